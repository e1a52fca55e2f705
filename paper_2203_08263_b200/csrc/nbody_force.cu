// sm_100a all-pairs softened gravity with a fused velocity-Verlet epilogue.
//
// Replaces the reference's O(N^2) kernel `_accel_cy.accel_soa`
// (/root/reference/pkg/src/nbodybench/kernels/_accel_cy.pyx:114-152, rows at
// :24-111) and, fused into the same launch, `step_soa` (:205-237) plus the host
// `_kick` (kernels/__init__.py:220-227).
//
// Design (DESIGN.md has the roofline arithmetic):
//  * CUDA cores only.  Per interaction the FP32 core issues 12 FP32 lane-ops
//    (3 FADD, 3 FFMA for d2, 3 FMUL for m*r^3, 3 FFMA accumulate) and one
//    MUFU.RSQ.  Two target bodies are paired in each thread and every FP32 op is
//    the packed FFMA2/FADD2/FMUL2 form with the source body broadcast (.F32
//    operand), so the FP32 pipe -- not the issue slot -- is the bound.  A third
//    of the weights take m*2^(-1.5 log2 d2) through MUFU.LG2/EX2 instead (10
//    FP32 ops + 2 MUFU), balancing the FMA and XU pipes (NB_F32_EXP2_MASK).
//  * Source bodies are staged through shared memory in tiles of TJ packed
//    (x,y,z,m) 4-vectors, double-buffered with one __syncthreads per tile; the
//    inner loop reads them with broadcast LDS.128 (no bank conflicts: every lane
//    reads the same address).
//  * FP32 accuracy: each tile's partial sum is FP32 (<= TJ terms); tile partials
//    are accumulated in FP64 (a single FP32 chain misses 1e-5 at
//    N >= 131072, tile partials + FP64 outer sums are at ~1e-7).
//  * FP64: MUFU.RSQ64H seed + one cubic correction that yields m*r^3 directly
//    (16 DP ops + 1 MUFU per interaction, no slow-path branch).
//  * Work distribution is stream-K over the (i-block x 16-body source chunk)
//    space: a persistent grid of SMs x occupancy CTAs, each owning an equal
//    contiguous range of units, so every SM gets the same work at every N.  An
//    i-block split between CTAs is combined through FP64 partial slots by
//    fixup_kernel (programmatic dependent launch, 32-thread CTAs) in fixed CTA
//    order -- bitwise reproducible run to run -- which then runs the epilogue.
//  * NB_TRACE builds record per-CTA %globaltimer timelines (tools/trace_launches.py).
//  * Small N: the whole multi-step loop runs in one cooperative launch --
//    small_simulate_kernel (N <= 3584 FP32 / 2560 FP64: source split inside the
//    CTA, no global partials; between its first and last step the positions are
//    exchanged as tagged coherent records, the staging poll standing in for the
//    grid barrier) or simulate_kernel (up to 8192: the stream-K decomposition
//    with a grid barrier per step, bitwise identical to per-step launches).
#include "nbody_common.cuh"
#include "nbody_kernels.h"

#include <atomic>
#include <cooperative_groups.h>
#include <cstdlib>
#include <mutex>
#include <random>

// Tuning knobs (overridable with -D for variant sweeps, tools/variants.py).
#ifndef NB_F32_K
#define NB_F32_K 6
#endif
#ifndef NB_F32_T
#define NB_F32_T 256
#endif
#ifndef NB_F32_TJ
#define NB_F32_TJ 256
#endif
#ifndef NB_F32_MINB
#define NB_F32_MINB 1
#endif
#ifndef NB_F32_UNROLL
#define NB_F32_UNROLL 16
#endif
#ifndef NB_F32_PACKED
#define NB_F32_PACKED 1
#endif
#ifndef NB_F32_MATH
#define NB_F32_MATH 0
#endif
#ifndef NB_F32_SUMS_IN_REGS
#define NB_F32_SUMS_IN_REGS 0
#endif
#ifndef NB_F32_STAGEWISE
#define NB_F32_STAGEWISE 0
#endif
#ifndef NB_F32_SPLIT_ACC
// Experiment (0 = off, shipped): G > 0 runs a full tile in groups of G sources --
// distances and weights of the group first, then, behind a scheduling boundary
// (NB_F32_SPLIT_KIND 1: a warp barrier, 2: a single-trip loop ptxas cannot see
// through), the group's accumulating FFMA2s in (source, pair, x/y/z) order, so the
// three accumulates of a weight are adjacent and w comes from the operand reuse
// cache (the accumulate is the one instruction with three distinct register
// pairs; DESIGN 3.1.1).
#define NB_F32_SPLIT_ACC 0
#endif
#ifndef NB_F32_SPLIT_KIND
#define NB_F32_SPLIT_KIND 1
#endif
#ifndef NB_F64_SPLIT_ACC
#define NB_F64_SPLIT_ACC 0  // the same experiment for the FP64 core's accumulating DFMAs (G sources per group)
#endif
#ifndef NB_F32_EXP2_MASK
// Which (target pair q, source phase p = jj mod NB_F32_EXP2_PHASES) weights go
// through MUFU.LG2/EX2 instead of MUFU.RSQ + FMUL2s: bit q + (K/2)*p.  0 = none.
// Default: pair 0 on even sources, pair 1 on odd -- 1/3 of the weights.
#define NB_F32_EXP2_MASK 17
#endif
#ifndef NB_F32_EXP2_PHASES
#define NB_F32_EXP2_PHASES 2
#endif
#ifndef NB_TMA_MIN_N
#define NB_TMA_MIN_N 65536  // FP32 launches with >= this many targets and sources use TMA staging
#endif
#ifndef NB_CHUNK
#define NB_CHUNK 16
#endif
#ifndef NB_PARTIAL_GROUPS
// 1: the last, partial i-block skips its dead target groups and the stream-K
// schedule is balanced by cost (Sched); 0 (shipped): every unit computes all
// groups.  Measured -10 % at C3-f32 and -9 % at C2: the two extra unrolled
// loops push the FP32 step kernel from 248 to 255 registers and cost the
// source loop its uniform-datapath addressing (profiles/variants_r02_infix_pg.txt).
#define NB_PARTIAL_GROUPS 0
#endif
#ifndef NB_INFIX_DEFAULT
// 1: split i-blocks are finished inside the step kernel (ready flags); 0
// (shipped): by fixup_kernel.  NB_FIXUP_KERNEL=0/1 in the environment overrides
// at run time.  Measured -3 % at C3-f32 and -8 % at C2: with the fixup code
// after the source loop ptxas schedules the loop worse (general-register
// addressing, +6 MOVs per 16 sources; profiles/variants_r02_infix_pg.txt).
#define NB_INFIX_DEFAULT 0
#endif
#ifndef NB_PAIR_ODD_EXP2
// pair_kernel: every NB_PAIR_ODD_EXP2-th source pair of the odd target takes
// the LG2/EX2 weight form (0: always the rsqrt form; 4 measured best of
// 2/4/8/16: C2 -1.1 %, profiles/r02/pair_odd_exp2.log)
#define NB_PAIR_ODD_EXP2 4
#endif
#ifndef NB_PAIR_ODD_FIRST
#define NB_PAIR_ODD_FIRST 0  // pair_kernel: the odd target's source pair before (1) or after (0) the pairs'
#endif
#ifndef NB_FIXUP_THREADS
// Threads per fixup CTA (one split body each).  Small CTAs spread the
// latency-bound fixup over every SM: C2 +1.7 % against 256-thread CTAs
// (profiles/variants_r01_fixup_threads.txt).
#define NB_FIXUP_THREADS 32
#endif
#ifndef NB_F64_K
#define NB_F64_K 6
#endif
#ifndef NB_F64_T
#define NB_F64_T 256
#endif
#ifndef NB_F64_TJ
#define NB_F64_TJ 256
#endif
#ifndef NB_F64_MINB
#define NB_F64_MINB 1
#endif
#ifndef NB_F64_UNROLL
#define NB_F64_UNROLL 8
#endif
#ifndef NB_F64_STAGEWISE
#define NB_F64_STAGEWISE 1
#endif
#if NB_F64_MIXED  // nbody_common.cuh
#define F64_CORR(e) fma((e), 1.5, nb::sq_term_f32((e), 1.875f))
#else
#define F64_CORR(e) ((e) * fma((e), 1.875, 1.5))
#endif


namespace nb {

// NB_CHECK builds (python -m paper_2203_08263_b200._build --check) trap on any
// out-of-range index: the stand-in for compute-sanitizer, closed on this pool.
#ifdef NB_CHECK
#define NB_DCHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define NB_DCHECK(cond) do { } while (0)
#endif

#if NB_TRACE
// Timeline instrumentation (trace builds only, tools/trace_launches.py): thread 0
// of every CTA records (tag, cta, smid, t_entry, t_wait, t_end) in %globaltimer ns.
__device__ unsigned long long* g_trace = nullptr;
__device__ unsigned long long g_trace_n = 0;
__device__ unsigned long long g_trace_cap = 0;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Record: (tag, id, smid, t[0..4]); unused timestamps are 0.
__device__ __forceinline__ void trace_put(int tag, unsigned long long id, const unsigned long long* t, int nt) {
  if (threadIdx.x == 0 && g_trace) {
    const unsigned long long k = atomicAdd(&g_trace_n, 1ull);
    if (k < g_trace_cap) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      unsigned long long* r = g_trace + 8 * k;
      r[0] = tag; r[1] = id; r[2] = smid;
      for (int q = 0; q < 5; ++q) r[3 + q] = q < nt ? t[q] : 0ull;
    }
  }
}
__device__ __forceinline__ void trace_rec(int tag, unsigned long long t_entry, unsigned long long t_wait) {
  __syncthreads();
  const unsigned long long t[3] = {t_entry, t_wait, gtimer()};
  trace_put(tag, blockIdx.x, t, 3);
}
#define NB_TRACE_ENTRY() const unsigned long long nb_t_entry = gtimer()
#define NB_TRACE_WAITED() const unsigned long long nb_t_wait = gtimer()
#define NB_TRACE_END(tag) trace_rec(tag, nb_t_entry, nb_t_wait)
#else
#define NB_TRACE_ENTRY() do { } while (0)
#define NB_TRACE_WAITED() do { } while (0)
#define NB_TRACE_END(tag) do { } while (0)
#endif

template <typename R>
__host__ __device__ __forceinline__ Sched sched_of(const StepArgs<R>& a) {
  return Sched::make(a.units, a.grid, a.n_tiles, a.n_iblocks, a.sched_kg, a.sched_lg);
}

// ---------------------------------------------------------------- packed FP32x2
// Two FP32 lanes in one 64-bit register (lo = first body, hi = second).  The
// packed ops are written in PTX on .b64 operands so ptxas keeps each pair in an
// aligned register pair for the whole loop (no per-use MOVs); a pair built from
// one scalar ({x, x}) folds into the FFMA2 .F32 broadcast operand.
typedef unsigned long long f2x;
__device__ __forceinline__ f2x pk(float lo, float hi) {
  f2x r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk(f2x v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
#if NB_F32_PACKED
__device__ __forceinline__ f2x add2(f2x a, f2x b) {
  f2x d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2x mul2(f2x a, f2x b) {
  f2x d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) {
  f2x d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
#else  // ladder rung without packed FP32x2: the same arithmetic as scalar FADD/FMUL/FFMA
__device__ __forceinline__ f2x add2(f2x a, f2x b) {
  float al, ah, bl, bh;
  upk(a, al, ah);
  upk(b, bl, bh);
  return pk(__fadd_rn(al, bl), __fadd_rn(ah, bh));
}
__device__ __forceinline__ f2x mul2(f2x a, f2x b) {
  float al, ah, bl, bh;
  upk(a, al, ah);
  upk(b, bl, bh);
  return pk(__fmul_rn(al, bl), __fmul_rn(ah, bh));
}
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) {
  float al, ah, bl, bh, cl, ch;
  upk(a, al, ah);
  upk(b, bl, bh);
  upk(c, cl, ch);
  return pk(__fmaf_rn(al, bl, cl), __fmaf_rn(ah, bh, ch));
}
#endif

// m * d2^(-3/2) for one lane in the reference's algebraic forms (ladder rungs):
// NB_F32_MATH 1 = recip (_accel_cy.pyx:86-94), 2 = pow (_accel_cy.pyx:42-49).
__device__ __forceinline__ float w_reference_form(float d2, float m) {
#if NB_F32_MATH == 2
  return __fdiv_rn(m, powf(d2, 1.5f));
#else
  return __fmul_rn(m, __frcp_rn(__fmul_rn(d2, __fsqrt_rn(d2))));
#endif
}

// ---------------------------------------------------------------- staged source tiles
// Source body jj of a shared-memory tile of TJ bodies.  FP32 tiles hold packed
// 16-byte (x,y,z,m) bodies.  FP64 tiles hold two planes of 16-byte halves,
// (x,y)[TJ] then (z,m)[TJ]: the staging stores of a warp are then contiguous
// 512-byte runs (4 wavefronts), where a packed 32-byte body per lane puts only
// four lanes' halves in each 128-byte wavefront (8 wavefronts, 2x; the r01
// ncu capture counted those as 5.6M shared-store bank conflicts per launch).
// The inner loop's reads are warp-wide broadcasts either way.
template <int TJ>
__device__ __forceinline__ F4 tile_get(const F4* tb, int jj) { return tb[jj]; }
template <int TJ>
__device__ __forceinline__ D4 tile_get(const D4* tb, int jj) {
  const double2* p = reinterpret_cast<const double2*>(tb);
  const double2 a = p[jj], b = p[TJ + jj];
  return D4{a.x, a.y, b.x, b.y};
}
template <int TJ>
__device__ __forceinline__ void tile_put(F4* tb, int idx, const F4& v) { tb[idx] = v; }
template <int TJ>
__device__ __forceinline__ void tile_put(D4* tb, int idx, const D4& v) {
  double2* p = reinterpret_cast<double2*>(tb);
  p[idx] = make_double2(v.x, v.y);
  p[TJ + idx] = make_double2(v.z, v.w);
}

// ---------------------------------------------------------------- FP32 core
// K target bodies per thread as K/2 packed pairs.  The FP64 segment sums live in
// shared memory (3*K doubles per thread, touched once per tile) so the inner
// loop keeps its registers for the pairs and their temporaries.
template <int K_, bool MASK, int UNROLL_, bool UNI>
struct CoreF32 {
  using R = float;
  static constexpr int K = K_;
  static constexpr int KP = K / 2;
  // Odd K (the cluster kernel's 7 targets per thread): the last target runs as
  // one scalar FP32 lane beside the KP packed pairs, always in the rsqrt form.
  static constexpr bool ODD = (K & 1) != 0;
  static constexpr unsigned XMASK = NB_F32_EXP2_MASK & ((1u << (NB_F32_EXP2_PHASES * KP)) - 1u);  // LG2/EX2 weights
  static constexpr bool NEEDS_LM = XMASK != 0 && !UNI;  // needs log2(m_j) per source
  const float* lmt;  // this tile's log2(m_j) (NEEDS_LM)
#if NB_F32_SUMS_IN_REGS
  static constexpr int SMEM_SUMS = 1;
  double rs[3 * K];  // FP64 segment sums in registers (1 CTA/SM leaves room)
#else
  static constexpr int SMEM_SUMS = 3 * K;  // doubles per thread
#endif
  f2x nx[KP], ny[KP], nz[KP];  // negated target positions, paired
  f2x tx[KP], ty[KP], tz[KP];  // FP32 partial sums of the current tile
  float onx, ony, onz;          // ODD: the scalar target's negated position
  float otx, oty, otz;          // ODD: its FP32 partial sums of the current tile
  // ODD, full tiles: the odd target runs packed over source PAIRS (2p, 2p+1)
  // read from a pair-interleaved copy of the tile, tbi[2p] = (x0,x1,y0,y1),
  // tbi[2p+1] = (z0,z1,m0,m1): the same packed FFMA2/FADD2/FMUL2 stream per
  // interaction as the target pairs (a scalar lane costs twice the issue slots).
  const float4* tbi;
  f2x pnx, pny, pnz;            // the odd target's negated position, broadcast
  f2x ptx, pty, ptz;            // its FP32 partials: even / odd sources of the tile
  int selfj[K];
  f2x e2;
  float e2s;
  double* ss;  // this thread's FP64 sums: ss[(d*K + k) * stride]
  int stride;

  __device__ __forceinline__ void init(float eps2, double* s, int st) {
    e2 = pk(eps2, eps2);
    e2s = eps2;
    ss = s;
    stride = st;
#if NB_F32_SPLIT_ACC
    one = st > 0 ? 1 : 0;  // st is a launch constant > 0; opaque to the compiler below
    asm volatile("" : "+r"(one));
#endif
  }
  __device__ __forceinline__ void set_pair(int q, const F4& p0, const F4& p1) {
    // +0 + (-x) is a real FADD2 (not an identity for x = +-0), so the pair is
    // materialised once in an aligned register pair instead of being re-paired
    // from the scalar load registers at every use.
    nx[q] = add2(0ull, pk(-p0.x, -p1.x));
    ny[q] = add2(0ull, pk(-p0.y, -p1.y));
    nz[q] = add2(0ull, pk(-p0.z, -p1.z));
  }
  __device__ __forceinline__ void set_single(const F4& p) {  // ODD: target K-1
    onx = -p.x;
    ony = -p.y;
    onz = -p.z;
    pnx = add2(0ull, pk(-p.x, -p.x));
    pny = add2(0ull, pk(-p.y, -p.y));
    pnz = add2(0ull, pk(-p.z, -p.z));
  }
  // The odd target against source pair (2p, 2p+1) of the interleaved tile
  // (a, b = tbi[2p], tbi[2p+1]).
  __device__ __forceinline__ void interact_odd2(const float4& a, const float4& b, int p) {
    const f2x xs = pk(a.x, a.y), ys = pk(a.z, a.w), zs = pk(b.x, b.y), ms = pk(b.z, b.w);
    const f2x dx = add2(xs, pnx), dy = add2(ys, pny), dz = add2(zs, pnz);
    f2x d2 = fma2(dx, dx, e2);
    d2 = fma2(dy, dy, d2);
    d2 = fma2(dz, dz, d2);
    float d2a, d2b;
    upk(d2, d2a, d2b);
    f2x w;
    if (NB_PAIR_ODD_EXP2 && NB_F32_MATH == 0 && (p % NB_PAIR_ODD_EXP2) == 0) {
      // this source pair's weights by 2^(-1.5 log2 d2 + log2 m) (LG2/EX2): XU work for FMA work
      const f2x l = pk(lg2_mufu(d2a), lg2_mufu(d2b));
      const f2x e = UNI ? mul2(l, pk(-1.5f, -1.5f))
                        : fma2(l, pk(-1.5f, -1.5f), *reinterpret_cast<const f2x*>(lmt + 2 * p));
      float ea, eb;
      upk(e, ea, eb);
      w = pk(ex2_mufu(ea), ex2_mufu(eb));
    } else {
      const f2x r = pk(rsqrt_mufu(d2a), rsqrt_mufu(d2b));
      const f2x r2 = mul2(r, r);
      w = UNI ? mul2(r2, r) : mul2(mul2(r, ms), r2);
    }
    if (MASK) {
      float wa, wb;
      upk(w, wa, wb);
      if (2 * p == selfj[K - 1]) wa = 0.f;
      if (2 * p + 1 == selfj[K - 1]) wb = 0.f;
      w = pk(wa, wb);
    }
    ptx = fma2(w, dx, ptx);
    pty = fma2(w, dy, pty);
    ptz = fma2(w, dz, ptz);
  }
#if NB_F32_SUMS_IN_REGS
  __device__ __forceinline__ double& acc_ref(int i) { return rs[i]; }
  __device__ __forceinline__ double acc_val(int i) const { return rs[i]; }
#else
  __device__ __forceinline__ double& acc_ref(int i) { return ss[i * stride]; }
  __device__ __forceinline__ double acc_val(int i) const { return ss[i * stride]; }
#endif
  __device__ __forceinline__ double sum(int d, int k) const { return acc_val(d * K + k); }
  __device__ __forceinline__ void set_sum(int d, int k, double v) { acc_ref(d * K + k) = v; }
  __device__ __forceinline__ void zero_sums() {
#pragma unroll
    for (int i = 0; i < 3 * K; ++i) acc_ref(i) = 0.0;
  }
  __device__ __forceinline__ void begin_tile() {
#pragma unroll
    for (int q = 0; q < KP; ++q) tx[q] = ty[q] = tz[q] = 0ull;
    if constexpr (ODD) {
      otx = oty = otz = 0.f;
      ptx = pty = ptz = 0ull;
    }
  }
  // One source body against the K targets.  Written stage-wise across the KP
  // pairs with w in the first operand slot of the accumulating FFMA2s: the
  // measured best source form (tools/loop_bench.cu, +1.2 % over a per-pair
  // order): consecutive instructions share the broadcast source operand, and the
  // accumulate -- the instruction with three distinct register pairs, which the
  // register file cannot feed at full rate -- gets the most reuse.
  __device__ __forceinline__ f2x weight(f2x d2, f2x mj, f2x lmj, int jj, int q) const {
    return weight_p(d2, mj, lmj, jj, q, jj % NB_F32_EXP2_PHASES);
  }
  // phase: the source's LG2/EX2 phase (jj mod NB_F32_EXP2_PHASES, a compile-time
  // value in the unrolled callers)
  __device__ __forceinline__ f2x weight_p(f2x d2, f2x mj, f2x lmj, int jj, int q, int phase) const {
    float d2a, d2b;
    upk(d2, d2a, d2b);
    f2x w;
#if NB_F32_MATH == 0
    if ((XMASK >> (q + KP * phase)) & 1u) {
      // m d2^(-3/2) = 2^(-1.5 log2 d2 + log2 m): one FFMA2 and four MUFU ops in
      // place of three FMUL2 + two MUFU.RSQ -- moves FP32-pipe work onto the XU
      // pipe, which the rsqrt form leaves ~40 % idle.
      const f2x l = pk(lg2_mufu(d2a), lg2_mufu(d2b));
      const f2x e = UNI ? mul2(l, pk(-1.5f, -1.5f)) : fma2(l, pk(-1.5f, -1.5f), lmj);
      float ea, eb;
      upk(e, ea, eb);
      w = pk(ex2_mufu(ea), ex2_mufu(eb));
    } else {
    const f2x r = pk(rsqrt_mufu(d2a), rsqrt_mufu(d2b));
    // r^2 by FMUL2.  (Taking it from MUFU.RCP for some pairs, to shift work to
    // the XU pipe, was measured slower: the XU pipe saturates first.)
    const f2x r2 = mul2(r, r);
    // UNI (all masses equal): m is applied once to the finished sum, saving
    // one FMUL2 of 12 per interaction pair.
    w = UNI ? mul2(r2, r) : mul2(mul2(r, mj), r2);
    }
#else
    float ma, mb;
    upk(mj, ma, mb);
    w = pk(w_reference_form(d2a, UNI ? 1.f : ma), w_reference_form(d2b, UNI ? 1.f : mb));
#endif
    if (MASK) {
      float wa, wb;
      upk(w, wa, wb);
      if (jj == selfj[2 * q]) wa = 0.f;
      if (jj == selfj[2 * q + 1]) wb = 0.f;
      w = pk(wa, wb);
    }
    return w;
  }

  static constexpr int KG = KP;  // target groups (pairs) per thread
  __device__ __forceinline__ void interact(const F4& pj, int jj) { interact_g<KP>(pj, jj); }
  // One source body against the first NG target pairs (the rest are dead rows
  // of a partial i-block: skipped).
  template <int NG, bool SCALAR_ODD = true>
  __device__ __forceinline__ void interact_g(const F4& pj, int jj) {
    const f2x xj = pk(pj.x, pj.x), yj = pk(pj.y, pj.y), zj = pk(pj.z, pj.z), mj = pk(pj.w, pj.w);
    float lm = 0.f;
    if (NEEDS_LM) lm = lmt[jj];
    const f2x lmj = pk(lm, lm);
#if !NB_F32_STAGEWISE
#pragma unroll
    for (int q = 0; q < NG; ++q) {  // ladder rung: per-pair order
      const f2x dx = add2(xj, nx[q]), dy = add2(yj, ny[q]), dz = add2(zj, nz[q]);
      f2x d2 = fma2(dx, dx, e2);
      d2 = fma2(dy, dy, d2);
      d2 = fma2(dz, dz, d2);
      const f2x w = weight(d2, mj, lmj, jj, q);
      tx[q] = fma2(dx, w, tx[q]);
      ty[q] = fma2(dy, w, ty[q]);
      tz[q] = fma2(dz, w, tz[q]);
    }
#else
    f2x dx[NG], dy[NG], dz[NG], d2[NG], w[NG];
#pragma unroll
    for (int q = 0; q < NG; ++q) dx[q] = add2(xj, nx[q]);
#pragma unroll
    for (int q = 0; q < NG; ++q) dy[q] = add2(yj, ny[q]);
#pragma unroll
    for (int q = 0; q < NG; ++q) dz[q] = add2(zj, nz[q]);
#pragma unroll
    for (int q = 0; q < NG; ++q) d2[q] = fma2(dx[q], dx[q], e2);
#pragma unroll
    for (int q = 0; q < NG; ++q) d2[q] = fma2(dy[q], dy[q], d2[q]);
#pragma unroll
    for (int q = 0; q < NG; ++q) d2[q] = fma2(dz[q], dz[q], d2[q]);
#pragma unroll
    for (int q = 0; q < NG; ++q) w[q] = weight(d2[q], mj, lmj, jj, q);
#pragma unroll
    for (int q = 0; q < NG; ++q) {
      tx[q] = fma2(w[q], dx[q], tx[q]);
      ty[q] = fma2(w[q], dy[q], ty[q]);
      tz[q] = fma2(w[q], dz[q], tz[q]);
    }
#endif
    if constexpr (ODD && SCALAR_ODD && NG == KP) {
      const float dxs = __fadd_rn(pj.x, onx), dys = __fadd_rn(pj.y, ony), dzs = __fadd_rn(pj.z, onz);
      float d2s = __fmaf_rn(dxs, dxs, e2s);
      d2s = __fmaf_rn(dys, dys, d2s);
      d2s = __fmaf_rn(dzs, dzs, d2s);
      const float r = rsqrt_mufu(d2s);
      const float r2 = __fmul_rn(r, r);
      float ws = UNI ? __fmul_rn(r2, r) : __fmul_rn(__fmul_rn(r, pj.w), r2);
      if (MASK && jj == selfj[K - 1]) ws = 0.f;
      otx = __fmaf_rn(ws, dxs, otx);
      oty = __fmaf_rn(ws, dys, oty);
      otz = __fmaf_rn(ws, dzs, otz);
    }
  }
  // A full tile of TJ source bodies against the first NG pairs, unrolled
  // UNROLL_ deep.  (Software-pipelining stage A of body j+1 against stage B of
  // body j was measured slower: profiles/variants_r01_sweep2.txt, "pipe".)
#if NB_F32_SPLIT_ACC
  int one;  // 1 at run time (NB_F32_SPLIT_KIND 2: trip count of the boundary loops)
  __device__ __forceinline__ void split_boundary() const {
#if NB_F32_SPLIT_KIND == 1
    __syncwarp();
#endif
  }
  template <int TJ, int NG>
  __device__ __forceinline__ void full_tile_split(const F4* tb) {
    constexpr int G = NB_F32_SPLIT_ACC;
    static_assert(TJ % G == 0 && G % NB_F32_EXP2_PHASES == 0, "group size");
#pragma unroll(UNROLL_ / G > 0 ? UNROLL_ / G : 1)
    for (int j0 = 0; j0 < TJ; j0 += G) {
      f2x dx[G][NG], dy[G][NG], dz[G][NG], w[G][NG];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const F4 pj = tb[j0 + g];
        const f2x xj = pk(pj.x, pj.x), yj = pk(pj.y, pj.y), zj = pk(pj.z, pj.z), mj = pk(pj.w, pj.w);
        float lm = 0.f;
        if (NEEDS_LM) lm = lmt[j0 + g];
        const f2x lmj = pk(lm, lm);
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          dx[g][q] = add2(xj, nx[q]);
          dy[g][q] = add2(yj, ny[q]);
          dz[g][q] = add2(zj, nz[q]);
          f2x d2 = fma2(dx[g][q], dx[g][q], e2);
          d2 = fma2(dy[g][q], dy[g][q], d2);
          d2 = fma2(dz[g][q], dz[g][q], d2);
          w[g][q] = weight_p(d2, mj, lmj, j0 + g, q, g % NB_F32_EXP2_PHASES);
        }
      }
      split_boundary();
#if NB_F32_SPLIT_KIND == 2
#pragma unroll 1
      for (int r = 0; r < one; ++r)
#endif
      {
#pragma unroll
        for (int g = 0; g < G; ++g) {
#pragma unroll
          for (int q = 0; q < NG; ++q) {
            tx[q] = fma2(w[g][q], dx[g][q], tx[q]);
            ty[q] = fma2(w[g][q], dy[g][q], ty[q]);
            tz[q] = fma2(w[g][q], dz[g][q], tz[q]);
          }
        }
      }
      split_boundary();
    }
  }
#endif
  template <int TJ, int NG = KP>
  __device__ __forceinline__ void full_tile(const F4* tb) {
#if NB_F32_SPLIT_ACC
    if constexpr (!ODD) {
      full_tile_split<TJ, NG>(tb);
      return;
    }
#endif
    if constexpr (ODD && NG == KP) {
      // every source read from the pair-interleaved tile (tbi): the pairs'
      // broadcast bodies and the odd target's packed source pair alike
#pragma unroll UNROLL_ / 2
      for (int p = 0; p < TJ / 2; ++p) {
        const float4 a = tbi[2 * p], b = tbi[2 * p + 1];
        if (NB_PAIR_ODD_FIRST) interact_odd2(a, b, p);
        interact_g<NG, false>(F4{a.x, a.z, b.x, b.z}, 2 * p);
        interact_g<NG, false>(F4{a.y, a.w, b.y, b.w}, 2 * p + 1);
        if (!NB_PAIR_ODD_FIRST) interact_odd2(a, b, p);
      }
    } else {
#pragma unroll UNROLL_
      for (int jj = 0; jj < TJ; ++jj) interact_g<NG>(tile_get<TJ>(tb, jj), jj);
    }
  }
  __device__ __forceinline__ void end_tile() {
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      float a, b;
      upk(tx[q], a, b);
      acc_ref(0 * K + 2 * q) += (double)a;
      acc_ref(0 * K + 2 * q + 1) += (double)b;
      upk(ty[q], a, b);
      acc_ref(1 * K + 2 * q) += (double)a;
      acc_ref(1 * K + 2 * q + 1) += (double)b;
      upk(tz[q], a, b);
      acc_ref(2 * K + 2 * q) += (double)a;
      acc_ref(2 * K + 2 * q + 1) += (double)b;
    }
    if constexpr (ODD) {
      float ea, eb;
      upk(ptx, ea, eb);
      acc_ref(0 * K + K - 1) += (double)otx + ((double)ea + (double)eb);
      upk(pty, ea, eb);
      acc_ref(1 * K + K - 1) += (double)oty + ((double)ea + (double)eb);
      upk(ptz, ea, eb);
      acc_ref(2 * K + K - 1) += (double)otz + ((double)ea + (double)eb);
    }
  }
};

// ---------------------------------------------------------------- FP64 core
template <int K_, bool MASK, int UNROLL_, bool UNI>
struct CoreF64 {
  using R = double;
  static constexpr int K = K_;
  static constexpr int SMEM_SUMS = 1;
  static constexpr bool NEEDS_LM = false;
  const float* lmt;
  double nx[K], ny[K], nz[K];
  double sx[K], sy[K], sz[K];
  int selfj[K];
  double e2;

  __device__ __forceinline__ void init(double eps2, double*, int) {
    e2 = eps2;
#if NB_F64_SPLIT_ACC
    one = 1;
#endif
  }
  __device__ __forceinline__ void set_pair(int q, const D4& p0, const D4& p1) {
    nx[2 * q] = -p0.x; ny[2 * q] = -p0.y; nz[2 * q] = -p0.z;
    nx[2 * q + 1] = -p1.x; ny[2 * q + 1] = -p1.y; nz[2 * q + 1] = -p1.z;
  }
  __device__ __forceinline__ double sum(int d, int k) const { return d == 0 ? sx[k] : (d == 1 ? sy[k] : sz[k]); }
  __device__ __forceinline__ void set_sum(int d, int k, double v) {
    if (d == 0) sx[k] = v; else if (d == 1) sy[k] = v; else sz[k] = v;
  }
  __device__ __forceinline__ void zero_sums() {
#pragma unroll
    for (int k = 0; k < K; ++k) sx[k] = sy[k] = sz[k] = 0.0;
  }
  __device__ __forceinline__ void begin_tile() {}
  __device__ __forceinline__ void end_tile() {}
  static constexpr int KG = K / 2;  // target groups (pairs) per thread, as in the FP32 core
#if NB_F64_SPLIT_ACC
  int one;  // 1 at run time, from a kernel parameter (trip count of the boundary loop)
#endif
  template <int TJ, int NG = KG>
  __device__ __forceinline__ void full_tile(const D4* tb) {
#if NB_F64_SPLIT_ACC
    constexpr int G = NB_F64_SPLIT_ACC, NK = 2 * NG;
    static_assert(TJ % G == 0, "group size");
#pragma unroll(UNROLL_ / G > 0 ? UNROLL_ / G : 1)
    for (int j0 = 0; j0 < TJ; j0 += G) {
      double dx[G][NK], dy[G][NK], dz[G][NK], w[G][NK];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const D4 pj = tile_get<TJ>(tb, j0 + g);
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          dx[g][k] = pj.x + nx[k];
          dy[g][k] = pj.y + ny[k];
          dz[g][k] = pj.z + nz[k];
          double d2 = fma(dx[g][k], dx[g][k], e2);
          d2 = fma(dy[g][k], dy[g][k], d2);
          d2 = fma(dz[g][k], dz[g][k], d2);
          const double y = rsqrt_seed(d2);
          const double t = y * y;
          const double e = fma(-d2, t, 1.0);
          const double my3 = UNI ? t * y : pj.w * (t * y);
          const double q = F64_CORR(e);
          w[g][k] = fma(my3, q, my3);
          if (MASK && j0 + g == selfj[k]) w[g][k] = 0.0;
        }
      }
#pragma unroll 1
      for (int r = 0; r < one; ++r) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
#pragma unroll
          for (int k = 0; k < NK; ++k) {
            sx[k] = fma(w[g][k], dx[g][k], sx[k]);
            sy[k] = fma(w[g][k], dy[g][k], sy[k]);
            sz[k] = fma(w[g][k], dz[g][k], sz[k]);
          }
        }
      }
    }
#else
#pragma unroll UNROLL_
    for (int jj = 0; jj < TJ; ++jj) interact_g<NG>(tile_get<TJ>(tb, jj), jj);
#endif
  }
  // A full tile staged row-wise (packed 32-byte bodies, as a bulk copy leaves
  // them: the cluster kernel's per-warp tiles).
  template <int TJ>
  __device__ __forceinline__ void full_tile_rows(const D4* tb) {
#pragma unroll UNROLL_
    for (int jj = 0; jj < TJ; ++jj) interact_g<KG>(tb[jj], jj);
  }
  __device__ __forceinline__ void interact(const D4& pj, int jj) { interact_g<KG>(pj, jj); }
  // One source body against the first 2*NG targets (the rest are dead rows of a
  // partial i-block: skipped).
  template <int NG>
  __device__ __forceinline__ void interact_g(const D4& pj, int jj) {
    constexpr int NK = 2 * NG;
#if NB_F64_STAGEWISE
    // Stage-wise across the K targets with w in the first slot of the
    // accumulating DFMAs (the FP32 kernel's measured best source form).
    double dx[NK], dy[NK], dz[NK], d2[NK], w[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) dx[k] = pj.x + nx[k];
#pragma unroll
    for (int k = 0; k < NK; ++k) dy[k] = pj.y + ny[k];
#pragma unroll
    for (int k = 0; k < NK; ++k) dz[k] = pj.z + nz[k];
#pragma unroll
    for (int k = 0; k < NK; ++k) d2[k] = fma(dx[k], dx[k], e2);
#pragma unroll
    for (int k = 0; k < NK; ++k) d2[k] = fma(dy[k], dy[k], d2[k]);
#pragma unroll
    for (int k = 0; k < NK; ++k) d2[k] = fma(dz[k], dz[k], d2[k]);
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const double y = rsqrt_seed(d2[k]);
      const double t = y * y;
      const double e = fma(-d2[k], t, 1.0);
      const double my3 = UNI ? t * y : pj.w * (t * y);
      const double q = F64_CORR(e);
      w[k] = fma(my3, q, my3);
      if (MASK && jj == selfj[k]) w[k] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      sx[k] = fma(w[k], dx[k], sx[k]);
      sy[k] = fma(w[k], dy[k], sy[k]);
      sz[k] = fma(w[k], dz[k], sz[k]);
    }
#else
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const double dx = pj.x + nx[k], dy = pj.y + ny[k], dz = pj.z + nz[k];
      double d2 = fma(dx, dx, e2);
      d2 = fma(dy, dy, d2);
      d2 = fma(dz, dz, d2);
      // y0 ~ d2^-1/2 to ~2^-22; with e = 1 - d2*y0^2 the exact
      // m*d2^-3/2 = m*y0^3*(1-e)^-3/2 = m*y0^3*(1 + 1.5e + 1.875e^2 + O(e^3)).
      const double y = rsqrt_seed(d2);
      const double t = y * y;
      const double e = fma(-d2, t, 1.0);
      const double my3 = UNI ? t * y : pj.w * (t * y);
      const double q = F64_CORR(e);
      double w = fma(my3, q, my3);
      if (MASK && jj == selfj[k]) w = 0.0;
      sx[k] = fma(dx, w, sx[k]);
      sy[k] = fma(dy, w, sy[k]);
      sz[k] = fma(dz, w, sz[k]);
    }
#endif
  }
};

// ---------------------------------------------------------------- epilogue
// a = real(G * sum) and the reference's update of one body from its previous
// velocity v, previous acceleration ap and current position p (all loaded by
// the caller): exactly the reference's rounding sequence (no contraction).  On
// return v and ap hold the new velocity and acceleration (also stored).
template <typename R>
__device__ __forceinline__ void integrate_body(const StepArgs<R>& a, int64_t il, double tx, double ty, double tz,
                                               V4<R>& v, V4<R>& ap, V4<R> p) {
  // Uniform-mass kernels left m_j out of every term: apply it once here.
  const double gm = a.uniform_mass ? a.g * (double)(a.mass0 ? *a.mass0 : a.pos[0].w) : a.g;
  const R ax = (R)(tx * gm), ay = (R)(ty * gm), az = (R)(tz * gm);
  V4<R> an;
  an.x = ax; an.y = ay; an.z = az; an.w = R(0);
  if (a.mode != NB_STEP_MODE_ACCEL) {
    if (a.mode != NB_STEP_MODE_FIRST) {  // trapezoidal kick, kernels/__init__.py:223-227
      v.x = add_rn(v.x, mul_rn(sub_rn(ax, ap.x), a.f));
      v.y = add_rn(v.y, mul_rn(sub_rn(ay, ap.y), a.f));
      v.z = add_rn(v.z, mul_rn(sub_rn(az, ap.z), a.f));
    }
    if (a.mode != NB_STEP_MODE_FINAL) {  // kick-drift, _accel_cy.pyx:218-226
      const int64_t ig = a.i_begin + il;
      const R dvx = mul_rn(ax, a.dt), dvy = mul_rn(ay, a.dt), dvz = mul_rn(az, a.dt);
      p.x = add_rn(p.x, mul_rn(add_rn(v.x, mul_rn(a.half, dvx)), a.dt));
      p.y = add_rn(p.y, mul_rn(add_rn(v.y, mul_rn(a.half, dvy)), a.dt));
      p.z = add_rn(p.z, mul_rn(add_rn(v.z, mul_rn(a.half, dvz)), a.dt));
      NB_DCHECK(ig >= 0 && ig < a.n_all && il >= 0 && il < a.n_i);
      if (a.pub) st4_pub(a.pos_next + ig, p);
      else st4(a.pos_next + ig, p);
      for (int q = 0; q < a.n_peers; ++q) st4(a.peers[q] + ig, p);  // NVLink peer stores
      v.x = add_rn(v.x, dvx);
      v.y = add_rn(v.y, dvy);
      v.z = add_rn(v.z, dvz);
    }
    st4(a.vel + il, v);
  }
  st4(a.acc + il, an);
  ap = an;
}

template <typename R>
__device__ __forceinline__ void finalize_body(const StepArgs<R>& a, int64_t il, double tx,
                                              double ty, double tz) {
  NB_DCHECK(il >= 0 && il < a.n_i);
  if (a.carry_mode == 2) {
    tx = a.carry[il] + tx;
    ty = a.carry[a.n_i + il] + ty;
    tz = a.carry[2 * a.n_i + il] + tz;
  }
  if (a.carry_mode == 1) {
    a.carry[il] = tx;
    a.carry[a.n_i + il] = ty;
    a.carry[2 * a.n_i + il] = tz;
    return;
  }
  V4<R> v{}, ap{}, p{};
  if (a.mode != NB_STEP_MODE_ACCEL) {
    v = a.vel[il];
    if (a.mode != NB_STEP_MODE_FIRST) ap = a.acc[il];
    if (a.mode != NB_STEP_MODE_FINAL) p = ld4_cg(a.pos + a.i_begin + il);
  }
  integrate_body<R>(a, il, tx, ty, tz, v, ap, p);
}

// ---------------------------------------------------------------- stream-K kernel
// Coherent (L2) or read-only-path load of a source/target body: inside the
// persistent multi-step kernel positions change between steps of ONE launch, so
// they must not come through the non-coherent read-only path.
template <bool COH, typename B>
__device__ __forceinline__ B ldp(const B* p) {
  if constexpr (COH) return ld4_cg(p);
  else return ld4(p);
}

// ---------------------------------------------------------------- TMA (bulk-copy) staging
// With TMA staging (large FP32 launches, use_tma) source tiles arrive in shared
// memory by cp.async.bulk (the 1-D TMA path) on an mbarrier per buffer instead
// of LDG -> registers -> STS.  Thread 0 issues each tile (two copies when the
// circular source range wraps); every thread waits on the buffer's phase.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Full source tile against the ng live target groups of this i-block: the
// group count selects one of KG unrolled loops (a uniform branch outside the
// source loop), so a partial last i-block skips its dead rows' arithmetic.
template <class Core, int TJ, int NG>
__device__ __forceinline__ void full_tile_live(Core& core, const V4<typename Core::R>* tb, int ng) {
  if constexpr (NG > 1) {
    if (ng < NG) {
      full_tile_live<Core, TJ, NG - 1>(core, tb, ng);
      return;
    }
  }
  core.template full_tile<TJ, NG>(tb);
}

// ---------------------------------------------------------------- split i-block fixup
// Ready flags of the partial slots (in-kernel fixup): a slot's flag holds the
// launch's unique tag once its partials are visible at GPU scope.
__device__ __forceinline__ void flag_publish(unsigned long long* f, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long flag_load(const unsigned long long* f) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
  return v;
}

// The partial slot CTA cc of split i-block b wrote its segment of b into: a
// CTA's first segment goes to slot 2c, its last (when it has two) to 2c+1; so
// the first contributor cf used 2cf+1 unless its units start exactly at b.
__device__ __forceinline__ int64_t slot_of(const Sched& S, int64_t NT, int64_t b, int64_t cf, int64_t cc) {
  return (cc == cf && S.start(cf) != b * NT) ? 2 * cf + 1 : 2 * cc;
}

// One target body of a split i-block: the FP64 partials of the contributing
// CTAs cf..cl summed in ascending CTA order (L2 loads: other CTAs of this or an
// earlier launch wrote them), then the epilogue.
template <typename R, int IB>
__device__ __forceinline__ void fixup_one(const StepArgs<R>& a, int64_t slot_cf, int64_t b, int64_t o, int64_t cf,
                                          int64_t cl) {
  const int64_t il = b * IB + o;
  double tx = 0.0, ty = 0.0, tz = 0.0;
  for (int64_t cc = cf; cc <= cl; ++cc) {
    const int64_t sl = cc == cf ? slot_cf : 2 * cc;
    NB_DCHECK(sl >= 0 && sl < 2 * a.grid && cc < a.grid && o < IB);
    const double* q = a.slots + sl * 3 * IB + o;
    tx += __ldcg(q);
    ty += __ldcg(q + IB);
    tz += __ldcg(q + 2 * IB);
  }
  finalize_body<R>(a, il, tx, ty, tz);
}

// In-kernel fixup plan of a CTA (INFIX, see step_body): for the split
// i-blocks it contributed to -- the ones holding its first and its last unit --
// the i-block, its first and last contributing CTAs and the first one's slot.
// Computed in the kernel's prologue next to the schedule's other divisions; the
// code after the source loop then has none (with the 64-bit divisions there,
// ptxas gave the source loop worse code: general instead of uniform-datapath
// addressing, -3 % at C3).
struct FixPlan {
  long long b[2], cf[2], cl[2], slot_cf[2];
};

__device__ __forceinline__ void make_fix_plan(FixPlan& p, const Sched& S, int64_t NT, int64_t c) {
  const int64_t u_begin = S.start(c), u_end = S.start(c + 1);
  const int64_t bb[2] = {u_begin / NT, (u_end - 1) / NT};
  for (int k = 0; k < 2; ++k) {
    const int64_t b = bb[k];
    const int64_t cf = S.cta_of(b * NT), cl = S.cta_of(b * NT + NT - 1);
    const bool use = u_end > u_begin && cf != cl && !(k == 1 && bb[1] == bb[0]);
    p.b[k] = use ? b : -1;
    p.cf[k] = cf;
    p.cl[k] = cl;
    p.slot_cf[k] = slot_of(S, NT, b, cf, cf);
  }
}

// Wait for every contributor's ready flag, then finish this CTA's 1/m share of
// the i-block's bodies (m contributors).
template <typename R, int T, int IB>
__device__ __forceinline__ void infix_fixup(const StepArgs<R>& a, const FixPlan& p) {
  const int tid = threadIdx.x;
  const int64_t c = blockIdx.x;
  for (int k = 0; k < 2; ++k) {
    const int64_t b = p.b[k];
    if (b < 0) continue;
    const int64_t cf = p.cf[k], cl = p.cl[k];
    if (tid < 32) {  // warp 0: one lane per contributor polls its slot's flag
      for (int64_t cc = cf + tid; cc <= cl; cc += 32) {
        const unsigned long long* f = a.flags + (cc == cf ? p.slot_cf[k] : 2 * cc);
        while (flag_load(f) != a.tag) __nanosleep(64);
      }
    }
    __syncthreads();
    const int64_t m = cl - cf + 1, r = c - cf;
    const int64_t rows = min((int64_t)IB, a.n_i - b * IB);
    // (r+1)*rows/m with rows <= IB and m <= grid: 32-bit division suffices
    const int64_t o0 = (int64_t)((uint32_t)(r * rows) / (uint32_t)m);
    const int64_t o1 = (int64_t)((uint32_t)((r + 1) * rows) / (uint32_t)m);
    for (int64_t o = o0 + tid; o < o1; o += T) fixup_one<R, IB>(a, p.slot_cf[k], b, o, cf, cl);
  }
}

// One force(+update) pass of the stream-K decomposition: the body of
// step_kernel, shared with the persistent multi-step simulate_kernel.
//
// INFIX: split i-blocks are finished inside this launch instead of by
// fixup_kernel.  Every contributor publishes its slot with a ready flag; after
// its last unit a CTA waits for the flags of the (at most two) split i-blocks it
// contributed to and finishes its own 1/m share of their bodies (m
// contributors), summing the slots in the same ascending CTA order as
// fixup_kernel -- bitwise the same result, one kernel boundary per step fewer,
// and the fixup spread over all contributors.  Waiting on other CTAs of the
// launch is safe because the persistent grid is at most one wave (every CTA is
// resident; launch_step falls back to fixup_kernel otherwise) and a CTA only
// ever waits on CTAs of its own launch.
template <class Core, int T, int TJ, int CH, bool COH, bool TMA, bool INFIX = false>
__device__ __forceinline__ void step_body(const StepArgs<typename Core::R>& a,
                                          V4<typename Core::R> (*tile)[TJ], double* s_sums,
                                          uint64_t* mbar) {
  using R = typename Core::R;
  using B = V4<R>;
  constexpr int K = Core::K;
  constexpr int IB = T * K;
  constexpr int PER = TJ / T;  // tile elements staged per thread
  static_assert(TJ % T == 0, "tile must be a multiple of the block");
  static_assert(TJ % CH == 0, "tile must be a multiple of the stream-K chunk");

  const int tid = threadIdx.x;
  const int64_t c = blockIdx.x;
  const Sched S = sched_of(a);
  const int64_t NT = a.n_tiles;  // source chunks of CH bodies per i-block
  const int64_t u_begin = S.start(c), u_end = S.start(c + 1);

  __shared__ long long s_plan[INFIX ? sizeof(FixPlan) / 8 : 1];
  if constexpr (INFIX) {
    if (tid == 0) make_fix_plan(*reinterpret_cast<FixPlan*>(s_plan), S, NT, c);
  }
  Core core;
  core.init(a.eps2, s_sums + tid, T);
#if NB_F32_SPLIT_ACC
  if constexpr (sizeof(R) == 4) core.one = (int)(a.n_all >> 40) + 1;  // 1, from a kernel parameter: opaque to ptxas
#endif
#if NB_F64_SPLIT_ACC
  if constexpr (sizeof(R) == 8) core.one = (int)(a.n_all >> 40) + 1;
#endif
  uint32_t phase_bits = 0u;  // mbarrier phase parity of tile buffer b in bit b (TMA staging)
  __shared__ float tile_lm[2][Core::NEEDS_LM ? TJ : 1];  // log2(m_j) of the staged tiles

  for (int64_t u = u_begin; u < u_end;) {
    const int64_t b = u / NT;
    const int64_t t0 = u - b * NT;
    const int64_t t1 = min(NT, t0 + (u_end - u));
    // this segment's source offsets [s0, s1) within the j range
    const int64_t s0 = t0 * CH, s1 = min(t1 * CH, a.j_count);
#if NB_PARTIAL_GROUPS
    // live target groups: all but in the last, partial i-block
    const int ng = b == a.n_iblocks - 1 ? a.sched_lg : Core::KG;
#endif
#if NB_TRACE
    unsigned long long tseg[5];
    tseg[0] = gtimer();
#endif

#pragma unroll
    for (int q = 0; q < K / 2; ++q) {
      const int64_t i0 = b * IB + (2 * q) * T + tid, i1 = i0 + T;
      core.set_pair(q, ldp<COH>(a.pos + a.i_begin + (i0 < a.n_i ? i0 : a.n_i - 1)),
                    ldp<COH>(a.pos + a.i_begin + (i1 < a.n_i ? i1 : a.n_i - 1)));
    }
    core.zero_sums();

    // (FP32 only: FP64 tiles are stored as planes, which a contiguous bulk copy
    // does not produce.)
    constexpr bool kTma = TMA && !COH && sizeof(R) == 4;
    // TMA staging: thread 0 arms the tile's mbarrier with its byte count and
    // issues the bulk copies; everyone waits on the barrier's current phase.
    auto issue_tile = [&](int buf, int64_t lo) {
      if (tid == 0) {
        const int64_t cnt = min((int64_t)TJ, s1 - lo);
        int64_t jg = a.j_begin + lo;
        if (jg >= a.n_all) jg -= a.n_all;
        const int64_t n1 = min(cnt, a.n_all - jg);
        mbar_expect_tx(mbar + buf, (uint32_t)(cnt * sizeof(B)));
        bulk_g2s(tile[buf], a.pos + jg, (uint32_t)(n1 * sizeof(B)), mbar + buf);
        if (cnt > n1) bulk_g2s(tile[buf] + n1, a.pos, (uint32_t)((cnt - n1) * sizeof(B)), mbar + buf);
      }
    };
    B stage[PER];
    auto load_tile = [&](int64_t lo) {
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        const int64_t off = lo + r * T + tid;
        if (off < s1) {
          int64_t jg = a.j_begin + off;
          if (jg >= a.n_all) jg -= a.n_all;
          NB_DCHECK(jg >= 0 && jg < a.n_all);
          stage[r] = ldp<COH>(a.pos + jg);
        } else {
          stage[r] = B{};
        }
      }
    };
    auto store_tile = [&](int buf) {
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        tile_put<TJ>(tile[buf], r * T + tid, stage[r]);
        if (Core::NEEDS_LM) tile_lm[buf][r * T + tid] = lg2_mufu((float)stage[r].w);
      }
    };

    if (kTma) {
      if (s0 < s1) issue_tile(0, s0);
    } else {
      load_tile(s0);
      store_tile(0);
      __syncthreads();
    }
#if NB_TRACE
    tseg[1] = gtimer();
#endif

    int buf = 0;
    for (int64_t lo = s0; lo < s1; lo += TJ) {
      const bool more = lo + TJ < s1;
      if (kTma) {
        if (more) issue_tile(buf ^ 1, lo + TJ);  // buf^1 was released by the last __syncthreads
        mbar_wait(mbar + buf, (phase_bits >> buf) & 1u);
        phase_bits ^= 1u << buf;
        if (Core::NEEDS_LM) {
#pragma unroll
          for (int r = 0; r < PER; ++r) tile_lm[buf][r * T + tid] = lg2_mufu((float)tile[buf][r * T + tid].w);
          __syncthreads();
        }
      } else if (more) {
        load_tile(lo + TJ);
      }
      const int count = (int)min((int64_t)TJ, s1 - lo);
      if (Core::MASK_SELF) {
        int64_t base = a.j_begin + lo;
        if (base >= a.n_all) base -= a.n_all;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          int64_t rel = a.i_begin + b * IB + k * T + tid - base;
          if (rel < 0) rel += a.n_all;
          core.selfj[k] = rel < count ? (int)rel : -1;
        }
      }
      core.begin_tile();
      core.lmt = tile_lm[buf];
      const B* tb = tile[buf];
      if (count == TJ) {
#if NB_PARTIAL_GROUPS
        full_tile_live<Core, TJ, Core::KG>(core, tb, ng);
#else
        core.template full_tile<TJ>(tb);
#endif
      } else {
        int jj = 0;
#pragma unroll 1
        for (; jj + 4 <= count; jj += 4) {
          core.interact(tile_get<TJ>(tb, jj), jj);
          core.interact(tile_get<TJ>(tb, jj + 1), jj + 1);
          core.interact(tile_get<TJ>(tb, jj + 2), jj + 2);
          core.interact(tile_get<TJ>(tb, jj + 3), jj + 3);
        }
#pragma unroll 1
        for (; jj < count; ++jj) core.interact(tile_get<TJ>(tb, jj), jj);
      }
      core.end_tile();
      if (!kTma && more) store_tile(buf ^ 1);
      buf ^= 1;
      __syncthreads();
    }

#if NB_TRACE
    tseg[2] = gtimer();
#endif
    if (t0 == 0 && t1 == NT) {
      // The whole source range of this i-block was ours: finish directly.
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int64_t il = b * IB + k * T + tid;
        if (il < a.n_i) finalize_body<R>(a, il, core.sum(0, k), core.sum(1, k), core.sum(2, k));
      }
    } else {
      // Split i-block: publish this segment's FP64 partial sums; fixup_kernel
      // (stream-ordered after this launch) combines the contributors of the
      // i-block in ascending CTA order -- deterministic -- and runs the epilogue.
      const int64_t slot = (u == u_begin) ? 2 * c : 2 * c + 1;
      NB_DCHECK(slot >= 0 && slot < 2 * a.grid && u >= u_begin && u < u_end);
      double* sp = a.slots + slot * 3 * IB;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        sp[k * T + tid] = core.sum(0, k);
        sp[IB + k * T + tid] = core.sum(1, k);
        sp[2 * IB + k * T + tid] = core.sum(2, k);
      }
      if (INFIX) {  // every thread's partials, then the slot's ready flag (release at GPU scope)
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          flag_publish(a.flags + slot, a.tag);
        }
      }
    }
#if NB_TRACE
    __syncthreads();
    tseg[3] = gtimer();
    tseg[4] = (unsigned long long)(s1 - s0);
    trace_put(4, (unsigned long long)c | ((unsigned long long)(u - u_begin) << 32), tseg, 5);
#endif
    u += t1 - t0;
  }
  if constexpr (INFIX) {
    __syncthreads();
    infix_fixup<R, T, IB>(a, *reinterpret_cast<const FixPlan*>(s_plan));
  }
  if (a.n_peers) __threadfence_system();  // peer stores visible before the rank barrier
}

template <class Core, int T, int TJ, int MINB, int CH, bool TMA, bool INFIX>
__global__ void __launch_bounds__(T, MINB) step_kernel(const StepArgs<typename Core::R> a) {
  __shared__ alignas(128) V4<typename Core::R> tile[2][TJ];
  __shared__ double s_sums[Core::SMEM_SUMS * T];
  __shared__ alignas(8) uint64_t mbar[2];
  if (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(mbar, 1);
      mbar_init(mbar + 1, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  // Programmatic dependent launch: wait for the previous kernel in the stream
  // (positions it wrote), then let the fixup kernel be scheduled as our CTAs drain.
  NB_TRACE_ENTRY();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  NB_TRACE_WAITED();
  asm volatile("griddepcontrol.launch_dependents;");
  step_body<Core, T, TJ, CH, false, TMA, INFIX>(a, tile, s_sums, mbar);
  NB_TRACE_END(1);
}

// ---------------------------------------------------------------- cluster split-source kernel
// Mid-size FP32 launches (C2: N = 16384; the per-rank size of C3 at 8 GPUs).
// Stream-K there splits every i-block between ~14 CTAs, and the FP64 partial
// slots, the fixup launch and the two kernel boundaries around it cost ~10 % of
// a 116 us step (profiles/trace_C2_r01.md).  This kernel splits the SOURCES
// instead, inside a 2-CTA cluster: cluster c owns i-block c of IBC = 32*K
// targets (every warp holds all of them, K per lane), and each of its 16 warps
// runs one 1/16 slice of the source range out of its own double-buffered tiles
// (cp.async.bulk on a per-warp mbarrier: no CTA-wide barrier in the loop).  The
// 16 slice sums of a target are then added in fixed slice order, the peer
// CTA's through distributed shared memory, and CTA r runs the epilogue of half
// r of the i-block: no partial slots, no fixup launch, bitwise reproducible.
// With 74 clusters on 148 SMs, K = 7 covers N <= 16576 (C2: 1.2 % dead lanes).
// The kernel is instantiated for K = NB_PAIR_KMIN .. NB_PAIR_K targets per lane
// (74 * 32 * K target slots: 4736, 7104, 9472, 11840, 14208, 16576) and a launch
// takes the smallest K that holds its targets (pair_clusters).
#ifndef NB_PAIR_K
#define NB_PAIR_K 7
#endif
#ifndef NB_PAIR_KMIN
#define NB_PAIR_KMIN 2
#endif
#ifndef NB_PAIR_TJ
#define NB_PAIR_TJ 256
#endif
#ifndef NB_PAIR_SHFL
// 1: the pair-interleaved tile copy by neighbour-lane shuffles (conflict-free
// shared loads/stores); 0: each lane copies a source pair (32-byte stride, 2
// wavefronts per access).
#define NB_PAIR_SHFL 1
#endif
#ifndef NB_PAIR_UNROLL
#define NB_PAIR_UNROLL 32
#endif
constexpr int PR_T = 256;             // threads per CTA
constexpr int PR_W = PR_T / 32;       // warps = source slices per CTA
constexpr int PR_CL = 2;              // CTAs per cluster
constexpr int PR_S = PR_W * PR_CL;    // source slices per i-block

template <int K, bool M, bool U> struct CorePair : CoreF32<K, M, NB_PAIR_UNROLL, U> {
  static constexpr bool MASK_SELF = M;
};

template <class Core, int TJ>
constexpr int64_t pair_smem_bytes() {
  return (int64_t)PR_W * 3 * TJ * sizeof(F4) + (Core::NEEDS_LM ? (int64_t)PR_W * 2 * TJ * 4 : 0) +
         (int64_t)3 * Core::K * PR_T * 8 + PR_W * 2 * 8;
}

template <class Core, int TJ>
__global__ void __cluster_dims__(PR_CL, 1, 1) __launch_bounds__(PR_T, 1) pair_kernel(const StepArgs<float> a) {
  using B = F4;
  constexpr int K = Core::K;
  constexpr int IBC = 32 * K;
  extern __shared__ __align__(128) unsigned char pr_smem[];
  B* tiles = reinterpret_cast<B*>(pr_smem);                                        // [warp][2][TJ]
  float4* ilv = reinterpret_cast<float4*>(tiles + PR_W * 2 * TJ);                  // [warp][TJ] interleaved
  float* lms = reinterpret_cast<float*>(ilv + PR_W * TJ);                          // [warp][2][TJ] (NEEDS_LM)
  double* sums = reinterpret_cast<double*>(lms + (Core::NEEDS_LM ? PR_W * 2 * TJ : 0));  // [3K][PR_T]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sums + 3 * K * PR_T);               // [warp][2]
  cooperative_groups::cluster_group cluster = cooperative_groups::this_cluster();
  const int tid = threadIdx.x, lane = tid & 31;
  // (A warp index through __shfl_sync -- provably uniform, tile addresses in
  // uniform registers as in the step kernel -- measured the same.)
  const int warp = tid >> 5;
  const int rank = (int)cluster.block_rank();
  const int64_t blk = blockIdx.x / PR_CL;
  // this warp's slice [s0, s1) of the j range (multiples of 16 bodies but the end)
  const int64_t per = (a.j_count + PR_S * 16 - 1) / (PR_S * 16) * 16;
  const int sl = rank * PR_W + warp;
  const int64_t s0 = min(a.j_count, sl * per), s1 = min(a.j_count, s0 + per);
  NB_DCHECK(blk * IBC < a.n_i && s0 >= 0 && s0 <= s1 && s1 <= a.j_count && rank < PR_CL);
  B* tw = tiles + warp * 2 * TJ;
  float* lw = lms + warp * 2 * TJ;
  uint64_t* bw = bars + warp * 2;
  if (lane == 0) {
    mbar_init(bw, 1);
    mbar_init(bw + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  NB_TRACE_ENTRY();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  NB_TRACE_WAITED();
  asm volatile("griddepcontrol.launch_dependents;");

  Core core;
  core.init(a.eps2, sums + tid, PR_T);
#pragma unroll
  for (int q = 0; q < K / 2; ++q) {
    const int64_t i0 = blk * IBC + (2 * q) * 32 + lane, i1 = i0 + 32;
    core.set_pair(q, ld4(a.pos + a.i_begin + (i0 < a.n_i ? i0 : a.n_i - 1)),
                  ld4(a.pos + a.i_begin + (i1 < a.n_i ? i1 : a.n_i - 1)));
  }
  if constexpr (Core::ODD) {
    const int64_t i0 = blk * IBC + (K - 1) * 32 + lane;
    core.set_single(ld4(a.pos + a.i_begin + (i0 < a.n_i ? i0 : a.n_i - 1)));
  }
  core.zero_sums();

  // lane 0 arms the buffer's mbarrier and issues the tile (two copies when the
  // circular source range wraps); the warp waits on the buffer's phase
  auto issue = [&](int buf, int64_t lo) {
    if (lane == 0) {
      const int64_t cnt = min((int64_t)TJ, s1 - lo);
      int64_t jg = a.j_begin + lo;
      if (jg >= a.n_all) jg -= a.n_all;
      const int64_t n1 = min(cnt, a.n_all - jg);
      NB_DCHECK(cnt > 0 && cnt <= TJ && jg >= 0 && jg + n1 <= a.n_all && cnt - n1 <= a.n_all);
      mbar_expect_tx(bw + buf, (uint32_t)(cnt * sizeof(B)));
      bulk_g2s(tw + buf * TJ, a.pos + jg, (uint32_t)(n1 * sizeof(B)), bw + buf);
      if (cnt > n1) bulk_g2s(tw + buf * TJ + n1, a.pos, (uint32_t)((cnt - n1) * sizeof(B)), bw + buf);
    }
  };
  uint32_t phase_bits = 0u;
  if (s0 < s1) issue(0, s0);
  int buf = 0;
  for (int64_t lo = s0; lo < s1; lo += TJ) {
    const bool more = lo + TJ < s1;
    mbar_wait(bw + buf, (phase_bits >> buf) & 1u);
    phase_bits ^= 1u << buf;
    if (more) issue(buf ^ 1, lo + TJ);  // buf^1 was released by the __syncwarp below
    const B* tb = tw + buf * TJ;
    const int count = (int)min((int64_t)TJ, s1 - lo);
    if (Core::ODD && count == TJ) {
      // Pair-interleaved copy of the tile for the odd target (and log2 m_j):
      // lane l reads body j = l + 32i (contiguous 16-byte loads), swaps halves
      // with its neighbour l^1 and writes ONE float4 -- (x0,x1,y0,y1) from the
      // even lane, (z0,z1,m0,m1) from the odd one -- so loads and stores are
      // conflict-free.
      float4* ti = ilv + warp * TJ;
#if NB_PAIR_SHFL
#pragma unroll
      for (int j = lane; j < TJ; j += 32) {
        const B b = tb[j];
        const float ox = __shfl_xor_sync(0xffffffffu, b.x, 1), oy = __shfl_xor_sync(0xffffffffu, b.y, 1);
        const float oz = __shfl_xor_sync(0xffffffffu, b.z, 1), ow = __shfl_xor_sync(0xffffffffu, b.w, 1);
        ti[j] = (lane & 1) ? make_float4(oz, b.z, ow, b.w) : make_float4(b.x, ox, b.y, oy);
        if (Core::NEEDS_LM) lw[buf * TJ + j] = lg2_mufu(b.w);
      }
#else
#pragma unroll 1
      for (int p = lane; p < TJ / 2; p += 32) {
        const B b0 = tb[2 * p], b1 = tb[2 * p + 1];
        ti[2 * p] = make_float4(b0.x, b1.x, b0.y, b1.y);
        ti[2 * p + 1] = make_float4(b0.z, b1.z, b0.w, b1.w);
        if (Core::NEEDS_LM) {
          lw[buf * TJ + 2 * p] = lg2_mufu(b0.w);
          lw[buf * TJ + 2 * p + 1] = lg2_mufu(b1.w);
        }
      }
#endif
      __syncwarp();
      core.tbi = ti;
    } else if (Core::NEEDS_LM) {
      for (int r = lane; r < count; r += 32) lw[buf * TJ + r] = lg2_mufu(tb[r].w);
      __syncwarp();
    }
    if (Core::MASK_SELF) {
      int64_t base = a.j_begin + lo;
      if (base >= a.n_all) base -= a.n_all;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        int64_t rel = a.i_begin + blk * IBC + k * 32 + lane - base;
        if (rel < 0) rel += a.n_all;
        core.selfj[k] = rel < count ? (int)rel : -1;
      }
    }
    core.begin_tile();
    core.lmt = lw + buf * TJ;
    if (count == TJ) {
      core.template full_tile<TJ>(tb);
    } else {
      int jj = 0;
#pragma unroll 1
      for (; jj + 4 <= count; jj += 4) {
        core.interact(tb[jj], jj);
        core.interact(tb[jj + 1], jj + 1);
        core.interact(tb[jj + 2], jj + 2);
        core.interact(tb[jj + 3], jj + 3);
      }
#pragma unroll 1
      for (; jj < count; ++jj) core.interact(tb[jj], jj);
    }
    core.end_tile();
    buf ^= 1;
    __syncwarp();
  }

  // every slice's FP64 sums (in shared memory) visible to both CTAs
  cluster.sync();
  // CTA r: targets [r*IBC/2, (r+1)*IBC/2) of the i-block; slice order 0..15
  const double* part[PR_CL];
#pragma unroll
  for (int r = 0; r < PR_CL; ++r) part[r] = cluster.map_shared_rank(sums, r);
  for (int t = rank * (IBC / 2) + tid; t < (rank + 1) * (IBC / 2); t += PR_T) {
    const int k = t >> 5, l = t & 31;
    NB_DCHECK(k < K && t < IBC);
    double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int s = 0; s < PR_S; ++s) {
      const double* q = part[s / PR_W] + (s % PR_W) * 32 + l;
#pragma unroll
      for (int d = 0; d < 3; ++d) acc[d] += q[(d * K + k) * PR_T];
    }
    const int64_t il = blk * IBC + t;
    if (il < a.n_i) finalize_body<float>(a, il, acc[0], acc[1], acc[2]);
  }
  cluster.sync();  // the peer's sums stay alive until both CTAs have read them
  NB_TRACE_END(5);
  if (a.n_peers) __threadfence_system();
}

// ---------------------------------------------------------------- FP64 cluster split-source kernel
// The same decomposition for FP64 (mid-size N in the reference's default
// precision: the persistent stream-K kernel spends ~a third of a step at
// N = 4096 on partial slots, the fixup pass and two grid barriers): 2-CTA
// clusters, K = 2 or 4 targets per lane (4736 / 9472 target slots on 148 SMs),
// 16 warp slices of the sources, each streamed by cp.async.bulk through the
// warp's own double-buffered tiles of packed 32-byte bodies (read row-wise:
// warp-wide broadcasts), slice sums reduced in fixed order through DSMEM.
#ifndef NB_PAIR64_UNROLL
#define NB_PAIR64_UNROLL 8
#endif
// minimum fill (1/1000) of the wave's target slots for K = 2 / K = 4 (1001 =
// never): the measured break-even against the persistent / stream-K paths
// (profiles/r02/pair_f64.txt) -- K = 2 wins from 2561 targets (above the small-N
// kernel's range: +29 ... +44 % per launch), K = 4 from ~8150 (+3 % at 8192, +17 %
// at 9472; below that its dead lanes cost more than the fixups it removes).
#ifndef NB_PAIR64_FILL2
#define NB_PAIR64_FILL2 540
#endif
#ifndef NB_PAIR64_FILL4
#define NB_PAIR64_FILL4 860
#endif
template <int K, bool M, bool U> struct CorePair64 : CoreF64<K, M, NB_PAIR64_UNROLL, U> {
  static constexpr bool MASK_SELF = M;
};
template <class Core, int TJ>
constexpr int64_t pair64_smem_bytes() {
  return (int64_t)PR_W * 2 * TJ * sizeof(D4) + (int64_t)3 * Core::K * PR_T * 8 + PR_W * 2 * 8;
}

template <class Core, int TJ>
__global__ void __cluster_dims__(PR_CL, 1, 1) __launch_bounds__(PR_T, 1) pair_kernel_f64(const StepArgs<double> a) {
  using B = D4;
  constexpr int K = Core::K;
  constexpr int IBC = 32 * K;
  extern __shared__ __align__(128) unsigned char pr_smem[];
  B* tiles = reinterpret_cast<B*>(pr_smem);                                 // [warp][2][TJ]
  double* sums = reinterpret_cast<double*>(tiles + PR_W * 2 * TJ);          // [3K][PR_T]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sums + 3 * K * PR_T);        // [warp][2]
  cooperative_groups::cluster_group cluster = cooperative_groups::this_cluster();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)cluster.block_rank();
  const int64_t blk = blockIdx.x / PR_CL;
  const int64_t per = (a.j_count + PR_S * 16 - 1) / (PR_S * 16) * 16;
  const int sl = rank * PR_W + warp;
  const int64_t s0 = min(a.j_count, sl * per), s1 = min(a.j_count, s0 + per);
  NB_DCHECK(blk * IBC < a.n_i && s0 >= 0 && s0 <= s1 && s1 <= a.j_count && rank < PR_CL);
  B* tw = tiles + warp * 2 * TJ;
  uint64_t* bw = bars + warp * 2;
  if (lane == 0) {
    mbar_init(bw, 1);
    mbar_init(bw + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  NB_TRACE_ENTRY();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  NB_TRACE_WAITED();
  asm volatile("griddepcontrol.launch_dependents;");

  Core core;
  core.init(a.eps2, nullptr, 0);
#pragma unroll
  for (int q = 0; q < K / 2; ++q) {
    const int64_t i0 = blk * IBC + (2 * q) * 32 + lane, i1 = i0 + 32;
    core.set_pair(q, ld4(a.pos + a.i_begin + (i0 < a.n_i ? i0 : a.n_i - 1)),
                  ld4(a.pos + a.i_begin + (i1 < a.n_i ? i1 : a.n_i - 1)));
  }
  core.zero_sums();

  auto issue = [&](int buf, int64_t lo) {
    if (lane == 0) {
      const int64_t cnt = min((int64_t)TJ, s1 - lo);
      int64_t jg = a.j_begin + lo;
      if (jg >= a.n_all) jg -= a.n_all;
      const int64_t n1 = min(cnt, a.n_all - jg);
      NB_DCHECK(cnt > 0 && cnt <= TJ && jg >= 0 && jg + n1 <= a.n_all && cnt - n1 <= a.n_all);
      mbar_expect_tx(bw + buf, (uint32_t)(cnt * sizeof(B)));
      bulk_g2s(tw + buf * TJ, a.pos + jg, (uint32_t)(n1 * sizeof(B)), bw + buf);
      if (cnt > n1) bulk_g2s(tw + buf * TJ + n1, a.pos, (uint32_t)((cnt - n1) * sizeof(B)), bw + buf);
    }
  };
  uint32_t phase_bits = 0u;
  if (s0 < s1) issue(0, s0);
  int buf = 0;
  for (int64_t lo = s0; lo < s1; lo += TJ) {
    const bool more = lo + TJ < s1;
    mbar_wait(bw + buf, (phase_bits >> buf) & 1u);
    phase_bits ^= 1u << buf;
    if (more) issue(buf ^ 1, lo + TJ);  // buf^1 was released by the __syncwarp below
    const B* tb = tw + buf * TJ;
    const int count = (int)min((int64_t)TJ, s1 - lo);
    if (Core::MASK_SELF) {
      int64_t base = a.j_begin + lo;
      if (base >= a.n_all) base -= a.n_all;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        int64_t rel = a.i_begin + blk * IBC + k * 32 + lane - base;
        if (rel < 0) rel += a.n_all;
        core.selfj[k] = rel < count ? (int)rel : -1;
      }
    }
    if (count == TJ) {
      core.template full_tile_rows<TJ>(tb);
    } else {
      int jj = 0;
#pragma unroll 1
      for (; jj + 4 <= count; jj += 4) {
        core.interact(tb[jj], jj);
        core.interact(tb[jj + 1], jj + 1);
        core.interact(tb[jj + 2], jj + 2);
        core.interact(tb[jj + 3], jj + 3);
      }
#pragma unroll 1
      for (; jj < count; ++jj) core.interact(tb[jj], jj);
    }
    buf ^= 1;
    __syncwarp();
  }
  // this thread's slice sums (registers) into the CTA's shared block
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int k = 0; k < K; ++k) sums[(d * K + k) * PR_T + tid] = core.sum(d, k);

  cluster.sync();  // every slice's sums visible to both CTAs
  const double* part[PR_CL];
#pragma unroll
  for (int r = 0; r < PR_CL; ++r) part[r] = cluster.map_shared_rank(sums, r);
  for (int t = rank * (IBC / 2) + tid; t < (rank + 1) * (IBC / 2); t += PR_T) {
    const int k = t >> 5, l = t & 31;
    NB_DCHECK(k < K && t < IBC);
    double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int s = 0; s < PR_S; ++s) {
      const double* q = part[s / PR_W] + (s % PR_W) * 32 + l;
#pragma unroll
      for (int d = 0; d < 3; ++d) acc[d] += q[(d * K + k) * PR_T];
    }
    const int64_t il = blk * IBC + t;
    if (il < a.n_i) finalize_body<double>(a, il, acc[0], acc[1], acc[2]);
  }
  cluster.sync();  // the peer's sums stay alive until both CTAs have read them
  NB_TRACE_END(5);
  if (a.n_peers) __threadfence_system();
}

// ---------------------------------------------------------------- split i-block fixup
template <typename R, int IB>
__device__ __forceinline__ void fixup_body(const StepArgs<R>& a, int64_t il);

// One thread per target body of a split i-block: sum the FP64 partials of the
// contributing CTAs cf..cl in ascending order (slot 2c holds a CTA's first
// segment, 2c+1 its last) and run the epilogue.  Bodies of i-blocks one CTA
// covered whole were finished by step_kernel and are skipped.
template <typename R, int IB>
__global__ void __launch_bounds__(NB_FIXUP_THREADS) fixup_kernel(const StepArgs<R> a) {
  NB_TRACE_ENTRY();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  NB_TRACE_WAITED();
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t il = blockIdx.x * (int64_t)NB_FIXUP_THREADS + threadIdx.x;
  fixup_body<R, IB>(a, il);
  NB_TRACE_END(2);
  if (a.n_peers) __threadfence_system();  // peer stores visible before the rank barrier
}

template <typename R, int IB>
__device__ __forceinline__ void fixup_body(const StepArgs<R>& a, int64_t il) {
  if (il >= a.n_i) return;
  const Sched S = sched_of(a);
  const int64_t NT = a.n_tiles;
  const int64_t b = il / IB, o = il - b * IB;
  const int64_t cf = S.cta_of(b * NT), cl = S.cta_of(b * NT + NT - 1);
  if (cf == cl) return;
  fixup_one<R, IB>(a, slot_of(S, NT, b, cf, cf), b, o, cf, cl);
}

// ---------------------------------------------------------------- persistent multi-step kernel
// Small N is launch-bound (C1: 1M interactions per evaluation, ~0.4 us of math
// against several us of launch + fixup per step); used for N <= 8192 (measured:
// C1 1.6x faster; at C2 the per-launch path with PDL is already as fast).  This kernel runs the whole
// velocity-Verlet loop of kernels.simulate in ONE cooperative launch: every step
// is the same stream-K pass as step_kernel, a grid-wide barrier, the split-i-block
// fixup spread over all CTAs, and a second barrier before the next step reads
// the new positions.  Same decomposition, same partial-sum order: results are
// bitwise identical to the per-launch path (tested).
template <class Core, int T, int TJ, int MINB, int CH>
__global__ void __launch_bounds__(T, MINB) simulate_kernel(StepArgs<typename Core::R> a,
                                                          V4<typename Core::R>* pos_a,
                                                          V4<typename Core::R>* pos_b, int64_t steps,
                                                          int any_split) {
  using R = typename Core::R;
  constexpr int IB = T * Core::K;
  __shared__ alignas(128) V4<R> tile[2][TJ];
  __shared__ double s_sums[Core::SMEM_SUMS * T];
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  for (int64_t s = 0; s <= steps; ++s) {
#if NB_TRACE
    unsigned long long tt[5];
    tt[0] = gtimer();
#endif
    a.mode = s == 0 ? NB_STEP_MODE_FIRST : (s < steps ? NB_STEP_MODE_KICK_DRIFT : NB_STEP_MODE_FINAL);
    a.pos = (s & 1) ? pos_b : pos_a;
    a.pos_next = (s & 1) ? pos_a : pos_b;
    step_body<Core, T, TJ, CH, true, false>(a, tile, s_sums, nullptr);
#if NB_TRACE
    __syncthreads();
    tt[1] = gtimer();
    tt[2] = tt[3] = tt[1];
#endif
    if (any_split) {
      grid.sync();  // every partial slot of this step is written
#if NB_TRACE
      tt[2] = gtimer();
#endif
      for (int64_t il = blockIdx.x * (int64_t)T + threadIdx.x; il < a.n_i; il += (int64_t)gridDim.x * T)
        fixup_body<R, IB>(a, il);
#if NB_TRACE
      __syncthreads();
      tt[3] = gtimer();
#endif
    }
    grid.sync();  // all new positions/velocities visible; nobody still reads the old buffer
#if NB_TRACE
    tt[4] = gtimer();
    trace_put(3, (unsigned long long)blockIdx.x | ((unsigned long long)s << 32), tt, 5);
#endif
  }
}

// ---------------------------------------------------------------- small-N cooperative simulate
// For a few thousand bodies (C1: N = 1024) the stream-K pass spreads one or two
// i-blocks over up to 148 CTAs, and every step then writes and re-reads ~2 MB
// of FP64 partial slots (C1: ~5 us each way, profiles/trace_C1_r01.md).  This
// kernel keeps the source split INSIDE the CTA instead: a CTA owns 2*PPW
// targets (PPW pairs; PPW = 8 or 4), each of its 8 warps holds all of them on
// PPW lanes x G = 32/PPW lane groups, so the CTA runs S = 8*G source splits;
// each thread runs one target pair over its split, and the S partial sums are
// combined by a shuffle butterfly over the lane groups and a fixed-order pass
// over the 8 warps -- no global partials, no fixup, bitwise reproducible.  Each
// step stages all N bodies into shared memory split-major (split s holds
// j = s, s+S, ... contiguously, padded so a warp's lane groups read disjoint
// banks), then one grid barrier per step (per-CTA release/acquire flags in its
// place measured slower beyond ~32 CTAs: every CTA polls every flag).  Same Core arithmetic as the main kernel (the FP32 split is
// <= N/S terms in FP32 before the FP64 sums).
#ifndef NB_SMALL_T
#define NB_SMALL_T 256
#endif
// Bytes of skew per source split of the small-N kernel's shared layout (FP64).
template <typename R>
__host__ __device__ constexpr int64_t small_split_skew() { return sizeof(R) == 8 ? 16 : 0; }
// A staged body at a 16-byte-aligned shared address (FP64 bodies as two halves).
__device__ __forceinline__ void st_body(unsigned char* p, const F4& b) { *reinterpret_cast<F4*>(p) = b; }
__device__ __forceinline__ void st_body(unsigned char* p, const D4& b) {
  double2* q = reinterpret_cast<double2*>(p);
  q[0] = make_double2(b.x, b.y);
  q[1] = make_double2(b.z, b.w);
}
// Position only: the staged body's mass (fourth word) stays as step 0 left it.
__device__ __forceinline__ void st_body_xyz(unsigned char* p, const F4& b) {
  *reinterpret_cast<float2*>(p) = make_float2(b.x, b.y);
  reinterpret_cast<float*>(p)[2] = b.z;
}
__device__ __forceinline__ void st_body_xyz(unsigned char* p, const D4& b) {
  double2* q = reinterpret_cast<double2*>(p);
  q[0] = make_double2(b.x, b.y);
  reinterpret_cast<double*>(p)[2] = b.z;
}
template <typename B> __device__ __forceinline__ B ld_body(const unsigned char* p);
template <> __device__ __forceinline__ F4 ld_body<F4>(const unsigned char* p) {
  return *reinterpret_cast<const F4*>(p);
}
template <> __device__ __forceinline__ D4 ld_body<D4>(const unsigned char* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = q[0], b = q[1];
  return D4{a.x, a.y, b.x, b.y};
}
constexpr int SN_T = NB_SMALL_T;  // threads per CTA (8 warps)

// Bodies per split in shared memory: ceil(N/S) rounded up to 1 mod 8, so the
// splits of one warp's lane groups start 4 banks apart (FP32 bodies; FP64 ones
// take two 16-byte halves, 8 banks apart).
__host__ __device__ inline int64_t small_split_stride(int64_t n, int splits) {
  const int64_t L = (n + splits - 1) / splits;
  return L + (((1 - L) % 8) + 8) % 8;
}

template <bool M, bool U> struct SmallF32 : CoreF32<2, M, 4, U> { static constexpr bool MASK_SELF = M; };
template <bool M, bool U> struct SmallF64 : CoreF64<2, M, 4, U> { static constexpr bool MASK_SELF = M; };

// cols (optional): simulate()'s device column block (x, y, z, m at 0, n, 2n, 3n;
// vx, vy, vz at 4n, 5n, 6n).  Step 0 then reads the initial state straight from
// the columns and the last step writes the final positions and velocities back
// into them, so the host API needs no pack/unpack launches around the simulate.
template <class Core, int PPW>
__global__ void __launch_bounds__(SN_T) small_simulate_kernel(StepArgs<typename Core::R> a,
                                                              V4<typename Core::R>* pos_a,
                                                              V4<typename Core::R>* pos_b, int64_t steps,
                                                              int64_t L, typename Core::R* cols,
                                                              typename Core::R* cols_out) {
  using R = typename Core::R;
  using B = V4<R>;
  constexpr int G = 32 / PPW;        // lane groups per warp
  constexpr int S = (SN_T / 32) * G; // source splits per CTA
  constexpr int TB = 2 * PPW;        // target bodies per CTA
  extern __shared__ __align__(128) unsigned char sn_smem[];
  // S splits of L bodies, split-major (split s holds j = s, s+S, ...), each
  // split SB bytes: FP64 splits carry a 16-byte skew so the 8 lane groups of a
  // warp, which read 8 consecutive splits, and the staging stores of 8
  // consecutive lanes fall in distinct 4-bank groups (conflict-free; 32-byte
  // bodies at an L*32-byte split stride would pair up 2-way).
  constexpr int64_t SKEW = small_split_skew<R>();
  const int64_t SB = L * (int64_t)sizeof(B) + SKEW;
  float* slm = reinterpret_cast<float*>(sn_smem + S * SB);            // log2(m_j) (FP32), slot() layout
  double* ssum = reinterpret_cast<double*>(slm + (Core::NEEDS_LM ? S * L : 0));
  double* red = ssum + Core::SMEM_SUMS * SN_T;                        // [8 warps][TB targets][3]
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pr = lane % PPW, sub = lane / PPW;
  const int s = warp * G + sub;  // this thread's source split: j = s + S*jj
  const int64_t n = a.n_all;
  const int64_t i0 = blockIdx.x * (int64_t)TB + 2 * pr;
  const int cnt = s < n ? (int)((n - s + S - 1) / S) : 0;
  auto body_at = [&](int64_t j) { return sn_smem + (j % S) * SB + (j / S) * (int64_t)sizeof(B); };
  auto slot = [&](int64_t j) {
    const int64_t q = (j % S) * L + j / S;
    NB_DCHECK(j >= 0 && j < n && q >= 0 && q < S * L);
    return q;
  };

  Core core;
  core.init(a.eps2, ssum + tid, SN_T);
  core.lmt = slm + s * L;
  if (Core::MASK_SELF) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int64_t i = i0 + k;
      core.selfj[k] = (i < n && (int)(i % S) == s) ? (int)(i / S) : -1;
    }
  }
  // The epilogue thread of body il keeps its velocity and previous acceleration
  // in registers for the whole launch (it is the only one that updates them).
  const int64_t il = blockIdx.x * (int64_t)TB + tid;
  // steps < 0: one force evaluation only (mode ACCEL: acc written, nothing moves)
  B vel{}, acc_prev{};
  if (tid < TB && il < n && steps >= 0) {
    if (cols) {
      vel.x = cols[4 * n + il];
      vel.y = cols[5 * n + il];
      vel.z = cols[6 * n + il];
    } else {
      vel = a.vel[il];
    }
  }
  const int64_t last = steps < 0 ? 0 : steps;
  for (int64_t st = 0; st <= last; ++st) {
    a.mode = steps < 0 ? NB_STEP_MODE_ACCEL
                       : (st == 0 ? NB_STEP_MODE_FIRST : (st < steps ? NB_STEP_MODE_KICK_DRIFT : NB_STEP_MODE_FINAL));
    a.pos = (st & 1) ? pos_b : pos_a;
    a.pos_next = (st & 1) ? pos_a : pos_b;
    // step 0 of a column-block run: the packed buffer holds no state yet
    a.mass0 = (cols && st == 0) ? cols + 3 * n : nullptr;
    // Tagged exchange (a.tag != 0): the drift of step st stores every body as one
    // coherent record whose fourth word is the tag of step st+1 instead of the
    // mass, and step st+1 stages by polling each record until it carries that
    // tag -- the staging read IS the grid-wide wait (one L2 round trip in place
    // of barrier + read).  Masses and log2 m stay in shared memory from step 0.
    // Buffer reuse is safe: a CTA overwrites buffer b (tag st+2) only after it
    // saw every record of the other buffer tagged st+1, and a CTA publishes
    // those only after it finished staging buffer b.  The first and the last
    // drift (st = 0, steps-1) store real masses and are followed by the grid
    // barrier: a polled buffer then never holds anything but masses (sign bit
    // clear) or this launch's own earlier tags -- no stale data of another launch
    // or process can match -- and the launch leaves the current buffer as every
    // other kernel expects it.
    const bool tagged_out = a.tag != 0 && st >= 1 && st < steps - 1;     // this step's drift publishes tags
    const bool tagged_in = a.tag != 0 && st >= 2 && st <= steps - 1;     // this step's staging polls them
    a.pub = tagged_out ? 1 : 0;
#if NB_TRACE
    unsigned long long tt[5];
    tt[0] = gtimer();
#endif
    if (tagged_in) {
      const R want = tag_word(R(0), a.tag + (unsigned long long)st);
      if (a.uniform_mass) a.mass0 = reinterpret_cast<const R*>(body_at(0)) + 3;  // a.pos[0].w is a tag
      for (int64_t j0 = tid; j0 < n; j0 += 4 * SN_T) {
        B b[4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (j0 + r * SN_T < n) b[r] = ld4_pub(a.pos + j0 + r * SN_T);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t j = j0 + r * SN_T;
          if (j < n) {
            while (!same_word(b[r].w, want)) b[r] = ld4_pub(a.pos + j);
            st_body_xyz(body_at(j), b[r]);
          }
        }
      }
    } else {
      for (int64_t j = tid; j < n; j += SN_T) {  // positions moved last step: coherent loads
        B b;
        if (cols && st == 0) {
          b.x = cols[j];
          b.y = cols[n + j];
          b.z = cols[2 * n + j];
          b.w = cols[3 * n + j];
        } else {
          b = ld4_cg(a.pos + j);
        }
        st_body(body_at(j), b);
        if (Core::NEEDS_LM) slm[slot(j)] = lg2_mufu((float)b.w);
      }
    }
    __syncthreads();
#if NB_TRACE
    tt[1] = gtimer();
#endif
    const int64_t ia = i0 < n ? i0 : n - 1, ib = i0 + 1 < n ? i0 + 1 : n - 1;
    core.set_pair(0, ld_body<B>(body_at(ia)), ld_body<B>(body_at(ib)));
    core.zero_sums();
    core.begin_tile();
    const unsigned char* tb = sn_smem + s * SB;
    NB_DCHECK(cnt >= 0 && cnt <= L);
    int jj = 0;
#pragma unroll 1
    for (; jj + 4 <= cnt; jj += 4) {
      core.interact(ld_body<B>(tb + jj * sizeof(B)), jj);
      core.interact(ld_body<B>(tb + (jj + 1) * sizeof(B)), jj + 1);
      core.interact(ld_body<B>(tb + (jj + 2) * sizeof(B)), jj + 2);
      core.interact(ld_body<B>(tb + (jj + 3) * sizeof(B)), jj + 3);
    }
#pragma unroll 1
    for (; jj < cnt; ++jj) core.interact(ld_body<B>(tb + jj * sizeof(B)), jj);
    core.end_tile();
#if NB_TRACE
    tt[2] = gtimer();
#endif
    // S splits -> 1: butterfly over the lane groups (a + b == b + a, so every
    // lane ends with the same bits), then the 8 warps in ascending order.
    double v[6];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      v[2 * d] = core.sum(d, 0);
      v[2 * d + 1] = core.sum(d, 1);
    }
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
      for (int x = PPW; x < 32; x *= 2) v[q] += __shfl_xor_sync(0xffffffffu, v[q], x);
    if (sub == 0) {
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        NB_DCHECK((warp * TB + 2 * pr + 1) * 3 + d < (SN_T / 32) * TB * 3);
        red[(warp * TB + 2 * pr) * 3 + d] = v[2 * d];
        red[(warp * TB + 2 * pr + 1) * 3 + d] = v[2 * d + 1];
      }
    }
    __syncthreads();
    if (tid < TB && il < n) {
      double t[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int w = 0; w < SN_T / 32; ++w)
#pragma unroll
        for (int d = 0; d < 3; ++d) t[d] += red[(w * TB + tid) * 3 + d];
      B pcur = ld_body<B>(body_at(il));
      if (tagged_out) pcur.w = tag_word(R(0), a.tag + (unsigned long long)st + 1);
      integrate_body<R>(a, il, t[0], t[1], t[2], vel, acc_prev, pcur);
      if (cols && st == last) {  // final state back into the columns (positions did not move in this step)
        const B pf = ld_body<B>(body_at(il));
        R* co = cols_out ? cols_out : cols;
        co[il] = pf.x;
        co[n + il] = pf.y;
        co[2 * n + il] = pf.z;
        co[4 * n + il] = vel.x;
        co[5 * n + il] = vel.y;
        co[6 * n + il] = vel.z;
      }
    }
#if NB_TRACE
    __syncthreads();
    tt[3] = gtimer();
#endif
    // new positions visible; nobody still reads the old buffer, sp or red
    if (st < steps) {
      if (tagged_out) __syncthreads();  // (the next staging's tag poll is the grid-wide wait)
      else grid.sync();
    }
#if NB_TRACE
    tt[4] = gtimer();
    trace_put(6, (unsigned long long)blockIdx.x | ((unsigned long long)st << 32), tt, 5);
#endif
  }
}

template <typename R>
int64_t small_smem_bytes(int64_t n, int ppw, bool needs_lm) {
  const int splits = (SN_T / 32) * (32 / ppw);
  const int64_t L = small_split_stride(n, splits);
  const int64_t sums = sizeof(R) == 4 ? 6 : 1;  // Core::SMEM_SUMS doubles per thread
  return splits * (L * (int64_t)sizeof(V4<R>) + small_split_skew<R>()) + (needs_lm ? splits * L * 4 : 0) +
         sums * SN_T * 8 +
         (SN_T / 32) * 2 * ppw * 3 * 8;
}

// ---------------------------------------------------------------- configurations
// Both precisions: 256 threads x 6 target bodies = 1536-body i-blocks, 256-body
// source tiles (FP32: 3 packed FFMA2 pairs per thread).
template <bool M, bool U> struct CoreF32M : CoreF32<NB_F32_K, M, NB_F32_UNROLL, U> {
  static constexpr bool MASK_SELF = M;
};
template <bool M, bool U> struct CoreF64M : CoreF64<NB_F64_K, M, NB_F64_UNROLL, U> {
  static constexpr bool MASK_SELF = M;
};

template <typename R> struct Cfg;
template <> struct Cfg<float> {
  static constexpr int T = NB_F32_T, TJ = NB_F32_TJ, MINB = NB_F32_MINB;
  template <bool M, bool U> using Core = CoreF32M<M, U>;
};
template <> struct Cfg<double> {
  static constexpr int T = NB_F64_T, TJ = NB_F64_TJ, MINB = NB_F64_MINB;
  template <bool M, bool U> using Core = CoreF64M<M, U>;
};

template <typename R, bool M, bool U, bool TMA, bool INFIX>
static const void* kernel_ptr() {
  using C = Cfg<R>;
  return reinterpret_cast<const void*>(
      &step_kernel<typename C::template Core<M, U>, C::T, C::TJ, C::MINB, NB_CHUNK, TMA, INFIX>);
}

template <typename R, bool INFIX>
static const void* step_fn_i(bool mask, bool uni, bool tma) {
  if constexpr (sizeof(R) == 4) {  // (TMA staging is FP32-only)
    if (tma) {
      if (mask) return uni ? kernel_ptr<R, true, true, true, INFIX>() : kernel_ptr<R, true, false, true, INFIX>();
      return uni ? kernel_ptr<R, false, true, true, INFIX>() : kernel_ptr<R, false, false, true, INFIX>();
    }
  }
  if (mask) return uni ? kernel_ptr<R, true, true, false, INFIX>() : kernel_ptr<R, true, false, false, INFIX>();
  return uni ? kernel_ptr<R, false, true, false, INFIX>() : kernel_ptr<R, false, false, false, INFIX>();
}

// The step kernel for (exclude-self, uniform-mass, TMA staging, in-kernel fixup).
template <typename R>
static const void* step_fn(bool mask, bool uni, bool tma, bool infix) {
  return infix ? step_fn_i<R, true>(mask, uni, tma) : step_fn_i<R, false>(mask, uni, tma);
}

// TMA (bulk-copy) staging of the source tiles, FP32, launches with >=
// NB_TMA_MIN_N targets and sources, enabled by NB_TMA=1.  Measured within noise
// of the register path at N=131072 (71.6 % vs 71.8 %) and 3 % slower at
// N=16384 (profiles/variants_r01_tma.txt), so it is off by default.
template <typename R>
static bool use_tma(int64_t n_i, int64_t j_count) {
  if (sizeof(R) != 4) return false;
  static int enabled = -1;
  if (enabled < 0) {
    const char* env = getenv("NB_TMA");
    enabled = env ? atoi(env) != 0 : 0;
  }
  return enabled && n_i >= NB_TMA_MIN_N && j_count >= NB_TMA_MIN_N;
}

template <typename R>
StepGeometry step_geometry(int64_t n_i, int64_t j_count) {
  using C = Cfg<R>;
  StepGeometry g{};
  g.threads = C::T;
  g.i_block = C::T * C::template Core<false, false>::K;
  g.tile = C::TJ;
  g.n_iblocks = (n_i + g.i_block - 1) / g.i_block;
  g.n_tiles = j_count > 0 ? (j_count + NB_CHUNK - 1) / NB_CHUNK : 1;  // stream-K chunks
  g.units = g.n_iblocks * g.n_tiles;
  return g;
}

// Persistent grid of a step kernel: SMs x its resident CTAs per SM (cached per
// device and kernel).  NB_GRID_OVERRIDE=<ctas> replaces it (experiments).
static int grid_for(const void* fn, int threads) {
  struct Entry { int dev; const void* fn; int grid; };
  static Entry cache[64];
  static int used = 0;
  static std::mutex mu;  // host threads may launch concurrently on different streams
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  for (int k = 0; k < used; ++k)
    if (cache[k].dev == dev && cache[k].fn == fn) return cache[k].grid;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0);
  int grid = sms * (per_sm < 1 ? 1 : per_sm);
  if (const char* env = getenv("NB_GRID_OVERRIDE")) {
    const int v = atoi(env);
    if (v > 0) grid = v;
  }
  if (used < 64) cache[used++] = Entry{dev, fn, grid};
  return grid;
}

// Largest persistent grid over every step-kernel variant of this precision
// (sizes the stream-K slot workspace).
template <typename R>
int max_grid() {
  // Cached per device (every step launch sizes its workspace with it: at small
  // N the host side of a launch is on simulate()'s critical path).
  static std::atomic<int> cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64) {
    const int c = cache[dev].load(std::memory_order_relaxed);
    if (c > 0) return c;
  }
  int best = 1;
  for (int m = 0; m < 16; ++m) {
    const int g = grid_for(step_fn<R>(m & 1, m & 2, m & 4, m & 8), Cfg<R>::T);
    best = g > best ? g : best;
  }
  if (dev >= 0 && dev < 64) cache[dev].store(best, std::memory_order_relaxed);
  return best;
}

// Unique, nonzero tag per launch for the slots' ready flags: a per-process
// random salt in the high bits, a launch counter in the low ones, so a flag
// left in a reused workspace by any earlier launch never equals a live tag.
static unsigned long long next_tag() {
  static std::atomic<unsigned long long> counter{0};
  static const unsigned long long salt = [] {
    std::random_device rd;
    return ((unsigned long long)rd() << 32 | rd()) & 0xffffff0000000000ull;
  }();
  return salt | ((counter.fetch_add(1) + 1) & 0xffffffffffull);
}

// n consecutive tag values no earlier launch of this process was given (the
// small-N kernel's per-step record tags): tag, tag+1, ... tag+n-1, never 0.
static unsigned long long reserve_tags(unsigned long long n) {
  static std::atomic<unsigned long long> next{1};
  return next.fetch_add(n);
}

// Resident CTAs per SM x SMs for a kernel (cached): the most CTAs that can be
// co-resident, which the in-kernel fixup's waits require of the launch grid.
static int resident_capacity(const void* fn, int threads) {
  struct Entry { int dev; const void* fn; int cap; };
  static Entry cache[64];
  static int used = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  for (int k = 0; k < used; ++k)
    if (cache[k].dev == dev && cache[k].fn == fn) return cache[k].cap;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0);
  const int cap = sms * per_sm;
  if (used < 64) cache[used++] = Entry{dev, fn, cap};
  return cap;
}

// In-kernel split-i-block fixup unless NB_FIXUP_KERNEL=1 (the separate
// fixup_kernel launch, kept for A/B measurements and over-subscribed grids).
static bool infix_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* env = getenv("NB_FIXUP_KERNEL");
    v = env ? (atoi(env) != 0 ? 0 : 1) : NB_INFIX_DEFAULT;
  }
  return v == 1;
}

// Cost-balanced schedule parameters of a launch (Sched): the live target
// groups of the last i-block (NB_FULL_GROUPS=1 computes every group there, the
// plain equal-units split, for A/B measurements).
template <typename R>
static void set_sched(StepArgs<R>& a, const StepGeometry& g) {
  constexpr int KG = Cfg<R>::template Core<false, false>::KG;
  static int full = -1;
  if (full < 0) {
    const char* env = getenv("NB_FULL_GROUPS");
    full = (env && atoi(env) != 0) ? 1 : 0;
  }
  const int64_t rows_last = a.n_i - (g.n_iblocks - 1) * (int64_t)g.i_block;
  const int64_t live = (rows_last + 2 * (int64_t)g.threads - 1) / (2 * (int64_t)g.threads);
  a.sched_kg = KG;
  a.sched_lg = (full || !NB_PARTIAL_GROUPS) ? KG : (int)(live < 1 ? 1 : (live > KG ? KG : live));
}

// The persistent grid capped so every CTA owns at least one unit: a CTA's cost
// share must be >= the most expensive unit (cost / grid >= kg).
template <typename R>
static int capped_grid(const StepArgs<R>& a, int grid) {
  const int64_t cost = Sched::make(a.units, 1, a.n_tiles, a.n_iblocks, a.sched_kg, a.sched_lg).cost;
  const int64_t cap = cost / a.sched_kg;
  return (int)(grid < cap ? grid : (cap < 1 ? 1 : cap));
}

// Any i-block whose units are split between CTAs (needs a fixup).
template <typename R>
static bool any_split_iblock(const StepArgs<R>& a) {
  const Sched S = sched_of(a);
  for (int64_t b = 0; b < a.n_iblocks; ++b)
    if (S.cta_of(b * a.n_tiles) != S.cta_of(b * a.n_tiles + a.n_tiles - 1)) return true;
  return false;
}

// SMs of the current device (cached per device).
static int sm_count() {
  static std::atomic<int> cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64) {
    const int c = cache[dev].load(std::memory_order_relaxed);
    if (c > 0) return c;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cache[dev].store(sms, std::memory_order_relaxed);
  return sms;
}

// Clusters of an FP32 launch through pair_kernel (0: the stream-K path) and its
// targets per lane K: the smallest K whose one wave of 2-CTA clusters (74 * 32 * K
// target slots on 148 SMs) holds the launch's targets, taken when the slots are
// filled at least to the measured break-even against the stream-K / persistent
// paths (profiles/r02/pair_kfam.txt: K = 2 from 3585 targets -- a 10-step simulate
// at N = 4096 takes 13.1 us per evaluation against the small-N kernel's 15.0, the
// crossover is ~3600 --, K = 3, 4 over their whole range, K = 5, 6,
// 7 from 88.7 / 90 / 92.7 %: K = 7 from 15367 targets, where stream-K needs its 11th i-block) and every warp's source slice holds at least one
// full tile.  NB_PAIR=0 / 1 turns it off / on wherever the targets fit one wave
// (A/B measurements, tests).
static int pair_clusters(int64_t n_i, int64_t j_count, int* k_out = nullptr) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("NB_PAIR");
    env = e ? atoi(e) : -1;
  }
  if (env == 0 || n_i < 1) return 0;
  const int64_t waves = sm_count() / PR_CL;
  int64_t k = (n_i + waves * 32 - 1) / (waves * 32);
  if (k < NB_PAIR_KMIN) k = NB_PAIR_KMIN;
  if (k > NB_PAIR_K) return 0;
  const int64_t ibc = 32 * k;
  const int64_t ncl = (n_i + ibc - 1) / ibc;
  if (ncl > waves) return 0;
  if (env != 1) {
    // minimum fill of the wave's target slots, in 1/1000
    static const int min_fill[8] = {1000, 1000, 757, 0, 0, 887, 900, 927};
    // (>= 128 sources per warp slice: partial tiles included, still ahead of the other paths)
    if (n_i * 1000 < waves * ibc * min_fill[k] || j_count < (int64_t)PR_S * NB_PAIR_TJ / 2) return 0;
  }
  if (k_out) *k_out = (int)k;
  return (int)ncl;
}

template <class Core>
static const void* pair_fn_of() {
  return reinterpret_cast<const void*>(&pair_kernel<Core, NB_PAIR_TJ>);
}

struct PairFn {
  const void* fn;
  int64_t smem;
};
template <class Core>
static PairFn pair_entry() {
  return PairFn{pair_fn_of<Core>(), pair_smem_bytes<Core, NB_PAIR_TJ>()};
}
template <int K>
static PairFn pair_entry_k(bool mask_self, bool uni) {
  if constexpr (K < NB_PAIR_KMIN || K > NB_PAIR_K) {
    return PairFn{nullptr, 0};
  } else {
    if (mask_self) return uni ? pair_entry<CorePair<K, true, true>>() : pair_entry<CorePair<K, true, false>>();
    return uni ? pair_entry<CorePair<K, false, true>>() : pair_entry<CorePair<K, false, false>>();
  }
}
static PairFn pair_entry_of(int k, bool mask_self, bool uni) {
  switch (k) {
    case 2: return pair_entry_k<2>(mask_self, uni);
    case 3: return pair_entry_k<3>(mask_self, uni);
    case 4: return pair_entry_k<4>(mask_self, uni);
    case 5: return pair_entry_k<5>(mask_self, uni);
    case 6: return pair_entry_k<6>(mask_self, uni);
    case 7: return pair_entry_k<7>(mask_self, uni);
    default: return PairFn{nullptr, 0};
  }
}

template <typename R>
static cudaError_t launch_pair_fn(StepArgs<R>& a, const PairFn& pf, int ncl, cudaStream_t stream);

static cudaError_t launch_pair(StepArgs<float> a, int flags, int ncl, int k, cudaStream_t stream) {
  const bool mask_self = (flags & 1) != 0, uni = (flags & 2) != 0;
  a.uniform_mass = uni ? 1 : 0;
  return launch_pair_fn<float>(a, pair_entry_of(k, mask_self, uni), ncl, stream);
}

// FP64: K = 2 (up to 4736 targets on 148 SMs) or 4 (9472), taken where measured
// faster than the persistent / stream-K paths (profiles/r02/pair_f64.txt).
static int pair64_clusters(int64_t n_i, int64_t j_count, int* k_out = nullptr) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("NB_PAIR");
    env = e ? atoi(e) : -1;
  }
  if (env == 0 || n_i < 1) return 0;
  const int64_t waves = sm_count() / PR_CL;
  const int64_t need = (n_i + waves * 32 - 1) / (waves * 32);
  const int64_t k = need <= 2 ? 2 : 4;
  if (need > 4) return 0;
  const int64_t ibc = 32 * k;
  const int64_t ncl = (n_i + ibc - 1) / ibc;
  if (ncl > waves) return 0;
  if (env != 1) {
    static const int min_fill[5] = {1000, 1000, NB_PAIR64_FILL2, 1000, NB_PAIR64_FILL4};  // 1/1000 of the slots
    // (>= 128 sources per warp slice: measured faster from 2561 sources on, partial tiles included)
    if (n_i * 1000 < waves * ibc * min_fill[k] || j_count < (int64_t)PR_S * NB_PAIR_TJ / 2) return 0;
  }
  if (k_out) *k_out = (int)k;
  return (int)ncl;
}
template <class Core>
static PairFn pair64_entry() {
  return PairFn{reinterpret_cast<const void*>(&pair_kernel_f64<Core, NB_PAIR_TJ>), pair64_smem_bytes<Core, NB_PAIR_TJ>()};
}
template <int K>
static PairFn pair64_entry_k(bool mask_self, bool uni) {
  if (mask_self) return uni ? pair64_entry<CorePair64<K, true, true>>() : pair64_entry<CorePair64<K, true, false>>();
  return uni ? pair64_entry<CorePair64<K, false, true>>() : pair64_entry<CorePair64<K, false, false>>();
}
static cudaError_t launch_pair64(StepArgs<double> a, int flags, int ncl, int k, cudaStream_t stream) {
  const bool mask_self = (flags & 1) != 0, uni = (flags & 2) != 0;
  a.uniform_mass = uni ? 1 : 0;
  return launch_pair_fn<double>(a, k == 2 ? pair64_entry_k<2>(mask_self, uni) : pair64_entry_k<4>(mask_self, uni), ncl,
                                stream);
}

template <typename R>
static cudaError_t launch_pair_fn(StepArgs<R>& a, const PairFn& pf, int ncl, cudaStream_t stream) {
  if (!pf.fn) return cudaErrorInvalidValue;
  const void* fn = pf.fn;
  const int64_t smem = pf.smem;
  {  // opt in to the dynamic shared memory once per (device, kernel)
    struct Opt { int dev; const void* fn; };
    static Opt opts[64];
    static int n_opts = 0;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    bool done = false;
    for (int k = 0; k < n_opts; ++k) done = done || (opts[k].dev == dev && opts[k].fn == fn);
    if (!done) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      if (n_opts < 64) opts[n_opts++] = Opt{dev, fn};
    }
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ncl * PR_CL));
  cfg.blockDim = dim3(PR_T);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {&a};
  cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
  count_launch();
  return e;
}

template <typename R>
cudaError_t launch_step(StepArgs<R> a, int flags, cudaStream_t stream) {
  if constexpr (sizeof(R) == 4) {
    int k = 0;
    if (const int ncl = pair_clusters(a.n_i, a.j_count, &k)) return launch_pair(a, flags, ncl, k, stream);
  } else {
    int k = 0;
    if (const int ncl = pair64_clusters(a.n_i, a.j_count, &k)) return launch_pair64(a, flags, ncl, k, stream);
  }
  const StepGeometry g = step_geometry<R>(a.n_i, a.j_count);
  a.n_tiles = g.n_tiles;
  a.n_iblocks = g.n_iblocks;
  a.units = g.units;
  set_sched<R>(a, g);
  const bool tma = use_tma<R>(a.n_i, a.j_count);
  using C = Cfg<R>;
  constexpr int IB = C::T * C::template Core<false, false>::K;
  const bool mask_self = (flags & 1) != 0, uni = (flags & 2) != 0;
  a.uniform_mass = uni ? 1 : 0;
  const void* fn = step_fn<R>(mask_self, uni, tma, false);
  const int grid = capped_grid<R>(a, grid_for(fn, C::T));
  a.grid = grid;
  // Any i-block split between CTAs needs a fixup: in this launch when the grid
  // is one resident wave, else by fixup_kernel.
  const bool split = any_split_iblock<R>(a);
  bool infix = false;
  if (split && infix_enabled()) {
    const void* fi = step_fn<R>(mask_self, uni, tma, true);
    if (grid <= resident_capacity(fi, C::T)) {
      fn = fi;
      infix = true;
      a.tag = next_tag();
    }
  }

  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(C::T);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {&a};
  cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
  count_launch();
  if (e != cudaSuccess) return e;

  if (split && !infix) {
    cfg.gridDim = dim3((unsigned)((a.n_i + NB_FIXUP_THREADS - 1) / NB_FIXUP_THREADS));
    cfg.blockDim = dim3(NB_FIXUP_THREADS);
    e = cudaLaunchKernelEx(&cfg, fixup_kernel<R, IB>, a);
    count_launch();
  }
  return e;
}

template <typename R>
const char* step_kernel_name(int64_t n_i, int64_t j_count) {
  if constexpr (sizeof(R) == 4) {
    if (pair_clusters(n_i, j_count)) return "pair_kernel";
  } else {
    if (pair64_clusters(n_i, j_count)) return "pair_kernel";
  }
  return "step_kernel";
}

template <typename R>
cudaError_t launch_simulate_persistent(StepArgs<R> a, int flags, V4<R>* pos_a, V4<R>* pos_b, int64_t steps,
                                       cudaStream_t stream) {
  const StepGeometry g = step_geometry<R>(a.n_i, a.j_count);
  a.n_tiles = g.n_tiles;
  a.n_iblocks = g.n_iblocks;
  a.units = g.units;
  set_sched<R>(a, g);
  const bool mask_self = (flags & 1) != 0, uni = (flags & 2) != 0;
  a.uniform_mass = uni ? 1 : 0;
  const int grid = capped_grid<R>(a, grid_for(step_fn<R>(mask_self, uni, false, false), Cfg<R>::T));
  a.grid = grid;
  int any_split = any_split_iblock<R>(a) ? 1 : 0;
  using C = Cfg<R>;
  void* args[] = {&a, &pos_a, &pos_b, &steps, &any_split};
  const void* fn;
  if (mask_self && uni)
    fn = reinterpret_cast<const void*>(&simulate_kernel<typename C::template Core<true, true>, C::T, C::TJ, C::MINB, NB_CHUNK>);
  else if (mask_self)
    fn = reinterpret_cast<const void*>(&simulate_kernel<typename C::template Core<true, false>, C::T, C::TJ, C::MINB, NB_CHUNK>);
  else if (uni)
    fn = reinterpret_cast<const void*>(&simulate_kernel<typename C::template Core<false, true>, C::T, C::TJ, C::MINB, NB_CHUNK>);
  else
    fn = reinterpret_cast<const void*>(&simulate_kernel<typename C::template Core<false, false>, C::T, C::TJ, C::MINB, NB_CHUNK>);
  // co-residency: the cooperative grid must fit the device at this occupancy
  int dev = 0, per_sm = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, C::T, 0);
  if (grid > per_sm * sms) return cudaErrorCooperativeLaunchTooLarge;
  cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(C::T), args, 0, stream);
  count_launch();
  return e;
}

template <class Core, int PPW>
static const void* small_fn() {
  return reinterpret_cast<const void*>(&small_simulate_kernel<Core, PPW>);
}
template <typename R, int PPW>
static const void* small_fn(bool mask_self, bool uni) {
  if constexpr (sizeof(R) == 4) {
    if (mask_self) return uni ? small_fn<SmallF32<true, true>, PPW>() : small_fn<SmallF32<true, false>, PPW>();
    return uni ? small_fn<SmallF32<false, true>, PPW>() : small_fn<SmallF32<false, false>, PPW>();
  } else {
    if (mask_self) return uni ? small_fn<SmallF64<true, true>, PPW>() : small_fn<SmallF64<true, false>, PPW>();
    return uni ? small_fn<SmallF64<false, true>, PPW>() : small_fn<SmallF64<false, false>, PPW>();
  }
}

// 8 targets per CTA (twice the CTAs) up to N = 3072 (FP32) / 1184 (FP64), else
// 16: the measured crossovers (profiles/small_n_r01.md; NB_SMALL_PPW=4|8 forces
// one).  When the 8-target grid exceeds what is co-resident (FP32 above N = 2368
// at 2 CTAs per SM), the 16-target form is taken instead of falling back to the
// stream-K paths.
template <typename R>
cudaError_t launch_simulate_small(StepArgs<R> a, int flags, V4<R>* pos_a, V4<R>* pos_b, int64_t steps,
                                  cudaStream_t stream, R* cols, R* cols_out) {
  const bool mask_self = (flags & 1) != 0, uni = (flags & 2) != 0;
  a.uniform_mass = uni ? 1 : 0;
  const int64_t n = a.n_all;
  NB_HT(10);
  int first = n <= (sizeof(R) == 4 ? 3072 : 1184) ? 4 : 8;
  bool forced = false;
  if (const char* env = getenv("NB_SMALL_PPW")) {  // (read per call: tools/small_n_bench.py)
    first = atoi(env) == 4 ? 4 : 8;
    forced = true;
  }
  bool needs_lm = false;
  if constexpr (sizeof(R) == 4) needs_lm = !uni && SmallF32<false, false>::NEEDS_LM;
  // Host-side launch preparation is on simulate()'s critical path at small N:
  // the co-resident capacity is cached per (device, kernel, shared-memory size)
  // and the opt-in shared-memory limit per (device, kernel) only ever raised.
  struct Cap { int dev; const void* fn; int64_t smem; int capacity; };
  struct Opt { int dev; const void* fn; int64_t smem; };
  static Cap caps[64];
  static Opt opts[32];
  static int n_caps = 0, n_opts = 0;
  static std::mutex mu;  // host threads may launch concurrently on different streams
  int ppw = first;
  const void* fn = nullptr;
  int64_t smem = 0, grid = 0;
  for (;;) {
    fn = ppw == 4 ? small_fn<R, 4>(mask_self, uni) : small_fn<R, 8>(mask_self, uni);
    smem = small_smem_bytes<R>(n, ppw, needs_lm);
    grid = (n + 2 * ppw - 1) / (2 * ppw);
    std::unique_lock<std::mutex> lock(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    Opt* opt = nullptr;
    for (int k = 0; k < n_opts; ++k)
      if (opts[k].dev == dev && opts[k].fn == fn) opt = &opts[k];
    cudaError_t fit = cudaSuccess;
    if (!opt || opt->smem < smem) {
      int smem_max = 0;
      cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      if (smem > smem_max) {
        fit = cudaErrorCooperativeLaunchTooLarge;
      } else {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        if (!opt && n_opts < 32) opt = &opts[n_opts++];
        if (opt) *opt = Opt{dev, fn, smem};
      }
    }
    if (fit == cudaSuccess) {
      int capacity = -1;
      for (int k = 0; k < n_caps; ++k)
        if (caps[k].dev == dev && caps[k].fn == fn && caps[k].smem == smem) capacity = caps[k].capacity;
      if (capacity < 0) {
        int per_sm = 0, sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, SN_T, (size_t)smem);
        capacity = per_sm * sms;
        if (n_caps < 64) caps[n_caps++] = Cap{dev, fn, smem, capacity};
      }
      if (grid > (int64_t)capacity) fit = cudaErrorCooperativeLaunchTooLarge;
    }
    lock.unlock();
    if (fit == cudaSuccess) break;
    if (ppw == 4 && !forced) {
      ppw = 8;  // half the CTAs
      continue;
    }
    return fit;
  }
  NB_HT(11);
  // Tagged position exchange between steps (NB_SMALL_TAGGED=0: a grid barrier
  // per step): steps+1 consecutive tags no earlier launch used.
  static const bool tagged = [] {
    const char* e = getenv("NB_SMALL_TAGGED");
    return !e || atoi(e) != 0;
  }();
  a.tag = (tagged && steps >= 3) ? reserve_tags((unsigned long long)steps + 1) : 0;
  a.pub = 0;
  int64_t L = small_split_stride(n, (SN_T / 32) * (32 / ppw));
  void* args[] = {&a, &pos_a, &pos_b, &steps, &L, &cols, &cols_out};
  NB_HT(12);
  cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(SN_T), args, (size_t)smem, stream);
  NB_HT(13);
  count_launch();
  return e;
}

#if NB_TRACE
int trace_setup(void* buf, int64_t cap) {
  unsigned long long* p = static_cast<unsigned long long*>(buf);
  unsigned long long c = (unsigned long long)cap, z = 0;
  if (cudaMemcpyToSymbol(g_trace, &p, sizeof(p)) != cudaSuccess) return 1;
  if (cudaMemcpyToSymbol(g_trace_cap, &c, sizeof(c)) != cudaSuccess) return 1;
  if (cudaMemcpyToSymbol(g_trace_n, &z, sizeof(z)) != cudaSuccess) return 1;
  return 0;
}
int64_t trace_count() {
  unsigned long long n = 0;
  cudaMemcpyFromSymbol(&n, g_trace_n, sizeof(n));
  return (int64_t)n;
}
#endif

template <typename R>
int64_t workspace_header_bytes() {
  return ((2 * (int64_t)max_grid<R>() * 8 + 255) / 256) * 256;
}

template <typename R>
int64_t step_workspace_bytes(int64_t n_i) {
  const StepGeometry g = step_geometry<R>(n_i, 1);
  const int64_t slots = 2 * (int64_t)max_grid<R>() * 3 * g.i_block * 8;
  return workspace_header_bytes<R>() + slots;
}

template StepGeometry step_geometry<float>(int64_t, int64_t);
template StepGeometry step_geometry<double>(int64_t, int64_t);
template cudaError_t launch_step<float>(StepArgs<float>, int, cudaStream_t);
template const char* step_kernel_name<float>(int64_t, int64_t);
template const char* step_kernel_name<double>(int64_t, int64_t);
template cudaError_t launch_step<double>(StepArgs<double>, int, cudaStream_t);
template cudaError_t launch_simulate_persistent<float>(StepArgs<float>, int, V4<float>*, V4<float>*, int64_t,
                                                      cudaStream_t);
template cudaError_t launch_simulate_persistent<double>(StepArgs<double>, int, V4<double>*, V4<double>*, int64_t,
                                                       cudaStream_t);
template int64_t workspace_header_bytes<float>();
template int64_t workspace_header_bytes<double>();
template int64_t step_workspace_bytes<float>(int64_t);
template int64_t step_workspace_bytes<double>(int64_t);
template cudaError_t launch_simulate_small<float>(StepArgs<float>, int, V4<float>*, V4<float>*, int64_t, cudaStream_t,
                                                  float*, float*);
template cudaError_t launch_simulate_small<double>(StepArgs<double>, int, V4<double>*, V4<double>*, int64_t,
                                                   cudaStream_t, double*, double*);

}  // namespace nb
