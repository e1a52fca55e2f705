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
//    operand), so the FP32 pipe -- not the issue slot -- is the bound.
//  * Source bodies are staged through shared memory in tiles of TJ packed
//    (x,y,z,m) 4-vectors, double-buffered with one __syncthreads per tile; the
//    inner loop reads them with broadcast LDS.128 (no bank conflicts: every lane
//    reads the same address).
//  * FP32 accuracy: each tile's partial sum is FP32 (<= TJ terms); tile partials
//    are accumulated in FP64 (a single FP32 chain misses 1e-5 at
//    N >= 131072, tile partials + FP64 outer sums are at ~1e-7).
//  * FP64: MUFU.RSQ64H seed + one cubic correction that yields m*r^3 directly
//    (16 DP ops + 1 MUFU per interaction, no slow-path branch).
//  * Work distribution is stream-K over the (i-block x j-tile) space: a
//    persistent grid of SMs x occupancy CTAs, each owning an equal contiguous
//    range of units, so every SM gets the same work at every N.  An i-block split
//    between CTAs is combined through FP64 partial slots; the last CTA to arrive
//    sums them in fixed CTA order (bitwise reproducible run to run) and runs the
//    epilogue.
#include "nbody_common.cuh"
#include "nbody_kernels.h"

namespace nb {

struct Sched {
  int64_t units;
  int64_t grid;
  __device__ __forceinline__ int64_t start(int64_t c) const { return c * units / grid; }
  // CTA owning unit u: the largest c with start(c) <= u.
  __device__ __forceinline__ int64_t cta_of(int64_t u) const {
    return ((u + 1) * grid + units - 1) / units - 1;
  }
};

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

// ---------------------------------------------------------------- FP32 core
// K target bodies per thread as K/2 packed pairs.  The FP64 segment sums live in
// shared memory (3*K doubles per thread, touched once per tile) so the inner
// loop keeps its registers for the pairs and their temporaries.
template <int K_, bool MASK>
struct CoreF32 {
  using R = float;
  static constexpr int K = K_;
  static constexpr int KP = K / 2;
  static constexpr int SMEM_SUMS = 3 * K;  // doubles per thread
  f2x nx[KP], ny[KP], nz[KP];  // negated target positions, paired
  f2x tx[KP], ty[KP], tz[KP];  // FP32 partial sums of the current tile
  int selfj[K];
  f2x e2;
  double* ss;  // this thread's FP64 sums: ss[(d*K + k) * stride]
  int stride;

  __device__ __forceinline__ void init(float eps2, double* s, int st) {
    e2 = pk(eps2, eps2);
    ss = s;
    stride = st;
  }
  __device__ __forceinline__ void set_pair(int q, const F4& p0, const F4& p1) {
    // +0 + (-x) is a real FADD2 (not an identity for x = +-0), so the pair is
    // materialised once in an aligned register pair instead of being re-paired
    // from the scalar load registers at every use.
    nx[q] = add2(0ull, pk(-p0.x, -p1.x));
    ny[q] = add2(0ull, pk(-p0.y, -p1.y));
    nz[q] = add2(0ull, pk(-p0.z, -p1.z));
  }
  __device__ __forceinline__ double sum(int d, int k) const { return ss[(d * K + k) * stride]; }
  __device__ __forceinline__ void set_sum(int d, int k, double v) { ss[(d * K + k) * stride] = v; }
  __device__ __forceinline__ void zero_sums() {
#pragma unroll
    for (int i = 0; i < 3 * K; ++i) ss[i * stride] = 0.0;
  }
  __device__ __forceinline__ void begin_tile() {
#pragma unroll
    for (int q = 0; q < KP; ++q) tx[q] = ty[q] = tz[q] = 0ull;
  }
  __device__ __forceinline__ void interact(const F4& pj, int jj) {
    const f2x xj = pk(pj.x, pj.x), yj = pk(pj.y, pj.y), zj = pk(pj.z, pj.z), mj = pk(pj.w, pj.w);
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      const f2x dx = add2(xj, nx[q]);
      const f2x dy = add2(yj, ny[q]);
      const f2x dz = add2(zj, nz[q]);
      f2x d2 = fma2(dx, dx, e2);
      d2 = fma2(dy, dy, d2);
      d2 = fma2(dz, dz, d2);
      float d2a, d2b;
      upk(d2, d2a, d2b);
      const f2x r = pk(rsqrt_mufu(d2a), rsqrt_mufu(d2b));
      const f2x r2 = mul2(r, r);
      const f2x mr = mul2(r, mj);
      f2x w = mul2(mr, r2);
      if (MASK) {
        float wa, wb;
        upk(w, wa, wb);
        if (jj == selfj[2 * q]) wa = 0.f;
        if (jj == selfj[2 * q + 1]) wb = 0.f;
        w = pk(wa, wb);
      }
      tx[q] = fma2(dx, w, tx[q]);
      ty[q] = fma2(dy, w, ty[q]);
      tz[q] = fma2(dz, w, tz[q]);
    }
  }
  __device__ __forceinline__ void end_tile() {
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      float a, b;
      upk(tx[q], a, b);
      ss[(0 * K + 2 * q) * stride] += (double)a;
      ss[(0 * K + 2 * q + 1) * stride] += (double)b;
      upk(ty[q], a, b);
      ss[(1 * K + 2 * q) * stride] += (double)a;
      ss[(1 * K + 2 * q + 1) * stride] += (double)b;
      upk(tz[q], a, b);
      ss[(2 * K + 2 * q) * stride] += (double)a;
      ss[(2 * K + 2 * q + 1) * stride] += (double)b;
    }
  }
};

// ---------------------------------------------------------------- FP64 core
template <int K_, bool MASK>
struct CoreF64 {
  using R = double;
  static constexpr int K = K_;
  static constexpr int SMEM_SUMS = 1;
  double nx[K], ny[K], nz[K];
  double sx[K], sy[K], sz[K];
  int selfj[K];
  double e2;

  __device__ __forceinline__ void init(double eps2, double*, int) { e2 = eps2; }
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
  __device__ __forceinline__ void interact(const D4& pj, int jj) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double dx = pj.x + nx[k], dy = pj.y + ny[k], dz = pj.z + nz[k];
      double d2 = fma(dx, dx, e2);
      d2 = fma(dy, dy, d2);
      d2 = fma(dz, dz, d2);
      // y0 ~ d2^-1/2 to ~2^-22; with e = 1 - d2*y0^2 the exact
      // m*d2^-3/2 = m*y0^3*(1-e)^-3/2 = m*y0^3*(1 + 1.5e + 1.875e^2 + O(e^3)).
      const double y = rsqrt_seed(d2);
      const double t = y * y;
      const double e = fma(-d2, t, 1.0);
      const double my3 = pj.w * (t * y);
      const double q = e * fma(e, 1.875, 1.5);
      double w = fma(my3, q, my3);
      if (MASK && jj == selfj[k]) w = 0.0;
      sx[k] = fma(dx, w, sx[k]);
      sy[k] = fma(dy, w, sy[k]);
      sz[k] = fma(dz, w, sz[k]);
    }
  }
};

// ---------------------------------------------------------------- epilogue
template <typename R>
__device__ __forceinline__ void finalize_body(const StepArgs<R>& a, int64_t il, double tx,
                                              double ty, double tz) {
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
  const R ax = (R)(tx * a.g), ay = (R)(ty * a.g), az = (R)(tz * a.g);
  V4<R> an;
  an.x = ax; an.y = ay; an.z = az; an.w = R(0);
  if (a.mode != NB_STEP_MODE_ACCEL) {
    V4<R> v = a.vel[il];
    if (a.mode != NB_STEP_MODE_FIRST) {  // trapezoidal kick, kernels/__init__.py:223-227
      const V4<R> ap = a.acc[il];
      v.x = add_rn(v.x, mul_rn(sub_rn(ax, ap.x), a.f));
      v.y = add_rn(v.y, mul_rn(sub_rn(ay, ap.y), a.f));
      v.z = add_rn(v.z, mul_rn(sub_rn(az, ap.z), a.f));
    }
    if (a.mode != NB_STEP_MODE_FINAL) {  // kick-drift, _accel_cy.pyx:218-226
      const int64_t ig = a.i_begin + il;
      V4<R> p = a.pos[ig];
      const R dvx = mul_rn(ax, a.dt), dvy = mul_rn(ay, a.dt), dvz = mul_rn(az, a.dt);
      p.x = add_rn(p.x, mul_rn(add_rn(v.x, mul_rn(a.half, dvx)), a.dt));
      p.y = add_rn(p.y, mul_rn(add_rn(v.y, mul_rn(a.half, dvy)), a.dt));
      p.z = add_rn(p.z, mul_rn(add_rn(v.z, mul_rn(a.half, dvz)), a.dt));
      st4(a.pos_next + ig, p);
      v.x = add_rn(v.x, dvx);
      v.y = add_rn(v.y, dvy);
      v.z = add_rn(v.z, dvz);
    }
    st4(a.vel + il, v);
  }
  st4(a.acc + il, an);
}

// ---------------------------------------------------------------- stream-K kernel
template <class Core, int T, int TJ, int MINB>
__global__ void __launch_bounds__(T, MINB) step_kernel(const StepArgs<typename Core::R> a) {
  using R = typename Core::R;
  using B = V4<R>;
  constexpr int K = Core::K;
  constexpr int IB = T * K;
  constexpr int PER = TJ / T;  // tile elements staged per thread
  static_assert(TJ % T == 0, "tile must be a multiple of the block");

  __shared__ B tile[2][TJ];
  __shared__ double s_sums[Core::SMEM_SUMS * T];
  __shared__ int s_last;

  const int tid = threadIdx.x;
  const int64_t c = blockIdx.x;
  const Sched S{a.units, a.grid};
  const int64_t NT = a.n_tiles;
  const int64_t u_begin = S.start(c), u_end = S.start(c + 1);

  Core core;
  core.init(a.eps2, s_sums + tid, T);

  for (int64_t u = u_begin; u < u_end;) {
    const int64_t b = u / NT;
    const int64_t t0 = u - b * NT;
    const int64_t t1 = min(NT, t0 + (u_end - u));

#pragma unroll
    for (int q = 0; q < K / 2; ++q) {
      const int64_t i0 = b * IB + (2 * q) * T + tid, i1 = i0 + T;
      core.set_pair(q, ld4(a.pos + a.i_begin + (i0 < a.n_i ? i0 : a.n_i - 1)),
                    ld4(a.pos + a.i_begin + (i1 < a.n_i ? i1 : a.n_i - 1)));
    }
    core.zero_sums();

    B stage[PER];
    auto load_tile = [&](int64_t t) {
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        const int64_t off = t * TJ + r * T + tid;
        if (off < a.j_count) {
          int64_t jg = a.j_begin + off;
          if (jg >= a.n_all) jg -= a.n_all;
          stage[r] = ld4(a.pos + jg);
        } else {
          stage[r] = B{};
        }
      }
    };
    auto store_tile = [&](int buf) {
#pragma unroll
      for (int r = 0; r < PER; ++r) tile[buf][r * T + tid] = stage[r];
    };

    load_tile(t0);
    store_tile(0);
    __syncthreads();

    for (int64_t t = t0; t < t1; ++t) {
      const int buf = (int)((t - t0) & 1);
      if (t + 1 < t1) load_tile(t + 1);
      const int64_t off0 = t * TJ;
      const int count = (int)max((int64_t)0, min((int64_t)TJ, a.j_count - off0));
      if (Core::MASK_SELF) {
        int64_t base = a.j_begin + off0;
        if (base >= a.n_all) base -= a.n_all;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          int64_t rel = a.i_begin + b * IB + k * T + tid - base;
          if (rel < 0) rel += a.n_all;
          core.selfj[k] = rel < count ? (int)rel : -1;
        }
      }
      core.begin_tile();
      const B* tb = tile[buf];
      if (count == TJ) {
#pragma unroll 4
        for (int jj = 0; jj < TJ; ++jj) core.interact(tb[jj], jj);
      } else {
#pragma unroll 1
        for (int jj = 0; jj < count; ++jj) core.interact(tb[jj], jj);
      }
      core.end_tile();
      if (t + 1 < t1) store_tile(buf ^ 1);
      __syncthreads();
    }

    if (t0 == 0 && t1 == NT) {
      // The whole source range of this i-block was ours: finish directly.
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int64_t il = b * IB + k * T + tid;
        if (il < a.n_i) finalize_body<R>(a, il, core.sum(0, k), core.sum(1, k), core.sum(2, k));
      }
    } else {
      // Split i-block: publish FP64 partials; the last CTA in combines them in
      // ascending CTA order (deterministic) and runs the epilogue.
      const int64_t slot = (u == u_begin) ? 2 * c : 2 * c + 1;
      double* sp = a.slots + slot * 3 * IB;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        sp[k * T + tid] = core.sum(0, k);
        sp[IB + k * T + tid] = core.sum(1, k);
        sp[2 * IB + k * T + tid] = core.sum(2, k);
      }
      __threadfence();
      __syncthreads();
      const int64_t cf = S.cta_of(b * NT), cl = S.cta_of(b * NT + NT - 1);
      if (tid == 0) {
        const unsigned prev = atomicAdd(a.counters + b, 1u);
        const int last = prev == (unsigned)(cl - cf);
        if (last) a.counters[b] = 0u;  // leave the workspace zeroed for the next launch
        s_last = last;
      }
      __syncthreads();
      if (s_last) {
        __threadfence();
        core.zero_sums();
        for (int64_t cc = cf; cc <= cl; ++cc) {
          const int64_t sl = (S.start(cc) / NT == b) ? 2 * cc : 2 * cc + 1;
          const double* q = a.slots + sl * 3 * IB;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            core.set_sum(0, k, core.sum(0, k) + __ldcg(q + k * T + tid));
            core.set_sum(1, k, core.sum(1, k) + __ldcg(q + IB + k * T + tid));
            core.set_sum(2, k, core.sum(2, k) + __ldcg(q + 2 * IB + k * T + tid));
          }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int64_t il = b * IB + k * T + tid;
          if (il < a.n_i) finalize_body<R>(a, il, core.sum(0, k), core.sum(1, k), core.sum(2, k));
        }
      }
    }
    u += t1 - t0;
  }
}

// ---------------------------------------------------------------- configurations
// FP32: 128 threads x 8 bodies (4 FFMA2 pairs) = 1024-body i-blocks, 256-body tiles.
// FP64: 128 threads x 4 bodies = 512-body i-blocks, 128-body tiles.
template <bool M> struct CoreF32M : CoreF32<8, M> { static constexpr bool MASK_SELF = M; };
template <bool M> struct CoreF64M : CoreF64<4, M> { static constexpr bool MASK_SELF = M; };

template <typename R> struct Cfg;
template <> struct Cfg<float> {
  static constexpr int T = 128, TJ = 256, MINB = 3;
  template <bool M> using Core = CoreF32M<M>;
};
template <> struct Cfg<double> {
  static constexpr int T = 128, TJ = 128, MINB = 3;
  template <bool M> using Core = CoreF64M<M>;
};

template <typename R, bool M>
static const void* kernel_ptr() {
  using C = Cfg<R>;
  return reinterpret_cast<const void*>(&step_kernel<typename C::template Core<M>, C::T, C::TJ, C::MINB>);
}

template <typename R>
StepGeometry step_geometry(int64_t n_i, int64_t j_count) {
  using C = Cfg<R>;
  StepGeometry g{};
  g.threads = C::T;
  g.i_block = C::T * C::template Core<false>::K;
  g.tile = C::TJ;
  g.n_iblocks = (n_i + g.i_block - 1) / g.i_block;
  g.n_tiles = j_count > 0 ? (j_count + C::TJ - 1) / C::TJ : 1;
  g.units = g.n_iblocks * g.n_tiles;
  return g;
}

template <typename R>
int max_grid() {
  static int cached[64] = {};
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev]) return cached[dev];
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int best = 1;
  for (int m = 0; m < 2; ++m) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, m ? kernel_ptr<R, true>() : kernel_ptr<R, false>(),
                                                  Cfg<R>::T, 0);
    if (per_sm < 1) per_sm = 1;
    best = best > sms * per_sm ? best : sms * per_sm;
  }
  cached[dev] = best;
  return best;
}

template <typename R>
cudaError_t launch_step(StepArgs<R> a, bool mask_self, cudaStream_t stream) {
  const StepGeometry g = step_geometry<R>(a.n_i, a.j_count);
  a.n_tiles = g.n_tiles;
  a.n_iblocks = g.n_iblocks;
  a.units = g.units;
  int grid = max_grid<R>();
  if ((int64_t)grid > g.units) grid = (int)g.units;
  a.grid = grid;
  using C = Cfg<R>;
  if (mask_self)
    step_kernel<typename C::template Core<true>, C::T, C::TJ, C::MINB><<<grid, C::T, 0, stream>>>(a);
  else
    step_kernel<typename C::template Core<false>, C::T, C::TJ, C::MINB><<<grid, C::T, 0, stream>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <typename R>
int64_t step_workspace_bytes(int64_t n_i) {
  const StepGeometry g = step_geometry<R>(n_i, 1);
  const int64_t counters = ((g.n_iblocks * 4 + 255) / 256) * 256;
  const int64_t slots = 2 * (int64_t)max_grid<R>() * 3 * g.i_block * 8;
  return counters + slots;
}

template StepGeometry step_geometry<float>(int64_t, int64_t);
template StepGeometry step_geometry<double>(int64_t, int64_t);
template cudaError_t launch_step<float>(StepArgs<float>, bool, cudaStream_t);
template cudaError_t launch_step<double>(StepArgs<double>, bool, cudaStream_t);
template int64_t step_workspace_bytes<float>(int64_t);
template int64_t step_workspace_bytes<double>(int64_t);

}  // namespace nb
