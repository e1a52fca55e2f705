// Shared device/host helpers for the sm_100a N-body kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

// 1: the e^2 term of the FP64 rsqrt corrections on the FP32/INT pipes
// (sq_term_f32): 15 DP ops per force interaction instead of 16 (NB_F64_MIXED),
// 12 per potential pair instead of 13 (NB_DIAG_MIXED).  Measured slower on
// B200 -- force -7 %, potential -12 % (profiles/variants_r01_f64_mixed.txt):
// the DP pipe is not the only limit at ~90 % busy (the extra issue slots and
// register reads cost more than the DP op saves), so both default to off.
#ifndef NB_F64_MIXED
#define NB_F64_MIXED 0
#endif
#ifndef NB_DIAG_MIXED
#define NB_DIAG_MIXED 0
#endif

namespace nb {

// Packed 4-vectors of the system precision: (x, y, z, m) for positions,
// (vx, vy, vz, 0) for velocities, (ax, ay, az, 0) for accelerations.
struct __align__(16) F4 { float x, y, z, w; };
struct __align__(32) D4 { double x, y, z, w; };

template <typename R> struct Vec;
template <> struct Vec<float> { using T = F4; };
template <> struct Vec<double> { using T = D4; };
template <typename R> using V4 = typename Vec<R>::T;

// ---------------------------------------------------------------- loads/stores
__device__ __forceinline__ F4 ld4(const F4* p) {
  float4 v = __ldg(reinterpret_cast<const float4*>(p));
  return F4{v.x, v.y, v.z, v.w};
}
__device__ __forceinline__ D4 ld4(const D4* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  double2 a = __ldg(q), b = __ldg(q + 1);
  return D4{a.x, a.y, b.x, b.y};
}
// Coherent (L2) loads for buffers another CTA of the same launch wrote.
__device__ __forceinline__ F4 ld4_cg(const F4* p) {
  float4 v = __ldcg(reinterpret_cast<const float4*>(p));
  return F4{v.x, v.y, v.z, v.w};
}
__device__ __forceinline__ D4 ld4_cg(const D4* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  double2 a = __ldcg(q), b = __ldcg(q + 1);
  return D4{a.x, a.y, b.x, b.y};
}
__device__ __forceinline__ void st4(F4* p, F4 v) {
  *reinterpret_cast<float4*>(p) = make_float4(v.x, v.y, v.z, v.w);
}
__device__ __forceinline__ void st4(D4* p, D4 v) {
  double2* q = reinterpret_cast<double2*>(p);
  q[0] = make_double2(v.x, v.y);
  q[1] = make_double2(v.z, v.w);
}

// Single-transaction, gpu-coherent accesses of one packed body: 128 bits (FP32)
// or 256 bits (FP64, LDG/STG.E.ENL2.256 on sm_100a) in ONE relaxed gpu-scope
// access of an aligned 16- / 32-byte record, i.e. at most one 32-byte sector, so
// a reader sees a record entirely old or entirely new.  The small-N kernel's
// tagged position exchange rests on that: the record's fourth word carries the
// step tag, and no other data is consumed under it.
__device__ __forceinline__ F4 ld4_pub(const F4* p) {
  F4 v;
  asm volatile("ld.relaxed.gpu.global.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ D4 ld4_pub(const D4* p) {
  D4 v;
  asm volatile("ld.relaxed.gpu.global.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st4_pub(F4* p, F4 v) {
  asm volatile("st.relaxed.gpu.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void st4_pub(D4* p, D4 v) {
  asm volatile("st.relaxed.gpu.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
               : "memory");
}
// Step tag <-> the bit pattern of a body's fourth word.  Sign bit set: never the
// pattern of a valid (positive, finite) mass.  No arithmetic touches the word.
__device__ __forceinline__ float tag_word(float, unsigned long long t) {
  return __uint_as_float(0x80000000u | (unsigned)(t & 0x7fffffffull));
}
__device__ __forceinline__ double tag_word(double, unsigned long long t) {
  return __longlong_as_double((long long)(0x8000000000000000ull | (t & 0x7fffffffffffffffull)));
}
__device__ __forceinline__ bool same_word(float a, float b) { return __float_as_uint(a) == __float_as_uint(b); }
__device__ __forceinline__ bool same_word(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b);
}

// ---------------------------------------------------------------- exact IEEE ops
// The integrator must reproduce the reference's rounding sequence bit for bit
// (pkg/setup.py:7-8,17 builds with -ffp-contract=off), so every update op is an
// explicitly rounded intrinsic that the compiler may not contract into an FMA.
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// ---------------------------------------------------------------- MUFU
// Bare MUFU.RSQ (FTZ, <= 2 ulp): the force kernels' only transcendental.
__device__ __forceinline__ float rsqrt_mufu(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_mufu(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_mufu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Bare MUFU.RSQ64H seed (about 2^-22 relative); refined by the caller.
__device__ __forceinline__ double rsqrt_seed(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// c*e^2 for the quadratic term of the FP64 rsqrt corrections, computed off the
// DP pipe.  e = 1 - d2*y0^2 with a MUFU.RSQ64H seed y0 (21 significant bits, so
// y0^2 is exact) is either 0 or, in magnitude, in [2^-95, 2^-20]: the exact
// 1 - d2*y0^2 is a nonzero multiple of ulp(d2)*ulp(y0^2) ~ 2^-95 or zero.  For
// |e| in [2^-255, 1) the top three of the eleven exponent bits are 011, so the
// 32 bits from the lowest of them down (one funnel shift of the hi:lo pair)
// read as an FP32 number equal to -|e|*2^128: that exponent bit lands in the
// sign, the mantissa is truncated to 24 bits, 0 stays 0, and the sign squares
// away.  The square is formed on the FP32 pipe at that scale and the result, a
// positive FP32 F = c*e^2*2^128, maps back the same way: the FP64 with bits
// ((F >> 3) + 0x30000000 : F << 29) is F*2^-128 exactly (0 -> 2^-255, harmless
// next to 1).  Only the e^2 term is computed this way: it is ~2^-42 of the
// result, so the FP32 rounding (~2^-22 relative) costs ~2^-64; the linear term
// stays in FP64.  Per call: one DP op fewer for 2 FMUL + 3 INT ops
// (SHF.L.W, LEA.HI, IMAD.SHL).
__device__ __forceinline__ double sq_term_f32(double e, float c) {
  const unsigned lo = (unsigned)__double2loint(e), hi = (unsigned)__double2hiint(e);
  const float g = __uint_as_float(__funnelshift_l(lo, hi, 3));  // -|e|*2^128
  // (g * c*2^-128) is c*|e| (a normal number; the constant itself is an FP32
  // subnormal, exact for c = 1.875 or 0.375 -- no FTZ on these FMULs).
  const unsigned f = __float_as_uint((g * (c * 0x1p-128f)) * g);  // c*e^2*2^128
  return __hiloint2double((int)((f >> 3) + 0x30000000u), (int)(f << 29));
}

// Stream-K schedule over the (i-block x source chunk) units, balanced by COST:
// a unit of a full i-block costs kg (the target groups -- pairs of target
// bodies per thread -- it computes), a unit of the last, partial i-block only
// lg <= kg (its dead groups are skipped: step_body's full_tile_live).  CTA c
// owns the units whose cost positions fall in [c*cost/grid, (c+1)*cost/grid).
// With lg == kg this is the plain equal-units split (start(c) = c*units/grid).
struct Sched {
  int64_t units, grid;
  int64_t full_units;  // units of the i-blocks before the last one
  int64_t kg, lg;      // cost of a full-i-block unit, of a last-i-block unit
  int64_t cost;        // full_units*kg + (units - full_units)*lg
  __host__ __device__ static Sched make(int64_t units, int64_t grid, int64_t n_tiles, int64_t n_iblocks, int64_t kg,
                                        int64_t lg) {
    Sched S;
    S.units = units;
    S.grid = grid;
    S.full_units = (n_iblocks - 1) * n_tiles;
    S.kg = kg;
    S.lg = lg;
    S.cost = S.full_units * kg + (units - S.full_units) * lg;
    return S;
  }
  // cost position of the start of unit u, and the unit holding cost position x
  __host__ __device__ __forceinline__ int64_t pos(int64_t u) const {
    return u <= full_units ? u * kg : full_units * kg + (u - full_units) * lg;
  }
  __host__ __device__ __forceinline__ int64_t unit_at(int64_t x) const {
    return x < full_units * kg ? x / kg : full_units + (x - full_units * kg) / lg;
  }
  __host__ __device__ __forceinline__ int64_t start(int64_t c) const { return unit_at(c * cost / grid); }
  // CTA owning unit u: the largest c with start(c) <= u, i.e. c*cost/grid < pos(u+1).
  __host__ __device__ __forceinline__ int64_t cta_of(int64_t u) const {
    return (pos(u + 1) * grid + cost - 1) / cost - 1;
  }
};

// Launch counter for the gpu_launches claim (host side).
void count_launch(int n = 1);

}  // namespace nb
