// Shared device/host helpers for the sm_100a N-body kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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

// Launch counter for the gpu_launches claim (host side).
void count_launch(int n = 1);

}  // namespace nb
