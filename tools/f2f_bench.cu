// Throughput of FP64<->FP32 conversions (F2F) vs DFMA on sm_100a: decides whether
// the FP64 rsqrt refinement can move its low-order polynomial to the FP32 pipe.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int IT = 1024;
__global__ void k_f2f(float* out, const float* in) {
  double d[8]; float f[8];
  for (int k = 0; k < 8; ++k) { f[k] = in[(threadIdx.x + k) & 255]; d[k] = 0; }
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { d[k] = (double)f[k] * 1.0000001; f[k] = (float)d[k]; }
  }
  float s = 0; for (int k = 0; k < 8; ++k) s += f[k];
  if (s == 1234.f) out[0] = s;
}
__global__ void k_f2f_mix(float* out, const float* in) {   // conversions interleaved with independent DFMAs
  double d[8], a[8]; float f[8];
  for (int k = 0; k < 8; ++k) { f[k] = in[(threadIdx.x + k) & 255]; d[k] = 0; a[k] = in[(threadIdx.x * 3 + k) & 255]; }
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float e = (float)a[k];
      e = fmaf(e, 1.875f, 1.5f) * e;
      a[k] = fma(a[k], 0.999999, (double)e);
    }
  }
  double s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1234.) out[0] = (float)s;
}
__global__ void k_dfma(float* out, const float* in) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = in[(threadIdx.x + k) & 255];
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { a[k] = fma(a[k], 0.999999, 1e-7); a[k] = fma(a[k], 1.000001, -1e-7); }
  }
  double s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1234.) out[0] = (float)s;
}
// The planned FP64 weight: 14 DP ops + 2 F2F + 2 FP32 ops + 1 MUFU.RSQ64H per
// element.  If F2F shares the DP pipe this runs at 14 + 2*4 DP-op slots, if it
// runs on the XU pipe (with MUFU) at max(14/64, 3/16) per element.
__global__ void k_plan(float* out, const float* in) {
  double a[4], b[4];
  for (int k = 0; k < 4; ++k) { a[k] = in[(threadIdx.x + k) & 255]; b[k] = in[(threadIdx.x * 7 + k) & 255]; }
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double y;
      asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a[k]));
      double t = y * y;
      double e = fma(-a[k], t, 1.0);
      float ef = (float)e;
      ef = fmaf(ef, 1.875f, 1.5f) * ef;
      double m = b[k] * y;
      m = m * t;
      double w = fma(m, (double)ef, m);
      double s0 = fma(w, a[k], b[k]);
      double s1 = fma(w, s0, 1e-9);
      double s2 = fma(s1, 0.5, s0);
      double s3 = s2 + s1;
      double s4 = s3 * 0.999;
      double s5 = fma(s4, 1e-3, 1.0);
      double s6 = s5 - 1e-3;
      a[k] = fma(s6, 1e-12, a[k]);  // 14 DP ops incl. t, e, m, m*t, w
      b[k] = b[k] + 1e-30 * s6;
    }
  }
  double s = 0; for (int k = 0; k < 4; ++k) s += a[k] + b[k];
  if (s == 1234.) out[0] = (float)s;
}
__global__ void k_plan_nof2f(float* out, const float* in) {  // same with the polynomial in FP64 (16 DP ops)
  double a[4], b[4];
  for (int k = 0; k < 4; ++k) { a[k] = in[(threadIdx.x + k) & 255]; b[k] = in[(threadIdx.x * 7 + k) & 255]; }
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double y;
      asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a[k]));
      double t = y * y;
      double e = fma(-a[k], t, 1.0);
      double q = e * fma(e, 1.875, 1.5);
      double m = b[k] * y;
      m = m * t;
      double w = fma(m, q, m);
      double s0 = fma(w, a[k], b[k]);
      double s1 = fma(w, s0, 1e-9);
      double s2 = fma(s1, 0.5, s0);
      double s3 = s2 + s1;
      double s4 = s3 * 0.999;
      double s5 = fma(s4, 1e-3, 1.0);
      double s6 = s5 - 1e-3;
      a[k] = fma(s6, 1e-12, a[k]);
      b[k] = b[k] + 1e-30 * s6;
    }
  }
  double s = 0; for (int k = 0; k < 4; ++k) s += a[k] + b[k];
  if (s == 1234.) out[0] = (float)s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *d, *in; cudaMalloc(&d, 64); cudaMalloc(&in, 1024);
  float h[256]; for (int i = 0; i < 256; ++i) h[i] = 1.0f + i * 1e-3f; cudaMemcpy(in, h, 1024, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, double ops, void (*k)(float*, const float*)) {
    int blocks = p.multiProcessorCount * 4, thr = 256;
    k<<<blocks, thr>>>(d, in); k<<<blocks, thr>>>(d, in);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); k<<<blocks, thr>>>(d, in); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best; }
    double rate = ops * blocks * thr / (best * 1e-3);
    printf("%-10s %.1f ops/SM/clk\n", name, rate / p.multiProcessorCount / (clk * 1e3));
  };
  run("f2f_pair", 8.0 * IT * 2, k_f2f);        // F2F.F64.F32 + F2F.F32.F64 (+ DMUL) per element
  run("mix", 8.0 * IT, k_f2f_mix);            // per element: 2 F2F + 2 fp32 + 1 DFMA
  run("dfma", 8.0 * IT * 2, k_dfma);
  run("plan_f2f", 4.0 * IT, k_plan);        // elements/SM/clk
  run("plan_dp", 4.0 * IT, k_plan_nof2f);   // elements/SM/clk
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
