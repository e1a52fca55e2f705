// Register-file / operand microbenchmark for packed FP32x2 on sm_100a: how the
// number of distinct 64-bit register-pair operands of FFMA2 affects throughput.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2x;
__device__ __forceinline__ f2x pk(float lo, float hi) { f2x r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) { f2x d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
constexpr int IT = 2048;

// 3 distinct pairs per FFMA2
__global__ void k_three(float* out, float s, const float* in) {
  f2x a[8], b[8], c[8];
  for (int k = 0; k < 8; ++k) { a[k] = pk(in[(threadIdx.x + 7 * k + 2) & 255], in[(threadIdx.x + 11 * k + 5) & 255]); b[k] = pk(in[(threadIdx.x + k) & 255], in[(threadIdx.x + 3 * k + 1) & 255]); c[k] = pk(threadIdx.x, k); }
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = fma2(a[k], b[k], c[k]);
  }
  float r = 0; for (int k = 0; k < 8; ++k) { unsigned long long v = c[k]; r += __uint_as_float((unsigned)v); }
  if (r == 1234.f) out[0] = r;
}
// 2 distinct pairs (a shared b within groups of 3: like dx*w, dy*w, dz*w)
__global__ void k_shared(float* out, float s, const float* in) {
  f2x a[8], b[3], c[8];
  for (int k = 0; k < 8; ++k) { a[k] = pk(in[(threadIdx.x + 7 * k + 2) & 255], in[(threadIdx.x + 11 * k + 5) & 255]); c[k] = pk(threadIdx.x, k); }
  for (int k = 0; k < 3; ++k) b[k] = pk(in[(threadIdx.x + k) & 255], in[(threadIdx.x + 3 * k + 1) & 255]);
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = fma2(a[k], b[k / 3], c[k]);
  }
  float r = 0; for (int k = 0; k < 8; ++k) { unsigned long long v = c[k]; r += __uint_as_float((unsigned)v); }
  if (r == 1234.f) out[0] = r;
}
// a*a + c (1 distinct pair + acc)
__global__ void k_square(float* out, float s, const float* in) {
  f2x a[8], c[8];
  for (int k = 0; k < 8; ++k) { a[k] = pk(in[(threadIdx.x + 7 * k + 2) & 255], in[(threadIdx.x + 11 * k + 5) & 255]); c[k] = pk(threadIdx.x, k); }
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = fma2(a[k], a[k], c[k]);
  }
  float r = 0; for (int k = 0; k < 8; ++k) { unsigned long long v = c[k]; r += __uint_as_float((unsigned)v); }
  if (r == 1234.f) out[0] = r;
}
// scalar FFMA with 3 distinct registers
__global__ void k_scalar3(float* out, float s, const float* in) {
  float a[8], b[8], c[8];
  for (int k = 0; k < 8; ++k) { a[k] = in[(threadIdx.x + 7 * k + 2) & 255]; b[k] = in[(threadIdx.x + 5 * k) & 255]; c[k] = threadIdx.x + k; }
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(c[k]) : "f"(a[k]), "f"(b[k]));
  }
  float r = 0; for (int k = 0; k < 8; ++k) r += c[k];
  if (r == 1234.f) out[0] = r;
}
// scalar FFMA, 16 chains of 3 distinct regs
__global__ void k_scalar3_16(float* out, float s, const float* in) {
  float a[16], b[16], c[16];
  for (int k = 0; k < 16; ++k) { a[k] = in[(threadIdx.x + 7 * k + 2) & 255]; b[k] = in[(threadIdx.x + 5 * k) & 255]; c[k] = threadIdx.x + k; }
  for (int it = 0; it < IT / 2; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(c[k]) : "f"(a[k]), "f"(b[k]));
  }
  float r = 0; for (int k = 0; k < 16; ++k) r += c[k];
  if (r == 1234.f) out[0] = r;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  float* d; cudaMalloc(&d, 64);
  float hin[256]; for (int i = 0; i < 256; ++i) hin[i] = 0.999f + i * 1e-7f;
  float* din; cudaMalloc(&din, sizeof(hin)); cudaMemcpy(din, hin, sizeof(hin), cudaMemcpyHostToDevice);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, double lane_ops_per_thread, void (*k)(float*, float, const float*), int threads, int bps) {
    int blocks = p.multiProcessorCount * bps;
    for (int w = 0; w < 2; ++w) k<<<blocks, threads>>>(d, 1.f, din);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); k<<<blocks, threads>>>(d, 1.f, din); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best; }
    double ops = lane_ops_per_thread * threads * (double)blocks / (best * 1e-3);
    printf("%-12s thr=%4d x%d/SM  %.1f lane-ops/SM/clk\n", name, threads, bps, ops / p.multiProcessorCount / (clk * 1e3));
  };
  for (int bps : {1, 2, 4}) {
    run("ffma2_3pair", 16.0 * IT, k_three, 256, bps);
    run("ffma2_shared", 16.0 * IT, k_shared, 256, bps);
    run("ffma2_square", 16.0 * IT, k_square, 256, bps);
    run("ffma_3reg", 8.0 * IT, k_scalar3, 256, bps);
    run("ffma_3reg16", 8.0 * IT, k_scalar3_16, 256, bps);
  }
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
