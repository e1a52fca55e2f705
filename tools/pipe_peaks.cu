// Pipe-throughput microbenchmark for the CUDA-core roofline of the N-body force
// kernels: FFMA (scalar), FFMA2 (packed f32x2), MUFU.RSQ and DFMA lane-ops/s on
// the whole chip.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// tools/pipe_peaks tools/pipe_peaks.cu ; run on a B200 via gpurun.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_ffma(float* out, float b0, float c0) {
  float b = b0 + threadIdx.x * 1e-9f, c = c0 * (1.f + threadIdx.x * 1e-9f);
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3f + k;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b, c);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma2(float* out, float b0, float c0) {
  float b = b0 + threadIdx.x * 1e-9f, c = c0 * (1.f + threadIdx.x * 1e-9f);
  float2 a[8];
  float2 bb = make_float2(b, b + 1e-7f), cc = make_float2(c, c * 0.5f);
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = make_float2(threadIdx.x * 1e-3f + k, k * 0.5f);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __ffma2_rn(a[k], bb, cc);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k].x + a[k].y;
  if (s == 12345.f) out[0] = s;
}

__device__ __forceinline__ float rsq(float x) {
  float y; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y;
}

__global__ void k_mufu(float* out, float b) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3f + k + 1.f;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = rsq(a[k]);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_dfma(double* out, double b, double c) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0.;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.) out[0] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("device %s sms=%d cc=%d.%d clock_khz=%d\n", p.name, p.multiProcessorCount, p.major, p.minor, clk_khz);
  float* df; double* dd; CK(cudaMalloc(&df, 64)); CK(cudaMalloc(&dd, 64));
  const int threads = 512, blocks = p.multiProcessorCount * 4;  // 2048 threads/SM
  const double lanes = double(threads) * blocks;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, double ops_per_thread, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double ops = ops_per_thread * lanes / (best * 1e-3);
    double per_sm_clk = ops / p.multiProcessorCount / (clk_khz * 1e3);
    printf("%-6s %10.3f ms  %.4e lane-ops/s  %.1f lane-ops/SM/clk@%dMHz  (x2 flop = %.2f TFLOP/s)\n",
           name, best, ops, per_sm_clk, clk_khz / 1000, 2 * ops / 1e12);
  };
  run("ffma", 8.0 * ITERS, [&] { k_ffma<<<blocks, threads>>>(df, 0.999f, 1e-4f); });
  run("ffma2", 16.0 * ITERS, [&] { k_ffma2<<<blocks, threads>>>(df, 0.999f, 1e-4f); });
  run("mufu", 8.0 * (ITERS / 4), [&] { k_mufu<<<blocks, threads>>>(df, 0.5f); });
  run("dfma", 8.0 * (ITERS / 4), [&] { k_dfma<<<blocks, threads>>>(dd, 0.999, 1e-4); });
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}
