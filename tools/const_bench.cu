// Inner-loop microbenchmark: source bodies broadcast from shared memory (LDS into
// vector registers) vs from constant memory (ULDC into uniform registers).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2x;
__device__ __forceinline__ f2x pk(float lo, float hi) { f2x r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ void upk(f2x v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ f2x add2(f2x a, f2x b) { f2x d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2x mul2(f2x a, f2x b) { f2x d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) { f2x d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ float rsq(float x) { float y; asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

constexpr int NJ = 2048, KP = 3, T = 128;
__constant__ float4 cj[NJ];

template <bool CONST>
__global__ void __launch_bounds__(T, 3) k(const float4* gj, const float4* gi, float* out, float eps2, int reps) {
  __shared__ float4 sj[NJ];
  if (!CONST) { for (int j = threadIdx.x; j < NJ; j += T) sj[j] = gj[j]; __syncthreads(); }
  f2x nx[KP], ny[KP], nz[KP], tx[KP], ty[KP], tz[KP];
  for (int q = 0; q < KP; ++q) {
    float4 a = gi[(blockIdx.x * T * 2 * KP + (2 * q) * T + threadIdx.x) & 65535];
    float4 b = gi[(blockIdx.x * T * 2 * KP + (2 * q + 1) * T + threadIdx.x) & 65535];
    nx[q] = add2(0ull, pk(-a.x, -b.x)); ny[q] = add2(0ull, pk(-a.y, -b.y)); nz[q] = add2(0ull, pk(-a.z, -b.z));
    tx[q] = ty[q] = tz[q] = 0ull;
  }
  const f2x e2 = pk(eps2, eps2);
  for (int r = 0; r < reps; ++r) {
#pragma unroll 8
    for (int j = 0; j < NJ; ++j) {
      const float4 p = CONST ? cj[j] : sj[j];
      const f2x xj = pk(p.x, p.x), yj = pk(p.y, p.y), zj = pk(p.z, p.z), mj = pk(p.w, p.w);
#pragma unroll
      for (int q = 0; q < KP; ++q) {
        f2x dx = add2(xj, nx[q]), dy = add2(yj, ny[q]), dz = add2(zj, nz[q]);
        f2x d2 = fma2(dx, dx, e2); d2 = fma2(dy, dy, d2); d2 = fma2(dz, dz, d2);
        float a, b; upk(d2, a, b);
        f2x rr = pk(rsq(a), rsq(b));
        f2x w = mul2(mul2(rr, mj), mul2(rr, rr));
        tx[q] = fma2(dx, w, tx[q]); ty[q] = fma2(dy, w, ty[q]); tz[q] = fma2(dz, w, tz[q]);
      }
    }
  }
  float s = 0;
  for (int q = 0; q < KP; ++q) { float a, b; upk(tx[q], a, b); s += a + b; upk(ty[q], a, b); s += a + b; upk(tz[q], a, b); s += a + b; }
  out[blockIdx.x * T + threadIdx.x] = s;
}

int main() {
  float4 h[NJ];
  for (int j = 0; j < NJ; ++j) h[j] = make_float4((j % 97) * 0.01f, (j % 89) * 0.013f, (j % 83) * 0.011f, 1.0f);
  cudaMemcpyToSymbol(cj, h, sizeof(h));
  float4 *gj, *gi; float* out;
  cudaMalloc(&gj, sizeof(h)); cudaMemcpy(gj, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMalloc(&gi, 65536 * sizeof(float4)); cudaMemset(gi, 0, 65536 * sizeof(float4));
  cudaMalloc(&out, 148 * 3 * T * sizeof(float));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = 148 * 3, reps = 8;
  for (int mode = 0; mode < 2; ++mode) {
    auto launch = [&] { if (mode) k<true><<<grid, T>>>(gj, gi, out, 1e-3f, reps); else k<false><<<grid, T>>>(gj, gi, out, 1e-3f, reps); };
    launch(); launch();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = best < ms ? best : ms; }
    double inter = (double)grid * T * 2 * KP * NJ * reps;
    double rate = inter / (best * 1e-3);
    printf("%s: %.4e interactions/s = %.1f%% of nominal FP32 (20 flop)\n", mode ? "constant(UR)" : "shared(LDS)", rate, 100 * 20 * rate / (148 * 128 * 2 * 1.965e9));
  }
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
