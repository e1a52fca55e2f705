// Inner-loop formulation microbenchmark (FP32 force, packed pairs): source order
// and operand placement variants of the same 12-op interaction.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2x;
__device__ __forceinline__ f2x pk(float lo, float hi) { f2x r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ void upk(f2x v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ f2x add2(f2x a, f2x b) { f2x d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2x mul2(f2x a, f2x b) { f2x d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) { f2x d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ float rsq(float x) { float y; asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

constexpr int NJ = 2048, T = 64;

template <int KP, int V>
__global__ void __launch_bounds__(T, 6) k(const float4* gj, const float4* gi, float* out, float eps2, int reps) {
  __shared__ float4 sj[NJ];
  for (int j = threadIdx.x; j < NJ; j += T) sj[j] = gj[j];
  __syncthreads();
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
      const float4 p = sj[j];
      const f2x xj = pk(p.x, p.x), yj = pk(p.y, p.y), zj = pk(p.z, p.z), mj = pk(p.w, p.w);
      if (V == 0) {  // current: per pair
#pragma unroll
        for (int q = 0; q < KP; ++q) {
          f2x dx = add2(xj, nx[q]), dy = add2(yj, ny[q]), dz = add2(zj, nz[q]);
          f2x d2 = fma2(dx, dx, e2); d2 = fma2(dy, dy, d2); d2 = fma2(dz, dz, d2);
          float a, b; upk(d2, a, b);
          f2x rr = pk(rsq(a), rsq(b));
          f2x w = mul2(mul2(rr, mj), mul2(rr, rr));
          tx[q] = fma2(dx, w, tx[q]); ty[q] = fma2(dy, w, ty[q]); tz[q] = fma2(dz, w, tz[q]);
        }
      } else if (V == 1) {  // stage-wise across pairs
        f2x dx[KP], dy[KP], dz[KP], d2[KP], rr[KP], w[KP];
#pragma unroll
        for (int q = 0; q < KP; ++q) dx[q] = add2(xj, nx[q]);
#pragma unroll
        for (int q = 0; q < KP; ++q) dy[q] = add2(yj, ny[q]);
#pragma unroll
        for (int q = 0; q < KP; ++q) dz[q] = add2(zj, nz[q]);
#pragma unroll
        for (int q = 0; q < KP; ++q) d2[q] = fma2(dx[q], dx[q], e2);
#pragma unroll
        for (int q = 0; q < KP; ++q) d2[q] = fma2(dy[q], dy[q], d2[q]);
#pragma unroll
        for (int q = 0; q < KP; ++q) d2[q] = fma2(dz[q], dz[q], d2[q]);
#pragma unroll
        for (int q = 0; q < KP; ++q) { float a, b; upk(d2[q], a, b); rr[q] = pk(rsq(a), rsq(b)); }
#pragma unroll
        for (int q = 0; q < KP; ++q) w[q] = mul2(mul2(rr[q], mj), mul2(rr[q], rr[q]));
#pragma unroll
        for (int q = 0; q < KP; ++q) { tx[q] = fma2(w[q], dx[q], tx[q]); ty[q] = fma2(w[q], dy[q], ty[q]); tz[q] = fma2(w[q], dz[q], tz[q]); }
      } else if (V == 2) {  // w in slot a for the accumulates
#pragma unroll
        for (int q = 0; q < KP; ++q) {
          f2x dx = add2(xj, nx[q]), dy = add2(yj, ny[q]), dz = add2(zj, nz[q]);
          f2x d2 = fma2(dx, dx, e2); d2 = fma2(dy, dy, d2); d2 = fma2(dz, dz, d2);
          float a, b; upk(d2, a, b);
          f2x rr = pk(rsq(a), rsq(b));
          f2x w = mul2(mul2(rr, mj), mul2(rr, rr));
          tx[q] = fma2(w, dx, tx[q]); ty[q] = fma2(w, dy, ty[q]); tz[q] = fma2(w, dz, tz[q]);
        }
      } else if (V >= 4) {  // stage-wise variants
        f2x dx[KP], dy[KP], dz[KP], d2[KP], rr[KP], w[KP];
#pragma unroll
        for (int q = 0; q < KP; ++q) dx[q] = (V == 6) ? add2(nx[q], xj) : add2(xj, nx[q]);
#pragma unroll
        for (int q = 0; q < KP; ++q) dy[q] = (V == 6) ? add2(ny[q], yj) : add2(yj, ny[q]);
#pragma unroll
        for (int q = 0; q < KP; ++q) dz[q] = (V == 6) ? add2(nz[q], zj) : add2(zj, nz[q]);
#pragma unroll
        for (int q = 0; q < KP; ++q) d2[q] = fma2(dx[q], dx[q], e2);
#pragma unroll
        for (int q = 0; q < KP; ++q) d2[q] = fma2(dy[q], dy[q], d2[q]);
#pragma unroll
        for (int q = 0; q < KP; ++q) d2[q] = fma2(dz[q], dz[q], d2[q]);
#pragma unroll
        for (int q = 0; q < KP; ++q) { float a, b; upk(d2[q], a, b); rr[q] = pk(rsq(a), rsq(b)); }
        if (V == 7) {
#pragma unroll
          for (int q = 0; q < KP; ++q) w[q] = mul2(mul2(mj, rr[q]), mul2(rr[q], rr[q]));
        } else {
#pragma unroll
          for (int q = 0; q < KP; ++q) w[q] = mul2(mul2(rr[q], mj), mul2(rr[q], rr[q]));
        }
        if (V == 4) {
#pragma unroll
          for (int q = 0; q < KP; ++q) tx[q] = fma2(w[q], dx[q], tx[q]);
#pragma unroll
          for (int q = 0; q < KP; ++q) ty[q] = fma2(w[q], dy[q], ty[q]);
#pragma unroll
          for (int q = 0; q < KP; ++q) tz[q] = fma2(w[q], dz[q], tz[q]);
        } else if (V == 5) {
#pragma unroll
          for (int q = 0; q < KP; ++q) { tx[q] = fma2(dx[q], w[q], tx[q]); ty[q] = fma2(dy[q], w[q], ty[q]); tz[q] = fma2(dz[q], w[q], tz[q]); }
        } else {
#pragma unroll
          for (int q = 0; q < KP; ++q) { tx[q] = fma2(w[q], dx[q], tx[q]); ty[q] = fma2(w[q], dy[q], ty[q]); tz[q] = fma2(w[q], dz[q], tz[q]); }
        }
      } else {  // V == 3: r2 first then mr (different dependency shape)
#pragma unroll
        for (int q = 0; q < KP; ++q) {
          f2x dx = add2(nx[q], xj), dy = add2(ny[q], yj), dz = add2(nz[q], zj);
          f2x d2 = fma2(dz, dz, e2); d2 = fma2(dy, dy, d2); d2 = fma2(dx, dx, d2);
          float a, b; upk(d2, a, b);
          f2x rr = pk(rsq(a), rsq(b));
          f2x r2 = mul2(rr, rr);
          f2x w = mul2(r2, mul2(mj, rr));
          tx[q] = fma2(dx, w, tx[q]); ty[q] = fma2(dy, w, ty[q]); tz[q] = fma2(dz, w, tz[q]);
        }
      }
    }
  }
  float s = 0;
  for (int q = 0; q < KP; ++q) { float a, b; upk(tx[q], a, b); s += a + b; upk(ty[q], a, b); s += a + b; upk(tz[q], a, b); s += a + b; }
  out[blockIdx.x * T + threadIdx.x] = s;
}

template <int KP, int V>
void run(const float4* gj, const float4* gi, float* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = 148 * 6, reps = 8;
  k<KP, V><<<grid, T>>>(gj, gi, out, 1e-3f, reps);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); k<KP, V><<<grid, T>>>(gj, gi, out, 1e-3f, reps); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = best < ms ? best : ms; }
  double rate = (double)grid * T * 2 * KP * NJ * reps / (best * 1e-3);
  printf("KP=%d V=%d: %.4e int/s = %.2f%% nominal\n", KP, V, rate, 100 * 20 * rate / (148 * 128 * 2 * 1.965e9));
}

int main() {
  float4 h[NJ];
  for (int j = 0; j < NJ; ++j) h[j] = make_float4((j % 97) * 0.01f, (j % 89) * 0.013f, (j % 83) * 0.011f, 1.0f);
  float4 *gj, *gi; float* out;
  cudaMalloc(&gj, sizeof(h)); cudaMemcpy(gj, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMalloc(&gi, 65536 * sizeof(float4)); cudaMemset(gi, 0, 65536 * sizeof(float4));
  cudaMalloc(&out, 148 * 6 * T * sizeof(float));
  run<3, 0>(gj, gi, out); run<3, 1>(gj, gi, out); run<3, 4>(gj, gi, out); run<3, 5>(gj, gi, out);
  run<3, 6>(gj, gi, out); run<3, 7>(gj, gi, out); run<4, 4>(gj, gi, out); run<4, 6>(gj, gi, out);
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
