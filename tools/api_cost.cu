// Host-side cost of the CUDA runtime calls on simulate()'s small-N critical path
// (nb_dev_simulate_cols), each timed alone over many repetitions on the GPU box.
// build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/api_cost.cu -o tools/api_cost
#include <chrono>
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_kernel(int* p) {
  if (p && threadIdx.x == 1 << 30) *p = 0;
}
__global__ void coop_kernel(int* p, int steps) {
  cooperative_groups::grid_group g = cooperative_groups::this_grid();
  for (int s = 0; s < steps; ++s) g.sync();
  if (p && threadIdx.x == 1 << 30) *p = 0;
}

struct BigArg { char b[296]; };
__global__ void coop_big(BigArg a, int steps) {
  extern __shared__ char sm[];
  cooperative_groups::grid_group g = cooperative_groups::this_grid();
  for (int s = 0; s < steps; ++s) g.sync();
  if (threadIdx.x == 1 << 30) sm[0] = a.b[0];
}

template <class F>
static double us(F f, int reps = 2000) {
  f();
  cudaDeviceSynchronize();
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) f();
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int* d = nullptr;
  cudaMalloc(&d, 1 << 20);
  void* h = nullptr;
  cudaMallocHost(&h, 1 << 20);
  const size_t bytes = 7 * 1024 * 8;  // C1's column block
  int dev = 0;
  cudaPointerAttributes attr;
  void* hd = nullptr;
  std::printf("%-58s %8.2f us\n", "cudaGetDevice", us([&] { cudaGetDevice(&dev); }));
  std::printf("%-58s %8.2f us\n", "cudaPointerGetAttributes (device ptr)", us([&] { cudaPointerGetAttributes(&attr, d); }));
  std::printf("%-58s %8.2f us\n", "cudaHostGetDevicePointer", us([&] { cudaHostGetDevicePointer(&hd, h, 0); }));
  std::printf("%-58s %8.2f us\n", "cudaStreamSynchronize (idle)", us([&] { cudaStreamSynchronize(st); }));
  std::printf("%-58s %8.2f us\n", "empty launch (async)", us([&] { empty_kernel<<<128, 256, 0, st>>>(d); }));
  cudaDeviceSynchronize();
  std::printf("%-58s %8.2f us\n", "empty launch + sync", us([&] { empty_kernel<<<128, 256, 0, st>>>(d); cudaStreamSynchronize(st); }));
  int steps = 0;
  void* args[] = {&d, &steps};
  std::printf("%-58s %8.2f us\n", "cooperative launch, 0 grid syncs (async)",
              us([&] { cudaLaunchCooperativeKernel((void*)coop_kernel, 128, 256, args, 0, st); }));
  cudaDeviceSynchronize();
  std::printf("%-58s %8.2f us\n", "cooperative launch, 0 grid syncs + sync",
              us([&] { cudaLaunchCooperativeKernel((void*)coop_kernel, 128, 256, args, 0, st); cudaStreamSynchronize(st); }));
  steps = 11;
  std::printf("%-58s %8.2f us\n", "cooperative launch, 11 grid syncs (128 CTAs) + sync",
              us([&] { cudaLaunchCooperativeKernel((void*)coop_kernel, 128, 256, args, 0, st); cudaStreamSynchronize(st); }));
  steps = 0;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(128);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  std::printf("%-58s %8.2f us\n", "cudaLaunchKernelEx cooperative attr, 0 syncs (async)",
              us([&] { cudaLaunchKernelExC(&cfg, (void*)coop_kernel, args); }));
  cudaDeviceSynchronize();
  std::printf("%-58s %8.2f us\n", "H2D 56 KiB pinned (async)", us([&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st); }));
  cudaDeviceSynchronize();
  std::printf("%-58s %8.2f us\n", "H2D 56 KiB pinned + sync", us([&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st); cudaStreamSynchronize(st); }));
  std::printf("%-58s %8.2f us\n", "D2H 56 KiB pinned + sync", us([&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st); cudaStreamSynchronize(st); }));
  std::printf("%-58s %8.2f us\n", "H2D + coop launch(0 syncs) + D2H + sync", us([&] {
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
    cudaLaunchCooperativeKernel((void*)coop_kernel, 128, 256, args, 0, st);
    cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st); }));
  std::printf("%-58s %8.2f us\n", "H2D + coop launch(0 syncs) + sync", us([&] {
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
    cudaLaunchCooperativeKernel((void*)coop_kernel, 128, 256, args, 0, st);
    cudaStreamSynchronize(st); }));
  // r02: simulate()'s launch in context -- legacy stream 0 vs a non-blocking
  // stream, 40 KB of dynamic shared memory, a 300-byte parameter block, and a
  // CUDA graph of (H2D + cooperative kernel) replayed
  BigArg big = {};
  int ss = 0;
  void* args2[] = {&big, &ss};
  cudaFuncSetAttribute((void*)coop_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  for (int pass = 0; pass < 2; ++pass) {
    cudaStream_t s2 = pass ? st : (cudaStream_t)0;
    const char* nm = pass ? "non-blocking stream" : "legacy stream 0";
    cudaDeviceSynchronize();
    std::printf("coop 128x256, 40KB dyn smem, 300B params, %-20s %8.2f us\n", nm,
                us([&] { cudaLaunchCooperativeKernel((void*)coop_big, 128, 256, args2, 40 * 1024, s2); }, 200));
    cudaDeviceSynchronize();
    std::printf("H2D + that coop + sync, %-35s %8.2f us\n", nm, us([&] {
      cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s2);
      cudaLaunchCooperativeKernel((void*)coop_big, 128, 256, args2, 40 * 1024, s2);
      cudaStreamSynchronize(s2); }, 500));
  }
  cudaGraph_t gr;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
  cudaError_t ce = cudaLaunchCooperativeKernel((void*)coop_big, 128, 256, args2, 40 * 1024, st);
  cudaError_t ee = cudaStreamEndCapture(st, &gr);
  cudaError_t ie = cudaGraphInstantiate(&ge, gr, 0);
  std::printf("graph capture: launch %d, end %d, instantiate %d\n", (int)ce, (int)ee, (int)ie);
  if (ie == cudaSuccess) {
    std::printf("%-58s %8.2f us\n", "graph launch (H2D + coop) async", us([&] { cudaGraphLaunch(ge, st); }, 200));
    cudaDeviceSynchronize();
    std::printf("%-58s %8.2f us\n", "graph launch (H2D + coop) + sync", us([&] { cudaGraphLaunch(ge, st); cudaStreamSynchronize(st); }, 500));
  }
  return 0;
}
