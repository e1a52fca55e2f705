// extern "C" boundary of libnbody_b200.so (declared in include/nbody_b200.h).
//
// nb_host_* mirror the reference's compiled-kernel FFI (the Cython functions of
// /root/reference/pkg/src/nbodybench/kernels/_accel_cy.pyx) and the step loop of
// kernels.simulate (kernels/__init__.py:230-253) on host pointers; nb_dev_* are
// the stream-ordered device-pointer entry points the Python host code drives.
#include <dlfcn.h>
#include <nccl.h>

#include <atomic>
#include <cmath>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "nbody_b200.h"
#include "nbody_kernels.h"

#if NB_TRACE
namespace nb {
double g_ht[16];
int g_ht_n = 0;
}  // namespace nb
using nb::g_ht;
using nb::g_ht_n;
#endif

namespace nb {
static std::atomic<int64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace nb

using namespace nb;

namespace {

thread_local std::string t_err;

int fail(int code, const std::string& msg) {
  t_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  t_err = std::string(where) + ": " + cudaGetErrorName(e) + ": " + cudaGetErrorString(e);
  return NB_ERR_CUDA + (int)e;
}
#define NB_CUDA(call)                                 \
  do {                                                \
    cudaError_t e_ = (call);                          \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

#ifndef NB_SMALL_MAX_N_F32
#define NB_SMALL_MAX_N_F32 3584
#endif
#ifndef NB_SMALL_MAX_N_F64
#define NB_SMALL_MAX_N_F64 2560
#endif

// Bodies up to which nb_dev_simulate runs the whole loop in one persistent
// cooperative launch (NB_PERSISTENT_MAX_N overrides, read per call; 0 disables).
int64_t persistent_max_n() {
  const char* env = getenv("NB_PERSISTENT_MAX_N");
  return env ? atoll(env) : 8192;
}

// Bodies up to which nb_dev_simulate uses the small-N cooperative kernel (source
// split inside the CTA): NB_SMALL_MAX_N overrides (0 disables; read per call so
// tests can switch paths), default by precision: the measured crossover with the
// stream-K persistent kernel (profiles/small_n_r01.md).
int64_t small_max_n(int precision_bytes) {
  const char* env = getenv("NB_SMALL_MAX_N");
  if (env) return atoll(env);
  return precision_bytes == 4 ? NB_SMALL_MAX_N_F32 : NB_SMALL_MAX_N_F64;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Make the device that owns `p` current for this runtime instance.  The library
// links its own (static) CUDA runtime, whose notion of the current device need
// not follow the host framework's (e.g. torch.cuda.set_device(local_rank)).
cudaError_t bind_device_of(const void* p) {
  cudaPointerAttributes attr;
  cudaError_t e = cudaPointerGetAttributes(&attr, p);
  if (e != cudaSuccess) return e;
  if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged) return cudaErrorInvalidDevicePointer;
  int cur = -1;
  if ((e = cudaGetDevice(&cur)) != cudaSuccess) return e;
  return cur == attr.device ? cudaSuccess : cudaSetDevice(attr.device);
}

template <typename R>
void fill_step_args(StepArgs<R>& a, const void* pos4, int64_t n_all, int64_t i_begin, int64_t n_i, int64_t j_begin,
                    int64_t j_count, double g, double eps2, double dt, int mode, double* carry, int carry_mode,
                    void* acc4, void* vel4, void* pos4_next, void* workspace, void* const* peers, int n_peers);

template <typename R>
int make_step_args(StepArgs<R>& a, const void* pos4, int64_t n_all, int64_t i_begin, int64_t n_i, int64_t j_begin,
             int64_t j_count, double g, double eps2, double dt, int mode, int flags,
             double* carry, int carry_mode, void* acc4, void* vel4, void* pos4_next,
             void* workspace, int64_t workspace_bytes, void* stream,
             void* const* peers, int n_peers) {
  if (n_all < 1 || i_begin < 0 || n_i < 0 || i_begin + n_i > n_all)
    return fail(NB_ERR_ARG, "target range [i_begin, i_begin+n_i) must lie in [0, n_all)");
  if (j_begin < 0 || j_begin >= n_all || j_count < 0 || j_count > n_all)
    return fail(NB_ERR_ARG, "source range must satisfy 0 <= j_begin < n_all and 0 <= j_count <= n_all");
  if (mode < NB_MODE_ACCEL || mode > NB_STEP_FINAL_KICK)
    return fail(NB_ERR_ARG, "mode must be NB_MODE_ACCEL or an NB_STEP_* mode");
  if (carry_mode < 0 || carry_mode > 2) return fail(NB_ERR_ARG, "carry_mode must be 0, 1 or 2");
  if (carry_mode != 0 && !carry) return fail(NB_ERR_ARG, "carry buffer required for carry_mode 1/2");
  if (!(g == g) || !(eps2 >= 0.0)) return fail(NB_ERR_ARG, "g must be a number and eps2 >= 0");
  if (n_peers < 0 || n_peers > kMaxPeers || (n_peers > 0 && !peers))
    return fail(NB_ERR_ARG, "n_peers must be in [0, 8] with a peer pointer array");
  for (int q = 0; q < n_peers; ++q)
    if (!peers[q] || !aligned16(peers[q]) || peers[q] == pos4)
      return fail(NB_ERR_ARG, "peer next-position buffers must be 16-byte aligned and must not alias pos4");
  if (n_i == 0) return -1;  // nothing to launch
  if (!pos4 || !aligned16(pos4)) return fail(NB_ERR_ARG, "pos4 must be a 16-byte aligned device pointer");
  const bool finalize = carry_mode != 1;
  if (finalize && (!acc4 || !aligned16(acc4))) return fail(NB_ERR_ARG, "acc4 must be a 16-byte aligned device pointer");
  if (finalize && mode != NB_MODE_ACCEL && (!vel4 || !aligned16(vel4)))
    return fail(NB_ERR_ARG, "vel4 required (16-byte aligned) for step modes");
  if (finalize && (mode == NB_STEP_FIRST || mode == NB_STEP_KICK_DRIFT)) {
    if (!pos4_next || !aligned16(pos4_next)) return fail(NB_ERR_ARG, "pos4_next required for drift modes");
    if (pos4_next == pos4) return fail(NB_ERR_ARG, "pos4_next must not alias pos4");
  }
  if (cudaError_t be = bind_device_of(pos4)) return cuda_fail(be, "pos4 is not a device pointer");
  const int64_t need = step_workspace_bytes<R>(n_i);
  if (!workspace || workspace_bytes < need)
    return fail(NB_ERR_WORKSPACE, "workspace smaller than nb_dev_workspace_bytes(): need " + std::to_string(need));
  fill_step_args<R>(a, pos4, n_all, i_begin, n_i, j_begin, j_count, g, eps2, dt, mode, carry, carry_mode, acc4, vel4,
                    pos4_next, workspace, peers, n_peers);
  return NB_OK;
}

// The StepArgs of a launch, unchecked: make_step_args validates first; the
// host entry points that allocated every buffer themselves call it directly.
template <typename R>
void fill_step_args(StepArgs<R>& a, const void* pos4, int64_t n_all, int64_t i_begin, int64_t n_i, int64_t j_begin,
                    int64_t j_count, double g, double eps2, double dt, int mode, double* carry, int carry_mode,
                    void* acc4, void* vel4, void* pos4_next, void* workspace, void* const* peers, int n_peers) {
  a = StepArgs<R>{};
  a.pos = static_cast<const V4<R>*>(pos4);
  a.n_all = n_all; a.i_begin = i_begin; a.n_i = n_i; a.j_begin = j_begin; a.j_count = j_count;
  a.eps2 = (R)eps2;
  a.g = g;
  a.dt = (R)dt; a.half = (R)0.5; a.f = (R)(0.5 * dt);
  a.mode = mode; a.carry_mode = carry_mode; a.carry = carry;
  a.acc = static_cast<V4<R>*>(acc4);
  a.vel = static_cast<V4<R>*>(vel4);
  a.pos_next = static_cast<V4<R>*>(pos4_next);
  a.flags = static_cast<unsigned long long*>(workspace);
  a.slots = reinterpret_cast<double*>(static_cast<char*>(workspace) + workspace_header_bytes<R>());
  a.n_peers = n_peers;
  for (int q = 0; q < n_peers; ++q) a.peers[q] = static_cast<V4<R>*>(peers[q]);
}

template <typename R>
int dev_step(const void* pos4, int64_t n_all, int64_t i_begin, int64_t n_i, int64_t j_begin,
             int64_t j_count, double g, double eps2, double dt, int mode, int flags,
             double* carry, int carry_mode, void* acc4, void* vel4, void* pos4_next,
             void* workspace, int64_t workspace_bytes, void* stream,
             void* const* peers = nullptr, int n_peers = 0) {
  StepArgs<R> a;
  int rc = make_step_args<R>(a, pos4, n_all, i_begin, n_i, j_begin, j_count, g, eps2, dt, mode, flags, carry,
                             carry_mode, acc4, vel4, pos4_next, workspace, workspace_bytes, stream, peers, n_peers);
  if (rc == -1) return NB_OK;
  if (rc) return rc;
  const int kf = flags & (NB_FLAG_EXCLUDE_SELF | NB_FLAG_UNIFORM_MASS);
  if (mode == NB_MODE_ACCEL && carry_mode == 0 && n_peers == 0 && i_begin == 0 && n_i == n_all && j_begin == 0 &&
      j_count == n_all && n_all <= small_max_n((int)sizeof(R))) {
    // small N, whole system: one evaluation of the small-N kernel (no partial slots)
    V4<R>* p = const_cast<V4<R>*>(static_cast<const V4<R>*>(pos4));
    cudaError_t e = launch_simulate_small<R>(a, kf, p, nullptr, -1, static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) return NB_OK;
    if (e != cudaErrorCooperativeLaunchTooLarge && e != cudaErrorNotSupported)
      return cuda_fail(e, "small_simulate_kernel");
    cudaGetLastError();  // fall through to the stream-K pass
  }
  cudaError_t e = launch_step<R>(a, kf, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "launch_step");
  return NB_OK;
}

// `events` (optional): steps+2 recorded events, one before every launch and one
// after the last, so a caller can time each force evaluation on the stream.
// cols (optional): the host API's device column block (x, y, z, m, vx, vy, vz;
// n each).  The small-N kernel then reads the initial state from it and writes
// the final state back (*cols_done = 1); every other path packs it into pos_a /
// vel4 here first and leaves the unpack to the caller (*cols_done = 0).
template <typename R>
int dev_simulate(void* pos_a, void* pos_b, void* vel4, void* acc4, int64_t n, double g, double dt,
                 double eps2, int64_t steps, int flags, void* ws, int64_t ws_bytes, void* stream,
                 int* final_in_b, cudaEvent_t* events = nullptr, R* cols = nullptr, int* cols_done = nullptr,
                 R* cols_out = nullptr) {
  if (steps < 1) return fail(NB_ERR_ARG, "steps must be >= 1");
  if (!(dt > 0.0)) return fail(NB_ERR_ARG, "dt must be positive");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cols_done) *cols_done = 0;
  if (!events && n <= small_max_n((int)sizeof(R))) {
    // small N: whole loop in one cooperative launch, source split inside the CTA
    StepArgs<R> a;
    int rc = make_step_args<R>(a, pos_a, n, 0, n, 0, n, g, eps2, dt, NB_STEP_FIRST, flags, nullptr, 0, acc4, vel4,
                               pos_b, ws, ws_bytes, stream, nullptr, 0);
    NB_HT(8);
    if (rc && rc != -1) return rc;
    if (rc == 0) {
      cudaError_t e = launch_simulate_small<R>(a, flags & (NB_FLAG_EXCLUDE_SELF | NB_FLAG_UNIFORM_MASS),
                                               static_cast<V4<R>*>(pos_a), static_cast<V4<R>*>(pos_b), steps, st,
                                               cols, cols_out);
      NB_HT(9);
      if (e == cudaSuccess) {
        if (final_in_b) *final_in_b = (steps & 1) ? 1 : 0;
        if (cols_done) *cols_done = cols ? (cols_out ? 2 : 1) : 0;
        return NB_OK;
      }
      if (e != cudaErrorCooperativeLaunchTooLarge && e != cudaErrorNotSupported)
        return cuda_fail(e, "small_simulate_kernel");
      cudaGetLastError();  // fall through to the stream-K paths
    }
  }
  if (cols) {  // the stream-K paths read the packed rows
    NB_CUDA(launch_pack_soa<R>(cols, cols + n, cols + 2 * n, cols + 3 * n, static_cast<V4<R>*>(pos_a), n, st));
    NB_CUDA(launch_pack_soa<R>(cols + 4 * n, cols + 5 * n, cols + 6 * n, nullptr, static_cast<V4<R>*>(vel4), n, st));
  }
  // (FP32 sizes the cluster split-source kernel covers go per step: it has no
  // partial slots, fixup pass or grid barriers to pay per step.)
  if (!events && n <= persistent_max_n() && strcmp(step_kernel_name<R>(n, n), "pair_kernel") != 0) {
    // small N: the whole loop in one cooperative launch (launch-bound otherwise)
    StepArgs<R> a;
    int rc = make_step_args<R>(a, pos_a, n, 0, n, 0, n, g, eps2, dt, NB_STEP_FIRST, flags, nullptr, 0, acc4, vel4,
                               pos_b, ws, ws_bytes, stream, nullptr, 0);
    if (rc && rc != -1) return rc;
    if (rc == 0) {
      cudaError_t e = launch_simulate_persistent<R>(a, flags & (NB_FLAG_EXCLUDE_SELF | NB_FLAG_UNIFORM_MASS),
                                                    static_cast<V4<R>*>(pos_a), static_cast<V4<R>*>(pos_b), steps, st);
      if (e == cudaSuccess) {
        if (final_in_b) *final_in_b = (steps & 1) ? 1 : 0;
        return NB_OK;
      }
      if (e != cudaErrorCooperativeLaunchTooLarge && e != cudaErrorNotSupported) return cuda_fail(e, "simulate_kernel");
      cudaGetLastError();  // fall through to per-step launches
    }
  }
  void* cur = pos_a;
  void* nxt = pos_b;
  for (int64_t s = 0; s < steps; ++s) {
    const int mode = s == 0 ? NB_STEP_FIRST : NB_STEP_KICK_DRIFT;
    if (events) NB_CUDA(cudaEventRecord(events[s], st));
    int rc = dev_step<R>(cur, n, 0, n, 0, n, g, eps2, dt, mode, flags, nullptr, 0, acc4, vel4, nxt, ws,
                         ws_bytes, stream);
    if (rc) return rc;
    void* t = cur; cur = nxt; nxt = t;
  }
  if (events) NB_CUDA(cudaEventRecord(events[steps], st));
  int rc = dev_step<R>(cur, n, 0, n, 0, n, g, eps2, dt, NB_STEP_FINAL_KICK, flags, nullptr, 0, acc4,
                       vel4, nullptr, ws, ws_bytes, stream);
  if (rc) return rc;
  if (events) NB_CUDA(cudaEventRecord(events[steps + 1], st));
  if (final_in_b) *final_in_b = cur == pos_b ? 1 : 0;
  return NB_OK;
}

template <typename R>
int dev_simulate_timed(void* pos_a, void* pos_b, void* vel4, void* acc4, int64_t n, double g, double dt,
                       double eps2, int64_t steps, int flags, void* ws, int64_t ws_bytes, void* stream,
                       int* final_in_b, float* launch_ms) {
  if (steps < 1) return fail(NB_ERR_ARG, "steps must be >= 1");
  if (!launch_ms) return fail(NB_ERR_ARG, "launch_ms must hold steps+1 floats");
  if (!pos_a) return fail(NB_ERR_ARG, "null device pointer");
  if (cudaError_t be = bind_device_of(pos_a)) return cuda_fail(be, "pos4 is not a device pointer");
  std::vector<cudaEvent_t> ev((size_t)steps + 2);
  for (auto& e : ev) NB_CUDA(cudaEventCreate(&e));
  int rc = dev_simulate<R>(pos_a, pos_b, vel4, acc4, n, g, dt, eps2, steps, flags, ws, ws_bytes, stream,
                           final_in_b, ev.data());
  if (!rc) {
    cudaError_t e = cudaEventSynchronize(ev.back());
    for (int64_t k = 0; k <= steps && e == cudaSuccess; ++k) e = cudaEventElapsedTime(&launch_ms[k], ev[k], ev[k + 1]);
    if (e != cudaSuccess) rc = cuda_fail(e, "event timing");
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

// Kernel flags for a host system: NB_FLAG_EXCLUDE_SELF unless the self pair
// adds exactly 0 ((R)eps2 > 0 and the largest self term m*eps2^-1.5 is finite
// with margin, else 0*inf = NaN), and NB_FLAG_UNIFORM_MASS when all masses are
// equal (m is then applied once per body instead of once per pair).
template <typename R>
int host_flags(const R* m, int64_t n, double eps2) {
  const double e = (double)(R)eps2;
  double mmax = 0.0;
  bool uniform = true;
  for (int64_t i = 0; i < n; ++i) {
    mmax = m[i] > mmax ? (double)m[i] : mmax;
    uniform = uniform && m[i] == m[0];
  }
  const double big = sizeof(R) == 4 ? 1e30 : 1e300;
  // Uniform-mass kernels form eps2^-1.5 without m (m is applied once per body),
  // so the test uses max(mmax, 1): a small uniform mass must not hide an
  // overflowing self term.
  const double mt = mmax > 1.0 ? mmax : 1.0;
  const bool mask = !(e > 0.0) || !(mt * (1.0 / e) / std::sqrt(e) < big);
  return (mask ? NB_FLAG_EXCLUDE_SELF : 0) | (uniform ? NB_FLAG_UNIFORM_MASS : 0);
}

// Device buffers of the synchronous host entry points (nb_host_*), kept between
// calls per device and only ever grown: a plugin-style caller (one
// accel_soa per force evaluation) pays no cudaMalloc/cudaFree per call.  One
// host call at a time (the mutex is held for the whole call).
struct Arena {
  void* p[12] = {};
  size_t cap[12] = {};
  void* host = nullptr;  // pinned staging: each call's uploads (and then downloads) as one block
  size_t host_cap = 0;
  // nb_host_simulate's own non-blocking stream: a launch on the legacy stream 0
  // costs ~1.6 us more host time (tools/api_cost.cu), which is on C1's path.
  cudaStream_t stream = nullptr;
};
std::mutex g_arena_mu;
Arena g_arenas[32];

struct DevBufs {
  std::lock_guard<std::mutex> lock{g_arena_mu};
  Arena* A = nullptr;
  int n = 0;
  cudaError_t err = cudaSuccess;
  DevBufs() {
    int d = 0;
    err = cudaGetDevice(&d);
    A = &g_arenas[(unsigned)d % 32u];
  }
  void* alloc(size_t bytes) {
    if (err != cudaSuccess || n >= 12) {
      if (err == cudaSuccess) err = cudaErrorMemoryAllocation;
      return nullptr;
    }
    if (bytes == 0) bytes = 16;
    const int k = n++;
    if (A->cap[k] < bytes) {
      if (A->p[k]) cudaFree(A->p[k]);
      A->p[k] = nullptr;
      A->cap[k] = 0;
      err = cudaMalloc(&A->p[k], bytes);
      if (err != cudaSuccess) return nullptr;
      A->cap[k] = bytes;
    }
    return A->p[k];
  }
  cudaStream_t stream() {
    if (err == cudaSuccess && !A->stream) err = cudaStreamCreateWithFlags(&A->stream, cudaStreamNonBlocking);
    return A->stream;
  }
  void* pinned(size_t bytes) {
    if (err != cudaSuccess) return nullptr;
    if (A->host_cap < bytes) {
      if (A->host) cudaFreeHost(A->host);
      A->host = nullptr;
      A->host_cap = 0;
      err = cudaMallocHost(&A->host, bytes);
      if (err != cudaSuccess) return nullptr;
      A->host_cap = bytes;
    }
    return A->host;
  }
};

// One upload of `k` host columns (n elements each, or 3n for an (n,3) AoS block
// when counts[c] == 3) through the pinned staging into consecutive device
// columns at d0; and one download of consecutive device columns.  Stream 0,
// synchronous where the host reads back.
template <typename R>
int upload_cols(DevBufs& B, R* d0, const R* const* cols, const int* counts, int k, int64_t n) {
  size_t total = 0;
  for (int c = 0; c < k; ++c) total += (size_t)counts[c] * n;
  R* h = static_cast<R*>(B.pinned(total * sizeof(R)));
  if (!h) return cuda_fail(B.err, "cudaMallocHost");
  size_t off = 0;
  for (int c = 0; c < k; ++c) {
    std::memcpy(h + off, cols[c], (size_t)counts[c] * n * sizeof(R));
    off += (size_t)counts[c] * n;
  }
  NB_CUDA(cudaMemcpyAsync(d0, h, total * sizeof(R), cudaMemcpyHostToDevice, 0));
  return NB_OK;
}
template <typename R>
int download_cols(DevBufs& B, const R* d0, R* const* cols, const int* counts, int k, int64_t n) {
  size_t total = 0;
  for (int c = 0; c < k; ++c) total += (size_t)counts[c] * n;
  NB_CUDA(cudaStreamSynchronize(0));  // every upload from the staging has landed
  R* h = static_cast<R*>(B.pinned(total * sizeof(R)));
  if (!h) return cuda_fail(B.err, "cudaMallocHost");
  NB_CUDA(cudaMemcpyAsync(h, d0, total * sizeof(R), cudaMemcpyDeviceToHost, 0));
  NB_CUDA(cudaStreamSynchronize(0));
  size_t off = 0;
  for (int c = 0; c < k; ++c) {
    std::memcpy(cols[c], h + off, (size_t)counts[c] * n * sizeof(R));
    off += (size_t)counts[c] * n;
  }
  return NB_OK;
}


template <typename R>
int host_accel(const R* px, const R* py, const R* pz, const R* pos_aos, const R* m, int64_t n, double g,
               double eps2, R* ax, R* ay, R* az) {
  if (n < 1) return fail(NB_ERR_ARG, "n must be >= 1");
  if (!m || !ax || !ay || !az || (!pos_aos && (!px || !py || !pz))) return fail(NB_ERR_ARG, "null host pointer");
  DevBufs B;
  void* dpos = B.alloc(sizeof(V4<R>) * n);
  void* dacc = B.alloc(sizeof(V4<R>) * n);
  void* dx = B.alloc(sizeof(R) * 4 * n);
  const int64_t wsb = step_workspace_bytes<R>(n);
  void* ws = B.alloc(wsb);  // scratch: no initialisation needed
  if (B.err != cudaSuccess) return cuda_fail(B.err, "cudaMalloc");
  R* d0 = static_cast<R*>(dx);
  int rc;
  if (pos_aos) {
    const R* cols[2] = {pos_aos, m};
    const int counts[2] = {3, 1};
    if ((rc = upload_cols<R>(B, d0, cols, counts, 2, n))) return rc;
    NB_CUDA(launch_pack_aos<R>(d0, d0 + 3 * n, static_cast<V4<R>*>(dpos), n, 0));
  } else {
    const R* cols[4] = {px, py, pz, m};
    const int counts[4] = {1, 1, 1, 1};
    if ((rc = upload_cols<R>(B, d0, cols, counts, 4, n))) return rc;
    NB_CUDA(launch_pack_soa<R>(d0, d0 + n, d0 + 2 * n, d0 + 3 * n, static_cast<V4<R>*>(dpos), n, 0));
  }
  if ((rc = dev_step<R>(dpos, n, 0, n, 0, n, g, eps2, 0.0, NB_MODE_ACCEL, host_flags<R>(m, n, eps2),
                        nullptr, 0, dacc, nullptr, nullptr, ws, wsb, nullptr)))
    return rc;
  NB_CUDA(launch_unpack_soa<R>(static_cast<V4<R>*>(dacc), d0, d0 + n, d0 + 2 * n, n, 0));
  R* out[3] = {ax, ay, az};
  const int counts[3] = {1, 1, 1};
  return download_cols<R>(B, d0, out, counts, 3, n);
}

template <typename R>
int host_step(R* px, R* py, R* pz, R* vx, R* vy, R* vz, R* pos_aos, R* vel_aos, const R* ax, const R* ay,
              const R* az, int64_t n, double dt) {
  if (n < 1) return fail(NB_ERR_ARG, "n must be >= 1");
  if (!ax || !ay || !az) return fail(NB_ERR_ARG, "null host pointer");
  if (pos_aos ? !vel_aos : (!px || !py || !pz || !vx || !vy || !vz)) return fail(NB_ERR_ARG, "null host pointer");
  DevBufs B;
  void* dpos = B.alloc(sizeof(V4<R>) * n);
  void* dvel = B.alloc(sizeof(V4<R>) * n);
  void* dacc = B.alloc(sizeof(V4<R>) * n);
  void* dx = B.alloc(sizeof(R) * 9 * n);
  if (B.err != cudaSuccess) return cuda_fail(B.err, "cudaMalloc");
  R* d0 = static_cast<R*>(dx);
  V4<R>* P = static_cast<V4<R>*>(dpos);
  V4<R>* V = static_cast<V4<R>*>(dvel);
  V4<R>* A = static_cast<V4<R>*>(dacc);
  int rc;
  // one upload: a (SoA) then positions and velocities (SoA columns or (n,3) blocks)
  if (pos_aos) {
    const R* cols[5] = {ax, ay, az, pos_aos, vel_aos};
    const int counts[5] = {1, 1, 1, 3, 3};
    if ((rc = upload_cols<R>(B, d0, cols, counts, 5, n))) return rc;
    NB_CUDA(launch_pack_aos<R>(d0 + 3 * n, nullptr, P, n, 0));
    NB_CUDA(launch_pack_aos<R>(d0 + 6 * n, nullptr, V, n, 0));
  } else {
    const R* cols[9] = {ax, ay, az, px, py, pz, vx, vy, vz};
    const int counts[9] = {1, 1, 1, 1, 1, 1, 1, 1, 1};
    if ((rc = upload_cols<R>(B, d0, cols, counts, 9, n))) return rc;
    NB_CUDA(launch_pack_soa<R>(d0 + 3 * n, d0 + 4 * n, d0 + 5 * n, nullptr, P, n, 0));
    NB_CUDA(launch_pack_soa<R>(d0 + 6 * n, d0 + 7 * n, d0 + 8 * n, nullptr, V, n, 0));
  }
  NB_CUDA(launch_pack_soa<R>(d0, d0 + n, d0 + 2 * n, nullptr, A, n, 0));
  NB_CUDA(launch_drift<R>(P, V, A, n, dt, 0));
  // one download: positions then velocities
  if (pos_aos) {
    NB_CUDA(launch_unpack_aos<R>(P, d0, n, 0));
    NB_CUDA(launch_unpack_aos<R>(V, d0 + 3 * n, n, 0));
    R* out[2] = {pos_aos, vel_aos};
    const int counts[2] = {3, 3};
    return download_cols<R>(B, d0, out, counts, 2, n);
  }
  NB_CUDA(launch_unpack_soa<R>(P, d0, d0 + n, d0 + 2 * n, n, 0));
  NB_CUDA(launch_unpack_soa<R>(V, d0 + 3 * n, d0 + 4 * n, d0 + 5 * n, n, 0));
  R* out[6] = {px, py, pz, vx, vy, vz};
  const int counts[6] = {1, 1, 1, 1, 1, 1};
  return download_cols<R>(B, d0, out, counts, 6, n);
}

// Whole simulate from host columns (inputs x, y, z, m, vx, vy, vz; outputs
// x, y, z, vx, vy, vz -- may alias the inputs).  One staging memcpy into the
// arena's pinned block, one H2D; at small N the simulate kernel reads the
// device column block itself and stores the final columns straight into the
// pinned block through its device mapping (no pack/unpack launches, no D2H);
// then one memcpy out.  Stream 0, synchronous.
template <typename R>
int host_simulate(const R* px, const R* py, const R* pz, const R* m, const R* vx, const R* vy, const R* vz,
                  int64_t n, double g, double dt, double eps2, int64_t steps, R* ox, R* oy, R* oz, R* ovx,
                  R* ovy, R* ovz) {
  if (n < 1) return fail(NB_ERR_ARG, "n must be >= 1");
  if (!px || !py || !pz || !vx || !vy || !vz || !m || !ox || !oy || !oz || !ovx || !ovy || !ovz)
    return fail(NB_ERR_ARG, "null host pointer");
  NB_HT(0);
  DevBufs B;
  void* pa = B.alloc(sizeof(V4<R>) * n);
  void* pb = B.alloc(sizeof(V4<R>) * n);
  void* dv = B.alloc(sizeof(V4<R>) * n);
  void* da = B.alloc(sizeof(V4<R>) * n);
  void* dx = B.alloc(sizeof(R) * 7 * n);
  const int64_t wsb = step_workspace_bytes<R>(n);
  void* ws = B.alloc(wsb);  // scratch: no initialisation needed
  if (B.err != cudaSuccess) return cuda_fail(B.err, "cudaMalloc");
  R* d0 = static_cast<R*>(dx);
  R* h = static_cast<R*>(B.pinned(sizeof(R) * 7 * n));
  if (!h) return cuda_fail(B.err, "cudaMallocHost");
  cudaStream_t st = B.stream();
  if (!st) return cuda_fail(B.err, "cudaStreamCreate");
  NB_HT(1);
  const R* cols[7] = {px, py, pz, m, vx, vy, vz};
  for (int c = 0; c < 7; ++c) std::memcpy(h + c * n, cols[c], sizeof(R) * n);
  NB_HT(2);
  R* hdev = nullptr;  // the pinned block's device mapping (UVA)
  if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&hdev), h, 0) != cudaSuccess) {
    cudaGetLastError();
    hdev = nullptr;
  }
  const bool small = steps >= 1 && dt > 0.0 && g == g && eps2 >= 0.0 && n <= small_max_n((int)sizeof(R));
  // (An H2D copy: reading the columns through the mapping inside the kernel
  // measured no faster at C1 -- the copy overlaps the launch's host time.)
  NB_CUDA(cudaMemcpyAsync(d0, h, sizeof(R) * 7 * n, cudaMemcpyHostToDevice, st));
  int in_b = 0, done = 0, rc;
  const int flags = host_flags<R>(m, n, eps2);
  NB_HT(3);
  bool launched = false;
  if (small) {
    // every buffer is this call's own: the small-N launch without re-validation
    StepArgs<R> a;
    fill_step_args<R>(a, pa, n, 0, n, 0, n, g, eps2, dt, NB_STEP_FIRST, nullptr, 0, da, dv, pb, ws, nullptr, 0);
    NB_HT(8);
    const cudaError_t e = launch_simulate_small<R>(a, flags, static_cast<V4<R>*>(pa), static_cast<V4<R>*>(pb), steps,
                                                   st, d0, hdev);
    NB_HT(9);
    if (e == cudaSuccess) {
      launched = true;
      in_b = (steps & 1) ? 1 : 0;
      done = hdev ? 2 : 1;
    } else if (e != cudaErrorCooperativeLaunchTooLarge && e != cudaErrorNotSupported) {
      return cuda_fail(e, "small_simulate_kernel");
    } else {
      cudaGetLastError();
    }
  }
  if (!launched && (rc = dev_simulate<R>(pa, pb, dv, da, n, g, dt, eps2, steps, flags, ws, wsb, st, &in_b,
                                         nullptr, d0, &done, hdev)))
    return rc;
  NB_HT(4);
  if (!done) {
    NB_CUDA(launch_unpack_soa<R>(static_cast<V4<R>*>(in_b ? pb : pa), d0, d0 + n, d0 + 2 * n, n, st));
    NB_CUDA(launch_unpack_soa<R>(static_cast<V4<R>*>(dv), d0 + 4 * n, d0 + 5 * n, d0 + 6 * n, n, st));
  }
  if (done != 2) NB_CUDA(cudaMemcpyAsync(h, d0, sizeof(R) * 7 * n, cudaMemcpyDeviceToHost, st));
  NB_HT(5);
  NB_CUDA(cudaStreamSynchronize(st));
  NB_HT(6);
  R* outs[7] = {ox, oy, oz, nullptr, ovx, ovy, ovz};
  for (int c = 0; c < 7; ++c)
    if (outs[c]) std::memcpy(outs[c], h + c * n, sizeof(R) * n);
  NB_HT(7);
  return NB_OK;
}

template <typename R>
int dev_pack(const void* x, const void* y, const void* z, const void* w, int64_t n, void* out4, void* stream) {
  if (n < 0) return fail(NB_ERR_ARG, "n must be >= 0");
  if (n == 0) return NB_OK;
  if (!x || !y || !z || !out4) return fail(NB_ERR_ARG, "null device pointer");
  if (cudaError_t be = bind_device_of(out4)) return cuda_fail(be, "out4 is not a device pointer");
  NB_CUDA(launch_pack_soa<R>(static_cast<const R*>(x), static_cast<const R*>(y), static_cast<const R*>(z),
                             static_cast<const R*>(w), static_cast<V4<R>*>(out4), n,
                             static_cast<cudaStream_t>(stream)));
  return NB_OK;
}

template <typename R>
int dev_unpack(const void* in4, int64_t n, void* x, void* y, void* z, void* stream) {
  if (n < 0) return fail(NB_ERR_ARG, "n must be >= 0");
  if (n == 0) return NB_OK;
  if (!in4 || !x || !y || !z) return fail(NB_ERR_ARG, "null device pointer");
  if (cudaError_t be = bind_device_of(in4)) return cuda_fail(be, "in4 is not a device pointer");
  NB_CUDA(launch_unpack_soa<R>(static_cast<const V4<R>*>(in4), static_cast<R*>(x), static_cast<R*>(y),
                               static_cast<R*>(z), n, static_cast<cudaStream_t>(stream)));
  return NB_OK;
}

// SURVEY.md 8(b)'s proposed minimal surface: the force pass alone and the update
// alone (the product path fuses them; these serve hosts that schedule the two).
// The masses are device-resident here, so whether the self term m*eps2^-1.5
// would overflow cannot be decided on the host: the self pair is always masked
// (one select per pair; a masked self pair and an unmasked finite one both add
// exactly 0, so the result equals the fused path's whenever that is finite).
template <typename R>
int dev_force(const void* pos_all, int64_t n_all, int64_t i_begin, int64_t n_i, double eps2, double g,
              void* acc_out, void* workspace, int64_t workspace_bytes, void* stream) {
  const int flags = NB_FLAG_EXCLUDE_SELF;
  return dev_step<R>(pos_all, n_all, i_begin, n_i, 0, n_all, g, eps2, 0.0, NB_MODE_ACCEL, flags, nullptr, 0,
                     acc_out, nullptr, nullptr, workspace, workspace_bytes, stream);
}

template <typename R>
int dev_update(void* pos_next, const void* pos_cur, void* vel, const void* acc, const void* acc_prev, int64_t n_i,
               double dt, int mode, void* stream) {
  if (n_i < 0) return fail(NB_ERR_ARG, "n_i must be >= 0");
  if (mode < NB_STEP_FIRST || mode > NB_STEP_FINAL_KICK) return fail(NB_ERR_ARG, "mode must be an NB_STEP_* mode");
  if (!(dt > 0.0)) return fail(NB_ERR_ARG, "dt must be positive");
  if (n_i == 0) return NB_OK;
  if (!pos_next || !pos_cur || !vel || !acc || (mode != NB_STEP_FIRST && !acc_prev))
    return fail(NB_ERR_ARG, "null device pointer");
  if (cudaError_t be = bind_device_of(vel)) return cuda_fail(be, "vel4 is not a device pointer");
  NB_CUDA(launch_update<R>(static_cast<V4<R>*>(pos_next), static_cast<const V4<R>*>(pos_cur),
                           static_cast<V4<R>*>(vel), static_cast<const V4<R>*>(acc),
                           static_cast<const V4<R>*>(acc_prev), n_i, dt, mode, static_cast<cudaStream_t>(stream)));
  return NB_OK;
}

// Column block of simulate()'s staging (header: nb_dev_load_cols_*).
template <typename R>
int dev_load_cols(const void* host_cols, void* dev_cols, int64_t n, int64_t n_i, void* pos4, void* vel4,
                  void* stream) {
  if (n < 1 || n_i < 0 || n_i > n) return fail(NB_ERR_ARG, "need n >= 1 and 0 <= n_i <= n");
  if (!host_cols || !dev_cols || !pos4 || (n_i && !vel4)) return fail(NB_ERR_ARG, "null pointer");
  if (!aligned16(pos4) || (n_i && !aligned16(vel4))) return fail(NB_ERR_ARG, "pos4/vel4 must be 16-byte aligned");
  if (cudaError_t be = bind_device_of(pos4)) return cuda_fail(be, "pos4 is not a device pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t ni = n_i > 0 ? n_i : 1;
  R* d = static_cast<R*>(dev_cols);
  NB_CUDA(cudaMemcpyAsync(d, host_cols, (size_t)(4 * n + 3 * ni) * sizeof(R), cudaMemcpyHostToDevice, st));
  NB_CUDA(launch_pack_soa<R>(d, d + n, d + 2 * n, d + 3 * n, static_cast<V4<R>*>(pos4), n, st));
  if (n_i)
    NB_CUDA(launch_pack_soa<R>(d + 4 * n, d + 4 * n + ni, d + 4 * n + 2 * ni, nullptr, static_cast<V4<R>*>(vel4),
                               n_i, st));
  return NB_OK;
}

template <typename R>
int dev_store_cols(const void* pos4, const void* vel4, int64_t n, int64_t n_i, void* dev_cols, void* host_cols,
                   void* stream) {
  if (n < 1 || n_i < 0 || n_i > n) return fail(NB_ERR_ARG, "need n >= 1 and 0 <= n_i <= n");
  if (!host_cols || !dev_cols || !pos4 || (n_i && !vel4)) return fail(NB_ERR_ARG, "null pointer");
  if (cudaError_t be = bind_device_of(pos4)) return cuda_fail(be, "pos4 is not a device pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t ni = n_i > 0 ? n_i : 1;
  R* d = static_cast<R*>(dev_cols);
  NB_CUDA(launch_unpack_soa<R>(static_cast<const V4<R>*>(pos4), d, d + n, d + 2 * n, n, st));
  if (n_i)
    NB_CUDA(launch_unpack_soa<R>(static_cast<const V4<R>*>(vel4), d + 4 * n, d + 4 * n + ni, d + 4 * n + 2 * ni,
                                 n_i, st));
  R* h = static_cast<R*>(host_cols);
  NB_CUDA(cudaMemcpyAsync(h, d, (size_t)(3 * n) * sizeof(R), cudaMemcpyDeviceToHost, st));  // x, y, z
  if (n_i)
    NB_CUDA(cudaMemcpyAsync(h + 4 * n, d + 4 * n, (size_t)(3 * ni) * sizeof(R), cudaMemcpyDeviceToHost, st));
  NB_CUDA(cudaStreamSynchronize(st));
  return NB_OK;
}

template <typename R>
int dev_simulate_cols(const void* host_cols, void* dev_cols, void* pos_a, void* pos_b, void* vel4, void* acc4,
                      int64_t n, double g, double dt, double eps2, int64_t steps, int flags, void* ws,
                      int64_t ws_bytes, void* stream, int* final_in_b) {
  // One H2D of the column block; the simulate reads it directly (small N) or
  // packs it itself; then the unpack (if the simulate did not write the columns)
  // and one D2H of positions and velocities.
  NB_HT(0);
  if (n < 1) return fail(NB_ERR_ARG, "need n >= 1");
  if (!host_cols || !dev_cols || !pos_a || !pos_b || !vel4 || !acc4) return fail(NB_ERR_ARG, "null pointer");
  if (!aligned16(pos_a) || !aligned16(vel4)) return fail(NB_ERR_ARG, "pos4/vel4 must be 16-byte aligned");
  if (cudaError_t be = bind_device_of(pos_a)) return cuda_fail(be, "pos4 is not a device pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  R* d = static_cast<R*>(dev_cols);
  NB_HT(1);
  NB_CUDA(cudaMemcpyAsync(d, host_cols, (size_t)(7 * n) * sizeof(R), cudaMemcpyHostToDevice, st));
  NB_HT(2);
  if (flags & NB_FLAG_AUTO)  // (while the copy runs) the flags of the staged masses
    flags = (flags & ~(NB_FLAG_AUTO | NB_FLAG_EXCLUDE_SELF | NB_FLAG_UNIFORM_MASS)) |
            host_flags<R>(static_cast<const R*>(host_cols) + 3 * n, n, eps2);
  // A pinned host block is mapped into the device's address space (UVA): the
  // small-N kernel then stores the final columns straight into it, and no D2H
  // copy follows (done == 2).
  R* hdev = nullptr;
  if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&hdev), const_cast<void*>(host_cols), 0) != cudaSuccess) {
    cudaGetLastError();
    hdev = nullptr;
  }
  int in_b = 0, done = 0;
  NB_HT(3);
  int rc = dev_simulate<R>(pos_a, pos_b, vel4, acc4, n, g, dt, eps2, steps, flags, ws, ws_bytes, stream, &in_b,
                           nullptr, d, &done, hdev);
  NB_HT(4);
  if (rc) return rc;
  if (final_in_b) *final_in_b = in_b;
  if (!done) {
    NB_CUDA(launch_unpack_soa<R>(static_cast<const V4<R>*>(in_b ? pos_b : pos_a), d, d + n, d + 2 * n, n, st));
    NB_CUDA(launch_unpack_soa<R>(static_cast<const V4<R>*>(vel4), d + 4 * n, d + 5 * n, d + 6 * n, n, st));
  }
  // one D2H of the whole block (the masses ride along unchanged: one copy's
  // latency instead of two at small N)
  if (done != 2)
    NB_CUDA(cudaMemcpyAsync(const_cast<void*>(host_cols), d, (size_t)(7 * n) * sizeof(R), cudaMemcpyDeviceToHost,
                            st));
  NB_HT(5);
  NB_CUDA(cudaStreamSynchronize(st));
  NB_HT(6);
  return NB_OK;
}

template <typename R>
int dev_drift(void* pos4, void* vel4, const void* acc4, int64_t n, double dt, void* stream) {
  if (n < 0) return fail(NB_ERR_ARG, "n must be >= 0");
  if (n == 0) return NB_OK;
  if (!pos4 || !vel4 || !acc4) return fail(NB_ERR_ARG, "null device pointer");
  if (cudaError_t be = bind_device_of(pos4)) return cuda_fail(be, "pos4 is not a device pointer");
  NB_CUDA(launch_drift<R>(static_cast<V4<R>*>(pos4), static_cast<V4<R>*>(vel4), static_cast<const V4<R>*>(acc4), n,
                          dt, static_cast<cudaStream_t>(stream)));
  return NB_OK;
}

template <typename R>
int dev_kick(void* vel4, const void* an, const void* ao, int64_t n, double factor, void* stream) {
  if (n < 0) return fail(NB_ERR_ARG, "n must be >= 0");
  if (n == 0) return NB_OK;
  if (!vel4 || !an || !ao) return fail(NB_ERR_ARG, "null device pointer");
  if (cudaError_t be = bind_device_of(vel4)) return cuda_fail(be, "vel4 is not a device pointer");
  NB_CUDA(launch_kick<R>(static_cast<V4<R>*>(vel4), static_cast<const V4<R>*>(an), static_cast<const V4<R>*>(ao), n,
                         factor, static_cast<cudaStream_t>(stream)));
  return NB_OK;
}

template <typename R>
int dev_energy(const void* pos4, const void* vel4, int64_t n, double g, double eps2, double* out6, void* ws,
               int64_t ws_bytes, void* stream) {
  if (n < 1) return fail(NB_ERR_ARG, "n must be >= 1");
  if (!pos4 || !vel4 || !out6) return fail(NB_ERR_ARG, "null device pointer");
  if (cudaError_t be = bind_device_of(pos4)) return cuda_fail(be, "pos4 is not a device pointer");
  if (!ws || ws_bytes < 8 * n) return fail(NB_ERR_WORKSPACE, "energy needs a workspace of 8*n bytes");
  NB_CUDA(launch_energy<R>(static_cast<const V4<R>*>(pos4), static_cast<const V4<R>*>(vel4), n, g, eps2, out6,
                           static_cast<double*>(ws), ws_bytes / 8, static_cast<cudaStream_t>(stream)));
  return NB_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int nb_host_accel_soa_f32(const float* px, const float* py, const float* pz, const float* m, int64_t n, double g,
                          double eps2, int recip, int64_t block, int threads, float* ax, float* ay, float* az) {
  (void)recip; (void)block; (void)threads;
  return host_accel<float>(px, py, pz, nullptr, m, n, g, eps2, ax, ay, az);
}
int nb_host_accel_soa_f64(const double* px, const double* py, const double* pz, const double* m, int64_t n,
                          double g, double eps2, int recip, int64_t block, int threads, double* ax, double* ay,
                          double* az) {
  (void)recip; (void)block; (void)threads;
  return host_accel<double>(px, py, pz, nullptr, m, n, g, eps2, ax, ay, az);
}
int nb_host_accel_aos_f32(const float* pos, const float* m, int64_t n, double g, double eps2, float* ax, float* ay,
                          float* az) {
  if (!pos) return fail(NB_ERR_ARG, "null host pointer");
  return host_accel<float>(nullptr, nullptr, nullptr, pos, m, n, g, eps2, ax, ay, az);
}
int nb_host_accel_aos_f64(const double* pos, const double* m, int64_t n, double g, double eps2, double* ax,
                          double* ay, double* az) {
  if (!pos) return fail(NB_ERR_ARG, "null host pointer");
  return host_accel<double>(nullptr, nullptr, nullptr, pos, m, n, g, eps2, ax, ay, az);
}
int nb_host_step_soa_f32(float* px, float* py, float* pz, float* vx, float* vy, float* vz, const float* ax,
                         const float* ay, const float* az, int64_t n, double dt, int threads) {
  (void)threads;
  return host_step<float>(px, py, pz, vx, vy, vz, nullptr, nullptr, ax, ay, az, n, dt);
}
int nb_host_step_soa_f64(double* px, double* py, double* pz, double* vx, double* vy, double* vz, const double* ax,
                         const double* ay, const double* az, int64_t n, double dt, int threads) {
  (void)threads;
  return host_step<double>(px, py, pz, vx, vy, vz, nullptr, nullptr, ax, ay, az, n, dt);
}
int nb_host_step_aos_f32(float* pos, float* vel, const float* ax, const float* ay, const float* az, int64_t n,
                         double dt) {
  if (!pos) return fail(NB_ERR_ARG, "null host pointer");
  return host_step<float>(nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, pos, vel, ax, ay, az, n, dt);
}
int nb_host_step_aos_f64(double* pos, double* vel, const double* ax, const double* ay, const double* az, int64_t n,
                         double dt) {
  if (!pos) return fail(NB_ERR_ARG, "null host pointer");
  return host_step<double>(nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, pos, vel, ax, ay, az, n, dt);
}
int nb_host_simulate_soa_f32(float* px, float* py, float* pz, float* vx, float* vy, float* vz, const float* m,
                             int64_t n, double g, double dt, double eps2, int64_t steps) {
  return host_simulate<float>(px, py, pz, m, vx, vy, vz, n, g, dt, eps2, steps, px, py, pz, vx, vy, vz);
}
int nb_host_simulate_soa_f64(double* px, double* py, double* pz, double* vx, double* vy, double* vz,
                             const double* m, int64_t n, double g, double dt, double eps2, int64_t steps) {
  return host_simulate<double>(px, py, pz, m, vx, vy, vz, n, g, dt, eps2, steps, px, py, pz, vx, vy, vz);
}
int nb_host_simulate_f32(const float* px, const float* py, const float* pz, const float* m, const float* vx,
                         const float* vy, const float* vz, int64_t n, double g, double dt, double eps2,
                         int64_t steps, float* out6, int device) {
  if (!out6) return fail(NB_ERR_ARG, "null host pointer");
  if (device >= 0) {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != device) NB_CUDA(cudaSetDevice(device));
  }
  return host_simulate<float>(px, py, pz, m, vx, vy, vz, n, g, dt, eps2, steps, out6, out6 + n, out6 + 2 * n,
                              out6 + 3 * n, out6 + 4 * n, out6 + 5 * n);
}
int nb_host_simulate_f64(const double* px, const double* py, const double* pz, const double* m, const double* vx,
                         const double* vy, const double* vz, int64_t n, double g, double dt, double eps2,
                         int64_t steps, double* out6, int device) {
  if (!out6) return fail(NB_ERR_ARG, "null host pointer");
  if (device >= 0) {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != device) NB_CUDA(cudaSetDevice(device));
  }
  return host_simulate<double>(px, py, pz, m, vx, vy, vz, n, g, dt, eps2, steps, out6, out6 + n, out6 + 2 * n,
                               out6 + 3 * n, out6 + 4 * n, out6 + 5 * n);
}

int64_t nb_dev_workspace_bytes(int precision_bytes, int64_t n_i) {
  if (n_i < 1) n_i = 1;
  if (precision_bytes == 4) return step_workspace_bytes<float>(n_i);
  if (precision_bytes == 8) return step_workspace_bytes<double>(n_i);
  fail(NB_ERR_ARG, "precision_bytes must be 4 or 8");
  return -1;
}

const char* nb_dev_step_kernel(int precision_bytes, int64_t n_i, int64_t j_count) {
  if (precision_bytes == 4) return step_kernel_name<float>(n_i, j_count);
  if (precision_bytes == 8) return step_kernel_name<double>(n_i, j_count);
  fail(NB_ERR_ARG, "precision_bytes must be 4 or 8");
  return nullptr;
}

int64_t nb_energy_workspace_bytes(int precision_bytes, int64_t n) {
  if (n < 1) n = 1;
  if (precision_bytes != 4 && precision_bytes != 8) {
    fail(NB_ERR_ARG, "precision_bytes must be 4 or 8");
    return -1;
  }
  return 8 * energy_workspace_entries(precision_bytes, n);
}

int nb_dev_step_f32(const void* pos4, int64_t n_all, int64_t i_begin, int64_t n_i, int64_t j_begin, int64_t j_count,
                    double g, double eps2, double dt, int mode, int flags, double* carry, int carry_mode,
                    void* acc4, void* vel4, void* pos4_next, void* workspace, int64_t workspace_bytes,
                    void* stream) {
  return dev_step<float>(pos4, n_all, i_begin, n_i, j_begin, j_count, g, eps2, dt, mode, flags, carry,
                         carry_mode, acc4, vel4, pos4_next, workspace, workspace_bytes, stream);
}
int nb_dev_step_f64(const void* pos4, int64_t n_all, int64_t i_begin, int64_t n_i, int64_t j_begin, int64_t j_count,
                    double g, double eps2, double dt, int mode, int flags, double* carry, int carry_mode,
                    void* acc4, void* vel4, void* pos4_next, void* workspace, int64_t workspace_bytes,
                    void* stream) {
  return dev_step<double>(pos4, n_all, i_begin, n_i, j_begin, j_count, g, eps2, dt, mode, flags, carry,
                          carry_mode, acc4, vel4, pos4_next, workspace, workspace_bytes, stream);
}
int nb_dev_step_p2p_f32(const void* pos4, int64_t n_all, int64_t i_begin, int64_t n_i, int64_t j_begin,
                        int64_t j_count, double g, double eps2, double dt, int mode, int flags, double* carry,
                        int carry_mode, void* acc4, void* vel4, void* pos4_next, void* const* peer_pos4_next,
                        int n_peers, void* workspace, int64_t workspace_bytes, void* stream) {
  return dev_step<float>(pos4, n_all, i_begin, n_i, j_begin, j_count, g, eps2, dt, mode, flags, carry, carry_mode,
                         acc4, vel4, pos4_next, workspace, workspace_bytes, stream, peer_pos4_next, n_peers);
}
int nb_dev_step_p2p_f64(const void* pos4, int64_t n_all, int64_t i_begin, int64_t n_i, int64_t j_begin,
                        int64_t j_count, double g, double eps2, double dt, int mode, int flags, double* carry,
                        int carry_mode, void* acc4, void* vel4, void* pos4_next, void* const* peer_pos4_next,
                        int n_peers, void* workspace, int64_t workspace_bytes, void* stream) {
  return dev_step<double>(pos4, n_all, i_begin, n_i, j_begin, j_count, g, eps2, dt, mode, flags, carry, carry_mode,
                          acc4, vel4, pos4_next, workspace, workspace_bytes, stream, peer_pos4_next, n_peers);
}
int nb_dev_simulate_f32(void* pos4_a, void* pos4_b, void* vel4, void* acc4, int64_t n, double g, double dt,
                        double eps2, int64_t steps, int flags, void* workspace, int64_t workspace_bytes,
                        void* stream, int* final_in_b) {
  return dev_simulate<float>(pos4_a, pos4_b, vel4, acc4, n, g, dt, eps2, steps, flags, workspace,
                             workspace_bytes, stream, final_in_b);
}
int nb_dev_simulate_f64(void* pos4_a, void* pos4_b, void* vel4, void* acc4, int64_t n, double g, double dt,
                        double eps2, int64_t steps, int flags, void* workspace, int64_t workspace_bytes,
                        void* stream, int* final_in_b) {
  return dev_simulate<double>(pos4_a, pos4_b, vel4, acc4, n, g, dt, eps2, steps, flags, workspace,
                              workspace_bytes, stream, final_in_b);
}
int nb_dev_simulate_timed_f32(void* pos4_a, void* pos4_b, void* vel4, void* acc4, int64_t n, double g, double dt,
                              double eps2, int64_t steps, int flags, void* workspace, int64_t workspace_bytes,
                              void* stream, int* final_in_b, float* launch_ms) {
  return dev_simulate_timed<float>(pos4_a, pos4_b, vel4, acc4, n, g, dt, eps2, steps, flags, workspace,
                                   workspace_bytes, stream, final_in_b, launch_ms);
}
int nb_dev_simulate_timed_f64(void* pos4_a, void* pos4_b, void* vel4, void* acc4, int64_t n, double g, double dt,
                              double eps2, int64_t steps, int flags, void* workspace, int64_t workspace_bytes,
                              void* stream, int* final_in_b, float* launch_ms) {
  return dev_simulate_timed<double>(pos4_a, pos4_b, vel4, acc4, n, g, dt, eps2, steps, flags, workspace,
                                    workspace_bytes, stream, final_in_b, launch_ms);
}
int nb_dev_pack_f32(const void* x, const void* y, const void* z, const void* w, int64_t n, void* out4,
                    void* stream) {
  return dev_pack<float>(x, y, z, w, n, out4, stream);
}
int nb_dev_pack_f64(const void* x, const void* y, const void* z, const void* w, int64_t n, void* out4,
                    void* stream) {
  return dev_pack<double>(x, y, z, w, n, out4, stream);
}
int nb_dev_unpack_f32(const void* in4, int64_t n, void* x, void* y, void* z, void* stream) {
  return dev_unpack<float>(in4, n, x, y, z, stream);
}
int nb_dev_unpack_f64(const void* in4, int64_t n, void* x, void* y, void* z, void* stream) {
  return dev_unpack<double>(in4, n, x, y, z, stream);
}
int nb_force_f32(const void* pos_all, int64_t n_all, int64_t i_begin, int64_t n_i, double eps2, double g,
                 void* acc_out, void* workspace, int64_t workspace_bytes, void* stream) {
  return dev_force<float>(pos_all, n_all, i_begin, n_i, eps2, g, acc_out, workspace, workspace_bytes, stream);
}
int nb_force_f64(const void* pos_all, int64_t n_all, int64_t i_begin, int64_t n_i, double eps2, double g,
                 void* acc_out, void* workspace, int64_t workspace_bytes, void* stream) {
  return dev_force<double>(pos_all, n_all, i_begin, n_i, eps2, g, acc_out, workspace, workspace_bytes, stream);
}
int nb_update_f32(void* pos_next, const void* pos_cur, void* vel, const void* acc, const void* acc_prev,
                  int64_t n_i, double dt, int mode, void* stream) {
  return dev_update<float>(pos_next, pos_cur, vel, acc, acc_prev, n_i, dt, mode, stream);
}
int nb_update_f64(void* pos_next, const void* pos_cur, void* vel, const void* acc, const void* acc_prev,
                  int64_t n_i, double dt, int mode, void* stream) {
  return dev_update<double>(pos_next, pos_cur, vel, acc, acc_prev, n_i, dt, mode, stream);
}
int nb_dev_simulate_cols_f32(void* host_cols, void* dev_cols, void* pos_a, void* pos_b, void* vel4, void* acc4,
                             int64_t n, double g, double dt, double eps2, int64_t steps, int flags, void* ws,
                             int64_t ws_bytes, void* stream, int* final_in_b) {
  return dev_simulate_cols<float>(host_cols, dev_cols, pos_a, pos_b, vel4, acc4, n, g, dt, eps2, steps, flags, ws,
                                  ws_bytes, stream, final_in_b);
}
int nb_dev_simulate_cols_f64(void* host_cols, void* dev_cols, void* pos_a, void* pos_b, void* vel4, void* acc4,
                             int64_t n, double g, double dt, double eps2, int64_t steps, int flags, void* ws,
                             int64_t ws_bytes, void* stream, int* final_in_b) {
  return dev_simulate_cols<double>(host_cols, dev_cols, pos_a, pos_b, vel4, acc4, n, g, dt, eps2, steps, flags, ws,
                                   ws_bytes, stream, final_in_b);
}
int nb_dev_load_cols_f32(const void* host_cols, void* dev_cols, int64_t n, int64_t n_i, void* pos4, void* vel4,
                         void* stream) {
  return dev_load_cols<float>(host_cols, dev_cols, n, n_i, pos4, vel4, stream);
}
int nb_dev_load_cols_f64(const void* host_cols, void* dev_cols, int64_t n, int64_t n_i, void* pos4, void* vel4,
                         void* stream) {
  return dev_load_cols<double>(host_cols, dev_cols, n, n_i, pos4, vel4, stream);
}
int nb_dev_store_cols_f32(const void* pos4, const void* vel4, int64_t n, int64_t n_i, void* dev_cols,
                          void* host_cols, void* stream) {
  return dev_store_cols<float>(pos4, vel4, n, n_i, dev_cols, host_cols, stream);
}
int nb_dev_store_cols_f64(const void* pos4, const void* vel4, int64_t n, int64_t n_i, void* dev_cols,
                          void* host_cols, void* stream) {
  return dev_store_cols<double>(pos4, vel4, n, n_i, dev_cols, host_cols, stream);
}
int nb_dev_drift_f32(void* pos4, void* vel4, const void* acc4, int64_t n, double dt, void* stream) {
  return dev_drift<float>(pos4, vel4, acc4, n, dt, stream);
}
int nb_dev_drift_f64(void* pos4, void* vel4, const void* acc4, int64_t n, double dt, void* stream) {
  return dev_drift<double>(pos4, vel4, acc4, n, dt, stream);
}
int nb_dev_kick_f32(void* vel4, const void* an, const void* ao, int64_t n, double factor, void* stream) {
  return dev_kick<float>(vel4, an, ao, n, factor, stream);
}
int nb_dev_kick_f64(void* vel4, const void* an, const void* ao, int64_t n, double factor, void* stream) {
  return dev_kick<double>(vel4, an, ao, n, factor, stream);
}
int nb_dev_energy_f32(const void* pos4, const void* vel4, int64_t n, double g, double eps2, double* out6, void* ws,
                      int64_t ws_bytes, void* stream) {
  return dev_energy<float>(pos4, vel4, n, g, eps2, out6, ws, ws_bytes, stream);
}
int nb_dev_energy_f64(const void* pos4, const void* vel4, int64_t n, double g, double eps2, double* out6, void* ws,
                      int64_t ws_bytes, void* stream) {
  return dev_energy<double>(pos4, vel4, n, g, eps2, out6, ws, ws_bytes, stream);
}

static int dev_init(int precision_bytes, int kind, uint64_t seed, int64_t n, void* pos4, void* vel4, void* stream) {
  if (n < 1) return fail(NB_ERR_ARG, "n must be >= 1");
  if (kind != NB_INIT_UNIFORM_CUBE && kind != NB_INIT_PLUMMER) return fail(NB_ERR_ARG, "unknown generator kind");
  if (!pos4 || !vel4 || !aligned16(pos4) || !aligned16(vel4)) return fail(NB_ERR_ARG, "pos4/vel4 must be 16-byte aligned device pointers");
  if (cudaError_t be = bind_device_of(pos4)) return cuda_fail(be, "pos4 is not a device pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (precision_bytes == 4)
    NB_CUDA(launch_init<float>(kind, seed, n, static_cast<V4<float>*>(pos4), static_cast<V4<float>*>(vel4), st));
  else
    NB_CUDA(launch_init<double>(kind, seed, n, static_cast<V4<double>*>(pos4), static_cast<V4<double>*>(vel4), st));
  return NB_OK;
}
int nb_dev_init_f32(int kind, uint64_t seed, int64_t n, void* pos4, void* vel4, void* stream) {
  return dev_init(4, kind, seed, n, pos4, vel4, stream);
}
int nb_dev_init_f64(int kind, uint64_t seed, int64_t n, void* pos4, void* vel4, void* stream) {
  return dev_init(8, kind, seed, n, pos4, vel4, stream);
}

const char* nb_last_error(void) { return t_err.c_str(); }

#if NB_TRACE
// Trace builds only (tools/trace_launches.py): per-CTA timeline records.
__attribute__((visibility("default"))) int nb_trace_setup(void* buf, int64_t capacity) {
  return nb::trace_setup(buf, capacity);
}
__attribute__((visibility("default"))) int64_t nb_trace_count(void) { return nb::trace_count(); }
__attribute__((visibility("default"))) int nb_host_trace(double* out, int cap) {
  const int k = g_ht_n < cap ? g_ht_n : cap;
  for (int q = 0; q < k; ++q) out[q] = g_ht[q];
  return k;
}
#endif
// ---------------------------------------------------------------- position exchange (NCCL)
// The per-step exchange of SURVEY.md 8(e) behind the C ABI, for hosts that are
// not Python (the Python driver uses torch.distributed's NCCL): communicator
// set-up and the in-place all-gather of a rank's position rows.  NCCL is
// resolved at run time from "libnccl.so.2" -- the copy the host process already
// loaded (e.g. PyTorch's) when there is one -- so the library has no link-time
// NCCL dependency and never carries a second NCCL into the process.
namespace {
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommInitAll) comm_init_all = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclCommUserRank) comm_user_rank = nullptr;
  decltype(&ncclCommCount) comm_count = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  std::string error;
};

const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "unknown");
      return;
    }
#define NB_NCCL_SYM(field, name)                                        \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));     \
  if (!api.field) { api.error = std::string("libnccl.so.2 lacks ") + name; return; }
    NB_NCCL_SYM(get_unique_id, "ncclGetUniqueId");
    NB_NCCL_SYM(comm_init_rank, "ncclCommInitRank");
    NB_NCCL_SYM(comm_init_all, "ncclCommInitAll");
    NB_NCCL_SYM(all_gather, "ncclAllGather");
    NB_NCCL_SYM(comm_destroy, "ncclCommDestroy");
    NB_NCCL_SYM(comm_user_rank, "ncclCommUserRank");
    NB_NCCL_SYM(comm_count, "ncclCommCount");
    NB_NCCL_SYM(group_start, "ncclGroupStart");
    NB_NCCL_SYM(group_end, "ncclGroupEnd");
    NB_NCCL_SYM(error_string, "ncclGetErrorString");
#undef NB_NCCL_SYM
  });
  return api;
}

int nccl_fail(ncclResult_t r, const char* where) {
  const NcclApi& api = nccl_api();
  t_err = std::string(where) + ": " + (api.error_string ? api.error_string(r) : "nccl error");
  return NB_ERR_NCCL + (int)r;
}
#define NB_NCCL(call)                                        \
  do {                                                       \
    ncclResult_t r_ = (call);                                \
    if (r_ != ncclSuccess) return nccl_fail(r_, #call);      \
  } while (0)
#define NB_NCCL_API(api)                                                         \
  const NcclApi& api = nccl_api();                                               \
  if (!api.all_gather) return fail(NB_ERR_NCCL_MISSING, api.error)
}  // namespace

int nb_comm_unique_id(void* id_out) {
  if (!id_out) return fail(NB_ERR_ARG, "id_out must hold NB_COMM_ID_BYTES bytes");
  NB_NCCL_API(api);
  ncclUniqueId id;
  NB_NCCL(api.get_unique_id(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return NB_OK;
}

int nb_comm_init_rank(int nranks, int rank, const void* id, void** comm_out) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(NB_ERR_ARG, "need 0 <= rank < nranks");
  if (!id || !comm_out) return fail(NB_ERR_ARG, "null id or comm_out");
  NB_NCCL_API(api);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  NB_NCCL(api.comm_init_rank(&c, nranks, uid, rank));
  *comm_out = c;
  return NB_OK;
}

int nb_comm_init_all(int ndev, const int* devs, void** comms_out) {
  if (ndev < 1 || !comms_out) return fail(NB_ERR_ARG, "need ndev >= 1 and comms_out[ndev]");
  NB_NCCL_API(api);
  std::vector<ncclComm_t> c((size_t)ndev, nullptr);
  NB_NCCL(api.comm_init_all(c.data(), ndev, devs));
  for (int q = 0; q < ndev; ++q) comms_out[q] = c[q];
  return NB_OK;
}

int nb_comm_allgather(void* buf, size_t bytes_per_rank, void* comm, void* stream) {
  if (!buf || !comm) return fail(NB_ERR_ARG, "null buffer or communicator");
  NB_NCCL_API(api);
  int rank = 0;
  NB_NCCL(api.comm_user_rank(static_cast<ncclComm_t>(comm), &rank));
  char* b = static_cast<char*>(buf);
  NB_NCCL(api.all_gather(b + (size_t)rank * bytes_per_rank, b, bytes_per_rank, ncclChar,
                         static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream)));
  return NB_OK;
}

int nb_comm_allgather_all(void* const* bufs, size_t bytes_per_rank, void* const* comms, void* const* streams,
                          int ndev) {
  if (ndev < 1 || !bufs || !comms || !streams) return fail(NB_ERR_ARG, "need ndev >= 1 and bufs/comms/streams");
  NB_NCCL_API(api);
  NB_NCCL(api.group_start());
  for (int q = 0; q < ndev; ++q) {
    int rank = 0;
    ncclResult_t r = api.comm_user_rank(static_cast<ncclComm_t>(comms[q]), &rank);
    if (r == ncclSuccess) {
      char* b = static_cast<char*>(bufs[q]);
      r = api.all_gather(b + (size_t)rank * bytes_per_rank, b, bytes_per_rank, ncclChar,
                         static_cast<ncclComm_t>(comms[q]), static_cast<cudaStream_t>(streams[q]));
    }
    if (r != ncclSuccess) {
      api.group_end();
      return nccl_fail(r, "ncclAllGather");
    }
  }
  NB_NCCL(api.group_end());
  return NB_OK;
}

int nb_comm_destroy(void* comm) {
  if (!comm) return NB_OK;
  NB_NCCL_API(api);
  NB_NCCL(api.comm_destroy(static_cast<ncclComm_t>(comm)));
  return NB_OK;
}

#ifndef NB_SRC_DIGEST
#define NB_SRC_DIGEST "unknown"
#endif
// The digest of the sources this library was compiled from (_build.py passes it):
// a prebuilt .so that travelled with a snapshot cannot pass for a rebuild of
// different sources (_native.verify_build).
const char* nb_version(void) { return "nbody_b200 0.2.0 (sm_100a) src:" NB_SRC_DIGEST; }
int64_t nb_launch_count(void) { return g_launches.load(); }

}  // extern "C"
