// Internal interface between the C ABI (nbody_capi.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "nbody_common.cuh"

#if NB_TRACE
#include <chrono>
namespace nb {
// Trace builds: host timestamps (ns, steady clock) of the last host simulate
// call's phases (tools/host_trace.py); defined in nbody_capi.cu.
extern double g_ht[16];
extern int g_ht_n;
}  // namespace nb
#define NB_HT(k) (nb::g_ht[(k)] = (double)std::chrono::duration_cast<std::chrono::nanoseconds>( \
                      std::chrono::steady_clock::now().time_since_epoch()).count(), \
                  nb::g_ht_n = (k) + 1 > nb::g_ht_n ? (k) + 1 : nb::g_ht_n)
#else
#define NB_HT(k) ((void)0)
#endif

namespace nb {

enum : int {
  NB_STEP_MODE_ACCEL = 0,
  NB_STEP_MODE_FIRST = 1,
  NB_STEP_MODE_KICK_DRIFT = 2,
  NB_STEP_MODE_FINAL = 3,
};

constexpr int kMaxPeers = 8;

template <typename R>
struct StepArgs {
  const V4<R>* pos;  // n_all packed (x,y,z,m): read-only during the launch
  int64_t n_all, i_begin, n_i, j_begin, j_count;
  R eps2;            // (R)eps2  (_accel_cy.pyx:119)
  double g;          // applied to the FP64 sum, then rounded to R
  R dt, half, f;     // (R)dt, (R)0.5, (R)(0.5*dt)  (_accel_cy.pyx:211-212; __init__.py:223)
  int mode, carry_mode;
  int uniform_mass;  // 1: every m_j equals pos[0].w; terms omit m_j, the sum is scaled once
  const R* mass0;    // where that mass is read instead of pos[0].w (nullptr: pos[0].w)
  double* carry;     // 3*n_i FP64 partial sums (SoA), carry_mode 1/2
  V4<R>* acc;        // n_i: a_prev in, a out
  V4<R>* vel;        // n_i
  V4<R>* pos_next;   // n_all: rows of this shard written by drift modes
  double* slots;     // stream-K partial slots (workspace)
  // In-kernel split-i-block fixup: one ready flag per slot (workspace header),
  // set to this launch's unique tag once the slot's partials are visible.
  unsigned long long* flags;
  unsigned long long tag;
  // 1: the drifted body is stored with ONE coherent 128-/256-bit access (st4_pub):
  // the small-N kernel's tagged position exchange (its fourth word is the step tag)
  int pub;
  int64_t units, n_tiles, n_iblocks;
  int64_t grid;
  // Cost-balanced stream-K (Sched in nbody_force.cu): target groups per thread
  // of a full i-block, and the live ones of the last (partial) i-block.
  int sched_kg, sched_lg;
  // Multi-GPU peer-store epilogue: the drifted rows are also stored straight
  // into every peer GPU's next-position buffer over NVLink (no all-gather).
  V4<R>* peers[kMaxPeers];
  int n_peers;
};

struct StepGeometry {
  int threads, i_block, tile;
  int64_t n_iblocks, n_tiles, units;
};

template <typename R> StepGeometry step_geometry(int64_t n_i, int64_t j_count);
// flags: bit 0 exclude the self pair explicitly, bit 1 uniform masses.
template <typename R> cudaError_t launch_step(StepArgs<R> a, int flags, cudaStream_t s);
// Which force kernel launch_step runs for a launch of this shape on the current
// device: "pair_kernel" (FP32 cluster split-source) or "step_kernel" (stream-K).
template <typename R> const char* step_kernel_name(int64_t n_i, int64_t j_count);
template <typename R> int64_t step_workspace_bytes(int64_t n_i);
// Whole simulate loop (steps drift steps + the final kick) in one cooperative launch.
template <typename R> cudaError_t launch_simulate_persistent(StepArgs<R> a, int flags, V4<R>* pos_a, V4<R>* pos_b,
                                                             int64_t steps, cudaStream_t s);
// Small N: the whole simulate loop in one cooperative launch with the source split
// inside each CTA (no global partials); cudaErrorCooperativeLaunchTooLarge when
// the grid or its shared memory does not fit.
// cols (optional): the host API's device column block, read at step 0 and
// written with the final state (no pack/unpack launches); cols_out (optional):
// where the final state goes instead -- the device view of the caller's
// pinned host block, so no D2H copy follows.
template <typename R> cudaError_t launch_simulate_small(StepArgs<R> a, int flags, V4<R>* pos_a, V4<R>* pos_b,
                                                        int64_t steps, cudaStream_t s, R* cols = nullptr,
                                                        R* cols_out = nullptr);
// Byte offset of the slot area inside the workspace: a 256-byte-aligned header
// holding the slots' ready flags (2 per CTA of the largest persistent grid).
template <typename R> int64_t workspace_header_bytes();

// Stand-alone O(N) kernels (nbody_update.cu).
template <typename R> cudaError_t launch_drift(V4<R>* pos, V4<R>* vel, const V4<R>* acc, int64_t n, double dt, cudaStream_t s);
template <typename R> cudaError_t launch_update(V4<R>* pos_next, const V4<R>* pos_cur, V4<R>* vel, const V4<R>* acc,
                                                const V4<R>* acc_prev, int64_t n, double dt, int mode, cudaStream_t s);
template <typename R> cudaError_t launch_kick(V4<R>* vel, const V4<R>* an, const V4<R>* ao, int64_t n, double factor, cudaStream_t s);
template <typename R> cudaError_t launch_pack_soa(const R* x, const R* y, const R* z, const R* w, V4<R>* out, int64_t n, cudaStream_t s);
template <typename R> cudaError_t launch_unpack_soa(const V4<R>* in, R* x, R* y, R* z, int64_t n, cudaStream_t s);
template <typename R> cudaError_t launch_pack_aos(const R* xyz, const R* w, V4<R>* out, int64_t n, cudaStream_t s);
template <typename R> cudaError_t launch_unpack_aos(const V4<R>* in, R* xyz, int64_t n, cudaStream_t s);
// kind 0: uniform cube, 1: Plummer sphere (BASELINE.json generators).
template <typename R> cudaError_t launch_init(int kind, unsigned long long seed, int64_t n, V4<R>* pos, V4<R>* vel,
                                              cudaStream_t s);
int64_t energy_workspace_entries(int precision_bytes, int64_t n);
#if NB_TRACE
int trace_setup(void* buf, int64_t cap);
int64_t trace_count();
#endif  // doubles of workspace the energy pass can use
template <typename R> cudaError_t launch_energy(const V4<R>* pos, const V4<R>* vel, int64_t n, double g, double eps2,
                                               double* out6, double* phi, int64_t phi_entries, cudaStream_t s);

}  // namespace nb
