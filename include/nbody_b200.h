/*
 * nbody_b200.h -- C ABI of libnbody_b200.so, the B200 (sm_100a) all-pairs
 * N-body hot path that sits behind the reference package's N-body entry point
 * (arXiv 2203.08263 artifact `nbodybench`).  Paths in citations are relative to
 * /root/reference/pkg/src/nbodybench/.
 *
 * Two families of entry points:
 *
 *  1. nb_host_*  -- HOST pointers, synchronous.  These are exactly the calls the
 *     reference's own FFI for this path makes into its compiled kernel module
 *     (Cython `_accel_cy`, bound through typed memoryviews), with the same
 *     argument order and meaning, plus the body count that a memoryview carries
 *     implicitly.  `block` and `threads` are accepted and ignored: the GPU uses
 *     its own tiling and all SMs.  `recip` selects the algebraic form on the CPU;
 *     the GPU always evaluates m*d*rsqrt(d2)^3, which the reference pins as
 *     equivalent to both forms (pkg/tests/test_kernels.py:220-227).  The library
 *     keeps the device buffers and a pinned staging block of these calls between
 *     calls (per device, grow-only); calls are serialized internally.
 *
 *  2. nb_dev_*   -- DEVICE pointers owned by the caller (e.g. torch tensors),
 *     stream-ordered, asynchronous.  These carry the packed HBM layout the
 *     kernels use and the i-shard / j-range arguments multi-GPU sharding needs.
 *
 * Packed layout (device): bodies are 4-vectors of the system precision,
 *   pos4[k] = (x, y, z, m),  vel4[k] = (vx, vy, vz, 0),  acc4[k] = (ax, ay, az, 0)
 * i.e. float4 (16 B) for *_f32 and double4 (32 B) for *_f64, 16 B aligned.
 *
 * Errors: every int-returning call returns 0 on success, else a nonzero code
 * (NB_ERR_* below, or a cudaError_t value + 1000); nb_last_error() describes
 * the last failure on the calling thread.  Argument errors are detected before
 * any device work.  Non-finite results are NOT checked (kernels/__init__.py:190-191).
 */
#ifndef NBODY_B200_H_
#define NBODY_B200_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define NB_OK 0
#define NB_ERR_ARG 1       /* invalid argument (sizes, null pointers, modes)      */
#define NB_ERR_WORKSPACE 2 /* workspace pointer null or smaller than required     */
#define NB_ERR_NODEV 3     /* no CUDA device / not an sm_100 device               */
#define NB_ERR_CUDA 1000   /* + cudaError_t                                       */
#define NB_ERR_NCCL 2000   /* + ncclResult_t (nb_comm_*)                           */
#define NB_ERR_NCCL_MISSING 4 /* libnccl.so.2 could not be loaded (nb_comm_*)      */

/* Update modes of the fused force+integrate step (nb_dev_step_*).
 * The velocity-Verlet loop of kernels.simulate (kernels/__init__.py:240-252) is
 *   A(p); [kick if step>0]; kick-drift; ... ; A(p); kick
 * and maps to NB_STEP_FIRST, NB_STEP_KICK_DRIFT x (steps-1), NB_STEP_FINAL_KICK.  */
#define NB_MODE_ACCEL 0      /* a only: acc4 <- G*sum                               */
#define NB_STEP_FIRST 1      /* step 0: dv=a*dt; p'=p+(v+half*dv)*dt; v+=dv; acc4<-a */
#define NB_STEP_KICK_DRIFT 2 /* step>0: v+=(a-acc4)*f, f=real(0.5*dt); then FIRST    */
#define NB_STEP_FINAL_KICK 3 /* after the loop: v+=(a-acc4)*f; acc4<-a; p unchanged */

/* Kernel flags (the `flags` argument of nb_dev_step_* / nb_dev_simulate_*). */
#define NB_FLAG_EXCLUDE_SELF 1 /* skip j == i explicitly: required when (real)eps2 == 0 (the
                                  self pair is 0*inf) or m*eps2^-1.5 overflows; otherwise the
                                  self pair is included and adds exactly 0                   */
#define NB_FLAG_UNIFORM_MASS 2 /* caller guarantees every m_j equals pos4[0].w: terms omit
                                  m_j and the sum is scaled by m once (one FMUL2 less per
                                  interaction pair)                                          */
#define NB_FLAG_AUTO 256       /* nb_dev_simulate_cols_* only: derive the two flags above
                                  from the host mass column itself (one pass over n masses
                                  in C, instead of the caller's)                            */

/* ---------------------------------------------------------------- host (FFI mirror) */

/* Replaces _accel_cy.accel_soa (_accel_cy.pyx:114-152), called from
 * kernels.compute_accelerations (kernels/__init__.py:199-202). */
int nb_host_accel_soa_f32(const float* px, const float* py, const float* pz, const float* m,
                          int64_t n, double g, double eps2, int recip, int64_t block,
                          int threads, float* ax, float* ay, float* az);
int nb_host_accel_soa_f64(const double* px, const double* py, const double* pz,
                          const double* m, int64_t n, double g, double eps2, int recip,
                          int64_t block, int threads, double* ax, double* ay, double* az);

/* Replaces _accel_cy.accel_aos (_accel_cy.pyx:155-202): pos is C-contiguous (n,3). */
int nb_host_accel_aos_f32(const float* pos, const float* m, int64_t n, double g, double eps2,
                          float* ax, float* ay, float* az);
int nb_host_accel_aos_f64(const double* pos, const double* m, int64_t n, double g,
                          double eps2, double* ax, double* ay, double* az);

/* Replaces _accel_cy.step_soa (_accel_cy.pyx:205-237), in place. */
int nb_host_step_soa_f32(float* px, float* py, float* pz, float* vx, float* vy, float* vz,
                         const float* ax, const float* ay, const float* az, int64_t n,
                         double dt, int threads);
int nb_host_step_soa_f64(double* px, double* py, double* pz, double* vx, double* vy,
                         double* vz, const double* ax, const double* ay, const double* az,
                         int64_t n, double dt, int threads);

/* Replaces _accel_cy.step_aos (_accel_cy.pyx:240-259), in place on (n,3) arrays. */
int nb_host_step_aos_f32(float* pos, float* vel, const float* ax, const float* ay,
                         const float* az, int64_t n, double dt);
int nb_host_step_aos_f64(double* pos, double* vel, const double* ax, const double* ay,
                         const double* az, int64_t n, double dt);

/* Replaces the whole of kernels.simulate (kernels/__init__.py:230-253) for an SoA
 * system: runs `steps` velocity-Verlet steps (steps+1 force evaluations) on the
 * device and writes the final state back IN PLACE into px..vz (the caller passes
 * copies, as simulate's `state = sys_.copy()` does at :240). */
int nb_host_simulate_soa_f32(float* px, float* py, float* pz, float* vx, float* vy, float* vz,
                             const float* m, int64_t n, double g, double dt, double eps2,
                             int64_t steps);
int nb_host_simulate_soa_f64(double* px, double* py, double* pz, double* vx, double* vy,
                             double* vz, const double* m, int64_t n, double g, double dt,
                             double eps2, int64_t steps);

/* The same simulate with the inputs left untouched: x, y, z, m, vx, vy, vz
 * columns in, the final x, y, z, vx, vy, vz into out6 (6*n elements, column
 * after column), on CUDA device `device` (< 0: the library's current one).
 * The binding behind simulate()'s single-GPU path (the CPython module
 * paper_2203_08263_b200._hostpath). */
int nb_host_simulate_f32(const float* px, const float* py, const float* pz, const float* m,
                         const float* vx, const float* vy, const float* vz, int64_t n, double g,
                         double dt, double eps2, int64_t steps, float* out6, int device);
int nb_host_simulate_f64(const double* px, const double* py, const double* pz, const double* m,
                         const double* vx, const double* vy, const double* vz, int64_t n, double g,
                         double dt, double eps2, int64_t steps, double* out6, int device);

/* ---------------------------------------------------------------- device (packed) */

/* Workspace bytes a nb_dev_step_* call needs for an i-shard of n_i bodies;
 * precision_bytes is 4 or 8.  Scratch only (FP64 partial sums of i-blocks split
 * between CTAs): no initialisation needed, reusable across calls on one stream. */
int64_t nb_dev_workspace_bytes(int precision_bytes, int64_t n_i);

/* Name of the force kernel a nb_dev_step_* launch of n_i targets against
 * j_count sources runs on the current device: "pair_kernel" (FP32 launches
 * whose 224-target i-blocks fill one wave of 2-CTA clusters -- the source range
 * split over 16 warps and reduced through distributed shared memory) or
 * "step_kernel" (stream-K + split-i-block fixup).  Diagnostic (bench, tests);
 * NULL on a bad precision. */
const char* nb_dev_step_kernel(int precision_bytes, int64_t n_i, int64_t j_count);

/* Fused softened all-pairs force (+ optional velocity-Verlet update) for the
 * target rows [i_begin, i_begin+n_i) of pos4 (n_all bodies) against the source
 * bodies j in [j_begin, j_begin+j_count) taken modulo n_all (circular, so a
 * shard can take "everything after my slice" as one range).
 *
 *   a_i = G * sum_j m_j (p_j - p_i) / (|p_j - p_i|^2 + eps2)^(3/2)
 *
 * mode         NB_MODE_ACCEL or one of NB_STEP_* (see above).
 * flags        NB_FLAG_EXCLUDE_SELF | NB_FLAG_UNIFORM_MASS (see above).
 * carry        optional FP64 3*n_i buffer (SoA: x then y then z) of partial sums
 *              (without G):
 *              carry_mode 0: unused; 1: write the partial sums here and do not
 *              finalize (first phase of a split j range); 2: add carry before
 *              finalizing (second phase).
 * acc4         n_i entries: a_prev in (kick modes), a out.
 * vel4         n_i entries (step modes): updated in place.
 * pos4_next    n_all entries (STEP_FIRST / STEP_KICK_DRIFT): rows
 *              [i_begin, i_begin+n_i) receive the drifted (x,y,z,m).  Must not
 *              alias pos4.
 * stream       a cudaStream_t (NULL = legacy default stream).
 * Summation order: fixed per (n_i, j_count, GPU) -- results are bitwise
 * reproducible run to run.  A whole-system NB_MODE_ACCEL call at small N (the
 * small-N bounds of nb_dev_simulate_*) runs the small-N kernel, whose order
 * differs from the per-step path's (parity-tolerance equal, not bitwise). */
int nb_dev_step_f32(const void* pos4, int64_t n_all, int64_t i_begin, int64_t n_i,
                    int64_t j_begin, int64_t j_count, double g, double eps2, double dt,
                    int mode, int flags, double* carry, int carry_mode, void* acc4,
                    void* vel4, void* pos4_next, void* workspace, int64_t workspace_bytes,
                    void* stream);
int nb_dev_step_f64(const void* pos4, int64_t n_all, int64_t i_begin, int64_t n_i,
                    int64_t j_begin, int64_t j_count, double g, double eps2, double dt,
                    int mode, int flags, double* carry, int carry_mode, void* acc4,
                    void* vel4, void* pos4_next, void* workspace, int64_t workspace_bytes,
                    void* stream);

/* nb_dev_step_* with a fused NVLink peer-store epilogue (multi-GPU without an
 * all-gather): drift modes also store each drifted row into every buffer of
 * peer_pos4_next[0..n_peers) (up to 8 UVA pointers to the next-position buffers
 * of the other GPUs, e.g. from CUDA IPC / symmetric memory) and end with a
 * system-scope fence.  The caller orders steps across GPUs with a barrier
 * between the local-source pass and the remote-source pass of the next step. */
int nb_dev_step_p2p_f32(const void* pos4, int64_t n_all, int64_t i_begin, int64_t n_i,
                        int64_t j_begin, int64_t j_count, double g, double eps2, double dt,
                        int mode, int flags, double* carry, int carry_mode, void* acc4,
                        void* vel4, void* pos4_next, void* const* peer_pos4_next, int n_peers,
                        void* workspace, int64_t workspace_bytes, void* stream);
int nb_dev_step_p2p_f64(const void* pos4, int64_t n_all, int64_t i_begin, int64_t n_i,
                        int64_t j_begin, int64_t j_count, double g, double eps2, double dt,
                        int mode, int flags, double* carry, int carry_mode, void* acc4,
                        void* vel4, void* pos4_next, void* const* peer_pos4_next, int n_peers,
                        void* workspace, int64_t workspace_bytes, void* stream);

/* Device-resident kernels.simulate for one GPU: `steps` fused steps plus the final
 * evaluation and kick (steps+1 force evaluations), ping-ponging pos4_a <-> pos4_b.
 * On return (stream-ordered) the final positions are in pos4_a if steps is even,
 * else in pos4_b; *final_in_b reports which (may be NULL).  Small N runs the whole
 * loop in one cooperative launch: N <= 3584 (FP32) / 2560 (FP64) with the source
 * split inside each CTA (environment NB_SMALL_MAX_N overrides, 0 disables; its
 * summation order differs from the per-step path, results agree within the
 * parity tolerances), up to 8192 with the per-step decomposition (bitwise equal
 * to per-step launches; NB_PERSISTENT_MAX_N overrides).  Larger N: one launch
 * (plus a split-block fixup launch) per force evaluation. */
int nb_dev_simulate_f32(void* pos4_a, void* pos4_b, void* vel4, void* acc4, int64_t n,
                        double g, double dt, double eps2, int64_t steps, int flags,
                        void* workspace, int64_t workspace_bytes, void* stream,
                        int* final_in_b);
int nb_dev_simulate_f64(void* pos4_a, void* pos4_b, void* vel4, void* acc4, int64_t n,
                        double g, double dt, double eps2, int64_t steps, int flags,
                        void* workspace, int64_t workspace_bytes, void* stream,
                        int* final_in_b);

/* nb_dev_simulate_* plus per-launch device timing: launch_ms (host, steps+1
 * floats) receives the CUDA-event time of each force evaluation (fused step +
 * fixup) measured on `stream`.  Synchronizes the stream before returning. */
int nb_dev_simulate_timed_f32(void* pos4_a, void* pos4_b, void* vel4, void* acc4, int64_t n,
                              double g, double dt, double eps2, int64_t steps, int flags,
                              void* workspace, int64_t workspace_bytes, void* stream,
                              int* final_in_b, float* launch_ms);
int nb_dev_simulate_timed_f64(void* pos4_a, void* pos4_b, void* vel4, void* acc4, int64_t n,
                              double g, double dt, double eps2, int64_t steps, int flags,
                              void* workspace, int64_t workspace_bytes, void* stream,
                              int* final_in_b, float* launch_ms);

/* Boundary layout conversion on the device: the caller's
 * SoA columns (one contiguous H2D) into the packed rows, and back (one
 * contiguous D2H).  pack: out4[i] = (x[i], y[i], z[i], w ? w[i] : 0);
 * unpack: x[i], y[i], z[i] = in4[i].xyz.  All device pointers, n entries. */
int nb_dev_pack_f32(const void* x, const void* y, const void* z, const void* w, int64_t n,
                    void* out4, void* stream);
int nb_dev_pack_f64(const void* x, const void* y, const void* z, const void* w, int64_t n,
                    void* out4, void* stream);
int nb_dev_unpack_f32(const void* in4, int64_t n, void* x, void* y, void* z, void* stream);
int nb_dev_unpack_f64(const void* in4, int64_t n, void* x, void* y, void* z, void* stream);

/* SURVEY 8(b)'s proposed minimal pair, for hosts that schedule the force pass and
 * the update separately (the product path fuses them in nb_dev_step_* /
 * nb_dev_simulate_*):
 * nb_force: acc_out[k] = G * sum_j m_j d / (|d|^2 + eps2)^(3/2) for the targets
 *   [i_begin, i_begin+n_i) of pos_all against all n_all sources (the self pair is
 *   always excluded explicitly: the masses are device-resident, so an overflowing
 *   self term m*eps2^-1.5 cannot be ruled out on the host); workspace as for
 *   nb_dev_step_*.
 * nb_update: the step update of one shard's n_i rows with the reference's
 *   rounding (mode NB_STEP_FIRST / NB_STEP_KICK_DRIFT / NB_STEP_FINAL_KICK, as in
 *   the fused step): pos_next = drifted pos_cur (= pos_cur for the final kick),
 *   vel updated in place; acc_prev is read by the kick modes only. */
int nb_force_f32(const void* pos_all, int64_t n_all, int64_t i_begin, int64_t n_i, double eps2,
                 double g, void* acc_out, void* workspace, int64_t workspace_bytes, void* stream);
int nb_force_f64(const void* pos_all, int64_t n_all, int64_t i_begin, int64_t n_i, double eps2,
                 double g, void* acc_out, void* workspace, int64_t workspace_bytes, void* stream);
int nb_update_f32(void* pos_next, const void* pos_cur, void* vel, const void* acc,
                  const void* acc_prev, int64_t n_i, double dt, int mode, void* stream);
int nb_update_f64(void* pos_next, const void* pos_cur, void* vel, const void* acc,
                  const void* acc_prev, int64_t n_i, double dt, int mode, void* stream);

/* The same conversion fused with its transfer, for simulate()'s column staging:
 * one call each way (small N is host-latency-bound).  Column block layout, in
 * elements of the system precision: x, y, z, m of all n bodies at 0, n, 2n, 3n,
 * then vx, vy, vz of the n_i owned rows at 4n, 4n + ni, 4n + 2ni with
 * ni = max(n_i, 1) -- 4n + 3ni elements.  load: H2D of the whole block from
 * host_cols (pinned for an asynchronous copy), then pos4 (n rows, masses in .w)
 * and vel4 (n_i rows) packed from it; asynchronous.  store: pos4 and vel4
 * unpacked into dev_cols (the mass column is left as is), D2H of the x, y, z
 * and vx, vy, vz columns into the same places of host_cols, and a synchronize
 * of `stream` before returning. */
/* load_cols + simulate + store_cols in one call (an unsharded system, n_i = n):
 * host_cols in (the column block above, 7n elements), host_cols out (x, y, z,
 * vx, vy, vz of the final state, masses unchanged; one H2D and one D2H of the
 * block; synchronizes `stream`); *final_in_b as for nb_dev_simulate_*.  At
 * small N the simulate kernel reads and writes dev_cols itself (no pack/unpack
 * launches); pos4_a/b, vel4 and acc4 hold the final state either way. */
int nb_dev_simulate_cols_f32(void* host_cols, void* dev_cols, void* pos4_a, void* pos4_b, void* vel4,
                             void* acc4, int64_t n, double g, double dt, double eps2, int64_t steps,
                             int flags, void* workspace, int64_t workspace_bytes, void* stream,
                             int* final_in_b);
int nb_dev_simulate_cols_f64(void* host_cols, void* dev_cols, void* pos4_a, void* pos4_b, void* vel4,
                             void* acc4, int64_t n, double g, double dt, double eps2, int64_t steps,
                             int flags, void* workspace, int64_t workspace_bytes, void* stream,
                             int* final_in_b);
int nb_dev_load_cols_f32(const void* host_cols, void* dev_cols, int64_t n, int64_t n_i,
                         void* pos4, void* vel4, void* stream);
int nb_dev_load_cols_f64(const void* host_cols, void* dev_cols, int64_t n, int64_t n_i,
                         void* pos4, void* vel4, void* stream);
int nb_dev_store_cols_f32(const void* pos4, const void* vel4, int64_t n, int64_t n_i,
                          void* dev_cols, void* host_cols, void* stream);
int nb_dev_store_cols_f64(const void* pos4, const void* vel4, int64_t n, int64_t n_i,
                          void* dev_cols, void* host_cols, void* stream);

/* Stand-alone update kernels on packed arrays (n entries each): the kick-drift
 * of step_soa (_accel_cy.pyx:205-237) in place, and the trapezoidal kick of
 * _kick (kernels/__init__.py:220-227): v += (a_new - a_old) * real(factor). */
int nb_dev_drift_f32(void* pos4, void* vel4, const void* acc4, int64_t n, double dt,
                     void* stream);
int nb_dev_drift_f64(void* pos4, void* vel4, const void* acc4, int64_t n, double dt,
                     void* stream);
int nb_dev_kick_f32(void* vel4, const void* acc4_new, const void* acc4_old, int64_t n,
                    double factor, void* stream);
int nb_dev_kick_f64(void* vel4, const void* acc4_new, const void* acc4_old, int64_t n,
                    double factor, void* stream);

/* Softened potential energy  -G * sum_{i<j} m_i m_j / sqrt(|p_i-p_j|^2 + eps2)
 * and kinetic energy / momentum of the packed state (validation.py:134-145),
 * accumulated in FP64.  out6 (device, 6 doubles) <- (KE, PE, Px, Py, Pz, KE+PE).
 * workspace: device scratch of at least 8*n bytes (per-body potentials);
 * nb_energy_workspace_bytes(precision_bytes, n) is the size that lets the pass
 * split the sources into ranges (to fill the GPU at any N) and reduce on every
 * SM.  The reduction order is fixed for a given device and workspace size. */
int64_t nb_energy_workspace_bytes(int precision_bytes, int64_t n);
int nb_dev_energy_f32(const void* pos4, const void* vel4, int64_t n, double g, double eps2,
                      double* out6, void* workspace, int64_t workspace_bytes, void* stream);
int nb_dev_energy_f64(const void* pos4, const void* vel4, int64_t n, double g, double eps2,
                      double* out6, void* workspace, int64_t workspace_bytes, void* stream);

/* On-device initial conditions (BASELINE.json generators):
 * splitmix64 in closed form (core.py:92-113), FP64, rounded once to the system
 * precision.  NB_INIT_UNIFORM_CUBE: 7 draws per body, x = -1+2u, v = -0.1+0.2u,
 * m = 0.5+u (bit-identical to paper_2203_08263_b200.core.uniform_cube);
 * NB_INIT_PLUMMER: 3 draws per body, scale radius 1, v = 0, m = 1/n.
 * Writes n packed bodies to pos4 (x,y,z,m) and vel4 (vx,vy,vz,0). */
#define NB_INIT_UNIFORM_CUBE 0
#define NB_INIT_PLUMMER 1
int nb_dev_init_f32(int kind, uint64_t seed, int64_t n, void* pos4, void* vel4, void* stream);
int nb_dev_init_f64(int kind, uint64_t seed, int64_t n, void* pos4, void* vel4, void* stream);

/* ---------------------------------------------------------------- misc */

const char* nb_last_error(void);
/* ---------------------------------------------------------------- exchange (NCCL) */

/* The per-step position exchange of the i-sharded multi-GPU loop:
 * after a rank's fused step wrote its rows [r*n/P, (r+1)*n/P) of the next
 * positions, every rank needs all n.  These wrap NCCL (resolved at run time from
 * libnccl.so.2, the copy the process already uses when there is one) for hosts
 * that are not Python; the Python driver does the same through
 * torch.distributed.  Communicators are opaque (ncclComm_t); not re-entrant per
 * communicator.  Two set-ups:
 *  - one process per GPU: rank 0 calls nb_comm_unique_id, the host distributes
 *    the NB_COMM_ID_BYTES bytes, every rank calls nb_comm_init_rank;
 *  - one process driving ndev GPUs: nb_comm_init_all (ncclCommInitAll).
 * nb_comm_allgather: IN PLACE on `buf` (this rank's block is at
 * buf + rank*bytes_per_rank, every block is bytes_per_rank), stream-ordered on
 * `stream`; with packed float4/double4 rows, bytes_per_rank = rows * 16 / 32.
 * nb_comm_allgather_all: the same for all ndev GPUs of one process (grouped). */
#define NB_COMM_ID_BYTES 128
int nb_comm_unique_id(void* id_out);
int nb_comm_init_rank(int nranks, int rank, const void* id, void** comm_out);
int nb_comm_init_all(int ndev, const int* devs, void** comms_out);
int nb_comm_allgather(void* buf, size_t bytes_per_rank, void* comm, void* stream);
int nb_comm_allgather_all(void* const* bufs, size_t bytes_per_rank, void* const* comms,
                          void* const* streams, int ndev);
int nb_comm_destroy(void* comm);

/* "nbody_b200 <version> (sm_100a) src:<digest>": <digest> is the first 16 hex
 * digits of the SHA-256 over the library's sources (paper_2203_08263_b200/csrc/*
 * and this header) the build was compiled from. */
const char* nb_version(void);
/* Number of kernel launches this library has issued on the calling process. */
int64_t nb_launch_count(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif

#endif /* NBODY_B200_H_ */
