/*
 * nbody_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's CPU algorithm for the all-pairs
 * N-body hot path (arXiv 2203.08263 artifact `nbodybench`), used as the parity
 * checker for the sm_100a kernels and as the CPU baseline ("port") in bench.py.
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load this library.  The product path never does.
 *
 * Every function cites the reference file:line it restates.  Paths are
 * relative to /root/reference/pkg/src/nbodybench/.
 *
 * Arithmetic contract (mirrors setup.py:7-8,17 `-ffp-contract=off`): this file
 * MUST be compiled with -ffp-contract=off and without -ffast-math so every
 * a*b+c is two rounded operations, exactly like the reference build.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------- */
/* splitmix64 -- core.py:92-107 (closed form state_k = seed + k*gamma).       */
ORC_EXPORT void orc_splitmix64(uint64_t seed, int64_t count, uint64_t* out) {
  for (int64_t k = 0; k < count; ++k) {
    uint64_t z = seed + (uint64_t)(k + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    out[k] = z ^ (z >> 31);
  }
}

/* Unit doubles u = (z >> 11) * 2^-53 -- core.py:110-113. */
ORC_EXPORT void orc_units(uint64_t seed, int64_t count, double* out) {
  for (int64_t k = 0; k < count; ++k) {
    uint64_t z = seed + (uint64_t)(k + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    out[k] = (double)(z >> 11) * 0x1.0p-53;
  }
}

/* Order-fixed checksum: sum of (x+y)+z in double, ascending i -- core.py:244-254. */
ORC_EXPORT double orc_checksum_f64(const double* x, const double* y, const double* z, int64_t n) {
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) total += (x[i] + y[i]) + z[i];
  return total;
}
ORC_EXPORT double orc_checksum_f32(const float* x, const float* y, const float* z, int64_t n) {
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) total += ((double)x[i] + (double)y[i]) + (double)z[i];
  return total;
}

/* ------------------------------------------------------------------------- */
/* Per-precision kernels.  REAL / SFX / SQRT / POW are bound by the macro     */
/* below, like the reference's fused `real` type (_accel_cy.pyx:19-21).       */

#define DEFINE_PRECISION(REAL, SFX, SQRT, POW)                                              \
                                                                                            \
/* _row_recip -- _accel_cy.pyx:68-111: j-loop split around i (self skipped,                 \
   no branch); d2 = ((dx*dx + dy*dy) + dz*dz) + eps2; inv = 1/(d2*sqrt(d2));               \
   w = m*inv; t += d*w; partial added into out once per (i, j-range). */                    \
static void row_recip_##SFX(const REAL* px, const REAL* py, const REAL* pz,                \
                            const REAL* m, int64_t i, int64_t j0, int64_t j1, REAL eps2,   \
                            REAL* ox, REAL* oy, REAL* oz) {                                \
  const REAL pxi = px[i], pyi = py[i], pzi = pz[i];                                        \
  REAL tx = 0, ty = 0, tz = 0;                                                              \
  int64_t lim = i < j1 ? i : j1;                                                            \
  for (int pass = 0; pass < 2; ++pass) {                                                    \
    int64_t lo = pass == 0 ? j0 : (i + 1 > j0 ? i + 1 : j0);                                \
    int64_t hi = pass == 0 ? lim : j1;                                                      \
    for (int64_t j = lo; j < hi; ++j) {                                                     \
      REAL dx = px[j] - pxi, dy = py[j] - pyi, dz = pz[j] - pzi;                            \
      REAL d2 = dx * dx + dy * dy + dz * dz + eps2;                                         \
      REAL inv = (REAL)1.0 / (d2 * SQRT(d2));                                               \
      REAL w = m[j] * inv;                                                                  \
      tx = tx + dx * w;                                                                     \
      ty = ty + dy * w;                                                                     \
      tz = tz + dz * w;                                                                     \
    }                                                                                       \
  }                                                                                         \
  *ox += tx; *oy += ty; *oz += tz;                                                          \
}                                                                                           \
                                                                                            \
/* _row_pow -- _accel_cy.pyx:24-65: s = pow(d2, 1.5); t += m*d/s. */                        \
static void row_pow_##SFX(const REAL* px, const REAL* py, const REAL* pz,                  \
                          const REAL* m, int64_t i, int64_t j0, int64_t j1, REAL eps2,     \
                          REAL* ox, REAL* oy, REAL* oz) {                                  \
  const REAL pxi = px[i], pyi = py[i], pzi = pz[i];                                        \
  REAL tx = 0, ty = 0, tz = 0;                                                              \
  int64_t lim = i < j1 ? i : j1;                                                            \
  for (int pass = 0; pass < 2; ++pass) {                                                    \
    int64_t lo = pass == 0 ? j0 : (i + 1 > j0 ? i + 1 : j0);                                \
    int64_t hi = pass == 0 ? lim : j1;                                                      \
    for (int64_t j = lo; j < hi; ++j) {                                                     \
      REAL dx = px[j] - pxi, dy = py[j] - pyi, dz = pz[j] - pzi;                            \
      REAL d2 = dx * dx + dy * dy + dz * dz + eps2;                                         \
      REAL s = POW(d2, (REAL)1.5);                                                          \
      tx = tx + m[j] * dx / s;                                                              \
      ty = ty + m[j] * dy / s;                                                              \
      tz = tz + m[j] * dz / s;                                                              \
    }                                                                                       \
  }                                                                                         \
  *ox += tx; *oy += ty; *oz += tz;                                                          \
}                                                                                           \
                                                                                            \
/* accel_soa -- _accel_cy.pyx:114-152: zero, per-i rows (static schedule over i),          \
   optional j-blocking (tiles outer, i inner), then out *= G sequentially.                  \
   eps2 and G are rounded to REAL first (:119-120). */                                      \
ORC_EXPORT void orc_accel_soa_##SFX(const REAL* px, const REAL* py, const REAL* pz,        \
                                    const REAL* m, int64_t n, double g, double eps2,       \
                                    int recip, int64_t block, int threads,                 \
                                    REAL* ax, REAL* ay, REAL* az) {                        \
  const REAL geps = (REAL)eps2, gg = (REAL)g;                                               \
  if (threads < 1) threads = 1;                                                             \
  for (int64_t i = 0; i < n; ++i) { ax[i] = 0; ay[i] = 0; az[i] = 0; }                     \
  int64_t step = block > 0 ? block : n;                                                     \
  for (int64_t j0 = 0; j0 < n; j0 += step) {                                                \
    int64_t j1 = j0 + step < n ? j0 + step : n;                                             \
    _Pragma("omp parallel for schedule(static) num_threads(threads)")                       \
    for (int64_t i = 0; i < n; ++i) {                                                       \
      if (recip) row_recip_##SFX(px, py, pz, m, i, j0, j1, geps, &ax[i], &ay[i], &az[i]);  \
      else row_pow_##SFX(px, py, pz, m, i, j0, j1, geps, &ax[i], &ay[i], &az[i]);          \
    }                                                                                       \
  }                                                                                         \
  for (int64_t i = 0; i < n; ++i) { ax[i] *= gg; ay[i] *= gg; az[i] *= gg; }               \
}                                                                                           \
                                                                                            \
/* accel_soa restricted to the target rows [i0, i0+ni) (row sample of the same            \
   arithmetic; used for bounded CPU baselines and large-N spot checks). */                  \
ORC_EXPORT void orc_accel_rows_##SFX(const REAL* px, const REAL* py, const REAL* pz,       \
                                     const REAL* m, int64_t n, int64_t i0, int64_t ni,     \
                                     double g, double eps2, int threads,                   \
                                     REAL* ax, REAL* ay, REAL* az) {                       \
  const REAL geps = (REAL)eps2, gg = (REAL)g;                                               \
  if (threads < 1) threads = 1;                                                             \
  _Pragma("omp parallel for schedule(static) num_threads(threads)")                         \
  for (int64_t k = 0; k < ni; ++k) {                                                        \
    REAL x = 0, y = 0, z = 0;                                                               \
    row_recip_##SFX(px, py, pz, m, i0 + k, 0, n, geps, &x, &y, &z);                         \
    ax[k] = x * gg; ay[k] = y * gg; az[k] = z * gg;                                         \
  }                                                                                         \
}                                                                                           \
                                                                                            \
/* step_soa -- _accel_cy.pyx:205-237: dv = a*dt; p += (v + half*dv)*dt; v += dv,           \
   with dt and half rounded to REAL (:211-212). */                                          \
ORC_EXPORT void orc_step_soa_##SFX(REAL* px, REAL* py, REAL* pz, REAL* vx, REAL* vy,       \
                                   REAL* vz, const REAL* ax, const REAL* ay,               \
                                   const REAL* az, int64_t n, double dt, int threads) {    \
  const REAL dtt = (REAL)dt, half = (REAL)0.5;                                              \
  if (threads < 1) threads = 1;                                                             \
  _Pragma("omp parallel for schedule(static) num_threads(threads)")                         \
  for (int64_t i = 0; i < n; ++i) {                                                         \
    REAL dvx = ax[i] * dtt, dvy = ay[i] * dtt, dvz = az[i] * dtt;                           \
    px[i] += (vx[i] + half * dvx) * dtt;                                                    \
    py[i] += (vy[i] + half * dvy) * dtt;                                                    \
    pz[i] += (vz[i] + half * dvz) * dtt;                                                    \
    vx[i] += dvx; vy[i] += dvy; vz[i] += dvz;                                               \
  }                                                                                         \
}                                                                                           \
                                                                                            \
/* _kick -- kernels/__init__.py:220-227: v += (new - old) * f, f = dtype(factor). */       \
ORC_EXPORT void orc_kick_##SFX(REAL* vx, REAL* vy, REAL* vz, const REAL* nx,               \
                               const REAL* ny, const REAL* nz, const REAL* ox,             \
                               const REAL* oy, const REAL* oz, int64_t n, double factor) { \
  const REAL f = (REAL)factor;                                                              \
  for (int64_t i = 0; i < n; ++i) {                                                         \
    vx[i] += (nx[i] - ox[i]) * f;                                                           \
    vy[i] += (ny[i] - oy[i]) * f;                                                           \
    vz[i] += (nz[i] - oz[i]) * f;                                                           \
  }                                                                                         \
}                                                                                           \
                                                                                            \
/* simulate -- kernels/__init__.py:230-253, in place on the caller's copy:                 \
   for step: A(p); kick if step>0; kick-drift; swap.  Then A(p) and the final kick.        \
   steps+1 force evaluations in total. */                                                   \
ORC_EXPORT int orc_simulate_##SFX(REAL* px, REAL* py, REAL* pz, REAL* vx, REAL* vy,        \
                                  REAL* vz, const REAL* m, int64_t n, double g, double dt, \
                                  double eps2, int64_t steps, int recip, int64_t block,    \
                                  int threads) {                                           \
  REAL* buf = (REAL*)calloc((size_t)(6 * n), sizeof(REAL));                                 \
  if (!buf) return 1;                                                                       \
  REAL *acc = buf, *prev = buf + 3 * n;                                                     \
  const double half_dt = 0.5 * dt;                                                          \
  for (int64_t s = 0; s < steps; ++s) {                                                     \
    orc_accel_soa_##SFX(px, py, pz, m, n, g, eps2, recip, block, threads, acc, acc + n,    \
                        acc + 2 * n);                                                       \
    if (s > 0)                                                                              \
      orc_kick_##SFX(vx, vy, vz, acc, acc + n, acc + 2 * n, prev, prev + n, prev + 2 * n,  \
                     n, half_dt);                                                           \
    orc_step_soa_##SFX(px, py, pz, vx, vy, vz, acc, acc + n, acc + 2 * n, n, dt, threads); \
    REAL* t = acc; acc = prev; prev = t;                                                    \
  }                                                                                         \
  orc_accel_soa_##SFX(px, py, pz, m, n, g, eps2, recip, block, threads, acc, acc + n,      \
                      acc + 2 * n);                                                         \
  orc_kick_##SFX(vx, vy, vz, acc, acc + n, acc + 2 * n, prev, prev + n, prev + 2 * n, n,   \
                 half_dt);                                                                  \
  free(buf);                                                                                \
  return 0;                                                                                 \
}

DEFINE_PRECISION(double, f64, sqrt, pow)
DEFINE_PRECISION(float, f32, sqrtf, powf)

/* ------------------------------------------------------------------------- */
/* High-precision row-sampled oracle for large N: the term   */
/* of validation.py:61-79 (m_j (p_j - p_i) / (d2)^1.5, self term zero) with   */
/* every operation and the sum in long double (x87 80-bit), then times G.     */
/* Inputs are the system's values widened exactly to long double, like       */
/* validation._state_of (validation.py:41-46) widens FP32 systems to double.  */
#define DEFINE_ROWS_LD(REAL, SFX)                                                           \
ORC_EXPORT void orc_accel_rows_ld_##SFX(const REAL* px, const REAL* py, const REAL* pz,    \
                                        const REAL* m, int64_t n, const int64_t* rows,     \
                                        int64_t nrows, double g, double eps2, int threads, \
                                        double* out3) {                                    \
  if (threads < 1) threads = 1;                                                             \
  _Pragma("omp parallel for schedule(dynamic, 1) num_threads(threads)")                     \
  for (int64_t r = 0; r < nrows; ++r) {                                                     \
    const int64_t i = rows[r];                                                              \
    const long double xi = px[i], yi = py[i], zi = pz[i], e2 = (long double)eps2;           \
    long double sx = 0, sy = 0, sz = 0;                                                     \
    for (int64_t j = 0; j < n; ++j) {                                                       \
      if (j == i) continue;                                                                 \
      long double dx = (long double)px[j] - xi, dy = (long double)py[j] - yi;               \
      long double dz = (long double)pz[j] - zi;                                             \
      long double d2 = dx * dx + dy * dy + dz * dz + e2;                                    \
      long double w = (long double)m[j] / (d2 * sqrtl(d2));                                 \
      sx += dx * w; sy += dy * w; sz += dz * w;                                             \
    }                                                                                       \
    out3[3 * r + 0] = (double)(sx * (long double)g);                                        \
    out3[3 * r + 1] = (double)(sy * (long double)g);                                        \
    out3[3 * r + 2] = (double)(sz * (long double)g);                                        \
  }                                                                                         \
}
DEFINE_ROWS_LD(double, f64)
DEFINE_ROWS_LD(float, f32)

/* Physics diagnostics -- validation.py:134-145: kinetic energy, softened     */
/* potential energy -G sum_{i<j} m_i m_j / sqrt(d2 + eps2), momentum.  Sums   */
/* are long double per row, rows combined in ascending i.                    */
ORC_EXPORT void orc_diagnostics_f64(const double* px, const double* py, const double* pz,
                                    const double* vx, const double* vy, const double* vz,
                                    const double* m, int64_t n, double g, double eps2,
                                    int threads, double* out6) {
  if (threads < 1) threads = 1;
  long double* rowpe = (long double*)calloc((size_t)n, sizeof(long double));
  if (!rowpe) { for (int k = 0; k < 6; ++k) out6[k] = NAN; return; }
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads)
  for (int64_t i = 0; i < n - 1; ++i) {
    long double s = 0;
    for (int64_t j = i + 1; j < n; ++j) {
      long double dx = (long double)px[j] - px[i], dy = (long double)py[j] - py[i];
      long double dz = (long double)pz[j] - pz[i];
      s += (long double)m[j] / sqrtl(dx * dx + dy * dy + dz * dz + (long double)eps2);
    }
    rowpe[i] = -(long double)g * (long double)m[i] * s;
  }
  long double ke = 0, pe = 0, mx = 0, my = 0, mz = 0;
  for (int64_t i = 0; i < n; ++i) {
    ke += 0.5L * m[i] * ((long double)vx[i] * vx[i] + (long double)vy[i] * vy[i] +
                         (long double)vz[i] * vz[i]);
    pe += rowpe[i];
    mx += (long double)m[i] * vx[i]; my += (long double)m[i] * vy[i];
    mz += (long double)m[i] * vz[i];
  }
  free(rowpe);
  out6[0] = (double)ke; out6[1] = (double)pe; out6[2] = (double)mx;
  out6[3] = (double)my; out6[4] = (double)mz; out6[5] = (double)(ke + pe);
}

ORC_EXPORT int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
