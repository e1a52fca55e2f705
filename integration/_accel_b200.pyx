# cython: language_level=3, boundscheck=False, wraparound=False
"""The Cython binding a maintainer would add to nbodybench (INTEGRATION.md §3):
the reference's backend protocol (_accel_cy.pyx:114,155,205,240 -- NAME,
accel_soa, accel_aos, step_soa, step_aos) over the C ABI of libnbody_b200.so,
with typed memoryviews exactly like the reference's own compiled backend.
Built by integration/build.py; exercised by tests/test_integration_binding.py."""

cdef extern from "nbody_b200.h":
    int nb_host_accel_soa_f32(const float*, const float*, const float*, const float*, long long,
                              double, double, int, long long, int, float*, float*, float*) nogil
    int nb_host_accel_soa_f64(const double*, const double*, const double*, const double*, long long,
                              double, double, int, long long, int, double*, double*, double*) nogil
    int nb_host_accel_aos_f32(const float*, const float*, long long, double, double,
                              float*, float*, float*) nogil
    int nb_host_accel_aos_f64(const double*, const double*, long long, double, double,
                              double*, double*, double*) nogil
    int nb_host_step_soa_f32(float*, float*, float*, float*, float*, float*, const float*, const float*,
                             const float*, long long, double, int) nogil
    int nb_host_step_soa_f64(double*, double*, double*, double*, double*, double*, const double*,
                             const double*, const double*, long long, double, int) nogil
    int nb_host_step_aos_f32(float*, float*, const float*, const float*, const float*, long long, double) nogil
    int nb_host_step_aos_f64(double*, double*, const double*, const double*, const double*, long long,
                             double) nogil
    const char* nb_last_error()

NAME = "b200"

ctypedef fused real:
    float
    double


cdef _check(int rc):
    if rc != 0:
        raise RuntimeError(nb_last_error().decode())


def accel_soa(real[::1] px, real[::1] py, real[::1] pz, real[::1] m, double g, double eps2,
              bint recip, Py_ssize_t block, int threads, real[::1] ax, real[::1] ay, real[::1] az):
    cdef int rc
    with nogil:
        if real is float:
            rc = nb_host_accel_soa_f32(&px[0], &py[0], &pz[0], &m[0], px.shape[0], g, eps2, recip, block,
                                       threads, &ax[0], &ay[0], &az[0])
        else:
            rc = nb_host_accel_soa_f64(&px[0], &py[0], &pz[0], &m[0], px.shape[0], g, eps2, recip, block,
                                       threads, &ax[0], &ay[0], &az[0])
    _check(rc)


def accel_aos(real[:, ::1] pos, real[::1] m, double g, double eps2, real[::1] ax, real[::1] ay,
              real[::1] az):
    cdef int rc
    with nogil:
        if real is float:
            rc = nb_host_accel_aos_f32(&pos[0, 0], &m[0], pos.shape[0], g, eps2, &ax[0], &ay[0], &az[0])
        else:
            rc = nb_host_accel_aos_f64(&pos[0, 0], &m[0], pos.shape[0], g, eps2, &ax[0], &ay[0], &az[0])
    _check(rc)


def step_soa(real[::1] px, real[::1] py, real[::1] pz, real[::1] vx, real[::1] vy, real[::1] vz,
             const real[::1] ax, const real[::1] ay, const real[::1] az, double dt, int threads):
    cdef int rc
    with nogil:
        if real is float:
            rc = nb_host_step_soa_f32(&px[0], &py[0], &pz[0], &vx[0], &vy[0], &vz[0], &ax[0], &ay[0],
                                      &az[0], px.shape[0], dt, threads)
        else:
            rc = nb_host_step_soa_f64(&px[0], &py[0], &pz[0], &vx[0], &vy[0], &vz[0], &ax[0], &ay[0],
                                      &az[0], px.shape[0], dt, threads)
    _check(rc)


def step_aos(real[:, ::1] pos, real[:, ::1] vel, const real[::1] ax, const real[::1] ay,
             const real[::1] az, double dt):
    cdef int rc
    with nogil:
        if real is float:
            rc = nb_host_step_aos_f32(&pos[0, 0], &vel[0, 0], &ax[0], &ay[0], &az[0], pos.shape[0], dt)
        else:
            rc = nb_host_step_aos_f64(&pos[0, 0], &vel[0, 0], &ax[0], &ay[0], &az[0], pos.shape[0], dt)
    _check(rc)
