/* CPython binding of simulate()'s single-GPU path: paper_2203_08263_b200._hostpath.
 *
 * The reference crosses into compiled code through Cython typed memoryviews
 * (/root/reference/pkg/src/nbodybench/kernels/_accel_cy.pyx:114-152), which
 * read the buffer pointers in C.  Through ctypes every NumPy pointer costs
 * ~2 us of Python (arr.ctypes.data) -- 16 us of a 100 us C1 simulate for the
 * eight arrays -- so this module takes the arrays through the buffer protocol
 * and calls nb_host_simulate_f32/f64 of the ALREADY LOADED libnbody_b200.so
 * (function addresses handed over by _native.lib(): one library per process,
 * NB_LIB_PATH variants included) with the GIL released.
 *
 *   bind(addr_f32, addr_f64)
 *   simulate(px, py, pz, m, vx, vy, vz, out6, g, dt, eps2, steps, device, itemsize) -> rc
 *
 * Every array must be C-contiguous with the float32 (itemsize 4) or float64
 * (8) item type the system precision names; inputs hold n elements, out6
 * holds 6*n.  Returns the C ABI's status (the caller raises with nb_last_error
 * on nonzero); TypeError for a buffer of another item type (the caller then
 * raises the reference's dtype ValueError), ValueError for bad lengths,
 * RuntimeError when unbound. */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

typedef int (*sim_f32_t)(const float*, const float*, const float*, const float*, const float*, const float*,
                         const float*, int64_t, double, double, double, int64_t, float*, int);
typedef int (*sim_f64_t)(const double*, const double*, const double*, const double*, const double*,
                         const double*, const double*, int64_t, double, double, double, int64_t, double*, int);

static sim_f32_t g_f32 = NULL;
static sim_f64_t g_f64 = NULL;

static PyObject* bind(PyObject* self, PyObject* args) {
  unsigned long long a32 = 0, a64 = 0;
  (void)self;
  if (!PyArg_ParseTuple(args, "KK", &a32, &a64)) return NULL;
  g_f32 = (sim_f32_t)(uintptr_t)a32;
  g_f64 = (sim_f64_t)(uintptr_t)a64;
  Py_RETURN_NONE;
}

static int item_kind(const Py_buffer* v) {
  /* 4: float32, 8: float64, 0: anything else */
  const char* f = v->format ? v->format : "B";
  if (*f == '<' || *f == '=' || *f == '@') ++f;
  if (f[0] == 'f' && f[1] == 0 && v->itemsize == 4) return 4;
  if (f[0] == 'd' && f[1] == 0 && v->itemsize == 8) return 8;
  return 0;
}

static PyObject* simulate(PyObject* self, PyObject* args) {
  PyObject* objs[8];
  double g, dt, eps2;
  long long steps;
  int device, want;
  (void)self;
  if (!PyArg_ParseTuple(args, "OOOOOOOOdddLii", &objs[0], &objs[1], &objs[2], &objs[3], &objs[4], &objs[5],
                        &objs[6], &objs[7], &g, &dt, &eps2, &steps, &device, &want))
    return NULL;
  if (!g_f32 || !g_f64) {
    PyErr_SetString(PyExc_RuntimeError, "_hostpath is not bound to libnbody_b200.so (call bind first)");
    return NULL;
  }
  Py_buffer v[8];
  int got = 0, kind = want, rc = 0;
  Py_ssize_t n = -1;
  for (; got < 8; ++got) {
    const int flags = got == 7 ? (PyBUF_C_CONTIGUOUS | PyBUF_FORMAT | PyBUF_WRITABLE)
                               : (PyBUF_C_CONTIGUOUS | PyBUF_FORMAT);
    if (PyObject_GetBuffer(objs[got], &v[got], flags) != 0) goto fail;
    const int k = item_kind(&v[got]);
    if (k != kind) {
      ++got;
      PyErr_SetString(PyExc_TypeError, "simulate buffers must all have the system precision's float type");
      goto fail;
    }
    const Py_ssize_t len = v[got].len / v[got].itemsize;
    if (got < 7) {
      if (n < 0) n = len;
      if (len != n) {
        ++got;
        PyErr_SetString(PyExc_ValueError, "simulate input columns must all hold n elements");
        goto fail;
      }
    } else if (len != 6 * n) {
      ++got;
      PyErr_SetString(PyExc_ValueError, "simulate output block must hold 6*n elements");
      goto fail;
    }
  }
  Py_BEGIN_ALLOW_THREADS
  if (kind == 4)
    rc = g_f32((const float*)v[0].buf, (const float*)v[1].buf, (const float*)v[2].buf, (const float*)v[3].buf,
               (const float*)v[4].buf, (const float*)v[5].buf, (const float*)v[6].buf, (int64_t)n, g, dt, eps2,
               (int64_t)steps, (float*)v[7].buf, device);
  else
    rc = g_f64((const double*)v[0].buf, (const double*)v[1].buf, (const double*)v[2].buf,
               (const double*)v[3].buf, (const double*)v[4].buf, (const double*)v[5].buf,
               (const double*)v[6].buf, (int64_t)n, g, dt, eps2, (int64_t)steps, (double*)v[7].buf, device);
  Py_END_ALLOW_THREADS
  for (int k = 0; k < 8; ++k) PyBuffer_Release(&v[k]);
  return PyLong_FromLong(rc);
fail:
  for (int k = 0; k < got; ++k) PyBuffer_Release(&v[k]);
  return NULL;
}

static PyMethodDef methods[] = {
    {"bind", bind, METH_VARARGS, "bind(addr_f32, addr_f64): nb_host_simulate_* of the loaded library"},
    {"simulate", simulate, METH_VARARGS,
     "simulate(px, py, pz, m, vx, vy, vz, out6, g, dt, eps2, steps, device, itemsize) -> C ABI status"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_hostpath", NULL, -1, methods,
                                    NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__hostpath(void) { return PyModule_Create(&module); }
