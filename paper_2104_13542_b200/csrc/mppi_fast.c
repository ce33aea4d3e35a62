/* mppi_fast.c — CPython entry for the single-controller latency path.
 *
 * Controller.control_step (reference controller.py:198-260) hands the joint
 * state to mppi_step (include/mppi_b200.h) once per step. Through ctypes that
 * call costs two staging copies (np.copyto of theta / theta_dot) plus the
 * ctypes argument conversion, ~1.5 us of a ~33 us end-to-end step. Here the
 * caller's float64 arrays are read through the buffer protocol and their
 * addresses go straight to mppi_step (which copies the 2d doubles into the
 * plan's pinned staging rows itself); anything that is not a C-contiguous
 * float64 vector of length d returns NotImplemented and the caller takes the
 * ctypes path, which converts. Plain C-ABI call: no torch, no numpy headers.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>

typedef int (*mppi_step_fn)(void* plan, const double* theta, const double* theta_dot, double* command_out,
                            void* info_out);

static int vec_f64(PyObject* o, Py_buffer* b, Py_ssize_t d) {
  if (PyObject_GetBuffer(o, b, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT) < 0) {
    PyErr_Clear();
    return 0;
  }
  if (b->format == NULL || b->format[0] != 'd' || b->format[1] != '\0' || b->len != d * (Py_ssize_t)sizeof(double)) {
    PyBuffer_Release(b);
    return 0;
  }
  return 1;
}

/* step(fn, plan, theta, theta_dot, command_addr, info_addr, d) -> status int
 * (or NotImplemented when theta / theta_dot need a conversion) */
static PyObject* fast_step(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 7) {
    PyErr_SetString(PyExc_TypeError, "step(fn, plan, theta, theta_dot, command_addr, info_addr, d)");
    return NULL;
  }
  mppi_step_fn fn = (mppi_step_fn)PyLong_AsVoidPtr(args[0]);
  void* plan = PyLong_AsVoidPtr(args[1]);
  double* cmd = (double*)PyLong_AsVoidPtr(args[4]);
  void* info = PyLong_AsVoidPtr(args[5]);
  const Py_ssize_t d = PyLong_AsSsize_t(args[6]);
  if (PyErr_Occurred()) return NULL;
  if (fn == NULL || plan == NULL) {
    PyErr_SetString(PyExc_ValueError, "null mppi_step or plan");
    return NULL;
  }
  Py_buffer bt, bv;
  if (!vec_f64(args[2], &bt, d)) Py_RETURN_NOTIMPLEMENTED;
  if (!vec_f64(args[3], &bv, d)) {
    PyBuffer_Release(&bt);
    Py_RETURN_NOTIMPLEMENTED;
  }
  int rc;
  Py_BEGIN_ALLOW_THREADS  /* the call waits for the device step, as the ctypes call did */
  rc = fn(plan, (const double*)bt.buf, (const double*)bv.buf, cmd, info);
  Py_END_ALLOW_THREADS
  PyBuffer_Release(&bv);
  PyBuffer_Release(&bt);
  return PyLong_FromLong(rc);
}

static PyMethodDef methods[] = {
    {"step", (PyCFunction)(void (*)(void))fast_step, METH_FASTCALL, "mppi_step on caller float64 vectors"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_mppi_fast", NULL, -1, methods};

PyMODINIT_FUNC PyInit__mppi_fast(void) { return PyModule_Create(&module); }
