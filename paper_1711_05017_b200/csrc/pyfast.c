/* pyfast.c -- CPython binding of the haptic-session query (gf_server_query),
 * the one call a real-time loop makes per frame (backend.cascade in a
 * session, energy.evaluate under haptic_session; the reference's per-frame
 * call is backend.cascade -> _core.cascade_3d, backend.py:153-164).
 *
 * ctypes costs ~2 us per frame on this path (argument marshalling, numpy
 * copies into staging buffers, the result copy); this module reads R and
 * t_eff straight from the caller's float64 buffers and returns a fresh
 * complex128[7] array.  It does not link the engine: the address of
 * gf_server_query is handed over once from the ctypes-loaded library
 * (bind()), so both paths share one library instance and its server table.
 * Inputs it cannot read in place (wrong dtype, not contiguous, wrong size)
 * return None and the caller takes the ctypes path. */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_1_7_API_VERSION
#include <numpy/arrayobject.h>
#include <stdint.h>
#include <string.h>

typedef int (*server_query_fn)(uint64_t, const double*, const double*, double*);
static server_query_fn g_query = NULL;

static PyObject* bind(PyObject* self, PyObject* args) {
  unsigned long long addr;
  if (!PyArg_ParseTuple(args, "K", &addr)) return NULL;
  g_query = (server_query_fn)(uintptr_t)addr;
  Py_RETURN_NONE;
}

/* a C-contiguous float64 buffer of exactly n doubles, or NULL */
static const double* f64_view(PyObject* o, Py_ssize_t n) {
  if (!PyArray_Check(o)) return NULL;
  PyArrayObject* a = (PyArrayObject*)o;
  if (PyArray_TYPE(a) != NPY_FLOAT64 || !PyArray_IS_C_CONTIGUOUS(a) || PyArray_SIZE(a) != n) return NULL;
  return (const double*)PyArray_DATA(a);
}

/* server_query(server_id, R, t_eff) -> complex128[7] | int rc | None */
static PyObject* server_query(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 3) {
    PyErr_SetString(PyExc_TypeError, "server_query(server_id, R, t_eff)");
    return NULL;
  }
  const unsigned long long id = PyLong_AsUnsignedLongLong(args[0]);
  if (PyErr_Occurred()) return NULL;
  const double* R = f64_view(args[1], 9);
  const double* t = f64_view(args[2], 3);
  if (!R || !t || !g_query) Py_RETURN_NONE;
  double out[14];
  int rc;
  Py_BEGIN_ALLOW_THREADS  /* the wait spins on host-mapped memory: let other threads run */
  rc = g_query((uint64_t)id, R, t, out);
  Py_END_ALLOW_THREADS
  if (rc) return PyLong_FromLong(rc);
  npy_intp dim = 7;
  PyObject* res = PyArray_SimpleNew(1, &dim, NPY_COMPLEX128);
  if (!res) return NULL;
  memcpy(PyArray_DATA((PyArrayObject*)res), out, sizeof out);
  return res;
}

static PyMethodDef methods[] = {
    {"bind", bind, METH_VARARGS, "bind(address of gf_server_query)"},
    {"server_query", (PyCFunction)(void (*)(void))server_query, METH_FASTCALL,
     "server_query(server_id, R, t_eff) -> complex128[7], or the int return code, or None"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_gf_fast", NULL, -1, methods};

PyMODINIT_FUNC PyInit__gf_fast(void) {
  import_array();
  return PyModule_Create(&module);
}
