/* pyfast.c — CPython entry for eager collectives: `_patfast.all_gather(...)` and
 * `_patfast.reduce_scatter(...)` take plain integers (device pointers, counts, stream handles)
 * or sequences of them and call patAllGather / patReduceScatter directly, instead of building
 * ctypes pointer arrays per call (comm.py). The C ABI's function addresses are handed over once
 * by `bind()` from the ctypes-loaded libpatb200.so, so this module links against nothing but
 * Python. Returns the patResult_t code; comm.py raises on non-zero like the ctypes path. */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

#define MAXR 8

typedef int (*coll_fn)(void*, const void* const*, void* const*, size_t, int, const void* const*);
typedef int (*rs_fn)(void*, const void* const*, void* const*, size_t, int, int, const void* const*);

static coll_fn g_ag = NULL;
static rs_fn g_rs = NULL;

static PyObject* bind(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 2) {
    PyErr_SetString(PyExc_TypeError, "bind(patAllGather address, patReduceScatter address)");
    return NULL;
  }
  void* a = PyLong_AsVoidPtr(args[0]);
  void* b = PyLong_AsVoidPtr(args[1]);
  if (PyErr_Occurred()) return NULL;
  g_ag = (coll_fn)a;
  g_rs = (rs_fn)b;
  Py_RETURN_NONE;
}

/* An int or a sequence of ints -> out[0..n); returns the element count or -1. */
static Py_ssize_t ptrs(PyObject* o, void** out) {
  if (PyLong_Check(o)) {
    out[0] = PyLong_AsVoidPtr(o);
    return PyErr_Occurred() ? -1 : 1;
  }
  PyObject* seq = PySequence_Fast(o, "expected an int or a sequence of ints");
  if (!seq) return -1;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  if (n > MAXR) {
    Py_DECREF(seq);
    PyErr_SetString(PyExc_ValueError, "more than 8 local ranks");
    return -1;
  }
  PyObject** items = PySequence_Fast_ITEMS(seq);
  for (Py_ssize_t i = 0; i < n; ++i) {
    out[i] = PyLong_AsVoidPtr(items[i]);
    if (PyErr_Occurred()) {
      Py_DECREF(seq);
      return -1;
    }
  }
  Py_DECREF(seq);
  return n;
}

/* all_gather(comm, send, recv, count, dtype, stream) */
static PyObject* all_gather(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 6) {
    PyErr_SetString(PyExc_TypeError, "all_gather(comm, send, recv, count, dtype, stream)");
    return NULL;
  }
  if (!g_ag) {
    PyErr_SetString(PyExc_RuntimeError, "_patfast not bound");
    return NULL;
  }
  void *s[MAXR] = {0}, *r[MAXR] = {0}, *st[MAXR] = {0}; /* short lists: the ABI sees NULL buffers */
  void* comm = PyLong_AsVoidPtr(args[0]);
  const size_t count = PyLong_AsSize_t(args[3]);
  const int dtype = (int)PyLong_AsLong(args[4]);
  if (PyErr_Occurred()) return NULL;
  const Py_ssize_t ns = ptrs(args[1], s), nr = ptrs(args[2], r), nst = ptrs(args[5], st);
  if (ns < 0 || nr < 0 || nst < 0) return NULL;
  if (ns != nr || ns != nst) {
    PyErr_SetString(PyExc_ValueError, "send, recv and stream lists differ in length");
    return NULL;
  }
  int rc;
  Py_BEGIN_ALLOW_THREADS rc = g_ag(comm, (const void* const*)s, (void* const*)r, count, dtype, (const void* const*)st);
  Py_END_ALLOW_THREADS return PyLong_FromLong(rc);
}

/* reduce_scatter(comm, send, recv, count, dtype, op, stream) */
static PyObject* reduce_scatter(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 7) {
    PyErr_SetString(PyExc_TypeError, "reduce_scatter(comm, send, recv, count, dtype, op, stream)");
    return NULL;
  }
  if (!g_rs) {
    PyErr_SetString(PyExc_RuntimeError, "_patfast not bound");
    return NULL;
  }
  void *s[MAXR] = {0}, *r[MAXR] = {0}, *st[MAXR] = {0}; /* short lists: the ABI sees NULL buffers */
  void* comm = PyLong_AsVoidPtr(args[0]);
  const size_t count = PyLong_AsSize_t(args[3]);
  const int dtype = (int)PyLong_AsLong(args[4]);
  const int op = (int)PyLong_AsLong(args[5]);
  if (PyErr_Occurred()) return NULL;
  const Py_ssize_t ns = ptrs(args[1], s), nr = ptrs(args[2], r), nst = ptrs(args[6], st);
  if (ns < 0 || nr < 0 || nst < 0) return NULL;
  if (ns != nr || ns != nst) {
    PyErr_SetString(PyExc_ValueError, "send, recv and stream lists differ in length");
    return NULL;
  }
  int rc;
  Py_BEGIN_ALLOW_THREADS rc =
      g_rs(comm, (const void* const*)s, (void* const*)r, count, dtype, op, (const void* const*)st);
  Py_END_ALLOW_THREADS return PyLong_FromLong(rc);
}

static PyMethodDef methods[] = {
    {"bind", (PyCFunction)(void (*)(void))bind, METH_FASTCALL, "bind the C ABI entry points"},
    {"all_gather", (PyCFunction)(void (*)(void))all_gather, METH_FASTCALL, "patAllGather"},
    {"reduce_scatter", (PyCFunction)(void (*)(void))reduce_scatter, METH_FASTCALL, "patReduceScatter"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_patfast", NULL, -1, methods, NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__patfast(void) { return PyModule_Create(&module); }
