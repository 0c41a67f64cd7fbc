/* _dagrt_fastcall: CPython METH_FASTCALL entry points for the three calls a
 * benchmark step makes per DAG (a launch batch, host reads, a graph run).
 * Argument marshalling only -- every call goes straight to libdagrt.so's
 * C ABI (include/dagrt.h); ctypes costs ~1-2 us per call on the B200 box's
 * host, comparable to a kernel launch.  Arguments are plain integers
 * (addresses and handles), results the dagrt_status. */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

#include "dagrt.h"

static int as_u64(PyObject* o, unsigned long long* v) {
  *v = PyLong_AsUnsignedLongLong(o);
  return !(*v == (unsigned long long)-1 && PyErr_Occurred());
}

/* launch_batch(ctx, descs_address, n) -> status */
static PyObject* fc_launch_batch(PyObject* self, PyObject* const* args, Py_ssize_t n) {
  unsigned long long c, d, k;
  if (n != 3 || !as_u64(args[0], &c) || !as_u64(args[1], &d) || !as_u64(args[2], &k)) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_TypeError, "launch_batch(ctx, descs, n)");
    return NULL;
  }
  return PyLong_FromLong(dagrt_launch_batch((dagrt_ctx)(uintptr_t)c,
                                            (const dagrt_launch_desc*)(uintptr_t)d, (int32_t)k));
}

/* host_read(ctx, array, off, nbytes, dst_address) -> status */
static PyObject* fc_host_read(PyObject* self, PyObject* const* args, Py_ssize_t n) {
  unsigned long long v[5];
  if (n != 5) {
    PyErr_SetString(PyExc_TypeError, "host_read(ctx, array, off, nbytes, dst)");
    return NULL;
  }
  for (int i = 0; i < 5; ++i)
    if (!as_u64(args[i], &v[i])) return NULL;
  return PyLong_FromLong(dagrt_host_read((dagrt_ctx)(uintptr_t)v[0], (dagrt_array)v[1], (size_t)v[2],
                                         (size_t)v[3], (void*)(uintptr_t)v[4]));
}

/* graph_run(ctx, graph, wait) -> status */
static PyObject* fc_graph_run(PyObject* self, PyObject* const* args, Py_ssize_t n) {
  unsigned long long c, g, w;
  if (n != 3 || !as_u64(args[0], &c) || !as_u64(args[1], &g) || !as_u64(args[2], &w)) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_TypeError, "graph_run(ctx, graph, wait)");
    return NULL;
  }
  return PyLong_FromLong(dagrt_graph_run((dagrt_ctx)(uintptr_t)c, (dagrt_graph)(uintptr_t)g, (int32_t)w));
}

static PyMethodDef kMethods[] = {
    {"launch_batch", (PyCFunction)(void (*)(void))fc_launch_batch, METH_FASTCALL, "dagrt_launch_batch"},
    {"host_read", (PyCFunction)(void (*)(void))fc_host_read, METH_FASTCALL, "dagrt_host_read"},
    {"graph_run", (PyCFunction)(void (*)(void))fc_graph_run, METH_FASTCALL, "dagrt_graph_run"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_dagrt_fastcall", NULL, -1, kMethods};

PyMODINIT_FUNC PyInit__dagrt_fastcall(void) { return PyModule_Create(&kModule); }
