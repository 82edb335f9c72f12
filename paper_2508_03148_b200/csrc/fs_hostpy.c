/* fs_hostpy.c -- CPython helper for the host side of a batch (not on the device
 * path): MetricsBundle.per_request for one instance,
 *   {request_id: {"ttft_s": a[o+i], "tpot_s": b[o+i], "e2e_s": c[o+i]}},
 * built directly from the batch's value lists (metrics.py:91-100 of the
 * reference builds the same dict request by request). api.metrics_many calls it
 * once per instance; at sweep scale (~260 K requests) the Python comprehension
 * was the largest host cost of simulate(). */
#define PY_SSIZE_T_CLEAN
#include <Python.h>

static PyObject *k_ttft, *k_tpot, *k_e2e;

static PyObject* per_request(PyObject* self, PyObject* args) {
  PyObject *ids, *a, *b, *c;
  Py_ssize_t o;
  if (!PyArg_ParseTuple(args, "O!O!O!O!n", &PyList_Type, &ids, &PyList_Type, &a, &PyList_Type,
                        &b, &PyList_Type, &c, &o))
    return NULL;
  const Py_ssize_t n = PyList_GET_SIZE(ids);
  if (o < 0 || o + n > PyList_GET_SIZE(a) || o + n > PyList_GET_SIZE(b) ||
      o + n > PyList_GET_SIZE(c)) {
    PyErr_SetString(PyExc_IndexError, "per_request: value lists shorter than offset + ids");
    return NULL;
  }
  PyObject* out = PyDict_New();
  if (!out) return NULL;
  for (Py_ssize_t i = 0; i < n; i++) {
    PyObject* in = PyDict_New();
    if (!in ||
        PyDict_SetItem(in, k_ttft, PyList_GET_ITEM(a, o + i)) < 0 ||
        PyDict_SetItem(in, k_tpot, PyList_GET_ITEM(b, o + i)) < 0 ||
        PyDict_SetItem(in, k_e2e, PyList_GET_ITEM(c, o + i)) < 0 ||
        PyDict_SetItem(out, PyList_GET_ITEM(ids, i), in) < 0) {
      Py_XDECREF(in);
      Py_DECREF(out);
      return NULL;
    }
    Py_DECREF(in);
  }
  return out;
}

static PyMethodDef methods[] = {
    {"per_request", per_request, METH_VARARGS,
     "per_request(ids, ttft, tpot, e2e, offset) -> {id: {'ttft_s', 'tpot_s', 'e2e_s'}}"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_fs_host", NULL, -1, methods};

PyMODINIT_FUNC PyInit__fs_host(void) {
  k_ttft = PyUnicode_InternFromString("ttft_s");
  k_tpot = PyUnicode_InternFromString("tpot_s");
  k_e2e = PyUnicode_InternFromString("e2e_s");
  if (!k_ttft || !k_tpot || !k_e2e) return NULL;
  return PyModule_Create(&module);
}
