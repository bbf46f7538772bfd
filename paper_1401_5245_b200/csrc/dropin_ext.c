/* _dropin -- CPython binding of the drop-in's per-image hot call.
 *
 * `detect_edges_mask(BitImage.from_array(a)).words` on a small host image
 * (bitimage.py:122-147 + SPEC.md:165-168) is one native call,
 * be_host_detect_u64_staged (include/bitedge.h); at C1/C2 sizes the whole call
 * is ~12 us of GPU round trip, so the binding's own overhead matters: ctypes
 * spends ~5 us converting 13 arguments and building the result.  This module
 * does it with METH_FASTCALL and the numpy C API, releases the GIL around the
 * native call, and keeps the calling thread's page-locked staging pair and
 * private stream (allocated by torch in Python, registered once per thread with
 * set_stage) in thread-local storage.
 *
 *   set_stage(in_ptr, in_bytes, out_ptr, out_bytes, stream, device) -> None
 *   detect_small(pix, fill_bit, edgeset, device) -> uint64 [H, ceil(W/64)] (read-only)
 *                                                  or None if this thread's stage
 *                                                  is missing / too small / on
 *                                                  another device
 */
#define PY_SSIZE_T_CLEAN
#define NPY_NO_DEPRECATED_API NPY_1_7_API_VERSION
#include <Python.h>
#include <numpy/arrayobject.h>
#include <stdint.h>

#include "../../include/bitedge.h"

typedef struct {
    uint8_t *in;
    int64_t in_n;
    uint64_t *out;
    int64_t out_n;
    void *stream;
    long device;
    int set;
} stage_t;

static _Thread_local stage_t g_stage;

static PyObject *set_stage(PyObject *self, PyObject *const *args, Py_ssize_t nargs) {
    (void)self;
    if (nargs != 6) {
        PyErr_SetString(PyExc_TypeError, "set_stage takes 6 arguments");
        return NULL;
    }
    stage_t s;
    s.in = (uint8_t *)PyLong_AsVoidPtr(args[0]);
    s.in_n = PyLong_AsLongLong(args[1]);
    s.out = (uint64_t *)PyLong_AsVoidPtr(args[2]);
    s.out_n = PyLong_AsLongLong(args[3]);
    s.stream = PyLong_AsVoidPtr(args[4]);
    s.device = PyLong_AsLong(args[5]);
    if (PyErr_Occurred()) return NULL;
    s.set = 1;
    g_stage = s;
    Py_RETURN_NONE;
}

static PyObject *detect_small(PyObject *self, PyObject *const *args, Py_ssize_t nargs) {
    (void)self;
    if (nargs != 4) {
        PyErr_SetString(PyExc_TypeError, "detect_small takes 4 arguments");
        return NULL;
    }
    if (!PyArray_Check(args[0])) {
        PyErr_SetString(PyExc_TypeError, "pix must be a numpy array");
        return NULL;
    }
    PyArrayObject *pix = (PyArrayObject *)args[0];
    const long fill = PyLong_AsLong(args[1]);
    const long edgeset = PyLong_AsLong(args[2]);
    const long device = PyLong_AsLong(args[3]);
    if (PyErr_Occurred()) return NULL;
    if (PyArray_NDIM(pix) != 2 || PyArray_TYPE(pix) != NPY_UINT8 || PyArray_STRIDE(pix, 1) != 1 ||
        PyArray_STRIDE(pix, 0) < PyArray_DIM(pix, 1)) {
        PyErr_SetString(PyExc_ValueError, "pix must be a uint8 [H, W] array with contiguous rows");
        return NULL;
    }
    const int64_t h = PyArray_DIM(pix, 0), w = PyArray_DIM(pix, 1);
    const int64_t wp = (w + 63) / 64;
    const stage_t st = g_stage;
    if (!st.set || st.device != device || st.in_n < h * w || st.out_n < h * wp * 8 + 128)
        Py_RETURN_NONE;                          /* Python (re)allocates the stage */
    npy_intp dims[2] = {(npy_intp)h, (npy_intp)wp};
    PyArrayObject *words = (PyArrayObject *)PyArray_SimpleNew(2, dims, NPY_UINT64);
    if (words == NULL) return NULL;
    int rc;
    Py_BEGIN_ALLOW_THREADS
    rc = be_host_detect_u64_staged((const uint8_t *)PyArray_DATA(pix), PyArray_STRIDE(pix, 0), h,
                                   w, (int)fill, (int)edgeset, st.in, st.in_n, st.out, st.out_n,
                                   NULL, (uint64_t *)PyArray_DATA(words), st.stream);
    Py_END_ALLOW_THREADS
    if (rc != 0) {
        Py_DECREF(words);
        PyErr_Format(rc < 0 ? PyExc_ValueError : PyExc_RuntimeError, "%s%s",
                     rc < 0 ? "" : "CUDA error: ", be_last_error());
        return NULL;
    }
    PyArray_CLEARFLAGS(words, NPY_ARRAY_WRITEABLE);
    return (PyObject *)words;
}

static PyMethodDef methods[] = {
    {"set_stage", (PyCFunction)(void (*)(void))set_stage, METH_FASTCALL,
     "Register this thread's page-locked staging pair and stream."},
    {"detect_small", (PyCFunction)(void (*)(void))detect_small, METH_FASTCALL,
     "One small host image: pack + edges on the device, uint64 words back."},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_dropin", NULL, -1, methods,
                                    NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__dropin(void) {
    import_array();
    return PyModule_Create(&module);
}
