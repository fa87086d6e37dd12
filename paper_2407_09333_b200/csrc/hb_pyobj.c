/* Host-side helper for the drop-in API: builds hash_batch's list[Digest].
 *
 * The reference's hash_batch returns one Python Digest object per message
 * (pkg/src/hetoc/crypto/batch.py:293-316); at 2^24 messages building those
 * objects costs far more than hashing them on the GPU (~70 %
 * of a 10^6 x 9 B batch already on the CPU path).  This builds the same
 * objects -- instances of the frozen dataclass `Digest` whose __dict__ holds
 * {"alg": alg, "data": <dlen bytes>}, exactly what its __init__ leaves -- in
 * one C loop over the digest array.  No hashing happens here.
 *
 *   _hb_pyobj.digest_list(Digest, alg: str, raw: bytes-like, dlen: int, count: int) -> list
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>

static PyObject* digest_list(PyObject* self, PyObject* args) {
    (void)self;
    PyTypeObject* cls = NULL;
    PyObject* alg = NULL;
    Py_buffer raw;
    Py_ssize_t dlen = 0, count = 0;
    if (!PyArg_ParseTuple(args, "O!Uy*nn", &PyType_Type, &cls, &alg, &raw, &dlen, &count)) return NULL;
    PyObject* list = NULL;
    PyObject* k_alg = NULL;
    PyObject* k_data = NULL;
    if (dlen <= 0 || count < 0 || raw.len < dlen * count) {
        PyErr_Format(PyExc_ValueError, "need %zd digests of %zd bytes, buffer holds %zd bytes", count, dlen, raw.len);
        goto done;
    }
    if (!(cls->tp_flags & Py_TPFLAGS_HEAPTYPE) || cls->tp_alloc == NULL) {
        PyErr_SetString(PyExc_TypeError, "cls must be a Python class");
        goto done;
    }
    k_alg = PyUnicode_InternFromString("alg");
    k_data = PyUnicode_InternFromString("data");
    list = PyList_New(count);
    if (!k_alg || !k_data || !list) goto fail;
    const char* p = (const char*)raw.buf;
    /* The new objects hold no reference cycles; keep the cyclic collector
     * from rescanning the growing list every few hundred allocations. */
    const int gc_was_enabled = PyGC_Disable();
    int rc = 0;
    for (Py_ssize_t i = 0; i < count && rc == 0; ++i) {
        PyObject* o = cls->tp_alloc(cls, 0); /* object.__new__(cls): no __init__ / __post_init__ */
        if (!o) {
            rc = -1;
            break;
        }
        PyList_SET_ITEM(list, i, o); /* the list owns it from here */
        /* object.__setattr__ (the generic slot, not the frozen class's
         * __setattr__): the instance's own attribute storage, as __init__ fills it */
        PyObject* b = PyBytes_FromStringAndSize(p + i * dlen, dlen);
        rc = b ? PyObject_GenericSetAttr(o, k_alg, alg) : -1;
        if (rc == 0) rc = PyObject_GenericSetAttr(o, k_data, b);
        Py_XDECREF(b);
    }
    if (gc_was_enabled) PyGC_Enable();
    if (rc == 0) goto done;
fail:
    Py_CLEAR(list);
done:
    Py_XDECREF(k_alg);
    Py_XDECREF(k_data);
    PyBuffer_Release(&raw);
    return list;
}

/* addr(obj) -> int: the address of a C-contiguous buffer (numpy array,
 * bytes, ...) -- what `ndarray.ctypes.data` returns, without building the
 * ctypes helper object (1.4 us per call, several per small engine call).  The
 * caller keeps obj alive while the address is in use. */
static PyObject* addr(PyObject* self, PyObject* obj) {
    (void)self;
    Py_buffer view;
    if (PyObject_GetBuffer(obj, &view, PyBUF_ANY_CONTIGUOUS) < 0) return NULL;
    PyObject* r = PyLong_FromVoidPtr(view.buf);
    PyBuffer_Release(&view);
    return r;
}

static PyMethodDef methods[] = {
    {"digest_list", digest_list, METH_VARARGS, "Digest objects over consecutive dlen-byte slices of a buffer."},
    {"addr", addr, METH_O, "Address of a contiguous buffer (ndarray.ctypes.data without the ctypes object)."},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {
    PyModuleDef_HEAD_INIT, "_hb_pyobj", NULL, -1, methods, NULL, NULL, NULL, NULL,
};

PyMODINIT_FUNC PyInit__hb_pyobj(void) { return PyModule_Create(&module); }
