/* pyfast.c -- CPython fast path for the drop-in backend calls.
 *
 * backend_cuda.cbc_encrypt / cbc_decrypt (the 7-argument contract of
 * _kernel.pyx:12-18 / :57-63) and encrypt_shared_iv spend most of a small
 * call's host time in Python: seven __array_interface__ lookups and buffer
 * checks (~1-3 us each).  This module takes the same arguments through the
 * buffer protocol, checks exactly what backend_cuda._check_args checks, and
 * calls the C ABI (include/gaes_b200.h) with the GIL released.  When any
 * argument is not a plain C-contiguous uint8 buffer of the expected shape it
 * returns None without side effects, and the Python path runs -- and raises
 * the reference's error messages.  It never computes anything itself.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

#include "gaes_b200.h"

typedef struct {
  Py_buffer b;
  int held;
} Buf;

static void release(Buf* bufs, int n) {
  for (int i = 0; i < n; i++)
    if (bufs[i].held) PyBuffer_Release(&bufs[i].b);
}

/* uint8 ("B" or unspecified format), C-contiguous, ndim dimensions. */
static int get_u8(PyObject* o, Buf* out, int ndim, int writable) {
  const int flags = PyBUF_C_CONTIGUOUS | PyBUF_FORMAT | (writable ? PyBUF_WRITABLE : 0);
  if (PyObject_GetBuffer(o, &out->b, flags) != 0) {
    PyErr_Clear();
    return 0;
  }
  out->held = 1;
  const char* f = out->b.format;
  if (out->b.itemsize != 1 || out->b.ndim != ndim || (f && !(f[0] == 'B' && f[1] == 0))) return 0;
  return 1;
}

/* cbc(decrypt, data, ivs, round_keys, sbox, mix_lut, shift_src, out) -> rc or None */
static PyObject* cbc(PyObject* self, PyObject* args) {
  int dec;
  PyObject *o[7];
  if (!PyArg_ParseTuple(args, "pOOOOOOO", &dec, &o[0], &o[1], &o[2], &o[3], &o[4], &o[5], &o[6])) return NULL;
  Buf b[7];
  memset(b, 0, sizeof(b));
  static const int ndim[7] = {2, 2, 2, 1, 3, 1, 2};
  int ok = 1;
  for (int i = 0; i < 7 && ok; i++) ok = get_u8(o[i], &b[i], ndim[i], i == 6);
  if (ok) {
    const Py_ssize_t* ds = b[0].b.shape;
    const Py_ssize_t n = ds[0], m = ds[1];
    ok = b[6].b.shape[0] == n && b[6].b.shape[1] == m && b[1].b.shape[0] == n && b[1].b.shape[1] == 16 &&
         b[2].b.shape[0] == 11 && b[2].b.shape[1] == 16 && b[3].b.shape[0] == 256 && b[4].b.shape[0] == 4 &&
         b[4].b.shape[1] == 4 && b[4].b.shape[2] == 256 && b[5].b.shape[0] == 16 && (n == 0 || (m > 0 && m % 16 == 0));
    const uint8_t* perm = (const uint8_t*)b[5].b.buf;
    for (int i = 0; i < 16 && ok; i++) ok = perm[i] < 16;
    if (ok) {
      int rc = 0;
      if (n) {
        Py_BEGIN_ALLOW_THREADS
        rc = (dec ? gaes_cbc_decrypt : gaes_cbc_encrypt)(
            (const uint8_t*)b[0].b.buf, (const uint8_t*)b[1].b.buf, (size_t)n, (size_t)m, (const uint8_t*)b[2].b.buf,
            (const uint8_t*)b[3].b.buf, (const uint8_t*)b[4].b.buf, perm, (uint8_t*)b[6].b.buf);
        Py_END_ALLOW_THREADS
      }
      release(b, 7);
      return PyLong_FromLong(rc);
    }
  }
  release(b, 7);
  Py_RETURN_NONE;
}

/* shared_iv(decrypt, data, iv(16 bytes-like), round_keys(176 bytes-like), out) -> rc or None */
static PyObject* shared_iv(PyObject* self, PyObject* args) {
  int dec;
  PyObject *od, *oiv, *ork, *oout;
  if (!PyArg_ParseTuple(args, "pOOOO", &dec, &od, &oiv, &ork, &oout)) return NULL;
  Buf b[4];
  memset(b, 0, sizeof(b));
  int ok = get_u8(od, &b[0], 2, 0) && get_u8(oout, &b[3], 2, 1);
  /* IV and round keys: any C-contiguous byte buffer (bytes, uint8 arrays) */
  for (int i = 1; i <= 2 && ok; i++) {
    ok = PyObject_GetBuffer(i == 1 ? oiv : ork, &b[i].b, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT) == 0;
    if (!ok) {
      PyErr_Clear();
      break;
    }
    b[i].held = 1;
    const char* f = b[i].b.format;
    ok = b[i].b.itemsize == 1 && (!f || (f[0] == 'B' && f[1] == 0));
  }
  if (ok) {
    const Py_ssize_t n = b[0].b.shape[0], m = b[0].b.shape[1];
    ok = b[1].b.len == 16 && b[2].b.len == 176 && b[3].b.shape[0] == n && b[3].b.shape[1] == m;
    if (ok) {
      int rc = 0;
      if (n) {
        Py_BEGIN_ALLOW_THREADS
        rc = (dec ? gaes_decrypt_shared_iv : gaes_encrypt_shared_iv)(
            (const uint8_t*)b[0].b.buf, (size_t)n, (size_t)m, (const uint8_t*)b[1].b.buf, (const uint8_t*)b[2].b.buf,
            (uint8_t*)b[3].b.buf);
        Py_END_ALLOW_THREADS
      }
      release(b, 4);
      return PyLong_FromLong(rc);
    }
  }
  release(b, 4);
  Py_RETURN_NONE;
}

/* cbc_std(decrypt, data, ivs, round_keys, out) -> rc or None: the same with
 * the device GF layer's standard tables (gaes_cbc_{en,de}crypt_std) */
static PyObject* cbc_std(PyObject* self, PyObject* args) {
  int dec;
  PyObject *o[4];
  if (!PyArg_ParseTuple(args, "pOOOO", &dec, &o[0], &o[1], &o[2], &o[3])) return NULL;
  Buf b[4];
  memset(b, 0, sizeof(b));
  static const int ndim[4] = {2, 2, 2, 2};
  int ok = 1;
  for (int i = 0; i < 4 && ok; i++) ok = get_u8(o[i], &b[i], ndim[i], i == 3);
  if (ok) {
    const Py_ssize_t n = b[0].b.shape[0], m = b[0].b.shape[1];
    ok = b[3].b.shape[0] == n && b[3].b.shape[1] == m && b[1].b.shape[0] == n && b[1].b.shape[1] == 16 &&
         b[2].b.shape[0] == 11 && b[2].b.shape[1] == 16;
    if (ok) {
      int rc = 0;
      if (n) {
        Py_BEGIN_ALLOW_THREADS
        rc = (dec ? gaes_cbc_decrypt_std : gaes_cbc_encrypt_std)((const uint8_t*)b[0].b.buf, (const uint8_t*)b[1].b.buf,
                                                               (size_t)n, (size_t)m, (const uint8_t*)b[2].b.buf,
                                                               (uint8_t*)b[3].b.buf);
        Py_END_ALLOW_THREADS
      }
      release(b, 4);
      return PyLong_FromLong(rc);
    }
  }
  release(b, 4);
  Py_RETURN_NONE;
}

/* PyInit must be visible despite -fvisibility=hidden */
static PyMethodDef methods[] = {
    {"cbc", cbc, METH_VARARGS, "7-argument backend call through the C ABI (None: use the checked Python path)"},
    {"cbc_std", cbc_std, METH_VARARGS, "gaes_cbc_{en,de}crypt_std through the C ABI (None: Python path)"},
    {"shared_iv", shared_iv, METH_VARARGS, "gaes_{en,de}crypt_shared_iv through the C ABI (None: Python path)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_pyfast", NULL, -1, methods};

PyMODINIT_FUNC PyInit__pyfast(void) { return PyModule_Create(&module); }
