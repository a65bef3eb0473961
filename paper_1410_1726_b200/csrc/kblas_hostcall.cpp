// CPython fast path for the numpy-vector call (kernels.gemv / symv_hemv /
// the offset API with numpy x and y, and their CommandQueue submissions).
//
// It is a thin binding of the C ABI entry kblas_mv_hostvec[_async]
// (include/kblas_b200.h) for the reference's numpy-in / numpy-out call
// shape (blockmv kernels.py:402-440, 443-486; offset.py:83-208): the
// vectors are taken through the buffer protocol and the scalars as Python
// numbers, with no ctypes marshalling (~6 us per call, scripts/
// queue_overhead.py).  Anything off the fast path -- x or y not a 1-D
// contiguous buffer of the operand dtype and length, a complex scalar for
// a real precision -- returns SLOW_PATH and the Python layer converts and
// validates exactly as before (same exceptions, same messages), then calls
// again.  The GIL is released around the library call.
//
// Links against libkblas_b200.so from the same directory (rpath $ORIGIN),
// so it shares the library instance ctypes loaded (caches, plans, counters).
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <cstdint>
#include <cstring>
#include <initializer_list>

#include "../../include/kblas_b200.h"

namespace {

constexpr long SLOW_PATH = -100;

struct Buf {
  Py_buffer view{};
  bool held = false;
  ~Buf() {
    if (held) PyBuffer_Release(&view);
  }
};

// struct-module format of the precision's element
bool format_ok(char prec, const char *fmt) {
  if (fmt == nullptr) return false;
  if (*fmt == '<' || *fmt == '=' || *fmt == '@') ++fmt;
  switch (prec) {
    case 's': return std::strcmp(fmt, "f") == 0;
    case 'd': return std::strcmp(fmt, "d") == 0;
    case 'c': return std::strcmp(fmt, "Zf") == 0;
    case 'z': return std::strcmp(fmt, "Zd") == 0;
  }
  return false;
}

Py_ssize_t esize(char prec) { return prec == 's' ? 4 : (prec == 'z' ? 16 : 8); }

// 1-D C-contiguous buffer of `len` elements of the precision (fmt_check) or
// of any 1-D shape of `len` elements (!fmt_check: y that is never read)
bool get_vec(PyObject *o, char prec, Py_ssize_t len, bool fmt_check, Buf *b) {
  if (!PyObject_CheckBuffer(o)) return false;
  if (PyObject_GetBuffer(o, &b->view, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT) != 0) {
    PyErr_Clear();
    return false;
  }
  b->held = true;
  if (b->view.ndim != 1 || b->view.shape == nullptr || b->view.shape[0] != len) return false;
  if (!fmt_check) return true;
  return b->view.itemsize == esize(prec) && format_ok(prec, b->view.format);
}

// scalar of the precision into out (16 bytes); false: off the fast path
bool get_scalar(PyObject *o, char prec, unsigned char *out) {
  double re, im = 0.0;
  if (PyFloat_CheckExact(o)) {
    re = PyFloat_AS_DOUBLE(o);
  } else if (PyLong_CheckExact(o)) {
    re = PyLong_AsDouble(o);
    if (re == -1.0 && PyErr_Occurred()) {
      PyErr_Clear();
      return false;
    }
  } else {
    Py_complex c = PyComplex_AsCComplex(o);
    if (c.real == -1.0 && PyErr_Occurred()) {
      PyErr_Clear();
      return false;
    }
    re = c.real;
    im = c.imag;
  }
  switch (prec) {
    case 's': {
      if (im != 0.0) return false;
      const float f = (float)re;
      std::memcpy(out, &f, 4);
      return true;
    }
    case 'd':
      if (im != 0.0) return false;
      std::memcpy(out, &re, 8);
      return true;
    case 'c': {
      const float f[2] = {(float)re, (float)im};
      std::memcpy(out, f, 8);
      return true;
    }
    case 'z': {
      const double d[2] = {re, im};
      std::memcpy(out, d, 16);
      return true;
    }
  }
  return false;
}

// mv_hostvec(prec, kind, op, hermitian, m, n, alpha, a_ptr, lda, offset_r,
//            offset_c, x, x_len, beta, y, y_len, out_ptr, stream, sync)
//   -> 0, a kblas return code, or SLOW_PATH
PyObject *mv_hostvec(PyObject *, PyObject *const *args, Py_ssize_t nargs) {
  if (nargs != 19) {
    PyErr_SetString(PyExc_TypeError, "mv_hostvec takes 19 arguments");
    return nullptr;
  }
  auto ch = [](PyObject *o, char *c) -> bool {
    if (!PyUnicode_Check(o) || PyUnicode_GET_LENGTH(o) != 1) return false;
    *c = (char)PyUnicode_READ_CHAR(o, 0);
    return true;
  };
  char prec, kind, op;
  if (!ch(args[0], &prec) || !ch(args[1], &kind) || !ch(args[2], &op)) {
    PyErr_SetString(PyExc_TypeError, "mv_hostvec: prec, kind and op are one-character strings");
    return nullptr;
  }
  prec = (char)(prec | 0x20);
  const long herm = PyLong_AsLong(args[3]);
  const long m = PyLong_AsLong(args[4]);
  const long n = PyLong_AsLong(args[5]);
  const uintptr_t a_ptr = (uintptr_t)PyLong_AsUnsignedLongLong(args[7]);
  const long lda = PyLong_AsLong(args[8]);
  const long off_r = PyLong_AsLong(args[9]);
  const long off_c = PyLong_AsLong(args[10]);
  const Py_ssize_t x_len = PyLong_AsSsize_t(args[12]);
  const Py_ssize_t y_len = PyLong_AsSsize_t(args[15]);
  const uintptr_t out_ptr = (uintptr_t)PyLong_AsUnsignedLongLong(args[16]);
  const uintptr_t stream = (uintptr_t)PyLong_AsUnsignedLongLong(args[17]);
  const int sync = PyObject_IsTrue(args[18]);
  if (PyErr_Occurred()) return nullptr;
  for (long v : {m, n, lda, off_r, off_c})
    if (v > 2147483647L) {
      PyErr_SetString(PyExc_ValueError, "mv_hostvec: a dimension exceeds the C ABI's 32-bit int range");
      return nullptr;
    }
  if (prec != 's' && prec != 'd' && prec != 'c' && prec != 'z') return PyLong_FromLong(SLOW_PATH);
  alignas(16) unsigned char alpha[16], beta[16];
  if (!get_scalar(args[6], prec, alpha) || !get_scalar(args[13], prec, beta)) return PyLong_FromLong(SLOW_PATH);
  bool beta_zero;
  {
    Py_complex b = PyComplex_AsCComplex(args[13]);
    if (PyErr_Occurred()) {
      PyErr_Clear();
      return PyLong_FromLong(SLOW_PATH);
    }
    beta_zero = b.real == 0.0 && b.imag == 0.0;
  }
  Buf xb, yb;
  if (!get_vec(args[11], prec, x_len, true, &xb)) return PyLong_FromLong(SLOW_PATH);
  // beta == 0: y is never read, only its length is checked
  if (!get_vec(args[14], prec, y_len, !beta_zero, &yb)) return PyLong_FromLong(SLOW_PATH);
  const void *hx = xb.view.buf;
  const void *hy = beta_zero ? nullptr : yb.view.buf;
  int rc;
  Py_BEGIN_ALLOW_THREADS
  rc = sync ? kblas_mv_hostvec(prec, kind, op, (int)herm, (int)m, (int)n, alpha, (const void *)a_ptr, (int)lda,
                               (int)off_r, (int)off_c, hx, beta, hy, (void *)out_ptr, (cudaStream_t)stream)
            : kblas_mv_hostvec_async(prec, kind, op, (int)herm, (int)m, (int)n, alpha, (const void *)a_ptr,
                                     (int)lda, (int)off_r, (int)off_c, hx, beta, hy, (void *)out_ptr,
                                     (cudaStream_t)stream);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(rc);
}

PyObject *last_plan(PyObject *, PyObject *) { return PyUnicode_FromString(kblas_last_plan()); }

PyMethodDef methods[] = {
    {"mv_hostvec", (PyCFunction)(void (*)(void))mv_hostvec, METH_FASTCALL,
     "numpy-vector call through kblas_mv_hostvec[_async]; returns 0, a kblas code or -100 (slow path)"},
    {"last_plan", last_plan, METH_NOARGS, "kblas_last_plan() of this thread"},
    {nullptr, nullptr, 0, nullptr},
};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_hostcall", "numpy-vector fast path of the KBLAS B200 API", -1,
                      methods};

}  // namespace

PyMODINIT_FUNC PyInit__hostcall(void) {
  PyObject *m = PyModule_Create(&module);
  if (m != nullptr) PyModule_AddIntConstant(m, "SLOW_PATH", SLOW_PATH);
  return m;
}
