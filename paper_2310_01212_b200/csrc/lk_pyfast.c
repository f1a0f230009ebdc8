/* lk_pyfast.c -- CPython fast path for NativeSession.trigger / wait.
 *
 * The per-task cost of the Python API is the wrapper, not the C ABI: a bare
 * ctypes trigger+wait pair costs ~0.3 us over the C loop, the Python methods
 * around it another ~0.7 us (tools/py_overhead.py).  This module performs the
 * common case of NativeSession.trigger / wait (native.py) in C and calls
 * lk_trigger / lk_wait (include/lk.h) directly:
 *   - a mask already validated and cached as its u64 words,
 *   - a WorkDescriptor object already staged in its slot for this worker set,
 *   - the timing row appended to session.timings (host.TimingLog rows), and
 *     an equal PhaseTiming returned.
 * Anything else goes to the session's Python path (slow_trigger/slow_wait,
 * called with the session from a weak reference), which holds the full rules
 * (validation messages, staging, foreign descriptors).  A failing C call is
 * raised through `raiser(rc, mask, is_wait)`.  native.py binds the two
 * methods as the session's own `trigger`/`wait`, so a task costs no Python
 * frame at all on the common path.  (Without the slow-path arguments a
 * decline returns None and an error its LK_E_* code, for the caller.)
 *
 * The two entry points are passed in as addresses taken from the ctypes
 * handle of liblk.so, so this module and ctypes share one loaded library
 * (one set of session claims and one thread-local last error).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

typedef int (*trigger_fn)(void*, const uint64_t*, uint32_t, uint32_t, const void*, uint64_t*);
typedef int (*wait_fn)(void*, const uint64_t*, uint32_t, uint64_t*);

typedef struct {
  PyObject_HEAD
  void* h;
  uint32_t nwords;
  trigger_fn trig;
  wait_fn wait;
  PyObject* staged;      /* dict slot -> (work, key, multi) */
  PyObject* mask_cache;  /* dict mask -> bytes (8 * nwords) */
  PyObject* rows;        /* list of (phase, ns, mask) */
  PyObject* limit;       /* 1 << num_workers */
  PyTypeObject* timing_type;
  PyTypeObject* work_type;
  PyObject* ph_trigger;
  PyObject* ph_wait;
  int keep_gil;          /* lk_trigger cannot spin (no lazy ack, no event ring): skip the GIL round trip */
  PyObject* slow_trigger;   /* NativeSession._trigger_slow (unbound) or NULL */
  PyObject* slow_wait;      /* NativeSession._wait_slow (unbound) or NULL */
  PyObject* wref;           /* weak reference to the session (no reference cycle) */
  PyObject* raiser;         /* raiser(rc, mask, is_wait) raises the LK_E_* code's exception */
} Fast;

static PyObject* g_zero;
static PyObject* g_empty;
static PyObject *s_slot, *s_phase, *s_cycles, *s_sm_mask;

static void fast_dealloc(Fast* f) {
  Py_XDECREF(f->staged);
  Py_XDECREF(f->mask_cache);
  Py_XDECREF(f->rows);
  Py_XDECREF(f->limit);
  Py_XDECREF(f->timing_type);
  Py_XDECREF(f->work_type);
  Py_XDECREF(f->ph_trigger);
  Py_XDECREF(f->ph_wait);
  Py_XDECREF(f->slow_trigger);
  Py_XDECREF(f->slow_wait);
  Py_XDECREF(f->wref);
  Py_XDECREF(f->raiser);
  Py_TYPE(f)->tp_free((PyObject*)f);
}

static int fast_init(Fast* f, PyObject* args, PyObject* kw) {
  unsigned long long h, trig, wt;
  unsigned int nwords;
  int keep_gil = 0;
  PyObject *staged, *cache, *rows, *limit, *tt, *wtp, *pt, *pw;
  PyObject *st = NULL, *sw = NULL, *wr = NULL, *rs = NULL;
  (void)kw;
  if (!PyArg_ParseTuple(args, "KIKKO!O!O!O!O!O!UU|pOOOO", &h, &nwords, &trig, &wt, &PyDict_Type, &staged,
                        &PyDict_Type, &cache, &PyList_Type, &rows, &PyLong_Type, &limit, &PyType_Type, &tt,
                        &PyType_Type, &wtp, &pt, &pw, &keep_gil, &st, &sw, &wr, &rs))
    return -1;
  f->keep_gil = keep_gil;
  if (st && sw && wr && rs) {
    if (!PyWeakref_CheckRef(wr)) {
      PyErr_SetString(PyExc_TypeError, "session must come as a weak reference");
      return -1;
    }
    Py_INCREF(st); Py_XSETREF(f->slow_trigger, st);
    Py_INCREF(sw); Py_XSETREF(f->slow_wait, sw);
    Py_INCREF(wr); Py_XSETREF(f->wref, wr);
    Py_INCREF(rs); Py_XSETREF(f->raiser, rs);
  }
  if (!h || !trig || !wt || nwords == 0) {
    PyErr_SetString(PyExc_ValueError, "null handle or entry point");
    return -1;
  }
  f->h = (void*)(uintptr_t)h;
  f->nwords = nwords;
  f->trig = (trigger_fn)(uintptr_t)trig;
  f->wait = (wait_fn)(uintptr_t)wt;
  Py_INCREF(staged); Py_XSETREF(f->staged, staged);
  Py_INCREF(cache); Py_XSETREF(f->mask_cache, cache);
  Py_INCREF(rows); Py_XSETREF(f->rows, rows);
  Py_INCREF(limit); Py_XSETREF(f->limit, limit);
  Py_INCREF(tt); Py_XSETREF(f->timing_type, (PyTypeObject*)tt);
  Py_INCREF(wtp); Py_XSETREF(f->work_type, (PyTypeObject*)wtp);
  Py_INCREF(pt); Py_XSETREF(f->ph_trigger, pt);
  Py_INCREF(pw); Py_XSETREF(f->ph_wait, pw);
  return 0;
}

/* The cached u64 words (a new reference to the bytes: another thread may
 * clear the cache while the GIL is released) of a valid mask
 * (0 < mask < 1 << num_workers), or NULL (no exception set) when the Python
 * path must handle it. */
static PyObject* mask_words(Fast* f, PyObject* mask) {
  if (!PyLong_CheckExact(mask)) return NULL;
  PyObject* b = PyDict_GetItemWithError(f->mask_cache, mask);   /* borrowed */
  if (!b) {
    PyErr_Clear();
    return NULL;
  }
  if (!PyBytes_CheckExact(b) || PyBytes_GET_SIZE(b) != (Py_ssize_t)(8 * f->nwords)) return NULL;
  Py_INCREF(b);   /* the comparisons below could run Python code */
  int gt = PyObject_RichCompareBool(mask, g_zero, Py_GT);
  int lt = gt == 1 ? PyObject_RichCompareBool(mask, f->limit, Py_LT) : 0;
  if (gt != 1 || lt != 1) {
    PyErr_Clear();
    Py_DECREF(b);
    return NULL;
  }
  return b;
}

/* Append (phase, ns, mask) to the timing rows and return an equal PhaseTiming
 * built like object.__new__ + __dict__ fill (host._materialize). */
static PyObject* record(Fast* f, PyObject* phase, uint64_t ns, PyObject* mask) {
  PyObject* cyc = PyLong_FromUnsignedLongLong(ns);
  if (!cyc) return NULL;
  PyObject* row = PyTuple_Pack(3, phase, cyc, mask);
  if (!row) {
    Py_DECREF(cyc);
    return NULL;
  }
  int rc = PyList_Append(f->rows, row);
  Py_DECREF(row);
  if (rc) {
    Py_DECREF(cyc);
    return NULL;
  }
  PyObject* t = PyBaseObject_Type.tp_new(f->timing_type, g_empty, NULL);
  if (!t) {
    Py_DECREF(cyc);
    return NULL;
  }
  PyObject* d = PyObject_GenericGetDict(t, NULL);
  if (!d || PyDict_SetItem(d, s_phase, phase) || PyDict_SetItem(d, s_cycles, cyc) ||
      PyDict_SetItem(d, s_sm_mask, mask)) {
    Py_XDECREF(d);
    Py_DECREF(cyc);
    Py_DECREF(t);
    return NULL;
  }
  Py_DECREF(d);
  Py_DECREF(cyc);
  return t;
}

/* The Python path for what the C path declines (None without one). */
static PyObject* decline(Fast* f, PyObject* slow, PyObject* const* args, Py_ssize_t nargs) {
  if (!slow) Py_RETURN_NONE;
  PyObject* sess = PyWeakref_GetObject(f->wref);   /* borrowed */
  if (!sess) return NULL;
  if (sess == Py_None) {
    PyErr_SetString(PyExc_ReferenceError, "session is gone");
    return NULL;
  }
  PyObject* callargs[3] = {sess, args[0], nargs > 1 ? args[1] : NULL};
  Py_INCREF(sess);
  PyObject* r = PyObject_Vectorcall(slow, callargs, (size_t)(nargs + 1), NULL);
  Py_DECREF(sess);
  return r;
}

/* A method object captured before the session closed: the handle is gone,
 * so never call into liblk.so.  The session's Python path raises its
 * "already disposed" UsageError; without one this is a RuntimeError. */
static PyObject* closed(Fast* f, PyObject* slow, PyObject* const* args, Py_ssize_t nargs) {
  if (slow && f->wref) {
    PyObject* sess = PyWeakref_GetObject(f->wref);   /* borrowed */
    if (sess && sess != Py_None) return decline(f, slow, args, nargs);
    PyErr_Clear();
  }
  PyErr_SetString(PyExc_RuntimeError, "LK session closed");
  return NULL;
}

static PyObject* fast_close(Fast* f, PyObject* unused) {
  (void)unused;
  f->h = NULL;
  Py_RETURN_NONE;
}

/* A failing C call: raised through the session's raiser (its LK_E_* code as an
 * int without one). */
static PyObject* failed(Fast* f, int rc, PyObject* mask, int is_wait) {
  if (!f->raiser) return PyLong_FromLong(rc);
  PyObject* r = PyObject_CallFunction(f->raiser, "iOi", rc, mask, is_wait);
  if (r) {   /* the raiser must raise */
    Py_DECREF(r);
    PyErr_Format(PyExc_RuntimeError, "LK error %d", rc);
  }
  return NULL;
}

static PyObject* fast_trigger(Fast* f, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 2) {
    PyErr_SetString(PyExc_TypeError, "trigger(mask, work)");
    return NULL;
  }
  PyObject *mask = args[0], *work = args[1];
  if (!f->h) return closed(f, f->slow_trigger, args, nargs);
  if (Py_TYPE(work) != f->work_type) return decline(f, f->slow_trigger, args, nargs);
  PyObject* mb = mask_words(f, mask);
  if (!mb) return decline(f, f->slow_trigger, args, nargs);
  PyObject* slot = PyObject_GetAttr(work, s_slot);
  if (!slot) {
    Py_DECREF(mb);
    return NULL;
  }
  PyObject* st = PyDict_GetItemWithError(f->staged, slot);   /* borrowed */
  unsigned long sl = PyLong_Check(slot) ? PyLong_AsUnsignedLong(slot) : (unsigned long)-1;
  Py_DECREF(slot);
  if (PyErr_Occurred()) {
    PyErr_Clear();
    Py_DECREF(mb);
    return decline(f, f->slow_trigger, args, nargs);
  }
  if (!st || !PyTuple_CheckExact(st) || PyTuple_GET_SIZE(st) != 3 || PyTuple_GET_ITEM(st, 0) != work ||
      sl > 0xFFFFFFFFul) {
    Py_DECREF(mb);
    return decline(f, f->slow_trigger, args, nargs);
  }
  /* staged for this worker set: key is the mask for payload kinds, else 0
   * (the entry is held across the comparisons, which could run Python code) */
  Py_INCREF(st);
  PyObject* key = PyObject_IsTrue(PyTuple_GET_ITEM(st, 2)) == 1 ? mask : g_zero;
  int same = PyObject_RichCompareBool(PyTuple_GET_ITEM(st, 1), key, Py_EQ);
  Py_DECREF(st);
  if (same != 1) {
    PyErr_Clear();
    Py_DECREF(mb);
    return decline(f, f->slow_trigger, args, nargs);
  }
  const uint64_t* m = (const uint64_t*)PyBytes_AS_STRING(mb);
  uint64_t ns = 0;
  int rc;
  if (f->keep_gil) {   /* a few stores and checks under the session mutex: ~100 ns */
    rc = f->trig(f->h, m, f->nwords, (uint32_t)sl, NULL, &ns);
  } else {
    Py_BEGIN_ALLOW_THREADS
    rc = f->trig(f->h, m, f->nwords, (uint32_t)sl, NULL, &ns);
    Py_END_ALLOW_THREADS
  }
  Py_DECREF(mb);
  if (rc) return failed(f, rc, mask, 0);
  return record(f, f->ph_trigger, ns, mask);
}

static PyObject* fast_wait(Fast* f, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 1) {
    PyErr_SetString(PyExc_TypeError, "wait(mask)");
    return NULL;
  }
  PyObject* mask = args[0];
  if (!f->h) return closed(f, f->slow_wait, args, nargs);
  PyObject* mb = mask_words(f, mask);
  if (!mb) return decline(f, f->slow_wait, args, nargs);
  const uint64_t* m = (const uint64_t*)PyBytes_AS_STRING(mb);
  uint64_t ns = 0;
  int rc;
  Py_BEGIN_ALLOW_THREADS
  rc = f->wait(f->h, m, f->nwords, &ns);
  Py_END_ALLOW_THREADS
  Py_DECREF(mb);
  if (rc) return failed(f, rc, mask, 1);
  return record(f, f->ph_wait, ns, mask);
}

static PyMethodDef fast_methods[] = {
    {"trigger", (PyCFunction)(void (*)(void))fast_trigger, METH_FASTCALL, "trigger(mask, work)"},
    {"wait", (PyCFunction)(void (*)(void))fast_wait, METH_FASTCALL, "wait(mask)"},
    {"close", (PyCFunction)fast_close, METH_NOARGS, "forget the session handle (later calls never reach liblk.so)"},
    {NULL, NULL, 0, NULL}};

static PyTypeObject FastType = {
    PyVarObject_HEAD_INIT(NULL, 0).tp_name = "paper_2310_01212_b200._lkfast.Fast",
    .tp_basicsize = sizeof(Fast),
    .tp_flags = Py_TPFLAGS_DEFAULT,
    .tp_new = PyType_GenericNew,
    .tp_init = (initproc)fast_init,
    .tp_dealloc = (destructor)fast_dealloc,
    .tp_methods = fast_methods,
    .tp_doc = "Fast(handle, nwords, lk_trigger, lk_wait, staged, mask_cache, rows, limit, PhaseTiming, "
              "WorkDescriptor, phase_trigger, phase_wait)",
};

static struct PyModuleDef moddef = {PyModuleDef_HEAD_INIT, "_lkfast", "CPython fast path for trigger/wait", -1,
                                    NULL, NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__lkfast(void) {
  if (PyType_Ready(&FastType) < 0) return NULL;
  g_zero = PyLong_FromLong(0);
  g_empty = PyTuple_New(0);
  s_slot = PyUnicode_InternFromString("slot");
  s_phase = PyUnicode_InternFromString("phase");
  s_cycles = PyUnicode_InternFromString("cycles");
  s_sm_mask = PyUnicode_InternFromString("sm_mask");
  if (!g_zero || !g_empty || !s_slot || !s_phase || !s_cycles || !s_sm_mask) return NULL;
  PyObject* m = PyModule_Create(&moddef);
  if (!m) return NULL;
  Py_INCREF(&FastType);
  if (PyModule_AddObject(m, "Fast", (PyObject*)&FastType) < 0) {
    Py_DECREF(&FastType);
    Py_DECREF(m);
    return NULL;
  }
  return m;
}
