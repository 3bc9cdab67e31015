/* _dgcore: native host-side graph construction for the drop-in API.
 *
 * The reference builds its graph in Python (graph.py:97-106: staleness check,
 * OpDef.shape rule, Node append, Expression handle).  Per training step the
 * PTB RNNLM builds ~1200 nodes, so construction and packing the node table for
 * the executor dominated the host side of a step.  This module implements
 *   - the Shape / Node / Expression storage as C base types (the Python
 *     classes in tensor.py / graph.py subclass them and keep every method),
 *   - GraphCore.add(kind, inputs, aux): the add_node fast path -- staleness
 *     checks, the shape rules of the built-in op kinds (happy path; anything
 *     irregular defers to the Python rule so errors are raised by the same
 *     code with the same messages), and the dg_node record encoding
 *     (include/dyngpu.h) into C buffers handed to dg_graph_append without a
 *     Python-level packing pass.
 * Kinds without a native rule (or re-registered by the user) go through the
 * Python OpDef.shape / OpDef.encode hooks and still land in the C records.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <structmember.h>
#include <stdint.h>
#include <string.h>

/* op codes (dyngpu.h dg_op) */
enum {
  OP_INPUT = 0, OP_PARAMETER = 1, OP_LOOKUP = 2, OP_LOOKUP_BATCH = 3, OP_ADD = 4, OP_CMULT = 5,
  OP_SCALAR_MUL = 6, OP_TANH = 7, OP_LOGISTIC = 8, OP_MATMUL = 9, OP_AFFINE = 10, OP_CONCATENATE = 11,
  OP_PICK_RANGE = 12, OP_SOFTMAX = 13, OP_PNLS = 14, OP_PNLS_BATCH = 15, OP_SUM_BATCHES = 16
};
#define HDR 13

/* ------------------------------------------------------------ base types */
typedef struct {
  PyObject_HEAD
  PyObject* dims; /* tuple of int */
  long batch;
  PyObject* enc;  /* unused slot kept for subclasses */
} ShapeObj;

typedef struct {
  PyObject_HEAD
  PyObject* kind;
  PyObject* inputs;
  PyObject* shape;
  PyObject* aux;
  long code;
} NodeObj;

typedef struct {
  PyObject_HEAD
  PyObject* graph;
  Py_ssize_t index;
  long generation;
} ExprObj;

static void shape_dealloc(ShapeObj* s) {
  Py_XDECREF(s->dims);
  Py_XDECREF(s->enc);
  Py_TYPE(s)->tp_free((PyObject*)s);
}
static void node_dealloc(NodeObj* n) {
  Py_XDECREF(n->kind);
  Py_XDECREF(n->inputs);
  Py_XDECREF(n->shape);
  Py_XDECREF(n->aux);
  Py_TYPE(n)->tp_free((PyObject*)n);
}
static void expr_dealloc(ExprObj* e) {
  Py_XDECREF(e->graph);
  Py_TYPE(e)->tp_free((PyObject*)e);
}

static PyMemberDef shape_members[] = {
    {"dims", T_OBJECT_EX, offsetof(ShapeObj, dims), 0, "dims tuple"},
    {"batch", T_LONG, offsetof(ShapeObj, batch), 0, "batch count"},
    {"_enc", T_OBJECT, offsetof(ShapeObj, enc), 0, "cache slot"},
    {NULL}};
static PyMemberDef node_members[] = {
    {"kind", T_OBJECT_EX, offsetof(NodeObj, kind), 0, NULL},
    {"inputs", T_OBJECT_EX, offsetof(NodeObj, inputs), 0, NULL},
    {"shape", T_OBJECT_EX, offsetof(NodeObj, shape), 0, NULL},
    {"aux", T_OBJECT, offsetof(NodeObj, aux), 0, NULL},
    {"code", T_LONG, offsetof(NodeObj, code), 0, NULL},
    {NULL}};
static PyMemberDef expr_members[] = {
    {"graph", T_OBJECT_EX, offsetof(ExprObj, graph), 0, NULL},
    {"index", T_PYSSIZET, offsetof(ExprObj, index), 0, NULL},
    {"generation", T_LONG, offsetof(ExprObj, generation), 0, NULL},
    {NULL}};

static PyTypeObject ShapeBaseType = {PyVarObject_HEAD_INIT(NULL, 0).tp_name = "_dgcore.ShapeBase",
                                     .tp_basicsize = sizeof(ShapeObj),
                                     .tp_dealloc = (destructor)shape_dealloc,
                                     .tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_BASETYPE,
                                     .tp_members = shape_members,
                                     .tp_new = PyType_GenericNew};
static PyTypeObject NodeBaseType = {PyVarObject_HEAD_INIT(NULL, 0).tp_name = "_dgcore.NodeBase",
                                    .tp_basicsize = sizeof(NodeObj),
                                    .tp_dealloc = (destructor)node_dealloc,
                                    .tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_BASETYPE,
                                    .tp_members = node_members,
                                    .tp_new = PyType_GenericNew};
static PyTypeObject ExprBaseType = {PyVarObject_HEAD_INIT(NULL, 0).tp_name = "_dgcore.ExprBase",
                                    .tp_basicsize = sizeof(ExprObj),
                                    .tp_dealloc = (destructor)expr_dealloc,
                                    .tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_BASETYPE,
                                    .tp_members = expr_members,
                                    .tp_new = PyType_GenericNew};

/* Python subclasses registered by setup(): instances are allocated directly */
static PyTypeObject* ShapeT = NULL;
static PyTypeObject* NodeT = NULL;
static PyTypeObject* ExprT = NULL;
static PyObject* Registry = NULL;  /* ops.REGISTRY */
static PyObject* FastKinds = NULL; /* kind str -> code for kinds with the built-in rule */
/* The heap subclasses are GC types, but the cycle collector cannot see the
   C fields (no tp_traverse on the bases), so tracking them buys nothing and
   makes every young-generation collection walk thousands of graph objects. */
static inline void untrack(PyObject* o) {
  if (o && PyObject_GC_IsTracked(o)) PyObject_GC_UnTrack(o);
}

/* tuples of ints/floats (index tuples, dims, pick ranges) cannot be in a cycle */
static void untrack_atomic_tuple(PyObject* t) {
  if (!t || !PyTuple_CheckExact(t) || !PyObject_GC_IsTracked(t)) return;
  for (Py_ssize_t k = 0, n = PyTuple_GET_SIZE(t); k < n; ++k) {
    PyObject* v = PyTuple_GET_ITEM(t, k);
    if (!PyLong_CheckExact(v) && !PyFloat_CheckExact(v)) return;
  }
  PyObject_GC_UnTrack(t);
}

static PyObject* s_shape = NULL, *s_encode = NULL, *s_handle = NULL, *s_rows = NULL, *s_dim = NULL,
                *s_data = NULL, *s_check_current = NULL, *s_code = NULL;

static PyObject* new_shape(PyObject* dims, long batch) {
  ShapeObj* s = (ShapeObj*)ShapeT->tp_alloc(ShapeT, 0);
  untrack((PyObject*)s);
  untrack_atomic_tuple(dims);
  if (!s) return NULL;
  Py_INCREF(dims);
  s->dims = dims;
  s->batch = batch;
  s->enc = NULL;
  return (PyObject*)s;
}

/* --------------------------------------------------------------- records */
typedef struct {
  char* p;
  Py_ssize_t n, cap, esz;
} Buf;

static int buf_reserve(Buf* b, Py_ssize_t extra) {
  if (b->n + extra <= b->cap) return 0;
  Py_ssize_t cap = b->cap ? b->cap : 1024;
  while (cap < b->n + extra) cap *= 2;
  char* p = (char*)PyMem_Realloc(b->p, (size_t)(cap * b->esz));
  if (!p) {
    PyErr_NoMemory();
    return -1;
  }
  b->p = p;
  b->cap = cap;
  return 0;
}

typedef struct {
  PyObject_HEAD
  PyObject* cg;    /* borrowed: the core is owned by its graph */
  PyObject* nodes; /* the graph's node list */
  long gen;
  Buf hdr, ins, ai, af, rebased;
  PyObject* fix; /* list of (ai position, parameter-like with .handle) */
} CoreObj;

static void core_dealloc(CoreObj* c) {
  Py_XDECREF(c->nodes);
  Py_XDECREF(c->fix);
  PyMem_Free(c->hdr.p);
  PyMem_Free(c->ins.p);
  PyMem_Free(c->ai.p);
  PyMem_Free(c->af.p);
  PyMem_Free(c->rebased.p);
  Py_TYPE(c)->tp_free((PyObject*)c);
}

static int core_init(CoreObj* c, PyObject* args, PyObject* kw) {
  PyObject *cg, *nodes;
  if (!PyArg_ParseTuple(args, "OO!", &cg, &PyList_Type, &nodes)) return -1;
  c->cg = cg;
  Py_XSETREF(c->nodes, Py_NewRef(nodes));
  c->gen = 0;
  c->hdr.esz = 4;
  c->ins.esz = 4;
  c->ai.esz = 8;
  c->af.esz = 4;
  c->rebased.esz = 4;
  Py_XSETREF(c->fix, PyList_New(0));
  return c->fix ? 0 : -1;
}

static PyObject* core_renew(CoreObj* c, PyObject* arg) {
  c->gen = PyLong_AsLong(arg);
  if (c->gen == -1 && PyErr_Occurred()) return NULL;
  c->hdr.n = c->ins.n = c->ai.n = c->af.n = 0;
  if (PyList_SetSlice(c->fix, 0, PyList_GET_SIZE(c->fix), NULL) < 0) return NULL;
  Py_RETURN_NONE;
}

/* append a node record; ai (n_ai int64) and af (n_af float) payloads */
static int put_record(CoreObj* c, long code, const int32_t* idx, int n_in, ShapeObj* sh, const int64_t* ai,
                      Py_ssize_t n_ai, const float* af, Py_ssize_t n_af) {
  if (buf_reserve(&c->hdr, HDR) || buf_reserve(&c->ins, n_in) || buf_reserve(&c->ai, n_ai) ||
      buf_reserve(&c->af, n_af))
    return -1;
  int32_t* h = (int32_t*)c->hdr.p + c->hdr.n;
  const Py_ssize_t r = PyTuple_GET_SIZE(sh->dims);
  h[0] = (int32_t)code;
  h[1] = n_in;
  h[2] = (int32_t)c->ins.n;
  h[3] = (int32_t)r;
  for (int d = 0; d < 4; ++d) h[4 + d] = d < r ? (int32_t)PyLong_AsLong(PyTuple_GET_ITEM(sh->dims, d)) : 1;
  h[8] = (int32_t)sh->batch;
  h[9] = (int32_t)c->ai.n;
  h[10] = (int32_t)n_ai;
  h[11] = (int32_t)c->af.n;
  h[12] = (int32_t)n_af;
  c->hdr.n += HDR;
  memcpy((int32_t*)c->ins.p + c->ins.n, idx, sizeof(int32_t) * (size_t)n_in);
  c->ins.n += n_in;
  if (n_ai) memcpy((int64_t*)c->ai.p + c->ai.n, ai, sizeof(int64_t) * (size_t)n_ai);
  c->ai.n += n_ai;
  if (n_af) memcpy((float*)c->af.p + c->af.n, af, sizeof(float) * (size_t)n_af);
  c->af.n += n_af;
  return 0;
}

static int add_fix(CoreObj* c, Py_ssize_t pos, PyObject* param) {
  PyObject* t = Py_BuildValue("(nO)", pos, param);
  if (!t) return -1;
  int rc = PyList_Append(c->fix, t);
  Py_DECREF(t);
  return rc;
}

/* Python fallback: od.shape(aux, in_shapes) and od.encode(aux) */
static PyObject* slow_shape(PyObject* od, PyObject* aux, PyObject* in_shapes) {
  PyObject* rule = PyObject_GetAttr(od, s_shape);
  if (!rule) return NULL;
  PyObject* r = PyObject_CallFunctionObjArgs(rule, aux, in_shapes, NULL);
  Py_DECREF(rule);
  return r;
}

static int slow_encode(CoreObj* c, PyObject* od, long code, PyObject* aux, const int32_t* idx, int n_in,
                       ShapeObj* sh) {
  PyObject* enc = PyObject_GetAttr(od, s_encode);
  if (!enc) return -1;
  PyObject* r = PyObject_CallOneArg(enc, aux);
  Py_DECREF(enc);
  if (!r) return -1;
  int rc = -1;
  PyObject *ai = NULL, *af = NULL, *aiseq = NULL;
  int64_t* aiv = NULL;
  Py_buffer view = {0};
  int have_view = 0;
  if (!PyTuple_Check(r) || PyTuple_GET_SIZE(r) != 2) {
    PyErr_SetString(PyExc_TypeError, "encode must return (aux_i, aux_f)");
    goto done;
  }
  ai = PyTuple_GET_ITEM(r, 0);
  af = PyTuple_GET_ITEM(r, 1);
  aiseq = PySequence_Fast(ai, "aux_i must be a sequence");
  if (!aiseq) goto done;
  Py_ssize_t n_ai = PySequence_Fast_GET_SIZE(aiseq);
  aiv = (int64_t*)PyMem_Malloc(sizeof(int64_t) * (size_t)(n_ai ? n_ai : 1));
  if (!aiv) {
    PyErr_NoMemory();
    goto done;
  }
  for (Py_ssize_t q = 0; q < n_ai; ++q) {
    aiv[q] = PyLong_AsLongLong(PySequence_Fast_GET_ITEM(aiseq, q));
    if (aiv[q] == -1 && PyErr_Occurred()) goto done;
  }
  const float* afp = NULL;
  Py_ssize_t n_af = 0;
  if (af != Py_None) {
    if (PyObject_GetBuffer(af, &view, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT) < 0) goto done;
    have_view = 1;
    if (view.itemsize != 4 || !view.format || strcmp(view.format, "f") != 0) {
      PyErr_SetString(PyExc_TypeError, "aux_f must be a contiguous float32 array");
      goto done;
    }
    afp = (const float*)view.buf;
    n_af = view.len / 4;
  }
  if ((code == OP_PARAMETER || code == OP_LOOKUP || code == OP_LOOKUP_BATCH) && n_ai > 0) {
    /* the handle slot is resolved at flush (parameters materialise lazily) */
    PyObject* owner = code == OP_PARAMETER ? aux : PyTuple_GetItem(aux, 0);
    if (!owner || add_fix(c, c->ai.n, owner) < 0) goto done;
  }
  rc = put_record(c, code, idx, n_in, sh, aiv, n_ai, afp, n_af);
done:
  if (have_view) PyBuffer_Release(&view);
  PyMem_Free(aiv);
  Py_XDECREF(aiseq);
  Py_DECREF(r);
  return rc;
}

static long get_long_attr(PyObject* o, PyObject* name, int* err) {
  PyObject* v = PyObject_GetAttr(o, name);
  if (!v) {
    *err = 1;
    return 0;
  }
  long x = PyLong_AsLong(v);
  Py_DECREF(v);
  if (x == -1 && PyErr_Occurred()) *err = 1;
  return x;
}

#define MAX_IN 64

/* GraphCore.add(kind, inputs, aux) -> Expression */
static PyObject* core_add(CoreObj* c, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs < 1 || nargs > 3) {
    PyErr_SetString(PyExc_TypeError, "add(kind, inputs=(), aux=None)");
    return NULL;
  }
  PyObject* kind = args[0];
  PyObject* inputs = nargs > 1 ? args[1] : NULL;
  PyObject* aux = nargs > 2 ? args[2] : Py_None;
  PyObject* seq = NULL;
  Py_ssize_t n_in = 0;
  if (inputs) {
    seq = PySequence_Fast(inputs, "inputs must be a sequence of expressions");
    if (!seq) return NULL;
    n_in = PySequence_Fast_GET_SIZE(seq);
  }
  int32_t idx_stack[MAX_IN];
  int32_t* idx = idx_stack;
  ShapeObj* shp_stack[MAX_IN];
  ShapeObj** shp = shp_stack;
  if (n_in > MAX_IN) {
    idx = (int32_t*)PyMem_Malloc(sizeof(int32_t) * (size_t)n_in);
    shp = (ShapeObj**)PyMem_Malloc(sizeof(ShapeObj*) * (size_t)n_in);
    if (!idx || !shp) {
      PyErr_NoMemory();
      goto fail0;
    }
  }
  const Py_ssize_t n_nodes = PyList_GET_SIZE(c->nodes);
  for (Py_ssize_t k = 0; k < n_in; ++k) {
    PyObject* e = PySequence_Fast_GET_ITEM(seq, k);
    if (!PyObject_TypeCheck(e, &ExprBaseType) || ((ExprObj*)e)->graph != c->cg || ((ExprObj*)e)->generation != c->gen ||
        ((ExprObj*)e)->index < 0 || ((ExprObj*)e)->index >= n_nodes) {
      /* the Python check raises StaleExpression with the reference message */
      PyObject* r = PyObject_CallMethodOneArg(c->cg, s_check_current, e);
      if (!r) goto fail0;
      Py_DECREF(r);
      PyErr_SetString(PyExc_TypeError, "graph inputs must be expressions of this graph");
      goto fail0;
    }
    const Py_ssize_t i = ((ExprObj*)e)->index;
    idx[k] = (int32_t)i;
    shp[k] = (ShapeObj*)((NodeObj*)PyList_GET_ITEM(c->nodes, i))->shape;
  }
  PyObject* codeobj = PyDict_GetItemWithError(FastKinds, kind);
  if (!codeobj && PyErr_Occurred()) goto fail0;
  long code = codeobj ? PyLong_AsLong(codeobj) : -1;
  PyObject* shape = NULL; /* new reference */
  /* ---- fast paths of the built-in rules (ops.py); irregular inputs defer to
     the Python rule, which raises the reference error */
  int64_t ai_small[4];
  Py_ssize_t n_ai = 0;
  float af_small[1];
  Py_ssize_t n_af = 0;
  PyObject* fixobj = NULL; /* borrowed */
  int done = 0;
  switch (code) {
    case OP_TANH:
    case OP_LOGISTIC:
      if (n_in == 1) {
        shape = Py_NewRef((PyObject*)shp[0]);
        done = 1;
      }
      break;
    case OP_SCALAR_MUL:
      if (n_in == 1 && PyFloat_CheckExact(aux)) {
        shape = Py_NewRef((PyObject*)shp[0]);
        af_small[0] = (float)PyFloat_AS_DOUBLE(aux);
        n_af = 1;
        done = 1;
      }
      break;
    case OP_ADD:
    case OP_CMULT:
      if (n_in == 2) {
        PyObject* da = shp[0]->dims;
        PyObject* db = shp[1]->dims;
        int same = da == db;
        if (!same) {
          same = PyObject_RichCompareBool(da, db, Py_EQ);
          if (same < 0) goto fail0;
        }
        const long ba = shp[0]->batch, bb = shp[1]->batch;
        if (same && (ba == bb || ba == 1 || bb == 1)) {
          shape = new_shape(da, ba > bb ? ba : bb);
          if (!shape) goto fail0;
          done = 1;
        }
      }
      break;
    case OP_PICK_RANGE:
      if (n_in == 1 && PyTuple_CheckExact(aux) && PyTuple_GET_SIZE(aux) == 2 && PyTuple_GET_SIZE(shp[0]->dims) == 1) {
        const long lo = PyLong_AsLong(PyTuple_GET_ITEM(aux, 0)), hi = PyLong_AsLong(PyTuple_GET_ITEM(aux, 1));
        if (PyErr_Occurred()) goto fail0;
        const long n = PyLong_AsLong(PyTuple_GET_ITEM(shp[0]->dims, 0));
        if (0 <= lo && lo < hi && hi <= n) {
          PyObject* d = Py_BuildValue("(l)", hi - lo);
          if (!d) goto fail0;
          shape = new_shape(d, shp[0]->batch);
          Py_DECREF(d);
          if (!shape) goto fail0;
          ai_small[0] = lo;
          ai_small[1] = hi;
          n_ai = 2;
          done = 1;
        }
      }
      break;
    case OP_AFFINE:
      if (n_in >= 3 && n_in % 2 == 1 && PyTuple_GET_SIZE(shp[0]->dims) == 1) {
        const long m = PyLong_AsLong(PyTuple_GET_ITEM(shp[0]->dims, 0));
        long batch = shp[0]->batch;
        int ok = 1;
        for (Py_ssize_t k = 1; k + 1 < n_in && ok; k += 2) {
          PyObject *wd = shp[k]->dims, *xd = shp[k + 1]->dims;
          if (PyTuple_GET_SIZE(wd) != 2 || PyTuple_GET_SIZE(xd) != 1) {
            ok = 0;
            break;
          }
          if (PyLong_AsLong(PyTuple_GET_ITEM(wd, 0)) != m ||
              PyLong_AsLong(PyTuple_GET_ITEM(wd, 1)) != PyLong_AsLong(PyTuple_GET_ITEM(xd, 0))) {
            ok = 0;
            break;
          }
          for (int q = 0; q < 2; ++q) {
            const long sb = shp[k + q]->batch;
            if (sb != 1) {
              if (batch != 1 && sb != batch) ok = 0;
              batch = sb;
            }
          }
        }
        if (PyErr_Occurred()) goto fail0;
        if (ok) {
          shape = new_shape(shp[0]->dims, batch);
          if (!shape) goto fail0;
          done = 1;
        }
      }
      break;
    case OP_PARAMETER:
      if (n_in == 0) {
        shape = PyObject_GetAttr(aux, s_shape);
        if (!shape) goto fail0;
        if (!PyObject_TypeCheck(shape, &ShapeBaseType)) {
          Py_CLEAR(shape);
          break;
        }
        int err = 0;
        ai_small[0] = get_long_attr(aux, s_handle, &err);
        if (err) goto fail_shape;
        n_ai = 1;
        fixobj = aux;
        done = 1;
      }
      break;
    case OP_LOOKUP_BATCH:
      if (n_in == 0 && PyTuple_CheckExact(aux) && PyTuple_GET_SIZE(aux) == 2 && PyTuple_CheckExact(PyTuple_GET_ITEM(aux, 1))) {
        PyObject* lp = PyTuple_GET_ITEM(aux, 0);
        PyObject* ids = PyTuple_GET_ITEM(aux, 1);
        const Py_ssize_t nid = PyTuple_GET_SIZE(ids);
        int err = 0;
        const long rows = get_long_attr(lp, s_rows, &err);
        const long dim = err ? 0 : get_long_attr(lp, s_dim, &err);
        const long handle = err ? 0 : get_long_attr(lp, s_handle, &err);
        if (err) goto fail0;
        if (nid == 0) break;
        int64_t* v = (int64_t*)PyMem_Malloc(sizeof(int64_t) * (size_t)(nid + 1));
        if (!v) {
          PyErr_NoMemory();
          goto fail0;
        }
        int ok = 1;
        v[0] = handle;
        for (Py_ssize_t q = 0; q < nid && ok; ++q) {
          const long x = PyLong_AsLong(PyTuple_GET_ITEM(ids, q));
          if (x == -1 && PyErr_Occurred()) {
            PyMem_Free(v);
            goto fail0;
          }
          if (x < 0 || x >= rows) ok = 0;
          v[q + 1] = x;
        }
        if (!ok) {
          PyMem_Free(v);
          break;
        }
        PyObject* d = Py_BuildValue("(l)", dim);
        if (!d) {
          PyMem_Free(v);
          goto fail0;
        }
        shape = new_shape(d, (long)nid);
        Py_DECREF(d);
        if (!shape) {
          PyMem_Free(v);
          goto fail0;
        }
        if (add_fix(c, c->ai.n, lp) < 0 || put_record(c, code, idx, (int)n_in, (ShapeObj*)shape, v, nid + 1, NULL, 0) < 0) {
          PyMem_Free(v);
          goto fail_shape;
        }
        PyMem_Free(v);
        done = 2; /* record written */
      }
      break;
    case OP_LOOKUP:
      if (n_in == 0 && PyTuple_CheckExact(aux) && PyTuple_GET_SIZE(aux) == 2 && PyLong_CheckExact(PyTuple_GET_ITEM(aux, 1))) {
        PyObject* lp = PyTuple_GET_ITEM(aux, 0);
        int err = 0;
        const long rows = get_long_attr(lp, s_rows, &err);
        const long dim = err ? 0 : get_long_attr(lp, s_dim, &err);
        const long handle = err ? 0 : get_long_attr(lp, s_handle, &err);
        if (err) goto fail0;
        const long x = PyLong_AsLong(PyTuple_GET_ITEM(aux, 1));
        if (x == -1 && PyErr_Occurred()) goto fail0;
        if (x < 0 || x >= rows) break; /* the Python rule raises IndexOutOfBounds */
        PyObject* d = Py_BuildValue("(l)", dim);
        if (!d) goto fail0;
        shape = new_shape(d, 1);
        Py_DECREF(d);
        if (!shape) goto fail0;
        const int64_t v[2] = {handle, x};
        if (add_fix(c, c->ai.n, lp) < 0 || put_record(c, code, idx, 0, (ShapeObj*)shape, v, 2, NULL, 0) < 0)
          goto fail_shape;
        done = 2;
      }
      break;
    case OP_CONCATENATE:
      if (n_in >= 1) {
        const long batch = shp[0]->batch;
        long total = 0;
        int ok = 1;
        for (Py_ssize_t k = 0; k < n_in && ok; ++k) {
          if (PyTuple_GET_SIZE(shp[k]->dims) != 1 || shp[k]->batch != batch) ok = 0;
          else total += PyLong_AsLong(PyTuple_GET_ITEM(shp[k]->dims, 0));
        }
        if (PyErr_Occurred()) goto fail0;
        if (ok) {
          PyObject* d = Py_BuildValue("(l)", total);
          if (!d) goto fail0;
          shape = new_shape(d, batch);
          Py_DECREF(d);
          if (!shape) goto fail0;
          done = 1;
        }
      }
      break;
    case OP_PNLS:
      if (n_in == 1 && PyLong_CheckExact(aux) && PyTuple_GET_SIZE(shp[0]->dims) == 1 && shp[0]->batch == 1) {
        const long lab = PyLong_AsLong(aux);
        if (lab == -1 && PyErr_Occurred()) goto fail0;
        const long n = PyLong_AsLong(PyTuple_GET_ITEM(shp[0]->dims, 0));
        if (0 <= lab && lab < n) {
          static PyObject* one1 = NULL;
          if (!one1) one1 = Py_BuildValue("(i)", 1);
          shape = new_shape(one1, 1);
          if (!shape) goto fail0;
          ai_small[0] = lab;
          n_ai = 1;
          done = 1;
        }
      }
      break;
    case OP_PNLS_BATCH:
      if (n_in == 1 && PyTuple_CheckExact(aux) && PyTuple_GET_SIZE(shp[0]->dims) == 1 &&
          PyTuple_GET_SIZE(aux) == shp[0]->batch) {
        const long n = PyLong_AsLong(PyTuple_GET_ITEM(shp[0]->dims, 0));
        const Py_ssize_t nl = PyTuple_GET_SIZE(aux);
        int64_t* v = (int64_t*)PyMem_Malloc(sizeof(int64_t) * (size_t)(nl ? nl : 1));
        if (!v) {
          PyErr_NoMemory();
          goto fail0;
        }
        int ok = 1;
        for (Py_ssize_t q = 0; q < nl && ok; ++q) {
          const long x = PyLong_AsLong(PyTuple_GET_ITEM(aux, q));
          if (x == -1 && PyErr_Occurred()) {
            PyMem_Free(v);
            goto fail0;
          }
          if (x < 0 || x >= n) ok = 0;
          v[q] = x;
        }
        if (!ok) {
          PyMem_Free(v);
          break;
        }
        static PyObject* one = NULL;
        if (!one) one = Py_BuildValue("(i)", 1);
        shape = new_shape(one, shp[0]->batch);
        if (!shape || put_record(c, code, idx, (int)n_in, (ShapeObj*)shape, v, nl, NULL, 0) < 0) {
          PyMem_Free(v);
          goto fail_shape;
        }
        PyMem_Free(v);
        done = 2;
      }
      break;
    case OP_SUM_BATCHES:
      if (n_in == 1) {
        shape = new_shape(shp[0]->dims, 1);
        if (!shape) goto fail0;
        done = 1;
      }
      break;
    case OP_INPUT:
      if (n_in == 0) {
        /* aux is a Tensor: its Shape, and its payload if already contiguous float32 */
        PyObject* sh = PyObject_GetAttr(aux, s_shape);
        if (!sh) goto fail0;
        if (!PyObject_TypeCheck(sh, &ShapeBaseType)) {
          Py_DECREF(sh);
          break;
        }
        PyObject* data = PyObject_GetAttr(aux, s_data);
        if (!data) {
          Py_DECREF(sh);
          goto fail0;
        }
        Py_buffer view;
        if (PyObject_GetBuffer(data, &view, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT) < 0) {
          PyErr_Clear();
          Py_DECREF(data);
          Py_DECREF(sh);
          break;
        }
        const int ok = view.itemsize == 4 && view.format && strcmp(view.format, "f") == 0;
        if (ok) {
          shape = sh;
          if (put_record(c, code, idx, 0, (ShapeObj*)shape, NULL, 0, (const float*)view.buf, view.len / 4) < 0) {
            PyBuffer_Release(&view);
            Py_DECREF(data);
            goto fail_shape;
          }
          done = 2;
        } else {
          Py_DECREF(sh);
        }
        PyBuffer_Release(&view);
        Py_DECREF(data);
      }
      break;
    default:
      break;
  }
  PyObject* od = NULL;
  if (!done) {
    /* Python rule + encode hooks (custom kinds, irregular inputs, errors) */
    od = PyDict_GetItemWithError(Registry, kind);
    if (!od) {
      if (!PyErr_Occurred()) PyErr_SetObject(PyExc_KeyError, kind);
      goto fail0;
    }
    int err = 0;
    code = get_long_attr(od, s_code, &err);
    if (err) goto fail0;
    PyObject* in_shapes = PyList_New(n_in);
    if (!in_shapes) goto fail0;
    for (Py_ssize_t k = 0; k < n_in; ++k) PyList_SET_ITEM(in_shapes, k, Py_NewRef((PyObject*)shp[k]));
    shape = slow_shape(od, aux, in_shapes);
    Py_DECREF(in_shapes);
    if (!shape) goto fail0;
    if (!PyObject_TypeCheck(shape, &ShapeBaseType)) {
      PyErr_SetString(PyExc_TypeError, "shape rule must return a Shape");
      goto fail_shape;
    }
    if (slow_encode(c, od, code, aux, idx, (int)n_in, (ShapeObj*)shape) < 0) goto fail_shape;
  } else if (done == 1) {
    if (fixobj && add_fix(c, c->ai.n, fixobj) < 0) goto fail_shape;
    if (put_record(c, code, idx, (int)n_in, (ShapeObj*)shape, ai_small, n_ai, af_small, n_af) < 0) goto fail_shape;
  }
  /* Node + Expression */
  {
    PyObject* tin = PyTuple_New(n_in);
    if (!tin) goto fail_shape;
    for (Py_ssize_t k = 0; k < n_in; ++k) {
      PyObject* v = PyLong_FromLong(idx[k]);
      if (!v) {
        Py_DECREF(tin);
        goto fail_shape;
      }
      PyTuple_SET_ITEM(tin, k, v);
    }
    NodeObj* nd = (NodeObj*)NodeT->tp_alloc(NodeT, 0);
    untrack((PyObject*)nd);
    if (!nd) {
      Py_DECREF(tin);
      goto fail_shape;
    }
    nd->kind = Py_NewRef(kind);
    untrack((PyObject*)tin);
    nd->inputs = tin;
    nd->shape = shape; /* steals */
    nd->aux = Py_NewRef(aux);
    untrack_atomic_tuple(aux);
    nd->code = code;
    int rc = PyList_Append(c->nodes, (PyObject*)nd);
    Py_DECREF(nd);
    if (rc < 0) goto fail0;
  }
  if (idx != idx_stack) PyMem_Free(idx);
  if (shp != shp_stack) PyMem_Free(shp);
  Py_XDECREF(seq);
  ExprObj* ex = (ExprObj*)ExprT->tp_alloc(ExprT, 0);
  untrack((PyObject*)ex);
  if (!ex) return NULL;
  ex->graph = Py_NewRef(c->cg);
  ex->index = PyList_GET_SIZE(c->nodes) - 1;
  ex->generation = c->gen;
  return (PyObject*)ex;
fail_shape:
  Py_XDECREF(shape);
fail0:
  if (idx != idx_stack) PyMem_Free(idx);
  if (shp != shp_stack) PyMem_Free(shp);
  Py_XDECREF(seq);
  return NULL;
}

/* GraphCore.pack(start) -> (hdr, n, ins, n_ins, ai, n_ai, af, n_af) raw pointers of the
 * records of nodes [start, end) with offsets rebased on the batch; parameter handles
 * are resolved first.  The pointers stay valid until the next add/renew. */
static PyObject* core_pack(CoreObj* c, PyObject* arg) {
  const Py_ssize_t start = PyLong_AsSsize_t(arg);
  if (start == -1 && PyErr_Occurred()) return NULL;
  const Py_ssize_t end = c->hdr.n / HDR;
  if (start < 0 || start > end) {
    PyErr_SetString(PyExc_IndexError, "pack start out of range");
    return NULL;
  }
  const Py_ssize_t nfix = PyList_GET_SIZE(c->fix);
  for (Py_ssize_t q = 0; q < nfix; ++q) {
    PyObject* t = PyList_GET_ITEM(c->fix, q);
    const Py_ssize_t pos = PyLong_AsSsize_t(PyTuple_GET_ITEM(t, 0));
    int err = 0;
    const long h = get_long_attr(PyTuple_GET_ITEM(t, 1), s_handle, &err);
    if (err) return NULL;
    ((int64_t*)c->ai.p)[pos] = h;
  }
  const Py_ssize_t n = end - start;
  c->rebased.n = 0;
  if (buf_reserve(&c->rebased, n * HDR + 1)) return NULL;
  int32_t* dst = (int32_t*)c->rebased.p;
  const int32_t* src = (const int32_t*)c->hdr.p + start * HDR;
  int32_t in0 = 0, ai0 = 0, af0 = 0;
  if (n > 0) {
    in0 = src[2];
    ai0 = src[9];
    af0 = src[11];
  }
  for (Py_ssize_t i = 0; i < n; ++i) {
    memcpy(dst + i * HDR, src + i * HDR, sizeof(int32_t) * HDR);
    dst[i * HDR + 2] -= in0;
    dst[i * HDR + 9] -= ai0;
    dst[i * HDR + 11] -= af0;
  }
  return Py_BuildValue("(KnKnKnKn)", (unsigned long long)(uintptr_t)dst, n,
                       (unsigned long long)(uintptr_t)((int32_t*)c->ins.p + in0), c->ins.n - in0,
                       (unsigned long long)(uintptr_t)((int64_t*)c->ai.p + ai0), c->ai.n - ai0,
                       (unsigned long long)(uintptr_t)((float*)c->af.p + af0), c->af.n - af0);
}

/* ---- composite builders: the node sequence of builders.py emitted without
   per-node Python frames (same kinds, same order, same shapes) */
static PyObject *k_affine = NULL, *k_pick = NULL, *k_logistic = NULL, *k_tanh = NULL, *k_cmult = NULL, *k_add = NULL;

static PyObject* add1(CoreObj* c, PyObject* kind, PyObject* a, PyObject* aux) {
  PyObject* t = PyTuple_Pack(1, a);
  if (!t) return NULL;
  PyObject* args[3] = {kind, t, aux};
  PyObject* r = core_add(c, args, 3);
  Py_DECREF(t);
  return r;
}

static PyObject* add2(CoreObj* c, PyObject* kind, PyObject* a, PyObject* b) {
  PyObject* t = PyTuple_Pack(2, a, b);
  if (!t) return NULL;
  PyObject* args[3] = {kind, t, Py_None};
  PyObject* r = core_add(c, args, 3);
  Py_DECREF(t);
  return r;
}

static PyObject* gate(CoreObj* c, PyObject* gates, long lo, long hi, PyObject* act) {
  PyObject* rng = Py_BuildValue("(ll)", lo, hi);
  if (!rng) return NULL;
  PyObject* p = add1(c, k_pick, gates, rng);
  Py_DECREF(rng);
  if (!p) return NULL;
  PyObject* r = add1(c, act, p, Py_None);
  Py_DECREF(p);
  return r;
}

/* GraphCore.lstm(b, wx, x, wh, h, c, H) -> (h', c'): builders.py
   RNNBuilder._lstm (i, f, o, g gate blocks of the affine output) */
static PyObject* lstm_generic(CoreObj* c, PyObject* const* args, long H) {
  PyObject *gates = NULL, *ig = NULL, *fg = NULL, *og = NULL, *gg = NULL, *fc = NULL, *igg = NULL, *nc = NULL,
           *tc = NULL, *nh = NULL, *ret = NULL;
  PyObject* ins = PyTuple_Pack(5, args[0], args[1], args[2], args[3], args[4]);
  if (!ins) return NULL;
  PyObject* aargs[3] = {k_affine, ins, Py_None};
  gates = core_add(c, aargs, 3);
  Py_DECREF(ins);
  if (!gates) return NULL;
  if (!(ig = gate(c, gates, 0, H, k_logistic))) goto done;
  if (!(fg = gate(c, gates, H, 2 * H, k_logistic))) goto done;
  if (!(og = gate(c, gates, 2 * H, 3 * H, k_logistic))) goto done;
  if (!(gg = gate(c, gates, 3 * H, 4 * H, k_tanh))) goto done;
  if (!(fc = add2(c, k_cmult, fg, args[5]))) goto done;
  if (!(igg = add2(c, k_cmult, ig, gg))) goto done;
  if (!(nc = add2(c, k_add, fc, igg))) goto done;
  if (!(tc = add1(c, k_tanh, nc, Py_None))) goto done;
  if (!(nh = add2(c, k_cmult, og, tc))) goto done;
  ret = PyTuple_Pack(2, nh, nc);
done:
  Py_XDECREF(gates);
  Py_XDECREF(ig);
  Py_XDECREF(fg);
  Py_XDECREF(og);
  Py_XDECREF(gg);
  Py_XDECREF(fc);
  Py_XDECREF(igg);
  Py_XDECREF(nc);
  Py_XDECREF(tc);
  Py_XDECREF(nh);
  return ret;
}


/* one record + Node for the fast composite path; returns the node index */
static Py_ssize_t emit(CoreObj* c, PyObject* kind, long code, const int32_t* idx, int n_in, PyObject* shape,
                       const int64_t* ai, Py_ssize_t n_ai, PyObject* aux) {
  if (put_record(c, code, idx, n_in, (ShapeObj*)shape, ai, n_ai, NULL, 0) < 0) return -1;
  PyObject* tin = PyTuple_New(n_in);
  if (!tin) return -1;
  for (int k = 0; k < n_in; ++k) {
    PyObject* v = PyLong_FromLong(idx[k]);
    if (!v) {
      Py_DECREF(tin);
      return -1;
    }
    PyTuple_SET_ITEM(tin, k, v);
  }
  untrack(tin);
  NodeObj* nd = (NodeObj*)NodeT->tp_alloc(NodeT, 0);
  if (!nd) {
    Py_DECREF(tin);
    return -1;
  }
  untrack((PyObject*)nd);
  nd->kind = Py_NewRef(kind);
  nd->inputs = tin;
  nd->shape = Py_NewRef(shape);
  nd->aux = Py_NewRef(aux);
  nd->code = code;
  const int rc = PyList_Append(c->nodes, (PyObject*)nd);
  Py_DECREF(nd);
  return rc < 0 ? -1 : PyList_GET_SIZE(c->nodes) - 1;
}

static PyObject* new_expr(CoreObj* c, Py_ssize_t index) {
  ExprObj* ex = (ExprObj*)ExprT->tp_alloc(ExprT, 0);
  if (!ex) return NULL;
  untrack((PyObject*)ex);
  ex->graph = Py_NewRef(c->cg);
  ex->index = index;
  ex->generation = c->gen;
  return (PyObject*)ex;
}

static long kind_code(PyObject* kind) {
  PyObject* v = PyDict_GetItemWithError(FastKinds, kind);
  return v ? PyLong_AsLong(v) : -1;
}

static long dim_at(ShapeObj* s, Py_ssize_t d) {
  return d < PyTuple_GET_SIZE(s->dims) ? PyLong_AsLong(PyTuple_GET_ITEM(s->dims, d)) : -1;
}

/* GraphCore.lstm(b, wx, x, wh, h, c, H) -> (h', c'): the 14 nodes of
   builders.py RNNBuilder._lstm (affine; i, f, o, g gate blocks; c' = f*c + i*g;
   h' = o*tanh(c')), written straight into the record buffers with only the
   two returned expressions materialised.  Anything irregular (re-registered
   kinds, shape or batch mismatches, foreign expressions) takes the generic
   node-by-node path, which raises the reference errors. */
static PyObject* core_lstm(CoreObj* c, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 7) {
    PyErr_SetString(PyExc_TypeError, "lstm(b, wx, x, wh, h, c, H)");
    return NULL;
  }
  const long H = PyLong_AsLong(args[6]);
  if (H == -1 && PyErr_Occurred()) return NULL;
  const long c_aff = kind_code(k_affine), c_pick = kind_code(k_pick), c_log = kind_code(k_logistic),
             c_tanh = kind_code(k_tanh), c_cm = kind_code(k_cmult), c_add = kind_code(k_add);
  if (PyErr_Occurred()) return NULL;
  const Py_ssize_t n_nodes = PyList_GET_SIZE(c->nodes);
  int32_t in[6];
  ShapeObj* sh[6];
  int ok = c_aff >= 0 && c_pick >= 0 && c_log >= 0 && c_tanh >= 0 && c_cm >= 0 && c_add >= 0 && H > 0;
  for (int k = 0; k < 6 && ok; ++k) {
    PyObject* e = args[k];
    if (!PyObject_TypeCheck(e, &ExprBaseType) || ((ExprObj*)e)->graph != c->cg || ((ExprObj*)e)->generation != c->gen ||
        ((ExprObj*)e)->index < 0 || ((ExprObj*)e)->index >= n_nodes) {
      ok = 0;
      break;
    }
    in[k] = (int32_t)((ExprObj*)e)->index;
    sh[k] = (ShapeObj*)((NodeObj*)PyList_GET_ITEM(c->nodes, in[k]))->shape;
  }
  /* b (4H) | wx (4H, X) | x (X) | wh (4H, H) | h (H) | c (H) */
  if (ok) {
    const long X = dim_at(sh[2], 0);
    ok = PyTuple_GET_SIZE(sh[0]->dims) == 1 && dim_at(sh[0], 0) == 4 * H && PyTuple_GET_SIZE(sh[1]->dims) == 2 &&
         dim_at(sh[1], 0) == 4 * H && dim_at(sh[1], 1) == X && PyTuple_GET_SIZE(sh[2]->dims) == 1 &&
         PyTuple_GET_SIZE(sh[3]->dims) == 2 && dim_at(sh[3], 0) == 4 * H && dim_at(sh[3], 1) == H &&
         PyTuple_GET_SIZE(sh[4]->dims) == 1 && dim_at(sh[4], 0) == H && PyTuple_GET_SIZE(sh[5]->dims) == 1 &&
         dim_at(sh[5], 0) == H;
    if (PyErr_Occurred()) return NULL;
  }
  long ba = 1, bn = 1;
  if (ok) {
    ba = sh[0]->batch;
    for (int k = 1; k < 5; ++k) {
      const long sb = sh[k]->batch;
      if (sb != 1) {
        if (ba != 1 && sb != ba) ok = 0;
        ba = sb;
      }
    }
    const long bc = sh[5]->batch;
    if (!(bc == ba || bc == 1 || ba == 1)) ok = 0;
    bn = ba > bc ? ba : bc;
  }
  if (!ok) return lstm_generic(c, args, H);

  PyObject *shA = NULL, *shG = NULL, *shN = NULL, *rng[4] = {NULL, NULL, NULL, NULL}, *ret = NULL, *eh = NULL,
           *ec = NULL;
  Py_ssize_t base = n_nodes, r = 0;
  if (!(shA = new_shape(sh[0]->dims, ba))) goto out;
  if (!(shG = new_shape(sh[4]->dims, ba))) goto out;
  if (bn == ba) {
    shN = Py_NewRef(shG);
  } else if (!(shN = new_shape(sh[4]->dims, bn))) {
    goto out;
  }
  for (int q = 0; q < 4; ++q) {
    if (!(rng[q] = Py_BuildValue("(ll)", q * H, (q + 1) * H))) goto out;
    untrack(rng[q]);
  }
  {
    const int32_t A = (int32_t)base;
    const int32_t iA[5] = {in[0], in[1], in[2], in[3], in[4]};
    r = emit(c, k_affine, c_aff, iA, 5, shA, NULL, 0, Py_None); /* base+0 */
    for (int q = 0; q < 4 && r >= 0; ++q) {                      /* pick, act: base+1+2q, base+2+2q */
      const int64_t lohi[2] = {(int64_t)q * H, (int64_t)(q + 1) * H};
      r = emit(c, k_pick, c_pick, &A, 1, shG, lohi, 2, rng[q]);
      if (r < 0) break;
      const int32_t p = (int32_t)r;
      r = q == 3 ? emit(c, k_tanh, c_tanh, &p, 1, shG, NULL, 0, Py_None)
                 : emit(c, k_logistic, c_log, &p, 1, shG, NULL, 0, Py_None);
    }
    if (r < 0) goto out;
    const int32_t ig = A + 2, fg = A + 4, og = A + 6, gg = A + 8;
    const int32_t fc_in[2] = {fg, in[5]}, igg_in[2] = {ig, gg}, nc_in[2] = {A + 9, A + 10};
    if ((r = emit(c, k_cmult, c_cm, fc_in, 2, shN, NULL, 0, Py_None)) < 0) goto out; /* base+9 */
    if ((r = emit(c, k_cmult, c_cm, igg_in, 2, shG, NULL, 0, Py_None)) < 0) goto out; /* base+10 */
    if ((r = emit(c, k_add, c_add, nc_in, 2, shN, NULL, 0, Py_None)) < 0) goto out; /* base+11 */
    const int32_t nc = A + 11;
    if ((r = emit(c, k_tanh, c_tanh, &nc, 1, shN, NULL, 0, Py_None)) < 0) goto out; /* base+12 */
    const int32_t nh_in[2] = {og, A + 12};
    if ((r = emit(c, k_cmult, c_cm, nh_in, 2, shN, NULL, 0, Py_None)) < 0) goto out; /* base+13 */
    if (!(eh = new_expr(c, base + 13)) || !(ec = new_expr(c, base + 11))) goto out;
    ret = PyTuple_Pack(2, eh, ec);
  }
out:
  Py_XDECREF(shA);
  Py_XDECREF(shG);
  Py_XDECREF(shN);
  for (int q = 0; q < 4; ++q) Py_XDECREF(rng[q]);
  Py_XDECREF(eh);
  Py_XDECREF(ec);
  return ret;
}

/* Tree-LSTM (builders.py TreeLSTM._compose / encode): the node sequence of
   one leaf or one binary internal cell, node for node, without per-node
   Python frames; returns (h, c). */
static PyObject* tree_compose(CoreObj* c, PyObject* gates, PyObject* t1, PyObject* t2, long H) {
  PyObject *ig = NULL, *og = NULL, *gg = NULL, *cc = NULL, *tc = NULL, *h = NULL, *ret = NULL;
  if (!(ig = gate(c, gates, 0, H, k_logistic))) goto out;
  if (!(og = gate(c, gates, 3 * H, 4 * H, k_logistic))) goto out;
  if (!(gg = gate(c, gates, 4 * H, 5 * H, k_tanh))) goto out;
  if (!(cc = add2(c, k_cmult, ig, gg))) goto out;
  if (t1) Py_SETREF(cc, add2(c, k_add, cc, t1));
  if (!cc) goto out;
  if (t2) Py_SETREF(cc, add2(c, k_add, cc, t2));
  if (!cc) goto out;
  if (!(tc = add1(c, k_tanh, cc, Py_None))) goto out;
  if (!(h = add2(c, k_cmult, og, tc))) goto out;
  ret = PyTuple_Pack(2, h, cc);
out:
  Py_XDECREF(ig);
  Py_XDECREF(og);
  Py_XDECREF(gg);
  Py_XDECREF(cc);
  Py_XDECREF(tc);
  Py_XDECREF(h);
  return ret;
}

/* GraphCore.tree_leaf(b, wx, x, H) -> (h, c) */
static PyObject* core_tree_leaf(CoreObj* c, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 4) {
    PyErr_SetString(PyExc_TypeError, "tree_leaf(b, wx, x, H)");
    return NULL;
  }
  const long H = PyLong_AsLong(args[3]);
  if (H == -1 && PyErr_Occurred()) return NULL;
  PyObject* ins = PyTuple_Pack(3, args[0], args[1], args[2]);
  if (!ins) return NULL;
  PyObject* aargs[3] = {k_affine, ins, Py_None};
  PyObject* gates = core_add(c, aargs, 3);
  Py_DECREF(ins);
  if (!gates) return NULL;
  PyObject* r = tree_compose(c, gates, NULL, NULL, H);
  Py_DECREF(gates);
  return r;
}

/* GraphCore.tree_node(b, u1, h1, u2, h2, c1, c2, H) -> (h, c) */
static PyObject* core_tree_node(CoreObj* c, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 8) {
    PyErr_SetString(PyExc_TypeError, "tree_node(b, u1, h1, u2, h2, c1, c2, H)");
    return NULL;
  }
  const long H = PyLong_AsLong(args[7]);
  if (H == -1 && PyErr_Occurred()) return NULL;
  PyObject *gates = NULL, *f1 = NULL, *f2 = NULL, *t1 = NULL, *t2 = NULL, *ret = NULL;
  PyObject* ins = PyTuple_Pack(5, args[0], args[1], args[2], args[3], args[4]);
  if (!ins) return NULL;
  PyObject* aargs[3] = {k_affine, ins, Py_None};
  gates = core_add(c, aargs, 3);
  Py_DECREF(ins);
  if (!gates) return NULL;
  if (!(f1 = gate(c, gates, H, 2 * H, k_logistic))) goto out;
  if (!(f2 = gate(c, gates, 2 * H, 3 * H, k_logistic))) goto out;
  if (!(t1 = add2(c, k_cmult, f1, args[5]))) goto out;
  if (!(t2 = add2(c, k_cmult, f2, args[6]))) goto out;
  ret = tree_compose(c, gates, t1, t2, H);
out:
  Py_XDECREF(gates);
  Py_XDECREF(f1);
  Py_XDECREF(f2);
  Py_XDECREF(t1);
  Py_XDECREF(t2);
  return ret;
}

/* one step through a stack of LSTM layers: pexprs[l] = (wx, wh, b); returns
   (hs', cs') as new lists (builders.py RNNBuilder._step, cell = "lstm") */
static int lstm_stack_step(CoreObj* c, PyObject* pexprs, PyObject* hs, PyObject* cs, PyObject* x, PyObject* Hobj,
                           PyObject** nhs_out, PyObject** ncs_out) {
  const Py_ssize_t L = PyList_GET_SIZE(pexprs);
  PyObject* nhs = PyList_New(L);
  PyObject* ncs = PyList_New(L);
  if (!nhs || !ncs) goto fail;
  PyObject* inp = x;
  for (Py_ssize_t l = 0; l < L; ++l) {
    PyObject* pe = PyList_GET_ITEM(pexprs, l);
    if (!PyTuple_CheckExact(pe) || PyTuple_GET_SIZE(pe) != 3) {
      PyErr_SetString(PyExc_TypeError, "layer parameters must be (wx, wh, b)");
      goto fail;
    }
    PyObject* a[7] = {PyTuple_GET_ITEM(pe, 2), PyTuple_GET_ITEM(pe, 0), inp,   PyTuple_GET_ITEM(pe, 1),
                      PyList_GET_ITEM(hs, l), PyList_GET_ITEM(cs, l), Hobj};
    PyObject* r = core_lstm(c, a, 7);
    if (!r) goto fail;
    PyList_SET_ITEM(nhs, l, Py_NewRef(PyTuple_GET_ITEM(r, 0)));
    PyList_SET_ITEM(ncs, l, Py_NewRef(PyTuple_GET_ITEM(r, 1)));
    Py_DECREF(r);
    inp = PyList_GET_ITEM(nhs, l);
  }
  *nhs_out = nhs;
  *ncs_out = ncs;
  return 0;
fail:
  Py_XDECREF(nhs);
  Py_XDECREF(ncs);
  return -1;
}

static int check_stack_args(PyObject* pexprs, PyObject* hs, PyObject* cs) {
  if (!PyList_CheckExact(pexprs) || !PyList_CheckExact(hs) || !PyList_CheckExact(cs) ||
      PyList_GET_SIZE(hs) != PyList_GET_SIZE(pexprs) || PyList_GET_SIZE(cs) != PyList_GET_SIZE(pexprs)) {
    PyErr_SetString(PyExc_TypeError, "layer lists (params, hs, cs) must be lists of equal length");
    return -1;
  }
  return 0;
}

/* GraphCore.lstm_step(pexprs, hs, cs, x, H) -> (hs', cs') */
static PyObject* core_lstm_step(CoreObj* c, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 5) {
    PyErr_SetString(PyExc_TypeError, "lstm_step(pexprs, hs, cs, x, H)");
    return NULL;
  }
  if (check_stack_args(args[0], args[1], args[2]) < 0) return NULL;
  PyObject *nhs, *ncs;
  if (lstm_stack_step(c, args[0], args[1], args[2], args[3], args[4], &nhs, &ncs) < 0) return NULL;
  PyObject* r = PyTuple_Pack(2, nhs, ncs);
  Py_DECREF(nhs);
  Py_DECREF(ncs);
  return r;
}

/* GraphCore.lstm_transduce(pexprs, hs, cs, xs, H) -> [top h per step]
   (builders.py RNNState.transduce over lstm_step) */
static PyObject* core_lstm_transduce(CoreObj* c, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 5) {
    PyErr_SetString(PyExc_TypeError, "lstm_transduce(pexprs, hs, cs, xs, H)");
    return NULL;
  }
  if (check_stack_args(args[0], args[1], args[2]) < 0) return NULL;
  PyObject* xs = PySequence_Fast(args[3], "xs must be a sequence");
  if (!xs) return NULL;
  const Py_ssize_t T = PySequence_Fast_GET_SIZE(xs);
  PyObject* outs = PyList_New(T);
  PyObject* hs = Py_NewRef(args[1]);
  PyObject* cs = Py_NewRef(args[2]);
  if (!outs) goto fail;
  for (Py_ssize_t t = 0; t < T; ++t) {
    PyObject *nhs, *ncs;
    if (lstm_stack_step(c, args[0], hs, cs, PySequence_Fast_GET_ITEM(xs, t), args[4], &nhs, &ncs) < 0) goto fail;
    Py_SETREF(hs, nhs);
    Py_SETREF(cs, ncs);
    PyList_SET_ITEM(outs, t, Py_NewRef(PyList_GET_ITEM(hs, PyList_GET_SIZE(hs) - 1)));
  }
  Py_DECREF(hs);
  Py_DECREF(cs);
  Py_DECREF(xs);
  return outs;
fail:
  Py_XDECREF(outs);
  Py_XDECREF(hs);
  Py_XDECREF(cs);
  Py_DECREF(xs);
  return NULL;
}

static PyMethodDef core_methods[] = {
    {"add", (PyCFunction)(void (*)(void))core_add, METH_FASTCALL, "add(kind, inputs=(), aux=None) -> Expression"},
    {"renew", (PyCFunction)core_renew, METH_O, "renew(generation)"},
    {"pack", (PyCFunction)core_pack, METH_O, "pack(start) -> raw record pointers"},
    {"lstm", (PyCFunction)(void (*)(void))core_lstm, METH_FASTCALL, "lstm(b, wx, x, wh, h, c, H) -> (h, c)"},
    {"tree_leaf", (PyCFunction)(void (*)(void))core_tree_leaf, METH_FASTCALL, "tree_leaf(b, wx, x, H) -> (h, c)"},
    {"tree_node", (PyCFunction)(void (*)(void))core_tree_node, METH_FASTCALL,
     "tree_node(b, u1, h1, u2, h2, c1, c2, H) -> (h, c)"},
    {"lstm_step", (PyCFunction)(void (*)(void))core_lstm_step, METH_FASTCALL,
     "lstm_step(pexprs, hs, cs, x, H) -> (hs, cs)"},
    {"lstm_transduce", (PyCFunction)(void (*)(void))core_lstm_transduce, METH_FASTCALL,
     "lstm_transduce(pexprs, hs, cs, xs, H) -> outputs"},
    {NULL}};

static PyTypeObject CoreType = {PyVarObject_HEAD_INIT(NULL, 0).tp_name = "_dgcore.GraphCore",
                                .tp_basicsize = sizeof(CoreObj),
                                .tp_dealloc = (destructor)core_dealloc,
                                .tp_flags = Py_TPFLAGS_DEFAULT,
                                .tp_methods = core_methods,
                                .tp_init = (initproc)core_init,
                                .tp_new = PyType_GenericNew};

/* setup(ShapeCls, NodeCls, ExprCls, registry, fast_kinds) */
static PyObject* mod_setup(PyObject* self, PyObject* args) {
  PyObject *st, *nt, *et, *reg, *fk;
  if (!PyArg_ParseTuple(args, "O!O!O!O!O!", &PyType_Type, &st, &PyType_Type, &nt, &PyType_Type, &et, &PyDict_Type,
                        &reg, &PyDict_Type, &fk))
    return NULL;
  if (!PyType_IsSubtype((PyTypeObject*)st, &ShapeBaseType) || !PyType_IsSubtype((PyTypeObject*)nt, &NodeBaseType) ||
      !PyType_IsSubtype((PyTypeObject*)et, &ExprBaseType)) {
    PyErr_SetString(PyExc_TypeError, "setup needs subclasses of ShapeBase / NodeBase / ExprBase");
    return NULL;
  }
  Py_XSETREF(ShapeT, (PyTypeObject*)Py_NewRef(st));
  Py_XSETREF(NodeT, (PyTypeObject*)Py_NewRef(nt));
  Py_XSETREF(ExprT, (PyTypeObject*)Py_NewRef(et));
  Py_XSETREF(Registry, Py_NewRef(reg));
  Py_XSETREF(FastKinds, Py_NewRef(fk));
  Py_RETURN_NONE;
}

/* int_tuple(seq) == tuple(map(int, seq)), without a call per exact int */
static PyObject* mod_int_tuple(PyObject* self, PyObject* seq) {
  PyObject* t = PySequence_Tuple(seq);
  if (!t) return NULL;
  const Py_ssize_t n = PyTuple_GET_SIZE(t);
  for (Py_ssize_t k = 0; k < n; ++k) {
    PyObject* v = PyTuple_GET_ITEM(t, k);
    if (PyLong_CheckExact(v)) continue;
    PyObject* iv = PyNumber_Long(v);
    if (!iv) {
      Py_DECREF(t);
      return NULL;
    }
    if (Py_REFCNT(t) == 1 && t != seq) {
      PyTuple_SET_ITEM(t, k, iv);
      Py_DECREF(v);
    } else { /* PySequence_Tuple returned the caller's tuple: copy first */
      PyObject* c = PyTuple_GetSlice(t, 0, n);
      Py_DECREF(t);
      if (!c) {
        Py_DECREF(iv);
        return NULL;
      }
      t = c;
      Py_DECREF(PyTuple_GET_ITEM(t, k));
      PyTuple_SET_ITEM(t, k, iv);
    }
  }
  untrack(t);
  return t;
}

static PyMethodDef mod_methods[] = {{"setup", mod_setup, METH_VARARGS, "register the Python subclasses"},
                                    {"int_tuple", mod_int_tuple, METH_O, "tuple(map(int, seq))"},
                                    {NULL}};

static struct PyModuleDef moddef = {PyModuleDef_HEAD_INIT, "_dgcore", "native graph construction", -1, mod_methods};

PyMODINIT_FUNC PyInit__dgcore(void) {
  if (PyType_Ready(&ShapeBaseType) < 0 || PyType_Ready(&NodeBaseType) < 0 || PyType_Ready(&ExprBaseType) < 0 ||
      PyType_Ready(&CoreType) < 0)
    return NULL;
  PyObject* m = PyModule_Create(&moddef);
  if (!m) return NULL;
  s_shape = PyUnicode_InternFromString("shape");
  k_affine = PyUnicode_InternFromString("affine");
  k_pick = PyUnicode_InternFromString("pick_range");
  k_logistic = PyUnicode_InternFromString("logistic");
  k_tanh = PyUnicode_InternFromString("tanh");
  k_cmult = PyUnicode_InternFromString("cmult");
  k_add = PyUnicode_InternFromString("add");
  s_encode = PyUnicode_InternFromString("encode");
  s_handle = PyUnicode_InternFromString("handle");
  s_rows = PyUnicode_InternFromString("rows");
  s_dim = PyUnicode_InternFromString("dim");
  s_data = PyUnicode_InternFromString("data");
  s_check_current = PyUnicode_InternFromString("check_current");
  s_code = PyUnicode_InternFromString("code");
  Py_INCREF(&ShapeBaseType);
  Py_INCREF(&NodeBaseType);
  Py_INCREF(&ExprBaseType);
  Py_INCREF(&CoreType);
  if (PyModule_AddObject(m, "ShapeBase", (PyObject*)&ShapeBaseType) < 0 ||
      PyModule_AddObject(m, "NodeBase", (PyObject*)&NodeBaseType) < 0 ||
      PyModule_AddObject(m, "ExprBase", (PyObject*)&ExprBaseType) < 0 ||
      PyModule_AddObject(m, "GraphCore", (PyObject*)&CoreType) < 0)
    return NULL;
  return m;
}
