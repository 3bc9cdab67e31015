// Native executor behind include/dyngpu.h.
//
// Replaces the reference's per-node interpreter (pkg/src/dyncore/graph.py:115-164)
// with a batching planner:
//   1. rewrite left-deep chains of equal-shape `add` nodes (the loss chain,
//      bench/tasks.py:419,439,558, and Tree-LSTM cell sums builders.py:255-257)
//      into one n-ary prefix-sum unit, so the per-step loss terms do not
//      serialise the graph;
//   2. schedule units by list scheduling over dependency levels: a signature
//      group (kind, shapes, shared parameter identity, aux) is launched when one
//      of its ready members becomes urgent (its ALAP level is reached), and it
//      then takes every ready member -> recurrent steps batch across layers,
//      non-recurrent branches (output affine, pnls, masks) batch across all
//      time steps, tree nodes batch by height;
//   3. lay every group's outputs out contiguously in the forward arena (same
//      total bytes as the reference bump allocator, so PoolExhausted and
//      alloc_count semantics are unchanged) and upload one table blob per call;
//   4. backward walks the groups in reverse; parameter gradients accumulate in
//      place (the default sink, graph.py:51-63), weight gradients of every use
//      of a parameter are aggregated into ONE GEMM (K = all rows), lookup rows
//      are flushed by an atomic-free sorted segmented scatter-add.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/dyngpu.h"
#include "kernels.cuh"

namespace dg {

// --------------------------------------------------------------------- errors
static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define DG_CUDA_TRY(expr)                                                          \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) return fail(DG_CUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
  } while (0)

// ------------------------------------------------------------ param registry
struct Param {
  int kind = 0;  // 0 dense, 1 lookup
  int64_t rows = 0, cols = 0;
  float* val = nullptr;
  float* grad = nullptr;
  bool alive = false;
  std::vector<uint8_t> touched_bits;
  std::vector<int64_t> touched_list;  // insertion order; sorted on read
  int64_t size() const { return rows * cols; }
  std::vector<int32_t> sort_cnt;  // scatter planning scratch (all zero at rest)
  void* dp_dev = nullptr;         // DP merge staging (dg_lookup_merge)
  size_t dp_cap = 0;
};

static std::mutex g_param_mu;
static std::vector<Param> g_params;
// bumped whenever a parameter's device storage may move: cached plans embed
// parameter pointers, so it is part of their key
static std::atomic<uint64_t> g_param_epoch{1};

static Param* param_at(int64_t h) {
  if (h < 0 || h >= (int64_t)g_params.size() || !g_params[h].alive) return nullptr;
  return &g_params[h];
}

static void touch(Param& p, int64_t id) {
  if (!p.touched_bits[id]) {
    p.touched_bits[id] = 1;
    p.touched_list.push_back(id);
  }
}

static std::vector<int64_t> touched_sorted(Param& p) {
  std::vector<int64_t> v = p.touched_list;
  std::sort(v.begin(), v.end());
  return v;
}

static void touched_clear(Param& p) {
  for (int64_t id : p.touched_list) p.touched_bits[id] = 0;
  p.touched_list.clear();
}

// ------------------------------------------------------------------ staging
// One table blob per forward/backward call: built on the host, copied with a
// single H2D into the head of the workspace; kernels read it from there.
struct Pinned {
  void* ptr = nullptr;
  size_t cap = 0;
  cudaEvent_t ev = nullptr;
  bool pending = false;
};

// Written straight into a pinned staging slot when one is attached (no host
// copy before the H2D); a plan that outgrows the slot moves to a vector.
struct Blob {
  std::vector<uint8_t> vec;
  uint8_t* ext = nullptr;
  size_t ext_cap = 0;
  Pinned* slot = nullptr;
  size_t n = 0;
  uint8_t* data() { return ext ? ext : vec.data(); }
  const uint8_t* data() const { return ext ? ext : vec.data(); }
  size_t size() const { return n; }
  bool empty() const { return n == 0; }
  size_t push_bytes(const void* p, size_t bytes, size_t align = 16) {
    const size_t off = (n + align - 1) & ~(align - 1);
    if (ext && off + bytes > ext_cap) {  // spill
      vec.assign(ext, ext + n);
      ext = nullptr;
      slot = nullptr;
    }
    if (!ext && vec.size() < off + bytes) vec.resize(std::max(off + bytes, 2 * vec.size()));
    if (bytes) std::memcpy(data() + off, p, bytes);
    n = off + bytes;
    return off;
  }
  template <class T>
  size_t push(const std::vector<T>& v) {
    return push_bytes(v.data(), v.size() * sizeof(T));
  }
};

// -------------------------------------------------------------------- graph
struct Node {
  int kind, n_in, in_off, rank;
  int dims[4];
  int batch;
  int64_t elem;
  int64_t ai_off, ai_len, af_off, af_len;
  float* val = nullptr;
  float* grad = nullptr;
  int64_t size() const { return elem * batch; }
};

static inline size_t round64(size_t n) { return (n + 63) & ~size_t(63); }

enum UnitKind { U_NODE = 0, U_CHAIN = 1, U_CELL = 2, U_RNN = 3, U_GRUA = 4, U_GRUB = 5, U_PNLS2 = 6 };

struct Unit {
  int type;                 // U_NODE / U_CHAIN / U_CELL
  std::vector<int> nodes;   // U_NODE: {i}; U_CHAIN: add nodes in chain order;
                            // U_CELL: nodes in kernels.cuh CellArgs slot order
                            //         (picks, acts, prods, adds, tanh(c), h)
  std::vector<int> ins;     // external inputs (node indices) in slot order
  // U_CELL: children m, gate offsets into G (i, o, g, f0, f1), G width, H
  int m = 0;
  int off[5] = {0, 0, 0, 0, 0};
  int gw = 0, H = 0;
  int rnn = -1;  // U_RNN: index into Schedule::rnns
  int first() const { return nodes.front(); }
  int last() const { return nodes.back(); }
};

// A chain of LSTM steps sharing (Wx, Wh, b) whose h_t / c_t feed step t+1
// (builders.py:92-101), run by the persistent recurrence kernels (rnn.cu).
struct RnnChainPlan {
  std::vector<Unit> cells;  // per step: the U_CELL (m = 1) unit
  std::vector<int> G;       // per step: the gate affine node
  int64_t hb = -1, hWx = -1, hWh = -1;
  int H = 0, K_in = 0, B = 0, gw = 0;
  int off[4] = {0, 0, 0, 0};  // i, f, o, g gate offsets into G
  int src = -1;               // stacked producer chain (index in the stack)
  int cons = -1;              // consumer chain
  int n_s = 0, n_u = 0;
};
struct RnnStack {
  std::vector<RnnChainPlan> chains;
  int bs = 1, ctas = 0;
};

struct Group {
  int kind;                 // node kind, -1 add chain, -2 gated cell, -3 LSTM stack
  std::vector<int> units;   // unit ids, ascending
  int level = 0;            // scheduling level (groups of one level are independent)
};

struct Schedule {
  std::vector<Unit> units;
  std::vector<int> unit_of;        // node -> unit id (or -1 when not scheduled)
  std::vector<Group> groups;       // execution order (forward)
  std::vector<int> input_nodes;    // `input` leaves
  std::vector<int> lookup_nodes;   // lookup / lookup_batch leaves
  std::vector<int> param_nodes;
  std::vector<RnnStack> rnns;
};

struct AffineUse {  // weight-gradient aggregation (one GEMM per parameter)
  std::vector<uintptr_t> x_rows;  // device pointers (forward values)
  std::vector<uintptr_t> g_rows;  // device pointers (grad slots)
  int64_t n_in = 0, m = 0;
};

struct dg_graph_impl;

}  // namespace dg

namespace dg {
struct Schedule;
struct CachedPlan;
// Gradient of an INPUT leaf that the backward pass leaves as per-slice
// partial sums (the batch-1 initial states of the LSTM recurrences): the
// reference computes it during backward, but only gradient() can observe it,
// so the final slice sum runs when gradient() asks for that node.
struct LazyGrad {
  int node;
  float* dst;
  const float* part;
  int n_s, H;
};

}

struct dg_graph {
  // last schedule of this graph generation (forward then backward of the same
  // node set reuse it without rehashing the node table)
  mutable std::shared_ptr<const dg::Schedule> memo_sched;
  mutable std::vector<int> memo_active;
  mutable int memo_scope = -1;
  std::vector<char> bwd_overwrite;  // per node: grad slot overwritten by its only contributor (backward plan)
  int device = 0;
  cudaStream_t stream = nullptr;
  char* fwd_base = nullptr;
  size_t fwd_bytes = 0, fwd_cursor = 0;
  int64_t fwd_alloc_count = 0;
  char* bwd_base = nullptr;
  size_t bwd_bytes = 0, bwd_cursor = 0;
  int64_t bwd_alloc_count = 0;
  char* work_base = nullptr;
  size_t work_bytes = 0;
  std::vector<dg::Node> nodes;
  std::vector<int32_t> inputs;
  std::vector<int64_t> aux_i;
  std::vector<float> aux_f;
  int watermark = -1;
  int64_t forward_calls = 0;
  int64_t launches = 0;
  int64_t h2d_bytes = 0;
  int64_t d2h_bytes = 0;
  int64_t stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // live profiling: CUDA events around launches of the enabled op classes
  uint32_t prof_mask = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_pending[16];
  std::vector<int> prof_pending_cls;
  double prof_ms[16] = {0};
  double prof_flops[16] = {0};
  double prof_bytes[16] = {0};
  int64_t prof_count[16] = {0};
  std::vector<cudaEvent_t> event_pool;
  dg::Pinned pinned[2];
  int pin_idx = 0;
  // small-value cache: the last forward's target node (e.g. the loss) is
  // copied to pinned memory right after its forward launches, before any
  // backward kernels, so value(loss) waits for the forward only
  float* vcache = nullptr;
  cudaEvent_t vcache_ev = nullptr;
  int vcache_node = -1;
  int64_t vcache_n = 0;
  size_t blob_hint[2] = {1 << 20, 4 << 20};  // forward / backward table blob sizes seen
  bool has_grads = false;  // any backward in this generation
  bool counters_ready = false;  // split-K tile counters zeroed (first launch)
  // launch-plan cache (per graph object: plans embed its arena addresses and
  // stream): [0] forward plans, [1] backward plans, most recent first
  std::vector<std::shared_ptr<dg::CachedPlan>> pcache[2];
  mutable uint64_t memo_key = 0;   // structure hash of memo_sched
  uint64_t fwd_hist = 0;   // forward calls of this generation (placement history)
  std::vector<dg::LazyGrad> lazy;  // pending input-leaf gradients of the last backward
};

struct dg_trainer {
  dg::RuleArgs rule{};
  int sparse = 1;
  int64_t t = 0;
  struct Slot {
    int64_t handle;
    float* s0;
    float* s1;
  };
  std::vector<Slot> slots;
  void* segs_dev = nullptr;  // device TensorSeg table
  size_t segs_cap = 0;
  void* ids_dev = nullptr;   // device sorted ids for sparse rows
  size_t ids_cap = 0;
  dg::Pinned pinned;
};

namespace dg {

// ------------------------------------------------------------ pinned upload
static int pinned_acquire(Pinned& p, size_t n) {
  if (p.pending) {
    DG_CUDA_TRY(cudaEventSynchronize(p.ev));
    p.pending = false;
  }
  if (!p.ev) DG_CUDA_TRY(cudaEventCreateWithFlags(&p.ev, cudaEventDisableTiming));
  if (n > p.cap) {
    // growth (cudaHostAlloc synchronises the device): start at 4 MiB and
    // double, so a stream of slightly larger plans does not regrow every time
    if (p.ptr) DG_CUDA_TRY(cudaFreeHost(p.ptr));
    size_t cap = std::max<size_t>(p.cap ? 2 * p.cap : (4u << 20), 1 << 16);
    while (cap < n) cap *= 2;
    DG_CUDA_TRY(cudaHostAlloc(&p.ptr, cap, cudaHostAllocDefault));
    p.cap = cap;
  }
  return DG_OK;
}

// Process-wide ring of pinned staging buffers shared by every graph: a fresh
// graph must not pay cudaHostAlloc (slow, and it synchronises the device) on
// its first plan; a slot is reused once its previous upload has executed.
static Pinned& staging_slot() {
  static std::mutex mu;
  static Pinned ring[8];
  static int next = 0;
  static bool primed = false;
  std::lock_guard<std::mutex> lk(mu);
  if (!primed) {  // size every slot now: no allocation (device sync) on a later step
    primed = true;
    for (Pinned& q : ring) pinned_acquire(q, 4u << 20);
  }
  Pinned& p = ring[next];
  next = (next + 1) % 8;
  return p;
}

// plans build their table blob in place in the next staging slot
static int blob_attach(Blob& b, size_t hint) {
  Pinned& p = staging_slot();
  int rc = pinned_acquire(p, std::max<size_t>(hint, 1));
  if (rc) return rc;
  b.ext = static_cast<uint8_t*>(p.ptr);
  b.ext_cap = p.cap;
  b.slot = &p;
  return DG_OK;
}

static int upload(dg_graph* g, const Blob& blob, void* dst) {
  if (blob.empty()) return DG_OK;
  Pinned* p = blob.slot;
  if (!blob.ext) {  // spilled (or never attached): through a staging slot
    p = &staging_slot();
    int rc = pinned_acquire(*p, blob.size());
    if (rc) return rc;
    std::memcpy(p->ptr, blob.data(), blob.size());
  }
  DG_CUDA_TRY(cudaMemcpyAsync(dst, p->ptr, blob.size(), cudaMemcpyHostToDevice, g->stream));
  g->h2d_bytes += (int64_t)blob.size();
  DG_CUDA_TRY(cudaEventRecord(p->ev, g->stream));
  p->pending = true;
  return DG_OK;
}

// ----------------------------------------------------------- signatures
struct SigHash {
  uint64_t h = 1469598103934665603ull;
  void add(int64_t v) {  // one multiply-xorshift round per value
    h ^= static_cast<uint64_t>(v) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
  }
};


static int64_t param_handle_of(const dg_graph* g, int node) {
  const Node& n = g->nodes[node];
  if (n.kind != DG_OP_PARAMETER) return -1;
  return g->aux_i[n.ai_off];
}

// Signature of a unit: everything that must agree for one batched launch.
static uint64_t unit_signature(const dg_graph* g, const Unit& u) {
  SigHash s;
  if (u.type == U_RNN) {
    // stacks that become ready together share one persistent launch
    s.add(U_RNN);
    return s.h;
  }
  if (u.type == U_PNLS2) {  // widths and labels are per unit: one launch for all
    s.add(U_PNLS2);
    return s.h;
  }
  if (u.type == U_GRUA || u.type == U_GRUB) {
    s.add(u.type);
    s.add(u.H);
    s.add(u.gw);
    for (int k = 0; k < 3; ++k) s.add(u.off[k]);
    for (int x : u.ins) s.add(g->nodes[x].batch);
    return s.h;
  }
  if (u.type == U_CELL) {
    const Node& G = g->nodes[u.ins[0]];
    s.add(U_CELL);
    s.add(u.m);
    s.add(u.gw);
    s.add(u.H);
    s.add(G.batch);
    for (int k = 0; k < 3 + u.m; ++k) s.add(u.off[k]);
    for (int k = 1; k <= u.m; ++k) s.add(g->nodes[u.ins[k]].batch);
    return s.h;
  }
  const Node& n = g->nodes[u.last()];
  s.add(u.type);
  s.add(u.type == U_CHAIN ? -1 : n.kind);
  s.add(n.rank);
  for (int d = 0; d < n.rank; ++d) s.add(n.dims[d]);
  s.add(n.batch);
  s.add((int64_t)u.nodes.size());
  s.add((int64_t)u.ins.size());
  for (size_t k = 0; k < u.ins.size(); ++k) {
    const Node& in = g->nodes[u.ins[k]];
    s.add(in.batch);
    s.add(in.elem);
    s.add(in.rank);
    for (int d = 0; d < in.rank; ++d) s.add(in.dims[d]);
  }
  switch (n.kind) {
    case DG_OP_AFFINE: {
      // W operands must be the same parameter for a shared-weight GEMM; the
      // bias may be a shared parameter (epilogue) or a per-node value.
      for (size_t k = 0; k < u.ins.size(); ++k) {
        const int64_t h = param_handle_of(g, u.ins[k]);
        if (k == 0 || (k % 2) == 1) s.add(h);
        if ((k % 2) == 1 && (h < 0 || g->nodes[u.ins[k]].batch != 1)) s.add(1000000 + u.last());  // generic: singleton
      }
      break;
    }
    case DG_OP_SCALAR_MUL: {
      float f = g->aux_f[n.af_off];
      int32_t bits;
      std::memcpy(&bits, &f, 4);
      s.add(bits);
      break;
    }
    case DG_OP_PICK_RANGE:
      s.add(g->aux_i[n.ai_off]);
      s.add(g->aux_i[n.ai_off + 1]);
      break;
    default:
      break;
  }
  return s.h;
}

// ------------------------------------------------------------ cell matching
// Recognises the gated-cell pattern emitted by the reference builders:
//   LSTM step (builders.py:92-101):  h = o*tanh(f*c_prev + i*g)
//   Tree-LSTM compose (builders.py:250-274): h = o*tanh((i*g + f1*c1) + f2*c2),
//   leaves h = o*tanh(i*g)
// where i,f,o = logistic(pick_range(G, ...)), g = tanh(pick_range(G, ...)).
// Every internal node must be consumed exactly once (inside the cell); the
// cell state c and the output h may have any consumers.  Nodes keep their
// identity: the fused kernels write every node's value and gradient slot.
static bool match_cell(const dg_graph* g, int h, const std::vector<int>& consumers, const std::vector<char>& in_set,
                       const std::vector<char>& absorbed, Unit& u) {
  auto Nd = [&](int i) -> const Node& { return g->nodes[i]; };
  auto in = [&](int i, int k) { return g->inputs[Nd(i).in_off + k]; };
  const Node& hn = Nd(h);
  if (hn.kind != DG_OP_CMULT || hn.rank != 1 || !in_set[h] || absorbed[h]) return false;
  const int H = hn.dims[0], B = hn.batch;
  auto is_vec = [&](int i, int batch) {
    const Node& x = Nd(i);
    return x.rank == 1 && x.dims[0] == H && x.batch == batch;
  };
  auto inner = [&](int i) { return i >= 0 && in_set[i] && !absorbed[i] && consumers[i] == 1 && is_vec(i, B); };
  // gate: act = kind(pick_range(G, off, off+H)); returns pick, G and offset
  auto gate = [&](int act, int kind, int& pick, int& G, int& off) {
    if (!inner(act) || Nd(act).kind != kind) return false;
    const int p = in(act, 0);
    if (!inner(p) || Nd(p).kind != DG_OP_PICK_RANGE) return false;
    pick = p;
    G = in(p, 0);
    off = (int)g->aux_i[Nd(p).ai_off];
    return true;
  };
  int o_act = in(h, 0), tcn = in(h, 1);
  if (Nd(o_act).kind != DG_OP_LOGISTIC) std::swap(o_act, tcn);
  int p_o, G, off_o;
  if (!gate(o_act, DG_OP_LOGISTIC, p_o, G, off_o)) return false;
  const Node& Gn = Nd(G);
  if (Gn.rank != 1 || Gn.batch != B) return false;
  if (!inner(tcn) || Nd(tcn).kind != DG_OP_TANH) return false;
  const int c = in(tcn, 0);
  if (!in_set[c] || absorbed[c] || !is_vec(c, B)) return false;
  // left-deep sum c = ((t0 + t1) + t2) or a single product (at most 3 terms;
  // fixed arrays: this runs for every cmult of the graph)
  int adds_top_down[2], terms[3];
  int n_adds = 0, n_terms = 0;
  if (Nd(c).kind == DG_OP_CMULT) {
    terms[n_terms++] = c;
  } else if (Nd(c).kind == DG_OP_ADD) {
    int x = c, rev[3], n_rev = 0;
    for (;;) {
      if (n_adds == 2) return false;
      adds_top_down[n_adds++] = x;
      const int l = in(x, 0), r = in(x, 1);
      rev[n_rev++] = r;
      if (Nd(l).kind == DG_OP_ADD && inner(l)) {
        x = l;
        continue;
      }
      rev[n_rev++] = l;
      break;
    }
    for (int k = 0; k < n_rev; ++k) terms[k] = rev[n_rev - 1 - k];
    n_terms = n_rev;
  } else {
    return false;
  }
  const int m = n_terms - 1;
  if (m > 2) return false;
  int ig = -1, p_i = -1, p_g = -1, off_i = 0, off_g = 0;
  int fterm[2], fact[2], fpick[2], fext[2], foff[2], nf = 0;
  for (int t = 0; t < n_terms; ++t) {
    const int x = terms[t];
    if (Nd(x).kind != DG_OP_CMULT) return false;
    if (m == 0 ? (x != c) : !inner(x)) return false;
    const int a = in(x, 0), b = in(x, 1);
    int pa, Ga, oa, pb, Gb, ob;
    if (ig < 0 && gate(a, DG_OP_LOGISTIC, pa, Ga, oa) && gate(b, DG_OP_TANH, pb, Gb, ob) && Ga == G && Gb == G) {
      ig = t; p_i = pa; off_i = oa; p_g = pb; off_g = ob;
      continue;
    }
    if (ig < 0 && gate(b, DG_OP_LOGISTIC, pa, Ga, oa) && gate(a, DG_OP_TANH, pb, Gb, ob) && Ga == G && Gb == G) {
      ig = t; p_i = pa; off_i = oa; p_g = pb; off_g = ob;
      continue;
    }
    int fa = -1, ext = -1;
    if (gate(a, DG_OP_LOGISTIC, pa, Ga, oa) && Ga == G) { fa = a; ext = b; }
    else if (gate(b, DG_OP_LOGISTIC, pa, Ga, oa) && Ga == G) { fa = b; ext = a; }
    if (fa < 0 || nf == 2) return false;
    const Node& en = Nd(ext);
    if (en.rank != 1 || en.dims[0] != H || (en.batch != B && en.batch != 1)) return false;
    fterm[nf] = x;
    fact[nf] = fa;
    fpick[nf] = pa;
    fext[nf] = ext;
    foff[nf] = oa;
    ++nf;
  }
  if (ig < 0) return false;
  // the fused kernel sums i*g first: exact for two terms (commutative), and
  // for more terms only when the reference order already starts with i*g
  if (m >= 2 && ig != 0) return false;
  u = Unit();
  u.nodes.reserve(9 + 4 * m);
  u.ins.reserve(1 + m);
  u.type = U_CELL;
  u.m = m;
  u.H = H;
  u.gw = (int)Gn.elem;
  u.off[0] = off_i;
  u.off[1] = off_o;
  u.off[2] = off_g;
  for (int k = 0; k < m; ++k) u.off[3 + k] = foff[k];
  u.ins.push_back(G);
  for (int k = 0; k < m; ++k) u.ins.push_back(fext[k]);
  const int i_act = in(terms[ig], Nd(in(terms[ig], 0)).kind == DG_OP_LOGISTIC ? 0 : 1);
  const int g_act = in(terms[ig], Nd(in(terms[ig], 0)).kind == DG_OP_LOGISTIC ? 1 : 0);
  // picks i, f[m], o, g | acts i, f[m], o, g | prods ig, f[m] | adds[m] bottom-up | tanh(c) | h
  u.nodes.push_back(p_i);
  for (int k = 0; k < m; ++k) u.nodes.push_back(fpick[k]);
  u.nodes.push_back(p_o);
  u.nodes.push_back(p_g);
  u.nodes.push_back(i_act);
  for (int k = 0; k < m; ++k) u.nodes.push_back(fact[k]);
  u.nodes.push_back(o_act);
  u.nodes.push_back(g_act);
  u.nodes.push_back(terms[ig]);
  for (int k = 0; k < m; ++k) u.nodes.push_back(fterm[k]);
  for (int k = n_adds - 1; k >= 0; --k) u.nodes.push_back(adds_top_down[k]);
  u.nodes.push_back(tcn);
  u.nodes.push_back(h);
  // distinct internal nodes, none of them an external input
  int all[32];
  const int na = (int)u.nodes.size();
  if (na > 32) return false;
  std::copy(u.nodes.begin(), u.nodes.end(), all);
  std::sort(all, all + na);
  if (std::adjacent_find(all, all + na) != all + na) return false;
  for (int x : u.ins)
    if (std::binary_search(all, all + na, x)) return false;
  if ((int)u.nodes.size() != 9 + 4 * m) return false;  // + G and m external states = nslot
  return true;
}

// GRU step (builders.py:102-110), matched from its output nh = add(kh, zc):
//   zr = affine(b, Wx, x, Wh, h); z = logistic(pick(zr, z)); r = logistic(pick(zr, r))
//   cx = pick(affine(b, Wx, x), c); rh = cmult(r, h); mh = matmul(Wh, rh); ch = pick(mh, c)
//   cand = tanh(add(cx, ch)); keep = add(input(ones), scalar_mul(z, -1))
//   nh = add(cmult(keep, h), cmult(z, cand))
// as two units around the matmul (kernels.cuh GruArgs slot order).  Every
// internal node has exactly one consumer; z (two consumers, both in part B),
// cx and rh are part A's outputs.
static bool match_gru(const dg_graph* g, int nh, const std::vector<int>& consumers, const std::vector<char>& in_set,
                      const std::vector<char>& absorbed, Unit& ua, Unit& ub) {
  auto Nd = [&](int i) -> const Node& { return g->nodes[i]; };
  auto in = [&](int i, int k) { return g->inputs[Nd(i).in_off + k]; };
  const Node& hn = Nd(nh);
  if (hn.kind != DG_OP_ADD || hn.rank != 1 || !in_set[nh] || absorbed[nh]) return false;
  const int H = hn.dims[0], B = hn.batch;
  auto vec = [&](int i, bool b1_ok) {
    const Node& x = Nd(i);
    return x.rank == 1 && x.dims[0] == H && (x.batch == B || (b1_ok && x.batch == 1));
  };
  auto inner = [&](int i, int kind) {
    return i >= 0 && in_set[i] && !absorbed[i] && consumers[i] == 1 && Nd(i).kind == kind && vec(i, false);
  };
  auto pick = [&](int p, int& src, int& off) {
    if (!inner(p, DG_OP_PICK_RANGE)) return false;
    src = in(p, 0);
    off = (int)g->aux_i[Nd(p).ai_off];
    return Nd(src).rank == 1 && Nd(src).batch == B && Nd(src).dims[0] == 3 * H;
  };
  const int kh = in(nh, 0), zc = in(nh, 1);
  if (!inner(kh, DG_OP_CMULT) || !inner(zc, DG_OP_CMULT)) return false;
  const int keep = in(kh, 0), h = in(kh, 1), z = in(zc, 0), cand = in(zc, 1);
  if (!inner(keep, DG_OP_ADD) || !vec(h, true) || !inner(cand, DG_OP_TANH)) return false;
  if (!in_set[z] || absorbed[z] || consumers[z] != 2 || Nd(z).kind != DG_OP_LOGISTIC || !vec(z, false)) return false;
  const int ones = in(keep, 0), nz = in(keep, 1);
  if (Nd(ones).kind != DG_OP_INPUT || !vec(ones, true) || !inner(nz, DG_OP_SCALAR_MUL) || in(nz, 0) != z ||
      g->aux_f[Nd(nz).af_off] != -1.f)
    return false;
  const int sv = in(cand, 0);
  if (!inner(sv, DG_OP_ADD)) return false;
  const int cx = in(sv, 0), ch = in(sv, 1);
  int ax, off_c, mh, off_ch;
  if (!pick(cx, ax, off_c) || !pick(ch, mh, off_ch)) return false;
  if (Nd(mh).kind != DG_OP_MATMUL || consumers[mh] != 1 || !in_set[mh] || absorbed[mh]) return false;
  const int rh = in(mh, 1);
  if (!inner(rh, DG_OP_CMULT) || in(rh, 1) != h) return false;
  const int r = in(rh, 0);
  if (!inner(r, DG_OP_LOGISTIC)) return false;
  int zr, off_r, zr2, off_z;
  if (!pick(in(r, 0), zr, off_r) || !pick(in(z, 0), zr2, off_z) || zr != zr2) return false;
  if (Nd(zr).kind != DG_OP_AFFINE || Nd(ax).kind != DG_OP_AFFINE || !in_set[zr] || !in_set[ax]) return false;
  ua = Unit();
  ua.type = U_GRUA;
  ua.m = -1;
  ua.H = H;
  ua.gw = 3 * H;
  ua.off[0] = off_z;
  ua.off[1] = off_r;
  ua.off[2] = off_c;
  ua.ins = {zr, ax, h};
  ua.nodes = {in(z, 0), z, in(r, 0), r, cx, rh};
  ub = Unit();
  ub.type = U_GRUB;
  ub.m = -1;
  ub.H = H;
  ub.gw = 3 * H;
  ub.off[0] = off_ch;
  ub.ins = {mh, cx, z, ones, h};
  ub.nodes = {ch, sv, cand, nz, keep, kh, zc, nh};
  // distinct nodes, no external input inside
  std::vector<int> all(ua.nodes);
  all.insert(all.end(), ub.nodes.begin(), ub.nodes.end());
  std::sort(all.begin(), all.end());
  if (std::adjacent_find(all.begin(), all.end()) != all.end()) return false;
  for (int x : {zr, ax, h, mh, ones})
    if (std::binary_search(all.begin(), all.end(), x)) return false;
  return true;
}

// ------------------------------------------------------------- LSTM chains
// Device limits the planner sizes persistent launches against (sm_100a B200:
// 148 SMs, 227 KB opt-in shared memory per CTA).  Fixed constants so the plan
// is the same with or without a device (host-only planner tests).
static constexpr int kSmCount = 148;
static constexpr size_t kSmemMax = 227 * 1024 - 1024;  // dynamic (static step tables aside)
static constexpr int kFlagInts = 65536;  // arrival counters (rnn.cu), end of the counter region
static constexpr bool kStackChains = false;

// CJ (dG columns staged per chunk) for a backward launch: the largest multiple
// of 32 (<= max gw) that fits next to the resident W^T slices.
static int rnn_pick_cj(int gw, int gw_c, int bs) {
  int cj = std::max(gw, gw_c);
  cj = (cj + 31) & ~31;
  while (cj > 32 && rnn_bwd_smem(gw, gw_c, bs, cj) > kSmemMax) cj -= 32;
  return cj;
}

// Groups matched LSTM cells (m = 1) into chains and stacks:
//   step t+1 of a chain: gates = affine(b, Wx, x, Wh, h_t) with the same three
//   parameters, c_prev = c_t, and G consumed only by the cell's 4 picks;
//   chain b is stacked on chain a when x^b_t = h^a_t for every t.
// A stack becomes one U_RNN unit when its external inputs do not depend on it
// and its persistent launches fit the device (CTAs <= SMs, shared memory).
// Returns per cell index the stack id (or -1).
static std::vector<int> find_rnn_stacks(const dg_graph* g, const std::vector<Unit>& cells,
                                        const std::vector<int>& consumers, const std::vector<char>& in_set,
                                        const std::vector<int>& active, std::vector<RnnStack>& stacks) {
  const int nc = (int)cells.size();
  std::vector<int> stack_of(nc, -1);
  if (nc < 2 || !rnn_enabled()) return stack_of;
  auto Nd = [&](int i) -> const Node& { return g->nodes[i]; };
  auto in = [&](int i, int k) { return g->inputs[Nd(i).in_off + k]; };
  const int N = (int)g->nodes.size();
  // eligibility + per-cell descriptors
  struct CellInfo {
    bool ok = false;
    int G = -1, x = -1, hp = -1, cp = -1, h = -1, c = -1, B = 0, H = 0, K = 0;
    int64_t hb = -1, hWx = -1, hWh = -1;
  };
  std::vector<CellInfo> ci(nc);
  std::unordered_map<int, int> cell_by_h;
  for (int k = 0; k < nc; ++k) {
    const Unit& u = cells[k];
    CellInfo& c = ci[k];
    if (u.m != 1 || u.nodes.size() != 13) continue;
    const int G = u.ins[0];
    const Node& Gn = Nd(G);
    if (Gn.kind != DG_OP_AFFINE || Gn.n_in != 5 || !in_set[G] || consumers[G] != 4) continue;
    const int pb = in(G, 0), pwx = in(G, 1), pwh = in(G, 3);
    bool params = true;
    for (int p : {pb, pwx, pwh})
      params = params && Nd(p).kind == DG_OP_PARAMETER && Nd(p).batch == 1;
    if (!params) continue;
    c.G = G;
    c.x = in(G, 2);
    c.hp = in(G, 4);
    c.cp = u.ins[1];
    c.h = u.nodes[12];
    c.c = u.nodes[10];
    c.B = Gn.batch;
    c.H = u.H;
    c.K = (int)Nd(c.x).elem;
    if ((int)Gn.elem != u.gw || Nd(c.hp).elem != c.H || Nd(c.x).rank != 1 || Nd(c.hp).rank != 1) continue;
    auto bok = [&](int i) { return Nd(i).batch == 1 || Nd(i).batch == c.B; };
    if (!bok(c.x) || !bok(c.hp) || !bok(c.cp)) continue;
    c.hb = param_handle_of(g, pb);
    c.hWx = param_handle_of(g, pwx);
    c.hWh = param_handle_of(g, pwh);
    c.ok = true;
    cell_by_h[c.h] = k;
  }
  auto same_sig = [&](int a, int b) {
    const Unit &ua = cells[a], &ub = cells[b];
    const CellInfo &x = ci[a], &y = ci[b];
    return x.hb == y.hb && x.hWx == y.hWx && x.hWh == y.hWh && x.B == y.B && x.H == y.H && x.K == y.K &&
           ua.gw == ub.gw && std::equal(ua.off, ua.off + 4, ub.off);
  };
  // recurrent links p -> k (unique successor)
  std::vector<int> pred(nc, -1), succ(nc, -1), nsucc(nc, 0);
  for (int k = 0; k < nc; ++k) {
    if (!ci[k].ok) continue;
    auto it = cell_by_h.find(ci[k].hp);
    if (it == cell_by_h.end()) continue;
    const int p = it->second;
    if (p == k || !ci[p].ok || ci[p].c != ci[k].cp || !same_sig(p, k)) continue;
    pred[k] = p;
    nsucc[p]++;
  }
  for (int k = 0; k < nc; ++k) {
    if (pred[k] < 0) continue;
    if (nsucc[pred[k]] != 1) {
      pred[k] = -1;
      continue;
    }
    succ[pred[k]] = k;
  }
  // chains (T >= 2), in order of their first cell
  std::vector<std::vector<int>> chains;
  std::vector<int> chain_of(nc, -1), step_of(nc, -1);
  for (int k = 0; k < nc; ++k) {
    if (!ci[k].ok || pred[k] >= 0 || succ[k] < 0) continue;
    std::vector<int> ch;
    for (int x = k; x >= 0; x = succ[x]) ch.push_back(x);
    for (size_t t = 0; t < ch.size(); ++t) {
      chain_of[ch[t]] = (int)chains.size();
      step_of[ch[t]] = (int)t;
    }
    chains.push_back(std::move(ch));
  }
  if (chains.empty()) return stack_of;
  // stacking (x^b_t == h^a_t for all t, one wavefront launch) is off: each
  // chain's input projection b + Wx x_t is one batched tensor-core GEMM over
  // all steps before its recurrence, so the layers run one after the other
  // and the recurrent kernels keep only Wh resident
  const int nch = (int)chains.size();
  std::vector<int> src(nch, -1), cons(nch, -1);
  for (int b = 0; b < nch && kStackChains; ++b) {
    const auto& cb = chains[b];
    auto it = cell_by_h.find(ci[cb[0]].x);
    if (it == cell_by_h.end()) continue;
    const int a = chain_of[it->second];
    if (a < 0 || a == b || step_of[it->second] != 0 || chains[a].size() != cb.size() || cons[a] >= 0) continue;
    if (ci[chains[a][0]].B != ci[cb[0]].B) continue;
    bool all = true;
    for (size_t t = 0; t < cb.size() && all; ++t) all = ci[cb[t]].x == ci[chains[a][t]].h;
    if (!all) continue;
    src[b] = a;
    cons[a] = b;
  }
  // stacks: walk from each bottom chain (no src) up through consumers.
  // mark / seen are stamped per stack (no O(N) clears per chain)
  std::vector<int> mark(N, -1), seen(N, -1), dfs;
  for (int bot = 0; bot < nch; ++bot) {
    if (src[bot] >= 0) continue;
    std::vector<int> order;
    for (int x = bot; x >= 0; x = cons[x]) order.push_back(x);
    // the stack's nodes and external inputs
    int lo = N;
    std::vector<int> ext;
    for (size_t li = 0; li < order.size(); ++li) {
      for (int k : chains[order[li]]) {
        mark[ci[k].G] = bot;
        lo = std::min(lo, ci[k].G);
        for (int x : cells[k].nodes) {
          mark[x] = bot;
          lo = std::min(lo, x);
        }
      }
      const auto& ch = chains[order[li]];
      ext.push_back(ci[ch[0]].hp);
      ext.push_back(ci[ch[0]].cp);
      if (li == 0)
        for (int k : ch) ext.push_back(ci[k].x);
    }
    // acyclic: no external input may depend on a node of the stack.  Inputs
    // precede their consumers, so only ancestors with index > lo can be
    // stack nodes: a backward walk bounded below by lo.
    bool cyclic = false;
    for (int x : ext) {
      if (cyclic) break;
      if (x < lo) continue;
      dfs.clear();
      dfs.push_back(x);
      while (!dfs.empty() && !cyclic) {
        const int i = dfs.back();
        dfs.pop_back();
        if (seen[i] == bot) continue;
        seen[i] = bot;
        if (mark[i] == bot) {
          cyclic = true;
          break;
        }
        const Node& n = Nd(i);
        for (int q = 0; q < n.n_in; ++q) {
          const int s2 = g->inputs[n.in_off + q];
          if (s2 >= lo && seen[s2] != bot) dfs.push_back(s2);
        }
      }
    }
    if (cyclic) continue;
    // geometry and device fit
    RnnStack st;
    const CellInfo& c0 = ci[chains[order[0]][0]];
    st.bs = rnn_rows_per_cta(c0.B);
    int ctas = 0;
    bool fits = true;
    for (size_t li = 0; li < order.size(); ++li) {
      const auto& ch = chains[order[li]];
      const CellInfo& cc = ci[ch[0]];
      RnnChainPlan cp;
      for (size_t t = 0; t < ch.size(); ++t) {
        cp.cells.push_back(cells[ch[t]]);
        cp.G.push_back(ci[ch[t]].G);
      }
      cp.hb = cc.hb;
      cp.hWx = cc.hWx;
      cp.hWh = cc.hWh;
      cp.H = cc.H;
      cp.K_in = cc.K;
      cp.B = cc.B;
      cp.gw = cells[ch[0]].gw;
      const Unit& u0 = cells[ch[0]];
      cp.off[0] = u0.off[0];  // i
      cp.off[1] = u0.off[3];  // f
      cp.off[2] = u0.off[1];  // o
      cp.off[3] = u0.off[2];  // g
      cp.src = li > 0 ? (int)li - 1 : -1;
      cp.cons = li + 1 < order.size() ? (int)li + 1 : -1;
      cp.n_s = (cp.B + st.bs - 1) / st.bs;
      cp.n_u = (cp.H + kRnnUnits - 1) / kRnnUnits;
      ctas += cp.n_s * cp.n_u;
      if (rnn_fwd_smem(cp.H, st.bs) > kSmemMax) fits = false;
      st.chains.push_back(std::move(cp));
    }
    for (auto& cp : st.chains) {
      const int gwc = cp.cons >= 0 ? st.chains[cp.cons].gw : 0;
      if (rnn_bwd_smem(cp.gw, gwc, st.bs, rnn_pick_cj(cp.gw, gwc, st.bs)) > kSmemMax) fits = false;
    }
    st.ctas = ctas;
    if (!fits || ctas > kSmCount || (int)st.chains.size() > kRnnMaxChains) continue;
    int flags = 0;
    for (auto& cp : st.chains) flags += cp.n_s * (int)cp.cells.size();
    if (flags > kFlagInts) continue;
    const int sid = (int)stacks.size();
    for (int li : order)
      for (int k : chains[li]) stack_of[k] = sid;
    stacks.push_back(std::move(st));
  }
  return stack_of;
}

// ------------------------------------------------------------- scheduling
// Builds units (with cell fusion and add-chain rewrite) and the group order
// for the node set `active` (ascending).  scope_hi bounds the consumer-count
// scope.
// host-side planning timers (DG_PLAN_TIMING=1 prints per call to stderr)
struct PlanTimer {
  bool on;
  std::chrono::steady_clock::time_point t0;
  const char* what;
  std::string acc;
  explicit PlanTimer(const char* w) : what(w) {
    const char* e = std::getenv("DG_PLAN_TIMING");
    on = e && e[0] == '1';
    t0 = std::chrono::steady_clock::now();
  }
  void lap(const char* name) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    char buf[64];
    std::snprintf(buf, sizeof buf, " %s %.0fus", name, std::chrono::duration<double, std::micro>(t - t0).count());
    acc += buf;
    t0 = t;
  }
  ~PlanTimer() {
    if (on) std::fprintf(stderr, "[plan] %s:%s\n", what, acc.c_str());
  }
};

static void build_schedule(const dg_graph* g, const std::vector<int>& active, int scope_hi, Schedule& S) {
  PlanTimer tm("build_schedule");
  const int N = (int)g->nodes.size();
  S = Schedule();
  S.unit_of.assign(N, -1);
  std::vector<char> in_set(N, 0);
  for (int i : active) in_set[i] = 1;

  // consumer counts over all nodes <= scope_hi (backward correctness needs the
  // full scope; see header comment)
  std::vector<int> consumers(N, 0);
  for (int i = 0; i <= scope_hi && i < N; ++i) {
    const Node& n = g->nodes[i];
    for (int k = 0; k < n.n_in; ++k) consumers[g->inputs[n.in_off + k]]++;
  }
  auto same_shape = [&](int a, int b) {
    const Node& x = g->nodes[a];
    const Node& y = g->nodes[b];
    if (x.batch != y.batch || x.rank != y.rank) return false;
    for (int d = 0; d < x.rank; ++d)
      if (x.dims[d] != y.dims[d]) return false;
    return true;
  };
  tm.lap("consumers");
  // gated cells first (they own their internal add chains)
  std::vector<char> absorbed(N, 0);
  std::vector<Unit> cells;
  std::vector<int> cell_of(N, -1);
  for (int i : active) {
    if (g->nodes[i].kind != DG_OP_CMULT) continue;
    Unit cu;
    if (match_cell(g, i, consumers, in_set, absorbed, cu)) {
      for (int x : cu.nodes) {
        absorbed[x] = 1;
        cell_of[x] = (int)cells.size();
      }
      cells.push_back(std::move(cu));
    }
  }
  // GRU steps: two units each (part A before the recurrent matmul, part B after)
  {
    static const bool gru_on = [] {
      const char* e = std::getenv("DG_GRU_FUSE");
      return !(e && e[0] == '0');
    }();
    for (int i : active) {
      if (!gru_on || g->nodes[i].kind != DG_OP_ADD || absorbed[i]) continue;
      Unit ua, ub;
      if (!match_gru(g, i, consumers, in_set, absorbed, ua, ub)) continue;
      for (Unit* pu : {&ua, &ub}) {
        for (int x : pu->nodes) {
          absorbed[x] = 1;
          cell_of[x] = (int)cells.size();
        }
        cells.push_back(std::move(*pu));
      }
    }
  }
  // class-factored softmax terms: add(pnls(class scores), pnls(word scores))
  {
    static const bool on = [] {
      const char* e = std::getenv("DG_PNLS2");
      return !(e && e[0] == '0');
    }();
    auto Nd = [&](int i) -> const Node& { return g->nodes[i]; };
    auto in = [&](int i, int k) { return g->inputs[Nd(i).in_off + k]; };
    auto term = [&](int p) {
      return p >= 0 && in_set[p] && !absorbed[p] && consumers[p] == 1 && Nd(p).kind == DG_OP_PNLS &&
             Nd(p).batch == 1 && Nd(in(p, 0)).rank == 1 && Nd(in(p, 0)).batch == 1;
    };
    for (int i : active) {
      if (!on || Nd(i).kind != DG_OP_ADD || absorbed[i] || Nd(i).batch != 1) continue;
      const int p1 = in(i, 0), p2 = in(i, 1);
      if (p1 == p2 || !term(p1) || !term(p2)) continue;
      Unit u;
      u.type = U_PNLS2;
      u.m = -1;
      u.ins = {in(p1, 0), in(p2, 0)};
      u.nodes = {p1, p2, i};
      for (int x : u.nodes) {
        absorbed[x] = 1;
        cell_of[x] = (int)cells.size();
      }
      cells.push_back(std::move(u));
    }
  }
  tm.lap("cells");
  // LSTM chains / stacks over the matched cells (persistent recurrence path)
  std::vector<int> rnn_of(N, -1);
  {
    std::vector<int> stack_of = find_rnn_stacks(g, cells, consumers, in_set, active, S.rnns);
    for (size_t k = 0; k < cells.size(); ++k) {
      if (stack_of[k] < 0) continue;
      for (int x : cells[k].nodes) rnn_of[x] = stack_of[k];
      rnn_of[cells[k].ins[0]] = stack_of[k];
    }
  }
  tm.lap("rnn");
  std::vector<char> rnn_made(S.rnns.size(), 0);
  auto chainable_add = [&](int i) {
    const Node& n = g->nodes[i];
    if (n.kind != DG_OP_ADD || absorbed[i] || rnn_of[i] >= 0) return false;
    const int a = g->inputs[n.in_off], b = g->inputs[n.in_off + 1];
    return same_shape(i, a) && same_shape(i, b);
  };

  // units
  std::vector<int> chain_next(N, -1);  // add node -> the add that extends it
  for (int i : active) {
    if (!chainable_add(i)) continue;
    const int p = g->inputs[g->nodes[i].in_off];
    if (p >= 0 && in_set[p] && chainable_add(p) && consumers[p] == 1 && chain_next[p] < 0) chain_next[p] = i;
  }
  std::vector<char> has_prev(N, 0);
  for (int i : active)
    if (chain_next[i] >= 0) has_prev[chain_next[i]] = 1;

  for (int i : active) {
    const Node& n = g->nodes[i];
    if (S.unit_of[i] >= 0) continue;
    if (n.kind == DG_OP_INPUT) { S.input_nodes.push_back(i); continue; }
    if (n.kind == DG_OP_PARAMETER) { S.param_nodes.push_back(i); continue; }
    if (n.kind == DG_OP_LOOKUP || n.kind == DG_OP_LOOKUP_BATCH) { S.lookup_nodes.push_back(i); continue; }
    Unit u;
    if (rnn_of[i] >= 0) {
      const int sid = rnn_of[i];
      if (rnn_made[sid]) continue;
      rnn_made[sid] = 1;
      u.type = U_RNN;
      u.rnn = sid;
      // slot-major node order: each slot's nodes of all steps are placed
      // contiguously (h_0..h_{T-1} form one dense [T*B x H] block, which the
      // layers above read as a regular GEMM operand)
      for (const RnnChainPlan& cp : S.rnns[sid].chains) {
        const size_t T = cp.G.size();
        for (size_t t = 0; t < T; ++t) {
          const Node& G = g->nodes[cp.G[t]];
          u.nodes.push_back(cp.G[t]);
          for (int k = 0; k < G.n_in; ++k) u.ins.push_back(g->inputs[G.in_off + k]);
          u.ins.push_back(cp.cells[t].ins[1]);
        }
        for (int k = 0; k < 13; ++k)
          for (size_t t = 0; t < T; ++t) u.nodes.push_back(cp.cells[t].nodes[k]);
      }
    } else if (cell_of[i] >= 0) {
      u = std::move(cells[cell_of[i]]);
    } else if (chainable_add(i) && !has_prev[i] && chain_next[i] >= 0) {
      u.type = U_CHAIN;
      int c = i;
      u.ins.push_back(g->inputs[n.in_off]);
      u.ins.push_back(g->inputs[n.in_off + 1]);
      u.nodes.push_back(c);
      while (chain_next[c] >= 0) {
        c = chain_next[c];
        u.nodes.push_back(c);
        u.ins.push_back(g->inputs[g->nodes[c].in_off + 1]);
      }
    } else {
      u.type = U_NODE;
      u.nodes.push_back(i);
      for (int k = 0; k < n.n_in; ++k) u.ins.push_back(g->inputs[n.in_off + k]);
    }
    const int id = (int)S.units.size();
    for (int x : u.nodes) S.unit_of[x] = id;
    S.units.push_back(std::move(u));
  }

  tm.lap("units");
  const int U = (int)S.units.size();
  if (U == 0) return;
  // unit dependency graph
  std::vector<std::vector<int>> succ(U);
  std::vector<int> indeg(U, 0);
  for (int u = 0; u < U; ++u) {
    std::vector<int> preds;
    for (int x : S.units[u].ins) {
      const int pu = x >= 0 && x < N ? S.unit_of[x] : -1;
      if (pu >= 0 && pu != u) preds.push_back(pu);
    }
    std::sort(preds.begin(), preds.end());
    preds.erase(std::unique(preds.begin(), preds.end()), preds.end());
    indeg[u] = (int)preds.size();
    for (int p : preds) succ[p].push_back(u);
  }
  // heights over a real topological order (a chain or cell unit is created at
  // its first node, but later terms of a loss chain are built after it)
  std::vector<int> topo;
  topo.reserve(U);
  {
    std::vector<int> deg = indeg;
    for (int u = 0; u < U; ++u)
      if (deg[u] == 0) topo.push_back(u);
    for (size_t q = 0; q < topo.size(); ++q)
      for (int c : succ[topo[q]])
        if (--deg[c] == 0) topo.push_back(c);
  }
  std::vector<int> height(U, 0);
  for (int q = (int)topo.size() - 1; q >= 0; --q) {
    const int u = topo[q];
    for (int c : succ[u]) height[u] = std::max(height[u], height[c] + 1);
  }
  int L = 0;
  for (int u = 0; u < U; ++u) L = std::max(L, height[u]);
  std::vector<int> alap(U);
  for (int u = 0; u < U; ++u) alap[u] = L - height[u];
  std::vector<uint64_t> sig(U);
  for (int u = 0; u < U; ++u) sig[u] = unit_signature(g, S.units[u]);

  tm.lap("deps+sig");
  // list scheduling
  std::unordered_map<uint64_t, std::vector<int>> ready;
  std::vector<uint64_t> ready_keys;  // insertion-ordered keys for determinism
  auto add_ready = [&](int u) {
    auto it = ready.find(sig[u]);
    if (it == ready.end()) {
      ready.emplace(sig[u], std::vector<int>{u});
      ready_keys.push_back(sig[u]);
    } else {
      it->second.push_back(u);
    }
  };
  for (int u = 0; u < U; ++u)
    if (indeg[u] == 0) add_ready(u);
  int done = 0, level = 0;
  std::vector<int> newly;
  while (done < U) {
    // urgent signatures at this level
    std::vector<std::pair<int, uint64_t>> urgent;  // (min unit id, key)
    int min_alap = 1 << 30;
    for (uint64_t k : ready_keys) {
      const auto& v = ready[k];
      int ma = 1 << 30, mu = 1 << 30;
      for (int u : v) {
        ma = std::min(ma, alap[u]);
        mu = std::min(mu, u);
      }
      min_alap = std::min(min_alap, ma);
      if (ma <= level) urgent.push_back({mu, k});
    }
    if (urgent.empty()) {
      level = std::max(level + 1, min_alap);
      continue;
    }
    std::sort(urgent.begin(), urgent.end());
    newly.clear();
    for (auto& uk : urgent) {
      std::vector<int> members = std::move(ready[uk.second]);
      ready.erase(uk.second);
      ready_keys.erase(std::find(ready_keys.begin(), ready_keys.end(), uk.second));
      std::sort(members.begin(), members.end());
      Group gr;
      const Unit& u0 = S.units[members[0]];
      gr.kind = u0.type == U_CHAIN ? -1 : u0.type == U_CELL ? -2 : u0.type == U_RNN ? -3
              : u0.type == U_GRUA ? -4 : u0.type == U_GRUB ? -5 : u0.type == U_PNLS2 ? -6
              : g->nodes[u0.last()].kind;
      gr.units = members;
      for (int u : members) {
        ++done;
        for (int c : succ[u])
          if (--indeg[c] == 0) newly.push_back(c);
      }
      gr.level = level;
      S.groups.push_back(std::move(gr));
    }
    for (int c : newly) add_ready(c);
    ++level;
  }
  tm.lap("list");
}

// Schedules depend only on the graph's structure (kinds, wiring, shapes,
// parameter identities, structural aux such as pick offsets) -- not on lookup
// ids, labels or input payloads -- so they are cached by a structural hash:
// minibatches of equal padded length reuse one schedule.
static uint64_t structure_hash(const dg_graph* g, const std::vector<int>& active, int scope_hi) {
  SigHash h;
  h.add(scope_hi);
  h.add((int64_t)active.size());
  for (int i : active) h.add(i);
  for (int i = 0; i <= scope_hi; ++i) {
    const Node& n = g->nodes[i];
    h.add(n.kind);
    h.add(n.batch);
    h.add(n.rank);
    for (int d = 0; d < n.rank; ++d) h.add(n.dims[d]);
    h.add(n.n_in);
    for (int k = 0; k < n.n_in; ++k) h.add(i - g->inputs[n.in_off + k]);
    switch (n.kind) {
      case DG_OP_PARAMETER:
      case DG_OP_LOOKUP:
      case DG_OP_LOOKUP_BATCH:
        h.add(g->aux_i[n.ai_off]);  // table / parameter identity (not the ids)
        break;
      case DG_OP_PICK_RANGE:
        for (int64_t q = 0; q < n.ai_len; ++q) h.add(g->aux_i[n.ai_off + q]);
        break;
      case DG_OP_SCALAR_MUL: {
        int32_t bits;
        std::memcpy(&bits, &g->aux_f[n.af_off], 4);
        h.add(bits);
        break;
      }
      default:
        break;
    }
  }
  return h.h;
}

static std::shared_ptr<const Schedule> get_schedule(const dg_graph* g, const std::vector<int>& active, int scope_hi) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, std::shared_ptr<const Schedule>> cache;
  static const bool on = [] {
    const char* e = std::getenv("DG_SCHED_CACHE");
    return !(e && e[0] == '0');
  }();
  if (g->memo_sched && g->memo_scope == scope_hi && g->memo_active == active) return g->memo_sched;
  const uint64_t key = structure_hash(g, active, scope_hi);
  g->memo_key = key;
  if (on) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      g->memo_sched = it->second;
      g->memo_active = active;
      g->memo_scope = scope_hi;
      return it->second;
    }
  }
  auto S = std::make_shared<Schedule>();
  build_schedule(g, active, scope_hi, *S);
  if (on) {
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() >= 256) cache.clear();
    cache.emplace(key, S);
  }
  g->memo_sched = S;
  g->memo_active = active;
  g->memo_scope = scope_hi;
  return S;
}

// ----------------------------------------------------------------- planning
// A plan = host-built table blob + deferred launch closures that read the
// blob's device base.
enum OpClass {
  C_GEMM_FWD = 0, C_GEMM_DX = 1, C_GEMM_DW = 2, C_PNLS_FWD = 3, C_PNLS_BWD = 4,
  C_ELEMWISE = 5, C_GATHER = 6, C_SCATTER = 7, C_COLSUM = 8, C_OTHER = 9, C_RNN_FWD = 10,
  C_RNN_BWD = 11, C_NCLASS = 12
};

struct OpMeta {
  int cls = C_OTHER;
  double flops = 0, bytes = 0;  // algorithmic work of the launch
};

struct Plan {
  Blob blob;
  std::vector<std::function<int(char*)>> ops;  // arg: device blob base
  int rnn_bwd_ctas = 0;   // CTAs of the last backward cluster recurrence planned
  size_t rnn_bwd_op = 0;  // ops.size() right after it (early dW only directly behind it)
  std::vector<LazyGrad> lazy;
  size_t lazy_floats = 0;  // used part of the lazy-partials region
  std::vector<OpMeta> meta;
  size_t scratch_need = 0;
  void tag(int cls, double flops, double bytes) {
    meta.resize(ops.size());
    meta.back() = OpMeta{cls, flops, bytes};
  }
};

// The data-dependent part of a plan's table blob: input payloads, lookup
// ids and pickneglogsoftmax labels.  Everything else in a plan (schedule,
// placement, row-pointer tables, launch configurations, TMA descriptors) is
// a function of the graph's structure hash, the arena cursors and the
// parameter storage, so a plan built once is replayed for every later graph
// of the same structure with only these entries rewritten.
struct PatchRec {
  struct Payload {
    int node;
    size_t off, bytes;
  };
  struct Ids {
    int node, q0, width;  // aux_i[ai_off + q0 .. ai_off + ai_len) as int64 (8) or int32 (4)
    size_t off;
  };
  std::vector<Payload> payload;
  std::vector<Ids> ids;
};
static thread_local PatchRec* g_rec = nullptr;  // recorder of the plan being built
// stream the launch closures issue into: the graph's stream, or the private
// capture stream while a cached plan is recorded into a CUDA graph
static thread_local cudaStream_t g_launch_stream = nullptr;

struct RecScope {
  explicit RecScope(PatchRec* r) { g_rec = r; }
  ~RecScope() { g_rec = nullptr; }
};

static void rec_payload(int node, size_t off, size_t bytes) {
  if (g_rec) g_rec->payload.push_back({node, off, bytes});
}
static void rec_ids(int node, int q0, int width, size_t off) {
  if (g_rec) g_rec->ids.push_back({node, q0, width, off});
}

struct CachedPlan {
  uint64_t key = 0;
  std::vector<uint8_t> tmpl;  // blob bytes of the static part
  std::vector<std::function<int(char*)>> ops;
  std::vector<OpMeta> meta;
  PatchRec patch;
  std::vector<LazyGrad> lazy;
  int64_t kernel_launches = 0;  // launches issued by `ops` (counted at build)
  cudaGraphExec_t exec = nullptr;
  int replays = 0;
  ~CachedPlan() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

template <class T>
static inline T* at(char* base, size_t off) {
  return reinterpret_cast<T*>(base + off);
}

static bool all_aligned16(const std::vector<uintptr_t>& v) {
  for (uintptr_t p : v)
    if (p & 15) return false;
  return true;
}

// pointers helpers
static inline uintptr_t P(const float* p) { return reinterpret_cast<uintptr_t>(p); }

// rounds: split a group's (node j, slot) targets so that no round writes the
// same target from two different nodes (same-node duplicates are handled by
// one thread in the elementwise kernels).  Returns per-round masks.
static std::vector<std::vector<char>> conflict_rounds(const std::vector<std::vector<int>>& targets,
                                                      bool same_node_ok) {
  // targets[j] = target node ids for node j (one per slot)
  const size_t n = targets.size();
  std::vector<std::vector<char>> rounds;
  std::vector<int> round_of(n, -1);
  std::vector<std::unordered_map<int, int>> owner;  // per round: target -> node j
  bool any_conflict = false;
  {
    std::unordered_map<int, int> seen;
    for (size_t j = 0; j < n && !any_conflict; ++j) {
      for (size_t k = 0; k < targets[j].size(); ++k) {
        int t = targets[j][k];
        auto it = seen.find(t);
        if (it != seen.end() && (!same_node_ok || it->second != (int)j)) {
          any_conflict = true;
          break;
        }
        seen[t] = (int)j;
      }
    }
  }
  if (!any_conflict) {
    rounds.push_back(std::vector<char>(n, 1));
    return rounds;
  }
  // node-granular greedy rounds; intra-node duplicates (not same_node_ok) are
  // split further by the caller through slot masks
  for (size_t j = 0; j < n; ++j) {
    int r = 0;
    for (;; ++r) {
      if (r == (int)owner.size()) {
        owner.emplace_back();
        rounds.push_back(std::vector<char>(n, 0));
      }
      bool ok = true;
      for (int t : targets[j]) {
        auto it = owner[r].find(t);
        if (it != owner[r].end() && it->second != (int)j) { ok = false; break; }
      }
      if (ok) break;
    }
    for (int t : targets[j]) owner[r][t] = (int)j;
    rounds[r][j] = 1;
  }
  return rounds;
}

// workspace layout: [0, W/8) table blob | [W/8, W-17MiB) scratch (split-K
// partials, dX temporaries, column-sum partials) | 16 MiB dummy gradient
// target | 1 MiB zeroed split-K tile counters
static constexpr size_t kDummyBytes = 16u << 20;
static constexpr size_t kCounterBytes = 1u << 20;
static inline size_t blob_cap(const dg_graph* g) { return (g->work_bytes / 8) & ~size_t(255); }
static inline char* scratch_base(dg_graph* g) { return g->work_base + blob_cap(g); }
// per-slice partial sums of lazily summed input-leaf gradients (LazyGrad):
// written by the backward recurrence, read when gradient() asks
static constexpr size_t kLazyBytes = 1u << 20;
static inline size_t scratch_bytes(dg_graph* g) {
  return g->work_bytes - blob_cap(g) - kDummyBytes - kCounterBytes - kLazyBytes;
}
static inline float* lazy_base(dg_graph* g) {
  return reinterpret_cast<float*>(g->work_base + g->work_bytes - kDummyBytes - kCounterBytes - kLazyBytes);
}
static inline float* dummy_base(dg_graph* g) {
  return reinterpret_cast<float*>(g->work_base + g->work_bytes - kDummyBytes - kCounterBytes);
}
static inline int* counter_base(dg_graph* g) {
  return reinterpret_cast<int*>(g->work_base + g->work_bytes - kCounterBytes);
}
// [0, kScatterCtrBase) split-K tile counters | kScatterCtrs lookup-scatter
// segment counters | kFlagInts recurrence arrival flags
static constexpr int kScatterCtrs = 8192;
static constexpr int kCounterCap = (int)(kCounterBytes / 4) - kFlagInts - kScatterCtrs;
static constexpr int kScatterCtrBase = kCounterCap;
// persistent-recurrence arrival counters (zeroed by each rnn launch)
static inline int* flag_base(dg_graph* g) { return counter_base(g) + kCounterCap + kScatterCtrs; }

// Same-level affine problems accumulate into one grouped GEMM launch.
struct GemmBatch {
  int level = -1;
  int cls = 0;
  bool a_kmajor = false, b_nmajor = false;
  std::vector<GemmProblem> probs;
  int64_t temp_floats = 0;  // dX temporaries at the head of the scratch region
  std::vector<std::function<int()>> post;
  double bytes = 0;
  std::vector<int> targets;  // nodes written with += (dX): must be disjoint per launch
  bool nowait = false;       // TMA launches skip griddepcontrol.wait (overlap window)
};

template <class T>
static inline const T* dev_at(dg_graph* g, size_t off) {
  return reinterpret_cast<const T*>(g->work_base + off);
}

// true when two entries of a row-pointer table coincide (strictly increasing
// tables -- the common, contiguous case -- are answered without sorting)
static bool has_duplicate_rows(const std::vector<uintptr_t>& rows) {
  bool increasing = true;
  for (size_t i = 1; i < rows.size() && increasing; ++i) increasing = rows[i] > rows[i - 1];
  if (increasing) return false;
  std::vector<uintptr_t> u = rows;
  std::sort(u.begin(), u.end());
  return std::adjacent_find(u.begin(), u.end()) != u.end();
}

// Row table (device address inside the plan blob) -> dense block: when the
// rows are equally spaced (row i at base + i*ld) the operand is rewritten as
// base/ld, which the TMA path (and vectorised epilogues) need.
static bool regularize(dg_graph* g, const Plan& plan, Operand& op, int64_t n_rows, int64_t row_len) {
  if (!op.rows) return op.base && (reinterpret_cast<uintptr_t>(op.base) & 15) == 0 && op.ld % 4 == 0 &&
                       op.ld >= row_len;
  const char* dev = reinterpret_cast<const char*>(op.rows);
  if (dev < g->work_base || dev >= g->work_base + plan.blob.size()) return false;
  const uintptr_t* r = reinterpret_cast<const uintptr_t*>(plan.blob.data() + (dev - g->work_base));
  if (n_rows < 1 || (r[0] & 15)) return false;
  const int64_t step = n_rows > 1 ? (int64_t)(r[1] - r[0]) : (int64_t)row_len * 4;
  if (step <= 0 || step % 16 || step / 4 < row_len) return false;
  for (int64_t i = 2; i < n_rows; ++i)
    if ((int64_t)(r[i] - r[i - 1]) != step) return false;
  op.base = reinterpret_cast<const float*>(r[0]);
  op.ld = step / 4;
  op.rows = nullptr;
  return true;
}

// TMA tensor-core path for one problem (tmagemm.cu): regular operands, wide
// enough for 128 x 128 tiles, residual copies in the scratch at lo_base.
static bool tma_try(dg_graph* g, const Plan& plan, const GemmProblem& p0, bool a_kmajor, bool b_nmajor,
                    float* lo_base, int64_t lo_cap, TmaGemmPlan* out) {
  if (!tma_gemm_enabled() || p0.n_seg != 1) return false;
  const int64_t K = p0.seg[0].K;
  if (p0.M < 128 || p0.N < 128 || K < 128 || K > (int64_t)1 << 30) return false;
  GemmProblem p = p0;
  const bool a_mn = a_kmajor, b_mn = !b_nmajor;
  if (!regularize(g, plan, p.seg[0].A, a_mn ? K : p.M, a_mn ? p.M : K)) return false;
  if (!regularize(g, plan, p.seg[0].B, b_mn ? K : p.N, b_mn ? p.N : K)) return false;
  regularize(g, plan, p.C, p.M, p.N);  // optional: vectorised epilogue
  const int64_t la = tma_lo_floats(a_mn ? K : p.M, a_mn ? p.M : K);
  const int64_t lb = tma_lo_floats(b_mn ? K : p.N, b_mn ? p.N : K);
  const int64_t la_p = (la + 63) & ~int64_t(63);
  if (!tma_conv_enabled() && la_p + lb > lo_cap) return false;  // residual copies need scratch
  TmaOperands o{};
  o.M = p.M;
  o.N = p.N;
  o.K = (int)K;
  o.a_mn = a_mn;
  o.b_mn = b_mn;
  o.A = p.seg[0].A.base;
  o.lda = p.seg[0].A.ld;
  o.B = p.seg[0].B.base;
  o.ldb = p.seg[0].B.ld;
  o.A_lo = lo_base;
  o.B_lo = lo_base + la_p;
  // split-K partials: the scratch past the residual copies (all of it when the
  // converter warps form the residuals); tile counters in the zeroed region
  const int64_t lo_used = tma_conv_enabled() ? 0 : ((la_p + lb + 63) & ~int64_t(63));
  if (lo_cap - lo_used >= (int64_t)128 * 128) {
    o.ws = lo_base + lo_used;
    o.ws_floats = lo_cap - lo_used;
    o.cnt = counter_base(g);
    o.cnt_cap = kScatterCtrBase;
  }
  o.C = p.C;
  o.bias = p.bias;
  o.accumulate = p.accumulate;
  return tma_gemm_make(o, out);
}

static void flush_gemm(dg_graph* g, Plan& plan, GemmBatch& gb) {
  if (gb.probs.empty()) {
    gb = GemmBatch();
    return;
  }
  const int64_t temp = (gb.temp_floats + 63) & ~int64_t(63);
  float* work = reinterpret_cast<float*>(scratch_base(g)) + temp;
  const int64_t cap = (int64_t)(scratch_bytes(g) / 4) - temp;
  // dense wide problems: TMA + warp-specialised tcgen05; problems of the batch
  // that share a kernel and write disjoint outputs go up to kTmaGroup per
  // launch with one split factor (small weight-gradient GEMMs fill a wave
  // together instead of each splitting K eight ways)
  std::vector<GemmProblem> rest;
  std::vector<std::pair<TmaGemmPlan, double>> tmas;
  for (const GemmProblem& p : gb.probs) {
    TmaGemmPlan tp;
    if (tma_try(g, plan, p, gb.a_kmajor, gb.b_nmajor, work, cap, &tp)) {
      // only the first launch of an overlap window skips the wait: the later
      // ones wait for their predecessor (which never waited for the window's
      // recurrence) and so never race on the shared workspace
      if (gb.nowait && tmas.empty()) tp.args.nowait = 1;
      tmas.push_back({tp, 4.0 * ((double)p.M * p.seg[0].K + (double)p.seg[0].K * p.N + 2.0 * p.M * p.N)});
    } else {
      rest.push_back(p);
    }
  }
  static const bool group_on = [] {
    const char* e = std::getenv("DG_TMA_GROUP");
    return !(e && e[0] == '0');
  }();
  std::vector<char> used(tmas.size(), 0);
  for (size_t i = 0; i < tmas.size(); ++i) {
    if (used[i]) continue;
    std::vector<size_t> grp{i};
    used[i] = 1;
    for (size_t j = i + 1; j < tmas.size() && group_on && (int)grp.size() < kTmaGroup; ++j) {
      if (used[j]) continue;
      bool ok = true;
      for (size_t q : grp) ok = ok && tma_gemm_groupable(tmas[q].first, tmas[j].first);
      if (!ok) continue;
      grp.push_back(j);
      used[j] = 1;
    }
    if (grp.size() == 1) {
      const TmaGemmPlan tp = tmas[i].first;
      plan.ops.push_back([tp](char*) {
      const cudaStream_t st = g_launch_stream; return launch_tma_gemm(tp, true, true, st); });
      plan.tag(gb.cls, tp.flops, tmas[i].second);
      continue;
    }
    std::vector<TmaGemmPlan> ps;
    double flops = 0, bytes = 0;
    for (size_t q : grp) {
      ps.push_back(tmas[q].first);
      flops += tmas[q].first.flops;
      bytes += tmas[q].second;
    }
    std::vector<TmaGemmPlan*> pp;
    for (auto& x : ps) pp.push_back(&x);
    tma_gemm_regroup(pp.data(), (int)pp.size());
    plan.ops.push_back([ps](char*) {
      const cudaStream_t st = g_launch_stream;
      const TmaGemmPlan* arr[kTmaGroup];
      for (size_t q = 0; q < ps.size(); ++q) arr[q] = &ps[q];
      return launch_tma_gemm_group(arr, (int)ps.size(), st);
    });
    plan.tag(gb.cls, flops, bytes);
  }
  auto post = std::move(gb.post);
  if (rest.empty()) {
    if (!post.empty()) {
      plan.ops.push_back([post](char*) {
        int n = 0;
        for (auto& f : post) n += f();
        return n;
      });
      plan.tag(gb.cls, 0.0, 0.0);
    }
    gb = GemmBatch();
    return;
  }
  // other wide problems run on the cp.async tensor-core kernel (tcgen05
  // 3xTF32), the rest on the grouped SIMT kernel
  const bool tc = tc_gemm_eligible(rest);
  static const bool log_rest = [] {
    const char* e = std::getenv("DG_GEMM_LOG");
    return e && e[0] == '1';
  }();
  if (log_rest)
    for (const GemmProblem& p : rest)
      std::fprintf(stderr, "[gemm-rest] cls %d M %d N %d K %lld segs %d tc %d\n", gb.cls, (int)p.M, (int)p.N,
                   (long long)(p.n_seg ? p.seg[0].K : 0), (int)p.n_seg, (int)tc);
  GemmLaunch L = tc ? tc_gemm_plan(rest, gb.a_kmajor, gb.b_nmajor)
                    : gemm_plan(rest, gb.a_kmajor, gb.b_nmajor, cap, kCounterCap);
  const size_t off = plan.blob.push(rest);
  const GemmProblem* pdev = dev_at<GemmProblem>(g, off);
  int* counters = counter_base(g);
  plan.ops.push_back([L, pdev, work, counters, post, tc](char*) {
      const cudaStream_t st = g_launch_stream;
    int n = tc ? launch_tc_gemm(L, pdev, st) : launch_gemm_group(L, pdev, work, counters, st);
    for (auto& f : post) n += f();
    return n;
  });
  double bytes = 0;
  for (const GemmProblem& p : rest) bytes += 4.0 * ((double)p.M * p.seg[0].K + (double)p.seg[0].K * p.N + 2.0 * p.M * p.N);
  plan.tag(gb.cls, L.flops, bytes);
  gb = GemmBatch();
}

static GemmBatch& gemm_batch_for(dg_graph* g, Plan& plan, GemmBatch& gb, int level, int cls, bool ak, bool bn) {
  if (!gb.probs.empty() && (gb.level != level || gb.cls != cls || gb.a_kmajor != ak || gb.b_nmajor != bn))
    flush_gemm(g, plan, gb);
  gb.level = level;
  gb.cls = cls;
  gb.a_kmajor = ak;
  gb.b_nmajor = bn;
  return gb;
}

}  // namespace dg

using namespace dg;

// =========================================================================
// C-ABI
// =========================================================================

extern "C" {

static bool dry_run();
static bool cuda_graphs_on();
static void warm_graph_runtime();

const char* dg_last_error(void) { return g_err.c_str(); }
int dg_abi_version(void) { return 1; }

int dg_param_register(int kind, int64_t rows, int64_t cols, float* values, float* grad, int64_t* handle) {
  if (rows < 1 || cols < 1) return fail(DG_BAD_SHAPE, "parameter needs rows >= 1 and cols >= 1");
  std::lock_guard<std::mutex> lk(g_param_mu);
  Param p;
  p.kind = kind;
  p.rows = rows;
  p.cols = cols;
  p.val = values;
  p.grad = grad;
  p.alive = true;
  if (kind == 1) p.touched_bits.assign(rows, 0);
  g_params.push_back(std::move(p));
  *handle = (int64_t)g_params.size() - 1;
  g_param_epoch++;
  return DG_OK;
}

int dg_param_rebind(int64_t h, float* values, float* grad) {
  std::lock_guard<std::mutex> lk(g_param_mu);
  Param* p = param_at(h);
  if (!p) return fail(DG_INDEX, "unknown parameter handle");
  p->val = values;
  p->grad = grad;
  g_param_epoch++;
  return DG_OK;
}

int dg_param_release(int64_t h) {
  std::lock_guard<std::mutex> lk(g_param_mu);
  Param* p = param_at(h);
  if (!p) return fail(DG_INDEX, "unknown parameter handle");
  p->alive = false;
  g_param_epoch++;
  p->touched_bits.clear();
  p->touched_list.clear();
  if (p->dp_dev) cudaFree(p->dp_dev);  // best effort (may run at interpreter exit)
  p->dp_dev = nullptr;
  p->dp_cap = 0;
  return DG_OK;
}

int dg_touched_count(int64_t h, int64_t* n) {
  Param* p = param_at(h);
  if (!p) return fail(DG_INDEX, "unknown parameter handle");
  *n = (int64_t)p->touched_list.size();
  return DG_OK;
}

int dg_touched_get(int64_t h, int64_t* ids, int64_t cap) {
  Param* p = param_at(h);
  if (!p) return fail(DG_INDEX, "unknown parameter handle");
  std::vector<int64_t> v = touched_sorted(*p);
  if ((int64_t)v.size() > cap) return fail(DG_INDEX, "touched buffer too small");
  std::copy(v.begin(), v.end(), ids);
  return DG_OK;
}

int dg_touched_add(int64_t h, const int64_t* ids, int64_t n) {
  Param* p = param_at(h);
  if (!p || p->kind != 1) return fail(DG_INDEX, "not a lookup parameter");
  for (int64_t i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= p->rows) return fail(DG_INDEX, "touched id out of range");
    touch(*p, ids[i]);
  }
  return DG_OK;
}

int dg_touched_clear(int64_t h) {
  Param* p = param_at(h);
  if (!p) return fail(DG_INDEX, "unknown parameter handle");
  touched_clear(*p);
  return DG_OK;
}

// ------------------------------------------------------------------ graph

int dg_graph_create(int device, void* fwd_base, size_t fwd_bytes, void* bwd_base, size_t bwd_bytes, void* work_base,
                    size_t work_bytes, dg_graph** out) {
  if (!fwd_base || !bwd_base || !work_base) return fail(DG_CONFIG, "null arena");
  dg_graph* g = new dg_graph();
  g->device = device;
  g->fwd_base = static_cast<char*>(fwd_base);
  g->fwd_bytes = fwd_bytes;
  g->bwd_base = static_cast<char*>(bwd_base);
  g->bwd_bytes = bwd_bytes;
  g->work_base = static_cast<char*>(work_base);
  g->work_bytes = work_bytes;
  if (work_bytes < (64u << 20)) {
    delete g;
    return fail(DG_CONFIG, "workspace must be at least 64 MiB");
  }
  if (cuda_graphs_on() && !dry_run()) warm_graph_runtime();
  *out = g;
  return DG_OK;
}

int dg_graph_destroy(dg_graph* g) {
  if (!g) return DG_OK;
  g->pcache[0].clear();
  g->pcache[1].clear();
  if (g->vcache_ev) {
    cudaEventSynchronize(g->vcache_ev);
    cudaEventDestroy(g->vcache_ev);
  }
  for (auto& p : g->pinned) {
    if (p.pending) cudaEventSynchronize(p.ev);
    if (p.ptr) cudaFreeHost(p.ptr);
    if (p.ev) cudaEventDestroy(p.ev);
  }
  delete g;
  return DG_OK;
}

int dg_graph_set_stream(dg_graph* g, void* stream) {
  g->stream = static_cast<cudaStream_t>(stream);
  return DG_OK;
}

int dg_graph_renew(dg_graph* g) {
  g->memo_sched.reset();
  g->memo_scope = -1;
  g->nodes.clear();
  g->inputs.clear();
  g->aux_i.clear();
  g->aux_f.clear();
  g->watermark = -1;
  g->vcache_node = -1;
  // the reference zeroes the used backward prefix here (arena.py:85-92); the
  // device backward slots are zeroed when a backward pass allocates them
  g->fwd_cursor = 0;
  g->bwd_cursor = 0;
  g->has_grads = false;
  g->fwd_hist = 0;
  g->lazy.clear();
  return DG_OK;
}

int dg_graph_append(dg_graph* g, const dg_node* nodes, int32_t n, const int32_t* inputs, int32_t n_inputs,
                    const int64_t* aux_i, int64_t n_aux_i, const float* aux_f, int64_t n_aux_f) {
  const int in_base = (int)g->inputs.size();
  const int64_t ai_base = (int64_t)g->aux_i.size(), af_base = (int64_t)g->aux_f.size();
  const int first = (int)g->nodes.size();
  g->inputs.insert(g->inputs.end(), inputs, inputs + n_inputs);
  g->aux_i.insert(g->aux_i.end(), aux_i, aux_i + n_aux_i);
  g->aux_f.insert(g->aux_f.end(), aux_f, aux_f + n_aux_f);
  g->nodes.reserve(g->nodes.size() + n);
  for (int i = 0; i < n; ++i) {
    const dg_node& r = nodes[i];
    Node x;
    x.kind = r.kind;
    x.n_in = r.n_in;
    x.in_off = r.in_off + in_base;
    x.rank = r.rank;
    x.elem = 1;
    for (int d = 0; d < 4; ++d) {
      x.dims[d] = d < r.rank ? r.dims[d] : 1;
      if (d < r.rank) x.elem *= r.dims[d];
    }
    x.batch = r.batch;
    x.ai_off = r.aux_i_off + ai_base;
    x.ai_len = r.aux_i_len;
    x.af_off = r.aux_f_off + af_base;
    x.af_len = r.aux_f_len;
    if (x.kind < 0 || x.kind >= DG_OP_COUNT) return fail(DG_INTERNAL, "bad op kind");
    for (int k = 0; k < x.n_in; ++k) {
      const int src = g->inputs[x.in_off + k];
      if (src < 0 || src >= first + i) return fail(DG_STALE, "input refers to a later or unknown node");
    }
    if (x.kind == DG_OP_PARAMETER || x.kind == DG_OP_LOOKUP || x.kind == DG_OP_LOOKUP_BATCH) {
      Param* p = param_at(g->aux_i[x.ai_off]);
      if (!p) return fail(DG_INDEX, "node references an unknown parameter");
      if (x.kind != DG_OP_PARAMETER) {
        for (int64_t q = 1; q < x.ai_len; ++q) {
          const int64_t id = g->aux_i[x.ai_off + q];
          if (id < 0 || id >= p->rows) return fail(DG_INDEX, "lookup row out of range");
        }
      }
    }
    g->nodes.push_back(x);
  }
  return DG_OK;
}

// ---------------------------------------------------------------- forward

// DG_DRYRUN=1: plan everything, launch nothing (host-side planner profiling
// without a device; results are meaningless)
static bool dry_run() {
  static const bool on = [] {
    const char* e = std::getenv("DG_DRYRUN");
    return e && e[0] == '1';
  }();
  return on;
}

// DG_NVTX=1: NVTX ranges around planning and around every launch group
// (named by op class), for nsys / ncu --nvtx timelines
static bool nvtx_on() {
  static const bool on = [] {
    const char* e = std::getenv("DG_NVTX");
    return e && e[0] == '1';
  }();
  return on;
}
static const char* const kClassName[C_NCLASS] = {"gemm_fwd", "gemm_dx", "gemm_dw", "pnls_fwd", "pnls_bwd",
                                                 "elementwise", "gather", "scatter_add", "bias_colsum", "other",
                                                 "rnn_fwd", "rnn_bwd"};
struct NvtxRange {
  bool on;
  explicit NvtxRange(const char* name) : on(nvtx_on()) {
    if (on) nvtxRangePushA(name);
  }
  ~NvtxRange() {
    if (on) nvtxRangePop();
  }
};

// run launch closures in order (with CUDA events around the profiled op
// classes); adds the kernel launches issued to *launched
static int run_ops(dg_graph* g, std::vector<std::function<int(char*)>>& ops, std::vector<OpMeta>& meta,
                   int64_t* launched, cudaStream_t stream) {
  g_launch_stream = stream;
  meta.resize(ops.size());
  for (size_t q = 0; q < ops.size(); ++q) {
    const OpMeta& mt = meta[q];
    const bool prof = (g->prof_mask >> mt.cls) & 1u;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (prof) {
      for (cudaEvent_t* e : {&e0, &e1}) {
        if (g->event_pool.empty()) {
          DG_CUDA_TRY(cudaEventCreate(e));
        } else {
          *e = g->event_pool.back();
          g->event_pool.pop_back();
        }
      }
      DG_CUDA_TRY(cudaEventRecord(e0, g->stream));
    }
    static const bool op_timing = [] {
      const char* e = std::getenv("DG_PLAN_TIMING");
      return e && e[0] == '2';
    }();
    const auto t_op = std::chrono::steady_clock::now();
    NvtxRange nv(mt.cls >= 0 && mt.cls < C_NCLASS ? kClassName[mt.cls] : "op");
    int n = ops[q](g->work_base);
    if (op_timing)
      std::fprintf(stderr, "[op] class %d launches %d host %.1f us\n", mt.cls, n,
                   std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_op).count());
    if (n < 0) return fail(DG_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(cudaGetLastError()));
    *launched += n;
    if (prof) {
      DG_CUDA_TRY(cudaEventRecord(e1, g->stream));
      g->prof_pending[mt.cls].push_back({e0, e1});
      g->prof_flops[mt.cls] += mt.flops;
      g->prof_bytes[mt.cls] += mt.bytes;
      g->prof_count[mt.cls] += 1;
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DG_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return DG_OK;
}

static int prepare_launch(dg_graph* g, const Blob& blob) {
  const size_t blob_bytes = (blob.size() + 255) & ~size_t(255);
  if (blob_bytes > blob_cap(g)) return fail(DG_CONFIG, "plan tables exceed the workspace");
  if (dry_run()) return DG_OK;
  if (!g->counters_ready) {
    // split-K tile counters start (and are always left) at zero
    DG_CUDA_TRY(cudaMemsetAsync(g->work_base + g->work_bytes - (1u << 20), 0, 1u << 20, g->stream));
    g->counters_ready = true;
  }
  return upload(g, blob, g->work_base);
}

static int launch_plan(dg_graph* g, Plan& plan, int64_t* launched = nullptr) {
  int rc = prepare_launch(g, plan.blob);
  if (rc || dry_run()) return rc;
  int64_t n = 0;
  rc = run_ops(g, plan.ops, plan.meta, &n, g->stream);
  g->launches += n;
  if (launched) *launched = n;
  return rc;
}

static bool plan_cache_on() {
  static const bool on = [] {
    const char* e = std::getenv("DG_PLAN_CACHE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// CUDA-graph replay of cached plans is opt-in (DG_CUDA_GRAPH=1): on the PTB
// headline the loop is device-bound once plans are cached, and a capture
// (~0.1-0.2 ms host) only pays off for plans that recur many times
static bool cuda_graphs_on() {
  static const bool on = [] {
    const char* e = std::getenv("DG_CUDA_GRAPH");
    return e && e[0] == '1';
  }();
  return on;
}

static uint64_t mix64(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  return h * 0xff51afd7ed558ccdull;
}

// key of a plan: structure, the node range, the placement history of this
// generation, arena cursors, parameter storage epoch, stream
static uint64_t plan_key(const dg_graph* g, int which, int lo, int hi) {
  uint64_t h = mix64(g->memo_key, (uint64_t)which);
  h = mix64(h, (uint64_t)(uint32_t)lo);
  h = mix64(h, (uint64_t)(uint32_t)hi);
  h = mix64(h, g->fwd_hist);
  h = mix64(h, (uint64_t)g->fwd_cursor);
  h = mix64(h, (uint64_t)g->bwd_cursor);
  h = mix64(h, g_param_epoch.load());
  h = mix64(h, (uint64_t)reinterpret_cast<uintptr_t>(g->stream));
  return h;
}

static CachedPlan* plan_cache_find(dg_graph* g, int which, uint64_t key) {
  if (!plan_cache_on()) return nullptr;
  auto& v = g->pcache[which];
  for (size_t i = 0; i < v.size(); ++i)
    if (v[i]->key == key) {
      if (i) std::rotate(v.begin(), v.begin() + i, v.begin() + i + 1);
      return v[0].get();
    }
  return nullptr;
}

// keep a freshly launched plan (its closures move into the cache)
static void plan_cache_store(dg_graph* g, int which, uint64_t key, Plan& plan, size_t static_ops,
                             size_t static_bytes, PatchRec&& rec, int64_t launched_static) {
  if (!plan_cache_on() || dry_run()) return;
  auto cp = std::make_shared<CachedPlan>();
  cp->key = key;
  cp->tmpl.assign(plan.blob.data(), plan.blob.data() + static_bytes);
  plan.meta.resize(plan.ops.size());
  cp->ops.assign(std::make_move_iterator(plan.ops.begin()), std::make_move_iterator(plan.ops.begin() + static_ops));
  cp->meta.assign(plan.meta.begin(), plan.meta.begin() + static_ops);
  cp->patch = std::move(rec);
  cp->lazy = plan.lazy;
  cp->kernel_launches = launched_static;
  auto& v = g->pcache[which];
  v.insert(v.begin(), std::move(cp));
  if (v.size() > 32) v.pop_back();
}

// blob for a cached plan: the template with this graph's data written in
static void blob_from_template(const dg_graph* g, const CachedPlan& cp, Blob& B) {
  B.push_bytes(cp.tmpl.data(), cp.tmpl.size(), 16);
  uint8_t* d = B.data();
  for (const PatchRec::Payload& p : cp.patch.payload)
    std::memcpy(d + p.off, g->aux_f.data() + g->nodes[p.node].af_off, p.bytes);
  for (const PatchRec::Ids& r : cp.patch.ids) {
    const Node& x = g->nodes[r.node];
    const int64_t* src = g->aux_i.data() + x.ai_off + r.q0;
    const int64_t n = x.ai_len - r.q0;
    if (r.width == 8) {
      std::memcpy(d + r.off, src, (size_t)n * 8);
    } else {
      int32_t* o = reinterpret_cast<int32_t*>(d + r.off);
      for (int64_t q = 0; q < n; ++q) o[q] = (int32_t)src[q];
    }
  }
}

// per host thread: the private non-blocking stream cached plans are recorded
// on (captures are synchronous host calls, so one per thread serves every
// graph); the first use also pays the runtime's one-time graph set-up with a
// throwaway capture
static cudaStream_t capture_stream() {
  static thread_local cudaStream_t cs = nullptr;
  if (!cs && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    cs = nullptr;
  }
  return cs;
}

static void warm_graph_runtime() {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaStream_t cs = capture_stream();
    void* buf = nullptr;
    if (!cs || cudaMalloc(&buf, 256) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      cudaMemsetAsync(buf, 0, 256, cs);
      if (cudaStreamEndCapture(cs, &graph) == cudaSuccess && graph &&
          cudaGraphInstantiateWithFlags(&exec, graph, 0) == cudaSuccess) {
        cudaGraphLaunch(exec, cs);
        cudaStreamSynchronize(cs);
      }
    }
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    cudaFree(buf);
    cudaGetLastError();
  });
}

// upload the blob, replay the cached static ops (as a CUDA graph from the
// second use on), then the per-call tail ops of `tail`
static int launch_cached(dg_graph* g, CachedPlan& cp, Plan& tail) {
  int rc = prepare_launch(g, tail.blob);
  if (rc || dry_run()) return rc;
  bool profiling = false;
  for (const OpMeta& m : cp.meta) profiling = profiling || ((g->prof_mask >> m.cls) & 1u);
  int64_t n = 0;
  // a structure seen for the third time is recorded as a CUDA graph (the
  // capture + instantiate, ~0.1-0.2 ms, pays off only for plans that recur)
  if (cuda_graphs_on() && !profiling && cp.replays >= 2 && !cp.exec && cp.replays != -1000) {
    // recorded on a private non-blocking stream (the graph's own stream may
    // be the legacy default stream, which cannot be captured); replayed on
    // the graph's stream
    PlanTimer ct("graph-capture");
    cudaStream_t cs = capture_stream();
    if (!cs) return fail(DG_CUDA, "cannot create the capture stream");
    cudaGraph_t graph = nullptr;
    bool ok = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    int64_t n_cap = 0;
    int rc_cap = ok ? run_ops(g, cp.ops, cp.meta, &n_cap, cs) : DG_CUDA;
    ok = cudaStreamEndCapture(cs, &graph) == cudaSuccess && ok && rc_cap == DG_OK;
    ct.lap("capture");
    if (ok) ok = cudaGraphInstantiateWithFlags(&cp.exec, graph, 0) == cudaSuccess;
    ct.lap("instantiate");
    if (graph) cudaGraphDestroy(graph);
    if (!ok) {
      cudaGetLastError();  // capture unsupported for this plan: replay op by op
      cp.exec = nullptr;
      cp.replays = -1000;
    }
  }
  g->stats[5]++;  // plan-cache hits (cumulative)
  if (cp.exec && !profiling) {
    PlanTimer lt("graph-launch");
    DG_CUDA_TRY(cudaGraphLaunch(cp.exec, g->stream));
    lt.lap("launch");
    n += cp.kernel_launches;
    g->stats[6]++;  // CUDA-graph replays (cumulative)
  } else {
    rc = run_ops(g, cp.ops, cp.meta, &n, g->stream);
    if (rc) return rc;
  }
  if (cp.replays >= 0) cp.replays++;
  rc = run_ops(g, tail.ops, tail.meta, &n, g->stream);
  g->launches += n;
  return rc;
}

// scratch region of the workspace (after the table blob half)


// dX += G W for one row set: rows of G (device table), W column-major m x K.
// Rows landing on one target (broadcast x, shared x) go through a dense temp
// and a deterministic segmented row reduce (same scheme as the affine path).
static void push_dx_problem(dg_graph* g, Plan& plan, GemmBatch& batch, const float* const* g_rows_dev, bool g_al,
                            const float* W, int m, int K, const std::vector<uintptr_t>& dxrows) {
  Blob& B = plan.blob;
  const bool dup = has_duplicate_rows(dxrows);
  GemmProblem pr{};
  pr.M = (int)dxrows.size();
  pr.N = K;
  pr.n_seg = 1;
  pr.seg[0].K = m;
  pr.seg[0].A.rows = g_rows_dev;
  pr.seg[0].A.rows_aligned = g_al;
  pr.seg[0].B.base = W;
  pr.seg[0].B.ld = m;
  batch.bytes += 4.0 * ((double)pr.M * m + (double)m * pr.N + 2.0 * pr.M * pr.N);
  if (!dup) {
    pr.accumulate = 1;
    pr.C.rows = dev_at<const float*>(g, B.push(dxrows));
  } else {
    const int64_t R = (int64_t)dxrows.size();
    std::vector<int> order(R);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return dxrows[x] < dxrows[y]; });
    std::vector<uintptr_t> tgt;
    std::vector<int32_t> seg;
    for (int64_t q = 0; q < R; ++q) {
      if (q == 0 || dxrows[order[q]] != dxrows[order[q - 1]]) {
        tgt.push_back(dxrows[order[q]]);
        seg.push_back((int32_t)q);
      }
    }
    seg.push_back((int32_t)R);
    std::vector<int64_t> pos(R);
    for (int64_t q = 0; q < R; ++q) pos[order[q]] = q;
    float* temp = reinterpret_cast<float*>(scratch_base(g)) + batch.temp_floats;
    batch.temp_floats += (R * K + 63) & ~int64_t(63);
    std::vector<uintptr_t> crow(R);
    for (int64_t r = 0; r < R; ++r) crow[r] = P(temp + pos[r] * K);
    pr.accumulate = 0;
    pr.C.rows = dev_at<const float*>(g, B.push(crow));
    float* const* tg =
        const_cast<float* const*>(reinterpret_cast<const float* const*>(dev_at<float*>(g, B.push(tgt))));
    const int* sg = dev_at<int>(g, B.push(seg));
    const int n_t = (int)tgt.size();
    batch.post.push_back([tg, sg, temp, n_t, K]() {
      return launch_row_reduce_scatter(tg, sg, temp, n_t, K, g_launch_stream);
    });
  }
  batch.probs.push_back(pr);
}

// Persistent LSTM recurrence (rnn.cu) for a group of U_RNN units: stacks are
// packed into launches (same rows-per-CTA, CTAs <= SMs).  Backward also plans
// the batched gradients of the stacks' external inputs (x_t of the bottom
// chain, h_{-1}; c_{-1} broadcast sums) and registers the weight / bias
// gradient rows for the aggregated dW GEMMs and column sums.
static void plan_rnn_group(dg_graph* g, const Schedule& S, const Group& gr, Plan& plan, bool bwd,
                           std::unordered_map<int64_t, AffineUse>* wuse,
                           std::unordered_map<int64_t, std::vector<uintptr_t>>* buse, GemmBatch* gb) {
  Blob& B = plan.blob;
  // pack
  std::vector<std::vector<int>> launches;
  {
    std::vector<int> cur;
    int cur_bs = -1, cur_ctas = 0, cur_chains = 0, cur_flags = 0;
    for (int u : gr.units) {
      const RnnStack& sk = S.rnns[S.units[u].rnn];
      int fl = 0;
      for (auto& cp : sk.chains) fl += cp.n_s * (int)cp.cells.size();
      if (!cur.empty() && (sk.bs != cur_bs || cur_ctas + sk.ctas > kSmCount ||
                           cur_chains + (int)sk.chains.size() > kRnnMaxChains || cur_flags + fl > kFlagInts)) {
        launches.push_back(cur);
        cur.clear();
        cur_ctas = cur_chains = cur_flags = 0;
      }
      cur.push_back(S.units[u].rnn);
      cur_bs = sk.bs;
      cur_ctas += sk.ctas;
      cur_chains += (int)sk.chains.size();
      cur_flags += fl;
    }
    if (!cur.empty()) launches.push_back(cur);
  }
  if (!bwd) {
    // input projections of every step, batched: G_t = b + Wx x_t (the
    // recurrent kernels add Wh h_{t-1})
    for (int u : gr.units) {
      for (const RnnChainPlan& cp : S.rnns[S.units[u].rnn].chains) {
        const int T = (int)cp.G.size(), Bt = cp.B;
        std::vector<uintptr_t> xrows((size_t)T * Bt), crow((size_t)T * Bt);
        for (int t = 0; t < T; ++t) {
          const Node& Gn = g->nodes[cp.G[t]];
          const Node& xn = g->nodes[g->inputs[Gn.in_off + 2]];
          for (int b = 0; b < Bt; ++b) {
            xrows[(size_t)t * Bt + b] = P(xn.val + (xn.batch == 1 ? 0 : (int64_t)b * cp.K_in));
            crow[(size_t)t * Bt + b] = P(Gn.val + (int64_t)b * cp.gw);
          }
        }
        GemmBatch& bt = gemm_batch_for(g, plan, *gb, gr.level, C_GEMM_FWD, false, false);
        GemmProblem pr{};
        pr.M = T * Bt;
        pr.N = cp.gw;
        pr.n_seg = 1;
        pr.accumulate = 0;
        pr.seg[0].K = cp.K_in;
        pr.seg[0].A.rows = dev_at<const float*>(g, B.push(xrows));
        pr.seg[0].A.rows_aligned = all_aligned16(xrows);
        pr.seg[0].B.base = param_at(cp.hWx)->val;
        pr.seg[0].B.ld = cp.gw;
        pr.C.rows = dev_at<const float*>(g, B.push(crow));
        pr.C.rows_aligned = all_aligned16(crow);
        pr.bias.base = param_at(cp.hb)->val;
        pr.bias.ld = 0;
        bt.probs.push_back(pr);
        bt.bytes += 4.0 * ((double)pr.M * cp.K_in + (double)cp.K_in * pr.N + (double)pr.M * pr.N);
      }
    }
    flush_gemm(g, plan, *gb);
  }
  std::unordered_set<int> init_h_done, init_c_done;  // chains (by G_0) whose initial-state grads the kernel owns
  for (const auto& L : launches) {
    RnnArgs a{};
    std::vector<const RnnChainPlan*> cps;
    a.flags = flag_base(g);
    a.gx = bwd ? 0 : 1;
    a.bs = S.rnns[L[0]].bs;
    int cta = 0, flag = 0;
    double flops = 0, bytes = 0;
    a.cj = 1 << 30;
    bool vec_ok = true;
    for (int sid : L) {
      const RnnStack& sk = S.rnns[sid];
      const int base = a.n_chains;
      for (const RnnChainPlan& cp : sk.chains) {
        cps.push_back(&cp);
        RnnChain& c = a.ch[a.n_chains++];
        const int T = (int)cp.G.size();
        c.T = T;
        c.B = cp.B;
        c.H = cp.H;
        c.K_in = bwd ? cp.K_in : 0;  // forward: recurrent part only (gx mode)
        c.gw = cp.gw;
        c.off_i = cp.off[0];
        c.off_f = cp.off[1];
        c.off_o = cp.off[2];
        c.off_g = cp.off[3];
        c.n_s = cp.n_s;
        c.n_u = cp.n_u;
        c.cta0 = cta;
        cta += cp.n_s * cp.n_u;
        c.src = cp.src >= 0 ? base + cp.src : -1;
        c.cons = cp.cons >= 0 ? base + cp.cons : -1;
        c.flag0 = flag;
        flag += cp.n_s * T;
        c.Wx = param_at(cp.hWx)->val;
        c.Wh = param_at(cp.hWh)->val;
        c.bias = param_at(cp.hb)->val;
        std::vector<uintptr_t> vals((size_t)T * kRnnSlots), grads;
        std::vector<int32_t> b1(T);
        if (bwd) grads.resize((size_t)T * kRnnSlots);
        for (int t = 0; t < T; ++t) {
          const Node& Gn = g->nodes[cp.G[t]];
          const int x = g->inputs[Gn.in_off + 2], hp = g->inputs[Gn.in_off + 4];
          const Unit& cu = cp.cells[t];
          const int cprev = cu.ins[1];
          int slot[kRnnSlots];
          slot[0] = cp.G[t];
          slot[1] = cprev;
          for (int k = 0; k < 13; ++k) slot[2 + k] = cu.nodes[k];
          slot[15] = x;
          slot[16] = hp;
          for (int k : {0, 15, 16}) vec_ok = vec_ok && (P(g->nodes[slot[k]].val) & 15) == 0;
          if (bwd) vec_ok = vec_ok && (P(g->nodes[slot[0]].grad) & 15) == 0;
          for (int k = 0; k < kRnnSlots; ++k) {
            vals[(size_t)t * kRnnSlots + k] = P(g->nodes[slot[k]].val);
            if (bwd) grads[(size_t)t * kRnnSlots + k] = P(g->nodes[slot[k]].grad);
          }
          const bool bb = cp.B > 1;
          b1[t] = (bb && g->nodes[x].batch == 1 ? 1 : 0) | (bb && g->nodes[hp].batch == 1 ? 2 : 0) |
                  (bb && g->nodes[cprev].batch == 1 ? 4 : 0);
        }
        vec_ok = vec_ok && cp.K_in % 4 == 0 && cp.H % 4 == 0 && cp.gw % 4 == 0 && cp.off[0] % 4 == 0 &&
                 cp.off[1] % 4 == 0 && cp.off[2] % 4 == 0 && cp.off[3] % 4 == 0;
        c.val = dev_at<const float*>(g, B.push(vals));
        if (bwd) c.grad = dev_at<float*>(g, B.push(grads));
        c.b1 = dev_at<int>(g, B.push(b1));
        const double gwd = cp.gw, bd = cp.B;
        flops += bwd ? 2.0 * bd * gwd * cp.H * (T - 1) : 2.0 * bd * gwd * cp.H * T;
        bytes += 4.0 * bd * cp.H * T * (bwd ? 30 : 17);
      }
      for (int k = base; k < a.n_chains; ++k) {
        const RnnChain& c = a.ch[k];
        if (c.cons >= 0 && bwd) flops += 2.0 * c.B * a.ch[c.cons].gw * c.H * c.T;
      }
    }
    a.ctas = cta;
    a.n_flags = flag;
    a.vec = vec_ok ? 1 : 0;
    a.trace = rnn_trace_enabled() ? (std::getenv("DG_RNN_TRACE")[0] == '2' ? 2 : 1) : 0;
    {
      static const int knob = std::getenv("DG_RNN_KNOB") ? std::atoi(std::getenv("DG_RNN_KNOB")) : 0;
      a.knob = knob;
    }
    // cluster mode: one cluster per (chain, batch slice) exchanging through
    // distributed shared memory; needs equal unit-block counts (<= 16)
    int cl = a.ch[0].n_u;
    // a one-CTA "cluster" has nothing to exchange: the global-counter kernels serve it
    bool use_cl = rnn_cluster_enabled() && cl >= 2 && cl <= 16;
    for (int k = 0; k < a.n_chains; ++k) use_cl = use_cl && a.ch[k].n_u == cl;
    size_t smem = 0, smem_cl = 0;
    if (bwd) {
      for (int k = 0; k < a.n_chains; ++k) {
        const int gwc = a.ch[k].cons >= 0 ? a.ch[a.ch[k].cons].gw : 0;
        a.cj = std::min(a.cj, rnn_pick_cj(a.ch[k].gw, gwc, a.bs));
        if (use_cl) {
          int cj = a.cj;
          while (cj > 32 && rnn_bwd_cl_smem(a.ch[k].H, gwc, a.bs, cj) > kSmemMax) cj -= 32;
          a.cj = cj;
        }
      }
      for (int k = 0; k < a.n_chains; ++k) {
        const int gwc = a.ch[k].cons >= 0 ? a.ch[a.ch[k].cons].gw : 0;
        smem = std::max(smem, rnn_bwd_smem(a.ch[k].gw, gwc, a.bs, a.cj));
        smem_cl = std::max(smem_cl, rnn_bwd_cl_smem(a.ch[k].H, gwc, a.bs, a.cj));
      }
    } else {
      a.cj = 0;
      for (int k = 0; k < a.n_chains; ++k) {
        smem = std::max(smem, rnn_fwd_smem(a.ch[k].K_in + a.ch[k].H, a.bs));  // K_in = 0 (gx mode)
        smem_cl = std::max(smem_cl, rnn_fwd_cl_smem(a.ch[k].K_in, a.ch[k].H, a.bs));
      }
    }
    use_cl = use_cl && smem_cl <= kSmemMax;
    // decided here, not at launch: the initial-state gradients below exist
    // only in the cluster backward kernel
    use_cl = use_cl && rnn_cluster_fits(a, bwd, smem_cl, cl);
    // initial-state gradients inside the backward cluster kernel (one more
    // reduce-scatter round gives dh_{-1}): per-row h_{-1} is accumulated in
    // place, batch-1 h_{-1} / c_{-1} leave per-slice row sums that one
    // rnn_part_sum_kernel adds up -- now for computed / parameter targets,
    // on gradient() for INPUT leaves (LazyGrad)
    RnnPartSum eager{};
    if (bwd && use_cl) {
      std::vector<int> own_h;
      const size_t cap = kLazyBytes / 4;
      for (int k = 0; k < a.n_chains; ++k) {
        const RnnChainPlan& cp = *cps[k];
        RnnChain& c = a.ch[k];
        const int hnode = g->inputs[g->nodes[cp.G[0]].in_off + 4];
        const int cnode = cp.cells[0].ins[1];
        const Node& hn = g->nodes[hnode];
        const Node& cn = g->nodes[cnode];
        const size_t need = (size_t)cp.n_s * cp.H;
        auto add_part = [&](int node, float*& part) {
          part = lazy_base(g) + plan.lazy_floats;
          plan.lazy_floats += (need + 63) & ~size_t(63);
          const Node& x = g->nodes[node];
          if (x.kind == DG_OP_INPUT) {
            plan.lazy.push_back(LazyGrad{node, x.grad, part, cp.n_s, cp.H});
          } else {
            eager.H[eager.n] = cp.H;
            eager.n_s[eager.n] = cp.n_s;
            eager.dst[eager.n] = x.grad;
            eager.part[eager.n] = part;
            eager.n++;
          }
        };
        if (hn.batch == cp.B && std::find(own_h.begin(), own_h.end(), hnode) == own_h.end()) {
          c.h0 = 1;  // per row, in place (no other chain of this launch adds into it)
          own_h.push_back(hnode);
          init_h_done.insert(cp.G[0]);
        } else if (hn.batch == 1 && cp.B > 1 && plan.lazy_floats + need <= cap) {
          c.h0 = 2;
          add_part(hnode, c.h0_part);
          init_h_done.insert(cp.G[0]);
        }
        if (cn.batch == 1 && cp.B > 1 && plan.lazy_floats + need <= cap) {
          c.c0 = 1;
          add_part(cnode, c.c0_part);
          init_c_done.insert(cp.G[0]);
        }
      }
    }
    plan.ops.push_back([a, smem, smem_cl, use_cl, cl, bwd](char*) {
      const cudaStream_t st = g_launch_stream;
      if (use_cl) {
        // residency was checked while planning; the fallback kernels do not
        // produce the initial-state gradients the plan counts on
        const int n = launch_rnn_cluster(a, bwd, smem_cl, cl, st);
        return n == -2 ? -1 : n;
      }
      return launch_rnn(a, bwd, smem, st);
    });
    plan.tag(bwd ? C_RNN_BWD : C_RNN_FWD, flops, bytes);
    plan.rnn_bwd_ctas = bwd && use_cl && !eager.n ? a.ctas : 0;
    plan.rnn_bwd_op = plan.ops.size();
    if (eager.n) {
      plan.ops.push_back([eager](char*) { return launch_rnn_part_sum(eager, g_launch_stream); });
      plan.tag(C_ELEMWISE, 0.0, 0.0);
    }
  }
  if (!bwd) return;

  // ---- backward: gradients leaving the stacks, weight / bias aggregation
  RnnC0 c0{};
  for (int u : gr.units) {
    const RnnStack& sk = S.rnns[S.units[u].rnn];
    for (const RnnChainPlan& cp : sk.chains) {
      const int T = (int)cp.G.size();
      const int Bt = cp.B;
      std::vector<uintptr_t> grows((size_t)T * Bt), xrows((size_t)T * Bt), hrows((size_t)T * Bt);
      std::vector<uintptr_t> dxrows, g0rows;
      for (int t = 0; t < T; ++t) {
        const Node& Gn = g->nodes[cp.G[t]];
        const Node& xn = g->nodes[g->inputs[Gn.in_off + 2]];
        const Node& hn = g->nodes[g->inputs[Gn.in_off + 4]];
        for (int b = 0; b < Bt; ++b) {
          const size_t q = (size_t)t * Bt + b;
          grows[q] = P(Gn.grad + (int64_t)b * cp.gw);
          xrows[q] = P(xn.val + (xn.batch == 1 ? 0 : (int64_t)b * cp.K_in));
          hrows[q] = P(hn.val + (hn.batch == 1 ? 0 : (int64_t)b * cp.H));
          if (cp.src < 0) dxrows.push_back(P(xn.grad + (xn.batch == 1 ? 0 : (int64_t)b * cp.K_in)));
        }
      }
      // weight / bias gradients: one aggregated GEMM per parameter later
      {
        AffineUse& ux = (*wuse)[cp.hWx];
        ux.n_in = cp.K_in;
        ux.m = cp.gw;
        ux.x_rows.insert(ux.x_rows.end(), xrows.begin(), xrows.end());
        ux.g_rows.insert(ux.g_rows.end(), grows.begin(), grows.end());
        AffineUse& uh = (*wuse)[cp.hWh];
        uh.n_in = cp.H;
        uh.m = cp.gw;
        uh.x_rows.insert(uh.x_rows.end(), hrows.begin(), hrows.end());
        uh.g_rows.insert(uh.g_rows.end(), grows.begin(), grows.end());
        auto& bv = (*buse)[cp.hb];
        bv.insert(bv.end(), grows.begin(), grows.end());
      }
      const bool g_al = all_aligned16(grows);
      const float* const* g_dev = dev_at<const float*>(g, B.push(grows));
      // gradients leaving the chain, batched across the group's chains: one
      // grouped launch unless two problems write the same node (then flush)
      auto add_dx = [&](const std::vector<int>& target_nodes, const float* W, int K,
                        const std::vector<uintptr_t>& rows) {
        GemmBatch& bt = gemm_batch_for(g, plan, *gb, gr.level, C_GEMM_DX, false, true);
        bool clash = false;
        for (int tnode : target_nodes)
          clash = clash || std::find(bt.targets.begin(), bt.targets.end(), tnode) != bt.targets.end();
        if (clash) flush_gemm(g, plan, *gb);
        GemmBatch& b2 = gemm_batch_for(g, plan, *gb, gr.level, C_GEMM_DX, false, true);
        push_dx_problem(g, plan, b2, g_dev, g_al, W, cp.gw, K, rows);
        b2.targets.insert(b2.targets.end(), target_nodes.begin(), target_nodes.end());
      };
      // x_t of the bottom chain: dX = dG Wx over every step
      if (cp.src < 0) {
        std::vector<int> xs;
        for (int t = 0; t < T; ++t) xs.push_back(g->inputs[g->nodes[cp.G[t]].in_off + 2]);
        add_dx(xs, param_at(cp.hWx)->val, cp.K_in, dxrows);
      }
      // h_{-1}: dX = dG_0 Wh (unless the backward kernel produced it)
      if (!init_h_done.count(cp.G[0])) {
        const Node& G0 = g->nodes[cp.G[0]];
        const int hnode = g->inputs[G0.in_off + 4];
        const Node& hn = g->nodes[hnode];
        std::vector<uintptr_t> hd(Bt);
        for (int b = 0; b < Bt; ++b) hd[b] = P(hn.grad + (hn.batch == 1 ? 0 : (int64_t)b * cp.H));
        add_dx({hnode}, param_at(cp.hWh)->val, cp.H, hd);
      }
      // c_{-1} broadcast over the batch: batch sum of dc_0 * f_0
      const Node& cpn = g->nodes[cp.cells[0].ins[1]];
      if (cpn.batch == 1 && Bt > 1 && !init_c_done.count(cp.G[0])) {
        if (c0.n == kRnnMaxChains) {
          plan.ops.push_back([c0](char*) {
      const cudaStream_t st = g_launch_stream; return launch_rnn_c0(c0, st); });
          plan.tag(C_ELEMWISE, 0.0, 0.0);
          c0 = RnnC0{};
        }
        c0.H[c0.n] = cp.H;
        c0.B[c0.n] = Bt;
        c0.dst[c0.n] = cpn.grad;
        c0.dc[c0.n] = g->nodes[cp.cells[0].nodes[10]].grad;
        c0.af[c0.n] = g->nodes[cp.cells[0].nodes[5]].val;
        c0.n++;
      }
    }
  }
  flush_gemm(g, plan, *gb);
  if (c0.n) {
    plan.ops.push_back([c0](char*) {
      const cudaStream_t st = g_launch_stream; return launch_rnn_c0(c0, st); });
    plan.tag(C_ELEMWISE, 0.0, 0.0);
  }
}

static int ew_kind_of(int kind) {
  switch (kind) {
    case DG_OP_TANH: return EW_TANH;
    case DG_OP_LOGISTIC: return EW_LOGISTIC;
    case DG_OP_SCALAR_MUL: return EW_SCALE;
    case DG_OP_ADD: return EW_ADD;
    case DG_OP_CMULT: return EW_CMULT;
    default: return -1;
  }
}

// forward launches for one group; node values are already placed
// affine groups whose W operands are all (batch-1) parameters run on the
// shared-weight GEMM; anything else takes the generic per-node kernel
static bool affine_gemm_ok(const dg_graph* g, const Node& n0) {
  const int terms = (n0.n_in - 1) / 2;
  if (terms > 4) return false;
  for (int k = 0; k < terms; ++k) {
    const Node& w = g->nodes[g->inputs[n0.in_off + 1 + 2 * k]];
    if (w.kind != DG_OP_PARAMETER || w.batch != 1) return false;
  }
  return true;
}

static void plan_pnls2(dg_graph* g, const Schedule& S, const std::vector<int>& units, Plan& plan, bool bwd) {
  Blob& B = plan.blob;
  const int n = (int)units.size();
  std::vector<uintptr_t> vals((size_t)5 * n), grads(bwd ? (size_t)5 * n : 0);
  std::vector<int32_t> width((size_t)2 * n), label((size_t)2 * n);
  double bytes = 0;
  for (int j = 0; j < n; ++j) {
    const Unit& u = S.units[units[j]];
    const int slot[5] = {u.ins[0], u.ins[1], u.nodes[0], u.nodes[1], u.nodes[2]};
    for (int k = 0; k < 5; ++k) {
      vals[(size_t)k * n + j] = P(g->nodes[slot[k]].val);
      if (bwd) grads[(size_t)k * n + j] = P(g->nodes[slot[k]].grad);
    }
    for (int k = 0; k < 2; ++k) {
      width[2 * j + k] = (int32_t)g->nodes[u.ins[k]].elem;
      const Node& pn = g->nodes[u.nodes[k]];
      label[2 * j + k] = (int32_t)g->aux_i[pn.ai_off];
      bytes += 4.0 * width[2 * j + k] * (bwd ? 3 : 1);
    }
  }
  const size_t ov = B.push(vals), ow = B.push(width), ol = B.push(label);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < 2; ++k) rec_ids(S.units[units[j]].nodes[k], 0, 4, ol + 4 * (size_t)(2 * j + k));
  const size_t og = bwd ? B.push(grads) : 0;
  Pnls2Args a{};
  a.n = n;
  plan.ops.push_back([a, ov, ow, ol, og, bwd](char* d) mutable {
    a.val = at<const float* const>(d, ov);
    a.width = at<const int>(d, ow);
    a.label = at<const int>(d, ol);
    if (!bwd) return launch_pnls2_fwd(a, g_launch_stream);
    a.grad = at<float* const>(d, og);
    return launch_pnls2_bwd(a, g_launch_stream);
  });
  plan.tag(bwd ? C_PNLS_BWD : C_PNLS_FWD, 0.0, bytes);
}

static GruArgs gru_args(const dg_graph* g, const Unit& u0, int n) {
  GruArgs a{};
  a.n = n;
  a.H = u0.H;
  a.gw = u0.gw;
  a.off0 = u0.off[0];
  a.off1 = u0.off[1];
  a.off2 = u0.off[2];
  const bool part_b = u0.type == U_GRUB;
  a.batch = g->nodes[u0.nodes.back()].batch;
  const int hslot = part_b ? 4 : 2;
  a.h_b1 = g->nodes[u0.ins[hslot]].batch == 1 && a.batch > 1;
  a.ones_b1 = part_b && g->nodes[u0.ins[3]].batch == 1 && a.batch > 1;
  a.nslot = part_b ? 13 : 9;
  return a;
}

// A gate-affine group immediately followed by the gated-cell group that
// consumes it (a Tree-LSTM level, its leaves, unchained LSTM cells): one
// fused launch (cellgemm.cu) when the level is small -- the generic path
// is a grouped GEMM plus cell_fwd_kernel, two launches whose dependent memory
// round trips dominate at a few rows.  Returns false (nothing planned) when
// the pair does not qualify.
// Checks one (affine, cell) level and fills A; with a plan, also pushes the
// level's row / slot tables into its blob (device pointers in A).
static bool affine_cell_level(dg_graph* g, const Schedule& S, size_t q, Plan* plan, AffCellArgs& A) {
  static const bool on = [] {
    const char* e = std::getenv("DG_AFFCELL");
    return !(e && e[0] == '0');
  }();
  if (!on || q + 1 >= S.groups.size()) return false;
  const Group& ga = S.groups[q];
  const Group& gc = S.groups[q + 1];
  if (ga.kind != DG_OP_AFFINE || gc.kind != -2 || ga.units.size() != gc.units.size()) return false;
  const int n = (int)gc.units.size();
  const Unit& c0 = S.units[gc.units[0]];
  const Node& a0 = g->nodes[S.units[ga.units[0]].last()];
  const int terms = (a0.n_in - 1) / 2;
  const int Bt = a0.batch;
  const int rows = n * Bt;
  if (terms < 1 || terms > kAffCellMaxTerms || c0.m > 2 || c0.H <= 0 || c0.gw != (int)a0.elem || c0.gw % c0.H)
    return false;
  if (rows > 64) return false;
  for (int k = 0; k < 3 + c0.m; ++k)
    if (c0.off[k] % c0.H) return false;
  // cell j <-> affine node: the cell's gate input
  std::unordered_map<int, int> pos;
  for (int j = 0; j < n; ++j) pos[S.units[ga.units[j]].last()] = j;
  std::vector<int> aff(n);
  for (int j = 0; j < n; ++j) {
    const Unit& cu = S.units[gc.units[j]];
    auto it = pos.find(cu.ins[0]);
    if (it == pos.end()) return false;
    aff[j] = S.units[ga.units[it->second]].last();
    if (g->nodes[cu.ins[0]].batch != Bt) return false;
    for (int k = 0; k < cu.m; ++k)
      if (g->nodes[cu.ins[1 + k]].batch != Bt) return false;  // no broadcast external c
  }
  // shared parameters: the same bias row and weights in every member
  const Node& b0 = g->nodes[g->inputs[a0.in_off]];
  if (b0.kind != DG_OP_PARAMETER || b0.batch != 1) return false;
  A = AffCellArgs{};
  int kp = 0;
  for (int t = 0; t < terms; ++t) {
    const Node& w = g->nodes[g->inputs[a0.in_off + 1 + 2 * t]];
    const Node& x = g->nodes[g->inputs[a0.in_off + 2 + 2 * t]];
    if (w.kind != DG_OP_PARAMETER || w.batch != 1) return false;
    A.W[t] = w.val;
    A.K[t] = (int)x.elem;
    A.koff[t] = kp;
    kp += (A.K[t] + 3) & ~3;
  }
  for (int j = 0; j < n; ++j) {
    const Node& aj = g->nodes[aff[j]];
    if (aj.n_in != a0.n_in || aj.batch != Bt || g->nodes[g->inputs[aj.in_off]].val != b0.val) return false;
    for (int t = 0; t < terms; ++t)
      if (g->nodes[g->inputs[aj.in_off + 1 + 2 * t]].val != A.W[t]) return false;
  }
  A.kpad = kp;
  if (affine_cell_smem(rows, kp, c0.gw, c0.H) > 200 * 1024) return false;
  A.rows = rows;
  A.terms = terms;
  A.bias = b0.val;
  CellArgs& a = A.cell;
  a.n = n;
  a.m = c0.m;
  a.H = c0.H;
  a.gw = c0.gw;
  a.batch = Bt;
  a.off_i = c0.off[0];
  a.off_o = c0.off[1];
  a.off_g = c0.off[2];
  for (int k = 0; k < c0.m; ++k) a.off_f[k] = c0.off[3 + k];
  a.nslot = 10 + 5 * c0.m;
  if (!plan) return true;
  Blob& B = plan->blob;
  for (int t = 0; t < terms; ++t) {
    std::vector<uintptr_t> xr((size_t)rows);
    for (int j = 0; j < n; ++j) {
      const Node& x = g->nodes[g->inputs[g->nodes[aff[j]].in_off + 2 + 2 * t]];
      for (int b = 0; b < Bt; ++b) xr[(size_t)j * Bt + b] = P(x.val + (x.batch == 1 ? 0 : (int64_t)b * A.K[t]));
    }
    A.x[t] = dev_at<const float*>(g, B.push(xr));
  }
  std::vector<uintptr_t> vals((size_t)a.nslot * n);
  for (int j = 0; j < n; ++j) {
    const Unit& u = S.units[gc.units[j]];
    int sl = 0;
    for (int x : u.ins) vals[(size_t)(sl++) * n + j] = P(g->nodes[x].val);
    for (int x : u.nodes) vals[(size_t)(sl++) * n + j] = P(g->nodes[x].val);
  }
  a.val = dev_at<const float*>(g, B.push(vals));
  return true;
}

// A small affine / matmul level followed by its activation group (simple
// RNN steps: tanh(affine(b, Wx, x, Wh, h)), builders.py:90-91) or a
// concatenate -> matmul -> tanh level (TreeRNN compose: tanh(matmul(W,
// concatenate([e1, e2]))), builders.py:183-210): the same fused launch as a
// gated-cell level, the activation in place of the cell.  Fills A (and, with
// a plan, pushes its tables); returns the number of groups it covers.
static size_t act_level(dg_graph* g, const Schedule& S, size_t q, Plan* plan, AffCellArgs& A) {
  static const bool on = [] {
    const char* e = std::getenv("DG_AFFCELL");
    return !(e && e[0] == '0');
  }();
  if (!on || q + 1 >= S.groups.size()) return 0;
  const Group& g0 = S.groups[q];
  const bool tree = g0.kind == DG_OP_CONCATENATE;
  if (g0.kind != DG_OP_AFFINE && !tree) return 0;
  if (tree && q + 2 >= S.groups.size()) return 0;
  const Group& gm = tree ? S.groups[q + 1] : g0;  // the affine / matmul group
  const Group& gt = S.groups[q + (tree ? 2 : 1)];
  if (tree && gm.kind != DG_OP_MATMUL) return 0;
  if (gt.kind != DG_OP_TANH && gt.kind != DG_OP_LOGISTIC) return 0;
  const int n = (int)gt.units.size();
  if ((int)gm.units.size() != n || (int)g0.units.size() != n) return 0;
  std::unordered_map<int, int> mpos, cpos;
  for (int j = 0; j < n; ++j) mpos[S.units[gm.units[j]].last()] = j;
  if (tree)
    for (int j = 0; j < n; ++j) cpos[S.units[g0.units[j]].last()] = j;
  std::vector<int> mm(n), act(n), cat(n, -1);
  for (int j = 0; j < n; ++j) {
    act[j] = S.units[gt.units[j]].last();
    auto it = mpos.find(g->inputs[g->nodes[act[j]].in_off]);
    if (it == mpos.end()) return 0;
    mm[j] = S.units[gm.units[it->second]].last();
    if (tree) {
      auto ic = cpos.find(g->inputs[g->nodes[mm[j]].in_off + 1]);
      if (ic == cpos.end()) return 0;
      cat[j] = S.units[g0.units[ic->second]].last();
    }
  }
  const Node& m0 = g->nodes[mm[0]];
  const int Bt = m0.batch, gw = (int)m0.elem, rows = n * Bt;
  if (m0.rank != 1 || rows > 64 || gw <= 0) return 0;
  A = AffCellArgs{};
  int kp = 0, terms = 0;
  if (!tree) {
    terms = (m0.n_in - 1) / 2;
    if (terms < 1 || terms > kAffCellMaxTerms) return 0;
    const Node& b0 = g->nodes[g->inputs[m0.in_off]];
    if (b0.kind != DG_OP_PARAMETER || b0.batch != 1) return 0;
    A.bias = b0.val;
    for (int t = 0; t < terms; ++t) {
      const Node& w = g->nodes[g->inputs[m0.in_off + 1 + 2 * t]];
      if (w.kind != DG_OP_PARAMETER || w.batch != 1) return 0;
      A.W[t] = w.val;
      A.K[t] = (int)g->nodes[g->inputs[m0.in_off + 2 + 2 * t]].elem;
    }
  } else {
    const Node& w = g->nodes[g->inputs[m0.in_off]];
    const Node& c0 = g->nodes[cat[0]];
    if (w.kind != DG_OP_PARAMETER || w.batch != 1 || w.rank != 2 || c0.rank != 1) return 0;
    terms = c0.n_in;
    if (terms < 1 || terms > kAffCellMaxTerms) return 0;
    int k0 = 0;
    for (int t = 0; t < terms; ++t) {  // W [e1; e2] = W[:, part 1] e1 + W[:, part 2] e2
      const Node& x = g->nodes[g->inputs[c0.in_off + t]];
      if (x.rank != 1) return 0;
      A.W[t] = w.val + (int64_t)k0 * gw;
      A.K[t] = (int)x.elem;
      k0 += A.K[t];
    }
    if (k0 != (int)c0.elem) return 0;
  }
  for (int t = 0; t < terms; ++t) {
    A.koff[t] = kp;
    kp += (A.K[t] + 3) & ~3;
  }
  for (int j = 0; j < n; ++j) {  // same parameters and shapes in every member
    const Node& mj = g->nodes[mm[j]];
    if (mj.n_in != m0.n_in || mj.batch != Bt || mj.elem != m0.elem || g->nodes[act[j]].batch != Bt) return 0;
    if (!tree) {
      if (g->nodes[g->inputs[mj.in_off]].val != A.bias) return 0;
      for (int t = 0; t < terms; ++t)
        if (g->nodes[g->inputs[mj.in_off + 1 + 2 * t]].val != A.W[t]) return 0;
    } else {
      const Node& cj = g->nodes[cat[j]];
      if (g->nodes[g->inputs[mj.in_off]].val != A.W[0] || cj.n_in != terms || cj.batch != Bt) return 0;
      for (int t = 0; t < terms; ++t)
        if (g->nodes[g->inputs[cj.in_off + t]].elem != A.K[t] || g->nodes[g->inputs[cj.in_off + t]].batch != Bt)
          return 0;
    }
  }
  A.kpad = kp;
  if (affine_cell_smem(rows, kp, gw, gw) > 200 * 1024) return 0;
  A.rows = rows;
  A.terms = terms;
  A.act = gt.kind == DG_OP_TANH ? 1 : 2;
  CellArgs& a = A.cell;
  a.n = n;
  a.H = gw;
  a.gw = gw;
  a.batch = Bt;
  a.nslot = 2;
  const size_t used = tree ? 3 : 2;
  if (!plan) return used;
  Blob& B = plan->blob;
  for (int t = 0; t < terms; ++t) {
    std::vector<uintptr_t> xr((size_t)rows);
    for (int j = 0; j < n; ++j) {
      const Node& x = tree ? g->nodes[g->inputs[g->nodes[cat[j]].in_off + t]]
                           : g->nodes[g->inputs[g->nodes[mm[j]].in_off + 2 + 2 * t]];
      for (int b = 0; b < Bt; ++b) xr[(size_t)j * Bt + b] = P(x.val + (x.batch == 1 ? 0 : (int64_t)b * A.K[t]));
    }
    A.x[t] = dev_at<const float*>(g, B.push(xr));
  }
  std::vector<uintptr_t> vals((size_t)2 * n);
  for (int j = 0; j < n; ++j) {
    vals[j] = P(g->nodes[mm[j]].val);
    vals[(size_t)n + j] = P(g->nodes[act[j]].val);
  }
  a.val = dev_at<const float*>(g, B.push(vals));
  if (tree) {
    const int kc = (int)g->nodes[cat[0]].elem;
    std::vector<uintptr_t> cr((size_t)rows);
    for (int j = 0; j < n; ++j)
      for (int b = 0; b < Bt; ++b) cr[(size_t)j * Bt + b] = P(g->nodes[cat[j]].val + (int64_t)b * kc);
    A.cat = dev_at<float*>(g, B.push(cr));
  }
  return used;
}

static double affine_cell_flops(const AffCellArgs& A) { return 2.0 * A.rows * A.cell.gw * A.kpad; }
static double affine_cell_bytes(const AffCellArgs& A) {
  return 4.0 * ((double)A.rows * A.kpad + (double)A.kpad * A.cell.gw + 14.0 * A.rows * A.cell.H);
}

static bool plan_affine_cell_fwd(dg_graph* g, const Schedule& S, size_t q, Plan& plan, GemmBatch& gb) {
  AffCellArgs A;
  if (!affine_cell_level(g, S, q, nullptr, A)) return false;
  flush_gemm(g, plan, gb);
  affine_cell_level(g, S, q, &plan, A);
  plan.ops.push_back([A](char*) { return launch_affine_cell_fwd(A, g_launch_stream); });
  plan.tag(C_GEMM_FWD, affine_cell_flops(A), affine_cell_bytes(A));
  return true;
}

// A run of >= 2 consecutive (affine, cell) levels with at most two weight
// sets and one hidden size (the leaves and compose levels of a Tree-LSTM):
// one cooperative launch for all of them (cellgemm.cu tree_fwd_kernel).
// Returns the number of groups consumed (0: not applicable).
static size_t plan_tree_fwd(dg_graph* g, const Schedule& S, size_t q, Plan& plan, GemmBatch& gb) {
  static const bool on = [] {
    const char* e = std::getenv("DG_TREE_PERSIST");
    return !(e && e[0] == '0');
  }();
  if (!on) return 0;
  std::vector<AffCellArgs> lv;
  TreeFwdArgs T{};
  size_t qq = q;
  for (;; qq += 2) {
    AffCellArgs A;
    if (!affine_cell_level(g, S, qq, nullptr, A)) break;
    if (!lv.empty() && A.cell.H != lv[0].cell.H) break;
    int w = -1;
    for (int k = 0; k < T.n_wsets; ++k) {
      const AffCellArgs& W = T.wset[k];
      bool same = W.terms == A.terms && W.cell.gw == A.cell.gw && W.kpad == A.kpad && W.bias == A.bias;
      for (int t = 0; t < A.terms && same; ++t) same = W.W[t] == A.W[t] && W.K[t] == A.K[t] && W.koff[t] == A.koff[t];
      if (same) w = k;
    }
    if (w < 0) {
      if (T.n_wsets == 2) break;
      w = T.n_wsets++;
      T.wset[w] = A;
      T.wfloats[w] = (A.cell.gw / A.cell.H) * kAffCellUnits * A.kpad;
    }
    A.wslot = w;
    T.max_rows = std::max(T.max_rows, A.rows);
    lv.push_back(A);
    if (tree_fwd_smem(T) > 200 * 1024) {
      lv.pop_back();
      break;
    }
  }
  // cooperative launch: one CTA per kAffCellUnits units, all co-resident
  if (lv.size() < 2 || (lv[0].cell.H + kAffCellUnits - 1) / kAffCellUnits > kSmCount) return 0;
  flush_gemm(g, plan, gb);
  double flops = 0, bytes = 0;
  for (size_t l = 0; l < lv.size(); ++l) {
    affine_cell_level(g, S, q + 2 * l, &plan, lv[l]);
    lv[l].wslot = (lv[l].cell.gw == T.wset[0].cell.gw && lv[l].W[0] == T.wset[0].W[0]) ? 0 : 1;
    flops += affine_cell_flops(lv[l]);
    bytes += affine_cell_bytes(lv[l]);
  }
  T.H = lv[0].cell.H;
  T.n_levels = (int)lv.size();
  T.levels = dev_at<AffCellArgs>(g, plan.blob.push(lv));
  plan.ops.push_back([T](char*) { return launch_tree_fwd(T, g_launch_stream); });
  plan.tag(C_GEMM_FWD, flops, bytes);
  return 2 * lv.size();
}

static void plan_forward_group(dg_graph* g, const Schedule& S, const Group& gr, Plan& plan, GemmBatch& gb) {
  Blob& B = plan.blob;
  std::vector<int> nodes;
  for (int u : gr.units) nodes.push_back(S.units[u].last());
  const int n = (int)nodes.size();
  const Node& n0 = g->nodes[nodes[0]];
  if (!(gr.kind == DG_OP_AFFINE && affine_gemm_ok(g, n0))) flush_gemm(g, plan, gb);

  if (gr.kind == -3) {  // persistent LSTM stacks
    plan_rnn_group(g, S, gr, plan, false, nullptr, nullptr, &gb);
    return;
  }
  if (gr.kind == -6) {  // class-factored softmax terms
    plan_pnls2(g, S, gr.units, plan, false);
    return;
  }
  if (gr.kind == -4 || gr.kind == -5) {  // fused GRU parts
    const Unit& u0 = S.units[gr.units[0]];
    GruArgs a = gru_args(g, u0, n);
    std::vector<uintptr_t> vals((size_t)a.nslot * n);
    for (int j = 0; j < n; ++j) {
      const Unit& u = S.units[gr.units[j]];
      int s = 0;
      for (int x : u.ins) vals[(size_t)(s++) * n + j] = P(g->nodes[x].val);
      for (int x : u.nodes) vals[(size_t)(s++) * n + j] = P(g->nodes[x].val);
    }
    const size_t ov = B.push(vals);
    const bool part_b = gr.kind == -5;
    plan.ops.push_back([a, ov, part_b](char* d) mutable {
      a.val = at<const float* const>(d, ov);
      return launch_gru_fwd(a, part_b, g_launch_stream);
    });
    plan.tag(C_ELEMWISE, 0.0, 4.0 * n * (double)a.batch * a.H * (part_b ? 13 : 9));
    return;
  }
  if (gr.kind == -2) {  // fused gated cells
    const Unit& u0 = S.units[gr.units[0]];
    CellArgs a{};
    a.n = n;
    a.m = u0.m;
    a.H = u0.H;
    a.gw = u0.gw;
    a.batch = g->nodes[u0.ins[0]].batch;
    a.off_i = u0.off[0];
    a.off_o = u0.off[1];
    a.off_g = u0.off[2];
    for (int k = 0; k < u0.m; ++k) {
      a.off_f[k] = u0.off[3 + k];
      a.cext_b1[k] = g->nodes[u0.ins[1 + k]].batch == 1 && a.batch > 1;
    }
    a.nslot = 10 + 5 * u0.m;
    std::vector<uintptr_t> vals((size_t)a.nslot * n);
    for (int j = 0; j < n; ++j) {
      const Unit& u = S.units[gr.units[j]];
      int s = 0;
      for (int x : u.ins) vals[(size_t)(s++) * n + j] = P(g->nodes[x].val);
      for (int x : u.nodes) vals[(size_t)(s++) * n + j] = P(g->nodes[x].val);
    }
    const size_t ov = B.push(vals);
    plan.ops.push_back([a, ov](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
      a.val = at<const float* const>(d, ov);
      return launch_cell_fwd(a, st);
    });
    plan.tag(C_ELEMWISE, 0.0, 4.0 * n * (double)a.batch * a.H * (3 + a.m + 2.0 * (9 + 5 * a.m)));
    return;
  }
  if (gr.kind == -1) {  // add chain
    const int len = (int)S.units[gr.units[0]].nodes.size();
    std::vector<uintptr_t> ins((len + 1) * n), outs(len * n);
    for (int j = 0; j < n; ++j) {
      const Unit& u = S.units[gr.units[j]];
      for (int i = 0; i <= len; ++i) ins[i * n + j] = P(g->nodes[u.ins[i]].val);
      for (int i = 0; i < len; ++i) outs[i * n + j] = P(g->nodes[u.nodes[i]].val);
    }
    const size_t oi = B.push(ins), oo = B.push(outs);
    ChainArgs a{};
    a.n = n;
    a.len = len;
    a.size = (int)n0.size();
    plan.ops.push_back([a, oi, oo](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
      a.ins = at<const float* const>(d, oi);
      a.outs = at<float* const>(d, oo);
      return launch_chain_fwd(a, st);
    });
    return;
  }

  auto in_vals = [&](int slot) {
    std::vector<uintptr_t> v(n);
    for (int j = 0; j < n; ++j) v[j] = P(g->nodes[g->inputs[g->nodes[nodes[j]].in_off + slot]].val);
    return v;
  };
  std::vector<uintptr_t> outs(n);
  for (int j = 0; j < n; ++j) outs[j] = P(g->nodes[nodes[j]].val);
  const Node& in0 = g->nodes[g->inputs[n0.in_off]];

  switch (gr.kind) {
    case DG_OP_TANH:
    case DG_OP_LOGISTIC:
    case DG_OP_SCALAR_MUL:
    case DG_OP_ADD:
    case DG_OP_CMULT: {
      EwArgs a{};
      a.kind = ew_kind_of(gr.kind);
      a.n = n;
      a.elem = (int)n0.elem;
      a.batch = n0.batch;
      a.scalar = gr.kind == DG_OP_SCALAR_MUL ? g->aux_f[n0.af_off] : 0.f;
      a.a_b1 = (in0.batch == 1 && n0.batch > 1);
      const size_t oa = B.push(in_vals(0));
      size_t ob = 0;
      if (n0.n_in > 1) {
        a.b_b1 = (g->nodes[g->inputs[n0.in_off + 1]].batch == 1 && n0.batch > 1);
        ob = B.push(in_vals(1));
      }
      const size_t oo = B.push(outs);
      const bool binary = n0.n_in > 1;
      plan.ops.push_back([a, oa, ob, oo, binary](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
        a.a = at<const float* const>(d, oa);
        a.b = binary ? at<const float* const>(d, ob) : nullptr;
        a.out = at<float* const>(d, oo);
        return launch_ew_fwd(a, st);
      });
      plan.tag(C_ELEMWISE, 0.0, 4.0 * (double)n0.size() * n * (binary ? 3 : 2));
      return;
    }
    case DG_OP_PICK_RANGE: {
      PickArgs a{};
      a.n = n;
      a.batch = n0.batch;
      a.in_elem = (int)in0.elem;
      a.lo = (int)g->aux_i[n0.ai_off];
      a.width = (int)n0.elem;
      const size_t oi = B.push(in_vals(0)), oo = B.push(outs);
      plan.ops.push_back([a, oi, oo](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
        a.in = at<const float* const>(d, oi);
        a.out = at<float* const>(d, oo);
        return launch_pick_fwd(a, st);
      });
      return;
    }
    case DG_OP_CONCATENATE: {
      ConcatArgs a{};
      a.n = n;
      a.batch = n0.batch;
      a.parts = n0.n_in;
      a.total = (int)n0.elem;
      std::vector<int32_t> offs(a.parts + 1, 0);
      for (int k = 0; k < a.parts; ++k) offs[k + 1] = offs[k] + (int)g->nodes[g->inputs[n0.in_off + k]].elem;
      std::vector<uintptr_t> ins((size_t)a.parts * n);
      for (int k = 0; k < a.parts; ++k) {
        auto v = in_vals(k);
        std::copy(v.begin(), v.end(), ins.begin() + (size_t)k * n);
      }
      const size_t of = B.push(offs), oi = B.push(ins), oo = B.push(outs);
      plan.ops.push_back([a, of, oi, oo](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
        a.offs = at<const int>(d, of);
        a.in = at<const float* const>(d, oi);
        a.out = at<float* const>(d, oo);
        return launch_concat_fwd(a, st);
      });
      return;
    }
    case DG_OP_SUM_BATCHES: {
      SumBatchesArgs a{};
      a.n = n;
      a.batch = in0.batch;
      a.elem = (int)in0.elem;
      const size_t oi = B.push(in_vals(0)), oo = B.push(outs);
      plan.ops.push_back([a, oi, oo](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
        a.in = at<const float* const>(d, oi);
        a.out = at<float* const>(d, oo);
        return launch_sum_batches_fwd(a, st);
      });
      return;
    }
    case DG_OP_SOFTMAX:
    case DG_OP_PNLS:
    case DG_OP_PNLS_BATCH: {
      RowArgs a{};
      a.batch = in0.batch;
      a.rows = n * in0.batch;
      a.width = (int)in0.elem;
      const size_t oi = B.push(in_vals(0)), oo = B.push(outs);
      size_t ol = 0;
      const bool pnls = gr.kind != DG_OP_SOFTMAX;
      if (pnls) {
        std::vector<int32_t> labels;
        labels.reserve(a.rows);
        for (int j = 0; j < n; ++j) {
          const Node& x = g->nodes[nodes[j]];
          for (int64_t q = 0; q < x.ai_len; ++q) labels.push_back((int32_t)g->aux_i[x.ai_off + q]);
        }
        ol = B.push(labels);
        for (int j = 0, k = 0; j < n; k += (int)g->nodes[nodes[j]].ai_len, ++j) rec_ids(nodes[j], 0, 4, ol + 4 * k);
      }
      plan.ops.push_back([a, oi, oo, ol, pnls](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
        a.in = at<const float* const>(d, oi);
        a.out = at<float* const>(d, oo);
        if (pnls) {
          a.labels = at<const int>(d, ol);
          return launch_pnls_fwd(a, st);
        }
        return launch_softmax_fwd(a, st);
      });
      plan.tag(pnls ? C_PNLS_FWD : C_ELEMWISE, 0.0, (double)a.rows * a.width * 4 * (pnls ? 1 : 2));
      return;
    }
    case DG_OP_MATMUL: {
      const Node& x = g->nodes[g->inputs[n0.in_off + 1]];
      MatmulArgs a{};
      a.n = n;
      a.batch = n0.batch;
      a.m = in0.dims[0];
      a.k = in0.dims[1];
      a.p = x.rank == 1 ? 1 : x.dims[1];
      a.a_b1 = in0.batch == 1 && n0.batch > 1;
      a.x_b1 = x.batch == 1 && n0.batch > 1;
      const size_t oa = B.push(in_vals(0)), ox = B.push(in_vals(1)), oo = B.push(outs);
      plan.ops.push_back([a, oa, ox, oo](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
        a.a = at<const float* const>(d, oa);
        a.x = at<const float* const>(d, ox);
        a.out = at<float* const>(d, oo);
        return launch_matmul_fwd(a, st);
      });
      return;
    }
    case DG_OP_AFFINE: {
      const int terms = (n0.n_in - 1) / 2;
      const int m = (int)n0.elem;
      const int Bt = n0.batch;
      const bool gemm = affine_gemm_ok(g, n0);
      const Node& b0 = g->nodes[g->inputs[n0.in_off]];
      if (gemm) {
        GemmBatch& batch = gemm_batch_for(g, plan, gb, gr.level, C_GEMM_FWD, false, false);
        GemmProblem pr{};
        pr.M = n * Bt;
        pr.N = m;
        pr.n_seg = terms;
        pr.accumulate = 0;
        double kk = 0;
        for (int k = 0; k < terms; ++k) {
          const Node& xk0 = g->nodes[g->inputs[n0.in_off + 2 + 2 * k]];
          const int K = (int)xk0.elem;
          const bool xb1 = xk0.batch == 1 && Bt > 1;
          std::vector<uintptr_t> rows((size_t)n * Bt);
          for (int j = 0; j < n; ++j) {
            const float* xv = g->nodes[g->inputs[g->nodes[nodes[j]].in_off + 2 + 2 * k]].val;
            for (int b = 0; b < Bt; ++b) rows[(size_t)j * Bt + b] = P(xv + (xb1 ? 0 : (int64_t)b * K));
          }
          pr.seg[k].K = K;
          pr.seg[k].A.rows = dev_at<const float*>(g, B.push(rows));
          pr.seg[k].A.rows_aligned = all_aligned16(rows);
          // W column-major m x K == row-major K x m (W^T): B(k, n) = W[n + k*m]
          pr.seg[k].B.base = g->nodes[g->inputs[n0.in_off + 1 + 2 * k]].val;
          pr.seg[k].B.ld = m;
          kk += K;
        }
        std::vector<uintptr_t> crow((size_t)n * Bt);
        for (int j = 0; j < n; ++j)
          for (int b = 0; b < Bt; ++b) crow[(size_t)j * Bt + b] = P(g->nodes[nodes[j]].val + (int64_t)b * m);
        pr.C.rows = dev_at<const float*>(g, B.push(crow));
        pr.C.rows_aligned = all_aligned16(crow);
        // a parameter bias (same storage for every member, the signature keys
        // on its handle) is a single broadcast row; otherwise a row table
        if (b0.kind == DG_OP_PARAMETER) {
          pr.bias.base = b0.val;
          pr.bias.ld = 0;
        } else {
          const bool bb1 = b0.batch == 1 && Bt > 1;
          std::vector<uintptr_t> brow((size_t)n * Bt);
          for (int j = 0; j < n; ++j) {
            const float* bv = g->nodes[g->inputs[g->nodes[nodes[j]].in_off]].val;
            for (int b = 0; b < Bt; ++b) brow[(size_t)j * Bt + b] = P(bv + (bb1 ? 0 : (int64_t)b * m));
          }
          pr.bias.rows = dev_at<const float*>(g, B.push(brow));
        }
        batch.probs.push_back(pr);
        batch.bytes += 4.0 * ((double)pr.M * kk + kk * pr.N + (double)pr.M * pr.N);
      } else {
        AffineGenericArgs a{};
        a.n = n;
        a.batch = Bt;
        a.m = m;
        a.terms = terms;
        a.b_b1 = b0.batch == 1 && Bt > 1;
        std::vector<uintptr_t> w((size_t)terms * n), x((size_t)terms * n);
        for (int k = 0; k < terms && k < 8; ++k) {
          const Node& wk = g->nodes[g->inputs[n0.in_off + 1 + 2 * k]];
          const Node& xk = g->nodes[g->inputs[n0.in_off + 2 + 2 * k]];
          a.kdim[k] = (int)xk.elem;
          a.w_b1[k] = wk.batch == 1 && Bt > 1;
          a.x_b1[k] = xk.batch == 1 && Bt > 1;
          for (int j = 0; j < n; ++j) {
            const Node& nj = g->nodes[nodes[j]];
            w[(size_t)k * n + j] = P(g->nodes[g->inputs[nj.in_off + 1 + 2 * k]].val);
            x[(size_t)k * n + j] = P(g->nodes[g->inputs[nj.in_off + 2 + 2 * k]].val);
          }
        }
        const size_t ob = B.push(in_vals(0)), ow = B.push(w), ox = B.push(x), oo = B.push(outs);
        plan.ops.push_back([a, ob, ow, ox, oo](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
          a.bias = at<const float* const>(d, ob);
          a.w = at<const float* const>(d, ow);
          a.x = at<const float* const>(d, ox);
          a.out = at<float* const>(d, oo);
          return launch_affine_generic_fwd(a, st);
        });
      }
      return;
    }
    default:
      return;
  }
}

static int finish_forward(dg_graph* g, const Schedule& S, int lo, int upto, size_t cur, uint64_t pkey);

static int do_forward(dg_graph* g, int upto) {
  const int lo = g->watermark + 1;
  if (upto < lo) return DG_OK;
  // arena accounting first (arena.py:48-56): same rounded total as the
  // reference's per-node bump allocation, checked before any launch
  size_t need = 0;
  for (int i = lo; i <= upto; ++i) {
    const Node& x = g->nodes[i];
    if (x.kind == DG_OP_PARAMETER) continue;
    const size_t nb = (size_t)x.size() * 4;
    if (round64(nb) > g->fwd_bytes - g->fwd_cursor - need) {
      char buf[160];
      std::snprintf(buf, sizeof buf, "forward|%zu|%zu", nb, g->fwd_bytes - g->fwd_cursor - need);
      return fail(DG_POOL_EXHAUSTED, buf);
    }
    need += round64(nb);
  }

  PlanTimer tm("forward");
  NvtxRange nv_fwd("dg_forward");
  std::vector<int> active;
  active.reserve(upto - lo + 1);
  for (int i = lo; i <= upto; ++i) active.push_back(i);
  const std::shared_ptr<const Schedule> Sp = get_schedule(g, active, upto);
  const Schedule& S = *Sp;
  tm.lap("schedule");

  // placement: inputs first (one contiguous block filled by a single copy),
  // then lookups, then groups in execution order
  size_t cur = g->fwd_cursor;
  auto place = [&](int i) {
    Node& x = g->nodes[i];
    x.val = reinterpret_cast<float*>(g->fwd_base + cur);
    cur += round64((size_t)x.size() * 4);
  };
  for (int i : S.param_nodes) g->nodes[i].val = param_at(g->aux_i[g->nodes[i].ai_off])->val;
  const size_t in_begin = cur;
  for (int i : S.input_nodes) place(i);
  const size_t in_end = cur;
  for (int i : S.lookup_nodes) place(i);
  for (const Group& gr : S.groups)
    for (int u : gr.units)
      for (int i : S.units[u].nodes) place(i);

  const uint64_t pkey = plan_key(g, 0, lo, upto);
  if (CachedPlan* hit = plan_cache_find(g, 0, pkey)) {
    // same structure as an earlier graph: its plan with this graph's data
    Plan tail;
    int rc = blob_attach(tail.blob, hit->tmpl.size());
    if (rc) return rc;
    blob_from_template(g, *hit, tail.blob);
    tm.lap("cached");
    rc = launch_cached(g, *hit, tail);
    if (rc) return rc;
    tm.lap("launch");
    return finish_forward(g, S, lo, upto, cur, pkey);
  }
  PatchRec rec;
  RecScope rec_scope(&rec);
  Plan plan;
  {
    const int rc0 = blob_attach(plan.blob, g->blob_hint[0]);  // no regrowth copies while planning
    if (rc0) return rc0;
  }
  Blob& B = plan.blob;
  // input payloads: laid out in the blob exactly like the arena block
  size_t in_blob = 0;
  if (in_end > in_begin) {
    std::vector<uint8_t> block(in_end - in_begin, 0);
    for (int i : S.input_nodes) {
      const Node& x = g->nodes[i];
      const size_t off = reinterpret_cast<char*>(x.val) - (g->fwd_base + in_begin);
      std::memcpy(block.data() + off, g->aux_f.data() + x.af_off, (size_t)x.size() * 4);
    }
    in_blob = B.push_bytes(block.data(), block.size(), 64);
    for (int i : S.input_nodes)
      rec_payload(i, in_blob + (reinterpret_cast<char*>(g->nodes[i].val) - (g->fwd_base + in_begin)),
                  (size_t)g->nodes[i].size() * 4);
    char* dst = g->fwd_base + in_begin;
    const size_t nbytes = in_end - in_begin;
    plan.ops.push_back([dst, in_blob, nbytes](char* d) {
      const cudaStream_t st = g_launch_stream;
      return cudaMemcpyAsync(dst, d + in_blob, nbytes, cudaMemcpyDeviceToDevice, st) == cudaSuccess ? 0 : -1;
    });
  }
  // lookups: one gather per table
  {
    std::unordered_map<int64_t, std::pair<std::vector<int64_t>, std::vector<uintptr_t>>> by_table;
    std::unordered_map<int64_t, std::vector<int>> nodes_of;
    std::vector<int64_t> order;
    for (int i : S.lookup_nodes) {
      const Node& x = g->nodes[i];
      const int64_t h = g->aux_i[x.ai_off];
      nodes_of[h].push_back(i);
      auto it = by_table.find(h);
      if (it == by_table.end()) {
        order.push_back(h);
        it = by_table.emplace(h, std::make_pair(std::vector<int64_t>{}, std::vector<uintptr_t>{})).first;
      }
      const int64_t dim = x.elem;
      for (int64_t q = 1; q < x.ai_len; ++q) {
        it->second.first.push_back(g->aux_i[x.ai_off + q]);
        it->second.second.push_back(P(x.val + (q - 1) * dim));
      }
    }
    for (int64_t h : order) {
      Param* p = param_at(h);
      auto& pr = by_table[h];
      const size_t oid = B.push(pr.first), orow = B.push(pr.second);
      {
        size_t k = 0;
        for (int i : nodes_of[h]) {
          rec_ids(i, 1, 8, oid + 8 * k);
          k += (size_t)g->nodes[i].ai_len - 1;
        }
      }
      const float* table = p->val;
      const int dim = (int)p->cols;
      const int rows = (int)pr.first.size();
      plan.ops.push_back([table, dim, oid, orow, rows](char* d) {
      const cudaStream_t st = g_launch_stream;
        return launch_gather_rows(table, dim, at<const int64_t>(d, oid), at<float* const>(d, orow), rows, st);
      });
      plan.tag(C_GATHER, 0.0, 8.0 * rows * dim + 8.0 * rows);
    }
  }
  tm.lap("place+inputs");
  {
    GemmBatch gb;
    for (size_t q = 0; q < S.groups.size(); ++q) {
      if (const size_t used = plan_tree_fwd(g, S, q, plan, gb)) {
        q += used - 1;  // every level of the run went into one launch
        continue;
      }
      {
        AffCellArgs A;
        if (const size_t used = act_level(g, S, q, nullptr, A)) {
          flush_gemm(g, plan, gb);
          act_level(g, S, q, &plan, A);
          plan.ops.push_back([A](char*) { return launch_affine_cell_fwd(A, g_launch_stream); });
          plan.tag(C_GEMM_FWD, affine_cell_flops(A), affine_cell_bytes(A));
          q += used - 1;
          continue;
        }
      }
      if (plan_affine_cell_fwd(g, S, q, plan, gb)) {
        ++q;  // the cell group went into the same launch
        continue;
      }
      plan_forward_group(g, S, S.groups[q], plan, gb);
    }
    flush_gemm(g, plan, gb);
  }
  tm.lap("groups");
  g->blob_hint[0] = std::max(g->blob_hint[0], plan.blob.size() + plan.blob.size() / 4);
  int64_t launched = 0;
  int rc = launch_plan(g, plan, &launched);
  if (rc) return rc;
  tm.lap("launch");
  plan_cache_store(g, 0, pkey, plan, plan.ops.size(), plan.blob.size(), std::move(rec), launched);
  return finish_forward(g, S, lo, upto, cur, pkey);
}

// bookkeeping after a forward's launches (planned or cached)
static int finish_forward(dg_graph* g, const Schedule& S, int lo, int upto, size_t cur, uint64_t pkey) {
  {
    const Node& tn = g->nodes[upto];
    g->vcache_node = -1;
    if (tn.kind != DG_OP_PARAMETER && tn.size() <= 64 && !dry_run()) {
      if (!g->vcache) {
        // slots of one process-wide pinned block (cudaHostAlloc synchronises
        // the device, so it must not run per graph)
        static std::mutex mu;
        static float* block = nullptr;
        static int next = 0;
        std::lock_guard<std::mutex> lk(mu);
        if (!block) DG_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&block), 4096 * 64 * sizeof(float), 0));
        g->vcache = block + 64 * (next++ % 4096);
        DG_CUDA_TRY(cudaEventCreateWithFlags(&g->vcache_ev, cudaEventDisableTiming));
      }
      DG_CUDA_TRY(cudaMemcpyAsync(g->vcache, tn.val, (size_t)tn.size() * 4, cudaMemcpyDeviceToHost, g->stream));
      DG_CUDA_TRY(cudaEventRecord(g->vcache_ev, g->stream));
      g->vcache_node = upto;
      g->vcache_n = tn.size();
      g->d2h_bytes += tn.size() * 4;
    }
  }
  g->fwd_cursor = cur;
  g->fwd_alloc_count += (int64_t)(S.input_nodes.size() + S.lookup_nodes.size());
  for (const Group& gr : S.groups)
    for (int u : gr.units) g->fwd_alloc_count += (int64_t)S.units[u].nodes.size();
  g->forward_calls += upto - lo + 1;
  g->watermark = upto;
  g->stats[0] = (int64_t)S.groups.size();
  g->stats[1] = (int64_t)S.units.size();
  g->stats[2] = (int64_t)(upto - lo + 1);
  g->fwd_hist = mix64(g->fwd_hist, pkey);
  return DG_OK;
}

int dg_forward(dg_graph* g, int32_t upto) {
  if (upto >= (int)g->nodes.size()) return fail(DG_STALE, "node index out of range");
  return do_forward(g, upto);
}

// --------------------------------------------------------------- backward

// Backward of a small affine group (a few rows: the tree levels' gate
// affines, per-word layers): dX through affine_dx_small_kernel (weights staged
// before the dependency wait, one launch) instead of the grouped split-K GEMM;
// weight / bias gradients registered for the aggregated dW GEMM / column sums
// exactly as the affine's generic backward does.
static bool plan_affine_dx_small(dg_graph* g, const Schedule& S, const Group& ga, Plan& plan, GemmBatch& gb,
                                 std::unordered_map<int64_t, AffineUse>& wuse,
                                 std::unordered_map<int64_t, std::vector<uintptr_t>>& buse) {
  static const bool on = [] {
    const char* e = std::getenv("DG_AFFCELL");
    return !(e && e[0] == '0');
  }();
  if (!on || ga.kind != DG_OP_AFFINE) return false;
  const int n = (int)ga.units.size();
  const Node& a0 = g->nodes[S.units[ga.units[0]].last()];
  const int terms = (a0.n_in - 1) / 2;
  const int Bt = a0.batch;
  const int rows = n * Bt;
  const int gw = (int)a0.elem;
  if (terms < 1 || terms > kAffCellMaxTerms || rows > 64 || a0.rank != 1) return false;
  const Node& b0 = g->nodes[g->inputs[a0.in_off]];
  if (b0.kind != DG_OP_PARAMETER || b0.batch != 1) return false;
  AffCellArgs A{};
  int Ktot = 0;
  for (int t = 0; t < terms; ++t) {
    const Node& w = g->nodes[g->inputs[a0.in_off + 1 + 2 * t]];
    if (w.kind != DG_OP_PARAMETER || w.batch != 1) return false;
    A.W[t] = w.val;
    A.K[t] = (int)g->nodes[g->inputs[a0.in_off + 2 + 2 * t]].elem;
    Ktot += A.K[t];
  }
  std::vector<int> targets;
  for (int u : ga.units) {
    const Node& aj = g->nodes[S.units[u].last()];
    if (aj.n_in != a0.n_in || aj.batch != Bt || aj.elem != a0.elem || g->nodes[g->inputs[aj.in_off]].val != b0.val)
      return false;
    for (int t = 0; t < terms; ++t) {
      const int x = g->inputs[aj.in_off + 2 + 2 * t];
      if (g->nodes[g->inputs[aj.in_off + 1 + 2 * t]].val != A.W[t] || g->nodes[x].batch != Bt) return false;
      targets.push_back(x);
    }
  }
  std::sort(targets.begin(), targets.end());
  if (std::adjacent_find(targets.begin(), targets.end()) != targets.end()) return false;
  if (affine_dx_small_smem(rows, gw) > 200 * 1024 || Ktot < 1) return false;
  flush_gemm(g, plan, gb);
  Blob& B = plan.blob;
  A.rows = rows;
  A.terms = terms;
  A.cell.gw = gw;
  std::vector<uintptr_t> grows((size_t)rows);
  for (int j = 0; j < n; ++j) {
    const Node& aj = g->nodes[S.units[ga.units[j]].last()];
    for (int b = 0; b < Bt; ++b) grows[(size_t)j * Bt + b] = P(aj.grad + (int64_t)b * gw);
  }
  const size_t ogr = B.push(grows);
  std::vector<size_t> ogx(terms);
  for (int t = 0; t < terms; ++t) {
    const Node& wn = g->nodes[g->inputs[a0.in_off + 1 + 2 * t]];
    std::vector<uintptr_t> xrows((size_t)rows), dxrows((size_t)rows);
    for (int j = 0; j < n; ++j) {
      const Node& aj = g->nodes[S.units[ga.units[j]].last()];
      const Node& x = g->nodes[g->inputs[aj.in_off + 2 + 2 * t]];
      for (int b = 0; b < Bt; ++b) {
        xrows[(size_t)j * Bt + b] = P(x.val + (int64_t)b * A.K[t]);
        dxrows[(size_t)j * Bt + b] = P(x.grad + (int64_t)b * A.K[t]);
      }
    }
    ogx[t] = B.push(dxrows);
    AffineUse& use = wuse[g->aux_i[wn.ai_off]];
    use.n_in = A.K[t];
    use.m = gw;
    use.x_rows.insert(use.x_rows.end(), xrows.begin(), xrows.end());
    use.g_rows.insert(use.g_rows.end(), grows.begin(), grows.end());
  }
  {
    auto& v = buse[g->aux_i[b0.ai_off]];
    v.insert(v.end(), grows.begin(), grows.end());
  }
  plan.ops.push_back([A, ogx, ogr](char* d) mutable {
    A.grow = at<const float* const>(d, ogr);
    for (size_t t = 0; t < ogx.size(); ++t) A.gx[t] = at<float* const>(d, ogx[t]);
    return launch_affine_dx_small(A, g_launch_stream);
  });
  plan.tag(C_GEMM_DX, 2.0 * rows * gw * Ktot, 4.0 * ((double)Ktot * gw + 2.0 * rows * Ktot + (double)rows * gw));
  return true;
}

// The weight gradient of a large parameter whose every use is already
// registered (the output layer's W once its affine group is planned), run
// while the backward recurrence just planned occupies its clusters: the
// persistent TMA GEMM is launched right behind the recurrence with
// programmatic dependent launch, on at most the SMs the recurrence leaves
// free, and without waiting for it (it neither reads nor writes anything the
// recurrence touches; the recurrence started only after every earlier kernel
// completed).  The next launch goes without PDL, so it waits for both.
static int sm_count_host() {
  static const int n = [] {
    int d = 0, v = 0;
    if (cudaGetDevice(&d) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess)
      v = 148;
    return v > 0 ? v : 148;
  }();
  return n;
}

static bool early_dw_on() {
  static const bool on = [] {
    const char* e = std::getenv("DG_EARLY_DW");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool plan_early_dw(dg_graph* g, Plan& plan, const AffineUse& use, Param* p, int grid_cap) {
  Blob& B = plan.blob;
  GemmProblem pr{};
  pr.M = (int)use.n_in;
  pr.N = (int)use.m;
  pr.n_seg = 1;
  pr.accumulate = 1;
  pr.seg[0].K = (int64_t)use.x_rows.size();
  pr.seg[0].A.rows = dev_at<const float*>(g, B.push(use.x_rows));
  pr.seg[0].A.rows_aligned = all_aligned16(use.x_rows);
  pr.seg[0].B.rows = dev_at<const float*>(g, B.push(use.g_rows));
  pr.seg[0].B.rows_aligned = all_aligned16(use.g_rows);
  pr.C.base = p->grad;
  pr.C.ld = use.m;
  float* work = reinterpret_cast<float*>(scratch_base(g));
  const int64_t cap = (int64_t)(scratch_bytes(g) / 4);
  TmaGemmPlan tp;
  if (!tma_try(g, plan, pr, true, false, work, cap, &tp) || !tp.pers) return false;
  tp.args.nowait = 1;
  tp.grid_cap = grid_cap;
  plan.ops.push_back([tp](char*) { return launch_tma_gemm(tp, true, true, g_launch_stream); });
  plan.tag(C_GEMM_DW, tp.flops, 4.0 * ((double)pr.seg[0].K * (pr.M + pr.N) + 2.0 * pr.M * pr.N));
  plan.ops.push_back([](char*) {
    pdl_skip_next();
    return 0;
  });
  plan.tag(C_OTHER, 0.0, 0.0);
  return true;
}

// Work for the SMs the second backward recurrence leaves free: column sums
// of biases whose uses are all plain affine nodes already planned (the
// output bias) and weight gradients whose every use is registered (the upper
// LSTM layer's), launched behind the recurrence without waiting for it; the
// next launch goes without PDL.  Scratch: the column-sum partials first, the
// GEMMs' split-K workspace after them.
static void plan_window_work(dg_graph* g, Plan& plan, std::unordered_map<int64_t, AffineUse>& wuse,
                             std::unordered_map<int64_t, std::vector<uintptr_t>>& buse,
                             const std::unordered_map<int64_t, int64_t>& rows_all,
                             const std::unordered_map<int64_t, int64_t>& brows_all,
                             const std::unordered_map<int64_t, int64_t>& brows_plain) {
  Blob& B = plan.blob;
  const size_t at_op = plan.rnn_bwd_op, n_before = plan.ops.size();
  static const bool elog = std::getenv("DG_EARLY_DW_LOG") != nullptr;
  // DG_WINDOW: bit 0 column sums (default), bit 1 weight gradients too (the
  // lite TMA kernels co-reside with the recurrence's CTAs and slow it:
  // 0.950 -> 1.013 ms per PTB step)
  static const int mode = [] {
    const char* e = std::getenv("DG_WINDOW");
    return e ? std::atoi(e) : 1;
  }();
  // bias column sums (wide rows only: the pass that can skip the wait)
  std::vector<int64_t> bkeys;
  for (auto& kv : buse) bkeys.push_back(kv.first);
  std::sort(bkeys.begin(), bkeys.end());
  struct Job {
    float* dst;
    size_t orow;
    int nr, width;
  };
  std::vector<Job> jobs;
  int64_t cw = 0;
  double cbytes = 0;
  for (int64_t h : bkeys) {
    const auto& rows = buse[h];
    const auto pa = brows_all.find(h), pp = brows_plain.find(h);
    Param* p = param_at(h);
    const int width = (int)p->size();
    if (!(mode & 1) || pa == brows_all.end() || pp == brows_plain.end() || pa->second != pp->second ||
        (int64_t)rows.size() != pp->second || width % 4 || width < 1024 || !all_aligned16(rows) ||
        (int)jobs.size() == kColsumGroup)
      continue;
    jobs.push_back({p->grad, B.push(rows), (int)rows.size(), width});
    cw += (((int64_t)(rows.size() + 31) / 32) * width + 63) & ~int64_t(63);
    cbytes += 4.0 * rows.size() * width + 8.0 * width;
  }
  float* work = reinterpret_cast<float*>(scratch_base(g));
  const int64_t wcap = (int64_t)(scratch_bytes(g) / 4);
  if (!jobs.empty() && cw < wcap / 2) {
    for (const Job& j : jobs)
      for (int64_t h : bkeys)
        if (param_at(h)->grad == j.dst) buse.erase(h);
    plan.ops.push_back([jobs, work, cw](char* d) {
      ColsumGroup G{};
      G.n = (int)jobs.size();
      G.nowait = 1;
      for (int q = 0; q < G.n; ++q)
        G.j[q] = ColsumJob{jobs[q].dst, at<const float* const>(d, jobs[q].orow), jobs[q].nr, jobs[q].width, 0, 0, 0,
                           nullptr, 1};
      return launch_colsum_group(G, work, cw, g_launch_stream);
    });
    plan.tag(C_COLSUM, 0.0, cbytes);
    if (elog) std::fprintf(stderr, "[early-dw] window: %zu column sums\n", jobs.size());
  } else {
    cw = 0;
  }
  // weight gradients complete by now
  std::vector<int64_t> wkeys;
  for (auto& kv : wuse) wkeys.push_back(kv.first);
  std::sort(wkeys.begin(), wkeys.end());
  GemmBatch gb;
  gemm_batch_for(g, plan, gb, -1, C_GEMM_DW, true, false);
  gb.nowait = cw == 0;  // behind the column sums the GEMMs simply wait for them
  gb.temp_floats = cw;
  std::vector<int64_t> taken;
  for (int64_t h : wkeys) {
    const AffineUse& use = wuse[h];
    const auto pa = rows_all.find(h);
    if (!(mode & 2) || pa == rows_all.end() || (int64_t)use.x_rows.size() != pa->second ||
        use.n_in * use.m < ((int64_t)1 << 18))
      continue;
    GemmProblem pr{};
    pr.M = (int)use.n_in;
    pr.N = (int)use.m;
    pr.n_seg = 1;
    pr.accumulate = 1;
    pr.seg[0].K = (int64_t)use.x_rows.size();
    pr.seg[0].A.rows = dev_at<const float*>(g, B.push(use.x_rows));
    pr.seg[0].A.rows_aligned = all_aligned16(use.x_rows);
    pr.seg[0].B.rows = dev_at<const float*>(g, B.push(use.g_rows));
    pr.seg[0].B.rows_aligned = all_aligned16(use.g_rows);
    pr.C.base = param_at(h)->grad;
    pr.C.ld = use.m;
    gb.probs.push_back(pr);
    gb.bytes += 4.0 * ((double)pr.seg[0].K * (pr.M + pr.N) + 2.0 * pr.M * pr.N);
    taken.push_back(h);
  }
  if (!gb.probs.empty()) {
    flush_gemm(g, plan, gb);
    for (int64_t h : taken) wuse.erase(h);
    if (elog) std::fprintf(stderr, "[early-dw] window: %zu weight gradients\n", taken.size());
  }
  if (plan.ops.size() == n_before) return;
  plan.ops.push_back([](char*) {
    pdl_skip_next();
    return 0;
  });
  plan.tag(C_OTHER, 0.0, 0.0);
  plan.meta.resize(plan.ops.size());
  std::rotate(plan.ops.begin() + at_op, plan.ops.begin() + n_before, plan.ops.end());
  std::rotate(plan.meta.begin() + at_op, plan.meta.begin() + n_before, plan.meta.end());
}

static void plan_backward_group(dg_graph* g, const Schedule& S, const Group& gr, Plan& plan, float* dummy,
                                std::unordered_map<int64_t, AffineUse>& wuse,
                                std::unordered_map<int64_t, std::vector<uintptr_t>>& buse, GemmBatch& gb) {
  Blob& B = plan.blob;
  if (!(gr.kind == DG_OP_AFFINE && affine_gemm_ok(g, g->nodes[S.units[gr.units[0]].last()]))) flush_gemm(g, plan, gb);
  if (gr.kind == -3) {
    plan_rnn_group(g, S, gr, plan, true, &wuse, &buse, &gb);
    return;
  }
  std::vector<int> all_nodes;
  for (int u : gr.units) all_nodes.push_back(S.units[u].last());
  const Node& n0 = g->nodes[all_nodes[0]];

  // targets per member for conflict rounds
  std::vector<std::vector<int>> targets(gr.units.size());
  for (size_t j = 0; j < gr.units.size(); ++j) targets[j] = S.units[gr.units[j]].ins;
  const bool ew = gr.kind == DG_OP_ADD || gr.kind == DG_OP_CMULT || gr.kind == DG_OP_TANH ||
                  gr.kind == DG_OP_LOGISTIC || gr.kind == DG_OP_SCALAR_MUL || gr.kind == -1 || gr.kind == -2 ||
                  gr.kind == -4 || gr.kind == -5 || gr.kind == -6;
  if (gr.kind == DG_OP_AFFINE) {
    // dX is conflict-free by construction (temp + segmented reduce); only the
    // per-node (non-parameter) bias needs rounds
    // (a parameter bias is aggregated into one column sum, no conflict)
    for (size_t j = 0; j < targets.size(); ++j) {
      const int b = targets[j][0];
      if (g->nodes[b].kind == DG_OP_PARAMETER) targets[j].clear();
      else targets[j] = {b};
    }
  }
  auto rounds = conflict_rounds(targets, ew);
  // intra-node duplicate slots in non-elementwise kinds (e.g. concatenate([x,x]))
  bool intra_dup = false;
  if (!ew && gr.kind != DG_OP_AFFINE) {
    for (auto& t : targets) {
      std::vector<int> s = t;
      std::sort(s.begin(), s.end());
      if (std::adjacent_find(s.begin(), s.end()) != s.end()) intra_dup = true;
    }
  }

  for (const auto& mask : rounds) {
    std::vector<int> nodes;
    std::vector<int> units;
    for (size_t j = 0; j < all_nodes.size(); ++j)
      if (mask[j]) { nodes.push_back(all_nodes[j]); units.push_back(gr.units[j]); }
    const int n = (int)nodes.size();
    if (n == 0) continue;
    if (gr.kind == -6) {  // class-factored softmax terms
      plan_pnls2(g, S, units, plan, true);
      continue;
    }
    if (gr.kind == -4 || gr.kind == -5) {  // fused GRU parts
      const Unit& u0 = S.units[units[0]];
      GruArgs a = gru_args(g, u0, n);
      std::vector<uintptr_t> vals((size_t)a.nslot * n), grads((size_t)a.nslot * n);
      for (int j = 0; j < n; ++j) {
        const Unit& u = S.units[units[j]];
        int s = 0;
        for (int x : u.ins) {
          vals[(size_t)s * n + j] = P(g->nodes[x].val);
          grads[(size_t)(s++) * n + j] = P(g->nodes[x].grad);
        }
        for (int x : u.nodes) {
          vals[(size_t)s * n + j] = P(g->nodes[x].val);
          grads[(size_t)(s++) * n + j] = P(g->nodes[x].grad);
        }
      }
      const size_t ov = B.push(vals), og = B.push(grads);
      const bool part_b = gr.kind == -5;
      plan.ops.push_back([a, ov, og, part_b](char* d) mutable {
        a.val = at<const float* const>(d, ov);
        a.grad = at<float* const>(d, og);
        return launch_gru_bwd(a, part_b, g_launch_stream);
      });
      plan.tag(C_ELEMWISE, 0.0, 4.0 * n * (double)a.batch * a.H * (part_b ? 26 : 18));
      continue;
    }
    if (gr.kind == -2) {  // fused gated cells
      const Unit& u0 = S.units[units[0]];
      CellArgs a{};
      a.n = n;
      a.m = u0.m;
      a.H = u0.H;
      a.gw = u0.gw;
      a.batch = g->nodes[u0.ins[0]].batch;
      a.off_i = u0.off[0];
      a.off_o = u0.off[1];
      a.off_g = u0.off[2];
      for (int k = 0; k < u0.m; ++k) {
        a.off_f[k] = u0.off[3 + k];
        a.cext_b1[k] = g->nodes[u0.ins[1 + k]].batch == 1 && a.batch > 1;
      }
      a.nslot = 10 + 5 * u0.m;
      std::vector<uintptr_t> vals((size_t)a.nslot * n), grads((size_t)a.nslot * n);
      for (int j = 0; j < n; ++j) {
        const Unit& u = S.units[units[j]];
        int s = 0;
        for (int x : u.ins) {
          vals[(size_t)s * n + j] = P(g->nodes[x].val);
          grads[(size_t)(s++) * n + j] = P(g->nodes[x].grad);
        }
        for (int x : u.nodes) {
          vals[(size_t)s * n + j] = P(g->nodes[x].val);
          grads[(size_t)(s++) * n + j] = P(g->nodes[x].grad);
        }
      }
      const size_t ov = B.push(vals), og = B.push(grads);
      plan.ops.push_back([a, ov, og](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
        a.val = at<const float* const>(d, ov);
        a.grad = at<float* const>(d, og);
        return launch_cell_bwd(a, st);
      });
      plan.tag(C_ELEMWISE, 0.0, 4.0 * n * (double)a.batch * a.H * (6 + 2 * a.m + 2.0 * (9 + 5 * a.m)));
      continue;
    }
    // slot passes: with intra-node duplicates, one pass per slot with every
    // other slot's gradient redirected to a dummy buffer
    const int n_slots = n0.n_in;
    const int passes = intra_dup ? n_slots : 1;
    for (int pass = 0; pass < passes; ++pass) {
      auto gin = [&](int slot) {
        std::vector<uintptr_t> v(n);
        for (int j = 0; j < n; ++j) {
          const bool live = !intra_dup || slot == pass;
          v[j] = live ? P(g->nodes[g->inputs[g->nodes[nodes[j]].in_off + slot]].grad) : P(dummy);
        }
        return v;
      };
      auto inval = [&](int slot) {
        std::vector<uintptr_t> v(n);
        for (int j = 0; j < n; ++j) v[j] = P(g->nodes[g->inputs[g->nodes[nodes[j]].in_off + slot]].val);
        return v;
      };
      std::vector<uintptr_t> gout(n), oval(n);
      for (int j = 0; j < n; ++j) {
        gout[j] = P(g->nodes[nodes[j]].grad);
        oval[j] = P(g->nodes[nodes[j]].val);
      }
      const Node& in0 = g->nodes[g->inputs[n0.in_off]];
      switch (gr.kind) {
        case -1: {
          const int len = (int)S.units[units[0]].nodes.size();
          std::vector<uintptr_t> gins((size_t)(len + 1) * n), gouts((size_t)len * n);
          for (int j = 0; j < n; ++j) {
            const Unit& u = S.units[units[j]];
            for (int i = 0; i <= len; ++i) gins[(size_t)i * n + j] = P(g->nodes[u.ins[i]].grad);
            for (int i = 0; i < len; ++i) gouts[(size_t)i * n + j] = P(g->nodes[u.nodes[i]].grad);
          }
          ChainArgs a{};
          a.n = n;
          a.len = len;
          a.size = (int)n0.size();
          {
            std::vector<uintptr_t> all(gins);
            all.insert(all.end(), gouts.begin(), gouts.end());
            a.distinct = has_duplicate_rows(all) ? 0 : 1;
          }
          const size_t og = B.push(gout), ogi = B.push(gins), ogo = B.push(gouts);
          plan.ops.push_back([a, og, ogi, ogo](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
            a.gfinal = at<const float* const>(d, og);
            a.gins = at<float* const>(d, ogi);
            a.gouts = at<float* const>(d, ogo);
            return launch_chain_bwd(a, st);
          });
          break;
        }
        case DG_OP_TANH:
        case DG_OP_LOGISTIC:
        case DG_OP_SCALAR_MUL:
        case DG_OP_ADD:
        case DG_OP_CMULT: {
          EwArgs a{};
          a.kind = ew_kind_of(gr.kind);
          a.n = n;
          a.elem = (int)n0.elem;
          a.batch = n0.batch;
          a.scalar = gr.kind == DG_OP_SCALAR_MUL ? g->aux_f[n0.af_off] : 0.f;
          const bool binary = n0.n_in > 1;
          a.a_b1 = in0.batch == 1 && n0.batch > 1;
          a.b_b1 = binary && g->nodes[g->inputs[n0.in_off + 1]].batch == 1 && n0.batch > 1;
          const size_t oa = B.push(inval(0)), oga = B.push(gin(0));
          size_t ob = 0, ogb = 0;
          if (binary) {
            ob = B.push(inval(1));
            ogb = B.push(gin(1));
          }
          const size_t ogo = B.push(gout), oov = B.push(oval);
          plan.ops.push_back([a, oa, oga, ob, ogb, ogo, oov, binary](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
            a.a = at<const float* const>(d, oa);
            a.ga = at<float* const>(d, oga);
            if (binary) {
              a.b = at<const float* const>(d, ob);
              a.gb = at<float* const>(d, ogb);
            }
            a.gout = at<const float* const>(d, ogo);
            a.oval = at<const float* const>(d, oov);
            return launch_ew_bwd(a, st);
          });
          plan.tag(C_ELEMWISE, 0.0, 4.0 * (double)n0.size() * n * (binary ? 6 : 4));
          break;
        }
        case DG_OP_PICK_RANGE: {
          PickArgs a{};
          a.n = n;
          a.batch = n0.batch;
          a.in_elem = (int)in0.elem;
          a.lo = (int)g->aux_i[n0.ai_off];
          a.width = (int)n0.elem;
          const size_t og = B.push(gout), oi = B.push(gin(0));
          plan.ops.push_back([a, og, oi](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
            a.gout = at<const float* const>(d, og);
            a.gin = at<float* const>(d, oi);
            return launch_pick_bwd(a, st);
          });
          break;
        }
        case DG_OP_CONCATENATE: {
          ConcatArgs a{};
          a.n = n;
          a.batch = n0.batch;
          a.parts = n0.n_in;
          a.total = (int)n0.elem;
          std::vector<int32_t> offs(a.parts + 1, 0);
          for (int k = 0; k < a.parts; ++k) offs[k + 1] = offs[k] + (int)g->nodes[g->inputs[n0.in_off + k]].elem;
          std::vector<uintptr_t> gins((size_t)a.parts * n);
          for (int k = 0; k < a.parts; ++k) {
            auto v = gin(k);
            std::copy(v.begin(), v.end(), gins.begin() + (size_t)k * n);
          }
          const size_t of = B.push(offs), og = B.push(gout), oi = B.push(gins);
          plan.ops.push_back([a, of, og, oi](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
            a.offs = at<const int>(d, of);
            a.gout = at<const float* const>(d, og);
            a.gin = at<float* const>(d, oi);
            return launch_concat_bwd(a, st);
          });
          break;
        }
        case DG_OP_SUM_BATCHES: {
          SumBatchesArgs a{};
          a.n = n;
          a.batch = in0.batch;
          a.elem = (int)in0.elem;
          const size_t og = B.push(gout), oi = B.push(gin(0));
          plan.ops.push_back([a, og, oi](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
            a.gout = at<const float* const>(d, og);
            a.gin = at<float* const>(d, oi);
            return launch_sum_batches_bwd(a, st);
          });
          break;
        }
        case DG_OP_SOFTMAX:
        case DG_OP_PNLS:
        case DG_OP_PNLS_BATCH: {
          RowArgs a{};
          a.batch = in0.batch;
          a.rows = n * in0.batch;
          a.width = (int)in0.elem;
          const bool pnls = gr.kind != DG_OP_SOFTMAX;
          const int x0 = g->inputs[n0.in_off];
          a.overwrite = pnls && x0 < (int)g->bwd_overwrite.size() && g->bwd_overwrite[x0] ? 1 : 0;
          size_t ol = 0;
          if (pnls) {
            std::vector<int32_t> labels;
            for (int j = 0; j < n; ++j) {
              const Node& x = g->nodes[nodes[j]];
              for (int64_t q = 0; q < x.ai_len; ++q) labels.push_back((int32_t)g->aux_i[x.ai_off + q]);
            }
            ol = B.push(labels);
            for (int j = 0, k = 0; j < n; k += (int)g->nodes[nodes[j]].ai_len, ++j) rec_ids(nodes[j], 0, 4, ol + 4 * k);
          }
          const size_t oi = B.push(inval(0)), og = B.push(gout), ov = B.push(oval), ogi = B.push(gin(0));
          plan.ops.push_back([a, oi, og, ov, ogi, ol, pnls](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
            a.in = at<const float* const>(d, oi);
            a.gout = at<const float* const>(d, og);
            a.oval = at<const float* const>(d, ov);
            a.gin = at<float* const>(d, ogi);
            if (pnls) {
              a.labels = at<const int>(d, ol);
              return launch_pnls_bwd(a, st);
            }
            return launch_softmax_bwd(a, st);
          });
          // logits read + dlogits written (and read, when accumulated)
          plan.tag(pnls ? C_PNLS_BWD : C_ELEMWISE, 0.0, (double)a.rows * a.width * 4 * (a.overwrite ? 2 : 3));
          break;
        }
        case DG_OP_MATMUL: {
          const Node& x = g->nodes[g->inputs[n0.in_off + 1]];
          MatmulArgs a{};
          a.n = n;
          a.batch = n0.batch;
          a.m = in0.dims[0];
          a.k = in0.dims[1];
          a.p = x.rank == 1 ? 1 : x.dims[1];
          a.a_b1 = in0.batch == 1 && n0.batch > 1;
          a.x_b1 = x.batch == 1 && n0.batch > 1;
          const size_t oa = B.push(inval(0)), ox = B.push(inval(1)), og = B.push(gout);
          const size_t oga = B.push(gin(0)), ogx = B.push(gin(1));
          plan.ops.push_back([a, oa, ox, og, oga, ogx](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
            a.a = at<const float* const>(d, oa);
            a.x = at<const float* const>(d, ox);
            a.gout = at<const float* const>(d, og);
            a.ga = at<float* const>(d, oga);
            a.gx = at<float* const>(d, ogx);
            return launch_matmul_bwd(a, st);
          });
          break;
        }
        case DG_OP_AFFINE: {
          const int terms = (n0.n_in - 1) / 2;
          const int m = (int)n0.elem;
          const int Bt = n0.batch;
          if (!affine_gemm_ok(g, n0)) {
            AffineGenericArgs a{};
            a.n = n;
            a.batch = Bt;
            a.m = m;
            a.terms = terms;
            a.b_b1 = in0.batch == 1 && Bt > 1;
            std::vector<uintptr_t> w((size_t)terms * n), x((size_t)terms * n), gw((size_t)terms * n),
                gx((size_t)terms * n);
            for (int k = 0; k < terms && k < 8; ++k) {
              const Node& wk = g->nodes[g->inputs[n0.in_off + 1 + 2 * k]];
              const Node& xk = g->nodes[g->inputs[n0.in_off + 2 + 2 * k]];
              a.kdim[k] = (int)xk.elem;
              a.w_b1[k] = wk.batch == 1 && Bt > 1;
              a.x_b1[k] = xk.batch == 1 && Bt > 1;
              auto wv = inval(1 + 2 * k), xv = inval(2 + 2 * k), gwv = gin(1 + 2 * k), gxv = gin(2 + 2 * k);
              for (int j = 0; j < n; ++j) {
                w[(size_t)k * n + j] = wv[j];
                x[(size_t)k * n + j] = xv[j];
                gw[(size_t)k * n + j] = gwv[j];
                gx[(size_t)k * n + j] = gxv[j];
              }
            }
            const size_t ob = B.push(inval(0)), ow = B.push(w), ox = B.push(x), og = B.push(gout);
            const size_t ogb = B.push(gin(0)), ogw = B.push(gw), ogx = B.push(gx);
            plan.ops.push_back([a, ob, ow, ox, og, ogb, ogw, ogx](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
              a.bias = at<const float* const>(d, ob);
              a.w = at<const float* const>(d, ow);
              a.x = at<const float* const>(d, ox);
              a.gout = at<const float* const>(d, og);
              a.gbias = at<float* const>(d, ogb);
              a.gw = at<float* const>(d, ogw);
              a.gx = at<float* const>(d, ogx);
              return launch_affine_generic_bwd(a, st);
            });
            break;
          }
          // G rows of this round
          std::vector<uintptr_t> grows((size_t)n * Bt);
          for (int j = 0; j < n; ++j)
            for (int b = 0; b < Bt; ++b) grows[(size_t)j * Bt + b] = P(g->nodes[nodes[j]].grad + (int64_t)b * m);
          // bias
          const Node& b0 = in0;
          if (b0.kind == DG_OP_PARAMETER) {
            auto& v = buse[g->aux_i[b0.ai_off]];
            v.insert(v.end(), grows.begin(), grows.end());
          } else {
            EwArgs a{};
            a.kind = EW_SCALE;
            a.scalar = 1.f;
            a.n = n;
            a.elem = m;
            a.batch = Bt;
            a.a_b1 = b0.batch == 1 && Bt > 1;
            const size_t og = B.push(gout), oga = B.push(gin(0));
            plan.ops.push_back([a, og, oga](char* d) mutable {
      const cudaStream_t st = g_launch_stream;
              a.gout = at<const float* const>(d, og);
              a.ga = at<float* const>(d, oga);
              return launch_ew_bwd(a, st);
            });
          }
          const bool g_al = all_aligned16(grows);
          const float* const* g_rows_dev = dev_at<const float*>(g, B.push(grows));
          // a grouped launch must not write one target from two problems
          {
            std::vector<int> mine;
            for (int j = 0; j < n; ++j)
              for (int k = 0; k < terms; ++k) mine.push_back(g->inputs[g->nodes[nodes[j]].in_off + 2 + 2 * k]);
            std::sort(mine.begin(), mine.end());
            bool clash = false;
            for (int x : gb.targets) clash = clash || std::binary_search(mine.begin(), mine.end(), x);
            // terms of one member sharing an x also clash inside one launch
            for (int k = 0; k + 1 < terms && !clash; ++k)
              for (int k2 = k + 1; k2 < terms && !clash; ++k2)
                for (int j = 0; j < n && !clash; ++j)
                  clash = g->inputs[g->nodes[nodes[j]].in_off + 2 + 2 * k] ==
                          g->inputs[g->nodes[nodes[j]].in_off + 2 + 2 * k2];
            if (clash) flush_gemm(g, plan, gb);
          }
          GemmBatch& batch = gemm_batch_for(g, plan, gb, gr.level, C_GEMM_DX, false, true);
          for (int k = 0; k < terms; ++k) {
            const Node& wn = g->nodes[g->inputs[n0.in_off + 1 + 2 * k]];
            const Node& xk0 = g->nodes[g->inputs[n0.in_off + 2 + 2 * k]];
            const int K = (int)xk0.elem;
            const bool xb1 = xk0.batch == 1 && Bt > 1;
            std::vector<uintptr_t> xrows((size_t)n * Bt), dxrows((size_t)n * Bt);
            for (int j = 0; j < n; ++j) {
              const Node& xj = g->nodes[g->inputs[g->nodes[nodes[j]].in_off + 2 + 2 * k]];
              for (int b = 0; b < Bt; ++b) {
                xrows[(size_t)j * Bt + b] = P(xj.val + (xb1 ? 0 : (int64_t)b * K));
                dxrows[(size_t)j * Bt + b] = P(xj.grad + (xb1 ? 0 : (int64_t)b * K));
              }
            }
            // weight-gradient aggregation (one GEMM per parameter later)
            AffineUse& use = wuse[g->aux_i[wn.ai_off]];
            use.n_in = K;
            use.m = m;
            use.x_rows.insert(use.x_rows.end(), xrows.begin(), xrows.end());
            use.g_rows.insert(use.g_rows.end(), grows.begin(), grows.end());
            // dX = G W   (B(k=i, n=t) = W[i + t*m]: n-major rows of W^T)
            const bool dup = has_duplicate_rows(dxrows);
            GemmProblem pr{};
            pr.M = n * Bt;
            pr.N = K;
            pr.n_seg = 1;
            pr.seg[0].K = m;
            pr.seg[0].A.rows = g_rows_dev;
            pr.seg[0].A.rows_aligned = g_al;
            pr.seg[0].B.base = wn.val;
            pr.seg[0].B.ld = m;
            batch.bytes += 4.0 * ((double)pr.M * m + (double)m * pr.N + 2.0 * pr.M * pr.N);
            if (!dup) {
              pr.accumulate = 1;
              pr.C.rows = dev_at<const float*>(g, B.push(dxrows));
            } else {
              // several rows land on one target (broadcast x, or one x shared
              // by group members): temp = G W densely, then a deterministic
              // segmented row reduce into the targets
              const int64_t R = (int64_t)n * Bt;
              std::vector<int> order(R);
              std::iota(order.begin(), order.end(), 0);
              std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return dxrows[x] < dxrows[y]; });
              std::vector<uintptr_t> tgt;
              std::vector<int32_t> seg;
              for (int64_t q = 0; q < R; ++q) {
                if (q == 0 || dxrows[order[q]] != dxrows[order[q - 1]]) {
                  tgt.push_back(dxrows[order[q]]);
                  seg.push_back((int32_t)q);
                }
              }
              seg.push_back((int32_t)R);
              std::vector<int64_t> pos(R);
              for (int64_t q = 0; q < R; ++q) pos[order[q]] = q;
              float* temp = reinterpret_cast<float*>(scratch_base(g)) + batch.temp_floats;
              batch.temp_floats += (R * K + 63) & ~int64_t(63);
              std::vector<uintptr_t> crow(R);
              for (int64_t r = 0; r < R; ++r) crow[r] = P(temp + pos[r] * K);
              pr.accumulate = 0;
              pr.C.rows = dev_at<const float*>(g, B.push(crow));
              float* const* tg = const_cast<float* const*>(reinterpret_cast<const float* const*>(
                  dev_at<float*>(g, B.push(tgt))));
              const int* sg = dev_at<int>(g, B.push(seg));
              const int n_t = (int)tgt.size();
              batch.post.push_back([tg, sg, temp, n_t, K]() {
                const cudaStream_t st = g_launch_stream;
                return launch_row_reduce_scatter(tg, sg, temp, n_t, K, st);
              });
            }
            batch.probs.push_back(pr);
            for (int j = 0; j < n; ++j) batch.targets.push_back(g->inputs[g->nodes[nodes[j]].in_off + 2 + 2 * k]);
            // two terms of one member on the same x: keep them in separate launches
            if (k + 1 < terms) {
              bool same = false;
              for (int j = 0; j < n && !same; ++j)
                for (int k2 = k + 1; k2 < terms && !same; ++k2)
                  same = g->inputs[g->nodes[nodes[j]].in_off + 2 + 2 * k] ==
                         g->inputs[g->nodes[nodes[j]].in_off + 2 + 2 * k2];
              if (same) {
                flush_gemm(g, plan, gb);
                gemm_batch_for(g, plan, gb, gr.level, C_GEMM_DX, false, true);
              }
            }
          }
          break;
        }
        default:
          break;
      }
    }
  }
}

int dg_backward(dg_graph* g, int32_t loss) {
  if (loss < 0 || loss >= (int)g->nodes.size()) return fail(DG_STALE, "loss index out of range");
  {
    const Node& L = g->nodes[loss];
    if (L.elem != 1 || L.batch != 1) return fail(DG_NON_SCALAR_LOSS, "backward needs a scalar");
  }
  int rc = do_forward(g, loss);
  if (rc) return rc;

  // slots for every node <= loss (graph.py:149-150): identical accounting
  size_t need = 0;
  for (int i = 0; i <= loss; ++i) {
    const size_t nb = (size_t)g->nodes[i].size() * 4;
    if (round64(nb) > g->bwd_bytes - g->bwd_cursor - need) {
      char buf[160];
      std::snprintf(buf, sizeof buf, "backward|%zu|%zu", nb, g->bwd_bytes - g->bwd_cursor - need);
      return fail(DG_POOL_EXHAUSTED, buf);
    }
    need += round64(nb);
  }
  // ancestors of the loss
  std::vector<char> anc(loss + 1, 0);
  anc[loss] = 1;
  for (int i = loss; i >= 0; --i) {
    if (!anc[i]) continue;
    const Node& x = g->nodes[i];
    for (int k = 0; k < x.n_in; ++k) anc[g->inputs[x.in_off + k]] = 1;
  }
  PlanTimer tm("backward");
  NvtxRange nv_bwd("dg_backward");
  std::vector<int> active;
  for (int i = 0; i <= loss; ++i)
    if (anc[i]) active.push_back(i);
  const std::shared_ptr<const Schedule> Sp = get_schedule(g, active, loss);
  const Schedule& S = *Sp;
  tm.lap("schedule");

  // slots written whole by their only contributor (the logits under a
  // pickneglogsoftmax group): placed after the zeroed range and overwritten
  // instead of accumulated, so the arena memset and the kernel's read of the
  // slot both skip them (a vocabulary-wide slot is the largest in the graph)
  std::vector<char>& overwrite = g->bwd_overwrite;
  overwrite.assign(loss + 1, 0);
  {
    std::vector<int> cons(loss + 1, 0);
    for (int i : active) {
      const Node& x = g->nodes[i];
      for (int k = 0; k < x.n_in; ++k) cons[g->inputs[x.in_off + k]]++;
    }
    for (const Group& gr : S.groups) {
      if (gr.kind != DG_OP_PNLS && gr.kind != DG_OP_PNLS_BATCH) continue;
      bool ok = true;
      std::vector<int> xs;
      for (int u : gr.units) {
        const int pn = S.units[u].last();
        const int x = g->inputs[g->nodes[pn].in_off];
        const int kx = g->nodes[x].kind;
        ok = ok && x != loss && cons[x] == 1 && kx != DG_OP_PARAMETER && kx != DG_OP_LOOKUP &&
             kx != DG_OP_LOOKUP_BATCH && kx != DG_OP_INPUT;
        xs.push_back(x);
      }
      if (ok)
        for (int x : xs) overwrite[x] = 1;
    }
    // the persistent recurrence backward (rnn.cu) stores every element of the
    // chain-internal gradient slots (gate affine, picks, activations, both
    // products, tanh(c)); only c_t and h_t can carry outside contributions
    for (const Group& gr : S.groups) {
      if (gr.kind != -3) continue;
      for (int u : gr.units)
        for (const RnnChainPlan& cp : S.rnns[S.units[u].rnn].chains)
          for (size_t t = 0; t < cp.G.size(); ++t) {
            overwrite[cp.G[t]] = 1;
            const std::vector<int>& cn = cp.cells[t].nodes;
            for (int k : {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 11}) overwrite[cn[k]] = 1;
          }
    }
  }
  // placement of grad slots: group order for scheduled units, then the rest
  const size_t begin = g->bwd_cursor;
  size_t cur = begin;
  std::vector<char> placed(loss + 1, 0);
  auto place = [&](int i) {
    if (placed[i]) return;
    placed[i] = 1;
    Node& x = g->nodes[i];
    x.grad = reinterpret_cast<float*>(g->bwd_base + cur);
    cur += round64((size_t)x.size() * 4);
  };
  for (const Group& gr : S.groups)
    for (int u : gr.units)
      for (int i : S.units[u].nodes)
        if (!overwrite[i]) place(i);
  for (int i = 0; i <= loss; ++i)
    if (!overwrite[i]) place(i);
  const size_t zero_end = cur;
  // overwritten slots: same group / unit order (slot-major recurrence blocks
  // stay dense GEMM operands), then the rest
  for (const Group& gr : S.groups)
    for (int u : gr.units)
      for (int i : S.units[u].nodes) place(i);
  for (int i = 0; i <= loss; ++i) place(i);
  // parameter nodes accumulate straight into the parameter's gradient (the
  // default sink adds the slot to p.gradient, graph.py:54-55)
  for (int i = 0; i <= loss; ++i)
    if (g->nodes[i].kind == DG_OP_PARAMETER) g->nodes[i].grad = param_at(g->aux_i[g->nodes[i].ai_off])->grad;

  Plan plan;
  {
    const int rc1 = blob_attach(plan.blob, g->blob_hint[1]);  // no regrowth copies while planning
    if (rc1) return rc1;
  }
  Blob& B = plan.blob;
  // static part (cached per structure) | per-call tail (lookup flush)
  const uint64_t pkey = plan_key(g, 1, 0, loss);
  CachedPlan* hit = plan_cache_find(g, 1, pkey);
  PatchRec rec;
  size_t n_wparams = hit ? (size_t)g->stats[4] : 0;
  if (hit) {
    blob_from_template(g, *hit, B);
    tm.lap("cached");
  } else {
    RecScope rec_scope(&rec);

    // zero the fresh slots (arena contract, graph.py:146-148) and seed dloss = 1
    {
      char* z0 = g->bwd_base + begin;
      const size_t zn = zero_end - begin;
      float* seed = g->nodes[loss].grad;
      plan.ops.push_back([z0, zn, seed](char*) {
        const cudaStream_t st = g_launch_stream;
        if (cudaMemsetAsync(z0, 0, zn, st) != cudaSuccess) return -1;
        return launch_fill(seed, 1, 1.f, st);
      });
    }
    // dummy gradient target for slot-serial passes
    float* dummy = dummy_base(g);
    std::unordered_map<int64_t, AffineUse> wuse;
    std::unordered_map<int64_t, std::vector<uintptr_t>> buse;
    tm.lap("place");
    {
      GemmBatch gb;
      static const bool per_kind = [] {
        const char* e = std::getenv("DG_PLAN_TIMING");
        return e && e[0] == '2';
      }();
      std::map<int, double> kt;
      // rows per weight key over all scheduled affine nodes, and over those in
      // plain affine groups: a key whose uses are all plain affine groups has
      // every use registered once its registered rows reach that count
      std::unordered_map<int64_t, int64_t> rows_all, rows_plain, brows_all, brows_plain;
      bool early_done = !early_dw_on(), early2_done = !early_dw_on();
      size_t early_op = 0;
      if (!early_done) {
        auto count = [&](int id, std::unordered_map<int64_t, int64_t>& m, std::unordered_map<int64_t, int64_t>& mb) {
          const Node& x = g->nodes[id];
          for (int t = 0; 2 + 2 * t < x.n_in; ++t) {
            const Node& wn = g->nodes[g->inputs[x.in_off + 1 + 2 * t]];
            if (wn.kind == DG_OP_PARAMETER) m[g->aux_i[wn.ai_off]] += x.batch;
          }
          const Node& bn = g->nodes[g->inputs[x.in_off]];
          if (bn.kind == DG_OP_PARAMETER) mb[g->aux_i[bn.ai_off]] += x.batch;
        };
        for (int id = 0; id < (int)g->nodes.size() && id < (int)S.unit_of.size(); ++id)
          if (g->nodes[id].kind == DG_OP_AFFINE && S.unit_of[id] >= 0) count(id, rows_all, brows_all);
        for (const Group& gq : S.groups)
          if (gq.kind == DG_OP_AFFINE)
            for (int u : gq.units) count(S.units[u].last(), rows_plain, brows_plain);
      }
      for (int q = (int)S.groups.size() - 1; q >= 0; --q) {
        const auto t0 = std::chrono::steady_clock::now();
        if (!plan_affine_dx_small(g, S, S.groups[q], plan, gb, wuse, buse))
          plan_backward_group(g, S, S.groups[q], plan, dummy, wuse, buse, gb);
        if (early_done && !early2_done && plan.rnn_bwd_ctas > 0 && plan.rnn_bwd_op > early_op &&
            plan.rnn_bwd_op <= plan.ops.size()) {
          // behind the second backward recurrence: column sums of biases and
          // weight gradients whose uses are all registered by now
          early2_done = true;
          plan_window_work(g, plan, wuse, buse, rows_all, brows_all, brows_plain);
        }
        if (!early_done && plan.rnn_bwd_ctas > 0 && plan.rnn_bwd_op > 0 && plan.rnn_bwd_op <= plan.ops.size()) {
          early_op = plan.rnn_bwd_op;
          early_done = true;  // behind the first backward recurrence only
          const int free_sms = sm_count_host() - plan.rnn_bwd_ctas;
          std::vector<int64_t> keys;
          for (auto& kv : wuse) keys.push_back(kv.first);
          std::sort(keys.begin(), keys.end());
          static const bool elog = std::getenv("DG_EARLY_DW_LOG") != nullptr;
          for (int64_t h : keys) {
            const AffineUse& use = wuse[h];
            const auto pa = rows_all.find(h), pp = rows_plain.find(h);
            if (elog)
              std::fprintf(stderr, "[early-dw] key %lld free %d all %lld plain %lld reg %zu size %lld\n", (long long)h,
                           free_sms, pa == rows_all.end() ? -1LL : (long long)pa->second,
                           pp == rows_plain.end() ? -1LL : (long long)pp->second, use.x_rows.size(),
                           (long long)(use.n_in * use.m));
            if (free_sms < 32 || pa == rows_all.end() || pp == rows_plain.end() || pa->second != pp->second ||
                (int64_t)use.x_rows.size() != pp->second || use.n_in * use.m < ((int64_t)1 << 21))
              continue;
            const size_t at_op = plan.rnn_bwd_op, n_before = plan.ops.size();
            if (plan_early_dw(g, plan, use, param_at(h), free_sms)) {
              // move the two ops directly behind the recurrence (ops planned
              // after it in this group follow them; the first runs without PDL)
              plan.meta.resize(plan.ops.size());
              std::rotate(plan.ops.begin() + at_op, plan.ops.begin() + n_before, plan.ops.end());
              std::rotate(plan.meta.begin() + at_op, plan.meta.begin() + n_before, plan.meta.end());
              if (elog) std::fprintf(stderr, "[early-dw] planned key %lld on %d SMs at op %zu of %zu\n", (long long)h, free_sms, at_op, n_before);
              wuse.erase(h);
              break;  // one overlapped GEMM
            }
          }
        }
        if (per_kind)
          kt[S.groups[q].kind] += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
      }
      flush_gemm(g, plan, gb);
      if (per_kind) {
        std::string o;
        for (auto& kv : kt) o += " k" + std::to_string(kv.first) + "=" + std::to_string((int)kv.second);
        std::fprintf(stderr, "[plan] backward groups by kind:%s\n", o.c_str());
      }
    }
    tm.lap("groups");

    // aggregated weight gradients: dW^T (K x m) += X^T G over every use
    std::vector<int64_t> wkeys;
    for (auto& kv : wuse) wkeys.push_back(kv.first);
    std::sort(wkeys.begin(), wkeys.end());
    {
      // rows of one parameter's uses -> the longest run where both the x rows
      // and the gradient rows are equally spaced (a dense block: TMA path) plus
      // the rest; the two parts accumulate into dW in two launches
      auto regular_run = [](const std::vector<uintptr_t>& a, const std::vector<uintptr_t>& b, int64_t la,
                            int64_t lb, size_t& best_lo, size_t& best_hi) {
        const size_t n = a.size();
        best_lo = best_hi = 0;
        size_t lo = 0;
        for (size_t i = 1; i <= n; ++i) {
          bool cont = i < n;
          if (cont && i - lo >= 2) {
            cont = a[i] - a[i - 1] == a[lo + 1] - a[lo] && b[i] - b[i - 1] == b[lo + 1] - b[lo];
          } else if (cont) {
            const int64_t sa = (int64_t)(a[i] - a[i - 1]), sb = (int64_t)(b[i] - b[i - 1]);
            cont = sa >= la * 4 && sb >= lb * 4 && sa % 16 == 0 && sb % 16 == 0 && (a[lo] & 15) == 0 &&
                   (b[lo] & 15) == 0;
          }
          if (!cont) {
            if (i - lo > best_hi - best_lo) {
              best_lo = lo;
              best_hi = i;
            }
            lo = i;
          }
        }
      };
      GemmBatch gb, gb_rest;
      std::vector<std::pair<std::vector<uintptr_t>, std::vector<uintptr_t>>> rest_rows;
      auto dw_problem = [&](const std::vector<uintptr_t>& xr, const std::vector<uintptr_t>& gr, const AffineUse& use,
                            Param* p, GemmBatch& bt) {
        GemmProblem pr{};
        pr.M = (int)use.n_in;
        pr.N = (int)use.m;
        pr.n_seg = 1;
        pr.accumulate = 1;
        pr.seg[0].K = (int64_t)xr.size();
        pr.seg[0].A.rows = dev_at<const float*>(g, B.push(xr));
        pr.seg[0].A.rows_aligned = all_aligned16(xr);
        pr.seg[0].B.rows = dev_at<const float*>(g, B.push(gr));
        pr.seg[0].B.rows_aligned = all_aligned16(gr);
        pr.C.base = p->grad;  // dW^T (n_in x m) row-major == dW column-major
        pr.C.ld = use.m;
        bt.probs.push_back(pr);
        bt.bytes += 4.0 * ((double)pr.seg[0].K * (pr.M + pr.N) + 2.0 * pr.M * pr.N);
      };
      gemm_batch_for(g, plan, gb, -1, C_GEMM_DW, true, false);
      std::vector<std::pair<int64_t, std::pair<std::vector<uintptr_t>, std::vector<uintptr_t>>>> rests;
      for (int64_t h : wkeys) {
        AffineUse& use = wuse[h];
        Param* p = param_at(h);
        size_t lo = 0, hi = 0;
        regular_run(use.x_rows, use.g_rows, use.n_in, use.m, lo, hi);
        if (hi - lo >= 128 && hi - lo < use.x_rows.size()) {
          std::vector<uintptr_t> xr(use.x_rows.begin() + lo, use.x_rows.begin() + hi);
          std::vector<uintptr_t> grr(use.g_rows.begin() + lo, use.g_rows.begin() + hi);
          dw_problem(xr, grr, use, p, gb);
          std::vector<uintptr_t> xo(use.x_rows.begin(), use.x_rows.begin() + lo), go(use.g_rows.begin(), use.g_rows.begin() + lo);
          xo.insert(xo.end(), use.x_rows.begin() + hi, use.x_rows.end());
          go.insert(go.end(), use.g_rows.begin() + hi, use.g_rows.end());
          rests.push_back({h, {std::move(xo), std::move(go)}});
        } else {
          dw_problem(use.x_rows, use.g_rows, use, p, gb);
        }
      }
      flush_gemm(g, plan, gb);
      if (!rests.empty()) {
        gemm_batch_for(g, plan, gb_rest, -1, C_GEMM_DW, true, false);
        for (auto& r : rests) dw_problem(r.second.first, r.second.second, wuse[r.first], param_at(r.first), gb_rest);
        flush_gemm(g, plan, gb_rest);
      }
    }
    tm.lap("dW");
    std::vector<int64_t> bkeys;
    for (auto& kv : buse) bkeys.push_back(kv.first);
    std::sort(bkeys.begin(), bkeys.end());
    // bias gradients: up to kColsumGroup column sums per pair of launches
    {
      float* work = reinterpret_cast<float*>(scratch_base(g));
      const int64_t wcap = (int64_t)(scratch_bytes(g) / 4);
      struct Job {
        float* dst;
        size_t orow;
        int nr, width, vec;
      };
      std::vector<Job> jobs;
      double bytes = 0;
      auto flush_jobs = [&] {
        if (jobs.empty()) return;
        plan.ops.push_back([jobs, work, wcap](char* d) {
        const cudaStream_t st = g_launch_stream;
          ColsumGroup G{};
          G.n = (int)jobs.size();
          for (int q = 0; q < G.n; ++q)
            G.j[q] = ColsumJob{jobs[q].dst, at<const float* const>(d, jobs[q].orow), jobs[q].nr, jobs[q].width, 0, 0, 0,
                               nullptr, jobs[q].vec};
          return launch_colsum_group(G, work, wcap, st);
        });
        plan.tag(C_COLSUM, 0.0, bytes);
        jobs.clear();
        bytes = 0;
      };
      for (int64_t h : bkeys) {
        auto& rows = buse[h];
        Param* p = param_at(h);
        jobs.push_back({p->grad, B.push(rows), (int)rows.size(), (int)p->size(), all_aligned16(rows) ? 1 : 0});
        bytes += 4.0 * rows.size() * p->size() + 8.0 * p->size();
        if ((int)jobs.size() == kColsumGroup) flush_jobs();
      }
      flush_jobs();
    }
    tm.lap("colsum");
    n_wparams = wuse.size();
  }
  const size_t static_ops = plan.ops.size(), static_bytes = plan.blob.size();
  // lookup flush: sorted segmented scatter-add per table (graph.py:57-63)
  {
    struct Rows {
      std::vector<std::pair<int64_t, uintptr_t>> v;
    };
    std::unordered_map<int64_t, Rows> by_table;
    std::vector<int64_t> order;
    for (int i = 0; i <= loss; ++i) {
      const Node& x = g->nodes[i];
      if (x.kind != DG_OP_LOOKUP && x.kind != DG_OP_LOOKUP_BATCH) continue;
      const int64_t h = g->aux_i[x.ai_off];
      Param* p = param_at(h);
      // touched includes non-ancestor lookups <= loss (graph.py:155-159)
      for (int64_t q = 1; q < x.ai_len; ++q) touch(*p, g->aux_i[x.ai_off + q]);
      if (!anc[i]) continue;
      auto it = by_table.find(h);
      if (it == by_table.end()) {
        order.push_back(h);
        it = by_table.emplace(h, Rows{}).first;
      }
      for (int64_t q = 1; q < x.ai_len; ++q)
        it->second.v.push_back({g->aux_i[x.ai_off + q], P(x.grad + (q - 1) * x.elem)});
    }
    tm.lap("scatter-collect");
    for (int64_t h : order) {
      auto& v = by_table[h].v;
      // stable counting sort by row id (ids < rows): unique ids sorted, then
      // each id's sources in graph order (deterministic segment sums)
      Param* pt = param_at(h);
      if ((int64_t)pt->sort_cnt.size() < pt->rows) pt->sort_cnt.assign(pt->rows, 0);
      std::vector<int32_t>& cnt = pt->sort_cnt;
      std::vector<int64_t> uids;
      for (auto& e : v)
        if (cnt[e.first]++ == 0) uids.push_back(e.first);
      std::sort(uids.begin(), uids.end());
      std::vector<int32_t> seg;
      seg.reserve(uids.size() + 1);
      int32_t pos = 0;
      for (int64_t u : uids) {
        seg.push_back(pos);
        const int32_t c = cnt[u];
        cnt[u] = pos;
        pos += c;
      }
      std::vector<uintptr_t> src(v.size());
      for (auto& e : v) src[cnt[e.first]++] = e.second;
      for (int64_t u : uids) cnt[u] = 0;
      seg.push_back((int32_t)v.size());
      Param* p = param_at(h);
      std::vector<ScatterItem> items;
      int n_part = 0, n_long = 0;
      const int n_items = plan_scatter_items(seg.data(), (int)uids.size(), items, &n_part, &n_long);
      const size_t ou = B.push(uids), oit = B.push(items), osrc = B.push(src);
      float* tg = p->grad;
      const int dim = (int)p->cols;
      float* partials = reinterpret_cast<float*>(scratch_base(g));
      int* ctr = counter_base(g) + kScatterCtrBase;
      if ((int64_t)n_part * dim * 4 > (int64_t)scratch_bytes(g) || n_long > kScatterCtrs)
        return fail(DG_POOL_EXHAUSTED, "workspace too small for the lookup scatter");
      plan.ops.push_back([tg, dim, ou, oit, osrc, n_items, partials, ctr](char* d) {
      const cudaStream_t st = g_launch_stream;
        return launch_scatter_rows(tg, dim, at<const int64_t>(d, ou), at<const ScatterItem>(d, oit), n_items,
                                   at<const float* const>(d, osrc), partials, ctr, 1.f, false, st);
      });
      plan.tag(C_SCATTER, 0.0, 4.0 * dim * ((double)src.size() + 2.0 * (double)uids.size()));
    }
  }
  tm.lap("scatter");
  g->blob_hint[1] = std::max(g->blob_hint[1], plan.blob.size() + plan.blob.size() / 4);
  if (hit) {
    rc = launch_cached(g, *hit, plan);  // plan.ops holds the tail only
    if (rc) return rc;
  } else {
    rc = prepare_launch(g, plan.blob);
    if (rc) return rc;
    if (!dry_run()) {
      std::vector<std::function<int(char*)>> tail_ops(std::make_move_iterator(plan.ops.begin() + static_ops),
                                                      std::make_move_iterator(plan.ops.end()));
      plan.meta.resize(plan.ops.size());
      std::vector<OpMeta> tail_meta(plan.meta.begin() + static_ops, plan.meta.end());
      plan.ops.resize(static_ops);
      plan.meta.resize(static_ops);
      int64_t n_static = 0, n_tail = 0;
      rc = run_ops(g, plan.ops, plan.meta, &n_static, g->stream);
      if (!rc) rc = run_ops(g, tail_ops, tail_meta, &n_tail, g->stream);
      g->launches += n_static + n_tail;
      if (rc) return rc;
      plan_cache_store(g, 1, pkey, plan, static_ops, static_bytes, std::move(rec), n_static);
    }
  }
  tm.lap("launch");
  g->lazy = hit ? hit->lazy : plan.lazy;  // supersedes the previous backward's
  g->bwd_cursor = cur;
  g->bwd_alloc_count += loss + 1;
  g->has_grads = true;
  g->stats[3] = (int64_t)S.groups.size();
  g->stats[4] = (int64_t)n_wparams;
  return DG_OK;
}

int dg_value(dg_graph* g, int32_t node, float* host_dst, int64_t n) {
  if (node < 0 || node >= (int)g->nodes.size()) return fail(DG_STALE, "node index out of range");
  int rc = do_forward(g, node);
  if (rc) return rc;
  const Node& x = g->nodes[node];
  if (n != x.size()) return fail(DG_SHAPE, "value buffer size mismatch");
  if (node == g->vcache_node && n == g->vcache_n) {
    DG_CUDA_TRY(cudaEventSynchronize(g->vcache_ev));
    std::memcpy(host_dst, g->vcache, (size_t)n * 4);
    return DG_OK;
  }
  DG_CUDA_TRY(cudaMemcpyAsync(host_dst, x.val, (size_t)n * 4, cudaMemcpyDeviceToHost, g->stream));
  g->d2h_bytes += n * 4;
  DG_CUDA_TRY(cudaStreamSynchronize(g->stream));
  return DG_OK;
}

int dg_gradient(dg_graph* g, int32_t node, float* host_dst, int64_t n) {
  if (node < 0 || node >= (int)g->nodes.size()) return fail(DG_STALE, "node index out of range");
  const Node& x = g->nodes[node];
  if (!g->has_grads || !x.grad) return fail(DG_SHAPE, "no backward pass has populated this node yet");
  if (n != x.size()) return fail(DG_SHAPE, "gradient buffer size mismatch");
  // slice sums left by the last backward for this INPUT leaf (LazyGrad)
  for (size_t i = 0; i < g->lazy.size();) {
    if (g->lazy[i].node != node) {
      ++i;
      continue;
    }
    RnnPartSum ps{};
    for (size_t q = i; q < g->lazy.size() && ps.n < kRnnMaxChains;) {
      if (g->lazy[q].node == node) {
        const LazyGrad& L = g->lazy[q];
        ps.H[ps.n] = L.H;
        ps.n_s[ps.n] = L.n_s;
        ps.dst[ps.n] = L.dst;
        ps.part[ps.n] = L.part;
        ps.n++;
        g->lazy.erase(g->lazy.begin() + (ptrdiff_t)q);
      } else {
        ++q;
      }
    }
    if (launch_rnn_part_sum(ps, g->stream) < 0) return fail(DG_CUDA, "initial-state gradient sum failed");
  }
  DG_CUDA_TRY(cudaMemcpyAsync(host_dst, x.grad, (size_t)n * 4, cudaMemcpyDeviceToHost, g->stream));
  DG_CUDA_TRY(cudaStreamSynchronize(g->stream));
  return DG_OK;
}

int dg_value_ptr(dg_graph* g, int32_t node, float** dev_ptr) {
  if (node < 0 || node > g->watermark) return fail(DG_STALE, "node not evaluated");
  *dev_ptr = g->nodes[node].val;
  return DG_OK;
}

int dg_graph_counters(dg_graph* g, int64_t* out8) {
  out8[0] = g->forward_calls;
  out8[1] = g->fwd_alloc_count;
  out8[2] = g->bwd_alloc_count;
  out8[3] = (int64_t)g->fwd_cursor;
  out8[4] = (int64_t)g->bwd_cursor;
  out8[5] = g->launches;
  out8[6] = g->h2d_bytes;
  out8[7] = g->d2h_bytes;
  return DG_OK;
}

int dg_schedule_stats(dg_graph* g, int32_t lo, int32_t hi, int64_t* out8) {
  // host-only: build the schedule of nodes [lo, hi] without touching the device
  if (lo < 0 || hi >= (int)g->nodes.size() || lo > hi) return fail(DG_STALE, "node range out of bounds");
  std::vector<int> active;
  for (int i = lo; i <= hi; ++i) active.push_back(i);
  Schedule S;
  build_schedule(g, active, hi, S);
  int64_t cells = 0, chains = 0, cell_nodes = 0;
  for (const Unit& u : S.units) {
    if (u.type == U_CELL) {
      ++cells;
      cell_nodes += (int64_t)u.nodes.size();
    }
    if (u.type == U_CHAIN) ++chains;
    if (u.type == U_RNN)
      for (const RnnChainPlan& cp : S.rnns[u.rnn].chains) {
        cells += (int64_t)cp.cells.size();
        cell_nodes += 13 * (int64_t)cp.cells.size();
      }
  }
  int64_t max_group = 0;
  for (const Group& gr : S.groups) max_group = std::max<int64_t>(max_group, (int64_t)gr.units.size());
  out8[0] = (int64_t)S.units.size();
  out8[1] = (int64_t)S.groups.size();
  out8[2] = cells;
  out8[3] = chains;
  out8[4] = cell_nodes;
  out8[5] = max_group;
  out8[6] = (int64_t)S.lookup_nodes.size();
  out8[7] = (int64_t)S.input_nodes.size();
  return DG_OK;
}

int dg_schedule_rnn_stats(dg_graph* g, int32_t lo, int32_t hi, int64_t* out4) {
  // host-only: persistent LSTM stacks of the schedule of nodes [lo, hi]
  if (lo < 0 || hi >= (int)g->nodes.size() || lo > hi) return fail(DG_STALE, "node range out of bounds");
  std::vector<int> active;
  for (int i = lo; i <= hi; ++i) active.push_back(i);
  Schedule S;
  build_schedule(g, active, hi, S);
  int64_t chains = 0, steps = 0, ctas = 0;
  for (const RnnStack& sk : S.rnns) {
    chains += (int64_t)sk.chains.size();
    ctas += sk.ctas;
    for (const RnnChainPlan& cp : sk.chains) steps += (int64_t)cp.cells.size();
  }
  out4[0] = (int64_t)S.rnns.size();
  out4[1] = chains;
  out4[2] = steps;
  out4[3] = ctas;
  return DG_OK;
}

int dg_rnn_trace(uint64_t* out, int64_t n) {
  if (rnn_trace_read(reinterpret_cast<unsigned long long*>(out), (size_t)n) != 0)
    return fail(DG_CUDA, "rnn trace read failed");
  return DG_OK;
}

int dg_profile_enable(dg_graph* g, uint32_t class_mask) {
  g->prof_mask = class_mask;
  return DG_OK;
}

int dg_profile_read(dg_graph* g, int32_t cls, double* out4) {
  if (cls < 0 || cls >= C_NCLASS) return fail(DG_INDEX, "profile class out of range");
  for (int c = 0; c < C_NCLASS; ++c) {
    for (auto& pr : g->prof_pending[c]) {
      DG_CUDA_TRY(cudaEventSynchronize(pr.second));
      float ms = 0.f;
      DG_CUDA_TRY(cudaEventElapsedTime(&ms, pr.first, pr.second));
      g->prof_ms[c] += ms;
      g->event_pool.push_back(pr.first);
      g->event_pool.push_back(pr.second);
    }
    g->prof_pending[c].clear();
  }
  out4[0] = g->prof_ms[cls];
  out4[1] = (double)g->prof_count[cls];
  out4[2] = g->prof_flops[cls];
  out4[3] = g->prof_bytes[cls];
  return DG_OK;
}

int dg_profile_reset(dg_graph* g) {
  double tmp[4];
  dg_profile_read(g, 0, tmp);
  for (int c = 0; c < 16; ++c) {
    g->prof_ms[c] = g->prof_flops[c] = g->prof_bytes[c] = 0;
    g->prof_count[c] = 0;
  }
  return DG_OK;
}

int dg_graph_plan_stats(dg_graph* g, int64_t* out8) {
  for (int i = 0; i < 8; ++i) out8[i] = g->stats[i];
  return DG_OK;
}

// ---------------------------------------------------------------- trainer

int dg_trainer_create(int rule, float lr, float momentum, float adagrad_eps, float beta1, float beta2,
                      float adam_eps, int sparse, dg_trainer** out) {
  if (rule < 0 || rule > 3) return fail(DG_BAD_SHAPE, "unknown trainer rule");
  dg_trainer* t = new dg_trainer();
  t->rule.rule = rule;
  t->rule.lr = lr;
  t->rule.momentum = momentum;
  t->rule.adagrad_eps = adagrad_eps;
  t->rule.beta1 = beta1;
  t->rule.beta2 = beta2;
  t->rule.adam_eps = adam_eps;
  t->sparse = sparse;
  *out = t;
  return DG_OK;
}

int dg_trainer_destroy(dg_trainer* t) {
  if (!t) return DG_OK;
  if (t->pinned.pending) cudaEventSynchronize(t->pinned.ev);
  if (t->pinned.ptr) cudaFreeHost(t->pinned.ptr);
  if (t->pinned.ev) cudaEventDestroy(t->pinned.ev);
  if (t->segs_dev) cudaFree(t->segs_dev);
  if (t->ids_dev) cudaFree(t->ids_dev);
  delete t;
  return DG_OK;
}

int dg_trainer_set(dg_trainer* t, float lr, int sparse) {
  t->rule.lr = lr;
  t->sparse = sparse;
  return DG_OK;
}

int dg_trainer_attach(dg_trainer* t, int64_t handle, float* s0, float* s1) {
  for (auto& s : t->slots)
    if (s.handle == handle) {
      s.s0 = s0;
      s.s1 = s1;
      return DG_OK;
    }
  t->slots.push_back({handle, s0, s1});
  return DG_OK;
}

int dg_trainer_step_count(dg_trainer* t, int64_t* step) {
  *step = t->t;
  return DG_OK;
}
int dg_trainer_set_step(dg_trainer* t, int64_t step) {
  t->t = step;
  return DG_OK;
}

int dg_trainer_update(dg_trainer* t, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  RuleArgs r = t->rule;
  if (r.rule == 3) {
    t->t += 1;
    // python floats: 1 - beta**t in double, then used as fp32 divisors (trainers.py:80-81)
    r.bc1 = (float)(1.0 - std::pow((double)t->rule.beta1, (double)t->t));
    r.bc2 = (float)(1.0 - std::pow((double)t->rule.beta2, (double)t->t));
    // (1 - beta) as python computes it in double, then fp32
    r.beta1 = t->rule.beta1;
    r.beta2 = t->rule.beta2;
  }
  // dense segments (+ lookups when not sparse), one multi-tensor launch
  std::vector<TensorSeg> segs;
  struct RowJob {
    Param* p;
    float* s0;
    float* s1;
    std::vector<int64_t> ids;
  };
  std::vector<RowJob> rows;
  int64_t blocks = 0;
  const int chunk = update_chunk();
  for (auto& s : t->slots) {
    Param* p = param_at(s.handle);
    if (!p) return fail(DG_INDEX, "trainer references a released parameter");
    if (p->kind == 0 || !t->sparse) {
      segs.push_back({p->val, p->grad, s.s0, s.s1, p->size()});
      blocks += (p->size() + chunk - 1) / chunk;
    } else if (!p->touched_list.empty()) {
      rows.push_back({p, s.s0, s.s1, touched_sorted(*p)});
    }
  }
  // host staging for the segment table and the sorted row ids
  size_t ids_total = 0;
  for (auto& j : rows) ids_total += j.ids.size();
  const size_t seg_bytes = segs.size() * sizeof(TensorSeg);
  const size_t total = seg_bytes + ids_total * 8 + 64;
  int rc = pinned_acquire(t->pinned, total);
  if (rc) return rc;
  if (t->segs_cap < seg_bytes + 1) {
    if (t->segs_dev) DG_CUDA_TRY(cudaFree(t->segs_dev));
    t->segs_cap = std::max<size_t>(seg_bytes * 2, 4096);
    DG_CUDA_TRY(cudaMalloc(&t->segs_dev, t->segs_cap));
  }
  if (t->ids_cap < ids_total * 8 + 8) {
    if (t->ids_dev) DG_CUDA_TRY(cudaFree(t->ids_dev));
    t->ids_cap = std::max<size_t>(ids_total * 16, 1 << 16);
    DG_CUDA_TRY(cudaMalloc(&t->ids_dev, t->ids_cap));
  }
  char* hp = static_cast<char*>(t->pinned.ptr);
  std::memcpy(hp, segs.data(), seg_bytes);
  size_t off = 0;
  for (auto& j : rows) {
    std::memcpy(hp + seg_bytes + off * 8, j.ids.data(), j.ids.size() * 8);
    off += j.ids.size();
  }
  if (seg_bytes) DG_CUDA_TRY(cudaMemcpyAsync(t->segs_dev, hp, seg_bytes, cudaMemcpyHostToDevice, st));
  if (ids_total)
    DG_CUDA_TRY(cudaMemcpyAsync(t->ids_dev, hp + seg_bytes, ids_total * 8, cudaMemcpyHostToDevice, st));
  DG_CUDA_TRY(cudaEventRecord(t->pinned.ev, st));
  t->pinned.pending = true;
  launch_update_dense(r, static_cast<const TensorSeg*>(t->segs_dev), (int)segs.size(), blocks, st);
  off = 0;
  for (auto& j : rows) {
    launch_update_rows(r, j.p->val, j.p->grad, j.s0, j.s1, (int)j.p->cols,
                       static_cast<const int64_t*>(t->ids_dev) + off, (int)j.ids.size(), st);
    off += j.ids.size();
  }
  // zero_gradients (params.py:114-119): dense grads were zeroed by the update
  // pass; sparse tables only ever hold gradient on touched rows, which the
  // row pass zeroed.  Clear touched sets.
  for (auto& s : t->slots) {
    Param* p = param_at(s.handle);
    touched_clear(*p);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DG_CUDA, std::string("update launch: ") + cudaGetErrorString(e));
  return DG_OK;
}

// --------------------------------------------------------------- DP helpers

// Host staging of the DP helpers: a pinned slot of the process-wide ring
// (reused once its previous upload has executed; no stream synchronisation)
// and a per-table device buffer, grown geometrically, whose scatter counter
// tail is zero at rest.
static int stage_to_device(const std::vector<uint8_t>& host, char* dev, cudaStream_t st) {
  if (host.empty()) return DG_OK;
  Pinned& slot = staging_slot();
  int rc = pinned_acquire(slot, host.size());
  if (rc) return rc;
  std::memcpy(slot.ptr, host.data(), host.size());
  DG_CUDA_TRY(cudaMemcpyAsync(dev, slot.ptr, host.size(), cudaMemcpyHostToDevice, st));
  DG_CUDA_TRY(cudaEventRecord(slot.ev, st));
  slot.pending = true;
  return DG_OK;
}

static int dp_buffer(Param& p, size_t need, cudaStream_t st) {
  constexpr size_t kCtr = sizeof(int) * 4096;
  if (p.dp_cap < need + kCtr) {
    if (p.dp_dev) DG_CUDA_TRY(cudaFree(p.dp_dev));  // implicit device sync, growth only
    p.dp_cap = std::max<size_t>(2 * (need + kCtr), 1 << 20);
    DG_CUDA_TRY(cudaMalloc(&p.dp_dev, p.dp_cap));
    DG_CUDA_TRY(cudaMemsetAsync(static_cast<char*>(p.dp_dev) + p.dp_cap - kCtr, 0, kCtr, st));
  }
  return DG_OK;
}

int dg_lookup_pack(int64_t handle, int64_t* ids_dev, float* rows_dev, int64_t cap, int64_t* n, void* stream) {
  Param* p = param_at(handle);
  if (!p || p->kind != 1) return fail(DG_INDEX, "not a lookup parameter");
  std::vector<int64_t> ids = touched_sorted(*p);
  *n = (int64_t)ids.size();
  if ((int64_t)ids.size() > cap) return fail(DG_INDEX, "pack capacity too small");
  if (ids.empty()) return DG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<uint8_t> host(ids.size() * 8);
  std::memcpy(host.data(), ids.data(), host.size());
  int rc = stage_to_device(host, reinterpret_cast<char*>(ids_dev), st);
  if (rc) return rc;
  launch_pack_rows(p->grad, (int)p->cols, ids_dev, rows_dev, (int)ids.size(), st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DG_CUDA, std::string("pack launch: ") + cudaGetErrorString(e));
  return DG_OK;
}

int dg_lookup_merge(int64_t handle, int32_t n_ranks, const int64_t* counts, const int64_t* ids_host,
                    const float* const* rank_rows, float div, void* stream) {
  // table_grad[id] = (sum over ranks, in rank order, of that rank's row) / div
  // for every id in the union; the union becomes the touched set
  // (average_slots + _load_average_into_model, parallel.py:55-65,105-109).
  Param* p = param_at(handle);
  if (!p || p->kind != 1) return fail(DG_INDEX, "not a lookup parameter");
  if (n_ranks <= 0 || !(div > 0.f)) return fail(DG_CONFIG, "merge needs n_ranks >= 1 and div > 0");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int dim = (int)p->cols;
  std::vector<uintptr_t> rows_src;
  std::vector<int64_t> ids_all;
  for (int r = 0; r < n_ranks; ++r) {
    if (counts[r] < 0) return fail(DG_CONFIG, "negative merge count");
    for (int64_t k = 0; k < counts[r]; ++k) {
      const int64_t id = ids_host[ids_all.size()];
      if (id < 0 || id >= p->rows) return fail(DG_INDEX, "merge id out of range");
      ids_all.push_back(id);
      rows_src.push_back(P(rank_rows[r] + k * dim));
    }
  }
  const int64_t n = (int64_t)ids_all.size();
  if (n == 0) return DG_OK;
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return ids_all[a] < ids_all[b]; });
  std::vector<int64_t> uids;
  std::vector<int32_t> seg;
  std::vector<uintptr_t> src(n);
  for (int64_t q = 0; q < n; ++q) {
    const int64_t id = ids_all[order[q]];
    if (q == 0 || id != ids_all[order[q - 1]]) {
      uids.push_back(id);
      seg.push_back((int32_t)q);
    }
    src[q] = rows_src[order[q]];
  }
  seg.push_back((int32_t)n);
  std::vector<ScatterItem> items;
  int n_part = 0, n_long = 0;
  const int n_items = plan_scatter_items(seg.data(), (int)uids.size(), items, &n_part, &n_long);
  if (n_long > 4096) return fail(DG_INTERNAL, "merge: too many long segments");
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t o_u = 0, o_it = al(uids.size() * 8), o_src = o_it + al(items.size() * sizeof(ScatterItem));
  const size_t o_part = o_src + al(src.size() * 8);
  const size_t need = o_part + (size_t)n_part * dim * 4;
  int rc = dp_buffer(*p, need, st);
  if (rc) return rc;
  std::vector<uint8_t> host(o_part, 0);
  std::memcpy(host.data() + o_u, uids.data(), uids.size() * 8);
  std::memcpy(host.data() + o_it, items.data(), items.size() * sizeof(ScatterItem));
  std::memcpy(host.data() + o_src, src.data(), src.size() * 8);
  char* d = static_cast<char*>(p->dp_dev);
  rc = stage_to_device(host, d, st);
  if (rc) return rc;
  int* ctr = reinterpret_cast<int*>(d + p->dp_cap - sizeof(int) * 4096);
  launch_scatter_rows(p->grad, dim, reinterpret_cast<const int64_t*>(d + o_u),
                      reinterpret_cast<const ScatterItem*>(d + o_it), n_items,
                      reinterpret_cast<const float* const*>(d + o_src), reinterpret_cast<float*>(d + o_part), ctr, div,
                      true, st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DG_CUDA, std::string("merge launch: ") + cudaGetErrorString(e));
  for (int64_t id : uids) touch(*p, id);
  return DG_OK;
}

int dg_scale(float* y, int64_t n, float alpha, void* stream) {
  launch_scale(y, n, alpha, static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DG_CUDA, cudaGetErrorString(e));
  return DG_OK;
}

}  // extern "C"
