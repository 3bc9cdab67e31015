/*
 * dyngpu.h — C-ABI of the B200 execution backend for dynamic ComputationGraphs.
 *
 * The reference (arXiv 1701.03980 desk-scale `dyncore`) has no native code and
 * no FFI: its hot path is the per-node Python interpreter in
 *   ComputationGraph._run_forward / backward  (pkg/src/dyncore/graph.py:115-164)
 * dispatching into the op catalog               (pkg/src/dyncore/ops.py:33-52, 98-527)
 * with gradients pushed through the sink         (pkg/src/dyncore/graph.py:51-66)
 * into Model storage                            (pkg/src/dyncore/params.py:55-119)
 * consumed by Trainer.update                    (pkg/src/dyncore/trainers.py:63-98).
 *
 * Each entry point below replaces one of those interfaces; the Python drop-in
 * (the paper_1701_03980_b200 package) keeps the reference's Python API and calls
 * these through ctypes.  Plain pointers and sizes only:
 * device buffers are allocated by the caller (PyTorch) and passed as raw
 * pointers; streams are cudaStream_t passed as void*.
 *
 * Every function returns a dg_status; on failure dg_last_error() returns a
 * thread-local message.  Status codes map 1:1 onto pkg/src/dyncore/errors.py.
 */
#ifndef DYNGPU_H
#define DYNGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes  (errors.py:8-86) ---------------------------------- */
typedef enum {
  DG_OK = 0,
  DG_POOL_EXHAUSTED = 1,   /* PoolExhausted   errors.py:8-16  */
  DG_NON_SCALAR_LOSS = 2,  /* NonScalarLoss   errors.py:47-48 */
  DG_STALE = 3,            /* StaleExpression errors.py:43-44 */
  DG_SHAPE = 4,            /* ShapeError      errors.py:39-40 */
  DG_INDEX = 5,            /* IndexOutOfBounds errors.py:31-32 */
  DG_BAD_SHAPE = 6,        /* BadShape        errors.py:27-28 */
  DG_CUDA = 7,             /* CUDA runtime failure (no reference analogue) */
  DG_CONFIG = 8,           /* ConfigError     errors.py:81-82 */
  DG_INTERNAL = 9
} dg_status;

/* ---- op kinds (ops.py:98-527 registry names) -------------------------- */
typedef enum {
  DG_OP_INPUT = 0,
  DG_OP_PARAMETER = 1,
  DG_OP_LOOKUP = 2,
  DG_OP_LOOKUP_BATCH = 3,
  DG_OP_ADD = 4,
  DG_OP_CMULT = 5,
  DG_OP_SCALAR_MUL = 6,
  DG_OP_TANH = 7,
  DG_OP_LOGISTIC = 8,
  DG_OP_MATMUL = 9,
  DG_OP_AFFINE = 10,
  DG_OP_CONCATENATE = 11,
  DG_OP_PICK_RANGE = 12,
  DG_OP_SOFTMAX = 13,
  DG_OP_PNLS = 14,        /* pickneglogsoftmax        */
  DG_OP_PNLS_BATCH = 15,  /* pickneglogsoftmax_batch  */
  DG_OP_SUM_BATCHES = 16,
  DG_OP_COUNT = 17
} dg_op;

/* One node record of the bulk node table (graph.py:39-48 `Node`).
 * inputs live in a separate int32 array at [in_off, in_off+n_in);
 * integer aux (param handle / lookup ids / labels / pick range) at
 * aux_i[aux_i_off .. +aux_i_len); float aux (scalar, input payload) at
 * aux_f[aux_f_off .. +aux_f_len).  Offsets are relative to the arrays passed
 * in the same dg_graph_append call. */
typedef struct {
  int32_t kind;
  int32_t n_in;
  int32_t in_off;
  int32_t rank;
  int32_t dims[4];
  int32_t batch;
  int32_t aux_i_off;
  int32_t aux_i_len;
  int32_t aux_f_off;
  int32_t aux_f_len;
} dg_node;

typedef struct dg_graph dg_graph;
typedef struct dg_trainer dg_trainer;

const char* dg_last_error(void);
int dg_abi_version(void);

/* ---- parameter registry  (params.py:84-111 add_parameters / add_lookup_parameters)
 * kind 0 = dense Parameter (rows x cols, column-major, cols==1 for vectors),
 * kind 1 = LookupParameter (rows x dim, row-major).  Storage is caller-owned
 * device memory; handles are process-global so any graph can reference any
 * model's parameters. */
int dg_param_register(int kind, int64_t rows, int64_t cols, float* values, float* grad, int64_t* handle);
/* rebind storage after the caller re-lays-out a model (values copied by caller) */
int dg_param_rebind(int64_t handle, float* values, float* grad);
int dg_param_release(int64_t handle);

/* touched-row set of a LookupParameter (params.py:41-52 `touched`), kept on the
 * host side of the library; sorted ascending, bit-exact with the reference */
int dg_touched_count(int64_t handle, int64_t* n);
int dg_touched_get(int64_t handle, int64_t* ids, int64_t cap);
int dg_touched_add(int64_t handle, const int64_t* ids, int64_t n);
int dg_touched_clear(int64_t handle);

/* ---- graph engine  (graph.py:69-172) ---------------------------------- */
/* ≙ ComputationGraph(pools) with new_poolset (arena.py:71-110): the forward and
 * backward arenas and a plan/scratch workspace are caller-owned device memory. */
int dg_graph_create(int device, void* fwd_base, size_t fwd_bytes, void* bwd_base, size_t bwd_bytes,
                    void* work_base, size_t work_bytes, dg_graph** out);
int dg_graph_destroy(dg_graph* g);
int dg_graph_set_stream(dg_graph* g, void* stream);
/* ≙ renew + PoolSet.reset_transient (graph.py:83-87, arena.py:85-92) */
int dg_graph_renew(dg_graph* g);
/* ≙ add_node, in bulk (graph.py:97-106); shapes were inferred by the caller */
int dg_graph_append(dg_graph* g, const dg_node* nodes, int32_t n, const int32_t* inputs, int32_t n_inputs,
                    const int64_t* aux_i, int64_t n_aux_i, const float* aux_f, int64_t n_aux_f);
/* ≙ _run_forward / forward_to (graph.py:115-130); asynchronous on the stream */
int dg_forward(dg_graph* g, int32_t upto);
/* ≙ backward (graph.py:139-164) incl. the default sink (graph.py:51-63):
 * parameter grads accumulate into registered grad storage, lookup rows into
 * the table gradient, touched sets updated.  Asynchronous. */
int dg_backward(dg_graph* g, int32_t loss);
/* ≙ value / gradient (graph.py:132-135, 166-172): D2H copy, synchronises */
int dg_value(dg_graph* g, int32_t node, float* host_dst, int64_t n);
int dg_gradient(dg_graph* g, int32_t node, float* host_dst, int64_t n);
/* device pointer of a node value (interop; valid until renew) */
int dg_value_ptr(dg_graph* g, int32_t node, float** dev_ptr);
/* counters: forward_calls (graph.py:78,124), Pool.alloc_count (arena.py:46,55),
 * pool cursors; out[0..7] = forward_calls, fwd_alloc_count, bwd_alloc_count,
 * fwd_cursor, bwd_cursor, launches (kernels enqueued since create),
 * h2d bytes (node tables + inputs), d2h bytes (values) */
int dg_graph_counters(dg_graph* g, int64_t* out8);
/* execution statistics of the last forward/backward plan (groups, fused cells...) */
int dg_graph_plan_stats(dg_graph* g, int64_t* out8);
/* live profiling: CUDA events around every launch of the enabled op classes
 * (bit c of class_mask; classes: 0 affine GEMM fwd, 1 dX GEMM, 2 aggregated dW
 * GEMM, 3 pnls fwd, 4 pnls bwd, 5 elementwise, 6 gather, 7 sorted scatter-add,
 * 8 bias column sums, 9 other, 10 persistent LSTM forward, 11 persistent LSTM
 * backward).  dg_profile_read syncs and returns
 * out4 = {total ms, launches, algorithmic flops, algorithmic bytes}. */
int dg_profile_enable(dg_graph* g, uint32_t class_mask);
/* host-only planner introspection for nodes [lo, hi]: out8 = {units, groups,
 * fused cells, add chains, nodes inside cells, largest group, lookup leaves,
 * input leaves}.  Touches no device memory. */
int dg_schedule_stats(dg_graph* g, int32_t lo, int32_t hi, int64_t* out8);
/* host-only: persistent LSTM stacks the planner forms over nodes [lo, hi]
 * (out4 = stacks, chains, steps, CTAs of one launch per stack) */
int dg_schedule_rnn_stats(dg_graph* g, int32_t lo, int32_t hi, int64_t* out4);
/* diagnostics: per-CTA globaltimer stamps of the last persistent LSTM launches
 * recorded with DG_RNN_TRACE=1 (out: 2 x 148 x 256 uint64) */
int dg_rnn_trace(uint64_t* out, int64_t n);
int dg_profile_read(dg_graph* g, int32_t cls, double* out4);
int dg_profile_reset(dg_graph* g);

/* ---- trainers  (trainers.py:21-98) ------------------------------------ */
/* rule: 0 sgd, 1 momentum, 2 adagrad, 3 adam */
int dg_trainer_create(int rule, float lr, float momentum, float adagrad_eps, float beta1, float beta2,
                      float adam_eps, int sparse, dg_trainer** out);
int dg_trainer_destroy(dg_trainer* t);
int dg_trainer_set(dg_trainer* t, float lr, int sparse);
/* attach a registered parameter with caller-owned state buffers (slot0/slot1
 * = vel | sq | m1,m2 per rule; may be NULL when the rule needs fewer) */
int dg_trainer_attach(dg_trainer* t, int64_t handle, float* slot0, float* slot1);
/* ≙ Trainer.update: dense rule on every dense parameter, sorted touched rows
 * (or every row when dense) of each lookup table, Adam t+=1 first, then
 * zero_gradients + clear touched.  Asynchronous on `stream`. */
int dg_trainer_update(dg_trainer* t, void* stream);
int dg_trainer_step_count(dg_trainer* t, int64_t* step);
int dg_trainer_set_step(dg_trainer* t, int64_t step);

/* ---- data-parallel exchange helpers (parallel.py:55-65,105-109) --------
 * dg_lookup_pack: copy the sorted touched rows of a lookup table's gradient
 * into rows_dev (n x dim) and their ids into ids_dev, for an all-gather.
 * dg_lookup_merge: ranks' packed rows (rank r: counts[r] rows at the device
 * pointer rank_rows[r], ids in ids_host, concatenated in rank order) replace
 * the table gradient on the union of ids with (sum in rank order) / div —
 * average_slots + _load_average_into_model for the touched rows — and the
 * union joins the touched set.  Both asynchronous on `stream` (host staging
 * goes through pinned memory; no stream synchronisation), deterministic. */
int dg_lookup_pack(int64_t handle, int64_t* ids_dev, float* rows_dev, int64_t cap, int64_t* n, void* stream);
int dg_lookup_merge(int64_t handle, int32_t n_ranks, const int64_t* counts, const int64_t* ids_host,
                    const float* const* rank_rows, float div, void* stream);
/* plain device helpers used by the sinks: y = alpha * y; zero */
int dg_scale(float* y, int64_t n, float alpha, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DYNGPU_H */
