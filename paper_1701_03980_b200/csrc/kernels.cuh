// Kernel launchers of the B200 executor (sm_100a).  Every launcher enqueues on
// the given stream and returns the number of kernels it launched (>= 0) so the
// executor can report gpu_launches; errors surface through cudaGetLastError.
//
// Group kernels operate on N same-signature nodes at once ("operation
// batching"); per-node operands are addressed through device pointer tables
// built by the planner (executor.cpp) and uploaded once per plan.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

namespace dg {

// Programmatic dependent launch: every kernel starts with pdl_prologue()
// (wait for the preceding grid's completion and memory, then let the next
// grid launch), and launch_k() launches with programmatic stream
// serialization, so a kernel's launch and CTA rasterisation overlap the tail
// of the one before it.  DG_PDL=0 launches without the attribute (the
// prologue is then a no-op).
__device__ __forceinline__ void pdl_prologue() {
#if defined(__CUDA_ARCH__)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
bool pdl_enabled();
// the next launch that asks pdl_enabled() goes without programmatic
// serialization (waits for every earlier grid of the stream)
void pdl_skip_next();

// 3xTF32 operand splits (x ~ hi + lo, products hi*hi + hi*lo + lo*hi).
// Both parts are rounded to nearest (cvt.rna), not truncated: a truncated
// split leaves lo with the sign of x, so the dropped lo*lo term has the sign
// of the product and accumulates as a bias over K; rounded parts have
// |lo| <= 2^-11 |x| with either sign.  tf32_rn_lo_of_raw is the residual for
// an operand the tensor core reads raw (its hardware hi = truncation).
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ uint32_t tf32_rn_hi(float x) { return tf32_rna(x); }
__device__ __forceinline__ uint32_t tf32_rn_lo(float x) { return tf32_rna(x - __uint_as_float(tf32_rna(x))); }
// cheap forms for finite operands inside hot loops: round-half-away of the
// magnitude in two integer ops (no NaN/Inf handling, which cvt.rna spends
// three more instructions on)
__device__ __forceinline__ uint32_t tf32_rn_bits(float x) { return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u; }
__device__ __forceinline__ float tf32_rn_lo_of_raw(float x) {
  return __uint_as_float(tf32_rn_bits(x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u)));
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args...);
}


// ---------------------------------------------------------------- elementwise
enum EwKind : int {
  EW_TANH = 0, EW_LOGISTIC = 1, EW_SCALE = 2, EW_ADD = 3, EW_CMULT = 4
};

struct EwArgs {
  int kind;
  int n;            // nodes in the group
  int elem;         // per-batch-element size of the output
  int batch;        // output batch
  int a_b1, b_b1;   // operand is batch-1 (broadcast over batch)
  float scalar;
  const float* const* a;   // [n] operand 0 values
  const float* const* b;   // [n] operand 1 values (binary only)
  float* const* out;       // [n] output values
  // backward
  const float* const* gout;  // [n]
  const float* const* oval;  // [n] output values (tanh/logistic backward)
  float* const* ga;          // [n] operand-0 grads
  float* const* gb;          // [n] operand-1 grads
};
int launch_ew_fwd(const EwArgs& a, cudaStream_t s);
int launch_ew_bwd(const EwArgs& a, cudaStream_t s);

// n-ary prefix sum for rewritten add chains: outs[i] = ins[0] + ... + ins[i+1]
struct ChainArgs {
  int n;       // chains in the group
  int len;     // number of add nodes in each chain (inputs = len + 1)
  int size;    // elements per value
  const float* const* ins;   // [(len+1) * n], slot-major
  float* const* outs;        // [len * n]
  const float* const* gfinal;  // [n] grad of the last add
  float* const* gins;        // [(len+1) * n]
  float* const* gouts;       // [len * n] grads of the intermediate adds (get gfinal)
  int distinct;              // backward: every gins / gouts slot distinct (element-parallel adds)
};
int launch_chain_fwd(const ChainArgs& a, cudaStream_t s);
int launch_chain_bwd(const ChainArgs& a, cudaStream_t s);

// ---------------------------------------------------------- fused gated cells
// One launch evaluates N same-signature gated cells (the 13-node LSTM step of
// builders.py:92-101 and the Tree-LSTM compositions of builders.py:250-274):
//   i,o = sigmoid(G[off_i|off_o]), g = tanh(G[off_g]), f_k = sigmoid(G[off_f[k]])
//   c = i*g (+ f_1*c_1) (+ f_2*c_2) ... (left-deep, the reference's order)
//   h = o * tanh(c)
// Every node of the pattern keeps its own value (and gradient) slot.
// Slot layout per cell (slot-major pointer tables, nslot = 10 + 5m):
//   0 G | 1..m c_ext | picks i,f[m],o,g | acts i,f[m],o,g | prod ig, prod f[m]
//   | adds[m] | tanh(c) | h        (c = adds[m-1], or prod ig when m == 0)
struct CellArgs {
  int n, batch, H, gw, m;
  int off_i, off_o, off_g;
  int off_f[2];
  int cext_b1[2];
  int nslot;
  const float* const* val;  // [nslot * n]
  float* const* grad;       // [nslot * n] (backward)
};
int launch_cell_fwd(const CellArgs& a, cudaStream_t s);
int launch_cell_bwd(const CellArgs& a, cudaStream_t s);

// GRU step (builders.py:102-110) in two fused parts around the recurrent
// matmul: part A (picks z, r of the gate affine zr, the candidate's input
// pick cx of ax, r*h), part B (candidate pick of Wh(r*h), cx + ch, tanh,
// 1 - z as input(ones) + (-1)*z, (1-z)*h + z*cand).  Slots: A = zr, ax, h |
// pz, z, pr, r, cx, rh; B = mh, cx, z, ones, h | ch, s, cand, nz, keep, kh,
// zc, nh.  One thread per (node, unit) loops over the batch (broadcast h /
// ones gradients are summed in batch order).
struct GruArgs {
  int n, batch, H, gw;    // gw: width of zr / ax / mh (3H)
  int off0, off1, off2;   // A: z, r offsets in zr, cx offset in ax; B: ch offset in mh
  int h_b1, ones_b1;      // broadcast (batch-1) h / ones under a batched step
  int nslot;
  const float* const* val;  // [nslot * n]
  float* const* grad;       // [nslot * n] (backward)
};
int launch_gru_fwd(const GruArgs& a, bool part_b, cudaStream_t s);
int launch_gru_bwd(const GruArgs& a, bool part_b, cudaStream_t s);

// Class-factored softmax term (builders.py:282-378 neg_log_softmax):
// s = add(pickneglogsoftmax(class_scores, c), pickneglogsoftmax(word_scores, i))
// as one unit: one block per unit computes both picked negative log
// softmaxes (rows of different widths) and their sum; backward adds
// g * (softmax - onehot) into both score rows.  Per unit slots:
// [0] class scores, [1] word scores, [2] pnls class, [3] pnls word, [4] s.
struct Pnls2Args {
  int n;
  const float* const* val;  // [5 * n]
  float* const* grad;       // [5 * n] (backward)
  const int* width;         // [2 * n]
  const int* label;         // [2 * n]
};
int launch_pnls2_fwd(const Pnls2Args& a, cudaStream_t s);
int launch_pnls2_bwd(const Pnls2Args& a, cudaStream_t s);

// gate affine + gated cell of a small level in one launch (cellgemm.cu):
// G = bias + sum_t W_t x_t (W_t column-major gw x K_t), then the cell
constexpr int kAffCellUnits = 4;  // hidden units per CTA
constexpr int kAffCellMaxTerms = 3;
struct AffCellArgs {
  CellArgs cell;  // val[0 * n + j] = the gate node (written whole)
  int rows;       // n * batch
  int terms;
  int K[kAffCellMaxTerms];
  int koff[kAffCellMaxTerms];  // 4-aligned offsets of the terms in the padded K
  int kpad;
  const float* W[kAffCellMaxTerms];
  const float* const* x[kAffCellMaxTerms];  // [rows] input rows per term
  const float* bias;                        // broadcast row (gw)
  float* const* gx[kAffCellMaxTerms];       // [rows] input gradient rows per term (backward)
  const float* const* grow;                 // [rows] gate gradient rows (backward)
  int wslot;                                // tree launches: which staged weight set
  // act != 0: no gated cell -- slot 0 = the affine / matmul node, slot 1 =
  // its activation (1 tanh, 2 logistic); bias may be null (matmul); cat (if
  // set): [rows] value rows of a concatenate node = the terms' inputs side by
  // side (TreeRNN: tanh(matmul(W, concatenate([e1, e2]))))
  int act;
  float* const* cat;
};
// every level of a tree in one cooperative launch (cellgemm.cu tree_fwd_kernel)
struct TreeFwdArgs {
  int H, n_levels, n_wsets, max_rows;
  int wfloats[2];            // shared-memory floats of each staged weight set
  AffCellArgs wset[2];       // weight set w: terms, K, koff, kpad, W, gw, H (its rows / tables unused)
  const AffCellArgs* levels;  // [n_levels] (device)
};
size_t tree_fwd_smem(const TreeFwdArgs& t);
int launch_tree_fwd(const TreeFwdArgs& t, cudaStream_t s);
constexpr int kAffCellCols = 8;  // backward: input columns per CTA
size_t affine_cell_smem(int rows, int kpad, int gw, int H);
int launch_affine_cell_fwd(const AffCellArgs& a, cudaStream_t s);
size_t affine_dx_small_smem(int rows, int gw);
int launch_affine_dx_small(const AffCellArgs& a, cudaStream_t s);

// ------------------------------------------- persistent LSTM recurrence (rnn.cu)
// One launch runs every step of a stack of LSTM chains (builders.py:92-101
// steps sharing Wx, Wh, b; x^l_t = h^{l-1}_t for stacked layers).  Per step t
// a chain has kRnnSlots node pointers: the 15 CellArgs slots for m = 1
// (G, c_prev, picks i,f,o,g, acts i,f,o,g, prod ig, prod fc, c, tanh c, h)
// followed by x_t and h_{t-1}.
constexpr int kRnnSlots = 17;
constexpr int kRnnMaxChains = 16;
constexpr int kRnnUnits = 16;  // hidden units per CTA
struct RnnChain {
  int T, B, H, K_in, gw;
  int off_i, off_f, off_o, off_g;
  int n_s, n_u;     // batch slices (of bs rows) x unit blocks (of kRnnUnits)
  int cta0;         // first CTA of the chain
  int src, cons;    // stacked producer (fwd) / consumer (bwd) chain, -1 none
  int flag0;        // this chain's arrival counters: [n_s][T]
  const float* Wx;  // column-major gw x K_in (W[row + k * gw])
  const float* Wh;  // column-major gw x H
  const float* bias;
  const float* const* val;  // [T][kRnnSlots] (device)
  float* const* grad;       // [T][kRnnSlots] (device, backward)
  const int* b1;            // [T] bit0 x_t, bit1 h_{t-1}, bit2 c_{t-1} is batch-1
  // initial-state gradients computed by the backward cluster kernel: h0 = 1
  // adds dh_{-1} into h_{-1}'s per-row slot, h0 = 2 writes per-slice row sums
  // to h0_part[n_s][H] (batch-1 h_{-1}); c0 = 1 writes per-slice row sums of
  // the batch-1 c_{-1} term to c0_part[n_s][H]
  int h0, c0;
  float* h0_part;
  float* c0_part;
};
struct RnnArgs {
  int n_chains, ctas, bs, cj, n_flags;
  int vec;     // every staged row is 16B aligned with a multiple-of-4 width (cp.async path)
  int trace;   // record the per-step timeline (rnn_trace_read)
  int knob;    // DG_RNN_KNOB: A/B switches of the recurrence kernels (diagnostics)
  int gx;      // G slots hold b + Wx x_t already (chains run with K_in = 0: recurrent part only)
  int* flags;  // zeroed by the launcher
  RnnChain ch[kRnnMaxChains];
};
// batch-1 c_{-1} gradients: dst[k][u] += sum_b dc[k][b][u] * af[k][b][u]
struct RnnC0 {
  int n;
  int H[kRnnMaxChains], B[kRnnMaxChains];
  float* dst[kRnnMaxChains];
  const float* dc[kRnnMaxChains];
  const float* af[kRnnMaxChains];
};
// dst[k][u] += sum_s part[k][s * H + u] for every item k (in order)
struct RnnPartSum {
  int n;
  int H[kRnnMaxChains], n_s[kRnnMaxChains];
  float* dst[kRnnMaxChains];
  const float* part[kRnnMaxChains];
};
int launch_rnn_part_sum(const RnnPartSum& a, cudaStream_t s);
// the cluster launch of these arguments can have every cluster resident
bool rnn_cluster_fits(const RnnArgs& a, bool backward, size_t smem, int cluster);
int rnn_rows_per_cta(int B);
size_t rnn_fwd_smem(int K, int bs);
size_t rnn_bwd_smem(int gw, int gw_c, int bs, int cj);
bool rnn_enabled();  // DG_RNN=0 disables the persistent path (A/B checks)
bool rnn_cluster_enabled();  // DG_RNN_CLUSTER=0 keeps the global-counter kernels
int launch_rnn(const RnnArgs& a, bool backward, size_t smem, cudaStream_t s);
// cluster variants (one cluster of n_u CTAs per chain slice, DSMEM exchange):
// returns -2 when the clusters cannot all be resident (caller falls back)
size_t rnn_fwd_cl_smem(int K_in, int H, int bs);
size_t rnn_bwd_cl_smem(int H, int gw_c, int bs, int cj);
int launch_rnn_cluster(const RnnArgs& a, bool backward, size_t smem, int cluster, cudaStream_t s);
int launch_rnn_c0(const RnnC0& a, cudaStream_t s);
bool rnn_trace_enabled();  // DG_RNN_TRACE=1
// [2][148][256] globaltimer stamps of the last launches (fwd, bwd)
int rnn_trace_read(unsigned long long* host, size_t n);

// --------------------------------------------------------------- structural
struct PickArgs {
  int n, batch, in_elem, lo, width;
  const float* const* in; float* const* out;
  const float* const* gout; float* const* gin;
};
int launch_pick_fwd(const PickArgs& a, cudaStream_t s);
int launch_pick_bwd(const PickArgs& a, cudaStream_t s);

struct ConcatArgs {
  int n, batch, parts, total;
  const int* offs;                 // [parts + 1] column offsets (device)
  const float* const* in;          // [parts * n]
  float* const* out;               // [n]
  const float* const* gout;
  float* const* gin;               // [parts * n]
};
int launch_concat_fwd(const ConcatArgs& a, cudaStream_t s);
int launch_concat_bwd(const ConcatArgs& a, cudaStream_t s);

struct SumBatchesArgs {
  int n, batch, elem;
  const float* const* in; float* const* out;
  const float* const* gout; float* const* gin;
};
int launch_sum_batches_fwd(const SumBatchesArgs& a, cudaStream_t s);
int launch_sum_batches_bwd(const SumBatchesArgs& a, cudaStream_t s);

// ----------------------------------------------------------------- row-wise
struct RowArgs {
  int rows;        // total rows (n nodes * batch)
  int width;       // row length
  int batch;       // rows per node
  const float* const* in;    // [n] node input values (rows batch-contiguous)
  float* const* out;         // [n] node outputs
  const int* labels;         // [rows] (pnls)
  const float* const* gout;  // [n]
  const float* const* oval;  // [n] (softmax backward)
  float* const* gin;         // [n]
  int overwrite;             // pnls backward: gin = (no accumulate; the slot's only contributor)
};
int launch_softmax_fwd(const RowArgs& a, cudaStream_t s);
int launch_softmax_bwd(const RowArgs& a, cudaStream_t s);
int launch_pnls_fwd(const RowArgs& a, cudaStream_t s);
int launch_pnls_bwd(const RowArgs& a, cudaStream_t s);

// ------------------------------------------------------------ lookup tables
// gather: out_rows[r] = table[ids[r]]  (one warp per row, 128-bit vectors)
int launch_gather_rows(const float* table, int dim, const int64_t* ids, float* const* out_rows, int rows,
                       cudaStream_t s);
// sorted segmented scatter of row gradients (graph.py:57-63):
//   for u in unique: table_grad[ids[u]] += scale * sum_{k in seg[u]..seg[u+1]} src_rows[k]
// (set_mean: table_grad[ids[u]] = sum / scale).  Deterministic: fixed
// summation order, no float atomics.  Segments longer than kScatterChunk rows
// are split into chunks (partials: n_partials x dim floats of scratch;
// counters: n_long ints, zero at rest and left at zero).
constexpr int kScatterChunk = 16;
struct ScatterItem {
  int u, k0, k1, chunk, nchunks, pbase, seg_slot, pad;
};
int plan_scatter_items(const int* seg, int n_unique, std::vector<ScatterItem>& items, int* n_partials, int* n_long);
int launch_scatter_rows(float* table_grad, int dim, const int64_t* uniq_ids, const ScatterItem* items, int n_items,
                        const float* const* src_rows, float* partials, int* counters, float scale, bool set_mean,
                        cudaStream_t s);

// ---------------------------------------------------------------- generic
// matmul (ops.py:252-301) per batch element, column-major element layout
struct MatmulArgs {
  int n, batch, m, k, p, a_b1, x_b1;
  const float* const* a; const float* const* x; float* const* out;
  const float* const* gout; float* const* ga; float* const* gx;
};
int launch_matmul_fwd(const MatmulArgs& a, cudaStream_t s);
int launch_matmul_bwd(const MatmulArgs& a, cudaStream_t s);

// affine with a per-element (batched) or non-parameter matrix: slow generic path
struct AffineGenericArgs {
  int n, batch, m, terms;
  int b_b1;
  const float* const* bias;   // [n]
  int kdim[8];                // per term (<= 8 terms)
  int w_b1[8];
  int x_b1[8];
  const float* const* w;      // [terms * n]
  const float* const* x;      // [terms * n]
  float* const* out;          // [n]
  const float* const* gout;
  float* const* gbias;
  float* const* gw;
  float* const* gx;
};
int launch_affine_generic_fwd(const AffineGenericArgs& a, cudaStream_t s);
int launch_affine_generic_bwd(const AffineGenericArgs& a, cudaStream_t s);

// column sums over gathered rows: dst[c] += sum_r rows[r][c]  (deterministic)
int launch_colsum_rows(float* dst, const float* const* rows, int n_rows, int width, float* work,
                       int64_t work_floats, cudaStream_t s);
// several column sums (the bias gradients of one backward) in one pair of launches
struct ColsumJob {
  float* dst;
  const float* const* rows;
  int n_rows, width;
  int chunks, pb0, fb0;  // filled by launch_colsum_group
  float* work;
  int vec;               // every row 16 B aligned (wide row-segment path)
};
constexpr int kColsumGroup = 8;
struct ColsumGroup {
  ColsumJob j[kColsumGroup];
  int n;
  int nowait;  // wide jobs only: the partial pass skips griddepcontrol.wait (launched behind an independent grid)
};
int launch_colsum_group(ColsumGroup G, float* work, int64_t work_floats, cudaStream_t s);
// row reduce-scatter: for t in targets: dst[t] += sum_{k in seg} src[k]  (src dense, width)
int launch_row_reduce_scatter(float* const* dst_rows, const int* seg, const float* src, int n_targets,
                              int width, cudaStream_t s);

// ------------------------------------------------------------------- GEMM
// C[M x N] (=|+=) sum_seg A_seg(m,k) B_seg(k,n) (+ bias_m(n)), fp32 SIMT.
struct Operand {
  const float* base;     // used when rows == nullptr: row(i) = base + i*ld
  int64_t ld;
  const float* const* rows;  // row pointer table (device) or nullptr
  int64_t rows_aligned;      // every row-table entry is 16B aligned (planner-checked)
};
struct GemmSeg {
  int64_t K;
  Operand A, B;
};
// One problem of a grouped launch; the table lives in device memory.
//   a_kmajor (per launch): A(m,k) = A.row(k)[m]   else A.row(m)[k]
//   b_nmajor (per launch): B(k,n) = B.row(n)[k]   else B.row(k)[n]
struct GemmProblem {
  int M, N, n_seg, accumulate;
  GemmSeg seg[4];
  Operand C;     // row(m) -> N contiguous outputs
  Operand bias;  // optional per-row bias (row(m)[n]); base == rows == nullptr -> none
  // filled by gemm_plan
  int tiles_n, tiles, splits, cta0;
  int counter0, vec_a, vec_b, pad_;
  int64_t work_off;
};
struct GemmLaunch {
  int cfg, n_probs, ctas;
  int cluster;  // > 0: split-K across a thread-block cluster of this size
  int chunk;    // tensor-core path: TMEM accumulator drain period (k-tiles)
  bool a_kmajor, b_nmajor;
  int64_t work_floats;
  double flops;
};
// host: choose tile config / split-K / CTA offsets (mutates probs)
GemmLaunch gemm_plan(std::vector<GemmProblem>& probs, bool a_kmajor, bool b_nmajor, int64_t work_cap_floats,
                     int counter_cap);
// counters: zero-initialised ints (>= sum of split problems' tiles); left zero
int launch_gemm_group(const GemmLaunch& L, const GemmProblem* probs_dev, float* work, int* counters,
                      cudaStream_t s);
// tcgen05 3xTF32 path (tcgemm.cu) for wide single-segment problems
bool tc_gemm_eligible(const std::vector<GemmProblem>& probs);
GemmLaunch tc_gemm_plan(std::vector<GemmProblem>& probs, bool a_kmajor, bool b_nmajor);
int launch_tc_gemm(const GemmLaunch& L, const GemmProblem* probs_dev, cudaStream_t s);
// DG_TC=0 in the environment disables the tensor-core path (A/B checks)
bool tc_gemm_enabled();

// TMA + warp-specialised tcgen05 3xTF32 path (tmagemm.cu) for single problems
// whose operands are dense blocks (row stride ld, 16B aligned).  The residual
// (lo) copies of A and B live in the workspace.
struct TmaGemmArgs {
  int M, N, K;
  int tiles_n, splits, accumulate, c_vec, pad_;
  int gsplit;  // split-K partials reduced through `ws` by the tile's last CTA (no cluster)
  int nowait;  // persistent kernel launched behind an independent grid: no griddepcontrol.wait
  int tstore;  // persistent kernel: C written by TMA tensor stores (map in TmaProb::mAl)
  Operand C, bias;
  float* ws;   // gsplit: one BM x BN partial per CTA of the launch
  int* cnt;    // gsplit: zeroed per-tile arrival counters (left zero)
};
struct TmaOperands {
  int M, N, K;
  bool a_mn, b_mn;      // A(m,k) = A[k*lda + m] (MN-major) else A[m*lda + k]; B(k,n) = B[k*ldb + n] else B[n*ldb + k]
  const float* A;
  int64_t lda;
  const float* B;
  int64_t ldb;
  float* A_lo;          // tma_lo_floats(rows, cols) floats each
  float* B_lo;
  Operand C, bias;
  int accumulate;
  float* ws;           // optional split-K partial workspace (ws_floats floats) + zeroed tile counters
  int64_t ws_floats;
  int* cnt;
  int cnt_cap;
};
constexpr int kTmaGroup = 4;  // problems per grouped TMA GEMM launch
struct TmaProb {
  CUtensorMap mAh, mAl, mBh, mBl;
  TmaGemmArgs args;
  int cta0;
};
struct TmaGroup {
  TmaProb p[kTmaGroup];
  int n;
};
struct TmaGemmPlan {
  CUtensorMap mAh, mAl, mBh, mBl;
  TmaGemmArgs args;
  bool a_mn, b_mn;
  bool conv;  // residuals formed in shared memory by converter warps (no lo copies)
  bool a_tmem;  // conv with A's hi/lo split stored in TMEM (MMAs read only B from shared memory)
  bool lite;    // a_tmem, K per split <= 1024 (768 when split): 2 stages, one accumulator, two CTAs per SM
  bool pers;    // lite-shaped single-split problem with many tiles: persistent CTAs, double-buffered
                // TMEM accumulators, each tile's epilogue overlapping the next tile's mainloop
  const float* a_src;
  const float* b_src;
  float* a_lo;
  float* b_lo;
  int64_t a_ld, a_rows, a_cols, a_colsp, b_ld, b_rows, b_cols, b_colsp;
  int ctas;
  int grid_cap;  // persistent kernel: at most this many CTAs (0: one per SM)
  int64_t ws_floats;
  int cnt_cap;
  double flops;
};
bool tma_gemm_enabled();  // DG_TMA=0 disables (A/B checks)
bool tma_conv_enabled();  // DG_TMA_CONV=0: pre-split residual copies instead of in-smem conversion
bool tma_at_enabled();    // DG_TMA_AT=0: A's split in shared memory instead of TMEM
bool tma_gsplit_enabled();  // DG_TMA_GSPLIT=0: split-K through a cluster's shared memory instead of the workspace
bool tma_pers_enabled();  // DG_TMA_PERS=0: no persistent variant
bool tma_tstore_enabled();  // DG_TMA_TSTORE=0: persistent epilogue with thread stores instead of TMA stores
bool tma_lite_enabled();  // DG_TMA_LITE=0: no two-CTA-per-SM variant for short-K (per split) GEMMs
int64_t tma_lo_floats(int64_t rows, int64_t cols);
bool tma_gemm_make(const TmaOperands& o, TmaGemmPlan* out);
// split_a / split_b: (re)compute the residual copies before the GEMM
int launch_tma_gemm(const TmaGemmPlan& p, bool split_a, bool split_b, cudaStream_t s);
// grouped launches (in-smem conversion only): same kernel, disjoint outputs
bool tma_gemm_groupable(const TmaGemmPlan& a, const TmaGemmPlan& b);
void tma_gemm_regroup(TmaGemmPlan* const* ps, int n);  // one split factor for the group
int launch_tma_gemm_group(const TmaGemmPlan* const* ps, int n, cudaStream_t s);
int tma_prof_read(long long* out);  // diagnostics: DG_TMA_DBG bit 10 wait timestamps [5][256][2]

// ------------------------------------------------------------- trainers
struct TensorSeg { float* w; float* g; float* s0; float* s1; int64_t n; };
int update_chunk();
struct RuleArgs {
  int rule;  // 0 sgd 1 momentum 2 adagrad 3 adam
  float lr, momentum, adagrad_eps, beta1, beta2, adam_eps;
  float bc1, bc2;  // Adam bias corrections 1-beta^t (computed in double on host)
};
// dense multi-tensor apply over `nseg` segments (device table), zeroes grads
int launch_update_dense(const RuleArgs& r, const TensorSeg* segs_dev, int nseg, int64_t total, cudaStream_t s);
// sparse rows: for u < n_rows: row ids[u] of (w,g,s0,s1) with width dim; zeroes those grad rows
int launch_update_rows(const RuleArgs& r, float* w, float* g, float* s0, float* s1, int dim, const int64_t* ids,
                       int n_rows, cudaStream_t s);

int launch_scale(float* y, int64_t n, float alpha, cudaStream_t s);
int launch_fill(float* y, int64_t n, float v, cudaStream_t s);
// pack rows: out[u] = table[ids[u]] (for DP exchange)
int launch_pack_rows(const float* table, int dim, const int64_t* ids, float* out, int n, cudaStream_t s);

}  // namespace dg
