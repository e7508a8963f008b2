/*
 * rgnn.h — C-ABI of librgnn: one relational-GNN layer (RGCN / RGAT / HGT),
 * forward and backward, on a typed heterograph, for NVIDIA B200 (sm_100a).
 *
 * The operations are those of the Hector hot path of arxiv 2412.04747 Ch. 3
 * (PAPER.md = P:line, SPEC.md = S:line; SURVEY.md §8(b) lists this boundary):
 *   - graph build: type sort, dst-CSR, src-CSC, compact (relation, source) pair
 *     index ("precompute this mapping and store it in a CSR-like format",
 *     P:774 §3.3.2; emitted preprocessing "converting COO to CSR", §3.3.6)
 *   - layer forward: typed segment GEMM Y[S] = X[G] x W[T] over compact pairs
 *     (§3.3.3, algo:gemm_template P:901-918; compact materialization
 *     P:764-776; linear-operator reordering P:820-823), edge logits (g-SDDMM,
 *     P:578-588; lst:ir_example P:739-745), edge softmax (lst:ir_example P:730-738),
 *     aggregation by destination (g-SpMM; Eq. 3.1)
 *   - layer backward (§3.3.5) over the dst-CSR and the src-CSC.
 * The model readings (HGT formula, RGAT message, norms, slope ...) are listed in
 * DESIGN.md "Readings".
 *
 * Conventions
 *   - Every pointer argument documented "device" must point to device memory
 *     of the current CUDA device; "host" pointers are ordinary host memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     All device work is enqueued on it.  Only rgnn_graph_build synchronises the
 *     stream (once, to read back the pair count and the validation flag).
 *   - Calls never abort and never throw across the ABI.  They return an
 *     rgnn_status; on failure a thread-local message is available from
 *     rgnn_last_error().  Output buffers are unspecified after a failure.
 *   - Node ids are global; node type t owns ids [node_type_ptr[t], node_type_ptr[t+1])
 *     ("nodes are presorted", §3.4.1).  Edge e = (src[e], dst[e], rel[e]);
 *     edge ids are positions in the COO arrays.
 *   - Feature/weight matrices are dense row-major.  dtype RGNN_F32 = float,
 *     RGNN_BF16 = bfloat16 (uint16 bit patterns).  Gradients are always float.
 */
#ifndef RGNN_H_
#define RGNN_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define RGNN_API __attribute__((visibility("default")))
#else
#define RGNN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RGNN_OK = 0,
  RGNN_ERR_INVALID_ARG = 1,   /* NULL/inconsistent sizes/unknown enum */
  RGNN_ERR_OUT_OF_RANGE = 2,  /* node or relation id out of range (message names the first bad edge) */
  RGNN_ERR_UNSUPPORTED = 3,   /* shape not supported (e.g. d_out not in {16,32,64,128}) */
  RGNN_ERR_OOM = 4,           /* the allocator callback returned NULL */
  RGNN_ERR_CUDA = 5,          /* a CUDA runtime error (message has the CUDA error string) */
  RGNN_ERR_NCCL = 6           /* NCCL missing or an NCCL call failed (library-owned collectives) */
} rgnn_status;

/* Thread-local description of the last failure on this thread ("" if none). */
RGNN_API const char* rgnn_last_error(void);
/* Library version and build string (static storage). */
RGNN_API const char* rgnn_version(void);

/* Device allocator callbacks.  Every device buffer the library owns (graph
 * index arrays, sort temporaries) is obtained through them, so the caller's
 * allocator (e.g. PyTorch's caching allocator) owns all device memory.
 * alloc must return a 256-byte aligned device pointer or NULL.  If both are
 * NULL the library uses cudaMallocAsync / cudaFreeAsync on the build stream. */
typedef void* (*rgnn_alloc_fn)(size_t bytes, void* stream, void* ctx);
typedef void (*rgnn_free_fn)(void* ptr, void* stream, void* ctx);

/* ------------------------------------------------------------------ graph */
typedef struct rgnn_graph_s* rgnn_graph_t;

/* Build the typed graph (C1 of SURVEY.md §8(c)).
 *   num_nodes, num_node_types, node_type_ptr (host, int64[T+1], ptr[0]=0, ptr[T]=num_nodes)
 *   num_rels R >= 1; num_edges E >= 0 (E = 0 is valid, compaction ratio 1.0)
 *   src, dst, rel: device int32[E] COO arrays (read only; not retained)
 *   dst_lo, dst_hi: the owned destination range; edges whose dst lies outside are
 *     dropped (destination partitioning for multi-GPU runs); pass 0, num_nodes on 1 GPU.
 *   On success *out receives a handle owning all index arrays.
 * Bit-exact contract: every exported array equals the oracle's C1 definition:
 *   CSR order = stable sort of edge ids by (dst, rel, src, eid); CSC order by
 *   (src, rel, dst, eid); pairs = distinct (rel, src) ascending; edge_pair[e] = rank
 *   of (rel_e, src_e).
 * Errors: INVALID_ARG (bad counts/pointers), OUT_OF_RANGE (an id outside
 *   [0,N) or [0,R); message names the first offending edge index),
 *   UNSUPPORTED (E >= 2^31 or key width 2*ceil(log2 N)+ceil(log2 R) > 64),
 *   OOM, CUDA.  Synchronises `stream` once. */
RGNN_API rgnn_status rgnn_graph_build(int64_t num_nodes, int32_t num_node_types, const int64_t* node_type_ptr,
                             int32_t num_rels, int64_t num_edges, const int32_t* src, const int32_t* dst,
                             const int32_t* rel, int64_t dst_lo, int64_t dst_hi, rgnn_alloc_fn alloc,
                             rgnn_free_fn free_fn, void* alloc_ctx, void* stream, rgnn_graph_t* out);

/* Build options. */
typedef struct {
  int32_t compact;      /* 1: one projected row per distinct (relation, source) pair ("compact
                           materialization", §3.3.2; the default of rgnn_graph_build);
                           0: one row per edge ("vanilla materialization"): the "pairs" are the
                           edges ordered by (rel, src, dst, eid), U = E, edge_pair a bijection. */
  int32_t reserved[7];  /* must be 0 */
} rgnn_graph_opts;

/* rgnn_graph_build with options (NULL is not allowed; zero-initialise and set `compact`).
 * Same arguments, contract and errors as rgnn_graph_build, plus INVALID_ARG for bad options. */
RGNN_API rgnn_status rgnn_graph_build_opts(int64_t num_nodes, int32_t num_node_types, const int64_t* node_type_ptr,
                                           int32_t num_rels, int64_t num_edges, const int32_t* src,
                                           const int32_t* dst, const int32_t* rel, int64_t dst_lo, int64_t dst_hi,
                                           const rgnn_graph_opts* opts, rgnn_alloc_fn alloc, rgnn_free_fn free_fn,
                                           void* alloc_ctx, void* stream, rgnn_graph_t* out);

typedef struct {
  int64_t num_nodes;
  int64_t num_edges;        /* edges kept (dst in [dst_lo, dst_hi)) */
  int64_t num_pairs;        /* U = distinct (rel, src) pairs among kept edges */
  int64_t max_in_degree;
  int64_t max_pair_degree;  /* largest number of edges sharing one pair */
  int64_t dst_lo, dst_hi;
  int32_t num_node_types;
  int32_t num_rels;
  double compaction_ratio;  /* U / E (1.0 if E == 0), §3.4.3 */
  int64_t device_bytes;     /* device memory the handle owns now (index arrays, work lists, cached
                               tile plans and norms; grows when a layer first uses a new plan) */
} rgnn_graph_info;

RGNN_API rgnn_status rgnn_graph_get_info(rgnn_graph_t g, rgnn_graph_info* out_host);

typedef enum {
  RGNN_ARR_ETYPE_PTR = 0,    /* int32[R+1]  edges per relation prefix (etype_ptr) */
  RGNN_ARR_ROW_PTR = 1,      /* int32[N+1]  dst-CSR row pointer */
  RGNN_ARR_CSR_SRC = 2,      /* int32[E]    source of each CSR entry */
  RGNN_ARR_CSR_REL = 3,      /* int32[E]    relation of each CSR entry */
  RGNN_ARR_CSR_EID = 4,      /* int32[E]    edge id of each CSR entry */
  RGNN_ARR_COL_PTR = 5,      /* int32[N+1]  src-CSC column pointer */
  RGNN_ARR_CSC_DST = 6,      /* int32[E] */
  RGNN_ARR_CSC_REL = 7,      /* int32[E] */
  RGNN_ARR_CSC_EID = 8,      /* int32[E] */
  RGNN_ARR_PAIR_REL_PTR = 9, /* int32[R+1]  unique_etype_ptr */
  RGNN_ARR_PAIR_SRC = 10,    /* int32[U]    unique_row_idx */
  RGNN_ARR_EDGE_PAIR = 11,   /* int32[E]    pair of each edge id */
  RGNN_ARR_CSR_PAIR = 12,    /* int32[E]    pair of each CSR entry */
  RGNN_ARR_CSC_PAIR = 13,    /* int32[E]    pair of each CSC entry */
  RGNN_ARR_COUNT = 14
} rgnn_array;

/* Copy one index array (as typed above) into caller memory.
 * dst_device: device buffer of `bytes` >= count*4.  Enqueued on `stream`.
 * Errors: INVALID_ARG (unknown array, buffer too small). */
RGNN_API rgnn_status rgnn_graph_export(rgnn_graph_t g, rgnn_array which, void* dst_device, size_t bytes, void* stream);
/* Element count of an index array. */
RGNN_API rgnn_status rgnn_graph_array_size(rgnn_graph_t g, rgnn_array which, int64_t* count);
/* Free the handle and all its arrays (through the free callback).  NULL is a no-op. */
RGNN_API rgnn_status rgnn_graph_destroy(rgnn_graph_t g);

/* ------------------------------------------------------------------ layer */
typedef enum { RGNN_RGCN = 0, RGNN_RGAT = 1, RGNN_HGT = 2 } rgnn_model;
typedef enum { RGNN_F32 = 0, RGNN_BF16 = 1 } rgnn_dtype;
/* RGCN per-edge multiplier 1/c_{v,r} of Eq. 3.1 (reading g1):
 *   MEAN 1/|{e' in in(v): rel e' = rel e}|, SYM 1/sqrt(outdeg(src) indeg(dst)) (GCN A*),
 *   NONE 1, CUSTOM the caller's float[E] array indexed by edge id. */
typedef enum { RGNN_NORM_MEAN = 0, RGNN_NORM_SYM = 1, RGNN_NORM_NONE = 2, RGNN_NORM_CUSTOM = 3 } rgnn_norm_kind;

typedef struct {
  int32_t model;       /* rgnn_model */
  int32_t dtype;       /* rgnn_dtype of X, the weights and the projected tables */
  int32_t d_in;        /* input feature width, one of 16, 32, 64, 128, 256 */
  int32_t d_out;       /* output width, one of 16, 32, 64, 128 */
  int32_t self_loop;   /* RGCN: add X W_0 (virtual self-loop); ignored otherwise */
  int32_t norm_kind;   /* RGCN: rgnn_norm_kind */
  float leaky_slope;   /* RGAT LeakyReLU slope (reading g6: 0.2) */
  int32_t gemm_impl;   /* 0 auto (bf16 -> tcgen05 when d_in % 64 == 0), 1 force SIMT, 2 force tcgen05 */
  int32_t no_reorder;  /* 1: linear-operator reordering off (F1 ablation, tab:optimizations P:1142-1188).
                          HGT projects K = X Wk, V = X Wv per node and then K~ = K[src] Watt, M = V[src] Wmsg
                          per (rel, src) pair instead of folding Wk Watt / Wv Wmsg; RGAT computes the
                          destination term as (X[dst] W_r) . b_r per (rel, dst) pair (lst:ir_example's ht,
                          attt) instead of X[dst] . (W_r b_r) (fig:linear_opt).  Ignored for RGCN
                          (no weight-weight product).  0 = the default reordered path. */
  int32_t num_heads;   /* HGT attention heads H in {0 or 1, 2, 4, 8} (F2; the traversal template's head
                          loop, algo:traversal_template P:926): head h owns output columns h*dh .. (h+1)*dh-1,
                          dh = d_out / H (a multiple of 8 for bf16, 4 for f32); l_{e,h} = mu_r K~_{e,h} . q_{v,h}
                          / sqrt(dh), a softmax per (destination, head).  UNSUPPORTED > 1 for RGCN / RGAT. */
  int32_t hgt_tail;    /* 1: HGT layer tail (F2, reading b12): out_v = GELU(h_v) A_type(v) + X_v, where h is
                          the attention aggregation; needs d_in == d_out and weights.A.  0: out = h. */
} rgnn_layer_desc;

/* Layer weights, device pointers in the layer dtype (mu and edge_norm: float).
 * Unused fields may be NULL. */
typedef struct {
  const void* W;           /* RGCN, RGAT: [R][d_in][d_out]  relation weights W_r */
  const void* W0;          /* RGCN: [d_in][d_out]           self-loop weight W_0 (self_loop=1) */
  const void* a;           /* RGAT: [R][d_out]  source attention vector w_s[r] (lst:ir_example) */
  const void* b;           /* RGAT: [R][d_out]  destination attention vector w_t[r] */
  const void* Wk;          /* HGT: [T][d_in][d_out] key projection per node type */
  const void* Wq;          /* HGT: [T][d_in][d_out] query projection per node type */
  const void* Wv;          /* HGT: [T][d_in][d_out] value projection per node type */
  const void* Watt;        /* HGT: [R][d_out][d_out] relation attention matrix */
  const void* Wmsg;        /* HGT: [R][d_out][d_out] relation message matrix */
  const float* mu;         /* HGT: [R] relation prior (not trained) */
  const float* edge_norm;  /* RGCN, norm_kind CUSTOM: [E] by edge id */
  const void* A;           /* HGT with hgt_tail: [T][d_out][d_out] target-type output linear (A-linear) */
} rgnn_weights;

/* Weight gradients, device float pointers, same shapes as rgnn_weights.
 * A NULL field is not computed (gradient pruning). */
typedef struct {
  float* dW;
  float* dW0;
  float* da;
  float* db;
  float* dWk;
  float* dWq;
  float* dWv;
  float* dWatt;
  float* dWmsg;
  float* dA;
} rgnn_weight_grads;

/* Bytes of the `saved` buffer (forward -> backward activations) and of the
 * `scratch` buffer (temporaries of one forward or backward call).  Both are
 * caller-owned device memory, 256-byte aligned.
 * Errors: INVALID_ARG / UNSUPPORTED for a bad descriptor. */
RGNN_API rgnn_status rgnn_layer_workspace(rgnn_graph_t g, const rgnn_layer_desc* desc, size_t* saved_bytes,
                                 size_t* scratch_bytes);

/* ------------------------------------------------------------------ communicator (multi-GPU)
 * Destination-partitioned multi-GPU layer (north_star: "the graph is partitioned by
 * destination-node range ... projected source features are exchanged with NCCL all-gather"; the
 * paper itself is single-GPU, §3.6.2).  One process per GPU.  Rank k owns the node rows
 * [node_ptr[k], node_ptr[k+1]) (features, outputs, dX) and builds its graph with dst_lo = node_ptr[k],
 * dst_hi = node_ptr[k+1]: the in-edges of its destinations, with sources anywhere.  The layer calls
 * take the communicator and then:
 *   forward : all-gather X in place (rank k's rows are read, the other rows of X are overwritten),
 *             one ncclBroadcast per owner on a library-owned high-priority stream, each chunk
 *             signalled by an event so the pair GEMM of the sources already present runs while
 *             the next chunk is in flight; node-side projections (HGT Q, RGCN self-loop, tail)
 *             run on the owned rows only; out rows outside the owned range are left untouched.
 *   backward: reads dout rows of the owned range only; the pair-side dX contributions of every
 *             source are summed onto their owners (one in-place ncclReduce per owner: a
 *             reduce-scatter with uneven counts), so dX rows [node_ptr[k], node_ptr[k+1]) hold the
 *             full gradient on rank k (other rows: this rank's partial contributions); every
 *             requested weight gradient is summed on all ranks (ncclAllReduce).
 * The exchanged tensor is X (variant X): N * d_in * b bytes per layer, against U_global * k * d_out *
 * b for the projected per-pair rows (variant P); with d_in = d_out and U > N (every BASELINE
 * config) X is the smaller, rgnn_comm_exchange_bytes reports both.
 * NCCL is loaded at run time (libnccl.so.2; in a PyTorch process the NCCL torch loaded).
 * Results are deterministic for a fixed world size (NCCL's fixed reduction order), not across sizes. */
#define RGNN_COMM_ID_BYTES 128
typedef struct rgnn_comm_s* rgnn_comm_t;

/* A fresh NCCL unique id (RGNN_COMM_ID_BYTES bytes into id_out, host).  Call on one rank and
 * distribute the bytes to the others out of band (e.g. torch.distributed broadcast).
 * Errors: INVALID_ARG (NULL), NCCL (libnccl.so.2 missing or ncclGetUniqueId failed). */
RGNN_API rgnn_status rgnn_comm_unique_id(void* id_out);

/* Create this rank's communicator on the current CUDA device (collective: every rank must call it
 * with the same id, world and node_ptr).  node_ptr: host int64[world+1], node_ptr[0] = 0,
 * non-decreasing, node_ptr[world] = N: the owned node rows of every rank.
 * Errors: INVALID_ARG (bad rank / world / node_ptr), NCCL, CUDA. */
RGNN_API rgnn_status rgnn_comm_create(int32_t rank, int32_t world, const void* unique_id, const int64_t* node_ptr,
                                      rgnn_comm_t* out);
/* Destroy (synchronises the comm stream).  NULL is a no-op. */
RGNN_API rgnn_status rgnn_comm_destroy(rgnn_comm_t comm);
RGNN_API rgnn_status rgnn_comm_info(rgnn_comm_t comm, int32_t* rank, int32_t* world);
/* Bytes one layer forward would exchange per rank under variant X (all-gather of X) and variant P
 * (all-gather of the projected per-(rel, src) rows of the whole graph, num_pairs_global rows of k
 * projections: 2 for HGT [K~|M], 1 otherwise), and the variant the library runs (0 = X).
 * Errors: INVALID_ARG. */
RGNN_API rgnn_status rgnn_comm_exchange_bytes(const rgnn_layer_desc* desc, int64_t num_nodes, int64_t num_pairs_global,
                                              int64_t* bytes_x, int64_t* bytes_p, int32_t* variant);

/* Forward: out[N][d_out] (float, device) = the layer output of every destination row in the
 * graph's owned range [dst_lo, dst_hi) (all rows on one GPU); zero in-degree rows hold only the
 * self-loop term for RGCN, zero otherwise (reading g10).  Rows outside the owned range are not
 * written.  X: device [N][d_in] in the layer dtype (read-only without a communicator; with one,
 * rows outside the owned range are overwritten by the all-gather, see above).
 * saved: written, needed by backward.  comm: NULL on one GPU; otherwise a communicator whose
 * node_ptr[rank], node_ptr[rank+1] equal the graph's dst_lo, dst_hi.
 * Errors: INVALID_ARG (NULL pointers for the model, bad desc, graph range != comm range),
 * UNSUPPORTED, CUDA, NCCL. */
RGNN_API rgnn_status rgnn_layer_forward(rgnn_graph_t g, const rgnn_layer_desc* desc, const void* X, const rgnn_weights* w,
                               float* out, void* saved, void* scratch, rgnn_comm_t comm, void* stream);

/* Backward of L = sum(out * dout) (reading g12).  `out` is the forward output
 * (read by RGAT/HGT for the softmax backward row term G_v . out_v), `saved` the
 * buffer written by the matching forward.  dout rows of the owned range are read.
 * dX: device float [N][d_in] (NULL = not computed): every row is written — the full
 * gradient on one GPU; on a partitioned graph without a communicator, this range's
 * contributions (their sum over the ranges is the gradient); with a communicator, the owned
 * rows hold the full gradient after the call.  dW: per-field device float (NULL = pruned),
 * summed over the ranks with a communicator.  Every requested output is fully overwritten
 * (no accumulation into caller data).  X: as written by the forward.
 * Errors: as for forward. */
RGNN_API rgnn_status rgnn_layer_backward(rgnn_graph_t g, const rgnn_layer_desc* desc, const void* X, const rgnn_weights* w,
                                const float* out, const void* saved, const float* dout, float* dX,
                                const rgnn_weight_grads* dW, void* scratch, rgnn_comm_t comm, void* stream);

/* ------------------------------------------------------------------ A1 primitive: typed segment GEMM
 * The paper's GEMM template Y[S] = X[G] x W[T] (§3.3.3, algo:gemm_template P:901-918),
 * the operator the layer calls for every projection (compact rows P:764-776), exported on its own
 * so a caller (and the D3 d-sweep) can run it at any width.  Rows 0..R-1 are split into
 * num_segments contiguous segments; for every row i of segment s
 *     Y[i][0:N] = X[G(i)][0:K] . W[w(s)]        G(i) = gather[i] (identity when gather is NULL),
 *                                               w(s) = seg_weight[s] (s when seg_weight is NULL).
 * A plan holds the row tiles of one segmentation (tiles never cross a segment); it is built once
 * and reused by every call with that segmentation. */
typedef struct rgnn_segments_s* rgnn_segments_t;

/* seg_ptr: host int64[num_segments+1], non-decreasing, seg_ptr[0] = 0 (R = seg_ptr[num_segments]).
 * seg_weight: host int32[num_segments] or NULL.  Device memory through alloc/free_fn (NULL: the
 * library's cudaMallocAsync on `stream`).  The call synchronises `stream` once (tile upload).
 * Errors: INVALID_ARG (decreasing seg_ptr, negative weight index, NULL out), OOM, CUDA. */
RGNN_API rgnn_status rgnn_segment_plan_create(int32_t num_segments, const int64_t* seg_ptr, const int32_t* seg_weight,
                                              rgnn_alloc_fn alloc, rgnn_free_fn free_fn, void* alloc_ctx, void* stream,
                                              rgnn_segments_t* out);
RGNN_API rgnn_status rgnn_segment_plan_destroy(rgnn_segments_t p);

/* Scratch bytes of rgnn_segment_gemm for these widths (the K-major bf16 weight image of the
 * tensor-core path; 0 for f32).  num_weights = number of matrices in W. */
RGNN_API rgnn_status rgnn_segment_gemm_workspace(rgnn_segments_t p, int32_t dtype, int32_t K, int32_t N,
                                                 int32_t num_weights, size_t* scratch_bytes);

/* X: device [*][K] in `dtype`; gather: device int32[R] or NULL; W: device [num_weights][K][N] in
 * `dtype` ([num_weights][N][K] when trans_w = 1, i.e. Y = X W^T); Y: device [R][N] in y_dtype
 * (BF16 only for dtype BF16; F32 always), fully overwritten; scratch: >= the workspace size.
 * dtype BF16 runs on the tcgen05 tensor cores (fp32 accumulation in TMEM): K a multiple of 64,
 * K <= 8192, N in {16, 32, 64, 128} or a multiple of 256 (<= 8192).  dtype F32 runs the SIMT FFMA
 * kernel (no TF32): K a multiple of 16, N in {16, 32, 64, 128, 256}.  Enqueued on `stream`.
 * Errors: INVALID_ARG (NULL pointers, weight index >= num_weights is not checked on the device:
 * caller contract), UNSUPPORTED (widths), CUDA. */
RGNN_API rgnn_status rgnn_segment_gemm(rgnn_segments_t p, int32_t dtype, const void* X, const int32_t* gather, int32_t K,
                                       const void* W, int32_t num_weights, int32_t N, int32_t trans_w, void* Y,
                                       int32_t y_dtype, void* scratch, size_t scratch_bytes, void* stream);

/* ------------------------------------------------------------------ F4: training step around the layers
 * a stacked-layer training step.  The paper's training measurement computes
 * "the negative log-likelihood loss by comparing the output with a precomputed random label
 * tensor" (§3.4.1); BASELINE.json's AIFB/AM configs stack 2 RGAT layers.  Between layers
 * the activation is ReLU (DESIGN.md b13), the optimiser plain SGD (b15).
 * All calls enqueue on `stream` and never synchronise it. */

/* a[i] = max(h[i], 0) converted to `dtype` (the next layer's input X), i in [0, n).
 * h: device float[n]; a: device [n] in dtype (may alias h only for RGNN_F32).
 * Errors: INVALID_ARG (NULL with n > 0, bad dtype), CUDA. */
RGNN_API rgnn_status rgnn_relu_forward(int64_t n, const float* h, void* a, int32_t dtype, void* stream);

/* dh[i] = h[i] > 0 ? da[i] : 0 (ReLU'(0) = 0), i in [0, n).  h, da, dh: device float[n];
 * dh may alias da (in place).  Errors: INVALID_ARG, CUDA. */
RGNN_API rgnn_status rgnn_relu_backward(int64_t n, const float* h, const float* da, float* dh, void* stream);

/* Scratch bytes of rgnn_nll_loss for n rows (per-block partial sums; caller-owned device memory). */
RGNN_API rgnn_status rgnn_nll_loss_workspace(int64_t n, int32_t c, size_t* scratch_bytes);

/* Mean negative log-likelihood of log_softmax over each row of logits (DESIGN.md b14):
 *   loss = -(1/num_labeled) sum_{v: 0 <= labels[v] < c} log softmax(logits[v])[labels[v]]
 *   dlogits[v] = (softmax(logits[v]) - onehot(labels[v])) / num_labeled   (labelled rows)
 *   dlogits[v] = 0                                                        (labels[v] < 0)
 * logits: device float[n][c], row-major; labels: device int32[n]; c in [1, 1024].
 * num_labeled: the number of rows with a label in [0, c), known to the caller (it built the
 * labels).  loss: device float[1], written by the call's last kernel: NaN if the rows the
 * device counted as labelled differ from num_labeled, or any label is >= c (the device-side
 * error report; the call itself cannot see device data without a sync).  dlogits: device
 * float[n][c] or NULL (loss only).  Deterministic: fixed grid, fixed reduction order.
 * Errors: INVALID_ARG (NULL pointers, c out of range, scratch too small), CUDA. */
RGNN_API rgnn_status rgnn_nll_loss(int64_t n, int32_t c, const float* logits, const int32_t* labels,
                                   int64_t num_labeled, float* loss, float* dlogits, void* scratch,
                                   size_t scratch_bytes, void* stream);

/* One parameter tensor of an SGD update: master -= lr * grad (float, device, n elements);
 * then, when shadow != NULL, shadow = master converted to shadow_dtype (the copy the layers read,
 * e.g. bf16 weights of the tensor-core path).  For an f32 layer, master is the weight itself. */
typedef struct {
  float* master;
  const float* grad;
  void* shadow;
  int64_t n;
} rgnn_sgd_tensor;

/* Plain SGD (theta <- theta - lr dL/dtheta, no momentum / weight decay; reading b15) over
 * `count` tensors (host array) in one launch per 32 tensors.  shadow_dtype: rgnn_dtype.
 * Errors: INVALID_ARG (NULL pointers, negative n, bad dtype), CUDA. */
RGNN_API rgnn_status rgnn_sgd_update(int32_t count, const rgnn_sgd_tensor* tensors, float lr,
                                     int32_t shadow_dtype, void* stream);

/* ------------------------------------------------------------------ profiling
 * When enabled, every kernel the library launches is bracketed by CUDA events
 * on its launch stream.  rgnn_profile_read synchronises those events and
 * writes a JSON object {"kernel": {"launches": n, "ms": total}, ...} into buf. */
RGNN_API rgnn_status rgnn_profile_enable(int32_t on);
RGNN_API rgnn_status rgnn_profile_reset(void);
RGNN_API rgnn_status rgnn_profile_read(char* buf, size_t len);

/* Number of kernels launched by the library since load (all threads). */
RGNN_API int64_t rgnn_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* RGNN_H_ */
