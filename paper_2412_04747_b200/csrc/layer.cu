// Layer forward / backward orchestration (C-ABI rgnn_layer_*).
//
// Forward, per model:
//   RGCN  A1 P = X[pair_src] W_rel (pairs) [+ X W_0 into out]  ->  A5 out_v += sum c_e P_pair
//   RGAT  A2 y_r = W_r b_r ; A1 P = X[pair_src] W_rel with epilogue s_p = P_p . a_rel  ->  A3-A5 fused
//   HGT   A2 F_{r,t} = [mu_r/sqrt(d) Wk_t Watt_r | Wv_t Wmsg_r] ; A1 [K~|M] = X[pair_src] F_{rel,type(src)},
//         Q = X Wq_type  ->  A3-A5 fused
// Backward: A6 dst-major, A7 pair-major, A8 typed-GEMM backward (dX = dP W^T reduced by source,
// dW = X[pair_src]^T dP per segment, two-level deterministic), then A2 unfolding.
#include <algorithm>

#include "comm.cuh"
#include "ops.cuh"
#include "traverse.cuh"

namespace rgnn {

void graph_norms(rgnn_graph_s* g, int kind, const float* custom, cudaStream_t s, float** csr_norm,
                 float** csc_norm);

namespace {

constexpr int GEMM_ROWS = 64;    // SIMT GEMM tile rows
constexpr int TC_ROWS = 128;     // tcgen05 tile rows
constexpr int WGRAD_ROWS = 2048;  // rows per weight-gradient partial
constexpr int WSUM_ROWS = 256;    // rows per weighted-row-sum partial (seg_wsum)

struct Segs {
  std::string key;
  std::vector<int64_t> ptr;
  std::vector<int32_t> w;  // empty: identity
};

Segs seg_pair_rel(const rgnn_graph_s* g) {
  return {"pair_rel", std::vector<int64_t>(g->pair_rel_ptr_h.begin(), g->pair_rel_ptr_h.end()), {}};
}
// pairs by (rel, src type); the weight of a non-empty segment is its active-combination index
Segs seg_pair_rt(const rgnn_graph_s* g) {
  return {"pair_rt", std::vector<int64_t>(g->pair_rt_ptr_h.begin(), g->pair_rt_ptr_h.end()), g->act_of_rt_h};
}
Segs seg_node_type(const rgnn_graph_s* g) { return {"node_type", g->node_type_ptr, {}}; }
Segs seg_all_nodes(const rgnn_graph_s* g) { return {"all_nodes", {0, g->N}, {0}}; }
Segs seg_dpair_rel(const rgnn_graph_s* g) {
  return {"dpair_rel", std::vector<int64_t>(g->dpair_rel_ptr_h.begin(), g->dpair_rel_ptr_h.end()), {}};
}

// A destination-partitioned graph (multi-GPU) owns the rows [dst_lo, dst_hi): its
// destination-side node work (HGT Q and its gradients, the RGCN self-loop, the HGT tail) runs on
// those rows only.
bool partitioned(const rgnn_graph_s* g) { return g->dst_lo != 0 || g->dst_hi != g->N; }
Segs seg_node_type_own(const rgnn_graph_s* g) {
  if (!partitioned(g)) return seg_node_type(g);
  std::vector<int64_t> p(g->node_type_ptr);
  for (auto& x : p) x = std::min(std::max(x, g->dst_lo), g->dst_hi);
  return {"node_type_own", p, {}};
}
Segs seg_own_nodes(const rgnn_graph_s* g) {
  if (!partitioned(g)) return seg_all_nodes(g);
  return {"own_nodes", {g->dst_lo, g->dst_hi}, {0}};
}

// The pairs of segmentation `sg` whose source lies in rank k's node rows (sources ascend within
// every pair segment: pairs sort by (rel, src)); the gaps between the segments' sub-ranges are
// segments of weight -1 (no tiles), so the tile plan covers exactly the chunk.
Segs seg_chunk(rgnn_graph_s* g, const Segs& sg, const rgnn_comm_s* cm, int k) {
  if (g->pair_src_h.size() != (size_t)g->U) {
    g->pair_src_h.resize(g->U);
    if (g->U)
      RGNN_CUDA(cudaMemcpy(g->pair_src_h.data(), g->pair_src, g->U * sizeof(int32_t), cudaMemcpyDeviceToHost));
  }
  const int64_t lo = cm->node_ptr[k], hi = cm->node_ptr[k + 1];
  Segs out{sg.key + "/chunk" + std::to_string(k) + "of" + std::to_string(cm->world) + "@" + std::to_string(lo), {}, {}};
  const int nseg = (int)sg.ptr.size() - 1;
  const int32_t* ps = g->pair_src_h.data();
  for (int i = 0; i < nseg; ++i) {
    const int32_t* b = ps + sg.ptr[i];
    const int32_t* e = ps + sg.ptr[i + 1];
    const int64_t a0 = std::lower_bound(b, e, (int32_t)lo) - ps, a1 = std::lower_bound(b, e, (int32_t)hi) - ps;
    if (!out.ptr.empty()) out.w.push_back(-1);  // gap up to this sub-range
    out.ptr.push_back(a0);
    out.ptr.push_back(a1);
    out.w.push_back(sg.w.empty() ? i : sg.w[i]);
  }
  if (out.ptr.empty()) out.ptr = {0, 0}, out.w = {-1};
  return out;
}

int64_t count_tiles(const Segs& sg, int rows) {
  int64_t n = 0;
  for (size_t i = 0; i + 1 < sg.ptr.size(); ++i) n += (sg.ptr[i + 1] - sg.ptr[i] + rows - 1) / rows;
  return n;
}

const Plan& plan(rgnn_graph_s* g, const Segs& sg, int rows, cudaStream_t s) {
  return get_plan(g, sg.key, sg.ptr, sg.w, rows, s);
}

struct Ctx {
  rgnn_graph_s* g;
  const rgnn_layer_desc* d;
  int dt, D, Din;
  size_t esz;
  cudaStream_t s;
  int H = 1;  // attention heads (HGT; F2)
  rgnn_comm_s* comm = nullptr;  // multi-GPU exchange (NULL on one GPU)
};

void check_desc(const rgnn_graph_s* g, const rgnn_layer_desc* d) {
  RGNN_CHECK(g && d, RGNN_ERR_INVALID_ARG, "NULL graph or descriptor");
  RGNN_CHECK(d->model >= 0 && d->model <= 2, RGNN_ERR_INVALID_ARG, "unknown model");
  RGNN_CHECK(d->dtype == F32 || d->dtype == BF16, RGNN_ERR_INVALID_ARG, "unknown dtype");
  RGNN_CHECK(d->d_out == 16 || d->d_out == 32 || d->d_out == 64 || d->d_out == 128, RGNN_ERR_UNSUPPORTED,
             "d_out must be one of 16, 32, 64, 128");
  RGNN_CHECK(d->d_in == 16 || d->d_in == 32 || d->d_in == 64 || d->d_in == 128 || d->d_in == 256,
             RGNN_ERR_UNSUPPORTED, "d_in must be one of 16, 32, 64, 128, 256");
  if (d->model == RGNN_RGAT)
    RGNN_CHECK(d->d_in == d->d_out, RGNN_ERR_UNSUPPORTED, "RGAT needs d_in == d_out");
  RGNN_CHECK(d->norm_kind >= 0 && d->norm_kind <= 3, RGNN_ERR_INVALID_ARG, "unknown norm_kind");
  RGNN_CHECK(d->gemm_impl >= 0 && d->gemm_impl <= 2, RGNN_ERR_INVALID_ARG, "unknown gemm_impl");
  RGNN_CHECK(d->no_reorder == 0 || d->no_reorder == 1, RGNN_ERR_INVALID_ARG, "no_reorder must be 0 or 1");
  const int H = d->num_heads <= 1 ? 1 : d->num_heads;
  RGNN_CHECK(d->num_heads >= 0 && (H == 1 || H == 2 || H == 4 || H == 8), RGNN_ERR_UNSUPPORTED,
             "num_heads must be 0/1, 2, 4 or 8");
  RGNN_CHECK(H == 1 || d->model == RGNN_HGT, RGNN_ERR_UNSUPPORTED, "num_heads > 1 is implemented for HGT only");
  RGNN_CHECK(d->hgt_tail == 0 || d->hgt_tail == 1, RGNN_ERR_INVALID_ARG, "hgt_tail must be 0 or 1");
  RGNN_CHECK(!d->hgt_tail || (d->model == RGNN_HGT && d->d_in == d->d_out), RGNN_ERR_UNSUPPORTED,
             "hgt_tail needs an HGT layer with d_in == d_out (residual)");
  RGNN_CHECK((d->d_out / H) % (d->dtype == BF16 ? 8 : 4) == 0, RGNN_ERR_UNSUPPORTED,
             "head width d_out / num_heads must be a multiple of 8 (bf16) or 4 (f32) elements");
}

// linear-operator reordering off (F1 ablation)
bool hgt_nr(const rgnn_layer_desc* d) { return d->model == RGNN_HGT && d->no_reorder; }
bool rgat_nr(const rgnn_layer_desc* d) { return d->model == RGNN_RGAT && d->no_reorder; }

// ---------------------------------------------------------------- workspace layout
struct Saved {
  void* P = nullptr;       // RGAT P [U][D] / HGT KM [U][2D]  (layer dtype)
  void* Q = nullptr;       // HGT Q [N][D]
  float* spair = nullptr;  // RGAT s [U]
  float2* stats = nullptr; // RGAT/HGT (m, sum) [N]
  float* y = nullptr;      // RGAT y [R][D]
  float* a32 = nullptr;    // RGAT a as fp32 [R][D]
  float* F32 = nullptr;    // HGT folded weights fp32 [n_act][Din][2D] (active (r, t) combinations)
  void* Fdt = nullptr;     // HGT folded weights in bf16
  void* KV = nullptr;      // HGT, reordering off: [K|V] = X [Wk|Wv]_type  [N][2D] (layer dtype)
  void* Wkv = nullptr;     //   [T][Din][2D]   [Wk_t | Wv_t]
  void* Bd = nullptr;      //   [R][2D][2D]    blockdiag(mu_r/sqrt(d) Watt_r, Wmsg_r)
  void* Pt = nullptr;      // RGAT, reordering off: X[dst] W_rel per (rel, dst) pair [UD][D] (layer dtype)
  float* tdp = nullptr;    //   Pt . b_rel per (rel, dst) pair [UD]
  float* te = nullptr;     //   the same per CSR entry [E]
  float* b32 = nullptr;    //   b as fp32 [R][D]
  float* H32 = nullptr;    // HGT tail: the attention aggregation h [N][D] fp32
  void* GH = nullptr;      //   GELU(h) [N][D] layer dtype
};

void layout_saved(const Ctx& c, Arena& ar, Saved& o) {
  const rgnn_graph_s* g = c.g;
  const int64_t U = g->U, N = g->N, R = g->R, T = g->T;
  switch (c.d->model) {
    case RGNN_RGCN:
      break;
    case RGNN_RGAT:
      o.P = ar.take<char>(U * c.D * c.esz);
      o.spair = ar.take<float>(U);
      o.stats = ar.take<float2>(N);
      o.y = ar.take<float>(R * c.D);
      o.a32 = ar.take<float>(R * c.D);
      if (rgat_nr(c.d)) {
        o.Pt = ar.take<char>(g->UD * c.D * c.esz);
        o.tdp = ar.take<float>(g->UD);
        o.te = ar.take<float>(g->E);
        o.b32 = ar.take<float>(R * c.D);
      }
      break;
    case RGNN_HGT:
      o.P = ar.take<char>(U * 2 * c.D * c.esz);
      o.Q = ar.take<char>(N * c.D * c.esz);
      o.stats = ar.take<float2>(N * c.H);
      if (c.d->hgt_tail) {
        o.H32 = ar.take<float>(N * c.D);
        o.GH = ar.take<char>(N * c.D * c.esz);
      }
      if (hgt_nr(c.d)) {
        o.KV = ar.take<char>(N * 2 * c.D * c.esz);
        o.Wkv = ar.take<char>(T * c.Din * 2 * c.D * c.esz);
        o.Bd = ar.take<char>(R * 4 * c.D * c.D * c.esz);
      } else {
        const int64_t A = std::max<int64_t>(g->n_act, 1);
        o.F32 = ar.take<float>(A * c.Din * 2 * c.D);
        if (c.dt == BF16) o.Fdt = ar.take<char>(A * c.Din * 2 * c.D * c.esz);
      }
      break;
  }
}

struct FwdScratch {
  Partial pt;         // split-row partial states
  void* P = nullptr;  // RGCN P
  void* bt = nullptr;  // tcgen05 path: K-major bf16 image of the GEMM weights
  float* csr_norm = nullptr;
  float* csc_norm = nullptr;
};
struct BwdScratch {
  Partial pt;
  void* bt = nullptr;     // tcgen05 path: K-major bf16 weight image
  float2* ebuf = nullptr;
  void* dP = nullptr;     // [U][D] or HGT [U][2D], layer dtype
  void* dXp = nullptr;    // [U][Din] layer dtype
  void* dQ = nullptr;     // HGT [N][D] layer dtype; RGAT dX fallback [N][D] fp32
  float* wsum = nullptr;  // RGAT [U]
  void* bx = nullptr;     // RGAT [U][D]  sum_e dz_e X_d per pair, layer dtype (bf16 path: b7)
  float* Bsum = nullptr;  // RGAT [R][Din]
  float* dF = nullptr;    // HGT [n_act][Din][2D]
  float* dFu = nullptr;   // HGT [n_act][Din][2D] per-combination unfold products
  void* GQ = nullptr;     // HGT [N][2D] = [G_v | Q_v] layer dtype
  void* Gt = nullptr;     // RGCN bf16 path: the upstream gradient in bf16 [N][D]
  float4* nst = nullptr;  // HGT [N] (m, 1/sum, G.out, 0)
  float2* wts = nullptr;  // HGT [E][H] (alpha_e, dl_e) per CSR entry (weighted pair SpMM)
  float* dKV32 = nullptr;  // HGT reordering off: per-node [dK|dV] [N][2D] fp32
  void* dKVdt = nullptr;   //   the same in the layer dtype (bf16 path; = dKV32 on the fp32 path)
  float* dXkv = nullptr;   //   dKV [Wk|Wv]^T  [N][Din]
  float* dBd = nullptr;    //   [R][2D][2D]
  float* dWkv = nullptr;   //   [T][Din][2D]
  float* dz = nullptr;     // RGAT reordering off: dz per CSR entry [E]
  float* dt = nullptr;     //   per (rel, dst) pair [UD]
  void* dPt = nullptr;     //   dt (x) b_rel [UD][D] layer dtype
  void* dXd = nullptr;     //   dPt W_rel^T [UD][Din] layer dtype
  float* dWt = nullptr;    //   X[dst]^T dPt per relation [R][Din][D]
  float* dH = nullptr;     // HGT tail: dL/dh [N][D]
  void* Gdt = nullptr;     //   dout in the layer dtype [N][D]
  float* partial = nullptr;
  float* csr_norm = nullptr;
  float* csc_norm = nullptr;
};

// RGNN_PAIRW=1: the destination-major pass writes (alpha_e, dl_e) per CSR entry and the pair pass is a
// weighted SpMM (k_pair_spmm); default: the pair-major backward recomputes them per edge from the pair
// rows and a per-node record.  Measured on mag HGT (B200): SpMM 1.03 ms + 0.05 ms of extra destination-pass
// writes vs 1.15 ms recomputing, but the per-edge weight gather is a random 8-byte read (+1 GB of DRAM
// sectors), so the recomputing kernels stay the default.
bool pair_spmm() {
  static const bool on = [] {
    const char* v = getenv("RGNN_PAIRW");
    return v && v[0] == '1';
  }();
  return on;
}

// RGAT pair pass, two designs:
//  * recompute: the pair pass re-derives z_e / alpha_e / dz_e per edge from [G_v | X_v] records (256 B per
//    edge at d = 64 bf16) and writes per-pair bx rows, summed per relation into B_r;
//  * weighted SpMM: the destination pass writes (alpha_e, dz_e) per CSR entry, the pair pass gathers only the
//    G rows (128 B per edge) and B_r is a weighted row sum of X over the (rel, dst) runs of dz.
// The SpMM is the default: AM (E/UD = 2.4) 2.53 -> 2.39 ms per step; mag (E/UD = 14.5, one hub row) 4.35 ->
// 4.02 ms once the long (rel, dst) runs are summed in chunks (dpair_sum 0.38 -> 0.08 ms; before that the
// recompute design was the faster one on mag, 4.81 vs 4.85 ms).  RGNN_RGATW=0 selects the recompute design.
bool rgat_spmm(const rgnn_graph_s* g, const rgnn_layer_desc* d) {
  static const int mode = [] {
    const char* v = getenv("RGNN_RGATW");
    return v ? atoi(v) : -1;
  }();
  (void)g;
  if (d->model != RGNN_RGAT || d->no_reorder || mode == 0) return false;
  return true;
}

// elements of the largest K-major weight image any GEMM of the layer builds (tcgen05 path)
int64_t bt_elems(const Ctx& c) {
  const int64_t R = c.g->R, T = c.g->T, Din = c.Din, D = c.D;
  if (c.d->model != RGNN_HGT) return std::max(R, (int64_t)1) * Din * D;
  const int64_t A = std::max<int64_t>(c.g->n_act, 1);
  return std::max({A * Din * 2 * D, T * Din * D, R * 4 * D * D, T * Din * 2 * D});
}

void layout_partial(const Ctx& c, Arena& ar, Partial& pt) {
  const int64_t rows = c.g->rows.n_slots * c.D;
  const int64_t pairs = c.g->pairs.n_slots * (c.d->model == RGNN_RGCN ? c.D : 2 * c.D);
  pt.acc = ar.take<float>(std::max<int64_t>({rows, pairs, c.g->n_dpair_chunks, 1}));  // also dpair_sum_w's partials
  pt.stat = ar.take<float2>(std::max<int64_t>(std::max(c.g->rows.n_slots * c.H, c.g->pairs.n_slots), 1));
}

void layout_fwd_scratch(const Ctx& c, Arena& ar, FwdScratch& o) {
  layout_partial(c, ar, o.pt);
  if (c.dt == BF16) o.bt = ar.take<char>(bt_elems(c) * 2);
  if (c.d->model == RGNN_RGCN) {
    o.P = ar.take<char>(c.g->U * c.D * c.esz);
    if (c.d->norm_kind == RGNN_NORM_CUSTOM) {
      o.csr_norm = ar.take<float>(c.g->E);
      o.csc_norm = ar.take<float>(c.g->E);
    }
  }
}

void layout_bwd_scratch(const Ctx& c, Arena& ar, BwdScratch& o) {
  const rgnn_graph_s* g = c.g;
  const int64_t U = g->U, N = g->N, E = g->E, R = g->R, T = g->T;
  const int model = c.d->model;
  layout_partial(c, ar, o.pt);
  if (c.dt == BF16) o.bt = ar.take<char>(bt_elems(c) * 2);
  int64_t width = 0, tiles = 0;
  auto need = [&](const Segs& sg, int64_t k1k2) {
    width = std::max(width, k1k2 * count_tiles(sg, WGRAD_ROWS));
    tiles = std::max(tiles, count_tiles(sg, WGRAD_ROWS));
  };
  if (model == RGNN_RGCN) {
    o.dP = ar.take<char>(U * c.D * c.esz);
    o.dXp = ar.take<char>(U * c.Din * c.esz);
    if (c.dt == BF16) o.Gt = ar.take<char>(N * c.D * c.esz);
    if (c.d->norm_kind == RGNN_NORM_CUSTOM) {
      o.csr_norm = ar.take<float>(E);
      o.csc_norm = ar.take<float>(E);
    }
    need(seg_pair_rel(g), (int64_t)c.Din * c.D);
    need(seg_all_nodes(g), (int64_t)c.Din * c.D);
  } else if (model == RGNN_RGAT) {
    o.dP = ar.take<char>(U * c.D * c.esz);
    o.dXp = ar.take<char>(U * c.Din * c.esz);
    o.dQ = ar.take<float>(N * c.D);
    o.wsum = ar.take<float>(U);
    if (rgat_spmm(g, c.d)) {
      o.wts = ar.take<float2>(E);
      o.dt = ar.take<float>(std::max<int64_t>(g->UD, 1));
      width = std::max(width, (int64_t)c.D * count_tiles(seg_dpair_rel(g), WSUM_ROWS));
    } else {
      o.bx = ar.take<char>(U * c.D * c.esz);
    }
    o.Bsum = ar.take<float>(R * c.Din);
    o.GQ = ar.take<char>(N * 2 * c.D * c.esz);
    o.nst = ar.take<float4>(N);
    need(seg_pair_rel(g), (int64_t)c.Din * c.D);
    width = std::max(width, (int64_t)c.D * count_tiles(seg_pair_rel(g), WSUM_ROWS));
    if (rgat_nr(c.d)) {
      o.dz = ar.take<float>(E);
      o.dt = ar.take<float>(g->UD);
      o.dPt = ar.take<char>(g->UD * c.D * c.esz);
      o.dXd = ar.take<char>(g->UD * c.Din * c.esz);
      o.dWt = ar.take<float>(R * c.Din * c.D);
      need(seg_dpair_rel(g), (int64_t)c.Din * c.D);
      width = std::max(width, (int64_t)c.D * count_tiles(seg_dpair_rel(g), WSUM_ROWS));
    }
  } else {
    o.dP = ar.take<char>(U * 2 * c.D * c.esz);
    o.dQ = ar.take<char>(N * c.D * c.esz);
    if (c.d->hgt_tail) {
      o.dH = ar.take<float>(N * c.D);
      o.Gdt = ar.take<char>(N * c.D * c.esz);
    }
    o.GQ = ar.take<char>(N * 2 * c.D * c.esz);
    if (pair_spmm()) o.wts = ar.take<float2>(E * c.H);
    else o.nst = ar.take<float4>(N * c.H);
    need(seg_node_type(g), (int64_t)c.Din * c.D);
    if (hgt_nr(c.d)) {
      o.dXp = ar.take<char>(U * 2 * c.D * c.esz);  // per-pair [dK|dV] rows
      o.dKV32 = ar.take<float>(N * 2 * c.D);
      o.dKVdt = c.dt == BF16 ? ar.take<char>(N * 2 * c.D * c.esz) : nullptr;
      o.dXkv = ar.take<float>(N * c.Din);
      o.dBd = ar.take<float>(R * 4 * c.D * c.D);
      o.dWkv = ar.take<float>(T * c.Din * 2 * c.D);
      need(seg_pair_rel(g), (int64_t)4 * c.D * c.D);
      need(seg_node_type(g), (int64_t)c.Din * 2 * c.D);
    } else {
      o.dXp = ar.take<char>(U * c.Din * c.esz);
      o.dF = ar.take<float>(std::max<int64_t>(g->n_act, 1) * c.Din * 2 * c.D);
      o.dFu = ar.take<float>(std::max<int64_t>(g->n_act, 1) * c.Din * 2 * c.D);
      need(seg_pair_rt(g), (int64_t)c.Din * 2 * c.D);
    }
  }
  o.partial = ar.take<float>(std::max<int64_t>(width, 1));
}

// The per-source reduction of the pair dX rows is fused into the node GEMM's epilogue when sources
// have few pairs on average (RGNN_FUSE_RED = 0 / 1 forces it off / on).
bool fuse_pair_reduce(const rgnn_graph_s* g) {
  static const int mode = [] {
    const char* v = getenv("RGNN_FUSE_RED");
    return v ? atoi(v) : -1;
  }();
  if (mode >= 0) return mode == 1;
  return g->N > 0 && 2 * g->U <= 9 * g->N;  // U/N <= 4.5 (mag 1.6, AM 4.1)
}

// A8 fused (bf16, tcgen05): the per-pair dX rows dP W^T and the pair weight gradient X[src]^T dP
// from one read of dP (k_pair_bwd_tc).  RGNN_FUSE_PAIR=0 runs the two kernels separately.
bool fused_pair_bwd(const Ctx& c, const Segs& sg, const void* X, const void* dP, int K2, const void* W, void* dXp,
                    float* dWout, int num_w, float* partial) {
  static const bool on = [] {
    const char* v = getenv("RGNN_FUSE_PAIR");
    return !(v && v[0] == '0');
  }();
  if (!on || c.dt != BF16 || c.d->gemm_impl == 1 || !pair_bwd_tc_supported(c.Din, K2)) return false;
  PairBwdArgs a;
  a.plan = &plan(c.g, sg, WGRAD_ROWS, c.s);
  a.X = X; a.gather = c.g->pair_src; a.K1 = c.Din;
  a.dP = dP; a.K2 = K2; a.W = W; a.Y = dXp;
  a.out = dWout; a.num_w = num_w; a.partial = partial;
  a.rows = sg.ptr.empty() ? 0 : sg.ptr.back();
  a.name = "pair_bwd_fused";
  pair_bwd_tc(a, c.s);
  return true;
}

// Single-edge pairs get their pair-gradient rows from the destination-major pass (which holds
// alpha_e, dl_e, q_v and G_v of the edge) instead of a gather in the pair-major pass; used when
// they are >= 30 % of the pairs (AM 71 %, wikikg2 91 %, mag 14 %).  RGNN_SINGLE=0 / 1 forces it.
// Not by default for RGAT's weighted-SpMM pair pass (spmm = true): its destination pass then stays at
// the register count that admits the staged-y kernel, and the pair pass handles the single-edge pairs
// with one gathered G row each (AM RGAT 2.296 -> 2.276 ms, measured).
bool single_in_dst(const rgnn_graph_s* g, bool spmm = false) {
  static const int mode = [] {
    const char* v = getenv("RGNN_SINGLE");
    return v ? atoi(v) : -1;
  }();
  if (mode >= 0) return mode == 1;
  if (spmm) return false;
  const int64_t n_single = g->pairs.n_items - g->pairs.n_multi;
  return 10 * n_single >= 3 * g->U;
}

// ---------------------------------------------------------------- GEMM selection
// Returns true when the tcgen05 kernel ran (it honours the fused row reduction; SIMT does not).
bool gemm(const Ctx& c, const Segs& sg, GemmArgs a) {
  bool want_tc = c.d->gemm_impl == 2 || (c.d->gemm_impl == 0 && c.dt == BF16);
  if (want_tc && gemm_tc_supported(a)) {
    const Plan& p = plan(c.g, sg, TC_ROWS, c.s);
    a.tiles = p.tiles;
    a.ntiles = p.count;
    a.y_rows = sg.ptr.empty() ? 0 : sg.ptr.back();
    a.a_rows = a.gather ? c.g->N : a.y_rows;
    gemm_tc(a, c.s);
    return true;
  }
  const Plan& p = plan(c.g, sg, GEMM_ROWS, c.s);
  a.tiles = p.tiles;
  a.ntiles = p.count;
  gemm_simt(a, c.s);
  return false;
}

// The source-side pair GEMM.  With a communicator it runs chunk by chunk of source owners: the own
// rows first (present at once), then each other owner's pairs after the event of that owner's
// broadcast, so the all-gather of chunk k+1 overlaps the GEMM of chunk k.
void pair_gemm(const Ctx& c, const Segs& sg, const GemmArgs& a) {
  if (!c.comm) {
    gemm(c, sg, a);
    return;
  }
  for (int j = 0; j <= c.comm->world; ++j) {
    const int k = j == 0 ? c.comm->rank : j - 1;
    if (j > 0 && k == c.comm->rank) continue;
    comm_wait_chunk(c.comm, k, c.s);
    gemm(c, seg_chunk(c.g, sg, c.comm, k), a);
  }
}

// dX[u] (+)= sum of the per-pair rows of source u, for every source row (pairs reach sources outside
// the owned range).  Owned rows accumulate when `own_acc` (their node-side term was written first)
// or are skipped when `skip_own` (a GEMM epilogue already added them); other rows are overwritten.
void reduce_pair_rows(const Ctx& c, const void* rows, int K, float* dX, bool own_acc, bool skip_own = false) {
  const rgnn_graph_s* g = c.g;
  const int64_t lo = partitioned(g) ? g->dst_lo : 0, hi = partitioned(g) ? g->dst_hi : g->N;
  if (lo > 0) seg_reduce_rows(lo, g->src_pair_ptr, g->src_pairs, rows, c.dt, K, dX, false, c.s);
  if (!skip_own && hi > lo)
    seg_reduce_rows(hi - lo, g->src_pair_ptr + lo, g->src_pairs, rows, c.dt, K, dX + lo * K, own_acc, c.s);
  if (hi < g->N)
    seg_reduce_rows(g->N - hi, g->src_pair_ptr + hi, g->src_pairs, rows, c.dt, K, dX + hi * K, false, c.s);
}

void do_wgrad(const Ctx& c, const Segs& sg, const void* A, int a_dt, int K1, const int32_t* gather, const void* Bm,
              int b_dt, int K2, float* out, int num_w, float* partial, const char* name) {
  WgradArgs w;
  w.name = name;
  w.allow_tc = c.d->gemm_impl == 2 || (c.d->gemm_impl == 0 && c.dt == BF16);
  w.plan = &plan(c.g, sg, WGRAD_ROWS, c.s);
  w.A = A;
  w.a_dtype = a_dt;
  w.K1 = K1;
  w.gather = gather;
  w.Bm = Bm;
  w.b_dtype = b_dt;
  w.K2 = K2;
  w.out = out;
  w.num_w = num_w;
  w.partial = partial;
  wgrad(w, c.s);
}

// ---------------------------------------------------------------- forward
void forward(const Ctx& c, const void* X, const rgnn_weights* w, float* out, const Saved& sv,
             const FwdScratch& sc) {
  rgnn_graph_s* g = c.g;
  const int model = c.d->model;
  if (model == RGNN_RGCN) {
    RGNN_CHECK(w->W && (!c.d->self_loop || w->W0), RGNN_ERR_INVALID_ARG, "RGCN needs W (and W0 with self_loop)");
    GemmArgs a;
    a.A = X; a.a_dtype = c.dt; a.K = c.Din; a.gather = g->pair_src;
    a.B = w->W; a.b_dtype = c.dt; a.Y = sc.P; a.y_dtype = c.dt; a.N = c.D;
    a.num_w = g->R; a.bt_scratch = sc.bt;
    a.name = "gemm_pairs_fwd";
    if (c.d->self_loop) {  // owned rows only; first, while the other owners' rows are in flight
      GemmArgs b;
      b.A = X; b.a_dtype = c.dt; b.K = c.Din; b.B = w->W0; b.b_dtype = c.dt; b.Y = out; b.y_dtype = F32; b.N = c.D;
      b.num_w = 1; b.bt_scratch = sc.bt;
      b.name = "gemm_selfloop_fwd";
      gemm(c, seg_own_nodes(g), b);
    }
    pair_gemm(c, seg_pair_rel(g), a);
    float *cn = sc.csr_norm, *xn = sc.csc_norm;
    graph_norms(g, c.d->norm_kind, w->edge_norm, c.s, &cn, &xn);
    rgcn_fwd_traverse(g, c.dt, c.D, cn, sc.P, out, c.d->self_loop != 0, sc.pt, c.s);
  } else if (model == RGNN_RGAT) {
    RGNN_CHECK(w->W && w->a && w->b, RGNN_ERR_INVALID_ARG, "RGAT needs W, a, b");
    const bool nr = rgat_nr(c.d);
    if (!nr) rgat_tpath_vectors(g->R, c.Din, c.D, w->W, w->b, c.dt, sv.y, c.s);
    convert_f32((int64_t)g->R * c.D, w->a, c.dt, sv.a32, c.s);
    if (nr) {
      // reordering off: attt = (X[dst] W_rel) . b_rel per (rel, dst) pair (the listing's ht),
      // then expanded to the CSR entries
      convert_f32((int64_t)g->R * c.D, w->b, c.dt, sv.b32, c.s);
      GemmArgs t;
      t.A = X; t.a_dtype = c.dt; t.K = c.Din; t.gather = g->dpair_dst;
      t.B = w->W; t.b_dtype = c.dt; t.Y = sv.Pt; t.y_dtype = c.dt; t.N = c.D;
      t.dotvec = sv.b32; t.dotout = sv.tdp;
      t.num_w = g->R; t.bt_scratch = sc.bt;
      t.name = "gemm_dpairs_fwd";
      gemm(c, seg_dpair_rel(g), t);
      dpair_expand(g, sv.tdp, sv.te, c.s);
    }
    GemmArgs a;
    a.A = X; a.a_dtype = c.dt; a.K = c.Din; a.gather = g->pair_src;
    a.B = w->W; a.b_dtype = c.dt; a.Y = sv.P; a.y_dtype = c.dt; a.N = c.D;
    a.dotvec = sv.a32; a.dotout = sv.spair;
    a.num_w = g->R; a.bt_scratch = sc.bt;
    a.name = "gemm_pairs_fwd";
    pair_gemm(c, seg_pair_rel(g), a);
    rgat_fwd_traverse(g, c.dt, c.D, sv.P, sv.spair, X, sv.y, nr ? sv.te : nullptr, c.d->leaky_slope, out, sv.stats,
                      sc.pt, c.s);
  } else {
    RGNN_CHECK(w->Wk && w->Wq && w->Wv && w->Watt && w->Wmsg && w->mu, RGNN_ERR_INVALID_ARG,
               "HGT needs Wk, Wq, Wv, Watt, Wmsg, mu");
    if (hgt_nr(c.d)) {
      // reordering off: [K|V] = X [Wk|Wv]_type per node, then [K~|M] = [K|V][src] blockdiag(.)_rel per pair
      if (c.comm) comm_wait_all(c.comm, c.s);  // every node's K, V (source side)
      hgt_nr_weights(g->R, g->T, c.Din, c.D, c.D / c.H, w->Wk, w->Wv, w->Watt, w->Wmsg, w->mu, c.dt, sv.Wkv, sv.Bd, c.s);
      GemmArgs k;
      k.A = X; k.a_dtype = c.dt; k.K = c.Din; k.B = sv.Wkv; k.b_dtype = c.dt; k.Y = sv.KV; k.y_dtype = c.dt;
      k.N = 2 * c.D; k.num_w = g->T; k.bt_scratch = sc.bt;
      k.name = "gemm_nodes_kv";
      gemm(c, seg_node_type(g), k);
      GemmArgs a;
      a.A = sv.KV; a.a_dtype = c.dt; a.K = 2 * c.D; a.gather = g->pair_src;
      a.B = sv.Bd; a.b_dtype = c.dt; a.Y = sv.P; a.y_dtype = c.dt; a.N = 2 * c.D;
      a.num_w = g->R; a.bt_scratch = sc.bt;
      a.name = "gemm_pairs_fwd";
      gemm(c, seg_pair_rel(g), a);
    } else {
      // the weight fold (A2) runs on the side stream while the Q GEMM (independent of it) runs here
      hgt_fold(g, c.Din, c.D, c.D / c.H, w->Wk, w->Wv, w->Watt, w->Wmsg, w->mu, c.dt, sv.F32, sv.Fdt, fork_side(c.s));
      GemmArgs a;
      a.A = X; a.a_dtype = c.dt; a.K = c.Din; a.gather = g->pair_src;
      a.B = c.dt == F32 ? (const void*)sv.F32 : sv.Fdt; a.b_dtype = c.dt;
      a.Y = sv.P; a.y_dtype = c.dt; a.N = 2 * c.D;
      a.num_w = std::max(g->n_act, 1); a.bt_scratch = sc.bt;
      a.name = "gemm_pairs_fwd";
      GemmArgs q;  // Q of the owned destinations: first, it needs only this rank's rows of X
      q.A = X; q.a_dtype = c.dt; q.K = c.Din; q.B = w->Wq; q.b_dtype = c.dt; q.Y = sv.Q; q.y_dtype = c.dt; q.N = c.D;
      q.num_w = g->T; q.bt_scratch = sc.bt;
      q.name = "gemm_nodes_fwd";
      gemm(c, seg_node_type_own(g), q);
      join_side(c.s);
      pair_gemm(c, seg_pair_rt(g), a);
    }
    if (hgt_nr(c.d)) {
      GemmArgs q;
      q.A = X; q.a_dtype = c.dt; q.K = c.Din; q.B = w->Wq; q.b_dtype = c.dt; q.Y = sv.Q; q.y_dtype = c.dt; q.N = c.D;
      q.num_w = g->T; q.bt_scratch = sc.bt;
      q.name = "gemm_nodes_fwd";
      gemm(c, seg_node_type_own(g), q);
    }
    float* h = c.d->hgt_tail ? sv.H32 : out;
    hgt_fwd_traverse(g, c.dt, c.D, c.H, sv.P, sv.Q, h, sv.stats, sc.pt, c.s);
    if (c.d->hgt_tail) {  // out = GELU(h) A_type + X  (F2, reading b12)
      RGNN_CHECK(w->A, RGNN_ERR_INVALID_ARG, "hgt_tail needs weights.A");
      const int64_t o0 = g->dst_lo * c.D, on = (g->dst_hi - g->dst_lo) * c.D;  // owned rows
      gelu_fwd(on, h + o0, static_cast<char*>(sv.GH) + o0 * c.esz, c.dt, c.s);
      GemmArgs t;
      t.A = sv.GH; t.a_dtype = c.dt; t.K = c.D; t.B = w->A; t.b_dtype = c.dt; t.Y = out; t.y_dtype = F32; t.N = c.D;
      t.num_w = g->T; t.bt_scratch = sc.bt;
      t.name = "tail_gemm_fwd";
      gemm(c, seg_node_type_own(g), t);
      add_dt(on, static_cast<const char*>(X) + o0 * c.esz, c.dt, out + o0, c.s);
    }
  }
}

// ---------------------------------------------------------------- backward
// HGT with reordering off, after A6/A7 produced dQ and d[K~|M] per pair:
//   d[K|V] per pair = d[K~|M] Bd_rel^T, summed per source node;  dX = dQ Wq^T + d[K|V] [Wk|Wv]^T;
//   dBd_r = sum_{pairs of r} [K|V][src]^T d[K~|M];  d[Wk|Wv]_t = X_t^T d[K|V]_t;  dWq as reordered.
void hgt_backward_nr(const Ctx& c, const void* X, const rgnn_weights* w, const Saved& sv, float* dX,
                     const rgnn_weight_grads* dW, const BwdScratch& sc) {
  rgnn_graph_s* g = c.g;
  const bool need_kv = dX || dW->dWk || dW->dWv;
  if (need_kv) {
    GemmArgs a;
    a.A = sc.dP; a.a_dtype = c.dt; a.K = 2 * c.D; a.B = sv.Bd; a.b_dtype = c.dt; a.transB = true;
    a.Y = sc.dXp; a.y_dtype = c.dt; a.N = 2 * c.D;
    a.num_w = g->R; a.bt_scratch = sc.bt;
    a.name = "gemm_pairs_dkv";
    gemm(c, seg_pair_rel(g), a);
    seg_reduce_rows(g->N, g->src_pair_ptr, g->src_pairs, sc.dXp, c.dt, 2 * c.D, sc.dKV32, false, c.s);
    if (c.dt == BF16) convert_dt((int64_t)g->N * 2 * c.D, sc.dKV32, sc.dKVdt, BF16, c.s);
  }
  const void* dKV = c.dt == BF16 ? sc.dKVdt : (const void*)sc.dKV32;
  if (dX) {
    // source side (every node): dX = d[K|V] [Wk|Wv]^T; then the owned rows add dQ Wq^T
    GemmArgs k;
    k.A = dKV; k.a_dtype = c.dt; k.K = 2 * c.D; k.B = sv.Wkv; k.b_dtype = c.dt; k.transB = true;
    k.Y = dX; k.y_dtype = F32; k.N = c.Din;
    k.num_w = g->T; k.bt_scratch = sc.bt;
    k.name = "gemm_nodes_dkv_dx";
    gemm(c, seg_node_type(g), k);
    GemmArgs q;
    q.A = sc.dQ; q.a_dtype = c.dt; q.K = c.D; q.B = w->Wq; q.b_dtype = c.dt; q.transB = true;
    q.Y = sc.dXkv; q.y_dtype = F32; q.N = c.Din;
    q.num_w = g->T; q.bt_scratch = sc.bt;
    q.name = "gemm_nodes_dx";
    gemm(c, seg_node_type_own(g), q);
    const int64_t o0 = g->dst_lo * c.Din;
    add_f32((g->dst_hi - g->dst_lo) * c.Din, sc.dXkv + o0, dX + o0, c.s);
  }
  if (dW->dWq)
    do_wgrad(c, seg_node_type_own(g), X, c.dt, c.Din, nullptr, sc.dQ, c.dt, c.D, dW->dWq, g->T, sc.partial,
             "wgrad_nodes");
  const bool need_bd = dW->dWatt || dW->dWmsg, need_wkv = dW->dWk || dW->dWv;
  if (need_bd)
    do_wgrad(c, seg_pair_rel(g), sv.KV, c.dt, 2 * c.D, g->pair_src, sc.dP, c.dt, 2 * c.D, sc.dBd, g->R, sc.partial,
             "wgrad_pairs");
  if (need_wkv)
    do_wgrad(c, seg_node_type(g), X, c.dt, c.Din, nullptr, dKV, c.dt, 2 * c.D, sc.dWkv, g->T, sc.partial,
             "wgrad_nodes_kv");
  if (need_bd || need_wkv)
    hgt_nr_split(g->R, g->T, c.Din, c.D, c.D / c.H, need_bd ? sc.dBd : nullptr, need_wkv ? sc.dWkv : nullptr, w->mu, dW->dWk,
                 dW->dWv, dW->dWatt, dW->dWmsg, c.s);
}

// RGAT with reordering off: A6/A7 read the per-edge destination term t_e and write dz_e; the
// destination side is then explicit: dt_j = sum of dz over the (rel, dst) pair j, dPt_j = dt_j b_rel,
// dX[dst] += dPt W_rel^T, dW_rel += X[dst]^T dPt, db_rel = sum_j dt_j Pt_j.
void rgat_backward_nr(const Ctx& c, const void* X, const rgnn_weights* w, const float* out, const Saved& sv,
                      const float* G, float* dX, const rgnn_weight_grads* dW, const BwdScratch& sc) {
  rgnn_graph_s* g = c.g;
  rgat_bwd_dst(g, c.dt, c.D, sv.P, sv.spair, X, nullptr, sv.te, sc.dz, c.d->leaky_slope, sv.stats, G, out, nullptr,
               sc.GQ, sc.nst, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, sc.pt, c.s);
  rgat_bwd_pair(g, c.dt, c.D, sv.P, sv.spair, nullptr, sv.te, w->a, c.d->leaky_slope, sc.GQ, sc.nst, nullptr, sc.dP,
                sc.wsum, nullptr, false, sc.pt, c.s);
  dpair_sum(g, sc.dz, sc.dt, c.s);
  const bool dst_side = dX || dW->dW;
  if (dst_side) dpair_outer(plan(g, seg_dpair_rel(g), WSUM_ROWS, c.s), sc.dt, w->b, c.dt, c.D, sc.dPt, c.s);
  if (dX) {
    GemmArgs a;
    a.A = sc.dP; a.a_dtype = c.dt; a.K = c.D; a.B = w->W; a.b_dtype = c.dt; a.transB = true;
    a.Y = sc.dXp; a.y_dtype = c.dt; a.N = c.Din;
    a.num_w = g->R; a.bt_scratch = sc.bt;
    a.name = "gemm_pairs_dx";
    gemm(c, seg_pair_rel(g), a);
    seg_reduce_rows(g->N, g->src_pair_ptr, g->src_pairs, sc.dXp, c.dt, c.Din, dX, false, c.s);
    GemmArgs b = a;
    b.A = sc.dPt; b.Y = sc.dXd;
    b.name = "gemm_dpairs_dx";
    gemm(c, seg_dpair_rel(g), b);
    ensure_dst_dpairs(g, c.s);
    seg_reduce_rows(g->N, g->dst_dpair_ptr, g->dst_dpairs, sc.dXd, c.dt, c.Din, dX, true, c.s);
  }
  if (dW->dW) {
    do_wgrad(c, seg_pair_rel(g), X, c.dt, c.Din, g->pair_src, sc.dP, c.dt, c.D, dW->dW, g->R, sc.partial, "wgrad_pairs");
    do_wgrad(c, seg_dpair_rel(g), X, c.dt, c.Din, g->dpair_dst, sc.dPt, c.dt, c.D, sc.dWt, g->R, sc.partial,
             "wgrad_dpairs");
    add_f32((int64_t)g->R * c.Din * c.D, sc.dWt, dW->dW, c.s);
  }
  if (dW->db) {
    const Plan& pd = plan(g, seg_dpair_rel(g), WSUM_ROWS, c.s);
    seg_wsum(&pd, sc.dt, sv.Pt, c.dt, c.D, nullptr, dW->db, g->R, sc.partial, c.s);
  }
  if (dW->da) {
    const Plan& pp = plan(g, seg_pair_rel(g), WSUM_ROWS, c.s);
    seg_wsum(&pp, sc.wsum, sv.P, c.dt, c.D, nullptr, dW->da, g->R, sc.partial, c.s);
  }
}

void backward(const Ctx& c, const void* X, const rgnn_weights* w, const float* out, const Saved& sv,
              const float* G, float* dX, const rgnn_weight_grads* dW, const BwdScratch& sc) {
  rgnn_graph_s* g = c.g;
  const int model = c.d->model;
  rgnn_weight_grads none{};
  if (!dW) dW = &none;
  if (model == RGNN_RGCN) {
    float *cn = sc.csr_norm, *xn = sc.csc_norm;
    graph_norms(g, c.d->norm_kind, w->edge_norm, c.s, &cn, &xn);
    // upstream gradient in the table dtype: bf16 copy on the bf16 path (gathered per edge and the
    // A operand of the self-loop tcgen05 GEMMs), G itself on the fp32 path
    const void* Gt = G;
    if (c.dt == BF16) {  // owned rows: the only rows of G the layer reads
      const int64_t o0 = g->dst_lo * c.D;
      convert_dt((g->dst_hi - g->dst_lo) * c.D, G + o0, static_cast<char*>(sc.Gt) + o0 * c.esz, BF16, c.s);
      Gt = sc.Gt;
    }
    rgcn_bwd_pair(g, c.dt, c.D, xn, Gt, sc.dP, sc.pt, c.s);
    const bool fused = dX && dW->dW &&
                       fused_pair_bwd(c, seg_pair_rel(g), X, sc.dP, c.D, w->W, sc.dXp, dW->dW, g->R, sc.partial);
    if (dX) {
      GemmArgs a;
      a.A = sc.dP; a.a_dtype = c.dt; a.K = c.D; a.B = w->W; a.b_dtype = c.dt; a.transB = true;
      a.Y = sc.dXp; a.y_dtype = c.dt; a.N = c.Din;
      a.num_w = g->R; a.bt_scratch = sc.bt;
      a.name = "gemm_pairs_dx";
      if (!fused) gemm(c, seg_pair_rel(g), a);
      if (c.d->self_loop) {  // dX = G W0^T, then + the per-source sum of the pair rows
        GemmArgs b;
        b.A = Gt; b.a_dtype = c.dt; b.K = c.D; b.B = w->W0; b.b_dtype = c.dt; b.transB = true;
        b.Y = dX; b.y_dtype = F32; b.N = c.Din;
        b.num_w = 1; b.bt_scratch = sc.bt;
        b.name = "gemm_selfloop_dx";
        gemm(c, seg_own_nodes(g), b);
      }
      reduce_pair_rows(c, sc.dXp, c.Din, dX, c.d->self_loop != 0);
    }
    if (dW->dW && !fused)
      do_wgrad(c, seg_pair_rel(g), X, c.dt, c.Din, g->pair_src, sc.dP, c.dt, c.D, dW->dW, g->R, sc.partial, "wgrad_pairs");
    if (dW->dW0 && c.d->self_loop)
      do_wgrad(c, seg_own_nodes(g), X, c.dt, c.Din, nullptr, Gt, c.dt, c.D, dW->dW0, 1, sc.partial, "wgrad_selfloop");
  } else if (model == RGNN_RGAT && rgat_nr(c.d)) {
    rgat_backward_nr(c, X, w, out, sv, G, dX, dW, sc);
  } else if (model == RGNN_RGAT) {
    float* dXt = dX ? dX : static_cast<float*>(sc.dQ);
    const bool single = single_in_dst(g, sc.wts != nullptr);
    rgat_bwd_dst(g, c.dt, c.D, sv.P, sv.spair, X, sv.y, nullptr, nullptr, c.d->leaky_slope, sv.stats, G, out, dXt,
                 sc.GQ, sc.wts ? nullptr : sc.nst, single ? g->csr_single : nullptr, w->a, sc.dP,
                 sc.wts ? nullptr : sc.bx, sc.wsum, sc.wts, sc.pt, c.s);
    rgat_bwd_pair(g, c.dt, c.D, sv.P, sv.spair, sv.y, nullptr, w->a, c.d->leaky_slope, sc.GQ, sc.nst, sc.wts, sc.dP,
                  sc.wsum, sc.bx, single, sc.pt, c.s);
    const bool fused = dX && dW->dW &&
                       fused_pair_bwd(c, seg_pair_rel(g), X, sc.dP, c.D, w->W, sc.dXp, dW->dW, g->R, sc.partial);
    if (dX) {
      GemmArgs a;
      a.A = sc.dP; a.a_dtype = c.dt; a.K = c.D; a.B = w->W; a.b_dtype = c.dt; a.transB = true;
      a.Y = sc.dXp; a.y_dtype = c.dt; a.N = c.Din;
      a.num_w = g->R; a.bt_scratch = sc.bt;
      a.name = "gemm_pairs_dx";
      if (!fused) gemm(c, seg_pair_rel(g), a);
      reduce_pair_rows(c, sc.dXp, c.Din, dX, true);  // owned rows hold the t-path term of the dst pass
    }
    if ((dW->dW || dW->db) && sc.wts) {  // B_r = sum_{e in r} dz_e X[d_e]: dz summed per (rel, dst) run, then
      dpair_sum_w(g, sc.wts, sc.dt, sc.pt.acc, c.s);  // a weighted row sum of X[dpair_dst] per relation
      const Plan& pp = plan(g, seg_dpair_rel(g), WSUM_ROWS, c.s);
      seg_wsum(&pp, sc.dt, X, c.dt, c.D, g->dpair_dst, sc.Bsum, g->R, sc.partial, c.s);
    } else if (dW->dW || dW->db) {  // B_r = the sum of the per-pair bx rows of relation r
      const Plan& pp = plan(g, seg_pair_rel(g), WSUM_ROWS, c.s);
      seg_wsum(&pp, nullptr, sc.bx, c.dt, c.D, nullptr, sc.Bsum, g->R, sc.partial, c.s);
    }
    if (dW->dW && !fused)
      do_wgrad(c, seg_pair_rel(g), X, c.dt, c.Din, g->pair_src, sc.dP, c.dt, c.D, dW->dW, g->R, sc.partial, "wgrad_pairs");
    if (dW->dW || dW->db) rgat_tpath_grads(g->R, c.Din, c.D, w->W, w->b, c.dt, sc.Bsum, dW->dW, dW->db, c.s);
    if (dW->da) {
      const Plan& pp = plan(g, seg_pair_rel(g), WSUM_ROWS, c.s);
      seg_wsum(&pp, sc.wsum, sv.P, c.dt, c.D, nullptr, dW->da, g->R, sc.partial, c.s);
    }
  } else {
    const bool single = single_in_dst(g);
    hgt_bwd_dst(g, c.dt, c.D, c.H, sv.P, sv.Q, sv.stats, G, out, sc.dQ, sc.GQ, sc.nst,
                single ? g->csr_single : nullptr, sc.dP, sc.wts, sc.pt, c.s);
    hgt_bwd_pair(g, c.dt, c.D, c.H, sv.P, sc.GQ, sc.nst, sc.wts, sc.dP, single, sc.pt, c.s);
    if (hgt_nr(c.d)) {
      hgt_backward_nr(c, X, w, sv, dX, dW, sc);
      return;
    }
    const bool needF = dW->dWk || dW->dWv || dW->dWatt || dW->dWmsg;
    const bool fused = dX && needF &&
                       fused_pair_bwd(c, seg_pair_rt(g), X, sc.dP, 2 * c.D, sv.Fdt, sc.dXp, sc.dF,
                                      std::max(g->n_act, 1), sc.partial);
    // the small unfold kernels (dF -> dWk, dWv, dWatt, dWmsg) only need dF: on the side stream, overlapped
    // with the node dX GEMM and the node weight gradient (joined before the layer returns)
    const bool unfold_side = needF && fused;
    if (unfold_side)
      hgt_unfold(g, c.Din, c.D, c.D / c.H, w->Wk, w->Wv, w->Watt, w->Wmsg, w->mu, c.dt, sc.dF, sc.dFu, dW->dWk, dW->dWv,
                 dW->dWatt, dW->dWmsg, fork_side(c.s));
    if (dX) {
      // per-pair rows first, then the node GEMM whose epilogue adds them per source (tcgen05 path)
      GemmArgs a;
      a.A = sc.dP; a.a_dtype = c.dt; a.K = 2 * c.D; a.B = c.dt == F32 ? (const void*)sv.F32 : sv.Fdt; a.b_dtype = c.dt;
      a.transB = true;
      a.Y = sc.dXp; a.y_dtype = c.dt; a.N = c.Din;
      a.num_w = std::max(g->n_act, 1); a.bt_scratch = sc.bt;
      a.name = "gemm_pairs_dx";
      if (!fused) gemm(c, seg_pair_rt(g), a);
      GemmArgs q;
      q.A = sc.dQ; q.a_dtype = c.dt; q.K = c.D; q.B = w->Wq; q.b_dtype = c.dt; q.transB = true;
      q.Y = dX; q.y_dtype = F32; q.N = c.Din;
      q.num_w = g->T; q.bt_scratch = sc.bt;
      q.name = "gemm_nodes_dx";
      // few pairs per source (U/N small): the node GEMM's epilogue adds each row's per-pair dX rows
      // (one thread per row, whole 16-byte vectors), saving dX's write + re-read by seg_reduce_rows
      if (fuse_pair_reduce(g)) {
        q.red_ptr = g->src_pair_ptr; q.red_list = g->src_pairs; q.red_rows = sc.dXp; q.red_dtype = c.dt;
      }
      const bool reduced_own = gemm(c, seg_node_type_own(g), q) && q.red_ptr != nullptr;
      reduce_pair_rows(c, sc.dXp, c.Din, dX, true, reduced_own);
    }
    if (dW->dWq)
      do_wgrad(c, seg_node_type_own(g), X, c.dt, c.Din, nullptr, sc.dQ, c.dt, c.D, dW->dWq, g->T, sc.partial,
               "wgrad_nodes");
    if (unfold_side) {
      join_side(c.s);
    } else if (needF) {
      if (!fused)
        do_wgrad(c, seg_pair_rt(g), X, c.dt, c.Din, g->pair_src, sc.dP, c.dt, 2 * c.D, sc.dF, std::max(g->n_act, 1),
                 sc.partial, "wgrad_pairs");
      hgt_unfold(g, c.Din, c.D, c.D / c.H, w->Wk, w->Wv, w->Watt, w->Wmsg, w->mu, c.dt, sc.dF, sc.dFu, dW->dWk, dW->dWv,
                 dW->dWatt, dW->dWmsg, c.s);
    }
  }
}

// HGT tail backward: dh = (dout A_type^T) * GELU'(h); the attention layer's backward with G = dh and
// out = h; then dX += dout (residual) and dA_t = sum_{v of type t} GELU(h_v)^T dout_v.
void tail_backward(const Ctx& c, const void* X, const rgnn_weights* w, const Saved& sv, const float* dout, float* dX,
                   const rgnn_weight_grads* dW, const BwdScratch& sc) {
  rgnn_graph_s* g = c.g;
  RGNN_CHECK(w->A, RGNN_ERR_INVALID_ARG, "hgt_tail needs weights.A");
  const int64_t o0 = g->dst_lo * c.D, n = (g->dst_hi - g->dst_lo) * c.D;  // owned rows
  const void* Gt = dout;
  if (c.dt == BF16) {
    convert_dt(n, dout + o0, static_cast<char*>(sc.Gdt) + o0 * c.esz, BF16, c.s);
    Gt = sc.Gdt;
  }
  GemmArgs t;
  t.A = Gt; t.a_dtype = c.dt; t.K = c.D; t.B = w->A; t.b_dtype = c.dt; t.transB = true;
  t.Y = sc.dH; t.y_dtype = F32; t.N = c.D;
  t.num_w = g->T; t.bt_scratch = sc.bt;
  t.name = "tail_gemm_dx";
  gemm(c, seg_node_type_own(g), t);
  gelu_bwd(n, sv.H32 + o0, sc.dH + o0, c.s);
  backward(c, X, w, sv.H32, sv, sc.dH, dX, dW, sc);
  if (dX) add_f32(n, dout + o0, dX + o0, c.s);  // residual (d_in == d_out)
  if (dW && dW->dA)
    do_wgrad(c, seg_node_type_own(g), sv.GH, c.dt, c.D, nullptr, Gt, c.dt, c.D, dW->dA, g->T, sc.partial,
             "tail_wgrad");
}

Ctx make_ctx(rgnn_graph_s* g, const rgnn_layer_desc* d, void* stream, rgnn_comm_s* comm = nullptr) {
  check_desc(g, d);
  Ctx c{g, d, d->dtype, d->d_out, d->d_in, d->dtype == F32 ? (size_t)4 : (size_t)2,
        static_cast<cudaStream_t>(stream), d->num_heads <= 1 ? 1 : d->num_heads, comm};
  if (comm) {
    RGNN_CHECK((int64_t)comm->node_ptr.size() == comm->world + 1 && comm->node_ptr[comm->world] == g->N,
               RGNN_ERR_INVALID_ARG, "communicator node_ptr[world] != the graph's number of nodes");
    RGNN_CHECK(comm->node_ptr[comm->rank] == g->dst_lo && comm->node_ptr[comm->rank + 1] == g->dst_hi,
               RGNN_ERR_INVALID_ARG, "the graph's destination range differs from the communicator's rows of this rank");
  }
  return c;
}

// every requested weight gradient with its element count (the backward's all-reduce list)
std::vector<std::pair<float*, size_t>> grad_list(const Ctx& c, const rgnn_weight_grads* dW) {
  std::vector<std::pair<float*, size_t>> v;
  if (!dW) return v;
  const size_t R = c.g->R, T = c.g->T, Din = c.Din, D = c.D;
  v.push_back({dW->dW, R * Din * D});
  v.push_back({c.d->self_loop ? dW->dW0 : nullptr, Din * D});
  v.push_back({dW->da, R * D});
  v.push_back({dW->db, R * D});
  v.push_back({dW->dWk, T * Din * D});
  v.push_back({dW->dWq, T * Din * D});
  v.push_back({dW->dWv, T * Din * D});
  v.push_back({dW->dWatt, R * D * D});
  v.push_back({dW->dWmsg, R * D * D});
  v.push_back({c.d->hgt_tail ? dW->dA : nullptr, T * D * D});
  if (c.d->model == RGNN_RGCN) v.resize(2);
  else if (c.d->model == RGNN_RGAT) v = {v[0], v[2], v[3]};
  else v = {v[4], v[5], v[6], v[7], v[8], v[9]};
  return v;
}

}  // namespace
}  // namespace rgnn

using namespace rgnn;

extern "C" {

rgnn_status rgnn_layer_workspace(rgnn_graph_t g, const rgnn_layer_desc* d, size_t* saved_bytes,
                                 size_t* scratch_bytes) {
  return guarded([&] {
    Ctx c = make_ctx(g, d, nullptr);
    RGNN_CHECK(saved_bytes && scratch_bytes, RGNN_ERR_INVALID_ARG, "NULL output");
    Arena a;
    a.measure_only = true;
    Saved sv;
    layout_saved(c, a, sv);
    *saved_bytes = std::max<size_t>(a.off, 256);
    Arena f, b;
    f.measure_only = b.measure_only = true;
    FwdScratch fs;
    BwdScratch bs;
    layout_fwd_scratch(c, f, fs);
    layout_bwd_scratch(c, b, bs);
    *scratch_bytes = std::max<size_t>(std::max(f.off, b.off), 256);
  });
}

rgnn_status rgnn_layer_forward(rgnn_graph_t g, const rgnn_layer_desc* d, const void* X, const rgnn_weights* w,
                               float* out, void* saved, void* scratch, rgnn_comm_t comm, void* stream) {
  return guarded([&] {
    Ctx c = make_ctx(g, d, stream, comm);
    RGNN_CHECK(X && w && out && saved && scratch, RGNN_ERR_INVALID_ARG, "NULL argument");
    size_t sb = 0, xb = 0;
    RGNN_CHECK(rgnn_layer_workspace(g, d, &sb, &xb) == RGNN_OK, RGNN_ERR_INVALID_ARG, "workspace query failed");
    Arena a{static_cast<char*>(saved), sb};
    Saved sv;
    layout_saved(c, a, sv);
    Arena f{static_cast<char*>(scratch), xb};
    FwdScratch fs;
    layout_fwd_scratch(c, f, fs);
    if (comm)  // in-place all-gather of X by owner chunks, overlapped with the pair GEMM (pair_gemm)
      comm_allgather_rows_begin(comm, const_cast<void*>(X), (size_t)c.Din * c.esz, c.s);
    forward(c, X, w, out, sv, fs);
    if (comm) comm_wait_all(comm, c.s);  // X complete on return (the backward reads it)
  });
}

rgnn_status rgnn_layer_backward(rgnn_graph_t g, const rgnn_layer_desc* d, const void* X, const rgnn_weights* w,
                                const float* out, const void* saved, const float* dout, float* dX,
                                const rgnn_weight_grads* dW, void* scratch, rgnn_comm_t comm, void* stream) {
  return guarded([&] {
    Ctx c = make_ctx(g, d, stream, comm);
    RGNN_CHECK(X && w && saved && dout && scratch, RGNN_ERR_INVALID_ARG, "NULL argument");
    RGNN_CHECK(d->model == RGNN_RGCN || out, RGNN_ERR_INVALID_ARG, "RGAT/HGT backward needs the forward output");
    size_t sb = 0, xb = 0;
    RGNN_CHECK(rgnn_layer_workspace(g, d, &sb, &xb) == RGNN_OK, RGNN_ERR_INVALID_ARG, "workspace query failed");
    Arena a{static_cast<char*>(const_cast<void*>(saved)), sb};
    Saved sv;
    layout_saved(c, a, sv);
    Arena b{static_cast<char*>(scratch), xb};
    BwdScratch bs;
    layout_bwd_scratch(c, b, bs);
    if (d->hgt_tail) {
      tail_backward(c, X, w, sv, dout, dX, dW, bs);
    } else {
      backward(c, X, w, out, sv, dout, dX, dW, bs);
    }
    if (comm) comm_reduce_grads(comm, dX, c.Din, grad_list(c, dW), c.s);
  });
}

}  // extern "C"

extern "C" rgnn_status rgnn_comm_exchange_bytes(const rgnn_layer_desc* d, int64_t num_nodes, int64_t num_pairs_global,
                                                int64_t* bytes_x, int64_t* bytes_p, int32_t* variant) {
  return guarded([&] {
    RGNN_CHECK(d && bytes_x && bytes_p && variant && num_nodes >= 0 && num_pairs_global >= 0, RGNN_ERR_INVALID_ARG,
               "bad argument");
    const int64_t b = d->dtype == RGNN_BF16 ? 2 : 4, k = d->model == RGNN_HGT ? 2 : 1;
    *bytes_x = num_nodes * d->d_in * b;
    *bytes_p = num_pairs_global * k * d->d_out * b;
    *variant = 0;  // X (the only variant implemented; the smaller one whenever U_global * k * d_out >= N * d_in)
  });
}
