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
Segs seg_pair_rt(const rgnn_graph_s* g) {
  return {"pair_rt", std::vector<int64_t>(g->pair_rt_ptr_h.begin(), g->pair_rt_ptr_h.end()), {}};
}
Segs seg_node_type(const rgnn_graph_s* g) { return {"node_type", g->node_type_ptr, {}}; }
Segs seg_all_nodes(const rgnn_graph_s* g) { return {"all_nodes", {0, g->N}, {0}}; }
Segs seg_dpair_rel(const rgnn_graph_s* g) {
  return {"dpair_rel", std::vector<int64_t>(g->dpair_rel_ptr_h.begin(), g->dpair_rel_ptr_h.end()), {}};
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
}

// ---------------------------------------------------------------- workspace layout
struct Saved {
  void* P = nullptr;       // RGAT P [U][D] / HGT KM [U][2D]  (layer dtype)
  void* Q = nullptr;       // HGT Q [N][D]
  float* spair = nullptr;  // RGAT s [U]
  float2* stats = nullptr; // RGAT/HGT (m, sum) [N]
  float* y = nullptr;      // RGAT y [R][D]
  float* a32 = nullptr;    // RGAT a as fp32 [R][D]
  float* F32 = nullptr;    // HGT folded weights fp32 [R*T][Din][2D]
  void* Fdt = nullptr;     // HGT folded weights in bf16
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
      break;
    case RGNN_HGT:
      o.P = ar.take<char>(U * 2 * c.D * c.esz);
      o.Q = ar.take<char>(N * c.D * c.esz);
      o.stats = ar.take<float2>(N);
      o.F32 = ar.take<float>(R * T * c.Din * 2 * c.D);
      if (c.dt == BF16) o.Fdt = ar.take<char>(R * T * c.Din * 2 * c.D * c.esz);
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
  float* bx = nullptr;    // RGAT [U][D]  sum_e dz_e X_d per pair
  float* Bsum = nullptr;  // RGAT [R][Din]
  float* dF = nullptr;    // HGT [R*T][Din][2D]
  void* GQ = nullptr;     // HGT [N][2D] = [G_v | Q_v] layer dtype
  void* Gt = nullptr;     // RGCN bf16 path: the upstream gradient in bf16 [N][D]
  float4* nst = nullptr;  // HGT [N] (m, 1/sum, G.out, 0)
  float* partial = nullptr;
  float* csr_norm = nullptr;
  float* csc_norm = nullptr;
};

void layout_partial(const Ctx& c, Arena& ar, Partial& pt) {
  const int64_t rows = c.g->rows.n_slots * c.D;
  const int64_t pairs = c.g->pairs.n_slots * (c.d->model == RGNN_RGCN ? c.D : 2 * c.D);
  pt.acc = ar.take<float>(std::max<int64_t>(std::max(rows, pairs), 1));
  pt.stat = ar.take<float2>(std::max<int64_t>(std::max(c.g->rows.n_slots, c.g->pairs.n_slots), 1));
}

void layout_fwd_scratch(const Ctx& c, Arena& ar, FwdScratch& o) {
  layout_partial(c, ar, o.pt);
  if (c.dt == BF16) {
    const int64_t R = c.g->R, T = c.g->T;
    int64_t n = c.d->model == RGNN_HGT ? std::max(R * T * c.Din * 2 * c.D, T * c.Din * c.D)
                                       : std::max(R, (int64_t)1) * c.Din * c.D;
    o.bt = ar.take<char>(n * 2);
  }
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
  if (c.dt == BF16) {
    int64_t n = model == RGNN_HGT ? std::max(R * T * c.Din * 2 * c.D, T * c.Din * c.D)
                                  : std::max(R, (int64_t)1) * c.Din * c.D;
    o.bt = ar.take<char>(n * 2);
  }
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
    o.bx = ar.take<float>(U * c.D);
    o.Bsum = ar.take<float>(R * c.Din);
    o.GQ = ar.take<char>(N * 2 * c.D * c.esz);
    o.nst = ar.take<float4>(N);
    need(seg_pair_rel(g), (int64_t)c.Din * c.D);
    width = std::max(width, (int64_t)c.D * count_tiles(seg_pair_rel(g), WSUM_ROWS));
  } else {
    o.dP = ar.take<char>(U * 2 * c.D * c.esz);
    o.dXp = ar.take<char>(U * c.Din * c.esz);
    o.dQ = ar.take<char>(N * c.D * c.esz);
    o.dF = ar.take<float>(R * T * c.Din * 2 * c.D);
    o.GQ = ar.take<char>(N * 2 * c.D * c.esz);
    o.nst = ar.take<float4>(N);
    need(seg_pair_rt(g), (int64_t)c.Din * 2 * c.D);
    need(seg_node_type(g), (int64_t)c.Din * c.D);
  }
  o.partial = ar.take<float>(std::max<int64_t>(width, 1));
}

// ---------------------------------------------------------------- GEMM selection
// Returns true when the tcgen05 kernel ran (it honours the fused row reduction; SIMT does not).
bool gemm(const Ctx& c, const Segs& sg, GemmArgs a) {
  bool want_tc = c.d->gemm_impl == 2 || (c.d->gemm_impl == 0 && c.dt == BF16);
  if (want_tc && gemm_tc_supported(a)) {
    const Plan& p = plan(c.g, sg, TC_ROWS, c.s);
    a.tiles = p.tiles;
    a.ntiles = p.count;
    gemm_tc(a, c.s);
    return true;
  }
  const Plan& p = plan(c.g, sg, GEMM_ROWS, c.s);
  a.tiles = p.tiles;
  a.ntiles = p.count;
  gemm_simt(a, c.s);
  return false;
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
    gemm(c, seg_pair_rel(g), a);
    if (c.d->self_loop) {
      GemmArgs b;
      b.A = X; b.a_dtype = c.dt; b.K = c.Din; b.B = w->W0; b.b_dtype = c.dt; b.Y = out; b.y_dtype = F32; b.N = c.D;
      b.num_w = 1; b.bt_scratch = sc.bt;
      b.name = "gemm_selfloop_fwd";
      gemm(c, seg_all_nodes(g), b);
    }
    float *cn = sc.csr_norm, *xn = sc.csc_norm;
    graph_norms(g, c.d->norm_kind, w->edge_norm, c.s, &cn, &xn);
    rgcn_fwd_traverse(g, c.dt, c.D, cn, sc.P, out, c.d->self_loop != 0, sc.pt, c.s);
  } else if (model == RGNN_RGAT) {
    RGNN_CHECK(w->W && w->a && w->b, RGNN_ERR_INVALID_ARG, "RGAT needs W, a, b");
    rgat_tpath_vectors(g->R, c.Din, c.D, w->W, w->b, c.dt, sv.y, c.s);
    convert_f32((int64_t)g->R * c.D, w->a, c.dt, sv.a32, c.s);
    GemmArgs a;
    a.A = X; a.a_dtype = c.dt; a.K = c.Din; a.gather = g->pair_src;
    a.B = w->W; a.b_dtype = c.dt; a.Y = sv.P; a.y_dtype = c.dt; a.N = c.D;
    a.dotvec = sv.a32; a.dotout = sv.spair;
    a.num_w = g->R; a.bt_scratch = sc.bt;
    a.name = "gemm_pairs_fwd";
    gemm(c, seg_pair_rel(g), a);
    rgat_fwd_traverse(g, c.dt, c.D, sv.P, sv.spair, X, sv.y, c.d->leaky_slope, out, sv.stats, sc.pt, c.s);
  } else {
    RGNN_CHECK(w->Wk && w->Wq && w->Wv && w->Watt && w->Wmsg && w->mu, RGNN_ERR_INVALID_ARG,
               "HGT needs Wk, Wq, Wv, Watt, Wmsg, mu");
    hgt_fold(g->R, g->T, c.Din, c.D, w->Wk, w->Wv, w->Watt, w->Wmsg, w->mu, c.dt, sv.F32, sv.Fdt, c.s);
    GemmArgs a;
    a.A = X; a.a_dtype = c.dt; a.K = c.Din; a.gather = g->pair_src;
    a.B = c.dt == F32 ? (const void*)sv.F32 : sv.Fdt; a.b_dtype = c.dt;
    a.Y = sv.P; a.y_dtype = c.dt; a.N = 2 * c.D;
    a.num_w = g->R * g->T; a.bt_scratch = sc.bt;
    a.name = "gemm_pairs_fwd";
    gemm(c, seg_pair_rt(g), a);
    GemmArgs q;
    q.A = X; q.a_dtype = c.dt; q.K = c.Din; q.B = w->Wq; q.b_dtype = c.dt; q.Y = sv.Q; q.y_dtype = c.dt; q.N = c.D;
    q.num_w = g->T; q.bt_scratch = sc.bt;
    q.name = "gemm_nodes_fwd";
    gemm(c, seg_node_type(g), q);
    hgt_fwd_traverse(g, c.dt, c.D, sv.P, sv.Q, out, sv.stats, sc.pt, c.s);
  }
}

// ---------------------------------------------------------------- backward
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
    if (c.dt == BF16) {
      convert_dt((int64_t)g->N * c.D, G, sc.Gt, BF16, c.s);
      Gt = sc.Gt;
    }
    rgcn_bwd_pair(g, c.dt, c.D, xn, Gt, sc.dP, sc.pt, c.s);
    if (dX) {
      GemmArgs a;
      a.A = sc.dP; a.a_dtype = c.dt; a.K = c.D; a.B = w->W; a.b_dtype = c.dt; a.transB = true;
      a.Y = sc.dXp; a.y_dtype = c.dt; a.N = c.Din;
      a.num_w = g->R; a.bt_scratch = sc.bt;
      a.name = "gemm_pairs_dx";
      gemm(c, seg_pair_rel(g), a);
      if (c.d->self_loop) {  // dX = G W0^T, then + the per-source sum of the pair rows
        GemmArgs b;
        b.A = Gt; b.a_dtype = c.dt; b.K = c.D; b.B = w->W0; b.b_dtype = c.dt; b.transB = true;
        b.Y = dX; b.y_dtype = F32; b.N = c.Din;
        b.num_w = 1; b.bt_scratch = sc.bt;
        b.name = "gemm_selfloop_dx";
        gemm(c, seg_all_nodes(g), b);
      }
      seg_reduce_rows(g->N, g->src_pair_ptr, g->src_pairs, sc.dXp, c.dt, c.Din, dX, c.d->self_loop != 0, c.s);
    }
    if (dW->dW) do_wgrad(c, seg_pair_rel(g), X, c.dt, c.Din, g->pair_src, sc.dP, c.dt, c.D, dW->dW, g->R, sc.partial, "wgrad_pairs");
    if (dW->dW0 && c.d->self_loop)
      do_wgrad(c, seg_all_nodes(g), X, c.dt, c.Din, nullptr, Gt, c.dt, c.D, dW->dW0, 1, sc.partial, "wgrad_selfloop");
  } else if (model == RGNN_RGAT) {
    float* dXt = dX ? dX : static_cast<float*>(sc.dQ);
    rgat_bwd_dst(g, c.dt, c.D, sv.P, sv.spair, X, sv.y, c.d->leaky_slope, sv.stats, G, out, dXt, sc.GQ, sc.nst, sc.pt,
                 c.s);
    rgat_bwd_pair(g, c.dt, c.D, sv.P, sv.spair, sv.y, w->a, c.d->leaky_slope, sc.GQ, sc.nst, sc.dP, sc.wsum, sc.bx,
                  sc.pt, c.s);
    if (dX) {
      GemmArgs a;
      a.A = sc.dP; a.a_dtype = c.dt; a.K = c.D; a.B = w->W; a.b_dtype = c.dt; a.transB = true;
      a.Y = sc.dXp; a.y_dtype = c.dt; a.N = c.Din;
      a.num_w = g->R; a.bt_scratch = sc.bt;
      a.name = "gemm_pairs_dx";
      gemm(c, seg_pair_rel(g), a);
      seg_reduce_rows(g->N, g->src_pair_ptr, g->src_pairs, sc.dXp, c.dt, c.Din, dX, true, c.s);
    }
    if (dW->dW || dW->db) {  // B_r = sum_{e in r} dz_e X[d_e] = sum of the per-pair bx rows of relation r
      const Plan& pp = plan(g, seg_pair_rel(g), WSUM_ROWS, c.s);
      seg_wsum(&pp, nullptr, sc.bx, F32, c.D, nullptr, sc.Bsum, g->R, sc.partial, c.s);
    }
    if (dW->dW) do_wgrad(c, seg_pair_rel(g), X, c.dt, c.Din, g->pair_src, sc.dP, c.dt, c.D, dW->dW, g->R, sc.partial, "wgrad_pairs");
    if (dW->dW || dW->db) rgat_tpath_grads(g->R, c.Din, c.D, w->W, w->b, c.dt, sc.Bsum, dW->dW, dW->db, c.s);
    if (dW->da) {
      const Plan& pp = plan(g, seg_pair_rel(g), WSUM_ROWS, c.s);
      seg_wsum(&pp, sc.wsum, sv.P, c.dt, c.D, nullptr, dW->da, g->R, sc.partial, c.s);
    }
  } else {
    hgt_bwd_dst(g, c.dt, c.D, sv.P, sv.Q, sv.stats, G, out, sc.dQ, sc.GQ, sc.nst, sc.pt, c.s);
    hgt_bwd_pair(g, c.dt, c.D, sv.P, sc.GQ, sc.nst, sc.dP, sc.pt, c.s);
    if (dX) {
      // per-pair rows first, then the node GEMM whose epilogue adds them per source (tcgen05 path)
      GemmArgs a;
      a.A = sc.dP; a.a_dtype = c.dt; a.K = 2 * c.D; a.B = c.dt == F32 ? (const void*)sv.F32 : sv.Fdt; a.b_dtype = c.dt;
      a.transB = true;
      a.Y = sc.dXp; a.y_dtype = c.dt; a.N = c.Din;
      a.num_w = g->R * g->T; a.bt_scratch = sc.bt;
      a.name = "gemm_pairs_dx";
      gemm(c, seg_pair_rt(g), a);
      GemmArgs q;
      q.A = sc.dQ; q.a_dtype = c.dt; q.K = c.D; q.B = w->Wq; q.b_dtype = c.dt; q.transB = true;
      q.Y = dX; q.y_dtype = F32; q.N = c.Din;
      q.num_w = g->T; q.bt_scratch = sc.bt;
      q.name = "gemm_nodes_dx";
      gemm(c, seg_node_type(g), q);
      seg_reduce_rows(g->N, g->src_pair_ptr, g->src_pairs, sc.dXp, c.dt, c.Din, dX, true, c.s);
    }
    if (dW->dWq) do_wgrad(c, seg_node_type(g), X, c.dt, c.Din, nullptr, sc.dQ, c.dt, c.D, dW->dWq, g->T, sc.partial, "wgrad_nodes");
    if (dW->dWk || dW->dWv || dW->dWatt || dW->dWmsg) {
      do_wgrad(c, seg_pair_rt(g), X, c.dt, c.Din, g->pair_src, sc.dP, c.dt, 2 * c.D, sc.dF, g->R * g->T, sc.partial, "wgrad_pairs");
      hgt_unfold(g->R, g->T, c.Din, c.D, w->Wk, w->Wv, w->Watt, w->Wmsg, w->mu, c.dt, sc.dF, dW->dWk, dW->dWv,
                 dW->dWatt, dW->dWmsg, c.s);
    }
  }
}

Ctx make_ctx(rgnn_graph_s* g, const rgnn_layer_desc* d, void* stream) {
  check_desc(g, d);
  Ctx c{g, d, d->dtype, d->d_out, d->d_in, d->dtype == F32 ? (size_t)4 : (size_t)2,
        static_cast<cudaStream_t>(stream)};
  return c;
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
                               float* out, void* saved, void* scratch, void* stream) {
  return guarded([&] {
    Ctx c = make_ctx(g, d, stream);
    RGNN_CHECK(X && w && out && saved && scratch, RGNN_ERR_INVALID_ARG, "NULL argument");
    size_t sb = 0, xb = 0;
    RGNN_CHECK(rgnn_layer_workspace(g, d, &sb, &xb) == RGNN_OK, RGNN_ERR_INVALID_ARG, "workspace query failed");
    Arena a{static_cast<char*>(saved), sb};
    Saved sv;
    layout_saved(c, a, sv);
    Arena f{static_cast<char*>(scratch), xb};
    FwdScratch fs;
    layout_fwd_scratch(c, f, fs);
    forward(c, X, w, out, sv, fs);
  });
}

rgnn_status rgnn_layer_backward(rgnn_graph_t g, const rgnn_layer_desc* d, const void* X, const rgnn_weights* w,
                                const float* out, const void* saved, const float* dout, float* dX,
                                const rgnn_weight_grads* dW, void* scratch, void* stream) {
  return guarded([&] {
    Ctx c = make_ctx(g, d, stream);
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
    backward(c, X, w, out, sv, dout, dX, dW, bs);
  });
}

}  // extern "C"
