// Host wrappers of the traversal kernels (traverse.cu).
#pragma once
#include "graph.cuh"

namespace rgnn {
// Partial states of heavy (split) rows / pairs (graph.cuh WorkPlan):
// acc [n_slots][width] fp32, stat [n_slots] ((m, sum) for softmax rows, (sum dz, 0) for RGAT pairs).
struct Partial {
  float* acc = nullptr;
  float2* stat = nullptr;
};
void rgcn_fwd_traverse(const rgnn_graph_s* g, int dtype, int D, const float* norm, const void* P, float* out,
                       bool accumulate, const Partial& pt, cudaStream_t s);
// HGT, H heads (head h = columns h*D/H .. (h+1)*D/H - 1): stats and the node records are [N][H]
void hgt_fwd_traverse(const rgnn_graph_s* g, int dtype, int D, int H, const void* KM, const void* Q, float* out,
                      float2* stats, const Partial& pt, cudaStream_t s);
// te != NULL (reordering off): the destination logit term per CSR entry instead of X_v . y_r
void rgat_fwd_traverse(const rgnn_graph_s* g, int dtype, int D, const void* P, const float* spair, const void* X,
                       const float* y, const float* te, float slope, float* out, float2* stats, const Partial& pt,
                       cudaStream_t s);
// also writes the per-node record GQ_v = [G_v | Q_v], nst_v = (m_v, 1/sum_v, G_v . out_v, 0) (nst may be
// NULL) of every destination with in-edges, and, when wts != NULL, (alpha_e, dl_e) per CSR entry and
// head (read by hgt_bwd_pair)
// single != NULL: the dKM rows of single-edge pairs (graph csr_single) are written here, and
// hgt_bwd_pair then runs with skip_single (its pair-major pass covers pairs with >= 2 edges)
void hgt_bwd_dst(const rgnn_graph_s* g, int dtype, int D, int H, const void* KM, const void* Q, const float2* stats,
                 const float* G, const float* out, void* dQ, void* GQ, float4* nst, const uint8_t* single, void* dKM,
                 float2* wts, const Partial& pt, cudaStream_t s);
// also writes the per-node record GX_v = [G_v | X_v], nst_v = (m_v, 1/sum_v, G_v . out_v, 0); with wts
// (weighted-SpMM pair pass) instead (alpha_e, dz_e) per CSR entry and GX_v = G_v ([N][D]), no bx, no nst.
// te != NULL (reordering off): t_e read from te, dz_e written per CSR entry into dz, dX untouched.
void rgat_bwd_dst(const rgnn_graph_s* g, int dtype, int D, const void* P, const float* spair, const void* X,
                  const float* y, const float* te, float* dz, float slope, const float2* stats, const float* G,
                  const float* out, float* dX, void* GX, float4* nst, const uint8_t* single, const void* a, void* dP,
                  void* bx, float* wsum, float2* wts, const Partial& pt, cudaStream_t s);
// G: upstream gradient rows in the layer dtype (bf16 copy on the bf16 path)
void rgcn_bwd_pair(const rgnn_graph_s* g, int dtype, int D, const float* csc_norm, const void* G, void* dP,
                   const Partial& pt, cudaStream_t s);
// te != NULL (reordering off): t_e = te[csc2csr[i]], bx not computed
// wts != NULL: weighted SpMM over the per-CSR-entry (alpha_e, dz_e) that rgat_bwd_dst wrote, GX = [N][D]
// bf16/fp32 rows of G (no bx); else the recomputing pair kernels over GX = [G_v | X_v] and nst
void rgat_bwd_pair(const rgnn_graph_s* g, int dtype, int D, const void* P, const float* spair, const float* y,
                   const float* te, const void* a, float slope, const void* GX, const float4* nst, const float2* wts,
                   void* dP, float* wsum, void* bx, bool skip_single, const Partial& pt, cudaStream_t s);
// wts != NULL: the weighted SpMM k_pair_spmm over the per-CSR-entry (alpha_e, dl_e) [E][H] that
// hgt_bwd_dst wrote (nst unused); else the recomputing pair kernels (alpha, dl from K~ / M and nst)
void hgt_bwd_pair(const rgnn_graph_s* g, int dtype, int D, int H, const void* KM, const void* GQ, const float4* nst,
                  const float2* wts, void* dKM, bool skip_single, const Partial& pt, cudaStream_t s);
}  // namespace rgnn
