// Host-side entry points of the kernels (internal).
#pragma once

#include "graph.cuh"

namespace rgnn {

enum DType { F32 = 0, BF16 = 1 };

// Typed segment GEMM  Y[row] = A[gather(row)] x B_w  for every tile (row0,row1,w)
// (the GEMM template Y[S] = X[G] x W[T], §3.3.3; segment MM P:634).
struct GemmArgs {
  const Tile* tiles = nullptr;
  int ntiles = 0;
  const void* A = nullptr;
  int a_dtype = F32;
  int K = 0;                        // A width
  const int32_t* gather = nullptr;  // NULL: identity
  const void* B = nullptr;          // weights: [w][K][N] or (transB) [w][N][K]
  int b_dtype = F32;
  bool transB = false;
  void* Y = nullptr;
  int y_dtype = F32;
  int N = 0;          // Y width (ldy = N)
  const float* dotvec = nullptr;  // optional epilogue: dotout[row] = sum_n Y_fp32[row][n] * dotvec[w][n]
  float* dotout = nullptr;
  const char* name = "gemm";      // profiling label of the launch
  // optional fused row reduction (tcgen05 path only): Y[row] += sum_{i in [red_ptr[row], red_ptr[row+1])}
  // red_rows[red_list[i]][:]  (rows of width N in red_dtype; used for dX += sum of per-pair dX rows by source)
  const int32_t* red_ptr = nullptr;
  const int32_t* red_list = nullptr;
  const void* red_rows = nullptr;
  int red_dtype = F32;
  int num_w = 0;                  // number of weight matrices in B (tcgen05 path: K-major image size)
  void* bt_scratch = nullptr;     // tcgen05 path: device buffer for num_w*K*N bf16 (K-major B image)
  int64_t y_rows = 0;             // rows of Y (and of A when not gathered); 0: unknown (no TMA path)
  int64_t a_rows = 0;             // rows of the gathered A table (0: unknown; bounds the TMA map only)
};
void gemm_simt(const GemmArgs& a, cudaStream_t s);
bool gemm_tc_supported(const GemmArgs& a);
void gemm_tc(const GemmArgs& a, cudaStream_t s);
// TMA generation of the tcgen05 GEMM (gemm_tma.cu), used by gemm_tc when enabled and applicable
bool gemm_tma_enabled(const GemmArgs& a);
void gemm_tma(const GemmArgs& a, const bf16* Bt, cudaStream_t s);

// Segmented weight gradient  out[w] = sum_{rows of w} A[gather(row)]^T Bm[row]   (fp32 out)
// Deterministic two-level reduction: per-tile partials, then per-segment sums in tile order.
struct WgradArgs {
  const Plan* plan = nullptr;  // tiles with pad = segment id, w = weight index
  const void* A = nullptr;
  int a_dtype = F32;
  int K1 = 0;
  const int32_t* gather = nullptr;
  const void* Bm = nullptr;  // [rows][K2], b_dtype
  int b_dtype = F32;
  int K2 = 0;
  float* out = nullptr;  // [num_w][K1][K2]
  int num_w = 0;
  float* partial = nullptr;  // scratch [ntiles][K1][K2]
  const char* name = "wgrad";
  bool allow_tc = false;  // bf16 operands: tcgen05 kernel (MN-major) when the widths allow
};
void wgrad(const WgradArgs& a, cudaStream_t s);
bool wgrad_tc_supported(const WgradArgs& a);
void wgrad_tc(const WgradArgs& a, cudaStream_t s);

// Fused pair-side backward (tcgen05, bf16): over the tiles of one plan (per-segment weight w),
//   Y[row] = dP[row] W_w^T  (W: [num_w][K1][K2] bf16; Y: [rows][K1] bf16)
//   out[w] = sum_{rows of w} X[gather(row)]^T dP[row]  (fp32 [num_w][K1][K2], two-level, deterministic)
struct PairBwdArgs {
  const Plan* plan = nullptr;
  const void* X = nullptr;
  const int32_t* gather = nullptr;
  int K1 = 0;
  const void* dP = nullptr;
  int K2 = 0;
  const void* W = nullptr;
  void* Y = nullptr;
  float* out = nullptr;
  int num_w = 0;
  float* partial = nullptr;  // scratch [ntiles][K1][K2]
  const char* name = "pair_bwd";
  int64_t rows = 0;          // rows of dP and Y (0: unknown, no TMA kernel)
};
bool pair_bwd_tc_supported(int K1, int K2);
void pair_bwd_tc(const PairBwdArgs& a, cudaStream_t s);
// warp-specialized TMA version (gemm_tma.cu), used by pair_bwd_tc when enabled and applicable
bool pair_bwd_ws_enabled(const PairBwdArgs& a);
void pair_bwd_ws(const PairBwdArgs& a, cudaStream_t s);
// the second level of the deterministic weight-gradient reduction (dense_ops.cu)
// out[seg_w[s]] = sum over the tiles of segment s of partial[tile] (width floats each), in tile order
void seg_partial_reduce(const Plan& p, const float* partial, int64_t width, float* out, cudaStream_t s);

// out[w][k] = sum_{rows of w} wt[row] * A[gather(row)][k]  (fp32 out; same two-level scheme)
void seg_wsum(const Plan* plan, const float* wt, const void* A, int a_dtype, int K, const int32_t* gather,
              float* out, int num_w, float* partial, cudaStream_t s);

// out[u][:] (+)= sum_{i in [ptr[u], ptr[u+1])} Y[list[i]][:]   (fp32 rows of width K)
void seg_reduce_rows(int64_t n, const int32_t* ptr, const int32_t* list, const void* Y, int y_dtype, int K, float* out,
                     bool accumulate, cudaStream_t s);

// A2 (linear-operator reordering): weight-weight products.
void rgat_tpath_vectors(int R, int d_in, int d_out, const void* W, const void* b, int dtype, float* y,
                        cudaStream_t s);
// F[a] for every active (r, t) combination a of g (graph.cuh): [mu_r/sqrt(dh) Wk_t Watt_r | Wv_t Wmsg_r]
// (dh = head width d / H; the per-head logit scale)
void hgt_fold(const rgnn_graph_s* g, int d_in, int d, int dh, const void* Wk, const void* Wv, const void* Watt,
              const void* Wmsg, const float* mu, int dtype, float* F32out, void* Fdt, cudaStream_t s);
// dWk, dWv, dWatt, dWmsg from dF[a] (fully overwritten; NULL outputs are skipped); P: scratch of dF's size
void hgt_unfold(const rgnn_graph_s* g, int d_in, int d, int dh, const void* Wk, const void* Wv, const void* Watt,
                const void* Wmsg, const float* mu, int dtype, const float* dF, float* P, float* dWk, float* dWv,
                float* dWatt, float* dWmsg, cudaStream_t s);
void rgat_tpath_grads(int R, int d_in, int d_out, const void* W, const void* b, int dtype, const float* Bsum,
                      float* dW, float* db, cudaStream_t s);
// F1 ablation (HGT, reordering off): un-folded weights and the split of their gradients.
void hgt_nr_weights(int R, int T, int d_in, int d, int dh, const void* Wk, const void* Wv, const void* Watt, const void* Wmsg,
                    const float* mu, int dtype, void* Wkv, void* Bd, cudaStream_t s);
void hgt_nr_split(int R, int T, int d_in, int d, int dh, const float* dBd, const float* dWkv, const float* mu, float* dWk,
                  float* dWv, float* dWatt, float* dWmsg, cudaStream_t s);
void add_f32(int64_t n, const float* x, float* y, cudaStream_t s);
// F2 HGT tail: gh = GELU(h) (erf form) in the layer dtype; dg *= GELU'(h); y += x (x in the layer dtype)
void gelu_fwd(int64_t n, const float* h, void* gh, int dtype, cudaStream_t s);
void gelu_bwd(int64_t n, const float* h, float* dg, cudaStream_t s);
void add_dt(int64_t n, const void* x, int dtype, float* y, cudaStream_t s);
// F1 ablation (RGAT, reordering off): per (rel, dst) pair -> CSR entries, CSR entries -> per pair,
// and the rank-1 rows dPt[j] = dt[j] b_rel(j) over a dpair_rel plan.
void dpair_expand(const rgnn_graph_s* g, const float* tdp, float* te, cudaStream_t s);
void dpair_sum(const rgnn_graph_s* g, const float* dz, float* dt, cudaStream_t s);
// sums w[i].y; part: g->n_dpair_chunks floats of scratch
void dpair_sum_w(const rgnn_graph_s* g, const float2* w, float* dt, float* part, cudaStream_t s);
void dpair_outer(const Plan& p, const float* dt, const void* b, int dtype, int D, void* dPt, cudaStream_t s);
void convert_f32(int64_t n, const void* in, int dtype, float* out, cudaStream_t s);
void convert_dt(int64_t n, const float* in, void* out, int dtype, cudaStream_t s);

}  // namespace rgnn
