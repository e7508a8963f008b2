// Edge-traversal kernels.
//
// Forward, destination-major over the dst-CSR:
//   A3 edge logits (g-SDDMM; RGAT: LeakyReLU(s_p + x_v . y_r), lst:ir_example
//      P:739-745 after reordering; HGT: K~_p . q_v with K~ pre-scaled by mu_r/sqrt(d)),
//   A4 edge softmax (lst:ir_example P:730-738) as an online max/sum rescale,
//   A5 attention- or norm-weighted aggregation of the compact pair rows (g-SpMM),
// all fused: logits and attention never touch HBM, only (m_v, sum_v) are saved.
//
// Work is edge-balanced (graph.cuh WorkPlan): heavy rows are cut into 512-edge chunks
// whose partial states are merged afterwards (k_merge_*), medium rows get one warp, and
// light rows (<= 64 edges) get one group of LPR lanes.  A lane always moves one 16-byte
// vector of a gathered row; in warp mode the EG = 32 / LPR groups stride over the row's
// edges, each with its own online-softmax state, merged by shuffles at the end.  UNR
// edges per group are loaded before they are used.
//
// Backward, destination-major (A6): recompute logits/alpha from (m_v, sum_v); the softmax
// backward row term sum_e alpha_e dalpha_e = G_v . out_v; dQ_v (HGT) or the t-path dX_v and
// per-edge (alpha_e, dz_e) (RGAT).  Backward, pair-major over the src-CSC (A7): per compact
// pair p the edges are contiguous in the CSC -> dP_p / [dK~_p | dM_p].  No float atomics.
#include <math_constants.h>

#include <algorithm>
#include <cstdlib>
#include <tuple>
#include <type_traits>

#include "ops.cuh"
#include "traverse.cuh"

namespace rgnn {
namespace {

#ifndef RGNN_UNR_D
#define RGNN_UNR_D 4
#endif
constexpr int UNR = RGNN_UNR_D;  // edges per group loaded ahead (dst-major and pair kernels)
#ifndef RGNN_UNR_P
#define RGNN_UNR_P 2
#endif
// launch bounds of the HGT destination-major kernels (tuning knobs: -DRGNN_FWD_MINB=n / -DRGNN_DST_MINB=n)
#ifdef RGNN_FWD_MINB
#define RGNN_FWD_LB __launch_bounds__(256, RGNN_FWD_MINB)
#else
#define RGNN_FWD_LB __launch_bounds__(256)
#endif
#ifndef RGNN_UNR_SGL
#define RGNN_UNR_SGL 2
#endif
#ifdef RGNN_RGAT_DST_MINB
#define RGNN_RGAT_DST_LB __launch_bounds__(256, RGNN_RGAT_DST_MINB)
#else
#define RGNN_RGAT_DST_LB __launch_bounds__(256)
#endif
#ifndef RGNN_UNR_WT
#define RGNN_UNR_WT 2
#endif
#ifndef RGNN_DST_MINB
#define RGNN_DST_MINB 3
#endif
#define RGNN_DST_LB __launch_bounds__(256, RGNN_DST_MINB)
#ifndef RGNN_PAIR_MINB
#define RGNN_PAIR_MINB 4
#endif
constexpr int UNR_P = RGNN_UNR_P;  // pair kernels with node records: two 16-byte row halves + a record per edge

template <class TP, int D>
struct Geo {
  static constexpr int V = Vec<TP>::N;  // elements per lane-vector
  static constexpr int LPR = D / V;     // lanes per row
  static constexpr int EG = 32 / LPR;   // lane groups per warp
  static_assert(LPR >= 1 && LPR <= 32 && (32 % LPR) == 0, "unsupported row width");
};

template <int V>
__device__ __forceinline__ void ld_f32(const float* p, float* o) {
#pragma unroll
  for (int i = 0; i < V; i += 4) {
    float4 x = __ldg(reinterpret_cast<const float4*>(p + i));
    o[i] = x.x; o[i + 1] = x.y; o[i + 2] = x.z; o[i + 3] = x.w;
  }
}
template <int V>
__device__ __forceinline__ void st_f32(float* p, const float* v) {
#pragma unroll
  for (int i = 0; i < V; i += 4) *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
}
// Round values to the table dtype and back (identity for fp32).  The softmax backward uses the
// upstream gradient G_v in both dalpha_e = G_v . M and the row term G_v . out_v; the pair-major
// pass reads G_v from the bf16 node record, so every pass rounds it the same way and the two
// terms cancel exactly where they should (e.g. a single-edge softmax, alpha = 1: dl = 0).
template <class TP, int V>
__device__ __forceinline__ void round_tp(float* v) {
  if constexpr (sizeof(TP) == 2) {
#pragma unroll
    for (int k = 0; k < V; ++k) v[k] = __bfloat162float(__float2bfloat16_rn(v[k]));
  }
}
// 4 consecutive elements of a table row as floats (8 B for bf16, 16 B for fp32)
__device__ __forceinline__ void ld4(const float* p, float* o) {
  float4 x = __ldg(reinterpret_cast<const float4*>(p));
  o[0] = x.x; o[1] = x.y; o[2] = x.z; o[3] = x.w;
}
__device__ __forceinline__ void ld4(const bf16* p, float* o) {
  uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
  o[0] = __uint_as_float(x.x << 16); o[1] = __uint_as_float(x.x & 0xffff0000u);
  o[2] = __uint_as_float(x.y << 16); o[3] = __uint_as_float(x.y & 0xffff0000u);
}
template <int V>
__device__ __forceinline__ void st_tp(float* p, const float* v) { st_f32<V>(p, v); }
template <int V>
__device__ __forceinline__ void st_tp(bf16* p, const float* v) { store16(p, v); }
__device__ __forceinline__ void st4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void st4(bf16* p, float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  *reinterpret_cast<uint2*>(p) = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
}

// 16-byte shared-memory load the compiler may not hoist (lane-private staging slots are re-read
// per edge instead of occupying registers)
__device__ __forceinline__ uint4 lds16(const uint4* p) {
  uint4 v;
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

// sum over the LPR lanes of one group (mask = the lanes executing this call)
template <int LPR>
__device__ __forceinline__ float gsum(float x, unsigned mask) {
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) x += __shfl_xor_sync(mask, x, o);
  return x;
}
template <int LPR>
__device__ __forceinline__ unsigned group_mask(int g) {
  return LPR == 32 ? 0xffffffffu : ((1u << LPR) - 1u) << (g * LPR);
}

__device__ __forceinline__ float safe_exp_diff(float a, float b) {  // exp(a - b), 0 when a = -inf
  return a == -CUDART_INF_F ? 0.f : __expf(a - b);
}

// Merge the online-softmax states of the EG groups of a warp (lanes with equal lane % LPR).
template <int LPR, int V>
__device__ __forceinline__ void merge_groups(float& m, float& s, float* acc) {
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) {
    float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    float mn = fmaxf(m, m2);
    float a = safe_exp_diff(m, mn), b = safe_exp_diff(m2, mn);
    s = s * a + s2 * b;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      float x2 = __shfl_xor_sync(0xffffffffu, acc[k], o);
      acc[k] = acc[k] * a + x2 * b;
    }
    m = mn;
  }
}

template <int LPR, int V>
__device__ __forceinline__ void sum_groups(float* acc) {
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
}

// Work-item bookkeeping shared by every kernel: warp mode (GROUP = false) gives one item to
// the whole warp and lets its groups stride over the edges; group mode gives one item per
// lane group.  The loop trip count `span` is warp-uniform in both modes (group mode: the
// longest item of the warp; light items are sorted by length so neighbours are alike), so
// the warp never diverges and shuffles always use the full mask.  init() returns false only
// when the whole warp has no item; lanes of an idle group see an empty range (has = false).
template <bool GROUP, int LPR>
struct Work {
  static constexpr int EG = 32 / LPR;
  int lane, g, c;
  int first, step, span;
  bool has;
  int4 item;
  __device__ __forceinline__ bool init(int64_t n, const int4* __restrict__ items) {
    return init(n, items, (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  }
  // warp w of the launch (persistent kernels stride w over the grid)
  __device__ __forceinline__ bool init(int64_t n, const int4* __restrict__ items, int64_t w) {
    lane = threadIdx.x & 31;
    g = lane / LPR;
    c = lane % LPR;
    first = GROUP ? 0 : g;
    step = GROUP ? 1 : EG;
    if (GROUP) {
      if (w * EG >= n) return false;
      const int64_t wi = w * EG + g;
      has = wi < n;
      item = has ? items[wi] : make_int4(0, 0, 0, -1);
      span = __reduce_max_sync(0xffffffffu, item.z - item.y);
    } else {
      if (w >= n) return false;
      has = true;
      item = items[w];
      span = item.z - item.y;
    }
    return true;
  }
  __device__ __forceinline__ bool writer() const { return has && (GROUP || g == 0); }
  __device__ __forceinline__ bool leader() const { return has && (GROUP ? c == 0 : lane == 0); }
  static constexpr unsigned mask = 0xffffffffu;
};

// Short items (<= SHORT_MAX edges, graph.cuh): each lane group owns KI items of the sorted list
// (group g of warp w: items w*EG*KI + g + EG*k, k < KI) and gathers edge t of all of them in
// the same step, so one dependent load chain (item -> index -> row) serves KI items instead of
// one.  Trip count = the longest of the warp's items (warp-uniform; the list is sorted).
template <int LPR, int KI>
struct WorkK {
  static constexpr int EG = 32 / LPR;
  int lane, g, c, span;
  int4 it[KI];
  __device__ __forceinline__ bool init(int64_t n, const int4* __restrict__ items) {
    lane = threadIdx.x & 31;
    g = lane / LPR;
    c = lane % LPR;
    const int64_t base = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * (int64_t)(EG * KI);
    if (base >= n) return false;
    int mx = 0;
#pragma unroll
    for (int k = 0; k < KI; ++k) {
      const int64_t j = base + g + (int64_t)EG * k;
      it[k] = j < n ? items[j] : make_int4(-1, 0, 0, -1);
      mx = max(mx, it[k].z - it[k].y);
    }
    span = __reduce_max_sync(0xffffffffu, mx);
    return true;
  }
  static constexpr unsigned mask = 0xffffffffu;
  // gather index of edge t of item k: the first edge's is carried in the item (w = -2 - index)
  __device__ __forceinline__ int64_t index(int k, int t, const int32_t* __restrict__ idx) const {
    return t == 0 ? (int64_t)(-2 - it[k].w) : (int64_t)idx[it[k].y + t];
  }
};

// ------------------------------------------------------------------ RGCN forward (A5)
// out_v (+)= sum_e norm_e P[pair_e]     (Eq. 3.1; self-loop X W_0 already in out when accumulate)
template <class TP, int D, bool GROUP>
__global__ void __launch_bounds__(256) k_rgcn_fwd(int64_t n, const int4* __restrict__ items, float* __restrict__ pacc,
                                                  const int32_t* __restrict__ csr_pair,
                                                  const float* __restrict__ norm, const TP* __restrict__ P,
                                                  float* __restrict__ out, bool accumulate) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR;
  Work<GROUP, LPR> w;
  if (!w.init(n, items)) return;
  const int64_t v = w.item.x;
  const int b = w.item.y, e = w.item.z, slot = w.item.w, c = w.c;
  float acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = 0.f;
  for (int t = 0; t < w.span; t += w.step * UNR) {
    const int i0 = b + t + w.first;
    uint4 raw[UNR];
    float wt[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      int i = i0 + u * w.step;
      wt[u] = 0.f;
      raw[u] = make_uint4(0, 0, 0, 0);
      if (i < e) {
        wt[u] = norm[i];
        raw[u] = ldg16(P + (int64_t)csr_pair[i] * D + c * V);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      float x[V];
      cvt16<TP>(raw[u], x);
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = fmaf(wt[u], x[k], acc[k]);
    }
  }
  if (!GROUP) sum_groups<LPR, V>(acc);
  if (!w.writer()) return;
  if (slot >= 0) {  // chunk of a heavy row: partial sum, merged by k_merge_sum
    st_f32<V>(pacc + (int64_t)slot * D + c * V, acc);
    return;
  }
  float* o = out + v * D + c * V;
  if (accumulate) {
    float prev[V];
    ld_f32<V>(o, prev);
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] += prev[k];
  }
  st_f32<V>(o, acc);
}

// ------------------------------------------------------------------ HGT forward (A3+A4+A5)
// KM row of pair p = [K~_p | M_p] (2D wide);  l_e = K~_p . q_v;  out_v = sum softmax(l)_e M_p.
// H heads (F2): head h owns columns h*dh..(h+1)*dh-1, i.e. LH = LPR/H consecutive lanes of a group;
// its logit is reduced over those lanes only and its online-softmax state lives in them, so
// per-lane state is per-head state; stats / partial stats are [id][H].
template <class TP, int D, bool GROUP, int H>
__global__ void RGNN_FWD_LB k_hgt_fwd(int64_t n, const int4* __restrict__ items, float* __restrict__ pacc,
                                                 float2* __restrict__ pstat, const int32_t* __restrict__ csr_pair,
                                                 const TP* __restrict__ KM, const TP* __restrict__ Q,
                                                 float* __restrict__ out, float2* __restrict__ stats) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR, LH = LPR / H;
  static_assert(LPR % H == 0, "a head must own whole 16-byte lane vectors");
  Work<GROUP, LPR> w;
  if (!w.init(n, items)) return;
  const int64_t v = w.item.x;
  const int b = w.item.y, e = w.item.z, slot = w.item.w, c = w.c, hd = c / LH;
  const bool hlead = w.has && (c % LH == 0) && (GROUP || w.g == 0);
  float q[V];
  cvt16<TP>(ldg16(Q + v * D + c * V), q);
  float m = -CUDART_INF_F, s = 0.f, acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = 0.f;
  for (int t = 0; t < w.span; t += w.step * UNR) {
    const int i0 = b + t + w.first;
    uint4 rk[UNR], rm[UNR];
    bool ok[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      int i = i0 + u * w.step;
      ok[u] = i < e;
      rk[u] = rm[u] = make_uint4(0, 0, 0, 0);
      if (ok[u]) {
        int64_t p = csr_pair[i];
        rk[u] = ldg16(KM + p * 2 * D + c * V);
        rm[u] = ldg16(KM + p * 2 * D + D + c * V);
      }
    }
    float l[UNR], mx = m;
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      float kx[V];
      cvt16<TP>(rk[u], kx);
      float d = 0.f;
#pragma unroll
      for (int k = 0; k < V; ++k) d = fmaf(kx[k], q[k], d);
      d = gsum<LH>(d, w.mask);
      l[u] = ok[u] ? d : -CUDART_INF_F;
      mx = fmaxf(mx, l[u]);
    }
    float sc = safe_exp_diff(m, mx);
    s *= sc;
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] *= sc;
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      float wt = safe_exp_diff(l[u], mx);
      s += wt;
      float mv[V];
      cvt16<TP>(rm[u], mv);
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = fmaf(wt, mv[k], acc[k]);
    }
    m = mx;
  }
  if (!GROUP) merge_groups<LPR, V>(m, s, acc);
  if (slot >= 0) {  // chunk of a heavy row: unnormalised state, merged by k_merge_softmax
    if (w.writer()) st_f32<V>(pacc + (int64_t)slot * D + c * V, acc);
    if (hlead) pstat[(int64_t)slot * H + hd] = make_float2(m, s);
    return;
  }
  float inv = s > 0.f ? 1.f / s : 0.f;
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] *= inv;
  if (w.writer()) st_f32<V>(out + v * D + c * V, acc);
  if (hlead) stats[v * H + hd] = make_float2(m, s);
}

// Short rows (<= SHORT_MAX in-edges, incl. empty rows), KI per lane group.
template <class TP, int D, int H, int KI>
__global__ void __launch_bounds__(256) k_hgt_fwd_k(int64_t n, const int4* __restrict__ items,
                                                   const int32_t* __restrict__ csr_pair, const TP* __restrict__ KM,
                                                   const TP* __restrict__ Q, float* __restrict__ out,
                                                   float2* __restrict__ stats) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR, LH = LPR / H;
  WorkK<LPR, KI> w;
  if (!w.init(n, items)) return;
  const int c = w.c, hd = c / LH;
  uint4 qr[KI];
  float m[KI], sm[KI], acc[KI][V];
#pragma unroll
  for (int k = 0; k < KI; ++k) {
    qr[k] = w.it[k].z > w.it[k].y ? ldg16(Q + (int64_t)w.it[k].x * D + c * V) : make_uint4(0, 0, 0, 0);
    m[k] = -CUDART_INF_F;
    sm[k] = 0.f;
#pragma unroll
    for (int j = 0; j < V; ++j) acc[k][j] = 0.f;
  }
  for (int t = 0; t < w.span; ++t) {
    uint4 rk[KI], rm[KI];
#pragma unroll
    for (int k = 0; k < KI; ++k) {
      const int i = w.it[k].y + t;
      rk[k] = rm[k] = make_uint4(0, 0, 0, 0);
      if (i < w.it[k].z) {
        const int64_t p = w.index(k, t, csr_pair);
        rk[k] = ldg16(KM + p * 2 * D + c * V);
        rm[k] = ldg16(KM + p * 2 * D + D + c * V);
      }
    }
#pragma unroll
    for (int k = 0; k < KI; ++k) {
      float kx[V], q[V];
      cvt16<TP>(rk[k], kx);
      cvt16<TP>(qr[k], q);
      float d = 0.f;
#pragma unroll
      for (int j = 0; j < V; ++j) d = fmaf(kx[j], q[j], d);
      d = gsum<LH>(d, w.mask);
      const float l = (w.it[k].y + t < w.it[k].z) ? d : -CUDART_INF_F;
      const float mx = fmaxf(m[k], l);
      const float sc = safe_exp_diff(m[k], mx), wt = safe_exp_diff(l, mx);
      sm[k] = sm[k] * sc + wt;
      float mv[V];
      cvt16<TP>(rm[k], mv);
#pragma unroll
      for (int j = 0; j < V; ++j) acc[k][j] = fmaf(wt, mv[j], acc[k][j] * sc);
      m[k] = mx;
    }
  }
#pragma unroll
  for (int k = 0; k < KI; ++k) {
    if (w.it[k].x < 0) continue;
    const int64_t v = w.it[k].x;
    const float inv = sm[k] > 0.f ? 1.f / sm[k] : 0.f;
#pragma unroll
    for (int j = 0; j < V; ++j) acc[k][j] *= inv;
    st_f32<V>(out + v * D + c * V, acc[k]);
    if (c % LH == 0) stats[v * H + hd] = make_float2(m[k], sm[k]);
  }
}

// ------------------------------------------------------------------ staged relation vectors
// The RGAT t-path reads y_r = W_r b_r (fp32, R x D) once per edge.  SY kernels stage all of y in
// shared memory once per (persistent) block and read the row of an edge's relation when it is used,
// instead of prefetching D floats per edge into registers through L1 (north_star: "shared-memory
// staging of relation weights").  Used when R * D * 4 <= kStageYMax bytes.
constexpr int kStageYMax = 48 * 1024;
// The warp half (heavy chunks, medium rows: few items) is staged and persistent only when y is small:
// measured on mag (R = 4, 1 KB: bwd warp half 0.70 -> 0.53 ms) and AM (R = 130, 33 KB: slower, the
// staging is not amortised over the few warp items per block).
constexpr int kStageYWarpMax = 8 * 1024;
__device__ __forceinline__ const float* stage_y(const float* __restrict__ y, int ny) {
  extern __shared__ float4 y_smem[];
  for (int i = threadIdx.x; i < ny / 4; i += blockDim.x) y_smem[i] = __ldg(reinterpret_cast<const float4*>(y) + i);
  __syncthreads();
  return reinterpret_cast<const float*>(y_smem);
}
// V floats of a staged row (volatile: read where it is used, not hoisted into the prefetch registers)
template <int V>
__device__ __forceinline__ void lds_f32(const float* p, float* o) {
#pragma unroll
  for (int i = 0; i < V; i += 4) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p + i));
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(o[i]), "=f"(o[i + 1]), "=f"(o[i + 2]), "=f"(o[i + 3]) : "r"(a));
  }
}

// ------------------------------------------------------------------ RGAT forward (A3+A4+A5)
// z_e = s_p + x_v . y_r (reordered t-path), l = LeakyReLU(z), out_v = sum softmax(l)_e P_p.
// Requires d_in == d_out == D (the x_v chunk lives in the same lanes as the row chunk).
// TE (reordering off, F1 ablation): the destination term t_e = (X_v W_r) . b_r is read per CSR
// entry from te[] (computed by the dst-pair GEMM) instead of x_v . y_r.
// SY: y staged in shared memory (persistent grid, stage_y); the edge's relation id is prefetched
// instead of its y row.
template <class TP, int D, bool GROUP, bool TE, bool SY, int UF = UNR>
__device__ __forceinline__ bool rgat_fwd_item(int64_t wid, int64_t n, const int4* __restrict__ items,
                                              float* __restrict__ pacc, float2* __restrict__ pstat,
                                              const int32_t* __restrict__ csr_pair, const int32_t* __restrict__ csr_rel,
                                              const TP* __restrict__ P, const float* __restrict__ spair,
                                              const TP* __restrict__ X, const float* __restrict__ y,
                                              const float* __restrict__ te, float slope, float* __restrict__ out,
                                              float2* __restrict__ stats) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR;
  constexpr int VY = SY ? 1 : V;  // prefetched y columns per edge
  Work<GROUP, LPR> w;
  if (!w.init(n, items, wid)) return false;
  const int64_t v = w.item.x;
  const int b = w.item.y, e = w.item.z, slot = w.item.w, c = w.c;
  float x[V];
  if (!TE) cvt16<TP>(ldg16(X + v * D + c * V), x);
  float m = -CUDART_INF_F, s = 0.f, acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = 0.f;
  for (int t = 0; t < w.span; t += w.step * UF) {
    const int i0 = b + t + w.first;
    uint4 rp[UF];
    float sp[UF], yv[UF][VY];
    int rel[UF];
    bool ok[UF];
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      int i = i0 + u * w.step;
      ok[u] = i < e;
      rp[u] = make_uint4(0, 0, 0, 0);
      sp[u] = 0.f;
      rel[u] = 0;
#pragma unroll
      for (int k = 0; k < VY; ++k) yv[u][k] = 0.f;
      if (ok[u]) {
        int64_t p = csr_pair[i];
        rp[u] = ldg16(P + p * D + c * V);
        sp[u] = spair[p];
        if (TE) yv[u][0] = te[i];
        else if (SY) rel[u] = csr_rel[i];
        else ld_f32<V>(y + (int64_t)csr_rel[i] * D + c * V, yv[u]);
      }
    }
    float l[UF], mx = m;
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      float t = 0.f;
      if (TE) {
        t = yv[u][0];
      } else {
        float yr[V];
        if constexpr (SY) lds_f32<V>(y + rel[u] * D + c * V, yr);
        else {
#pragma unroll
          for (int k = 0; k < V; ++k) yr[k] = yv[u][k % VY];
        }
#pragma unroll
        for (int k = 0; k < V; ++k) t = fmaf(x[k], yr[k], t);
        t = gsum<LPR>(t, w.mask);
      }
      float z = sp[u] + t;
      float lz = z > 0.f ? z : slope * z;
      l[u] = ok[u] ? lz : -CUDART_INF_F;
      mx = fmaxf(mx, l[u]);
    }
    float sc = safe_exp_diff(m, mx);
    s *= sc;
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] *= sc;
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      float wt = safe_exp_diff(l[u], mx);
      s += wt;
      float pv[V];
      cvt16<TP>(rp[u], pv);
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = fmaf(wt, pv[k], acc[k]);
    }
    m = mx;
  }
  if (!GROUP) merge_groups<LPR, V>(m, s, acc);
  if (slot >= 0) {
    if (w.writer()) st_f32<V>(pacc + (int64_t)slot * D + c * V, acc);
    if (w.leader()) pstat[slot] = make_float2(m, s);
    return true;
  }
  float inv = s > 0.f ? 1.f / s : 0.f;
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] *= inv;
  if (w.writer()) st_f32<V>(out + v * D + c * V, acc);
  if (w.leader()) stats[v] = make_float2(m, s);
  return true;
}

#ifndef RGNN_SY_MINB
#define RGNN_SY_MINB 4
#endif
#ifndef RGNN_SY_MINB_FWD
#define RGNN_SY_MINB_FWD RGNN_SY_MINB
#endif
#ifndef RGNN_SY_UNR
#define RGNN_SY_UNR 4  // edges per lane group in flight in the staged forward kernel
#endif
#ifndef RGNN_SY_MINB_SGL
#define RGNN_SY_MINB_SGL 3  // the single-edge-pair stores need more registers (64 spill)
#endif
template <class TP, int D, bool GROUP, bool TE>
__global__ void __launch_bounds__(256) k_rgat_fwd(int64_t n, const int4* __restrict__ items, float* __restrict__ pacc,
                                                  float2* __restrict__ pstat, const int32_t* __restrict__ csr_pair,
                                                  const int32_t* __restrict__ csr_rel, const TP* __restrict__ P,
                                                  const float* __restrict__ spair, const TP* __restrict__ X,
                                                  const float* __restrict__ y, const float* __restrict__ te,
                                                  float slope, float* __restrict__ out, float2* __restrict__ stats,
                                                  int ny) {
  rgat_fwd_item<TP, D, GROUP, TE, false>((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, n, items, pacc, pstat,
                                         csr_pair, csr_rel, P, spair, X, y, te, slope, out, stats);
}
// persistent, y staged in shared memory
template <class TP, int D, bool GROUP>
__global__ void __launch_bounds__(256, RGNN_SY_MINB_FWD) k_rgat_fwd_sy(
    int64_t n, const int4* __restrict__ items, float* __restrict__ pacc, float2* __restrict__ pstat,
    const int32_t* __restrict__ csr_pair, const int32_t* __restrict__ csr_rel, const TP* __restrict__ P,
    const float* __restrict__ spair, const TP* __restrict__ X, const float* __restrict__ y,
    const float* __restrict__ te, float slope, float* __restrict__ out, float2* __restrict__ stats, int ny) {
  const float* ys = stage_y(y, ny);
  const int64_t stride = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
       rgat_fwd_item<TP, D, GROUP, false, true, RGNN_SY_UNR>(wid, n, items, pacc, pstat, csr_pair, csr_rel, P, spair, X, ys, te, slope,
                                               out, stats);
       wid += stride) {
  }
}

// ------------------------------------------------------------------ HGT backward, dst-major (A6)
// alpha_e = exp(l_e - m_v)/sum_v ; dalpha_e = G_v . M_p ; dl_e = alpha_e (dalpha_e - G_v . out_v)
// dQ_v = sum_e dl_e K~_p   (layer dtype; heavy rows: fp32 partials merged by k_merge_sum)
template <class TP, int D, bool GROUP, int H, bool SGL, bool WT>
__global__ void RGNN_DST_LB k_hgt_bwd_dst(int64_t n, const int4* __restrict__ items,
                                                     float* __restrict__ pacc, const int32_t* __restrict__ csr_pair,
                                                     const TP* __restrict__ KM, const TP* __restrict__ Q,
                                                     const float2* __restrict__ stats, const float* __restrict__ Gr,
                                                     const float* __restrict__ out, TP* __restrict__ dQ,
                                                     TP* __restrict__ GQ, float4* __restrict__ nst,
                                                     const uint8_t* __restrict__ single, TP* __restrict__ dKM,
                                                     float2* __restrict__ wts) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR, LH = LPR / H;
  Work<GROUP, LPR> w;
  if (!w.init(n, items)) return;
  const int64_t v = w.item.x;
  const int b = w.item.y, e = w.item.z, slot = w.item.w, c = w.c, hd = c / LH;
  float dq[V];
#pragma unroll
  for (int k = 0; k < V; ++k) dq[k] = 0.f;
  if (w.span > 0) {
    float q[V], gv[V], ov[V];
    cvt16<TP>(ldg16(Q + v * D + c * V), q);
    ld_f32<V>(Gr + v * D + c * V, gv);
    round_tp<TP, V>(gv);  // G_v in the table precision everywhere (dalpha and the row term G_v . out_v)
    ld_f32<V>(out + v * D + c * V, ov);
    float go = 0.f;
#pragma unroll
    for (int k = 0; k < V; ++k) go = fmaf(gv[k], ov[k], go);
    go = gsum<LH>(go, w.mask);
    const float2 st = stats[v * H + hd];
    const float inv = 1.f / st.y;
    if (slot < 0 && e > b && w.writer()) {  // node record for the pair-major pass (heavy rows: k_hgt_node_prep)
      st_tp<V>(GQ + v * 2 * D + c * V, gv);
      st_tp<V>(GQ + v * 2 * D + D + c * V, q);
      if (nst && c % LH == 0) nst[v * H + hd] = make_float4(st.x + logf(st.y), go, 0.f, 0.f);
    }
    for (int t = 0; t < w.span; t += w.step * UNR) {
      const int i0 = b + t + w.first;
      uint4 rk[UNR], rm[UNR];
      int pid[UNR];  // SGL: the pair id when it has a single edge (its dKM row is written here), else -1
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        int i = i0 + u * w.step;
        rk[u] = rm[u] = make_uint4(0, 0, 0, 0);
        pid[u] = -1;
        if (i < e) {
          int64_t p = csr_pair[i];
          rk[u] = ldg16(KM + p * 2 * D + c * V);
          rm[u] = ldg16(KM + p * 2 * D + D + c * V);
          if (SGL && single[i]) pid[u] = (int)p;
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        int i = i0 + u * w.step;
        float kx[V], mv[V];
        cvt16<TP>(rk[u], kx);
        cvt16<TP>(rm[u], mv);
        float l = 0.f, da = 0.f;
#pragma unroll
        for (int k = 0; k < V; ++k) {
          l = fmaf(kx[k], q[k], l);
          da = fmaf(gv[k], mv[k], da);
        }
        l = gsum<LH>(l, w.mask);
        da = gsum<LH>(da, w.mask);
        float dl = (i < e) ? __expf(l - st.x) * inv * (da - go) : 0.f;
        if (WT && i < e && c % LH == 0)  // for k_pair_spmm
          wts[(int64_t)i * H + hd] = make_float2(__expf(l - st.x) * inv, dl);
#pragma unroll
        for (int k = 0; k < V; ++k) dq[k] = fmaf(dl, kx[k], dq[k]);
        if (SGL && pid[u] >= 0) {  // single-edge pair: dKM_p = [dl q_v | alpha G_v]
          const float alpha = __expf(l - st.x) * inv;
          float o[V];
#pragma unroll
          for (int k = 0; k < V; ++k) o[k] = dl * q[k];
          st_tp<V>(dKM + (int64_t)pid[u] * 2 * D + c * V, o);
#pragma unroll
          for (int k = 0; k < V; ++k) o[k] = alpha * gv[k];
          st_tp<V>(dKM + (int64_t)pid[u] * 2 * D + D + c * V, o);
        }
      }
    }
  }
  if (!GROUP) sum_groups<LPR, V>(dq);
  if (!w.writer()) return;
  if (slot >= 0) st_f32<V>(pacc + (int64_t)slot * D + c * V, dq);
  else st_tp<V>(dQ + v * D + c * V, dq);
}

// Short rows (<= SHORT_MAX in-edges, incl. empty rows), KI per lane group; also the node records.
template <class TP, int D, int H, int KI, bool SGL, bool WT>
__global__ void __launch_bounds__(256) k_hgt_bwd_dst_k(int64_t n, const int4* __restrict__ items,
                                                       const int32_t* __restrict__ csr_pair,
                                                       const TP* __restrict__ KM, const TP* __restrict__ Q,
                                                       const float2* __restrict__ stats, const float* __restrict__ Gr,
                                                       const float* __restrict__ out, TP* __restrict__ dQ,
                                                       TP* __restrict__ GQ, float4* __restrict__ nst,
                                                       const uint8_t* __restrict__ single, TP* __restrict__ dKM,
                                                       float2* __restrict__ wts) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR, LH = LPR / H;
  __shared__ uint4 sg[KI][256];  // G_v chunk (table dtype) of each item, lane-private
  WorkK<LPR, KI> w;
  if (!w.init(n, items)) return;
  const int c = w.c, hd = c / LH;
  uint4 qr[KI];
  float go[KI], lse[KI], dq[KI][V];
#pragma unroll
  for (int k = 0; k < KI; ++k) {
    const bool has = w.it[k].z > w.it[k].y;
    const int64_t v = has ? w.it[k].x : 0;
    qr[k] = make_uint4(0, 0, 0, 0);
    go[k] = 0.f;
    lse[k] = CUDART_INF_F;
#pragma unroll
    for (int j = 0; j < V; ++j) dq[k][j] = 0.f;
    if (has) {
      float gv[V], ov[V], q[V];
      qr[k] = ldg16(Q + v * D + c * V);
      ld_f32<V>(Gr + v * D + c * V, gv);
      round_tp<TP, V>(gv);  // G_v in the table precision everywhere (dalpha and the row term G_v . out_v)
      ld_f32<V>(out + v * D + c * V, ov);
      float x = 0.f;
#pragma unroll
      for (int j = 0; j < V; ++j) x = fmaf(gv[j], ov[j], x);
      go[k] = x;
      const float2 st = stats[v * H + hd];
      lse[k] = st.x + logf(st.y);
      cvt16<TP>(qr[k], q);
      st_tp<V>(GQ + v * 2 * D + c * V, gv);
      st_tp<V>(GQ + v * 2 * D + D + c * V, q);
      uint4 gpk;
      if constexpr (sizeof(TP) == 2) {
        store16(reinterpret_cast<bf16*>(&gpk), gv);
        sg[k][threadIdx.x] = gpk;
      } else {
        sg[k][threadIdx.x] = *reinterpret_cast<uint4*>(gv);
      }
    }
    go[k] = gsum<LH>(go[k], w.mask);
    if (nst && has && c % LH == 0) nst[v * H + hd] = make_float4(lse[k], go[k], 0.f, 0.f);
  }
  for (int t = 0; t < w.span; ++t) {
    uint4 rk[KI], rm[KI];
    int pid[KI];
#pragma unroll
    for (int k = 0; k < KI; ++k) {
      const int i = w.it[k].y + t;
      rk[k] = rm[k] = make_uint4(0, 0, 0, 0);
      pid[k] = -1;
      if (i < w.it[k].z) {
        const int64_t p = w.index(k, t, csr_pair);
        rk[k] = ldg16(KM + p * 2 * D + c * V);
        rm[k] = ldg16(KM + p * 2 * D + D + c * V);
        if (SGL && single[i]) pid[k] = (int)p;
      }
    }
#pragma unroll
    for (int k = 0; k < KI; ++k) {
      float kx[V], x[V];
      cvt16<TP>(rk[k], kx);
      cvt16<TP>(qr[k], x);
      float l = 0.f, da = 0.f;
#pragma unroll
      for (int j = 0; j < V; ++j) l = fmaf(kx[j], x[j], l);
      cvt16<TP>(rm[k], x);
      float gv[V];
      cvt16<TP>(lds16(&sg[k][threadIdx.x]), gv);
#pragma unroll
      for (int j = 0; j < V; ++j) da = fmaf(gv[j], x[j], da);
      l = gsum<LH>(l, w.mask);
      da = gsum<LH>(da, w.mask);
      const float dl = (w.it[k].y + t < w.it[k].z) ? __expf(l - lse[k]) * (da - go[k]) : 0.f;
      if (WT && w.it[k].y + t < w.it[k].z && c % LH == 0)
        wts[(int64_t)(w.it[k].y + t) * H + hd] = make_float2(__expf(l - lse[k]), dl);
#pragma unroll
      for (int j = 0; j < V; ++j) dq[k][j] = fmaf(dl, kx[j], dq[k][j]);
      if (SGL && pid[k] >= 0) {  // single-edge pair: dKM_p = [dl q_v | alpha G_v]
        const float alpha = __expf(l - lse[k]);
        float o[V], q[V];
        cvt16<TP>(qr[k], q);
#pragma unroll
        for (int j = 0; j < V; ++j) o[j] = dl * q[j];
        st_tp<V>(dKM + (int64_t)pid[k] * 2 * D + c * V, o);
#pragma unroll
        for (int j = 0; j < V; ++j) o[j] = alpha * gv[j];
        st_tp<V>(dKM + (int64_t)pid[k] * 2 * D + D + c * V, o);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < KI; ++k)
    if (w.it[k].x >= 0) st_tp<V>(dQ + (int64_t)w.it[k].x * D + c * V, dq[k]);
}

// ------------------------------------------------------------------ RGAT backward, dst-major (A6)
// dalpha_e = G_v . P_p ; dl_e = alpha_e (dalpha_e - G_v . out_v) ; dz_e = dl_e (z_e > 0 ? 1 : slope)
// dX_v = sum_e dz_e y_{r_e}  (destination side of the reordered t-path).  Also writes the node record
// GX_v = [G_v | X_v] (table dtype) and nst_v = (lse_v = m_v + log sum_v, G_v . out_v, 0, 0) read by the
// pair pass (alpha_e = exp(l_e - lse_v); 8 bytes per edge gathered instead of 16).
// TE (reordering off): t_e from te[], no dX t-path here; dz_e is written per CSR entry (dz_out)
// for the explicit destination-side GEMMs.
// WT: (alpha_e, dz_e) written per CSR entry into wts for the weighted-SpMM pair pass, the node record is
// the G row alone (GX [N][D]), no bx rows and no nst.
template <class TP, int D, bool GROUP, bool TE, bool SGL, bool WT, bool SY>
__device__ __forceinline__ bool rgat_bwd_dst_item(int64_t wid, int64_t n, const int4* __restrict__ items,
                                                      float* __restrict__ pacc, const int32_t* __restrict__ csr_pair,
                                                      const int32_t* __restrict__ csr_rel, const TP* __restrict__ P,
                                                      const float* __restrict__ spair, const TP* __restrict__ X,
                                                      const float* __restrict__ y, const float* __restrict__ te,
                                                      float* __restrict__ dz_out, float slope,
                                                      const float2* __restrict__ stats,
                                                      const float* __restrict__ Gr, const float* __restrict__ out,
                                                      float* __restrict__ dX, TP* __restrict__ GX,
                                                      float4* __restrict__ nst, const uint8_t* __restrict__ single,
                                                      const TP* __restrict__ avec, TP* __restrict__ dP,
                                                      TP* __restrict__ bx, float* __restrict__ wsum,
                                                      float2* __restrict__ wts) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR;
  // the single-edge stores and the weight writes need registers: fewer edges per step
  constexpr int UN = SGL ? RGNN_UNR_SGL : WT ? RGNN_UNR_WT : UNR;
  constexpr int VY = SY ? 1 : V;  // prefetched y columns per edge (SY: y staged, read when used)
  Work<GROUP, LPR> w;
  if (!w.init(n, items, wid)) return false;
  const int64_t v = w.item.x;
  const int b = w.item.y, e = w.item.z, slot = w.item.w, c = w.c;
  float dx[V];
#pragma unroll
  for (int k = 0; k < V; ++k) dx[k] = 0.f;
  if (w.span > 0) {
    float x[V], gv[V], ov[V];
    cvt16<TP>(ldg16(X + v * D + c * V), x);
    ld_f32<V>(Gr + v * D + c * V, gv);
    round_tp<TP, V>(gv);  // G_v in the table precision everywhere (dalpha and the row term G_v . out_v)
    ld_f32<V>(out + v * D + c * V, ov);
    float go = 0.f;
#pragma unroll
    for (int k = 0; k < V; ++k) go = fmaf(gv[k], ov[k], go);
    go = gsum<LPR>(go, w.mask);
    const float2 st = stats[v];
    const float inv = 1.f / st.y;
    if (slot < 0 && e > b && w.writer()) {  // node record (heavy rows: k_rgat_node_prep)
      if (WT) {
        st_tp<V>(GX + v * D + c * V, gv);
      } else {
        st_tp<V>(GX + v * 2 * D + c * V, gv);
        st_tp<V>(GX + v * 2 * D + D + c * V, x);
        if (w.leader()) nst[v] = make_float4(st.x + logf(st.y), go, 0.f, 0.f);
      }
    }
    for (int t = 0; t < w.span; t += w.step * UN) {
      const int i0 = b + t + w.first;
      uint4 rp[UN];
      float sp[UN], yv[UN][VY];
      int pid[UN], rel[UN], ry[UN];  // SGL: single-edge pair id (else -1) and its relation; SY: relation
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        int i = i0 + u * w.step;
        rp[u] = make_uint4(0, 0, 0, 0);
        sp[u] = 0.f;
        pid[u] = -1;
        rel[u] = 0;
        ry[u] = 0;
#pragma unroll
        for (int k = 0; k < VY; ++k) yv[u][k] = 0.f;
        if (i < e) {
          int64_t p = csr_pair[i];
          rp[u] = ldg16(P + p * D + c * V);
          sp[u] = spair[p];
          if (TE) {
            yv[u][0] = te[i];
          } else {
            const int r = csr_rel[i];
            if (SY) ry[u] = r;
            else ld_f32<V>(y + (int64_t)r * D + c * V, yv[u]);
            if (SGL && single[i]) {
              pid[u] = (int)p;
              rel[u] = r;
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        int i = i0 + u * w.step;
        float pv[V], yr[V];
        cvt16<TP>(rp[u], pv);
        if constexpr (SY) lds_f32<V>(y + ry[u] * D + c * V, yr);
        else {
#pragma unroll
          for (int k = 0; k < V; ++k) yr[k] = yv[u][k % VY];
        }
        float t = 0.f, da = 0.f;
#pragma unroll
        for (int k = 0; k < V; ++k) {
          if (!TE) t = fmaf(x[k], yr[k], t);
          da = fmaf(gv[k], pv[k], da);
        }
        t = TE ? yv[u][0] : gsum<LPR>(t, w.mask);
        da = gsum<LPR>(da, w.mask);
        float z = sp[u] + t;
        float l = z > 0.f ? z : slope * z;
        float alpha = __expf(l - st.x) * inv;
        float dz = alpha * (da - go) * (z > 0.f ? 1.f : slope);
        if (i < e) {
          if (WT && c == 0) wts[i] = make_float2(alpha, dz);
          if (TE) {
            if (c == 0) dz_out[i] = dz;
          } else {
#pragma unroll
            for (int k = 0; k < V; ++k) dx[k] = fmaf(dz, yr[k], dx[k]);
            if (SGL && pid[u] >= 0) {  // single-edge pair: dP_p = alpha G_v + dz a_r, bx_p = dz X_v, wsum_p = dz
              float av[V], o[V];
              cvt16<TP>(ldg16(avec + (int64_t)rel[u] * D + c * V), av);
#pragma unroll
              for (int k = 0; k < V; ++k) o[k] = fmaf(dz, av[k], alpha * gv[k]);
              st_tp<V>(dP + (int64_t)pid[u] * D + c * V, o);
              if (!WT) {
#pragma unroll
                for (int k = 0; k < V; ++k) o[k] = dz * x[k];
                st_tp<V>(bx + (int64_t)pid[u] * D + c * V, o);
              }
              if (c == 0) wsum[pid[u]] = dz;
            }
          }
        }
      }
    }
  }
  if (TE) return true;
  if (!GROUP) sum_groups<LPR, V>(dx);
  if (!w.writer()) return true;
  st_f32<V>((slot >= 0 ? pacc + (int64_t)slot * D : dX + v * D) + c * V, dx);
  return true;
}


template <class TP, int D, bool GROUP, bool TE, bool SGL, bool WT>
__global__ void RGNN_RGAT_DST_LB k_rgat_bwd_dst(int64_t n, const int4* __restrict__ items,
                                                      float* __restrict__ pacc, const int32_t* __restrict__ csr_pair,
                                                      const int32_t* __restrict__ csr_rel, const TP* __restrict__ P,
                                                      const float* __restrict__ spair, const TP* __restrict__ X,
                                                      const float* __restrict__ y, const float* __restrict__ te,
                                                      float* __restrict__ dz_out, float slope,
                                                      const float2* __restrict__ stats,
                                                      const float* __restrict__ Gr, const float* __restrict__ out,
                                                      float* __restrict__ dX, TP* __restrict__ GX,
                                                      float4* __restrict__ nst, const uint8_t* __restrict__ single,
                                                      const TP* __restrict__ avec, TP* __restrict__ dP,
                                                      TP* __restrict__ bx, float* __restrict__ wsum,
                                                      float2* __restrict__ wts, int ny) {
  rgat_bwd_dst_item<TP, D, GROUP, TE, SGL, WT, false>((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, n, items,
                                                      pacc, csr_pair, csr_rel, P, spair, X, y, te, dz_out, slope,
                                                      stats, Gr, out, dX, GX, nst, single, avec, dP, bx, wsum, wts);
}
// persistent, y staged in shared memory
template <class TP, int D, bool GROUP, bool SGL, bool WT>
__global__ void __launch_bounds__(256, SGL ? RGNN_SY_MINB_SGL : RGNN_SY_MINB) k_rgat_bwd_dst_sy(int64_t n, const int4* __restrict__ items,
                                                      float* __restrict__ pacc, const int32_t* __restrict__ csr_pair,
                                                      const int32_t* __restrict__ csr_rel, const TP* __restrict__ P,
                                                      const float* __restrict__ spair, const TP* __restrict__ X,
                                                      const float* __restrict__ y, const float* __restrict__ te,
                                                      float* __restrict__ dz_out, float slope,
                                                      const float2* __restrict__ stats,
                                                      const float* __restrict__ Gr, const float* __restrict__ out,
                                                      float* __restrict__ dX, TP* __restrict__ GX,
                                                      float4* __restrict__ nst, const uint8_t* __restrict__ single,
                                                      const TP* __restrict__ avec, TP* __restrict__ dP,
                                                      TP* __restrict__ bx, float* __restrict__ wsum,
                                                      float2* __restrict__ wts, int ny) {
  const float* ys = stage_y(y, ny);
  const int64_t stride = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
       rgat_bwd_dst_item<TP, D, GROUP, false, SGL, WT, true>(wid, n, items, pacc, csr_pair, csr_rel, P, spair, X, ys, te,
                                                           dz_out, slope, stats, Gr, out, dX, GX, nst, single, avec,
                                                           dP, bx, wsum, wts);
       wid += stride) {
  }
}

// ------------------------------------------------------------------ pair-major backward (A7)
// One group of LPR = D/4 lanes per light pair, one warp per medium pair or heavy chunk;
// each lane owns 4 fp32 columns.  The edges of pair p are csc[item.y, item.z).

// RGCN: dP_p = sum_{e in p} norm_e G[d_e]; G rows in the table dtype (bf16 copy on the bf16 path),
// one 16-byte vector per lane.
template <class TP, int D, bool GROUP>
__global__ void __launch_bounds__(256) k_rgcn_bwd_pair(int64_t n, const int4* __restrict__ items,
                                                       float* __restrict__ pacc, const int32_t* __restrict__ csc_dst,
                                                       const float* __restrict__ csc_norm,
                                                       const TP* __restrict__ Gr, TP* __restrict__ dP) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR;
  Work<GROUP, LPR> w;
  if (!w.init(n, items)) return;
  const int64_t p = w.item.x;
  const int b = w.item.y, e = w.item.z, slot = w.item.w, c = w.c;
  float acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = 0.f;
  for (int t = 0; t < w.span; t += w.step * UNR) {
    const int i0 = b + t + w.first;
    uint4 gr[UNR];
    float wt[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      int i = i0 + u * w.step;
      gr[u] = make_uint4(0, 0, 0, 0);
      wt[u] = 0.f;
      if (i < e) {
        wt[u] = csc_norm[i];
        gr[u] = ldg16(Gr + (int64_t)csc_dst[i] * D + c * V);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      float x[V];
      cvt16<TP>(gr[u], x);
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = fmaf(wt[u], x[k], acc[k]);
    }
  }
  if (!GROUP) sum_groups<LPR, V>(acc);
  if (!w.writer()) return;
  if (slot >= 0) st_f32<V>(pacc + (int64_t)slot * D + c * V, acc);
  else st_tp<V>(dP + p * D + c * V, acc);
}

template <class TP, int D, int KI>
__global__ void __launch_bounds__(256) k_rgcn_bwd_pair_k(int64_t n, const int4* __restrict__ items,
                                                         const int32_t* __restrict__ csc_dst,
                                                         const float* __restrict__ csc_norm,
                                                         const TP* __restrict__ Gr, TP* __restrict__ dP) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR;
  WorkK<LPR, KI> w;
  if (!w.init(n, items)) return;
  const int c = w.c;
  float acc[KI][V];
#pragma unroll
  for (int k = 0; k < KI; ++k)
#pragma unroll
    for (int j = 0; j < V; ++j) acc[k][j] = 0.f;
  for (int t = 0; t < w.span; ++t) {
    uint4 gr[KI];
    float wt[KI];
#pragma unroll
    for (int k = 0; k < KI; ++k) {
      const int i = w.it[k].y + t;
      gr[k] = make_uint4(0, 0, 0, 0);
      wt[k] = 0.f;
      if (i < w.it[k].z) {
        wt[k] = csc_norm[i];
        gr[k] = ldg16(Gr + w.index(k, t, csc_dst) * D + c * V);
      }
    }
#pragma unroll
    for (int k = 0; k < KI; ++k) {
      float x[V];
      cvt16<TP>(gr[k], x);
#pragma unroll
      for (int j = 0; j < V; ++j) acc[k][j] = fmaf(wt[k], x[j], acc[k][j]);
    }
  }
#pragma unroll
  for (int k = 0; k < KI; ++k)
    if (w.it[k].x >= 0) st_tp<V>(dP + (int64_t)w.it[k].x * D + c * V, acc[k]);
}

// RGAT, recomputing the edge terms from the destination's node record (no per-edge buffer):
// per pair p (relation r): P_p, y_r, s_p in registers; per edge e of p:
//   z_e = s_p + X_d . y_r, alpha_e = exp(LeakyReLU(z_e) - lse_d), dalpha_e = G_d . P_p,
//   dz_e = alpha_e (dalpha_e - G_d . out_d) (z_e > 0 ? 1 : slope);
// dP_p = sum alpha_e G_d + (sum dz_e) a_r, wsum_p = sum dz_e (-> da_r), bx_p = sum dz_e X_d (-> B_r).
template <class TP, int D>
__global__ void __launch_bounds__(256) k_rgat_node_prep(int64_t n, const int4* __restrict__ rows,
                                                        const float* __restrict__ Gr, const TP* __restrict__ X,
                                                        const float* __restrict__ out,
                                                        const float2* __restrict__ stats, TP* __restrict__ GX,
                                                        float4* __restrict__ nst) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR, EG = G::EG;
  const int lane = threadIdx.x & 31, g = lane / LPR, c = lane % LPR;
  const int64_t j = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * EG + g;
  if (j >= n) return;
  const int64_t v = rows[j].x;
  float gv[V], ov[V], xv[V];
  ld_f32<V>(Gr + v * D + c * V, gv);
  round_tp<TP, V>(gv);
  ld_f32<V>(out + v * D + c * V, ov);
  cvt16<TP>(ldg16(X + v * D + c * V), xv);
  float go = 0.f;
#pragma unroll
  for (int k = 0; k < V; ++k) go = fmaf(gv[k], ov[k], go);
  go = gsum<LPR>(go, group_mask<LPR>(g));
  if (!nst) {  // weighted-SpMM pair pass: the record is the G row alone ([N][D])
    st_tp<V>(GX + v * D + c * V, gv);
    return;
  }
  st_tp<V>(GX + v * 2 * D + c * V, gv);
  st_tp<V>(GX + v * 2 * D + D + c * V, xv);
  if (c == 0) {
    float2 st = stats[v];
    nst[v] = make_float4(st.y > 0.f ? st.x + logf(st.y) : CUDART_INF_F, go, 0.f, 0.f);
  }
}

// TE (reordering off): t_e = te[csc2csr[i]]; no bx (the destination side is done by GEMMs).
template <class TP, int D, bool GROUP, bool TE>
__global__ void __launch_bounds__(256, RGNN_PAIR_MINB) k_rgat_bwd_pair(int64_t n, const int4* __restrict__ items,
                                                          float* __restrict__ pacc, float2* __restrict__ pstat,
                                                          const int32_t* __restrict__ csc_dst,
                                                          const int32_t* __restrict__ csc_rel,
                                                          const int32_t* __restrict__ csc2csr,
                                                          const float* __restrict__ te,
                                                          const TP* __restrict__ P, const float* __restrict__ spair,
                                                          const float* __restrict__ y, const TP* __restrict__ avec,
                                                          float slope, const TP* __restrict__ GX,
                                                          const float4* __restrict__ nst, TP* __restrict__ dP,
                                                          float* __restrict__ wsum, TP* __restrict__ bx) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR;
  Work<GROUP, LPR> w;
  if (!w.init(n, items)) return;
  const int64_t p = w.item.x;
  const int b = w.item.y, e = w.item.z, slot = w.item.w, c = w.c;
  const int r = e > b ? csc_rel[b] : 0;
  float pv[V], yv[V];
  cvt16<TP>(ldg16(P + p * D + c * V), pv);
  if (!TE) ld_f32<V>(y + (int64_t)r * D + c * V, yv);
  const float sp = spair[p];
  float acc[V], ax[V], zs = 0.f;
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = ax[k] = 0.f;
  for (int t = 0; t < w.span; t += w.step * UNR_P) {
    const int i0 = b + t + w.first;
    uint4 rg[UNR_P], rx[UNR_P];
    float2 ns[UNR_P];
    float tv[UNR_P];
#pragma unroll
    for (int u = 0; u < UNR_P; ++u) {
      int i = i0 + u * w.step;
      ns[u] = make_float2(0.f, 0.f);
      rg[u] = rx[u] = make_uint4(0, 0, 0, 0);
      tv[u] = 0.f;
      if (i < e) {
        const int64_t d = csc_dst[i];
        rg[u] = ldg16(GX + d * 2 * D + c * V);
        if (TE) tv[u] = te[csc2csr[i]];
        else rx[u] = ldg16(GX + d * 2 * D + D + c * V);
        ns[u] = __ldg(reinterpret_cast<const float2*>(nst + d));
      }
    }
#pragma unroll
    for (int u = 0; u < UNR_P; ++u) {
      float gr[V], xd[V];
      cvt16<TP>(rg[u], gr);
      if (!TE) cvt16<TP>(rx[u], xd);
      float tt = 0.f, da = 0.f;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        if (!TE) tt = fmaf(xd[k], yv[k], tt);
        da = fmaf(gr[k], pv[k], da);
      }
      tt = TE ? tv[u] : gsum<LPR>(tt, w.mask);
      da = gsum<LPR>(da, w.mask);
      const bool ok = i0 + u * w.step < e;
      float z = sp + tt;
      float l = z > 0.f ? z : slope * z;
      float alpha = ok ? __expf(l - ns[u].x) : 0.f;
      float dz = alpha * (da - ns[u].y) * (z > 0.f ? 1.f : slope);
      zs += dz;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        acc[k] = fmaf(alpha, gr[k], acc[k]);
        if (!TE) ax[k] = fmaf(dz, xd[k], ax[k]);
      }
    }
  }
  if (!GROUP) {
    sum_groups<LPR, V>(acc);
    sum_groups<LPR, V>(ax);
    float z1[1] = {zs};
    sum_groups<LPR, 1>(z1);
    zs = z1[0];
  }
  if (!w.writer()) return;
  if (slot >= 0) {  // heavy pair chunk: [acc | ax] partial + sum dz
    st_f32<V>(pacc + (int64_t)slot * 2 * D + c * V, acc);
    st_f32<V>(pacc + (int64_t)slot * 2 * D + D + c * V, ax);
    if (c == 0) pstat[slot] = make_float2(zs, 0.f);
    return;
  }
  float av[V];
  cvt16<TP>(ldg16(avec + (int64_t)r * D + c * V), av);
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = fmaf(zs, av[k], acc[k]);
  st_tp<V>(dP + p * D + c * V, acc);
  if (!TE) st_tp<V>(bx + p * D + c * V, ax);
  if (c == 0) wsum[p] = zs;
}

// Group mode of the RGAT pair pass (reordered path): P_p and y_r chunks staged in shared memory
// (lane-private), one edge per step with the next destination id prefetched (as k_hgt_bwd_pair_s).
template <class TP, int D>
__global__ void __launch_bounds__(256, RGNN_PAIR_MINB) k_rgat_bwd_pair_s(
    int64_t n, const int4* __restrict__ items, float* __restrict__ pacc, float2* __restrict__ pstat,
    const int32_t* __restrict__ csc_dst, const int32_t* __restrict__ csc_rel, const int32_t* __restrict__ csc2csr,
    const float* __restrict__ te, const TP* __restrict__ P, const float* __restrict__ spair,
    const float* __restrict__ y, const TP* __restrict__ avec, float slope, const TP* __restrict__ GX,
    const float4* __restrict__ nst, TP* __restrict__ dP, float* __restrict__ wsum, TP* __restrict__ bx) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR;
  static_assert(V % 4 == 0, "y chunk as 16-byte fp32 vectors");
  __shared__ uint4 sst[1 + V / 4][256];  // [P chunk (table dtype) | y_r chunk (fp32, V/4 vectors)]
  Work<true, LPR> w;
  if (!w.init(n, items)) return;
  const int64_t p = w.item.x;
  const int b = w.item.y, e = w.item.z, slot = w.item.w, c = w.c;
  const int r = e > b ? csc_rel[b] : 0;
  sst[0][threadIdx.x] = w.has ? ldg16(P + p * D + c * V) : make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int j = 0; j < V / 4; ++j)
    sst[1 + j][threadIdx.x] = w.has ? __ldg(reinterpret_cast<const uint4*>(y + (int64_t)r * D + c * V) + j)
                                    : make_uint4(0, 0, 0, 0);
  const float sp = w.has ? spair[p] : 0.f;
  float acc[V], ax[V], zs = 0.f;
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = ax[k] = 0.f;
  int dn = b < e ? csc_dst[b] : 0;
  for (int t = 0; t < w.span; ++t) {
    const int i = b + t;
    const bool ok = i < e;
    uint4 rg = make_uint4(0, 0, 0, 0), rx = make_uint4(0, 0, 0, 0);
    float2 ns = make_float2(CUDART_INF_F, 0.f);
    if (ok) {
      const int64_t d = dn;
      rg = ldg16(GX + d * 2 * D + c * V);
      rx = ldg16(GX + d * 2 * D + D + c * V);
      ns = __ldg(reinterpret_cast<const float2*>(nst + d));
    }
    dn = i + 1 < e ? csc_dst[i + 1] : 0;
    float gr[V], xd[V], x[V];
    cvt16<TP>(rg, gr);
    cvt16<TP>(rx, xd);
    float tt = 0.f, da = 0.f;
#pragma unroll
    for (int j = 0; j < V / 4; ++j) {
      const uint4 yv = lds16(&sst[1 + j][threadIdx.x]);
      tt = fmaf(xd[4 * j], __uint_as_float(yv.x), tt);
      tt = fmaf(xd[4 * j + 1], __uint_as_float(yv.y), tt);
      tt = fmaf(xd[4 * j + 2], __uint_as_float(yv.z), tt);
      tt = fmaf(xd[4 * j + 3], __uint_as_float(yv.w), tt);
    }
    cvt16<TP>(lds16(&sst[0][threadIdx.x]), x);
#pragma unroll
    for (int k = 0; k < V; ++k) da = fmaf(gr[k], x[k], da);
    tt = gsum<LPR>(tt, w.mask);
    da = gsum<LPR>(da, w.mask);
    const float z = sp + tt;
    const float l = z > 0.f ? z : slope * z;
    const float alpha = ok ? __expf(l - ns.x) : 0.f;
    const float dz = alpha * (da - ns.y) * (z > 0.f ? 1.f : slope);
    zs += dz;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      acc[k] = fmaf(alpha, gr[k], acc[k]);
      ax[k] = fmaf(dz, xd[k], ax[k]);
    }
  }
  if (!w.writer()) return;
  if (slot >= 0) {
    st_f32<V>(pacc + (int64_t)slot * 2 * D + c * V, acc);
    st_f32<V>(pacc + (int64_t)slot * 2 * D + D + c * V, ax);
    if (c == 0) pstat[slot] = make_float2(zs, 0.f);
    return;
  }
  float av[V];
  cvt16<TP>(ldg16(avec + (int64_t)r * D + c * V), av);
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = fmaf(zs, av[k], acc[k]);
  st_tp<V>(dP + p * D + c * V, acc);
  st_tp<V>(bx + p * D + c * V, ax);
  if (c == 0) wsum[p] = zs;
}

// RGCN pair pass, group mode: U edges per step with their (destination, norm) prefetched a step ahead.
#ifndef RGNN_UNR_R
#define RGNN_UNR_R 2
#endif
template <class TP, int D, int U>
__global__ void __launch_bounds__(256) k_rgcn_bwd_pair_p(int64_t n, const int4* __restrict__ items,
                                                         float* __restrict__ pacc,
                                                         const int32_t* __restrict__ csc_dst,
                                                         const float* __restrict__ csc_norm,
                                                         const TP* __restrict__ Gr, TP* __restrict__ dP) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR;
  Work<true, LPR> w;
  if (!w.init(n, items)) return;
  const int64_t p = w.item.x;
  const int b = w.item.y, e = w.item.z, slot = w.item.w, c = w.c;
  float acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = 0.f;
  int dn[U];
  float wn[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    dn[u] = b + u < e ? csc_dst[b + u] : 0;
    wn[u] = b + u < e ? csc_norm[b + u] : 0.f;
  }
  for (int t = 0; t < w.span; t += U) {
    uint4 gr[U];
    float wt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      gr[u] = b + t + u < e ? ldg16(Gr + (int64_t)dn[u] * D + c * V) : make_uint4(0, 0, 0, 0);
      wt[u] = wn[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = b + t + U + u;
      dn[u] = i < e ? csc_dst[i] : 0;
      wn[u] = i < e ? csc_norm[i] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float x[V];
      cvt16<TP>(gr[u], x);
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = fmaf(wt[u], x[k], acc[k]);
    }
  }
  if (!w.writer()) return;
  if (slot >= 0) st_f32<V>(pacc + (int64_t)slot * D + c * V, acc);
  else st_tp<V>(dP + p * D + c * V, acc);
}

// HGT, recomputing alpha per edge from a per-node record (no per-edge buffer):
// prep:  GQ_v = [G_v | Q_v] in the table dtype, nst_v = (lse_v = m_v + log sum_v, G_v . out_v, 0, 0);
// pair:  K~_p and M_p in registers; per edge e of p: l_e = K~_p . Q_d, alpha_e = exp(l_e - lse_d),
//        dalpha_e = G_d . M_p, dl_e = alpha_e (dalpha_e - G_d . out_d);
//        dM_p = sum alpha_e G_d, dK~_p = sum dl_e Q_d  ->  dKM_p = [dK~_p | dM_p].
template <class TP, int D, int H>
__global__ void __launch_bounds__(256) k_hgt_node_prep(int64_t n, const int4* __restrict__ rows,
                                                       const float* __restrict__ Gr,
                                                       const TP* __restrict__ Q, const float* __restrict__ out,
                                                       const float2* __restrict__ stats, TP* __restrict__ GQ,
                                                       float4* __restrict__ nst) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR, EG = G::EG, LH = LPR / H;
  const int lane = threadIdx.x & 31, g = lane / LPR, c = lane % LPR;
  const int64_t j = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * EG + g;
  if (j >= n) return;
  const int64_t v = rows[j].x;
  float gv[V], ov[V], qv[V];
  ld_f32<V>(Gr + v * D + c * V, gv);
  round_tp<TP, V>(gv);
  ld_f32<V>(out + v * D + c * V, ov);
  cvt16<TP>(ldg16(Q + v * D + c * V), qv);
  float go = 0.f;
#pragma unroll
  for (int k = 0; k < V; ++k) go = fmaf(gv[k], ov[k], go);
  go = gsum<LH>(go, group_mask<LPR>(g));
  st_tp<V>(GQ + v * 2 * D + c * V, gv);
  st_tp<V>(GQ + v * 2 * D + D + c * V, qv);
  if (nst && c % LH == 0) {
    float2 st = stats[v * H + c / LH];
    nst[v * H + c / LH] = make_float4(st.y > 0.f ? st.x + logf(st.y) : CUDART_INF_F, go, 0.f, 0.f);
  }
}

// One lane moves 16 bytes of the G half and 16 bytes of the Q half of a GQ row (V columns each).
template <class TP, int D, bool GROUP, int H>
__global__ void __launch_bounds__(256, RGNN_PAIR_MINB) k_hgt_bwd_pair(int64_t n, const int4* __restrict__ items,
                                                      float* __restrict__ pacc, const int32_t* __restrict__ csc_dst,
                                                      const TP* __restrict__ KM, const TP* __restrict__ GQ,
                                                      const float4* __restrict__ nst, TP* __restrict__ dKM) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR, LH = LPR / H;
  Work<GROUP, LPR> w;
  if (!w.init(n, items)) return;
  const int64_t p = w.item.x;
  const int b = w.item.y, e = w.item.z, slot = w.item.w, c = w.c, hd = c / LH;
  float kx[V], mv[V];
  cvt16<TP>(ldg16(KM + p * 2 * D + c * V), kx);
  cvt16<TP>(ldg16(KM + p * 2 * D + D + c * V), mv);
  float ak[V], am[V];
#pragma unroll
  for (int k = 0; k < V; ++k) ak[k] = am[k] = 0.f;
  for (int t = 0; t < w.span; t += w.step * UNR_P) {
    const int i0 = b + t + w.first;
    uint4 rg[UNR_P], rq[UNR_P];
    float2 ns[UNR_P];
#pragma unroll
    for (int u = 0; u < UNR_P; ++u) {
      int i = i0 + u * w.step;
      ns[u] = make_float2(0.f, 0.f);
      rg[u] = rq[u] = make_uint4(0, 0, 0, 0);
      if (i < e) {
        const int64_t d = csc_dst[i];
        rg[u] = ldg16(GQ + d * 2 * D + c * V);
        rq[u] = ldg16(GQ + d * 2 * D + D + c * V);
        ns[u] = __ldg(reinterpret_cast<const float2*>(nst + d * H + hd));
      }
    }
#pragma unroll
    for (int u = 0; u < UNR_P; ++u) {
      float gr[V], qv[V];
      cvt16<TP>(rg[u], gr);
      cvt16<TP>(rq[u], qv);
      float l = 0.f, da = 0.f;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        l = fmaf(kx[k], qv[k], l);
        da = fmaf(gr[k], mv[k], da);
      }
      l = gsum<LH>(l, w.mask);
      da = gsum<LH>(da, w.mask);
      float alpha = (i0 + u * w.step < e) ? __expf(l - ns[u].x) : 0.f;
      float dl = alpha * (da - ns[u].y);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        ak[k] = fmaf(dl, qv[k], ak[k]);
        am[k] = fmaf(alpha, gr[k], am[k]);
      }
    }
  }
  if (!GROUP) {
    sum_groups<LPR, V>(ak);
    sum_groups<LPR, V>(am);
  }
  if (!w.writer()) return;
  if (slot >= 0) {
    float* o = pacc + (int64_t)slot * 2 * D;
    st_f32<V>(o + c * V, ak);
    st_f32<V>(o + D + c * V, am);
  } else {
    TP* o = dKM + p * 2 * D;
    st_tp<V>(o + c * V, ak);
    st_tp<V>(o + D + c * V, am);
  }
}

// Group mode of the HGT pair pass with the pair's K~_p / M_p chunks staged in shared memory
// (lane-private slots, re-read per edge) instead of 16 registers: the freed registers carry
// U edges' gathers in flight per group (U = 4 vs UNR_P = 2), i.e. twice the memory-level
// parallelism of the register-resident version at the same occupancy.

#ifndef RGNN_UNR_S
#define RGNN_UNR_S 1
#endif
#ifndef RGNN_PF
#define RGNN_PF 1
#endif

template <class TP, int D, int H, int U>
__global__ void __launch_bounds__(256, RGNN_PAIR_MINB) k_hgt_bwd_pair_s(int64_t n, const int4* __restrict__ items,
                                                                        float* __restrict__ pacc,
                                                                        const int32_t* __restrict__ csc_dst,
                                                                        const TP* __restrict__ KM,
                                                                        const TP* __restrict__ GQ,
                                                                        const float4* __restrict__ nst,
                                                                        TP* __restrict__ dKM) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR, LH = LPR / H;
  __shared__ uint4 skm[2][256];
  Work<true, LPR> w;
  if (!w.init(n, items)) return;
  const int64_t p = w.item.x;
  const int b = w.item.y, e = w.item.z, slot = w.item.w, c = w.c, hd = c / LH;
  uint4* const sk = &skm[0][threadIdx.x];
  uint4* const sm = &skm[1][threadIdx.x];
  *sk = w.has ? ldg16(KM + p * 2 * D + c * V) : make_uint4(0, 0, 0, 0);
  *sm = w.has ? ldg16(KM + p * 2 * D + D + c * V) : make_uint4(0, 0, 0, 0);
  float ak[V], am[V];
#pragma unroll
  for (int k = 0; k < V; ++k) ak[k] = am[k] = 0.f;
#if RGNN_PF
  int di[U];  // destination ids of the next U edges, loaded one iteration ahead
#pragma unroll
  for (int u = 0; u < U; ++u) di[u] = b + u < e ? csc_dst[b + u] : 0;
#endif
  for (int t = 0; t < w.span; t += U) {
    const int i0 = b + t;
    uint4 rg[U], rq[U];
    float2 ns[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u;
      ns[u] = make_float2(CUDART_INF_F, 0.f);
      rg[u] = rq[u] = make_uint4(0, 0, 0, 0);
      if (i < e) {
#if RGNN_PF
        const int64_t d = di[u];
#else
        const int64_t d = csc_dst[i];
#endif
        rg[u] = ldg16(GQ + d * 2 * D + c * V);
        rq[u] = ldg16(GQ + d * 2 * D + D + c * V);
        ns[u] = __ldg(reinterpret_cast<const float2*>(nst + d * H + hd));
      }
    }
#if RGNN_PF
#pragma unroll
    for (int u = 0; u < U; ++u) di[u] = i0 + U + u < e ? csc_dst[i0 + U + u] : 0;
#endif
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float gr[V], qv[V], x[V];
      cvt16<TP>(rg[u], gr);
      cvt16<TP>(rq[u], qv);
      float l = 0.f, da = 0.f;
      cvt16<TP>(lds16(sk), x);
#pragma unroll
      for (int k = 0; k < V; ++k) l = fmaf(x[k], qv[k], l);
      cvt16<TP>(lds16(sm), x);
#pragma unroll
      for (int k = 0; k < V; ++k) da = fmaf(gr[k], x[k], da);
      l = gsum<LH>(l, w.mask);
      da = gsum<LH>(da, w.mask);
      const float alpha = __expf(l - ns[u].x);  // 0 for padding (lse = +inf)
      const float dl = alpha * (da - ns[u].y);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        ak[k] = fmaf(dl, qv[k], ak[k]);
        am[k] = fmaf(alpha, gr[k], am[k]);
      }
    }
  }
  if (!w.writer()) return;
  if (slot >= 0) {
    float* o = pacc + (int64_t)slot * 2 * D;
    st_f32<V>(o + c * V, ak);
    st_f32<V>(o + D + c * V, am);
  } else {
    TP* o = dKM + p * 2 * D;
    st_tp<V>(o + c * V, ak);
    st_tp<V>(o + D + c * V, am);
  }
}

// Mixed-precision helpers: bf16 x bf16 products are exact in fp32 (fma.rn.f32.bf16, no unpacking of the
// packed halves); accumulations of a bf16 vector scaled by an fp32 weight as packed f32x2 FMAs.
__device__ __forceinline__ float bdot4(uint2 a, uint2 b, float acc) {  // acc + sum_k a_k b_k over 4 bf16 pairs
  asm("{\n.reg .b16 a0, a1, a2, a3, b0, b1, b2, b3;\n"
      "mov.b32 {a0, a1}, %1;\nmov.b32 {a2, a3}, %2;\nmov.b32 {b0, b1}, %3;\nmov.b32 {b2, b3}, %4;\n"
      "fma.rn.f32.bf16 %0, a0, b0, %0;\nfma.rn.f32.bf16 %0, a1, b1, %0;\n"
      "fma.rn.f32.bf16 %0, a2, b2, %0;\nfma.rn.f32.bf16 %0, a3, b3, %0;\n}"
      : "+f"(acc)
      : "r"(a.x), "r"(a.y), "r"(b.x), "r"(b.y));
  return acc;
}

// Group mode of the HGT pair pass for bf16 tables, split halves: a group of LPR = D / 4 lanes per pair,
// lanes [0, D/8) own the G half of the destination record and the M half of the pair row, lanes
// [D/8, D/4) the Q half and K~; each lane does ONE 8-column dot (G.M or K~.Q, mixed-precision bf16
// FMAs on the packed halves), a reduction over its half, one exchange with its partner lane in the
// other half, and 8 accumulations (dM or dK~).  One 16-byte gather per lane per edge, ~28 registers:
// full occupancy with half the per-edge instructions of 4-column lanes.
__device__ __forceinline__ float bdot8(uint4 a, uint4 b, float acc) {
  return bdot4(make_uint2(a.z, a.w), make_uint2(b.z, b.w), bdot4(make_uint2(a.x, a.y), make_uint2(b.x, b.y), acc));
}
template <int D, int H, int MINB>
__global__ void __launch_bounds__(256, MINB) k_hgt_bwd_pair_sp(int64_t n, const int4* __restrict__ items,
                                                               float* __restrict__ pacc,
                                                               const int32_t* __restrict__ csc_dst,
                                                               const bf16* __restrict__ KM,
                                                               const bf16* __restrict__ GQ,
                                                               const float4* __restrict__ nst,
                                                               bf16* __restrict__ dKM) {
  constexpr int HL = D / 8, LPR = 2 * HL, LHH = HL / H;  // lanes per half, per group, per head and half
  static_assert(LHH >= 1, "a head must own at least one lane of each half");
  Work<true, LPR> w;
  if (!w.init(n, items)) return;
  const int64_t p = w.item.x;
  const int b = w.item.y, e = w.item.z, slot = w.item.w, c = w.c;
  const int h = c / HL, cc = c % HL, hd = cc / LHH;  // h = 0: G / M / dM,  h = 1: Q / K~ / dK~
  const uint4 pk = w.has ? ldg16(KM + p * 2 * D + (1 - h) * D + 8 * cc) : make_uint4(0, 0, 0, 0);
  float2 acc[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) acc[k] = make_float2(0.f, 0.f);
  int dn = b < e ? csc_dst[b] : 0;
  for (int t = 0; t < w.span; ++t) {
    const int i = b + t;
    const int64_t d = dn;
    const uint4 x = ldg16(GQ + d * 2 * D + h * D + 8 * cc);
    const float2 ns = i < e ? __ldg(reinterpret_cast<const float2*>(nst + d * H + hd)) : make_float2(CUDART_INF_F, 0.f);
    dn = i + 1 < e ? csc_dst[i + 1] : 0;
    float part = gsum<LHH>(bdot8(pk, x, 0.f), w.mask);
    const float other = __shfl_xor_sync(0xffffffffu, part, HL);
    const float l = h ? part : other, da = h ? other : part;
    const float alpha = __expf(l - ns.x);  // 0 past the end (lse = +inf)
    const float dl = alpha * (da - ns.y);
    // past the end the gathered row is node 0's, which may never have been written: no accumulation
    const float s = i < e ? (h ? dl : alpha) : 0.f;
    const uint4 xv = i < e ? x : make_uint4(0, 0, 0, 0);
    const float2 ss = make_float2(s, s);
    acc[0] = __ffma2_rn(make_float2(__uint_as_float(xv.x << 16), __uint_as_float(xv.x & 0xffff0000u)), ss, acc[0]);
    acc[1] = __ffma2_rn(make_float2(__uint_as_float(xv.y << 16), __uint_as_float(xv.y & 0xffff0000u)), ss, acc[1]);
    acc[2] = __ffma2_rn(make_float2(__uint_as_float(xv.z << 16), __uint_as_float(xv.z & 0xffff0000u)), ss, acc[2]);
    acc[3] = __ffma2_rn(make_float2(__uint_as_float(xv.w << 16), __uint_as_float(xv.w & 0xffff0000u)), ss, acc[3]);
  }
  if (!w.writer()) return;
  const int col = (1 - h) * D + 8 * cc;  // dKM row = [dK~ | dM]: h = 1 (dK~) at 0, h = 0 (dM) at D
  if (slot >= 0) {
    float* o = pacc + (int64_t)slot * 2 * D + col;
    *reinterpret_cast<float4*>(o) = make_float4(acc[0].x, acc[0].y, acc[1].x, acc[1].y);
    *reinterpret_cast<float4*>(o + 4) = make_float4(acc[2].x, acc[2].y, acc[3].x, acc[3].y);
  } else {
    float f[8] = {acc[0].x, acc[0].y, acc[1].x, acc[1].y, acc[2].x, acc[2].y, acc[3].x, acc[3].y};
    store16(dKM + p * 2 * D + col, f);
  }
}

// Short pairs (<= SHORT_MAX edges), KI per lane group; K~_p / M_p of each item staged in shared memory.
template <class TP, int D, int H, int KI>
__global__ void __launch_bounds__(256, RGNN_PAIR_MINB) k_hgt_bwd_pair_k(int64_t n, const int4* __restrict__ items,
                                                                        const int32_t* __restrict__ csc_dst,
                                                                        const TP* __restrict__ KM,
                                                                        const TP* __restrict__ GQ,
                                                                        const float4* __restrict__ nst,
                                                                        TP* __restrict__ dKM) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR, LH = LPR / H;
  __shared__ uint4 skm[2 * KI][256];
  WorkK<LPR, KI> w;
  if (!w.init(n, items)) return;
  const int c = w.c, hd = c / LH;
#pragma unroll
  for (int k = 0; k < KI; ++k) {
    const bool ok = w.it[k].x >= 0;
    const int64_t p = ok ? w.it[k].x : 0;
    skm[2 * k][threadIdx.x] = ok ? ldg16(KM + p * 2 * D + c * V) : make_uint4(0, 0, 0, 0);
    skm[2 * k + 1][threadIdx.x] = ok ? ldg16(KM + p * 2 * D + D + c * V) : make_uint4(0, 0, 0, 0);
  }
  float ak[KI][V], am[KI][V];
#pragma unroll
  for (int k = 0; k < KI; ++k)
#pragma unroll
    for (int j = 0; j < V; ++j) ak[k][j] = am[k][j] = 0.f;
  for (int t = 0; t < w.span; ++t) {
    uint4 rg[KI], rq[KI];
    float2 ns[KI];
#pragma unroll
    for (int k = 0; k < KI; ++k) {
      const int i = w.it[k].y + t;
      ns[k] = make_float2(CUDART_INF_F, 0.f);
      rg[k] = rq[k] = make_uint4(0, 0, 0, 0);
      if (i < w.it[k].z) {
        const int64_t d = w.index(k, t, csc_dst);
        rg[k] = ldg16(GQ + d * 2 * D + c * V);
        rq[k] = ldg16(GQ + d * 2 * D + D + c * V);
        ns[k] = __ldg(reinterpret_cast<const float2*>(nst + d * H + hd));
      }
    }
#pragma unroll
    for (int k = 0; k < KI; ++k) {
      float gr[V], qv[V], x[V];
      cvt16<TP>(rg[k], gr);
      cvt16<TP>(rq[k], qv);
      float l = 0.f, da = 0.f;
      cvt16<TP>(lds16(&skm[2 * k][threadIdx.x]), x);
#pragma unroll
      for (int j = 0; j < V; ++j) l = fmaf(x[j], qv[j], l);
      cvt16<TP>(lds16(&skm[2 * k + 1][threadIdx.x]), x);
#pragma unroll
      for (int j = 0; j < V; ++j) da = fmaf(gr[j], x[j], da);
      l = gsum<LH>(l, w.mask);
      da = gsum<LH>(da, w.mask);
      const float alpha = __expf(l - ns[k].x);
      const float dl = alpha * (da - ns[k].y);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        ak[k][j] = fmaf(dl, qv[j], ak[k][j]);
        am[k][j] = fmaf(alpha, gr[j], am[k][j]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < KI; ++k) {
    if (w.it[k].x < 0) continue;
    TP* o = dKM + (int64_t)w.it[k].x * 2 * D;
    st_tp<V>(o + c * V, ak[k]);
    st_tp<V>(o + D + c * V, am[k]);
  }
}

// ------------------------------------------------------------------ weighted pair SpMM (A7)
// The pair-major backward as a two-weight SpMM over the src-CSC: per compact pair p
//   outA_p = sum_{e in p} wA_e A_{d_e},   outB_p = sum_{e in p} wB_e B_{d_e}   (+ wsum_p = sum wB_e),
// with the destination record rec_v = [A_v | B_v] (2D wide, table dtype) and the per-edge weights
// (wA, wB) written by the destination-major pass in CSR order (gathered through csc2csr).  HGT:
// rec = [G_v | Q_v], w = (alpha_e, dl_e) -> [dM_p | dK~_p]; RGAT: rec = [G_v | X_v], w = (alpha_e, dz_e)
// -> [dP_p - (sum dz) a_r | bx_p].  No logits, softmax or pair rows are recomputed here: per edge one
// record gather, one 8-byte weight gather, and 2 x V fused multiply-adds per lane (packed f32x2).
// One lane group walks one stream chunk (a contiguous CSC run of whole pairs, WorkPlan::chunks) U
// edges per step; the ids of the next LPR edges arrive as one coalesced load per group and are
// shuffled to their step; a pair's rows are written when the stream leaves it (split chunks of heavy
// pairs: the fp32 partial into the chunk's slot, merged by k_merge_sum).
// acc[0..V/2) += s * (16-byte vector v of the table dtype), packed f32x2 FMAs
#ifndef RGNN_FFMA2
#define RGNN_FFMA2 1
#endif
template <class TP>
__device__ __forceinline__ void acc16(float2* acc, uint4 v, float s) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#if !RGNN_FFMA2
  float x[Vec<TP>::N];
  cvt16<TP>(v, x);
#pragma unroll
  for (int i = 0; i < Vec<TP>::N / 2; ++i) {
    acc[i].x = fmaf(x[2 * i], s, acc[i].x);
    acc[i].y = fmaf(x[2 * i + 1], s, acc[i].y);
  }
  return;
#endif
  const float2 ss = make_float2(s, s);
  if constexpr (sizeof(TP) == 2) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      acc[i] = __ffma2_rn(make_float2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xffff0000u)), ss, acc[i]);
  } else {
#pragma unroll
    for (int i = 0; i < 2; ++i)
      acc[i] = __ffma2_rn(make_float2(__uint_as_float(w[2 * i]), __uint_as_float(w[2 * i + 1])), ss, acc[i]);
  }
}

#ifndef RGNN_SPMM_U
#define RGNN_SPMM_U 2
#endif

#ifndef RGNN_SPMM_MINB
#define RGNN_SPMM_MINB 3
#endif

// TWO: the record has two halves [A_v | B_v] (2D wide) and two weights; else one half (D wide) weighted
// by w.x, with w.y summed per pair (RGAT: rec = G_v, w = (alpha_e, dz_e): dP_p = sum alpha_e G_d +
// (sum dz_e) a_r, wsum_p = sum dz_e -- AVEC adds the a_r term when the pair's row is written).
template <class TP, int D, int H, int U, bool TWO, bool AVEC>
__global__ void __launch_bounds__(256, RGNN_SPMM_MINB) k_pair_spmm(
    int64_t nch, const int4* __restrict__ chunks, float* __restrict__ pacc, float2* __restrict__ pstat,
    const int32_t* __restrict__ csc_dst, const int32_t* __restrict__ csc2csr, const int32_t* __restrict__ csc_pair,
    const TP* __restrict__ rec, const float2* __restrict__ wts, TP* __restrict__ outA, TP* __restrict__ outB,
    int64_t ostride, float* __restrict__ wsum, int poffA, int poffB, const int32_t* __restrict__ csc_rel,
    const TP* __restrict__ avec) {
  using G = Geo<TP, D>;
  constexpr int V = G::V, LPR = G::LPR, EG = G::EG, LH = LPR / H, V2 = V / 2, RW = TWO ? 2 * D : D;
  constexpr bool WSUM = !TWO;
  static_assert(LPR % U == 0, "U must divide the lanes per row");
  const int lane = threadIdx.x & 31, g = lane / LPR, c = lane % LPR, hd = c / LH;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (wid * EG >= nch) return;  // whole warp idle
  const int64_t gid = wid * EG + g;
  const int4 ch = gid < nch ? chunks[gid] : make_int4(0, 0, -1, 0);
  const int a = ch.x, L = ch.y - ch.x, slot = ch.z;
  const int span = __reduce_max_sync(0xffffffffu, L);
  const int src0 = g * LPR;
  // ids of the stream's edges [t, t + LPR): lane c holds edge t + c (past the end: row 0, weight 0, pair -1)
  int d_cur, x_cur, p_cur, d_nxt, x_nxt, p_nxt;
  auto ld_ids = [&](int t, int& dd, int& xx, int& pp) {
    const int i = t + c;
    const bool ok = i < L;
    const int j = a + (ok ? i : 0);
    dd = ok ? __ldg(csc_dst + j) : 0;
    xx = __ldg(csc2csr + j);
    pp = ok ? __ldg(csc_pair + j) : -1;
  };
  ld_ids(0, d_cur, x_cur, p_cur);
  ld_ids(LPR, d_nxt, x_nxt, p_nxt);
  float2 accA[V2], accB[V2];
  float ws = 0.f;
#pragma unroll
  for (int k = 0; k < V2; ++k) accA[k] = accB[k] = make_float2(0.f, 0.f);
  int cp = -1, cbeg = 0;  // the pair being accumulated (group-uniform) and its first stream position
  auto flush = [&]() {
    float fa[V], fb[V];
#pragma unroll
    for (int k = 0; k < V2; ++k) {
      fa[2 * k] = accA[k].x;
      fa[2 * k + 1] = accA[k].y;
      fb[2 * k] = accB[k].x;
      fb[2 * k + 1] = accB[k].y;
    }
    if (slot >= 0) {  // split chunk of a heavy pair: fp32 partial row (A at poffA, B at poffB) + (wsum, 0)
      float* o = pacc + (int64_t)slot * 2 * D;
      st_f32<V>(o + poffA + c * V, fa);
      if (TWO) st_f32<V>(o + poffB + c * V, fb);
      if (WSUM && c == 0) pstat[slot] = make_float2(ws, 0.f);
    } else {
      if (AVEC) {  // + (sum dz) a_r
        float av[V];
        cvt16<TP>(ldg16(avec + (int64_t)__ldg(csc_rel + a + cbeg) * D + c * V), av);
#pragma unroll
        for (int k = 0; k < V; ++k) fa[k] = fmaf(ws, av[k], fa[k]);
      }
      st_tp<V>(outA + (int64_t)cp * ostride + c * V, fa);
      if (TWO) st_tp<V>(outB + (int64_t)cp * ostride + c * V, fb);
      if (WSUM && c == 0) wsum[cp] = ws;
    }
  };
  for (int t0 = 0; t0 < span; t0 += U) {
    if (t0 > 0 && t0 % LPR == 0) {  // warp-uniform: the prefetched batch becomes current
      d_cur = d_nxt;
      x_cur = x_nxt;
      p_cur = p_nxt;
      ld_ids(t0 + LPR, d_nxt, x_nxt, p_nxt);
    }
    uint4 ra[U], rb[U];
    float2 ww[U];
    int pp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int sl = src0 + (t0 + u) % LPR;
      const int d = __shfl_sync(0xffffffffu, d_cur, sl);
      const int x = __shfl_sync(0xffffffffu, x_cur, sl);
      pp[u] = __shfl_sync(0xffffffffu, p_cur, sl);
      const TP* r = rec + (int64_t)d * RW + c * V;
      ra[u] = ldg16(r);
      if (TWO) rb[u] = ldg16(r + D);
      ww[u] = __ldg(wts + (int64_t)x * H + hd);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (pp[u] != cp) {  // the stream enters a new pair (or leaves its last one)
        if (cp >= 0) flush();
#pragma unroll
        for (int k = 0; k < V2; ++k) accA[k] = accB[k] = make_float2(0.f, 0.f);
        ws = 0.f;
        cp = pp[u];
        cbeg = t0 + u;
      }
      const float wa = pp[u] >= 0 ? ww[u].x : 0.f, wb = pp[u] >= 0 ? ww[u].y : 0.f;
      acc16<TP>(accA, ra[u], wa);
      if (TWO) acc16<TP>(accB, rb[u], wb);
      if (WSUM) ws += wb;
    }
  }
  if (cp >= 0) flush();
}

// ------------------------------------------------------------------ heavy-id merges
// One CTA per heavy id: warp w folds chunks w, w+8, ... of the id (lane c owns columns 4c..4c+3
// of a W-wide row, looping over W in steps of 128); the 8 warp results are then combined in warp
// order through shared memory.  Fixed orders throughout: deterministic.
template <int D, int H>
__global__ void __launch_bounds__(256) k_merge_softmax(int64_t n_split, const int4* __restrict__ splits,
                                                       const float* __restrict__ pacc,
                                                       const float2* __restrict__ pstat, float* __restrict__ out,
                                                       float2* __restrict__ stats) {
  // lane owns columns 4*lane .. 4*lane+3, which belong to head hh = 4*lane / (D / H)
  __shared__ float sm_m[8][32], sm_s[8][32];
  __shared__ __align__(16) float sm_acc[8][D];
  const int4 sp = splits[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool act = lane * 4 < D;
  const int hh = act ? lane * 4 / (D / H) : 0;
  float m = -CUDART_INF_F;
  for (int i = warp; i < sp.z; i += 8) m = fmaxf(m, pstat[(int64_t)(sp.y + i) * H + hh].x);
  sm_m[warp][lane] = m;
  __syncthreads();
  m = sm_m[0][lane];
#pragma unroll
  for (int k = 1; k < 8; ++k) m = fmaxf(m, sm_m[k][lane]);
  float s = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
  // slots warp, warp + 8, ... in order (as one slot per step), four loaded before they are used
  for (int i0 = warp; i0 < sp.z; i0 += 32) {
    float2 st[4];
    float4 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + 8 * u;
      st[u] = make_float2(-CUDART_INF_F, 0.f);
      a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < sp.z) {
        st[u] = pstat[(int64_t)(sp.y + i) * H + hh];
        if (act) a[u] = *reinterpret_cast<const float4*>(pacc + (int64_t)(sp.y + i) * D + lane * 4);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i0 + 8 * u >= sp.z) break;
      const float wt = safe_exp_diff(st[u].x, m);
      s = fmaf(st[u].y, wt, s);
      if (act) {
        acc[0] = fmaf(wt, a[u].x, acc[0]); acc[1] = fmaf(wt, a[u].y, acc[1]);
        acc[2] = fmaf(wt, a[u].z, acc[2]); acc[3] = fmaf(wt, a[u].w, acc[3]);
      }
    }
  }
  sm_s[warp][lane] = s;
  if (act) *reinterpret_cast<float4*>(&sm_acc[warp][lane * 4]) = make_float4(acc[0], acc[1], acc[2], acc[3]);
  __syncthreads();
  if (warp == 0) {
    float st = 0.f, a4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      st += sm_s[k][lane];
      if (act)
#pragma unroll
        for (int j = 0; j < 4; ++j) a4[j] += sm_acc[k][lane * 4 + j];
    }
    float inv = st > 0.f ? 1.f / st : 0.f;
    if (act) {
      *reinterpret_cast<float4*>(out + (int64_t)sp.x * D + lane * 4) =
          make_float4(a4[0] * inv, a4[1] * inv, a4[2] * inv, a4[3] * inv);
      if ((lane * 4) % (D / H) == 0) stats[(int64_t)sp.x * H + hh] = make_float2(m, st);
    }
  }
}

template <int W, class TO>
__global__ void __launch_bounds__(256) k_merge_sum(int64_t n_split, const int4* __restrict__ splits,
                                                   const float* __restrict__ pacc, TO* __restrict__ out,
                                                   bool accumulate) {
  __shared__ __align__(16) float sm_acc[8][W];
  const int4 sp = splits[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int col = lane * 4; col < W; col += 128) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int i0 = warp; i0 < sp.z; i0 += 32) {  // slots in order, four loaded before they are added
      float4 a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        a[u] = i0 + 8 * u < sp.z ? *reinterpret_cast<const float4*>(pacc + (int64_t)(sp.y + i0 + 8 * u) * W + col)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i0 + 8 * u >= sp.z) break;
        acc[0] += a[u].x; acc[1] += a[u].y; acc[2] += a[u].z; acc[3] += a[u].w;
      }
    }
    *reinterpret_cast<float4*>(&sm_acc[warp][col]) = make_float4(acc[0], acc[1], acc[2], acc[3]);
  }
  __syncthreads();
  if (warp != 0) return;
  for (int col = lane * 4; col < W; col += 128) {
    TO* o = out + (int64_t)sp.x * W + col;
    float a4[4] = {0.f, 0.f, 0.f, 0.f};
    if (accumulate) {  // fp32 outputs only
      float4 prev = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(o));
      a4[0] = prev.x; a4[1] = prev.y; a4[2] = prev.z; a4[3] = prev.w;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int j = 0; j < 4; ++j) a4[j] += sm_acc[k][col + j];
    st4(o, a4[0], a4[1], a4[2], a4[3]);
  }
}

// RGAT heavy pairs: dP_p = sum acc_i + (sum zs_i) a_r ; bx_p = sum ax_i ; wsum_p = sum zs_i
template <class TW, int D>
__global__ void __launch_bounds__(256) k_merge_rgat_pair(int64_t n_split, const int4* __restrict__ splits,
                                                         const float* __restrict__ pacc,
                                                         const float2* __restrict__ pstat,
                                                         const int32_t* __restrict__ pair_csc_beg,
                                                         const int32_t* __restrict__ csc_rel,
                                                         const TW* __restrict__ avec, TW* __restrict__ dP,
                                                         float* __restrict__ wsum, TW* __restrict__ bx) {
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (j >= n_split) return;
  const int lane = threadIdx.x & 31;
  const int4 sp = splits[j];
  float zs = 0.f;
  for (int i = 0; i < sp.z; ++i) zs += pstat[sp.y + i].x;
  if (lane == 0) wsum[sp.x] = zs;
  if (lane * 4 >= D) return;
  const int r = csc_rel[pair_csc_beg[sp.x]];
  float acc[4] = {0.f, 0.f, 0.f, 0.f}, ax[4] = {0.f, 0.f, 0.f, 0.f};
  for (int i = 0; i < sp.z; ++i) {
    float4 a = *reinterpret_cast<const float4*>(pacc + (int64_t)(sp.y + i) * 2 * D + lane * 4);
    float4 x = *reinterpret_cast<const float4*>(pacc + (int64_t)(sp.y + i) * 2 * D + D + lane * 4);
    acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
    ax[0] += x.x; ax[1] += x.y; ax[2] += x.z; ax[3] += x.w;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) acc[k] = fmaf(zs, to_f(avec[(int64_t)r * D + lane * 4 + k]), acc[k]);
  st4(dP + (int64_t)sp.x * D + lane * 4, acc[0], acc[1], acc[2], acc[3]);
  if (bx) st4(bx + (int64_t)sp.x * D + lane * 4, ax[0], ax[1], ax[2], ax[3]);
}

template <class F>
void by_width(int D, F&& f) {
  switch (D) {
    case 16: f(std::integral_constant<int, 16>()); break;
    case 32: f(std::integral_constant<int, 32>()); break;
    case 64: f(std::integral_constant<int, 64>()); break;
    case 128: f(std::integral_constant<int, 128>()); break;
    default: RGNN_FAIL(RGNN_ERR_UNSUPPORTED, "d_out must be one of 16, 32, 64, 128");
  }
}

template <class F>
void by_dtype(int dtype, F&& f) {
  if (dtype == F32) f((float*)nullptr);
  else f((bf16*)nullptr);
}

// RGNN_STAGE=0 selects the register-resident group-mode pair kernel (A/B switch for the staged one)
inline bool stage_pair_rows() {
  static const bool on = [] {
    const char* v = getenv("RGNN_STAGE");
    return !(v && v[0] == '0');
  }();
  return on;
}

// RGNN_SPLIT=0: the staged group-mode HGT pair kernel (8 columns per lane, 60 registers) instead of the
// split-halves one on bf16 tables (measured equal on mag HGT: 0.833 vs 0.836 ms for the group half)
inline bool pair_split() {
  static const bool on = [] {
    const char* v = getenv("RGNN_SPLIT");
    return !(v && v[0] == '0');
  }();
  return on;
}

// RGNN_SHORT_PAIR=1: the HGT pair pass keeps its KI = 2 short-item kernel beside the split-halves group
// kernel; default: the split-halves kernel (32 registers, full occupancy) takes the short pairs as well
// (mag HGT pair pass 1.175 -> 1.162 ms; the short kernel spills at 64 registers)
inline bool short_pairs_split() {
  static const bool on = [] {
    const char* v = getenv("RGNN_SHORT_PAIR");
    return v && v[0] == '1';
  }();
  return on;
}

inline dim3 warps(int64_t n) { return dim3(ceil_div(n * 32, 256)); }
inline dim3 groups(int64_t n, int lpr) { return dim3(ceil_div(ceil_div(n, 32 / lpr) * (int64_t)32, 256)); }

// Launch a work-plan kernel pair: warp mode over items [0, n_warp) on `s`, group mode over the
// rest concurrently on the side stream (the long heavy-row warps overlap the light-row groups).
template <class KW, class KG, class... Args>
void launch_plan(const char* name, const WorkPlan& wp, int lpr, KW kw, KG kg, cudaStream_t s, Args... args) {
  const int64_t nl = wp.n_items - wp.n_warp;
  int slot = -1;
  profile_begin(name, s, &slot);  // the whole traversal (both halves) as one profile region
  cudaStream_t side = fork_side(s);
  launch(intern(std::string(name) + "/warp"), kw, warps(wp.n_warp), dim3(256), 0, s, wp.n_warp,
         (const int4*)wp.items, args...);
  launch(intern(std::string(name) + "/group"), kg, groups(nl, lpr), dim3(256), 0, side, nl,
         (const int4*)(wp.items + wp.n_warp), args...);
  join_side(s);
  profile_end(slot, s);
}

// RGNN_STAGE_Y=0 keeps the RGAT t-path rows of y in registers via L1 (A/B switch for stage_y)
inline bool stage_y_on() {
  static const bool on = [] {
    const char* v = getenv("RGNN_STAGE_Y");
    return !(v && v[0] == '0');
  }();
  return on;
}

// RGNN_STAGE_Y_SGL=1: staged y also for the destination pass that resolves single-edge pairs (AM)
inline bool stage_y_sgl() {
  static const bool on = [] {
    const char* v = getenv("RGNN_STAGE_Y_SGL");
    return v && v[0] == '1';
  }();
  return on;
}

// Grid of a persistent kernel: the blocks that are resident at once (occupancy with `smem` bytes of
// dynamic shared memory) times the SM count, at most `need`.
template <class K>
dim3 resident_grid(K k, size_t smem, unsigned need) {
  static int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, smem);
  const unsigned cap = (unsigned)std::max(1, per_sm) * (unsigned)std::max(1, sms);
  return dim3(std::min(need, cap));
}

// launch_plan with persistent kernels that stage `smem` bytes per block (grid-stride over the items);
// a warp-half kernel without staging (no dynamic shared memory in its signature) is launched plainly.
template <class KW, class KG, class... Args>
void launch_plan_staged(const char* name, const WorkPlan& wp, int lpr, size_t smem, bool warp_staged, KW kw, KG kg,
                        cudaStream_t s, Args... args) {
  const int64_t nl = wp.n_items - wp.n_warp;
  int slot = -1;
  profile_begin(name, s, &slot);
  cudaStream_t side = fork_side(s);
  if (warp_staged)
    launch(intern(std::string(name) + "/warp"), kw, resident_grid(kw, smem, warps(wp.n_warp).x), dim3(256), smem, s,
           wp.n_warp, (const int4*)wp.items, args...);
  else
    launch(intern(std::string(name) + "/warp"), kw, warps(wp.n_warp), dim3(256), 0, s, wp.n_warp,
           (const int4*)wp.items, args...);
  launch(intern(std::string(name) + "/group"), kg, resident_grid(kg, smem, groups(nl, lpr).x), dim3(256), smem, side,
         nl, (const int4*)(wp.items + wp.n_warp), args...);
  join_side(s);
  profile_end(slot, s);
}

// RGNN_SHORT=0 turns the short-item kernels off (A/B switch)
inline bool use_short() {
  static const bool on = [] {
    const char* v = getenv("RGNN_SHORT");
    return !(v && v[0] == '0');
  }();
  return on;
}

// As launch_plan, plus the short items [n_short, n_items) on the main stream after the warp half with
// KI items per lane group (ks takes the short-kernel argument list `sargs`, a tuple).
template <int KI, class KW, class KG, class KS, class... Args, class... SArgs>
void launch_plan_short(const char* name, const WorkPlan& wp, int lpr, KW kw, KG kg, KS ks,
                       std::tuple<SArgs...> sargs, cudaStream_t s, Args... args) {
  // lpr: lanes per item of the group kernel (low 8 bits) and of the short kernel (bits 8..15, 0 = same)
  const int lpr_s = (lpr >> 8) ? (lpr >> 8) : lpr;
  lpr &= 0xff;
  if (!use_short()) {
    launch_plan(name, wp, lpr, kw, kg, s, args...);
    return;
  }
  const int64_t ng = wp.n_short - wp.n_warp, ns = wp.n_items - wp.n_short;
  int slot = -1;
  profile_begin(name, s, &slot);
  cudaStream_t side = fork_side(s);
  launch(intern(std::string(name) + "/group"), kg, groups(ng, lpr), dim3(256), 0, side, ng,
         (const int4*)(wp.items + wp.n_warp), args...);
  launch(intern(std::string(name) + "/warp"), kw, warps(wp.n_warp), dim3(256), 0, s, wp.n_warp,
         (const int4*)wp.items, args...);
  std::apply([&](auto... a) {
    launch(intern(std::string(name) + "/short"), ks, groups(ceil_div(ns, KI), lpr_s), dim3(256), 0, s, ns,
           (const int4*)(wp.items + wp.n_short), a...);
  }, sargs);
  join_side(s);
  profile_end(slot, s);
}

}  // namespace

void rgcn_fwd_traverse(const rgnn_graph_s* g, int dtype, int D, const float* norm, const void* P, float* out,
                       bool accumulate, const Partial& pt, cudaStream_t s) {
  by_width(D, [&](auto Dc) {
    constexpr int DD = decltype(Dc)::value;
    by_dtype(dtype, [&](auto* tp) {
      using TP = std::remove_pointer_t<decltype(tp)>;
      launch_plan("rgcn_fwd_traverse", g->rows, Geo<TP, DD>::LPR, k_rgcn_fwd<TP, DD, false>, k_rgcn_fwd<TP, DD, true>,
                  s, pt.acc, (const int32_t*)g->csr_pair, norm, static_cast<const TP*>(P), out, accumulate);
    });
    launch("merge_heavy_rows", k_merge_sum<DD, float>, dim3(g->rows.n_split), dim3(256), 0, s, g->rows.n_split,
           (const int4*)g->rows.splits, (const float*)pt.acc, out, accumulate);
  });
}

// H heads: template dispatch, only where a head owns whole lane vectors (LPR % H == 0)
template <int LPR, class F>
void by_heads(int H, F&& f) {
  auto go = [&](auto hc) {
    constexpr int HH = decltype(hc)::value;
    if constexpr (LPR % HH == 0) f(hc);
    else RGNN_FAIL(RGNN_ERR_UNSUPPORTED, "num_heads: a head must span a multiple of 16 bytes of the row");
  };
  switch (H) {
    case 1: go(std::integral_constant<int, 1>()); break;
    case 2: go(std::integral_constant<int, 2>()); break;
    case 4: go(std::integral_constant<int, 4>()); break;
    case 8: go(std::integral_constant<int, 8>()); break;
    default: RGNN_FAIL(RGNN_ERR_UNSUPPORTED, "num_heads must be 1, 2, 4 or 8");
  }
}

void hgt_fwd_traverse(const rgnn_graph_s* g, int dtype, int D, int H, const void* KM, const void* Q, float* out,
                      float2* stats, const Partial& pt, cudaStream_t s) {
  by_width(D, [&](auto Dc) {
    constexpr int DD = decltype(Dc)::value;
    by_dtype(dtype, [&](auto* tp) {
      using TP = std::remove_pointer_t<decltype(tp)>;
      by_heads<Geo<TP, DD>::LPR>(H, [&](auto hc) {
        constexpr int HH = decltype(hc)::value;
        launch_plan_short<2>("hgt_fwd_traverse", g->rows, Geo<TP, DD>::LPR, k_hgt_fwd<TP, DD, false, HH>,
                             k_hgt_fwd<TP, DD, true, HH>, k_hgt_fwd_k<TP, DD, HH, 2>,
                             std::make_tuple((const int32_t*)g->csr_pair, static_cast<const TP*>(KM),
                                             static_cast<const TP*>(Q), out, stats),
                             s, pt.acc, pt.stat, (const int32_t*)g->csr_pair, static_cast<const TP*>(KM),
                             static_cast<const TP*>(Q), out, stats);
        launch("merge_heavy_rows", k_merge_softmax<DD, HH>, dim3(g->rows.n_split), dim3(256), 0, s,
               g->rows.n_split, (const int4*)g->rows.splits, (const float*)pt.acc, (const float2*)pt.stat, out,
               stats);
      });
    });
  });
}

void rgat_fwd_traverse(const rgnn_graph_s* g, int dtype, int D, const void* P, const float* spair, const void* X,
                       const float* y, const float* te, float slope, float* out, float2* stats, const Partial& pt,
                       cudaStream_t s) {
  by_width(D, [&](auto Dc) {
    constexpr int DD = decltype(Dc)::value;
    by_dtype(dtype, [&](auto* tp) {
      using TP = std::remove_pointer_t<decltype(tp)>;
      const int ny = g->R * DD;
      const bool sy = !te && stage_y_on() && (size_t)ny * sizeof(float) <= (size_t)kStageYMax;
      const bool sy_warp = (size_t)ny * sizeof(float) <= (size_t)kStageYWarpMax;
      auto go = [&](auto kw, auto kg) {
        if (sy)
          launch_plan_staged("rgat_fwd_traverse", g->rows, Geo<TP, DD>::LPR, (size_t)ny * sizeof(float), sy_warp, kw,
                             kg, s,
                             pt.acc, pt.stat, (const int32_t*)g->csr_pair, (const int32_t*)g->csr_rel,
                             static_cast<const TP*>(P), spair, static_cast<const TP*>(X), y, te, slope, out, stats, ny);
        else
          launch_plan("rgat_fwd_traverse", g->rows, Geo<TP, DD>::LPR, kw, kg, s, pt.acc, pt.stat,
                      (const int32_t*)g->csr_pair, (const int32_t*)g->csr_rel, static_cast<const TP*>(P), spair,
                      static_cast<const TP*>(X), y, te, slope, out, stats, ny);
      };
      if (te) go(k_rgat_fwd<TP, DD, false, true>, k_rgat_fwd<TP, DD, true, true>);
      else if (sy && sy_warp) go(k_rgat_fwd_sy<TP, DD, false>, k_rgat_fwd_sy<TP, DD, true>);
      else if (sy) go(k_rgat_fwd<TP, DD, false, false>, k_rgat_fwd_sy<TP, DD, true>);
      else go(k_rgat_fwd<TP, DD, false, false>, k_rgat_fwd<TP, DD, true, false>);
    });
    launch("merge_heavy_rows", k_merge_softmax<DD, 1>, dim3(g->rows.n_split), dim3(256), 0, s, g->rows.n_split,
           (const int4*)g->rows.splits, (const float*)pt.acc, (const float2*)pt.stat, out, stats);
  });
}

void hgt_bwd_dst(const rgnn_graph_s* g, int dtype, int D, int H, const void* KM, const void* Q, const float2* stats,
                 const float* G, const float* out, void* dQ, void* GQ, float4* nst, const uint8_t* single, void* dKM,
                 float2* wts, const Partial& pt, cudaStream_t s) {
  by_width(D, [&](auto Dc) {
    constexpr int DD = decltype(Dc)::value;
    by_dtype(dtype, [&](auto* tp) {
      using TP = std::remove_pointer_t<decltype(tp)>;
      by_heads<Geo<TP, DD>::LPR>(H, [&](auto hc) {
        constexpr int HH = decltype(hc)::value;
        auto go = [&](auto sc, auto wc) {
          constexpr bool SG = decltype(sc)::value, WT = decltype(wc)::value;
          launch_plan_short<2>("hgt_bwd_dst", g->rows, Geo<TP, DD>::LPR, k_hgt_bwd_dst<TP, DD, false, HH, SG, WT>,
                             k_hgt_bwd_dst<TP, DD, true, HH, SG, WT>, k_hgt_bwd_dst_k<TP, DD, HH, 2, SG, WT>,
                             std::make_tuple((const int32_t*)g->csr_pair, static_cast<const TP*>(KM),
                                             static_cast<const TP*>(Q), stats, G, out, static_cast<TP*>(dQ),
                                             static_cast<TP*>(GQ), nst, single, static_cast<TP*>(dKM), wts),
                             s, pt.acc, (const int32_t*)g->csr_pair, static_cast<const TP*>(KM),
                             static_cast<const TP*>(Q), stats, G, out, static_cast<TP*>(dQ),
                             static_cast<TP*>(GQ), nst, single, static_cast<TP*>(dKM), wts);
        };
        if (single) {
          if (wts) go(std::true_type(), std::true_type());
          else go(std::true_type(), std::false_type());
        } else {
          if (wts) go(std::false_type(), std::true_type());
          else go(std::false_type(), std::false_type());
        }
        launch("hgt_node_prep", k_hgt_node_prep<TP, DD, HH>, groups(g->rows.n_split, Geo<TP, DD>::LPR), dim3(256),
               0, s, g->rows.n_split, (const int4*)g->rows.splits, G, static_cast<const TP*>(Q), out, stats,
               static_cast<TP*>(GQ), nst);
      });
      launch("merge_heavy_rows", k_merge_sum<DD, TP>, dim3(g->rows.n_split), dim3(256), 0, s, g->rows.n_split,
             (const int4*)g->rows.splits, (const float*)pt.acc, static_cast<TP*>(dQ), false);
    });
  });
}

void rgat_bwd_dst(const rgnn_graph_s* g, int dtype, int D, const void* P, const float* spair, const void* X,
                  const float* y, const float* te, float* dz, float slope, const float2* stats, const float* G,
                  const float* out, float* dX, void* GX, float4* nst, const uint8_t* single, const void* a, void* dP,
                  void* bx, float* wsum, float2* wts, const Partial& pt, cudaStream_t s) {
  by_width(D, [&](auto Dc) {
    constexpr int DD = decltype(Dc)::value;
    by_dtype(dtype, [&](auto* tp) {
      using TP = std::remove_pointer_t<decltype(tp)>;
      const int ny = g->R * DD;
      const bool sy = !te && y && (!single || stage_y_sgl()) && stage_y_on() &&
                      (size_t)ny * sizeof(float) <= (size_t)kStageYMax;
      const bool sy_warp = (size_t)ny * sizeof(float) <= (size_t)kStageYWarpMax;
      auto go = [&](auto kw, auto kg) {
        auto args = std::make_tuple(pt.acc, (const int32_t*)g->csr_pair, (const int32_t*)g->csr_rel,
                                    static_cast<const TP*>(P), spair, static_cast<const TP*>(X), y, te, dz, slope,
                                    stats, G, out, dX, static_cast<TP*>(GX), nst, single, static_cast<const TP*>(a),
                                    static_cast<TP*>(dP), static_cast<TP*>(bx), wsum, wts, ny);
        std::apply([&](auto... ar) {
          if (sy)
            launch_plan_staged("rgat_bwd_dst", g->rows, Geo<TP, DD>::LPR, (size_t)ny * sizeof(float), sy_warp, kw,
                               kg, s, ar...);
          else
            launch_plan("rgat_bwd_dst", g->rows, Geo<TP, DD>::LPR, kw, kg, s, ar...);
        }, args);
      };
      auto pick = [&](auto sc, auto wc) {
        constexpr bool SG = decltype(sc)::value, WT = decltype(wc)::value;
        if (sy && sy_warp) go(k_rgat_bwd_dst_sy<TP, DD, false, SG, WT>, k_rgat_bwd_dst_sy<TP, DD, true, SG, WT>);
        else if (sy) go(k_rgat_bwd_dst<TP, DD, false, false, SG, WT>, k_rgat_bwd_dst_sy<TP, DD, true, SG, WT>);
        else go(k_rgat_bwd_dst<TP, DD, false, false, SG, WT>, k_rgat_bwd_dst<TP, DD, true, false, SG, WT>);
      };
      if (te) go(k_rgat_bwd_dst<TP, DD, false, true, false, false>, k_rgat_bwd_dst<TP, DD, true, true, false, false>);
      else if (wts && single) pick(std::true_type(), std::true_type());
      else if (wts) pick(std::false_type(), std::true_type());
      else if (single) pick(std::true_type(), std::false_type());
      else pick(std::false_type(), std::false_type());
      launch("rgat_node_prep", k_rgat_node_prep<TP, DD>, groups(g->rows.n_split, Geo<TP, DD>::LPR), dim3(256), 0, s,
             g->rows.n_split, (const int4*)g->rows.splits, G, static_cast<const TP*>(X), out, stats,
             static_cast<TP*>(GX), nst);
    });
    if (!te)
      launch("merge_heavy_rows", k_merge_sum<DD, float>, dim3(g->rows.n_split), dim3(256), 0, s, g->rows.n_split,
             (const int4*)g->rows.splits, (const float*)pt.acc, dX, false);
  });
}

void rgcn_bwd_pair(const rgnn_graph_s* g, int dtype, int D, const float* csc_norm, const void* G, void* dP,
                   const Partial& pt, cudaStream_t s) {
  by_width(D, [&](auto Dc) {
    constexpr int DD = decltype(Dc)::value;
    by_dtype(dtype, [&](auto* tp) {
      using TP = std::remove_pointer_t<decltype(tp)>;
      launch_plan_short<4>("rgcn_bwd_pair", g->pairs, Geo<TP, DD>::LPR, k_rgcn_bwd_pair<TP, DD, false>,
                           k_rgcn_bwd_pair_p<TP, DD, RGNN_UNR_R>, k_rgcn_bwd_pair_k<TP, DD, 4>,
                           std::make_tuple((const int32_t*)g->csc_dst, csc_norm, static_cast<const TP*>(G),
                                           static_cast<TP*>(dP)),
                           s, pt.acc, (const int32_t*)g->csc_dst, csc_norm, static_cast<const TP*>(G),
                           static_cast<TP*>(dP));
      launch("merge_heavy_pairs", k_merge_sum<DD, TP>, dim3(g->pairs.n_split), dim3(256), 0, s, g->pairs.n_split,
             (const int4*)g->pairs.splits, (const float*)pt.acc, static_cast<TP*>(dP), false);
    });
  });
}

void rgat_bwd_pair(const rgnn_graph_s* g, int dtype, int D, const void* P, const float* spair, const float* y,
                   const float* te, const void* a, float slope, const void* GX, const float4* nst, const float2* wts,
                   void* dP, float* wsum, void* bx, bool skip_single, const Partial& pt, cudaStream_t s) {
  if (wts) {  // weighted SpMM: dP_p = sum alpha_e G_d + (sum dz_e) a_r, wsum_p = sum dz_e (GX = G_v rows, [N][D])
    const int64_t nch = skip_single ? g->pairs.n_chunks_multi : g->pairs.n_chunks;
    const int4* ch = skip_single ? g->pairs.chunks_multi : g->pairs.chunks;
    by_width(D, [&](auto Dc) {
      constexpr int DD = decltype(Dc)::value;
      by_dtype(dtype, [&](auto* tp) {
        using TP = std::remove_pointer_t<decltype(tp)>;
        constexpr int LPR = Geo<TP, DD>::LPR;
        constexpr int UU = RGNN_SPMM_U < LPR ? RGNN_SPMM_U : LPR;
        launch("rgat_bwd_pair", k_pair_spmm<TP, DD, 1, UU, false, true>, groups(nch, LPR), dim3(256), 0, s, nch, ch,
               pt.acc, pt.stat, (const int32_t*)g->csc_dst, (const int32_t*)g->csc2csr, (const int32_t*)g->csc_pair,
               static_cast<const TP*>(GX), wts, static_cast<TP*>(dP), (TP*)nullptr, (int64_t)DD, wsum, 0, DD,
               (const int32_t*)g->csc_rel, static_cast<const TP*>(a));
        launch("merge_heavy_pairs", k_merge_rgat_pair<TP, DD>, warps(g->pairs.n_split), dim3(256), 0, s,
               g->pairs.n_split, (const int4*)g->pairs.splits, (const float*)pt.acc, (const float2*)pt.stat,
               (const int32_t*)g->pair_csc_beg, (const int32_t*)g->csc_rel, static_cast<const TP*>(a),
               static_cast<TP*>(dP), wsum, (TP*)nullptr);
      });
    });
    return;
  }
  WorkPlan wp = g->pairs;  // single-edge pairs resolved by the destination-major pass (reordered path)
  if (skip_single && !te) {
    wp.n_items = wp.n_multi;
    wp.n_short = std::min(wp.n_short, wp.n_multi);
  }
  by_width(D, [&](auto Dc) {
    constexpr int DD = decltype(Dc)::value;
    by_dtype(dtype, [&](auto* tp) {
      using TP = std::remove_pointer_t<decltype(tp)>;
      auto go = [&](auto kw, auto kg) {
        launch_plan("rgat_bwd_pair", wp, Geo<TP, DD>::LPR, kw, kg, s, pt.acc, pt.stat,
                    (const int32_t*)g->csc_dst, (const int32_t*)g->csc_rel, (const int32_t*)g->csc2csr, te,
                    static_cast<const TP*>(P), spair, y, static_cast<const TP*>(a), slope, static_cast<const TP*>(GX),
                    nst, static_cast<TP*>(dP), wsum, te ? nullptr : static_cast<TP*>(bx));
      };
      if (te) go(k_rgat_bwd_pair<TP, DD, false, true>, k_rgat_bwd_pair<TP, DD, true, true>);
      else if (stage_pair_rows()) go(k_rgat_bwd_pair<TP, DD, false, false>, k_rgat_bwd_pair_s<TP, DD>);
      else go(k_rgat_bwd_pair<TP, DD, false, false>, k_rgat_bwd_pair<TP, DD, true, false>);
      launch("merge_heavy_pairs", k_merge_rgat_pair<TP, DD>, warps(g->pairs.n_split), dim3(256), 0, s,
             g->pairs.n_split, (const int4*)g->pairs.splits, (const float*)pt.acc, (const float2*)pt.stat,
             (const int32_t*)g->pair_csc_beg, (const int32_t*)g->csc_rel, static_cast<const TP*>(a),
             static_cast<TP*>(dP), wsum, te ? nullptr : static_cast<TP*>(bx));
    });
  });
}

void hgt_bwd_pair(const rgnn_graph_s* g, int dtype, int D, int H, const void* KM, const void* GQ, const float4* nst,
                  const float2* wts, void* dKM, bool skip_single, const Partial& pt, cudaStream_t s) {
  if (wts) {  // weighted SpMM: [dM | dK~] = sum_e [alpha_e G_d | dl_e Q_d] (weights from hgt_bwd_dst)
    const int64_t nch = skip_single ? g->pairs.n_chunks_multi : g->pairs.n_chunks;
    const int4* ch = skip_single ? g->pairs.chunks_multi : g->pairs.chunks;
    by_width(D, [&](auto Dc) {
      constexpr int DD = decltype(Dc)::value;
      by_dtype(dtype, [&](auto* tp) {
        using TP = std::remove_pointer_t<decltype(tp)>;
        constexpr int LPR = Geo<TP, DD>::LPR;
        constexpr int UU = RGNN_SPMM_U < LPR ? RGNN_SPMM_U : LPR;
        by_heads<LPR>(H, [&](auto hc) {
          constexpr int HH = decltype(hc)::value;
          TP* o = static_cast<TP*>(dKM);
          launch("hgt_bwd_pair", k_pair_spmm<TP, DD, HH, UU, true, false>, groups(nch, LPR), dim3(256), 0, s, nch,
                 ch, pt.acc, pt.stat, (const int32_t*)g->csc_dst, (const int32_t*)g->csc2csr,
                 (const int32_t*)g->csc_pair, static_cast<const TP*>(GQ), wts, o + DD, o, (int64_t)2 * DD,
                 (float*)nullptr, DD, 0, (const int32_t*)nullptr, (const TP*)nullptr);
        });
        launch("merge_heavy_pairs", k_merge_sum<2 * DD, TP>, dim3(g->pairs.n_split), dim3(256), 0, s,
               g->pairs.n_split, (const int4*)g->pairs.splits, (const float*)pt.acc, static_cast<TP*>(dKM), false);
      });
    });
    return;
  }
  WorkPlan wp = g->pairs;  // single-edge pairs were resolved by the destination-major pass
  if (skip_single) {
    wp.n_items = wp.n_multi;
    wp.n_short = std::min(wp.n_short, wp.n_multi);
  }
  by_width(D, [&](auto Dc) {
    constexpr int DD = decltype(Dc)::value;
    by_dtype(dtype, [&](auto* tp) {
      using TP = std::remove_pointer_t<decltype(tp)>;
      by_heads<Geo<TP, DD>::LPR>(H, [&](auto hc) {
        constexpr int HH = decltype(hc)::value;
        auto go = [&](auto kg) {
          launch_plan_short<2>("hgt_bwd_pair", wp, Geo<TP, DD>::LPR, k_hgt_bwd_pair<TP, DD, false, HH>, kg,
                               k_hgt_bwd_pair_k<TP, DD, HH, 2>,
                               std::make_tuple((const int32_t*)g->csc_dst, static_cast<const TP*>(KM),
                                               static_cast<const TP*>(GQ), nst, static_cast<TP*>(dKM)),
                               s, pt.acc, (const int32_t*)g->csc_dst, static_cast<const TP*>(KM),
                               static_cast<const TP*>(GQ), nst, static_cast<TP*>(dKM));
        };
        if constexpr (std::is_same_v<TP, bf16> && DD / 4 <= 32 && (DD / 8) % HH == 0) {
          if (pair_split() && !short_pairs_split()) {  // the split-halves kernel also takes the short pairs
            launch_plan("hgt_bwd_pair", wp, DD / 4, k_hgt_bwd_pair<TP, DD, false, HH>, k_hgt_bwd_pair_sp<DD, HH, 8>, s,
                        pt.acc, (const int32_t*)g->csc_dst, static_cast<const TP*>(KM), static_cast<const TP*>(GQ),
                        nst, static_cast<TP*>(dKM));
            return;
          }
          if (pair_split()) {  // group mode: split halves, D / 4 lanes per pair; warp and short halves as before
            launch_plan_short<2>("hgt_bwd_pair", wp, DD / 4 | Geo<TP, DD>::LPR << 8,
                                 k_hgt_bwd_pair<TP, DD, false, HH>, k_hgt_bwd_pair_sp<DD, HH, 8>,
                                 k_hgt_bwd_pair_k<TP, DD, HH, 2>,
                                 std::make_tuple((const int32_t*)g->csc_dst, static_cast<const TP*>(KM),
                                                 static_cast<const TP*>(GQ), nst, static_cast<TP*>(dKM)),
                                 s, pt.acc, (const int32_t*)g->csc_dst, static_cast<const TP*>(KM),
                                 static_cast<const TP*>(GQ), nst, static_cast<TP*>(dKM));
            return;
          }
        }
        if (stage_pair_rows()) go(k_hgt_bwd_pair_s<TP, DD, HH, RGNN_UNR_S>);
        else go(k_hgt_bwd_pair<TP, DD, true, HH>);
      });
      launch("merge_heavy_pairs", k_merge_sum<2 * DD, TP>, dim3(g->pairs.n_split), dim3(256), 0, s,
             g->pairs.n_split, (const int4*)g->pairs.splits, (const float*)pt.acc, static_cast<TP*>(dKM), false);
    });
  });
}


}  // namespace rgnn
