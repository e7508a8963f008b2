// F4 training step around the layers (include/rgnn.h "F4"): ReLU between stacked layers,
// the NLL loss of log_softmax outputs against random labels (§3.4.1), and a
// multi-tensor SGD update with an optional low-precision shadow copy of each weight.
// All HBM-bound elementwise / row work: 16-byte vectors, grids sized to the SM count.
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace rgnn {
namespace {

constexpr int kSMs = 148;

inline dim3 vec_grid(int64_t n4) {
  return dim3((unsigned)std::min<int64_t>(std::max<int64_t>(ceil_div(n4, 256), 1), kSMs * 8));
}

// ------------------------------------------------------------------ ReLU
template <class TO>
__global__ void k_relu_fwd(int64_t n, const float* __restrict__ h, TO* __restrict__ a) {
  const int64_t n4 = n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 v = __ldg(reinterpret_cast<const float4*>(h) + i);
    v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
    if constexpr (sizeof(TO) == 4) {
      reinterpret_cast<float4*>(a)[i] = v;
    } else {
      __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
      uint2 o;
      o.x = *reinterpret_cast<uint32_t*>(&lo);
      o.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(a)[i] = o;
    }
  }
  const int64_t t = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) a[t] = from_f<TO>(fmaxf(h[t], 0.f));
}

__global__ void k_relu_bwd(int64_t n, const float* __restrict__ h, const float* da, float* dh) {
  const int64_t n4 = n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(h) + i);
    float4 g = reinterpret_cast<const float4*>(da)[i];
    g.x = x.x > 0.f ? g.x : 0.f; g.y = x.y > 0.f ? g.y : 0.f;
    g.z = x.z > 0.f ? g.z : 0.f; g.w = x.w > 0.f ? g.w : 0.f;
    reinterpret_cast<float4*>(dh)[i] = g;
  }
  const int64_t t = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) dh[t] = h[t] > 0.f ? da[t] : 0.f;
}

// ------------------------------------------------------------------ NLL of log_softmax
// One warp per row; the row lives in registers (PER values per lane, column j = lane + 32 k),
// so logits are read once and dlogits written once.  Per-warp sums -> per-block partials in
// fixed warp order -> one block sums the partials in fixed order (deterministic).
constexpr int kNllThreads = 256, kNllWarps = kNllThreads / 32;

struct NllPartial {
  double loss;
  long long count;
  int bad;
  int pad_;
};

template <int PER>
__global__ void __launch_bounds__(kNllThreads) k_nll_rows(int64_t n, int c, const float* __restrict__ z,
                                                         const int32_t* __restrict__ y, float inv_count,
                                                         float* __restrict__ dz, NllPartial* __restrict__ part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double wloss = 0.0;
  long long wcount = 0;
  int wbad = 0;
  for (int64_t row = (int64_t)blockIdx.x * kNllWarps + warp; row < n; row += (int64_t)gridDim.x * kNllWarps) {
    const float* zr = z + row * c;
    float v[PER];
    float m = -INFINITY;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int j = lane + 32 * k;
      v[k] = j < c ? __ldg(zr + j) : -INFINITY;
      m = fmaxf(m, v[k]);
    }
    m = warp_max(m);
    const int lab = __ldg(y + row);  // row-uniform
    const bool labelled = lab >= 0 && lab < c;
    if (lab >= c) wbad = 1;
    float zy = 0.f;
    if (labelled) {
      const int kl = lab >> 5;
#pragma unroll
      for (int k = 0; k < PER; ++k)
        if (k == kl) zy = v[k];
      zy = __shfl_sync(0xffffffffu, zy, lab & 31);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      v[k] = expf(v[k] - m);  // exp(-inf) = 0 for padding columns
      s += v[k];
    }
    s = group_sum<32>(s);
    if (labelled && lane == 0) {
      wloss -= (double)(zy - m) - (double)logf(s);  // log softmax at the label
      wcount += 1;
    }
    if (dz) {
      float* dr = dz + row * c;
      const float scale = labelled ? inv_count / s : 0.f;
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int j = lane + 32 * k;
        if (j < c) dr[j] = v[k] * scale - ((labelled && j == lab) ? inv_count : 0.f);
      }
    }
  }
  __shared__ NllPartial sp[kNllWarps];
  const int anybad = __any_sync(0xffffffffu, wbad);
  if (lane == 0) sp[warp] = NllPartial{wloss, wcount, anybad ? 1 : 0, 0};
  __syncthreads();
  if (threadIdx.x == 0) {
    NllPartial p{0.0, 0, 0, 0};
    for (int w = 0; w < kNllWarps; ++w) {
      p.loss += sp[w].loss;
      p.count += sp[w].count;
      p.bad |= sp[w].bad;
    }
    part[blockIdx.x] = p;
  }
}

// C in {64, 128, 256}: L = C / 8 lanes per row (8 values = two 16-byte vectors per lane), 32 / L
// rows per warp at once; the same per-block partials as k_nll_rows.
template <int C>
__global__ void __launch_bounds__(kNllThreads) k_nll_rows_v(int64_t n, const float* __restrict__ z,
                                                           const int32_t* __restrict__ y, float inv_count,
                                                           float* __restrict__ dz, NllPartial* __restrict__ part) {
  constexpr int L = C / 8, RPW = 32 / L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane / L, c = lane % L;
  const unsigned gmask = (L == 32) ? 0xffffffffu : (((1u << L) - 1u) << (g * L));
  double wloss = 0.0;
  long long wcount = 0;
  int wbad = 0;
  const int64_t stride = (int64_t)gridDim.x * kNllWarps * RPW;
  for (int64_t row = ((int64_t)blockIdx.x * kNllWarps + warp) * RPW + g; row - g < n; row += stride) {
    const bool has = row < n;
    float v[8];
    if (has) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(z + row * C + c * 8));
      const float4 b = __ldg(reinterpret_cast<const float4*>(z + row * C + c * 8 + 4));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = 0.f;
    }
    const int lab = has ? __ldg(y + row) : -1;
    float m = v[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) m = fmaxf(m, v[k]);
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const bool labelled = lab >= 0 && lab < C;
    if (lab >= C) wbad = 1;
    float zy = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (labelled && c * 8 + k == lab) zy = v[k];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = expf(v[k] - m);
      s += v[k];
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      zy += __shfl_xor_sync(0xffffffffu, zy, o);
    }
    if (labelled && c == 0) {
      wloss -= (double)(zy - m) - (double)logf(s);
      wcount += 1;
    }
    if (dz && has) {
      const float scale = labelled ? inv_count / s : 0.f;
      float o8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) o8[k] = v[k] * scale - ((labelled && c * 8 + k == lab) ? inv_count : 0.f);
      float* dr = dz + row * C + c * 8;
      *reinterpret_cast<float4*>(dr) = make_float4(o8[0], o8[1], o8[2], o8[3]);
      *reinterpret_cast<float4*>(dr + 4) = make_float4(o8[4], o8[5], o8[6], o8[7]);
    }
    (void)gmask;
  }
  // warp totals in lane order (fixed), then the block's warps in order
  double wl = wloss;
  long long wc = wcount;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    wl += __shfl_xor_sync(0xffffffffu, wl, o);
    wc += __shfl_xor_sync(0xffffffffu, wc, o);
  }
  __shared__ NllPartial sp[kNllWarps];
  const int anybad = __any_sync(0xffffffffu, wbad);
  if (lane == 0) sp[warp] = NllPartial{wl, wc, anybad ? 1 : 0, 0};
  __syncthreads();
  if (threadIdx.x == 0) {
    NllPartial p{0.0, 0, 0, 0};
    for (int w = 0; w < kNllWarps; ++w) {
      p.loss += sp[w].loss;
      p.count += sp[w].count;
      p.bad |= sp[w].bad;
    }
    part[blockIdx.x] = p;
  }
}

__global__ void __launch_bounds__(256) k_nll_final(int nparts, const NllPartial* __restrict__ part,
                                                   long long num_labeled, float* __restrict__ loss) {
  __shared__ double sl[256];
  __shared__ long long sc[256];
  __shared__ int sb[256];
  double l = 0.0;
  long long cnt = 0;
  int bad = 0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) {  // fixed assignment of partials to threads
    l += part[i].loss;
    cnt += part[i].count;
    bad |= part[i].bad;
  }
  sl[threadIdx.x] = l;
  sc[threadIdx.x] = cnt;
  sb[threadIdx.x] = bad;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {  // fixed tree
    if (threadIdx.x < o) {
      sl[threadIdx.x] += sl[threadIdx.x + o];
      sc[threadIdx.x] += sc[threadIdx.x + o];
      sb[threadIdx.x] |= sb[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (sb[0] || sc[0] != num_labeled) *loss = __int_as_float(0x7fc00000);  // NaN: device-side error
    else *loss = num_labeled ? (float)(sl[0] / (double)num_labeled) : 0.f;
  }
}

int nll_blocks(int64_t n) {
  return (int)std::min<int64_t>(std::max<int64_t>(ceil_div(n, kNllWarps), 1), kSMs * 64);  // tens of rows per warp, many rows in flight
}

// ------------------------------------------------------------------ SGD
constexpr int kSgdMax = 32;
struct SgdBatch {
  float* master[kSgdMax];
  const float* grad[kSgdMax];
  void* shadow[kSgdMax];
  int64_t n[kSgdMax];
};

template <class TS>
__global__ void k_sgd(SgdBatch b, float lr) {
  const int t = blockIdx.y;
  const int64_t n = b.n[t];
  float* __restrict__ w = b.master[t];
  const float* __restrict__ g = b.grad[t];
  TS* __restrict__ sh = static_cast<TS*>(b.shadow[t]);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(g)) & 15) == 0 &&
                   (sh == nullptr || (reinterpret_cast<uintptr_t>(sh) & (4 * sizeof(TS) - 1)) == 0);
  int64_t done = 0;
  if (vec) {
    const int64_t n4 = n >> 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
      float4 p = reinterpret_cast<float4*>(w)[i];
      const float4 d = __ldg(reinterpret_cast<const float4*>(g) + i);
      p.x -= lr * d.x; p.y -= lr * d.y; p.z -= lr * d.z; p.w -= lr * d.w;
      reinterpret_cast<float4*>(w)[i] = p;
      if (sh) {
        if constexpr (sizeof(TS) == 4) {
          reinterpret_cast<float4*>(sh)[i] = p;
        } else {
          __nv_bfloat162 lo = __floats2bfloat162_rn(p.x, p.y), hi = __floats2bfloat162_rn(p.z, p.w);
          uint2 o;
          o.x = *reinterpret_cast<uint32_t*>(&lo);
          o.y = *reinterpret_cast<uint32_t*>(&hi);
          reinterpret_cast<uint2*>(sh)[i] = o;
        }
      }
    }
    done = 4 * n4;
  }
  for (int64_t i = done + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const float p = w[i] - lr * g[i];
    w[i] = p;
    if (sh) sh[i] = from_f<TS>(p);
  }
}

}  // namespace
}  // namespace rgnn

using namespace rgnn;

extern "C" {

rgnn_status rgnn_relu_forward(int64_t n, const float* h, void* a, int32_t dtype, void* stream) {
  return guarded([&] {
    RGNN_CHECK(n >= 0, RGNN_ERR_INVALID_ARG, "negative n");
    RGNN_CHECK(dtype == RGNN_F32 || dtype == RGNN_BF16, RGNN_ERR_INVALID_ARG, "dtype");
    if (n == 0) return;
    RGNN_CHECK(h && a, RGNN_ERR_INVALID_ARG, "NULL h or a");
    RGNN_CHECK(dtype == RGNN_F32 || (const void*)h != a, RGNN_ERR_INVALID_ARG, "a may alias h only for F32");
    const size_t align = dtype == RGNN_F32 ? 16 : 8;
    RGNN_CHECK(((reinterpret_cast<uintptr_t>(h) & 15) | (reinterpret_cast<uintptr_t>(a) & (align - 1))) == 0,
               RGNN_ERR_INVALID_ARG, "h must be 16-byte aligned, a 16-byte (F32) / 8-byte (BF16) aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (dtype == RGNN_F32)
      launch("relu_fwd", k_relu_fwd<float>, vec_grid(n / 4), dim3(256), 0, s, n, h, static_cast<float*>(a));
    else
      launch("relu_fwd", k_relu_fwd<bf16>, vec_grid(n / 4), dim3(256), 0, s, n, h, static_cast<bf16*>(a));
  });
}

rgnn_status rgnn_relu_backward(int64_t n, const float* h, const float* da, float* dh, void* stream) {
  return guarded([&] {
    RGNN_CHECK(n >= 0, RGNN_ERR_INVALID_ARG, "negative n");
    if (n == 0) return;
    RGNN_CHECK(h && da && dh, RGNN_ERR_INVALID_ARG, "NULL h, da or dh");
    RGNN_CHECK(((reinterpret_cast<uintptr_t>(h) | reinterpret_cast<uintptr_t>(da) | reinterpret_cast<uintptr_t>(dh)) &
                15) == 0,
               RGNN_ERR_INVALID_ARG, "h, da and dh must be 16-byte aligned");
    launch("relu_bwd", k_relu_bwd, vec_grid(n / 4), dim3(256), 0, static_cast<cudaStream_t>(stream), n, h, da, dh);
  });
}

rgnn_status rgnn_nll_loss_workspace(int64_t n, int32_t c, size_t* scratch_bytes) {
  return guarded([&] {
    RGNN_CHECK(scratch_bytes && n >= 0, RGNN_ERR_INVALID_ARG, "NULL scratch_bytes or negative n");
    RGNN_CHECK(c >= 1 && c <= 1024, RGNN_ERR_INVALID_ARG, "c must be in [1, 1024]");
    *scratch_bytes = (size_t)nll_blocks(n) * sizeof(NllPartial);
  });
}

rgnn_status rgnn_nll_loss(int64_t n, int32_t c, const float* logits, const int32_t* labels, int64_t num_labeled,
                          float* loss, float* dlogits, void* scratch, size_t scratch_bytes, void* stream) {
  return guarded([&] {
    RGNN_CHECK(n >= 0 && num_labeled >= 0 && num_labeled <= n, RGNN_ERR_INVALID_ARG,
               "n and num_labeled must satisfy 0 <= num_labeled <= n");
    RGNN_CHECK(c >= 1 && c <= 1024, RGNN_ERR_INVALID_ARG, "c must be in [1, 1024]");
    RGNN_CHECK(loss, RGNN_ERR_INVALID_ARG, "NULL loss");
    RGNN_CHECK(n == 0 || (logits && labels), RGNN_ERR_INVALID_ARG, "NULL logits or labels");
    const int nb = nll_blocks(n);
    RGNN_CHECK(scratch && scratch_bytes >= (size_t)nb * sizeof(NllPartial), RGNN_ERR_INVALID_ARG,
               "scratch smaller than rgnn_nll_loss_workspace");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    NllPartial* part = static_cast<NllPartial*>(scratch);
    const float inv = num_labeled ? 1.f / (float)num_labeled : 0.f;
    const bool vec = (c == 64 || c == 128 || c == 256) &&
                     ((reinterpret_cast<uintptr_t>(logits) | reinterpret_cast<uintptr_t>(dlogits)) & 15) == 0;
    if (n > 0 && vec) {
      if (c == 64) launch("nll_loss", k_nll_rows_v<64>, dim3(nb), dim3(kNllThreads), 0, s, n, logits, labels, inv, dlogits, part);
      else if (c == 128) launch("nll_loss", k_nll_rows_v<128>, dim3(nb), dim3(kNllThreads), 0, s, n, logits, labels, inv, dlogits, part);
      else launch("nll_loss", k_nll_rows_v<256>, dim3(nb), dim3(kNllThreads), 0, s, n, logits, labels, inv, dlogits, part);
    } else if (n > 0) {
      const int per = (c + 31) / 32;
      auto go = [&](auto kern) {
        launch("nll_loss", kern, dim3(nb), dim3(kNllThreads), 0, s, n, (int)c, logits, labels, inv, dlogits, part);
      };
      if (per <= 1) go(k_nll_rows<1>);
      else if (per <= 2) go(k_nll_rows<2>);
      else if (per <= 4) go(k_nll_rows<4>);
      else if (per <= 8) go(k_nll_rows<8>);
      else if (per <= 16) go(k_nll_rows<16>);
      else go(k_nll_rows<32>);
    }
    launch("nll_final", k_nll_final, dim3(1), dim3(256), 0, s, n > 0 ? nb : 0, part, (long long)num_labeled, loss);
  });
}

rgnn_status rgnn_sgd_update(int32_t count, const rgnn_sgd_tensor* tensors, float lr, int32_t shadow_dtype,
                            void* stream) {
  return guarded([&] {
    RGNN_CHECK(count >= 0 && (count == 0 || tensors), RGNN_ERR_INVALID_ARG, "NULL tensors");
    RGNN_CHECK(shadow_dtype == RGNN_F32 || shadow_dtype == RGNN_BF16, RGNN_ERR_INVALID_ARG, "shadow_dtype");
    RGNN_CHECK(std::isfinite(lr), RGNN_ERR_INVALID_ARG, "lr must be finite");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (int32_t base = 0; base < count; base += kSgdMax) {
      SgdBatch b{};
      int m = 0;
      int64_t nmax = 0;
      for (int32_t i = base; i < std::min(count, base + kSgdMax); ++i) {
        const rgnn_sgd_tensor& t = tensors[i];
        RGNN_CHECK(t.n >= 0, RGNN_ERR_INVALID_ARG, "tensor " + std::to_string(i) + ": negative n");
        if (t.n == 0) continue;
        RGNN_CHECK(t.master && t.grad, RGNN_ERR_INVALID_ARG, "tensor " + std::to_string(i) + ": NULL master or grad");
        b.master[m] = t.master;
        b.grad[m] = t.grad;
        b.shadow[m] = t.shadow;
        b.n[m] = t.n;
        nmax = std::max(nmax, t.n);
        ++m;
      }
      if (m == 0) continue;
      dim3 grid((unsigned)std::min<int64_t>(std::max<int64_t>(ceil_div(nmax / 4 + 1, 256), 1), kSMs * 4), m);
      if (shadow_dtype == RGNN_BF16) launch("sgd_update", k_sgd<bf16>, grid, dim3(256), 0, s, b, lr);
      else launch("sgd_update", k_sgd<float>, grid, dim3(256), 0, s, b, lr);
    }
  });
}

}  // extern "C"
