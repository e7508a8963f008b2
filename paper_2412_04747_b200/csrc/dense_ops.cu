// SIMT dense kernels: typed segment GEMM (fp32 path; bf16 fallback shapes),
// segmented weight gradients, per-node row reduction, and the small
// weight-weight products of linear-operator reordering (A2).
//
// The fp32 path must match the fp64 oracle to 1e-4 with TF32 off, and tcgen05
// has no fp32 kind (SURVEY.md §0 finding 8), so fp32 GEMMs run on FFMA.  At
// d = 64 these GEMMs are HBM-bound (arithmetic intensity 16 flop/B fp32), so
// the kernel is organised for coalesced gathers and stores, not for FLOPs.
#include <cstdlib>
#include <type_traits>

#include "ops.cuh"

namespace rgnn {
namespace {

constexpr int BM = 64;  // rows per tile
constexpr int KC = 16;  // k chunk

template <class T> __device__ __forceinline__ float ldf(const T* p) { return to_f(*p); }

// 256 threads: tx = tid % 16 owns columns tx + 16 j, ty = tid / 16 owns rows 4 ty .. 4 ty + 3.
template <class TA, class TB, class TY, int N>
__global__ void __launch_bounds__(256) k_gemm_simt(const Tile* __restrict__ tiles, const TA* __restrict__ A, int K,
                                                   const int32_t* __restrict__ gather, const TB* __restrict__ B,
                                                   bool transB, TY* __restrict__ Y, const float* __restrict__ dotvec,
                                                   float* __restrict__ dotout) {
  constexpr int NJ = N / 16;
  __shared__ __align__(16) float As[KC][BM + 4];
  __shared__ __align__(16) float Bs[KC][N];
  const Tile t = tiles[blockIdx.x];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int nrows = t.row1 - t.row0;
  const TB* Bw = B + (size_t)t.w * K * N;

  // loader mapping for A: row lr = tid / 4 (0..63), 4 consecutive k at (tid % 4) * 4
  const int lr = tid >> 2, lk = (tid & 3) * 4;
  int64_t arow = -1;
  if (lr < nrows) {
    int64_t r = t.row0 + lr;
    arow = gather ? (int64_t)gather[r] : r;
  }
  float acc[4][NJ];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < K; k0 += KC) {
#pragma unroll
    for (int i = 0; i < 4; ++i) As[lk + i][lr] = arow >= 0 ? ldf(A + arow * K + k0 + lk + i) : 0.f;
    for (int idx = tid; idx < KC * N; idx += 256) {
      int kk = idx / N, n = idx % N;
      Bs[kk][n] = transB ? ldf(Bw + (size_t)n * K + k0 + kk) : ldf(Bw + (size_t)(k0 + kk) * N + n);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      float4 a4 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      float a[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        float b = Bs[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][j] = fmaf(a[i], b, acc[i][j]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int lrow = ty * 4 + i;
    int64_t row = t.row0 + lrow;
    if (dotvec) {  // per-row scalar epilogue: dot of the fp32 row with a per-weight vector
      float d = 0.f;
#pragma unroll
      for (int j = 0; j < NJ; ++j) d = fmaf(acc[i][j], dotvec[(size_t)t.w * N + tx + 16 * j], d);
      d = group_sum<16>(d);
      if (tx == 0 && lrow < nrows) dotout[row] = d;
    }
    if (lrow < nrows) {
#pragma unroll
      for (int j = 0; j < NJ; ++j) Y[row * N + tx + 16 * j] = from_f<TY>(acc[i][j]);
    }
  }
}

// fp32 typed segment GEMM for N = 64 / 128 (the layer widths): N threads per 64-row tile, thread
// (tx = tid % (N/8), ty = tid / (N/8)) owns rows 8 ty .. 8 ty + 7 and columns 4 tx .. 4 tx + 3 and
// N/2 + 4 tx .. N/2 + 4 tx + 3 as packed f32x2 accumulators (8 x 8 per thread: half the shared-memory reads
// per FMA of a 8 x 4 tile -- the 64-wide kernel was bound by the shared-memory pipe at 8 x 4); A (gathered rows) and B chunks of KC = 16 k are loaded as float4 into
// registers one chunk ahead and stored transposed (A) / as is (B) into double-buffered shared memory, so
// each k step is 2 + N/64 16-byte shared loads for 32 N/64 packed FMAs.  FFMA only (no TF32).
// NTH threads per 64-row tile, each owning 8 rows x 8 columns (N = NTH): (tx = tid % 8, ty = tid / 8).
template <int N>
__global__ void __launch_bounds__(N) k_gemm_f32(const Tile* __restrict__ tiles, const float* __restrict__ A, int K,
                                                const int32_t* __restrict__ gather, const float* __restrict__ B,
                                                bool transB, float* __restrict__ Y, const float* __restrict__ dotvec,
                                                float* __restrict__ dotout) {
  constexpr int NTH = N;                // threads: 8 x 8 outputs each over the 64 x N tile
  constexpr int NB = 2;                 // 4-column groups per thread (8 columns: 4 tx and 4 (tx + 8 .. ) strided)
  constexpr int AQ = BM * KC / 4 / NTH; // float4 of an A chunk per thread
  constexpr int BQ = KC * N / 4 / NTH;  // float4 of a B chunk per thread
  constexpr int TX = N / 8;             // threads along the columns
  __shared__ __align__(16) float As[2][KC][BM + 4];
  __shared__ __align__(16) float Bs[2][KC][N];
  const Tile t = tiles[blockIdx.x];
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const int nrows = t.row1 - t.row0;
  const float* Bw = B + (size_t)t.w * K * N;
  // A loader: float4 q of the 64 x 16 chunk: row (tid + NTH q) / 4, k quad (tid + NTH q) % 4
  int64_t arow[AQ];
#pragma unroll
  for (int q = 0; q < AQ; ++q) {
    const int r = (tid + NTH * q) >> 2;
    arow[q] = r < nrows ? (gather ? (int64_t)gather[t.row0 + r] : (int64_t)(t.row0 + r)) : -1;
  }
  float4 ra[AQ], rb[BQ];
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < AQ; ++q) {
      const int kq = (tid + NTH * q) & 3;
      ra[q] = arow[q] >= 0 ? __ldg(reinterpret_cast<const float4*>(A + arow[q] * K + k0 + 4 * kq))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < BQ; ++q) {
      const int idx = tid + NTH * q;
      if (!transB) {  // row kk of the chunk, 4 consecutive n
        const int kk = idx / (N / 4), n4 = idx % (N / 4);
        rb[q] = __ldg(reinterpret_cast<const float4*>(Bw + (size_t)(k0 + kk) * N + 4 * n4));
      } else {  // column n, 4 consecutive k
        const int n = idx / (KC / 4), k4 = idx % (KC / 4);
        rb[q] = __ldg(reinterpret_cast<const float4*>(Bw + (size_t)n * K + k0 + 4 * k4));
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < AQ; ++q) {
      const int r = (tid + NTH * q) >> 2, kq = (tid + NTH * q) & 3;
      As[buf][4 * kq + 0][r] = ra[q].x;
      As[buf][4 * kq + 1][r] = ra[q].y;
      As[buf][4 * kq + 2][r] = ra[q].z;
      As[buf][4 * kq + 3][r] = ra[q].w;
    }
#pragma unroll
    for (int q = 0; q < BQ; ++q) {
      const int idx = tid + NTH * q;
      if (!transB) {
        const int kk = idx / (N / 4), n4 = idx % (N / 4);
        *reinterpret_cast<float4*>(&Bs[buf][kk][4 * n4]) = rb[q];
      } else {
        const int n = idx / (KC / 4), k4 = idx % (KC / 4);
        Bs[buf][4 * k4 + 0][n] = rb[q].x;
        Bs[buf][4 * k4 + 1][n] = rb[q].y;
        Bs[buf][4 * k4 + 2][n] = rb[q].z;
        Bs[buf][4 * k4 + 3][n] = rb[q].w;
      }
    }
  };
  float2 acc[8][2 * NB];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 2 * NB; ++j) acc[i][j] = make_float2(0.f, 0.f);
  load(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += KC) {
    if (k0 + KC < K) load(k0 + KC);
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][8 * ty]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][8 * ty + 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float2 b[2 * NB];
#pragma unroll
      for (int h = 0; h < NB; ++h) {
        const float4 b4 = *reinterpret_cast<const float4*>(&Bs[buf][kk][(N / 2) * h + 4 * tx]);
        b[2 * h] = make_float2(b4.x, b4.y);
        b[2 * h + 1] = make_float2(b4.z, b4.w);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 2 * NB; ++j) acc[i][j] = __ffma2_rn(b[j], make_float2(a[i], a[i]), acc[i][j]);
    }
    if (k0 + KC < K) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int lrow = 8 * ty + i;
    const int64_t row = t.row0 + lrow;
    if (dotvec) {  // per-row scalar epilogue
      float d = 0.f;
#pragma unroll
      for (int h = 0; h < NB; ++h) {
        const float* dv = dotvec + (size_t)t.w * N + (N / 2) * h + 4 * tx;
        d = fmaf(acc[i][2 * h].x, dv[0], d);
        d = fmaf(acc[i][2 * h].y, dv[1], d);
        d = fmaf(acc[i][2 * h + 1].x, dv[2], d);
        d = fmaf(acc[i][2 * h + 1].y, dv[3], d);
      }
      d = group_sum<TX>(d);
      if (tx == 0 && lrow < nrows) dotout[row] = d;
    }
    if (lrow < nrows) {
#pragma unroll
      for (int h = 0; h < NB; ++h)
        *reinterpret_cast<float4*>(Y + row * N + (N / 2) * h + 4 * tx) =
            make_float4(acc[i][2 * h].x, acc[i][2 * h].y, acc[i][2 * h + 1].x, acc[i][2 * h + 1].y);
    }
  }
}

template <class TA, class TB, class TY>
void gemm_dispatch(const GemmArgs& a, cudaStream_t s) {
  const TA* A = static_cast<const TA*>(a.A);
  const TB* B = static_cast<const TB*>(a.B);
  TY* Y = static_cast<TY*>(a.Y);
  dim3 g(a.ntiles), b(256);
  if constexpr (std::is_same_v<TA, float> && std::is_same_v<TB, float> && std::is_same_v<TY, float>) {
    // RGNN_F32GEMM=0 keeps the 4 x 4-per-thread kernel for every width (A/B switch)
    static const bool f32k = [] {
      const char* v = getenv("RGNN_F32GEMM");
      return !(v && v[0] == '0');
    }();
    const bool al = (reinterpret_cast<uintptr_t>(a.A) & 15) == 0 && (reinterpret_cast<uintptr_t>(a.B) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(a.Y) & 15) == 0;
    if (f32k && al && (a.N == 64 || a.N == 128)) {
      if (a.N == 64)
        launch(a.name, k_gemm_f32<64>, g, dim3(64), 0, s, a.tiles, A, a.K, a.gather, B, a.transB, Y, a.dotvec,
               a.dotout);
      else
        launch(a.name, k_gemm_f32<128>, g, dim3(128), 0, s, a.tiles, A, a.K, a.gather, B, a.transB, Y, a.dotvec,
               a.dotout);
      return;
    }
  }
#define RGNN_GEMM_CASE(NN)                                                                                  \
  case NN:                                                                                                  \
    launch(a.name, k_gemm_simt<TA, TB, TY, NN>, g, b, 0, s, a.tiles, A, a.K, a.gather, B, a.transB, Y, \
           a.dotvec, a.dotout);                                                                             \
    break;
  switch (a.N) {
    RGNN_GEMM_CASE(16)
    RGNN_GEMM_CASE(32)
    RGNN_GEMM_CASE(64)
    RGNN_GEMM_CASE(128)
    RGNN_GEMM_CASE(256)
    default:
      RGNN_FAIL(RGNN_ERR_UNSUPPORTED, "gemm: N must be one of 16,32,64,128,256");
  }
#undef RGNN_GEMM_CASE
}

// ---------------------------------------------------------------- weight gradient
// grid (tiles, ceil(K1/64), ceil(K2/64)); 256 threads own a 4x4 block of a 64x64 output tile.
template <class TA, class TB>
__global__ void __launch_bounds__(256) k_wgrad(const Tile* __restrict__ tiles, const TA* __restrict__ A, int K1,
                                               const int32_t* __restrict__ gather, const TB* __restrict__ Bm,
                                               int K2, float* __restrict__ partial) {
  __shared__ __align__(16) float As[32][64 + 4];
  __shared__ __align__(16) float Bs[32][64 + 4];
  const Tile t = tiles[blockIdx.x];
  const int k1_0 = blockIdx.y * 64, k2_0 = blockIdx.z * 64;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float acc[4][4] = {};
  const int lrow = tid >> 3, lcol = (tid & 7) * 8;  // loader: 32 rows x 64 cols, 8 per thread
  for (int r0 = t.row0; r0 < t.row1; r0 += 32) {
    int r = r0 + lrow;
    bool ok = r < t.row1;
    int64_t ar = ok ? (gather ? (int64_t)gather[r] : (int64_t)r) : 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      int k1 = k1_0 + lcol + c, k2 = k2_0 + lcol + c;
      As[lrow][lcol + c] = (ok && k1 < K1) ? to_f(A[ar * K1 + k1]) : 0.f;
      Bs[lrow][lcol + c] = (ok && k2 < K2) ? to_f(Bm[(int64_t)r * K2 + k2]) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      float4 a4 = *reinterpret_cast<const float4*>(&As[rr][ty * 4]);
      float a[4] = {a4.x, a4.y, a4.z, a4.w};
      float b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[rr][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* out = partial + (size_t)blockIdx.x * K1 * K2;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int k1 = k1_0 + ty * 4 + i;
    if (k1 >= K1) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int k2 = k2_0 + tx + 16 * j;
      if (k2 < K2) out[(size_t)k1 * K2 + k2] = acc[i][j];
    }
  }
}

// fp32 weight gradient, 64 x 64 output block per CTA (grid as k_wgrad): 128 threads, thread (tx, ty) owns
// k1 = 8 ty .. 8 ty + 7 and k2 = 4 tx .. 4 tx + 3 as packed f32x2 accumulators; rows stream in chunks of
// 16 through double-buffered shared memory (float4 loads one chunk ahead, no transposition: both
// operands are read along their row), 3 16-byte shared loads per 16 packed FMAs.  Requires K1, K2
// multiples of 64 and 16-byte aligned rows.
__global__ void __launch_bounds__(128) k_wgrad_f32(const Tile* __restrict__ tiles, const float* __restrict__ A,
                                                   int K1, const int32_t* __restrict__ gather,
                                                   const float* __restrict__ Bm, int K2, float* __restrict__ partial) {
  constexpr int RC = 16;
  __shared__ __align__(16) float As[2][RC][64 + 4];
  __shared__ __align__(16) float Bs[2][RC][64 + 4];
  const Tile t = tiles[blockIdx.x];
  const int k1_0 = blockIdx.y * 64, k2_0 = blockIdx.z * 64;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float2 acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = make_float2(0.f, 0.f);
  float4 ra[2], rb[2];
  // loader: float4 q of a 16 x 64 chunk: row (tid + 128 q) / 16, column quad (tid + 128 q) % 16
  auto load = [&](int r0) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int idx = tid + 128 * q, rr = idx >> 4, c4 = idx & 15;
      const int r = r0 + rr;
      const bool ok = r < t.row1;
      const int64_t ar = ok ? (gather ? (int64_t)gather[r] : (int64_t)r) : 0;
      ra[q] = ok ? __ldg(reinterpret_cast<const float4*>(A + ar * K1 + k1_0 + 4 * c4)) : make_float4(0.f, 0.f, 0.f, 0.f);
      rb[q] = ok ? __ldg(reinterpret_cast<const float4*>(Bm + (int64_t)r * K2 + k2_0 + 4 * c4))
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int idx = tid + 128 * q, rr = idx >> 4, c4 = idx & 15;
      *reinterpret_cast<float4*>(&As[buf][rr][4 * c4]) = ra[q];
      *reinterpret_cast<float4*>(&Bs[buf][rr][4 * c4]) = rb[q];
    }
  };
  load(t.row0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int r0 = t.row0; r0 < t.row1; r0 += RC) {
    if (r0 + RC < t.row1) load(r0 + RC);
#pragma unroll
    for (int rr = 0; rr < RC; ++rr) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][rr][8 * ty]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][rr][8 * ty + 4]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[buf][rr][4 * tx]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float2 b0 = make_float2(b4.x, b4.y), b1 = make_float2(b4.z, b4.w);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        acc[i][0] = __ffma2_rn(b0, make_float2(a[i], a[i]), acc[i][0]);
        acc[i][1] = __ffma2_rn(b1, make_float2(a[i], a[i]), acc[i][1]);
      }
    }
    if (r0 + RC < t.row1) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  float* out = partial + (size_t)blockIdx.x * K1 * K2;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int k1 = k1_0 + 8 * ty + i;
    *reinterpret_cast<float4*>(out + (size_t)k1 * K2 + k2_0 + 4 * tx) =
        make_float4(acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y);
  }
}

// out[seg_w[s]][i] = sum over the tiles of segment s of partial[tile][i].  Block = (segment, 32
// consecutive elements); its 8 warps take interleaved tiles (lane = element), then the 8 warp sums
// are added in warp order: a fixed order, so the result is deterministic.
__global__ void __launch_bounds__(256) k_seg_partial_reduce(int nseg, const int32_t* __restrict__ seg_tile_ptr,
                                                            const int32_t* __restrict__ seg_w,
                                                            const float* __restrict__ partial, int64_t width,
                                                            float* __restrict__ out) {
  __shared__ float red[8][33];
  const int sidx = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // an empty segment contributes nothing (out was zeroed); several may share a weight index
  if (seg_tile_ptr[sidx] == seg_tile_ptr[sidx + 1]) return;
  const int64_t i = blockIdx.x * (int64_t)32 + lane;
  float acc = 0.f;
  if (i < width)
    for (int t = seg_tile_ptr[sidx] + warp; t < seg_tile_ptr[sidx + 1]; t += 8) acc += partial[(size_t)t * width + i];
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && i < width) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[k][lane];
    out[(size_t)seg_w[sidx] * width + i] = s;
  }
}

// The same sum for widths that are a multiple of 128: block = (segment, 128 consecutive elements), lane l of
// every warp owns elements 4l .. 4l+3 (16-byte loads), the 8 warps take interleaved tiles (two loads in
// flight per lane), warp sums added in warp order: fixed order, deterministic.  A quarter of the blocks of
// k_seg_partial_reduce (wikikg2: 535 segments x 4096-wide weight gradients).
__global__ void __launch_bounds__(256) k_seg_partial_reduce4(int nseg, const int32_t* __restrict__ seg_tile_ptr,
                                                             const int32_t* __restrict__ seg_w,
                                                             const float* __restrict__ partial, int64_t width,
                                                             float* __restrict__ out) {
  __shared__ float4 red[8][32];
  const int sidx = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = seg_tile_ptr[sidx], t1 = seg_tile_ptr[sidx + 1];
  if (t0 == t1) return;
  const int64_t i = blockIdx.x * (int64_t)128 + 4 * lane;
  auto ld = [&](int t) { return __ldg(reinterpret_cast<const float4*>(partial + (size_t)t * width + i)); };
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
  int t = t0 + warp;
  for (; t + 8 < t1; t += 16) {
    const float4 x = ld(t), y = ld(t + 8);
    a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
    b.x += y.x; b.y += y.y; b.z += y.z; b.w += y.w;
  }
  if (t < t1) {
    const float4 x = ld(t);
    a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
  }
  red[warp][lane] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
  __syncthreads();
  if (warp == 0) {
    float4 s = red[0][lane];
#pragma unroll
    for (int k = 1; k < 8; ++k) {
      const float4 x = red[k][lane];
      s.x += x.x; s.y += x.y; s.z += x.z; s.w += x.w;
    }
    *reinterpret_cast<float4*>(out + (size_t)seg_w[sidx] * width + i) = s;
  }
}

// per tile: partial[tile][k] = sum_rows wt[row] * A[gather(row)][k] (wt == NULL: weight 1).
// Lanes move 16-byte vectors: LPR = K / V lanes per row, RG = 256 / LPR row groups striding over
// the tile's rows; the groups' sums are combined in group order in shared memory (deterministic).
template <class TA>
__global__ void __launch_bounds__(256) k_seg_wsum(const Tile* __restrict__ tiles, const float* __restrict__ wt,
                                                  const TA* __restrict__ A, int K, const int32_t* __restrict__ gather,
                                                  float* __restrict__ partial) {
  constexpr int V = Vec<TA>::N;
  __shared__ __align__(16) float red[256 * V];
  const Tile t = tiles[blockIdx.x];
  const int LPR = K / V, RG = 256 / LPR;
  const int c = threadIdx.x % LPR, rg = threadIdx.x / LPR;
  float acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = 0.f;
  if (rg < RG) {
#pragma unroll 2
    for (int r = t.row0 + rg; r < t.row1; r += RG) {
      int64_t ar = gather ? (int64_t)gather[r] : (int64_t)r;
      float x[V];
      cvt16<TA>(ldg16(A + ar * K + c * V), x);
      const float wr = wt ? wt[r] : 1.f;
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = fmaf(wr, x[k], acc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < V; ++k) red[threadIdx.x * V + k] = acc[k];
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    float sum = 0.f;
    for (int g = 0; g < RG; ++g) sum += red[(g * LPR + k / V) * V + k % V];
    partial[(size_t)blockIdx.x * K + k] = sum;
  }
}

// out[u] (+)= sum of rows Y[list[i]], i in [ptr[u], ptr[u+1]).  One group of K*sizeof(TY)/16 lanes
// per node (one 16-byte vector per lane), 4 rows loaded ahead; the loop count is the longest
// list of the warp's nodes, so the warp stays converged.  Fixed summation order (deterministic).
template <class TY, int K>
__global__ void __launch_bounds__(256) k_seg_reduce_rows(int64_t n, const int32_t* __restrict__ ptr,
                                                         const int32_t* __restrict__ list, const TY* __restrict__ Y,
                                                         float* __restrict__ out, bool accumulate, int64_t ld) {
  constexpr int V = Vec<TY>::N, LPR = K / V, EG = 32 / LPR, UN = 4;
  const int lane = threadIdx.x & 31, g = lane / LPR, c = lane % LPR;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w * EG >= n) return;
  const int64_t u = w * EG + g;
  const bool has = u < n;
  const int b = has ? ptr[u] : 0, e = has ? ptr[u + 1] : 0;
  const int span = __reduce_max_sync(0xffffffffu, e - b);
  float acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = 0.f;
  int li[UN];  // row indices of the next batch, loaded one batch ahead (the list -> row chain is dependent)
#pragma unroll
  for (int q = 0; q < UN; ++q) li[q] = b + q < e ? list[b + q] : -1;
  for (int t = 0; t < span; t += UN) {
    uint4 raw[UN];
#pragma unroll
    for (int q = 0; q < UN; ++q) {
      raw[q] = make_uint4(0, 0, 0, 0);
      if (li[q] >= 0) raw[q] = ldg16(Y + (int64_t)li[q] * ld + c * V);
    }
#pragma unroll
    for (int q = 0; q < UN; ++q) li[q] = b + t + UN + q < e ? list[b + t + UN + q] : -1;
#pragma unroll
    for (int q = 0; q < UN; ++q) {
      float x[V];
      cvt16<TY>(raw[q], x);
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] += x[k];
    }
  }
  if (!has) return;
  float* o = out + u * ld + c * V;
#pragma unroll
  for (int k = 0; k < V; k += 4) {
    float4 prev = accumulate ? *reinterpret_cast<const float4*>(o + k) : make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4*>(o + k) =
        make_float4(prev.x + acc[k], prev.y + acc[k + 1], prev.z + acc[k + 2], prev.w + acc[k + 3]);
  }
}

// ---------------------------------------------------------------- A2 weight products
// y_r = W_r b_r  (t-path of RGAT after reordering: attt = (h_d W_r) . b_r = h_d . (W_r b_r))
template <class TW>
__global__ void k_rgat_y(int d_in, int d_out, const TW* W, const TW* b, float* y) {
  int r = blockIdx.x;
  for (int k = threadIdx.x; k < d_in; k += blockDim.x) {
    float acc = 0.f;
    for (int n = 0; n < d_out; ++n)
      acc = fmaf(to_f(W[((size_t)r * d_in + k) * d_out + n]), to_f(b[(size_t)r * d_out + n]), acc);
    y[(size_t)r * d_in + k] = acc;
  }
}

// F[r*T+t] = [ (mu_r/sqrt(d)) Wk_t Watt_r | Wv_t Wmsg_r ]   (d_in x 2d)
// A2 for HGT: one folded weight per ACTIVE (r, t) combination a (pairs of relation r whose source
// has type t): F[a] = [mu_r/sqrt(d) Wk_t Watt_r | Wv_t Wmsg_r]  (d_in x 2d).
template <class TW>
__global__ void k_hgt_fold(int T, int d_in, int d, int dh, const TW* Wk, const TW* Wv, const TW* Watt, const TW* Wmsg,
                           const float* mu, const int32_t* act_rt, float* F, TW* Fdt) {
  const int a = blockIdx.x, rt = act_rt[a], r = rt / T, t = rt % T;
  const float c = mu[r] * rsqrtf((float)dh);
  for (int idx = blockIdx.y * blockDim.x + threadIdx.x; idx < d_in * 2 * d; idx += blockDim.x * gridDim.y) {
    const int k = idx / (2 * d), n2 = idx % (2 * d);
    const bool key = n2 < d;
    const int n = key ? n2 : n2 - d;
    const TW* L = key ? Wk : Wv;
    const TW* Rm = key ? Watt : Wmsg;
    float acc = 0.f;
    for (int j = 0; j < d; ++j)
      acc = fmaf(to_f(L[((size_t)t * d_in + k) * d + j]), to_f(Rm[((size_t)r * d + j) * d + n]), acc);
    if (key) acc *= c;
    F[(size_t)a * d_in * 2 * d + idx] = acc;
    if (Fdt) Fdt[(size_t)a * d_in * 2 * d + idx] = from_f<TW>(acc);
  }
}

// F1 ablation, HGT without linear-operator reordering (R off): the un-folded weights
//   Wkv[t] = [Wk_t | Wv_t]                         (d_in x 2d, node GEMM KV = X Wkv_type)
//   Bd[r]  = blockdiag(mu_r/sqrt(d) Watt_r, Wmsg_r)  (2d x 2d, pair GEMM [K~|M] = KV[src] Bd_rel)
template <class TW>
__global__ void k_hgt_nr_weights(int R, int T, int d_in, int d, int dh, const TW* Wk, const TW* Wv, const TW* Watt,
                                 const TW* Wmsg, const float* mu, TW* Wkv, TW* Bd) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t n1 = (int64_t)T * d_in * 2 * d, n2 = (int64_t)R * 4 * d * d;
  if (i < n1) {
    const int64_t tk = i / (2 * d);
    const int c = (int)(i % (2 * d));
    Wkv[i] = c < d ? Wk[tk * d + c] : Wv[tk * d + c - d];
  } else if (i < n1 + n2) {
    const int64_t j = i - n1;
    const int r = (int)(j / (4 * d * d)), rem = (int)(j % (4 * d * d)), a = rem / (2 * d), b = rem % (2 * d);
    float v = 0.f;
    if (a < d && b < d) v = mu[r] * rsqrtf((float)dh) * to_f(Watt[((size_t)r * d + a) * d + b]);
    else if (a >= d && b >= d) v = to_f(Wmsg[((size_t)r * d + a - d) * d + b - d]);
    Bd[j] = from_f<TW>(v);
  }
}

// The weight gradients of the R-off path from dBd [R][2d][2d] and dWkv [T][d_in][2d] (diagonal
// blocks and column halves; the off-diagonal blocks of Bd are not parameters).
__global__ void k_hgt_nr_split(int R, int T, int d_in, int d, int dh, const float* dBd, const float* dWkv, const float* mu,
                               float* dWk, float* dWv, float* dWatt, float* dWmsg) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t n1 = (int64_t)R * d * d, n2 = (int64_t)T * d_in * d;
  if (i < n1) {
    const int r = (int)(i / (d * d)), a = (int)(i % (d * d)) / d, b = (int)(i % d);
    if (dBd && dWatt) dWatt[i] = mu[r] * rsqrtf((float)dh) * dBd[((size_t)r * 2 * d + a) * 2 * d + b];
    if (dBd && dWmsg) dWmsg[i] = dBd[((size_t)r * 2 * d + d + a) * 2 * d + d + b];
  } else if (i < n1 + n2) {
    const int64_t j = i - n1, tk = j / d;
    const int c = (int)(j % d);
    if (dWkv && dWk) dWk[j] = dWkv[tk * 2 * d + c];
    if (dWkv && dWv) dWv[j] = dWkv[tk * 2 * d + d + c];
  }
}

// F1 ablation, RGAT without reordering: the destination logit term per (rel, dst) pair j
// (a run of the dst-CSR) expanded to its CSR entries, and dz summed back per run (warp per run,
// fixed-order shuffle reduction).
__global__ void k_dpair_expand(int64_t UD, const int32_t* __restrict__ beg, const int32_t* __restrict__ cnt,
                               const float* __restrict__ tdp, float* __restrict__ te) {
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (j >= UD) return;
  const int lane = threadIdx.x & 31;
  const float v = tdp[j];
  for (int q = lane; q < cnt[j]; q += 32) te[beg[j] + q] = v;
}

__global__ void k_dpair_sum(int64_t UD, const int32_t* __restrict__ beg, const int32_t* __restrict__ cnt,
                            const float* __restrict__ dz, float* __restrict__ dt) {
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (j >= UD) return;
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (int q = lane; q < cnt[j]; q += 32) acc += dz[beg[j] + q];
  acc = group_sum<32>(acc);
  if (lane == 0) dt[j] = acc;
}

// dPt[row][:] = dt[row] * b[w][:] over the rows of each tile (w = relation)
template <class TW>
__global__ void k_dpair_outer(const Tile* __restrict__ tiles, const float* __restrict__ dt, const TW* __restrict__ b,
                              int D, TW* __restrict__ dPt) {
  const Tile t = tiles[blockIdx.x];
  for (int64_t idx = threadIdx.x; idx < (int64_t)(t.row1 - t.row0) * D; idx += blockDim.x) {
    const int64_t row = t.row0 + idx / D;
    const int k = (int)(idx % D);
    dPt[row * D + k] = from_f<TW>(dt[row] * to_f(b[(size_t)t.w * D + k]));
  }
}

// F2, HGT layer tail: GELU (exact, erf form) of the aggregation, its derivative, and the residual.
template <class TO>
__global__ void k_gelu_fwd(int64_t n, const float* __restrict__ h, TO* __restrict__ gh) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float x = h[i];
    gh[i] = from_f<TO>(0.5f * x * (1.f + erff(x * 0.70710678118654752f)));
  }
}
__global__ void k_gelu_bwd(int64_t n, const float* __restrict__ h, float* __restrict__ dg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float x = h[i];
    const float cdf = 0.5f * (1.f + erff(x * 0.70710678118654752f));
    const float pdf = 0.39894228040143268f * __expf(-0.5f * x * x);
    dg[i] *= cdf + x * pdf;
  }
}
template <class TX>
__global__ void k_add_dt(int64_t n, const TX* __restrict__ x, float* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += to_f(x[i]);
}

// y += x (fp32, 16-byte vectors when aligned)
__global__ void k_add_f32(int64_t n, const float* __restrict__ x, float* __restrict__ y) {
  const int64_t n4 = n >> 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = __ldg(reinterpret_cast<const float4*>(x) + i);
    float4 b = reinterpret_cast<float4*>(y)[i];
    b.x += a.x; b.y += a.y; b.z += a.z; b.w += a.w;
    reinterpret_cast<float4*>(y)[i] = b;
  }
  const int64_t t = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) y[t] += x[t];
}

// Unfold dF[a] (d_in x 2d, one per active (r, t)) into the four HGT weight gradients; every
// output is a fixed-order sum over the active combinations (deterministic).
//   dWk[t][k][j] = sum_{a=(r,t)} c_r sum_n dF[a][k][n] Watt[r][j][n],   dWv likewise with dF[a][k][d+n], Wmsg
// Step 1, block (a, k), 2d threads: P[a][k][j] = c_r dF[a][k][0:d] . Watt_r[j][:] (j < d) and
// P[a][k][d+j] = dF[a][k][d:2d] . Wmsg_r[j][:] (the dF row staged in shared memory, weight rows
// read as 16-byte vectors).  Step 2, block (t, k): the sum of P over the combinations of type t.
template <class TW>
__global__ void k_hgt_unfold_node_p(int T, int d_in, int d, int dh, const TW* Watt, const TW* Wmsg, const float* mu,
                                    const int32_t* act_rt, const float* dF, float* P) {
  extern __shared__ float fsm[];  // [2d]
  constexpr int V = Vec<TW>::N;
  const int a = blockIdx.x, k = blockIdx.y, tid = threadIdx.x, r = act_rt[a] / T;
  const size_t row = ((size_t)a * d_in + k) * 2 * d;
  fsm[tid] = dF[row + tid];
  __syncthreads();
  const bool key = tid < d;
  const int j = key ? tid : tid - d;
  const TW* W = (key ? Watt : Wmsg) + ((size_t)r * d + j) * d;
  const float* f = fsm + (key ? 0 : d);
  float acc = 0.f;
  for (int n0 = 0; n0 < d; n0 += V) {
    float w[V];
    load16(W + n0, w);
#pragma unroll
    for (int i = 0; i < V; ++i) acc = fmaf(f[n0 + i], w[i], acc);
  }
  P[row + tid] = key ? mu[r] * rsqrtf((float)dh) * acc : acc;
}

__global__ void k_hgt_unfold_node_sum(int d_in, int d, const int32_t* t_act_ptr, const int32_t* t_act, const float* P,
                                      float* dWk, float* dWv) {
  const int t = blockIdx.x, k = blockIdx.y, tid = threadIdx.x;
  float acc = 0.f;
  for (int i = t_act_ptr[t]; i < t_act_ptr[t + 1]; ++i) acc += P[((size_t)t_act[i] * d_in + k) * 2 * d + tid];
  float* out = tid < d ? dWk : dWv;
  if (out) out[((size_t)t * d_in + k) * d + (tid < d ? tid : tid - d)] = acc;
}

//   dWatt[r][j][n] = c_r sum_{a=(r,t)} sum_k Wk[t][k][j] dF[a][k][n],  dWmsg[r][j][n] = sum_a sum_k Wv[t][k][j] dF[a][k][d+n]
// Block (r, j), 2d threads: thread n < d -> dWatt[r][j][n], thread d + n -> dWmsg[r][j][n] (coalesced dF rows).
template <class TW>
__global__ void k_hgt_unfold_rel(int T, int d_in, int d, int dh, const TW* Wk, const TW* Wv, const float* mu,
                                 const int32_t* act_rt, const int32_t* r_act_ptr, const float* dF, float* dWatt,
                                 float* dWmsg) {
  const int r = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  const bool key = tid < d;
  float acc = 0.f;
  for (int a = r_act_ptr[r]; a < r_act_ptr[r + 1]; ++a) {
    const int t = act_rt[a] % T;
    const TW* W = (key ? Wk : Wv) + (size_t)t * d_in * d + j;
    const float* f = dF + (size_t)a * d_in * 2 * d + tid;
    for (int k = 0; k < d_in; ++k) acc = fmaf(to_f(W[(size_t)k * d]), f[(size_t)k * 2 * d], acc);
  }
  if (key) {
    if (dWatt) dWatt[((size_t)r * d + j) * d + tid] = mu[r] * rsqrtf((float)dh) * acc;
  } else if (dWmsg) {
    dWmsg[((size_t)r * d + j) * d + tid - d] = acc;
  }
}

// dW_r += Bsum_r^T b_r (outer product, destination side of the t-path); db_r = Bsum_r W_r
template <class TW>
__global__ void k_rgat_tpath_grads(int R, int d_in, int d_out, const TW* W, const TW* b, const float* Bsum, float* dW,
                                   float* db) {
  int r = blockIdx.x;
  if (dW)
    for (int idx = threadIdx.x; idx < d_in * d_out; idx += blockDim.x) {
      int k = idx / d_out, n = idx % d_out;
      dW[(size_t)r * d_in * d_out + idx] += Bsum[(size_t)r * d_in + k] * to_f(b[(size_t)r * d_out + n]);
    }
  if (db)
    for (int n = threadIdx.x; n < d_out; n += blockDim.x) {
      float acc = 0.f;
      for (int k = 0; k < d_in; ++k)
        acc = fmaf(Bsum[(size_t)r * d_in + k], to_f(W[((size_t)r * d_in + k) * d_out + n]), acc);
      db[(size_t)r * d_out + n] = acc;
    }
}

template <class TI>
__global__ void k_to_f32(int64_t n, const TI* in, float* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = to_f(in[i]);
}
template <class TO>
__global__ void k_from_f32(int64_t n, const float* in, TO* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = from_f<TO>(in[i]);
}

// fp32 -> bf16, 8 elements per thread (two 16-byte loads, one 16-byte store); scalar tail
__global__ void k_from_f32_bf16(int64_t n, const float* __restrict__ in, bf16* __restrict__ out) {
  const int64_t n8 = n >> 3;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(in) + 2 * i);
    const float4 b = __ldg(reinterpret_cast<const float4*>(in) + 2 * i + 1);
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    store16(out + 8 * i, v);
  }
  const int64_t t = 8 * n8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) out[t] = __float2bfloat16_rn(in[t]);
}

}  // namespace

void gemm_simt(const GemmArgs& a, cudaStream_t s) {
  RGNN_CHECK(a.K % KC == 0 && a.K > 0, RGNN_ERR_UNSUPPORTED, "gemm: K must be a positive multiple of 16");
  if (a.a_dtype == F32 && a.b_dtype == F32 && a.y_dtype == F32) gemm_dispatch<float, float, float>(a, s);
  else if (a.a_dtype == BF16 && a.b_dtype == BF16 && a.y_dtype == BF16) gemm_dispatch<bf16, bf16, bf16>(a, s);
  else if (a.a_dtype == BF16 && a.b_dtype == BF16 && a.y_dtype == F32) gemm_dispatch<bf16, bf16, float>(a, s);
  else if (a.a_dtype == F32 && a.b_dtype == BF16 && a.y_dtype == F32) gemm_dispatch<float, bf16, float>(a, s);
  else RGNN_FAIL(RGNN_ERR_UNSUPPORTED, "gemm: unsupported dtype combination");
}

void seg_partial_reduce(const Plan& p, const float* partial, int64_t width, float* out, cudaStream_t s) {
  const bool al = (reinterpret_cast<uintptr_t>(partial) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  // few long segments (mag: a handful of relation / type segments x ~400 tiles) keep the 32-element blocks:
  // 4x the blocks to spread the long tile loops over the SMs (measured: the 128-element blocks cost mag HGT
  // 0.033 -> 0.050 ms); many short ones (wikikg2: 535 x ~13 tiles, AM: 130 x ~14) take the float4 blocks
  if (width % 128 == 0 && al && p.count <= 64 * (int64_t)p.nseg)
    launch("wgrad_reduce", k_seg_partial_reduce4, dim3((unsigned)(width / 128), p.nseg), dim3(256), 0, s, p.nseg,
           p.seg_tile_ptr, p.seg_w, partial, width, out);
  else
    launch("wgrad_reduce", k_seg_partial_reduce, dim3(ceil_div(width, 32), p.nseg), dim3(256), 0, s, p.nseg,
           p.seg_tile_ptr, p.seg_w, partial, width, out);
}

void wgrad(const WgradArgs& a, cudaStream_t s) {
  const Plan& p = *a.plan;
  RGNN_CUDA(cudaMemsetAsync(a.out, 0, (size_t)a.num_w * a.K1 * a.K2 * sizeof(float), s));
  if (p.count == 0) return;
  dim3 g(p.count, ceil_div(a.K1, 64), ceil_div(a.K2, 64));
  if (a.allow_tc && wgrad_tc_supported(a)) {
    wgrad_tc(a, s);
    seg_partial_reduce(p, a.partial, (int64_t)a.K1 * a.K2, a.out, s);
    return;
  }
  auto go = [&](auto* A, auto* B) {
    using TA = std::remove_const_t<std::remove_pointer_t<decltype(A)>>;
    using TB = std::remove_const_t<std::remove_pointer_t<decltype(B)>>;
    launch(a.name, k_wgrad<TA, TB>, g, dim3(256), 0, s, p.tiles, A, a.K1, a.gather, B, a.K2, a.partial);
  };
  const bool a32 = a.a_dtype == F32, b32 = a.b_dtype == F32;
  static const bool f32k = [] {  // RGNN_F32GEMM=0: the 4 x 4-per-thread weight-gradient kernel (A/B switch)
    const char* v = getenv("RGNN_F32GEMM");
    return !(v && v[0] == '0');
  }();
  const bool al = (reinterpret_cast<uintptr_t>(a.A) & 15) == 0 && (reinterpret_cast<uintptr_t>(a.Bm) & 15) == 0;
  if (a32 && b32 && f32k && al && a.K1 % 64 == 0 && a.K2 % 64 == 0)
    launch(a.name, k_wgrad_f32, g, dim3(128), 0, s, p.tiles, static_cast<const float*>(a.A), a.K1, a.gather,
           static_cast<const float*>(a.Bm), a.K2, a.partial);
  else if (a32 && b32) go(static_cast<const float*>(a.A), static_cast<const float*>(a.Bm));
  else if (a32) go(static_cast<const float*>(a.A), static_cast<const bf16*>(a.Bm));
  else if (b32) go(static_cast<const bf16*>(a.A), static_cast<const float*>(a.Bm));
  else go(static_cast<const bf16*>(a.A), static_cast<const bf16*>(a.Bm));
  seg_partial_reduce(p, a.partial, (int64_t)a.K1 * a.K2, a.out, s);
}

void seg_wsum(const Plan* plan, const float* wt, const void* A, int a_dtype, int K, const int32_t* gather, float* out,
              int num_w, float* partial, cudaStream_t s) {
  const Plan& p = *plan;
  RGNN_CHECK(K % (a_dtype == F32 ? 4 : 8) == 0 && K <= (a_dtype == F32 ? 1024 : 2048), RGNN_ERR_UNSUPPORTED,
             "seg_wsum: K must be a multiple of the 16-byte vector width");
  RGNN_CUDA(cudaMemsetAsync(out, 0, (size_t)num_w * K * sizeof(float), s));
  if (p.count == 0) return;
  if (a_dtype == F32)
    launch("seg_wsum", k_seg_wsum<float>, dim3(p.count), dim3(256), 0, s, p.tiles, wt,
           static_cast<const float*>(A), K, gather, partial);
  else
    launch("seg_wsum", k_seg_wsum<bf16>, dim3(p.count), dim3(256), 0, s, p.tiles, wt,
           static_cast<const bf16*>(A), K, gather, partial);
  seg_partial_reduce(p, partial, (int64_t)K, out, s);
}

void seg_reduce_rows(int64_t n, const int32_t* ptr, const int32_t* list, const void* Y, int y_dtype, int K, float* out,
                     bool accumulate, cudaStream_t s) {
  auto go = [&](auto* ty, auto kc) {
    using TY = std::remove_pointer_t<decltype(ty)>;
    constexpr int KK = decltype(kc)::value;
    constexpr int LPR = KK / Vec<TY>::N;
    if constexpr (LPR >= 1 && LPR <= 32) {
      launch("seg_reduce_rows", k_seg_reduce_rows<TY, KK>, dim3(ceil_div(ceil_div(n, 32 / LPR) * 32, 256)),
             dim3(256), 0, s, n, ptr, list, static_cast<const TY*>(Y), out, accumulate, (int64_t)KK);
    } else {  // fp32 rows of 256: two column halves of 128 (row stride 256)
      constexpr int KH = KK / 2;
      for (int h = 0; h < 2; ++h)
        launch("seg_reduce_rows", k_seg_reduce_rows<TY, KH>, dim3(ceil_div(ceil_div(n, 32 / (KH / Vec<TY>::N)) * 32, 256)),
               dim3(256), 0, s, n, ptr, list, static_cast<const TY*>(Y) + h * KH, out + h * KH, accumulate,
               (int64_t)KK);
    }
  };
  auto by_k = [&](auto* ty) {
    switch (K) {
      case 16: go(ty, std::integral_constant<int, 16>()); break;
      case 32: go(ty, std::integral_constant<int, 32>()); break;
      case 64: go(ty, std::integral_constant<int, 64>()); break;
      case 128: go(ty, std::integral_constant<int, 128>()); break;
      case 256: go(ty, std::integral_constant<int, 256>()); break;
      default: RGNN_FAIL(RGNN_ERR_UNSUPPORTED, "seg_reduce_rows: width");
    }
  };
  if (y_dtype == F32) by_k((float*)nullptr);
  else by_k((bf16*)nullptr);
}

void rgat_tpath_vectors(int R, int d_in, int d_out, const void* W, const void* b, int dtype, float* y,
                        cudaStream_t s) {
  if (dtype == F32)
    launch("rgat_y", k_rgat_y<float>, dim3(R), dim3(std::min(d_in, 256)), 0, s, d_in, d_out,
           static_cast<const float*>(W), static_cast<const float*>(b), y);
  else
    launch("rgat_y", k_rgat_y<bf16>, dim3(R), dim3(std::min(d_in, 256)), 0, s, d_in, d_out,
           static_cast<const bf16*>(W), static_cast<const bf16*>(b), y);
}

void hgt_fold(const rgnn_graph_s* g, int d_in, int d, int dh, const void* Wk, const void* Wv, const void* Watt,
              const void* Wmsg, const float* mu, int dtype, float* F, void* Fdt, cudaStream_t s) {
  const dim3 grid(g->n_act, ceil_div(d_in * 2 * d, 256));
  if (dtype == F32)
    launch("hgt_fold", k_hgt_fold<float>, grid, dim3(256), 0, s, g->T, d_in, d, dh, static_cast<const float*>(Wk),
           static_cast<const float*>(Wv), static_cast<const float*>(Watt), static_cast<const float*>(Wmsg), mu,
           g->act_rt, F, static_cast<float*>(nullptr));
  else
    launch("hgt_fold", k_hgt_fold<bf16>, grid, dim3(256), 0, s, g->T, d_in, d, dh, static_cast<const bf16*>(Wk),
           static_cast<const bf16*>(Wv), static_cast<const bf16*>(Watt), static_cast<const bf16*>(Wmsg), mu,
           g->act_rt, F, static_cast<bf16*>(Fdt));
}

void hgt_unfold(const rgnn_graph_s* g, int d_in, int d, int dh, const void* Wk, const void* Wv, const void* Watt,
                const void* Wmsg, const float* mu, int dtype, const float* dF, float* P, float* dWk, float* dWv,
                float* dWatt, float* dWmsg, cudaStream_t s) {
  const int R = g->R, T = g->T;
  const size_t sm = 2 * d * sizeof(float);
  auto go = [&](auto* tw) {
    using TW = std::remove_pointer_t<decltype(tw)>;
    if ((dWk || dWv) && g->n_act > 0) {
      launch("hgt_unfold_node", k_hgt_unfold_node_p<TW>, dim3(g->n_act, d_in), dim3(2 * d), sm, s, T, d_in, d, dh,
             static_cast<const TW*>(Watt), static_cast<const TW*>(Wmsg), mu, g->act_rt, dF, P);
    }
    if (dWk || dWv)
      launch("hgt_unfold_node", k_hgt_unfold_node_sum, dim3(T, d_in), dim3(2 * d), 0, s, d_in, d, g->t_act_ptr,
             g->t_act, P, dWk, dWv);
    if (dWatt || dWmsg)
      launch("hgt_unfold_rel", k_hgt_unfold_rel<TW>, dim3(R, d), dim3(2 * d), 0, s, T, d_in, d, dh,
             static_cast<const TW*>(Wk), static_cast<const TW*>(Wv), mu, g->act_rt, g->r_act_ptr, dF, dWatt, dWmsg);
  };
  if (dtype == F32) go(static_cast<float*>(nullptr));
  else go(static_cast<bf16*>(nullptr));
}

void rgat_tpath_grads(int R, int d_in, int d_out, const void* W, const void* b, int dtype, const float* Bsum,
                      float* dW, float* db, cudaStream_t s) {
  if (dtype == F32)
    launch("rgat_tpath_grads", k_rgat_tpath_grads<float>, dim3(R), dim3(256), 0, s, R, d_in, d_out,
           static_cast<const float*>(W), static_cast<const float*>(b), Bsum, dW, db);
  else
    launch("rgat_tpath_grads", k_rgat_tpath_grads<bf16>, dim3(R), dim3(256), 0, s, R, d_in, d_out,
           static_cast<const bf16*>(W), static_cast<const bf16*>(b), Bsum, dW, db);
}

void hgt_nr_weights(int R, int T, int d_in, int d, int dh, const void* Wk, const void* Wv, const void* Watt, const void* Wmsg,
                    const float* mu, int dtype, void* Wkv, void* Bd, cudaStream_t s) {
  const int64_t n = (int64_t)T * d_in * 2 * d + (int64_t)R * 4 * d * d;
  if (dtype == F32)
    launch("hgt_nr_weights", k_hgt_nr_weights<float>, dim3(ceil_div(n, 256)), dim3(256), 0, s, R, T, d_in, d, dh,
           static_cast<const float*>(Wk), static_cast<const float*>(Wv), static_cast<const float*>(Watt),
           static_cast<const float*>(Wmsg), mu, static_cast<float*>(Wkv), static_cast<float*>(Bd));
  else
    launch("hgt_nr_weights", k_hgt_nr_weights<bf16>, dim3(ceil_div(n, 256)), dim3(256), 0, s, R, T, d_in, d, dh,
           static_cast<const bf16*>(Wk), static_cast<const bf16*>(Wv), static_cast<const bf16*>(Watt),
           static_cast<const bf16*>(Wmsg), mu, static_cast<bf16*>(Wkv), static_cast<bf16*>(Bd));
}

void hgt_nr_split(int R, int T, int d_in, int d, int dh, const float* dBd, const float* dWkv, const float* mu, float* dWk,
                  float* dWv, float* dWatt, float* dWmsg, cudaStream_t s) {
  const int64_t n = (int64_t)R * d * d + (int64_t)T * d_in * d;
  launch("hgt_nr_split", k_hgt_nr_split, dim3(ceil_div(n, 256)), dim3(256), 0, s, R, T, d_in, d, dh, dBd, dWkv, mu, dWk,
         dWv, dWatt, dWmsg);
}

void dpair_expand(const rgnn_graph_s* g, const float* tdp, float* te, cudaStream_t s) {
  launch("dpair_expand", k_dpair_expand, dim3(ceil_div(g->UD * 32, 256)), dim3(256), 0, s, g->UD,
         (const int32_t*)g->dpair_csr_beg, (const int32_t*)g->dpair_cnt, tdp, te);
}

// dt[j] = sum of w[i].y over the CSR entries of (rel, dst) run j.  A warp owns 32 consecutive runs: each
// lane sums its run when it has at most 32 entries; the warp's runs of 33 .. SPLIT_THRESH entries are then
// summed by the whole warp, one after the other, in lane order with a fixed shuffle tree.  Longer runs (the
// skewed in-degrees of a mag hub: ~10^5 in-edges per relation) are cut into SPLIT_CHUNK-entry chunks
// (graph dpair_chunks), one warp each (k_dpair_chunk_sum), and their partials added in chunk order
// (k_dpair_merge).  Deterministic throughout.
__global__ void k_dpair_sum_w(int64_t UD, const int32_t* __restrict__ beg, const int32_t* __restrict__ cnt,
                              const float2* __restrict__ w, float* __restrict__ dt) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int b = j < UD ? beg[j] : 0, n = j < UD ? cnt[j] : 0;
  const bool longrun = n > 32 && n <= SPLIT_THRESH;
  if (j < UD && n <= 32) {
    float acc = 0.f;
    for (int i = b; i < b + n; ++i) acc += w[i].y;
    dt[j] = acc;
  }
  unsigned todo = __ballot_sync(0xffffffffu, longrun);
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const int bb = __shfl_sync(0xffffffffu, b, src), nn = __shfl_sync(0xffffffffu, n, src);
    float acc = 0.f;
    for (int i = lane; i < nn; i += 32) acc += w[bb + i].y;
    acc = group_sum<32>(acc);
    if (lane == src) dt[j] = acc;
  }
}

__global__ void k_dpair_chunk_sum(int64_t n, const int4* __restrict__ chunks, const float2* __restrict__ w,
                                  float* __restrict__ part) {
  const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (k >= n) return;
  const int lane = threadIdx.x & 31;
  const int4 c = chunks[k];
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;  // four independent loads in flight per lane
  int i = c.y + lane;
  for (; i + 96 < c.z; i += 128) {
    a0 += w[i].y;
    a1 += w[i + 32].y;
    a2 += w[i + 64].y;
    a3 += w[i + 96].y;
  }
  for (; i < c.z; i += 32) a0 += w[i].y;
  float acc = group_sum<32>((a0 + a1) + (a2 + a3));
  if (lane == 0) part[c.w] = acc;
}

__global__ void k_dpair_merge(int64_t n, const int4* __restrict__ splits, const float* __restrict__ part,
                              float* __restrict__ dt) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int4 sp = splits[k];
  float acc = 0.f;
  for (int q = 0; q < sp.z; ++q) acc += part[sp.y + q];
  dt[sp.x] = acc;
}

void dpair_sum_w(const rgnn_graph_s* g, const float2* w, float* dt, float* part, cudaStream_t s) {
  launch("dpair_sum", k_dpair_sum_w, dim3(ceil_div(g->UD, 256)), dim3(256), 0, s, g->UD,
         (const int32_t*)g->dpair_csr_beg, (const int32_t*)g->dpair_cnt, w, dt);
  launch("dpair_sum/chunks", k_dpair_chunk_sum, dim3(ceil_div(g->n_dpair_chunks * 32, 256)), dim3(256), 0, s,
         g->n_dpair_chunks, (const int4*)g->dpair_chunks, w, part);
  launch("dpair_sum/merge", k_dpair_merge, dim3(ceil_div(g->n_dpair_splits, 256)), dim3(256), 0, s,
         g->n_dpair_splits, (const int4*)g->dpair_splits, (const float*)part, dt);
}

void dpair_sum(const rgnn_graph_s* g, const float* dz, float* dt, cudaStream_t s) {
  launch("dpair_sum", k_dpair_sum, dim3(ceil_div(g->UD * 32, 256)), dim3(256), 0, s, g->UD,
         (const int32_t*)g->dpair_csr_beg, (const int32_t*)g->dpair_cnt, dz, dt);
}

void dpair_outer(const Plan& p, const float* dt, const void* b, int dtype, int D, void* dPt, cudaStream_t s) {
  if (dtype == F32)
    launch("dpair_outer", k_dpair_outer<float>, dim3(p.count), dim3(256), 0, s, p.tiles, dt,
           static_cast<const float*>(b), D, static_cast<float*>(dPt));
  else
    launch("dpair_outer", k_dpair_outer<bf16>, dim3(p.count), dim3(256), 0, s, p.tiles, dt,
           static_cast<const bf16*>(b), D, static_cast<bf16*>(dPt));
}

namespace {
inline dim3 ew_grid(int64_t n) { return dim3((unsigned)std::min<int64_t>(std::max<int64_t>(ceil_div(n, 256), 1), 148 * 16)); }
}  // namespace

void gelu_fwd(int64_t n, const float* h, void* gh, int dtype, cudaStream_t s) {
  if (dtype == F32) launch("tail_gelu", k_gelu_fwd<float>, ew_grid(n), dim3(256), 0, s, n, h, static_cast<float*>(gh));
  else launch("tail_gelu", k_gelu_fwd<bf16>, ew_grid(n), dim3(256), 0, s, n, h, static_cast<bf16*>(gh));
}

void gelu_bwd(int64_t n, const float* h, float* dg, cudaStream_t s) {
  launch("tail_gelu_bwd", k_gelu_bwd, ew_grid(n), dim3(256), 0, s, n, h, dg);
}

void add_dt(int64_t n, const void* x, int dtype, float* y, cudaStream_t s) {
  if (dtype == F32) launch("tail_residual", k_add_dt<float>, ew_grid(n), dim3(256), 0, s, n, static_cast<const float*>(x), y);
  else launch("tail_residual", k_add_dt<bf16>, ew_grid(n), dim3(256), 0, s, n, static_cast<const bf16*>(x), y);
}

void add_f32(int64_t n, const float* x, float* y, cudaStream_t s) {
  RGNN_CHECK(((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0, RGNN_ERR_INVALID_ARG,
             "add_f32: unaligned buffers");
  launch("add_rows", k_add_f32, dim3(std::min<int64_t>(std::max<int64_t>(ceil_div(n / 4, 256), 1), 148 * 16)),
         dim3(256), 0, s, n, x, y);
}

void convert_f32(int64_t n, const void* in, int dtype, float* out, cudaStream_t s) {
  if (dtype == F32)
    RGNN_CUDA(cudaMemcpyAsync(out, in, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
  else
    launch("to_f32", k_to_f32<bf16>, dim3(ceil_div(n, 256)), dim3(256), 0, s, n, static_cast<const bf16*>(in), out);
}

void convert_dt(int64_t n, const float* in, void* out, int dtype, cudaStream_t s) {
  if (dtype == F32)
    RGNN_CUDA(cudaMemcpyAsync(out, in, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
  else if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15)
    launch("from_f32", k_from_f32<bf16>, dim3(ceil_div(n, 256)), dim3(256), 0, s, n, in, static_cast<bf16*>(out));
  else
    launch("from_f32", k_from_f32_bf16, dim3(std::min<int64_t>(std::max<int64_t>(ceil_div(n / 8, 256), 1), 148 * 16)),
           dim3(256), 0, s, n, in, static_cast<bf16*>(out));
}

}  // namespace rgnn
