// A1 on the 5th-generation tensor cores: typed segment GEMM  Y[row] = X[gather(row)] x W_w
// for the bf16 path (GEMM template Y[S] = X[G] x W[T], §3.3.3; compact rows P:764-776).
//
// One CTA per 128-row tile of one segment (tiles never cross a weight segment):
//   * 128 threads gather the tile's A rows (X[pair_src[row]], bf16, K-major) and the
//     segment's B = W_w^T (pre-transposed to K-major by k_transpose_kmajor) into shared
//     memory with cp.async, already in the 128-byte-swizzled canonical UMMA layout
//     (8-row x 128 B atoms, 16-byte chunk c of row r stored at chunk c ^ (r % 8));
//   * one elected thread issues tcgen05.mma.cta_group::1.kind::f16 (M=128, N=n_out,
//     K=16 per instruction) accumulating fp32 in TMEM, then tcgen05.commit -> mbarrier;
//   * the 4 warps read their 32 TMEM lanes (= tile rows) with tcgen05.ld.32x32b and
//     run the fused epilogue: optional per-row dot with a per-weight vector (RGAT
//     s_p = P_p . a_r, "per-row scalar"), conversion, and the row store.
// Several CTAs per SM (TMEM 512 columns / n_out columns each) overlap one tile's
// gather with another's MMA and epilogue.  At d = 64 the GEMM is HBM-bound
// (32 flop/B vs a ~213 flop/B ridge), so the design goal is bytes in flight.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "ops.cuh"
#include "tc_ptx.cuh"

namespace rgnn {
namespace {
using namespace tc;

// Persistent warp-specialized GEMM (k_gemm_ws) for contiguous A rows; the gathered GEMM
// (A = X[pair_src]) stays on k_gemm_tc, whose ~9 resident CTAs per SM keep more independent
// row gathers in flight (measured on B200: ws 0.30 vs 0.24 ms for mag pairs_fwd, while ws wins
// 5-17% on the ungathered GEMMs).  RGNN_GEMM_WS=0: never ws; RGNN_GEMM_WS=2: ws for all.
int ws_mode() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("RGNN_GEMM_WS");
    on = (e && e[0] == '0') ? 0 : (e && e[0] == '2') ? 2 : 1;
  }
  return on;
}

// K-major bf16 copy of the weights: Wt[w][n][k] = W[w][k][n] (or of W^T when transB: Wt[w][n][k] = W[w][n][k]).
template <class TW>
__global__ void k_transpose_kmajor(int64_t nw, int K, int N, const TW* __restrict__ W, bool transB,
                                   bf16* __restrict__ Wt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t per = (int64_t)K * N;
  if (i >= nw * per) return;
  int64_t w = i / per, r = i % per;
  int n = r / K, k = r % K;
  float v = transB ? to_f(W[w * per + (int64_t)n * K + k]) : to_f(W[w * per + (int64_t)k * N + n]);
  Wt[i] = __float2bfloat16_rn(v);
}

// N = n_out (multiple of 16, <= 256); KB = K / 64 (1..4).
template <class TY, int N, int KB>
__global__ void __launch_bounds__(128) k_gemm_tc(const Tile* __restrict__ tiles, const bf16* __restrict__ A,
                                                 const int32_t* __restrict__ gather, const bf16* __restrict__ Bt,
                                                 TY* __restrict__ Y, const float* __restrict__ dotvec,
                                                 float* __restrict__ dotout, const int32_t* __restrict__ red_ptr,
                                                 const int32_t* __restrict__ red_list,
                                                 const void* __restrict__ red_rows, int red_bf16) {
  constexpr int K = KB * 64;
  constexpr int NCOLS = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  constexpr uint32_t A_BYTES = 128 * 128;  // per K block
  constexpr uint32_t B_BYTES = N * 128;    // per K block
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + KB * A_BYTES;
  constexpr uint32_t OPS = KB * (A_BYTES + B_BYTES) > 128u * N * sizeof(TY) ? KB * (A_BYTES + B_BYTES)
                                                                            : 128u * N * sizeof(TY);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OPS);  // after operands / epilogue staging
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Tile t = tiles[blockIdx.x];
  const int nrows = t.row1 - t.row0;

  if (warp == 0) tmem_alloc<NCOLS>(tslot);
  if (tid == 32) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }

  // ---- gather A rows and B rows into swizzled smem (8 lanes per 128-byte row: coalesced)
  const uint32_t sA_u = smem_u32(sA), sB_u = smem_u32(sB);
  // the 8 gathered row indices of this thread, loaded together before any copy is issued
  int64_t src_row[8];
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int r = (it * 128 + tid) >> 3;
    const int rr = r < nrows ? r : nrows - 1;
    src_row[it] = gather ? (int64_t)__ldg(gather + t.row0 + rr) : (int64_t)(t.row0 + rr);
  }
#pragma unroll
  for (int kb = 0; kb < KB; ++kb) {
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      int idx = it * 128 + tid;
      int r = idx >> 3, c = idx & 7;
      cp_async16(sA_u + kb * A_BYTES + r * 128 + ((c ^ (r & 7)) << 4), A + src_row[it] * K + kb * 64 + c * 8);
    }
    const bf16* Bw = Bt + (size_t)t.w * N * K;
    for (int idx = tid; idx < N * 8; idx += 128) {
      int r = idx >> 3, c = idx & 7;
      cp_async16(sB_u + kb * B_BYTES + r * 128 + ((c ^ (r & 7)) << 4), Bw + (int64_t)r * K + kb * 64 + c * 8);
    }
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  // generic-proxy smem writes -> visible to the tensor core (async proxy)
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;

  if (tid == 0) {
    const uint32_t idesc = umma_idesc_bf16(N);
#pragma unroll
    for (int kb = 0; kb < KB; ++kb)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint64_t da = umma_desc_sw128(sA_u + kb * A_BYTES + k * 32);
        uint64_t db = umma_desc_sw128(sB_u + kb * B_BYTES + k * 32);
        umma_bf16(tmem, da, db, idesc, (kb | k) ? 1u : 0u);
      }
    umma_commit(bar);
  }
  mbar_wait(bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");

  // ---- epilogue: thread = tile row (TMEM lane 32*warp + lane); rows are staged per warp in
  // the (now idle) operand smem and written back as contiguous, coalesced 16-byte chunks.
  constexpr int RB = N * (int)sizeof(TY);  // bytes per output row
  constexpr int CH = RB / 16;
  uint8_t* stage = smem + warp * 32 * RB;
  const int r = warp * 32 + lane;
  const bool valid = r < nrows;
  const int64_t row = t.row0 + r;
  constexpr int NV = N < 32 ? N : 32;  // valid columns per 32-column TMEM load
  float dot = 0.f;
#pragma unroll
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    if (dotvec) {
#pragma unroll
      for (int i = 0; i < NV; ++i) dot = fmaf(v[i], __ldg(dotvec + (size_t)t.w * N + c0 + i), dot);
    }
    if (red_ptr && valid) {  // fused per-row reduction of gathered rows (fp32 or bf16)
      for (int j = red_ptr[row], je = red_ptr[row + 1]; j < je; ++j) {
        if (red_bf16) {
          const bf16* rr = static_cast<const bf16*>(red_rows) + (int64_t)red_list[j] * N + c0;
          if constexpr (NV % 8 == 0) {
#pragma unroll
            for (int i = 0; i < NV; i += 8) {
              float x[8];
              load16(rr + i, x);
#pragma unroll
              for (int q = 0; q < 8; ++q) v[i + q] += x[q];
            }
          } else {
#pragma unroll
            for (int i = 0; i < NV; ++i) v[i] += __bfloat162float(rr[i]);
          }
        } else {
          const float* rr = static_cast<const float*>(red_rows) + (int64_t)red_list[j] * N + c0;
#pragma unroll
          for (int i = 0; i < NV; i += 4) {
            float4 x = __ldg(reinterpret_cast<const float4*>(rr + i));
            v[i] += x.x; v[i + 1] += x.y; v[i + 2] += x.z; v[i + 3] += x.w;
          }
        }
      }
    }
    stage_vals<TY, NV, CH>(stage + lane * RB, lane, c0 * (int)sizeof(TY) / 16, v);
  }
  if (dotvec && valid) dotout[row] = dot;
  __syncwarp();
  const int rows_here = min(32, nrows - warp * 32);
  uint8_t* ybase = reinterpret_cast<uint8_t*>(Y) + (t.row0 + (int64_t)warp * 32) * RB;
#pragma unroll 4
  for (int k = lane; k < 32 * CH; k += 32) {
    const int rr = k / CH, j = k % CH;
    if (rr < rows_here)
      *reinterpret_cast<uint4*>(ybase + (int64_t)rr * RB + j * 16) =
          *reinterpret_cast<const uint4*>(stage + rr * RB + ((j ^ (rr & (CH - 1))) << 4));
  }

  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc<NCOLS>(tmem);
}

// ------------------------------------------------------------------ weight gradient on tcgen05
// partial[tile] = (sum_{rows of tile} A[gather(row)]^T Bm[row])  as  D[m = k2][n = k1]:
//   M = 128 covers K2 (the gradient width; for K2 = 64 the second 64-row half of the MMA
//   re-reads the same smem block through LBO = 0 and its lanes are ignored),
//   N = K1 (d_in), K = the rows, 16 per instruction.  Both operands are MN-major: a staged
//   row (128 B = 64 elements) is one 128B-swizzle line, 8 rows form a 1024-B atom (SBO),
//   64-element MN blocks sit at +LBO.  Rows past the tile end are zero-filled (cp.async
//   src-size 0) so they contribute nothing.  Two smem stages overlap the next sub-tile's
//   gather with the current MMAs; the accumulator stays in TMEM for the whole tile.
template <int K1, int K2>
__global__ void __launch_bounds__(128) k_wgrad_tc(const Tile* __restrict__ tiles, const bf16* __restrict__ A,
                                                  const int32_t* __restrict__ gather, const bf16* __restrict__ Bm,
                                                  float* __restrict__ partial) {
  constexpr int ROWS = 128;                  // rows per sub-tile (8 MMAs of K = 16)
  constexpr int KB1 = K1 / 64, KB2 = K2 / 64;  // 64-element MN blocks
  constexpr uint32_t BLK = ROWS * 128;       // bytes of one MN block of one sub-tile
  constexpr uint32_t STAGE = (KB1 + KB2) * BLK;
  constexpr int NCOLS = K1 <= 64 ? 64 : 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * STAGE);  // [2] stage-free barriers + [1] done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Tile t = tiles[blockIdx.x];
  const int nsub = (t.row1 - t.row0 + ROWS - 1) / ROWS;
  const uint32_t s_base = smem_u32(smem);

  if (warp == 0) tmem_alloc<NCOLS>(tslot);
  if (tid == 32) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }

  auto load = [&](int sub, int stage) {
    const uint32_t sb = s_base + stage * STAGE;
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      int idx = it * 128 + tid;
      int r = idx >> 3, c = idx & 7;
      int row = t.row0 + sub * ROWS + r;
      bool ok = row < t.row1;
      int rr = ok ? row : t.row0;
      int64_t xa = gather ? (int64_t)gather[rr] : (int64_t)rr;
      uint32_t off = r * 128 + ((c ^ (r & 7)) << 4);
#pragma unroll
      for (int j = 0; j < KB2; ++j) cp_async16_zfill(sb + j * BLK + off, Bm + (int64_t)rr * K2 + j * 64 + c * 8, ok);
#pragma unroll
      for (int j = 0; j < KB1; ++j)
        cp_async16_zfill(sb + (KB2 + j) * BLK + off, A + xa * K1 + j * 64 + c * 8, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  load(0, 0);
  __syncthreads();  // barrier init + TMEM address visible
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t idesc = umma_idesc_bf16_mn(K1);
  for (int sub = 0; sub < nsub; ++sub) {
    const int st = sub & 1;
    if (sub + 1 < nsub) {
      if (sub + 1 >= 2) mbar_wait(&bars[(sub + 1) & 1], ((sub - 1) >> 1) & 1);  // MMAs of sub-1 freed it
      load(sub + 1, (sub + 1) & 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t sb = s_base + st * STAGE;
#pragma unroll
      for (int k = 0; k < ROWS / 16; ++k) {
        uint64_t da = umma_desc_mn_sw128(sb + k * 2048, KB2 == 2 ? BLK : 0);
        uint64_t db = umma_desc_mn_sw128(sb + KB2 * BLK + k * 2048, BLK);
        umma_bf16(tmem, da, db, idesc, (sub | k) ? 1u : 0u);
      }
      umma_commit(&bars[st]);
      if (sub == nsub - 1) umma_commit(&bars[2]);
    }
  }
  mbar_wait(&bars[2], 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // epilogue: lane m = k2 (rows 0..K2-1 of D), columns n = k1; partial[tile][k1][k2]
  float* out = partial + (size_t)blockIdx.x * K1 * K2;
  if (warp * 32 < K2) {
#pragma unroll
    for (int c0 = 0; c0 < K1; c0 += 32) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
      const int m = warp * 32 + lane;
#pragma unroll
      for (int i = 0; i < 32; ++i) out[(size_t)(c0 + i) * K2 + m] = v[i];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc<NCOLS>(tmem);
}

template <int K1, int K2>
void launch_wgrad_tc(const WgradArgs& a, cudaStream_t s) {
  constexpr uint32_t STAGE = (K1 / 64 + K2 / 64) * 128 * 128;
  size_t smem = 1024 + 2 * STAGE + 64;
  auto k = k_wgrad_tc<K1, K2>;
  static bool attr_set = false;
  if (!attr_set) {
    RGNN_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  launch(a.name, k, dim3(a.plan->count), dim3(128), smem, s, a.plan->tiles, static_cast<const bf16*>(a.A), a.gather,
         static_cast<const bf16*>(a.Bm), a.partial);
}

// ------------------------------------------------------------------ fused pair-side backward (A8)
// One pass over the pair gradient rows dP (= dKM for HGT) of a 2048-row weight-gradient tile
// computes both products that read them:
//   partial[tile] = sum_{rows} X[gather(row)]^T dP[row]        (as k_wgrad_tc: D_w[m = k2][n = k1])
//   Y[row]        = dP[row] W_w^T   (W_w: [K1][K2] row-major, i.e. already K-major for this MMA)
// The staged dP sub-tile is read by the tensor cores twice: MN-major (weight gradient) and
// K-major (dX rows) -- the 128B-swizzled lines are the same bytes in both views.  The dX
// accumulator is double-buffered in TMEM; its epilogue (thread = row, bf16 row store) for
// sub-tile s runs while the MMAs of s+1 execute.  Saves one full read of dP versus the two
// separate kernels.
template <int K1, int K2, int S>
__global__ void __launch_bounds__(128) k_pair_bwd_tc(const Tile* __restrict__ tiles, const bf16* __restrict__ A,
                                                     const int32_t* __restrict__ gather, const bf16* __restrict__ Bm,
                                                     const bf16* __restrict__ Wm, bf16* __restrict__ Y,
                                                     float* __restrict__ partial) {
  constexpr int ROWS = 128;
  constexpr int KB1 = K1 / 64, KB2 = K2 / 64;
  constexpr uint32_t BLK = ROWS * 128;
  constexpr uint32_t STAGE = (KB1 + KB2) * BLK;
  constexpr uint32_t WBLK = K1 * 128;  // one 64-wide K block of the K1 weight rows
  constexpr int NCOLS = K1 <= 64 ? 256 : 512;  // D_w (K1) + 2 x D_x (K1)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // barriers: free[S] (stage s consumed by its MMAs), xready[2] (dX accumulator b written), done
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * STAGE + KB2 * WBLK);
  uint64_t* xready = bars + S;
  uint64_t* done = bars + S + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + S + 3);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Tile t = tiles[blockIdx.x];
  const int nsub = (t.row1 - t.row0 + ROWS - 1) / ROWS;
  const uint32_t s_base = smem_u32(smem);
  const uint32_t s_w = s_base + S * STAGE;

  if (warp == 0) tmem_alloc<NCOLS>(tslot);
  if (tid == 32) {
#pragma unroll
    for (int i = 0; i < S + 3; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // the segment's weight W_w (K1 rows of K2) into KB2 swizzled K blocks
  for (int idx = tid; idx < K1 * 8 * KB2; idx += 128) {
    const int kb = idx / (K1 * 8), rem = idx % (K1 * 8), n = rem >> 3, c = rem & 7;
    cp_async16(s_w + kb * WBLK + n * 128 + ((c ^ (n & 7)) << 4), Wm + ((int64_t)t.w * K1 + n) * K2 + kb * 64 + c * 8);
  }
  // sub-tile `sub` into stage sub % S; every call commits one cp.async group (empty past the end)
  auto load = [&](int sub) {
    if (sub < nsub) {
      const uint32_t sb = s_base + (sub % S) * STAGE;
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        int idx = it * 128 + tid;
        int r = idx >> 3, c = idx & 7;
        int row = t.row0 + sub * ROWS + r;
        bool ok = row < t.row1;
        int rr = ok ? row : t.row0;
        int64_t xa = gather ? (int64_t)gather[rr] : (int64_t)rr;
        uint32_t off = r * 128 + ((c ^ (r & 7)) << 4);
#pragma unroll
        for (int j = 0; j < KB2; ++j)
          cp_async16_zfill(sb + j * BLK + off, Bm + (int64_t)rr * K2 + j * 64 + c * 8, ok);
#pragma unroll
        for (int j = 0; j < KB1; ++j)
          cp_async16_zfill(sb + (KB2 + j) * BLK + off, A + xa * K1 + j * 64 + c * 8, ok);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  // prologue: S-1 sub-tiles in flight (the weight copies join the first group)
#pragma unroll
  for (int i = 0; i < S - 1; ++i) load(i);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t idesc_w = umma_idesc_bf16_mn(K1);
  const uint32_t idesc_x = umma_idesc_bf16(K1);

  auto epilogue_x = [&](int sb_i) {
    const int b = sb_i & 1;
    mbar_wait(&xready[b], (sb_i >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const int r = warp * 32 + lane;
    const int64_t row = (int64_t)t.row0 + sb_i * ROWS + r;
    const bool ok = row < t.row1;
#pragma unroll
    for (int c0 = 0; c0 < K1; c0 += 32) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + K1 + b * K1 + c0, v);
      if (ok) {
        bf16* yp = Y + row * K1 + c0;
#pragma unroll
        for (int q = 0; q < 4; ++q) store16(yp + 8 * q, v + 8 * q);
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  };

  for (int sub = 0; sub < nsub; ++sub) {
    const int st = sub % S;
    // refill the stage last used by sub-1 (its MMAs must have consumed it) with sub + S - 1
    if (sub >= 1 && sub + S - 1 < nsub) mbar_wait(&bars[(sub - 1) % S], ((sub - 1) / S) & 1);
    load(sub + S - 1);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(S - 1) : "memory");  // sub-tile `sub` landed
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t sb = s_base + st * STAGE;
#pragma unroll
      for (int k = 0; k < ROWS / 16; ++k) {  // weight gradient: D_w += dP^T X (both MN-major)
        uint64_t da = umma_desc_mn_sw128(sb + k * 2048, KB2 == 2 ? BLK : 0);
        uint64_t db = umma_desc_mn_sw128(sb + KB2 * BLK + k * 2048, BLK);
        umma_bf16(tmem, da, db, idesc_w, (sub | k) ? 1u : 0u);
      }
#pragma unroll
      for (int kb = 0; kb < KB2; ++kb)  // dX rows: D_x[sub & 1] = dP W^T (both K-major)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint64_t da = umma_desc_sw128(sb + kb * BLK + k * 32);
          uint64_t db = umma_desc_sw128(s_w + kb * WBLK + k * 32);
          umma_bf16(tmem + K1 + (sub & 1) * K1, da, db, idesc_x, (kb | k) ? 1u : 0u);
        }
      umma_commit(&bars[st]);
      umma_commit(&xready[sub & 1]);
      if (sub == nsub - 1) umma_commit(done);
    }
    if (sub >= 1) epilogue_x(sub - 1);
  }
  if (nsub > 0) epilogue_x(nsub - 1);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  float* out = partial + (size_t)blockIdx.x * K1 * K2;
  if (warp * 32 < K2) {
#pragma unroll
    for (int c0 = 0; c0 < K1; c0 += 32) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
      const int m = warp * 32 + lane;
#pragma unroll
      for (int i = 0; i < 32; ++i) out[(size_t)(c0 + i) * K2 + m] = v[i];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc<NCOLS>(tmem);
}

#ifndef RGNN_PAIR_BWD_STAGES
#define RGNN_PAIR_BWD_STAGES 2
#endif

template <int K1, int K2>
void launch_pair_bwd_tc(const PairBwdArgs& a, cudaStream_t s) {
  constexpr int S = RGNN_PAIR_BWD_STAGES;
  constexpr uint32_t STAGE = (K1 / 64 + K2 / 64) * 128 * 128;
  size_t smem = 1024 + S * STAGE + (K2 / 64) * K1 * 128 + 128;
  // at most two CTAs per SM: TMEM 2 x 256 columns (K1 = 64)
  smem = std::max(smem, (size_t)(232448 / 3) + 1);
  auto k = k_pair_bwd_tc<K1, K2, S>;
  static bool attr_set = false;
  if (!attr_set) {
    RGNN_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  launch(a.name, k, dim3(a.plan->count), dim3(128), smem, s, a.plan->tiles, static_cast<const bf16*>(a.X), a.gather,
         static_cast<const bf16*>(a.dP), static_cast<const bf16*>(a.W), static_cast<bf16*>(a.Y), a.partial);
}

// ------------------------------------------------------------------ persistent warp-specialized GEMM
// One CTA per SM loops over work items (tile, n-block) in static round robin; an item is a
// 128-row tile of one weight segment times an NT-column block of that segment's weight.
// Warps 4-7 gather the A rows (X[gather(row)]) and the weight's K-major rows of one 64-wide K
// block per smem stage with cp.async (S stages in a ring, up to S-1 in flight; a stage is handed
// to the MMA warp once the producers' own copies landed and were fenced for the async proxy);
// warp 8 issues the tcgen05.mma (M = 128, N = NT, K = 16) into one of two TMEM accumulators and
// commits the stage back to the producers and the accumulator to the epilogue; warps 0-3 (TMEM
// lane quarters) drain the previous item's accumulator (tcgen05.ld, optional per-row dot,
// bf16/fp32 pack, swizzled 128-byte row chunks staged per warp, coalesced row stores) while the
// next item is gathered and multiplied; warp 9 owns the TMEM allocation.  K is a runtime
// multiple of 64, so the same kernel serves the layer (d = 64/128) and the d-sweep of D3.
template <int NT, class TY>
struct WsCfg {
  static constexpr int NCOLS = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;
  static constexpr uint32_t A_BYTES = 128 * 128;
  static constexpr uint32_t B_BYTES = NT * 128;
  static constexpr uint32_t STAGE = A_BYTES + B_BYTES;
  static constexpr uint32_t RB = NT * sizeof(TY);       // tile row bytes
  static constexpr uint32_t CB = RB < 128 ? RB : 128;   // staged row-chunk bytes
  static constexpr int CC = CB / sizeof(TY);            // columns per staged chunk
  static constexpr int PC = CB / 16;                    // 16-byte pieces per row chunk
  static constexpr uint32_t STAGING = 4 * 32 * CB;      // 4 epilogue warps x 32 rows
  static constexpr int S_FIT = (int)((220 * 1024 - STAGING) / STAGE);
  static constexpr int S = S_FIT < 8 ? S_FIT : 8;
  static constexpr size_t SMEM = 1024 + (size_t)S * STAGE + STAGING + 256;
};

template <class TY, int NT>
__global__ void __launch_bounds__(320, 1) k_gemm_ws(const Tile* __restrict__ tiles, int ntiles, int nblk,
                                                    const bf16* __restrict__ A, const int32_t* __restrict__ gather,
                                                    int K, const bf16* __restrict__ Bt, int ntot, TY* __restrict__ Y,
                                                    const float* __restrict__ dotvec, float* __restrict__ dotout) {
  using C = WsCfg<NT, TY>;
  constexpr int S = C::S;
  static_assert(S >= 2, "not enough shared memory for two stages");
  const int KB = K >> 6, nitems = ntiles * nblk;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + S * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + C::STAGING);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t s_base = smem_u32(smem);

  if (warp == 9) tmem_alloc<2 * C::NCOLS>(tslot);
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 128);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp >= 4 && warp < 8) {
    // ------------------------------------------------ producers (warps 4-7, 128 threads)
    // thread ptid copies 16-byte chunk ptid % 8 of rows ptid / 8 + 16 i; the next item's row
    // indices are loaded while this item's copies are issued, so the gather never stalls issue
    const int ptid = tid - 128, c = ptid & 7, r0 = ptid >> 3;
    int st = 0, pend = 0, old = 0;
    uint32_t ph = 0;
    int64_t nxt[8];
    auto load_rows = [&](int item) {
      const Tile t = tiles[item / nblk];
      const int nrows = t.row1 - t.row0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = r0 + 16 * i, rr = r < nrows ? r : nrows - 1;
        nxt[i] = gather ? (int64_t)__ldg(gather + t.row0 + rr) : (int64_t)(t.row0 + rr);
      }
    };
    if (blockIdx.x < nitems) load_rows(blockIdx.x);
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int ti = it / nblk, nb = it - ti * nblk;
      const int w = tiles[ti].w;
      int64_t cur[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) cur[i] = nxt[i];
      if (it + (int)gridDim.x < nitems) load_rows(it + gridDim.x);
      const bf16* Bw = Bt + ((size_t)w * ntot + (size_t)nb * NT) * K;
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&empty[st], ph ^ 1);
        const uint32_t sa = s_base + st * C::STAGE, sb = sa + C::A_BYTES;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = r0 + 16 * i;
          cp_async16(sa + r * 128 + ((c ^ (r & 7)) << 4), A + cur[i] * K + kb * 64 + c * 8);
        }
#pragma unroll 4
        for (int r = r0; r < NT; r += 16)
          cp_async16(sb + r * 128 + ((c ^ (r & 7)) << 4), Bw + (int64_t)r * K + kb * 64 + c * 8);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        if (++pend == S - 1) {
          asm volatile("cp.async.wait_group %0;\n" ::"n"(S - 2) : "memory");
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          mbar_arrive(&full[old]);
          if (++old == S) old = 0;
          --pend;
        }
        if (++st == S) { st = 0; ph ^= 1; }
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    for (; pend > 0; --pend) {
      mbar_arrive(&full[old]);
      if (++old == S) old = 0;
    }
  } else if (warp == 8) {
    // ------------------------------------------------ MMA issuer (one thread)
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(NT);
      int st = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        mbar_wait(&tempty[acc], aph ^ 1);  // the epilogue drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t d_tmem = tmem + acc * C::NCOLS;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[st], ph);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t sa = s_base + st * C::STAGE, sb = sa + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(d_tmem, umma_desc_sw128(sa + k * 32), umma_desc_sw128(sb + k * 32), idesc, (kb | k) ? 1u : 0u);
          umma_commit(&empty[st]);  // stage free once these MMAs have read it
          if (++st == S) { st = 0; ph ^= 1; }
        }
        umma_commit(&tfull[acc]);  // accumulator complete
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ------------------------------------------------ epilogue (warps 0-3 = TMEM lane quarters)
    constexpr int NV = C::CC < 32 ? C::CC : 32;
    const int q = warp;
    uint8_t* stg = staging + q * 32 * C::CB;
    int acc = 0;
    uint32_t aph = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int ti = it / nblk, nb = it - ti * nblk;
      const Tile t = tiles[ti];
      const int nrows = t.row1 - t.row0;
      const int rows_here = min(32, nrows - q * 32);
      const int64_t row = t.row0 + q * 32 + lane;
      uint8_t* ybase = reinterpret_cast<uint8_t*>(Y + (t.row0 + (int64_t)q * 32) * ntot + (int64_t)nb * NT);
      const int64_t ystride = (int64_t)ntot * sizeof(TY);
      mbar_wait(&tfull[acc], aph);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t tb = tmem + acc * C::NCOLS + ((uint32_t)(q * 32) << 16);
      float dot = 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < NT; c0 += C::CC) {
#pragma unroll
        for (int s0 = 0; s0 < C::CC; s0 += 32) {
          float v[32];
          tmem_ld32(tb + c0 + s0, v);
          if (dotvec) {
#pragma unroll
            for (int i = 0; i < NV; ++i) dot = fmaf(v[i], __ldg(dotvec + (size_t)t.w * ntot + c0 + s0 + i), dot);
          }
          stage_vals<TY, NV, C::PC>(stg + lane * C::CB, lane, s0 * (int)sizeof(TY) / 16, v);
        }
        __syncwarp();
#pragma unroll
        for (int k = lane; k < 32 * C::PC; k += 32) {
          const int rr = k / C::PC, j = k % C::PC;
          if (rr < rows_here)
            *reinterpret_cast<uint4*>(ybase + rr * ystride + c0 * (int)sizeof(TY) + j * 16) =
                *reinterpret_cast<const uint4*>(stg + rr * C::CB + ((j ^ (rr & (C::PC - 1))) << 4));
        }
        __syncwarp();
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      mbar_arrive(&tempty[acc]);  // TMEM reads done: the MMA warp may reuse this accumulator
      if (dotvec && lane < rows_here) dotout[row] = dot;
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 9) tmem_dealloc<2 * C::NCOLS>(tmem);
}

template <class TY, int NT>
void launch_ws(const GemmArgs& a, const bf16* Bt, cudaStream_t s) {
  using C = WsCfg<NT, TY>;
  auto k = k_gemm_ws<TY, NT>;
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    RGNN_CUDA(cudaGetDevice(&dev));
    RGNN_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    RGNN_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  }
  const int nblk = a.N / NT;
  const int grid = std::min(a.ntiles * nblk, num_sms);
  launch(a.name, k, dim3(grid), dim3(320), C::SMEM, s, a.tiles, a.ntiles, nblk, static_cast<const bf16*>(a.A),
         a.gather, a.K, Bt, a.N, static_cast<TY*>(a.Y), a.dotvec, a.dotout);
}

template <class TY>
void ws_by_n(const GemmArgs& a, const bf16* Bt, cudaStream_t s) {
  switch (a.N < 256 ? a.N : 256) {
    case 16: launch_ws<TY, 16>(a, Bt, s); break;
    case 32: launch_ws<TY, 32>(a, Bt, s); break;
    case 64: launch_ws<TY, 64>(a, Bt, s); break;
    case 128: launch_ws<TY, 128>(a, Bt, s); break;
    case 256: launch_ws<TY, 256>(a, Bt, s); break;
    default: RGNN_FAIL(RGNN_ERR_UNSUPPORTED, "tcgen05 gemm: N");
  }
}

template <class TY, int N, int KB>
void launch_tc(const GemmArgs& a, const bf16* Bt, cudaStream_t s) {
  constexpr int NCOLS = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  // operands, reused by the epilogue's row staging (128 rows x N x sizeof(TY)) once the MMAs are done
  size_t smem = 1024 + std::max<size_t>(KB * (128 * 128 + N * 128), 128 * N * sizeof(TY)) + 64;
  // keep concurrent CTAs per SM within the 512 TMEM columns (alloc never waits)
  size_t floor_smem = (size_t)(232448 / (512 / NCOLS + 1)) + 1;
  smem = std::max(smem, floor_smem);
  auto k = k_gemm_tc<TY, N, KB>;
  static bool attr_set = false;
  if (!attr_set) {
    RGNN_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  launch(a.name, k, dim3(a.ntiles), dim3(128), smem, s, a.tiles, static_cast<const bf16*>(a.A), a.gather, Bt,
         static_cast<TY*>(a.Y), a.dotvec, a.dotout, a.red_ptr, a.red_list, a.red_rows, (int)(a.red_dtype == BF16));
}

template <class TY, int KB>
void by_n(const GemmArgs& a, const bf16* Bt, cudaStream_t s) {
  switch (a.N) {
    case 16: launch_tc<TY, 16, KB>(a, Bt, s); break;
    case 32: launch_tc<TY, 32, KB>(a, Bt, s); break;
    case 64: launch_tc<TY, 64, KB>(a, Bt, s); break;
    case 128: launch_tc<TY, 128, KB>(a, Bt, s); break;
    case 256: launch_tc<TY, 256, KB>(a, Bt, s); break;
    default: RGNN_FAIL(RGNN_ERR_UNSUPPORTED, "tcgen05 gemm: N");
  }
}

// k_gemm_tc holds a whole tile's K in shared memory: K <= 128, N <= 256, not both at the maximum.
bool fits_tc(const GemmArgs& a) { return a.K <= 128 && a.N <= 256 && !(a.K == 128 && a.N == 256); }

bool use_ws(const GemmArgs& a) {
  if (a.red_ptr != nullptr) return false;  // the fused reduce epilogue exists only in k_gemm_tc
  if (!fits_tc(a)) return true;
  const int mode = ws_mode();
  return mode == 2 || (mode == 1 && a.gather == nullptr);
}

}  // namespace

bool pair_bwd_tc_supported(int K1, int K2) { return K1 == 64 && (K2 == 64 || K2 == 128); }

void pair_bwd_tc(const PairBwdArgs& a, cudaStream_t s) {
  RGNN_CHECK(pair_bwd_tc_supported(a.K1, a.K2), RGNN_ERR_UNSUPPORTED, "fused pair backward: K1 = 64, K2 = 64 / 128");
  RGNN_CUDA(cudaMemsetAsync(a.out, 0, (size_t)a.num_w * a.K1 * a.K2 * sizeof(float), s));
  if (a.plan->count == 0) return;
  if (pair_bwd_ws_enabled(a)) pair_bwd_ws(a, s);
  else if (a.K2 == 64) launch_pair_bwd_tc<64, 64>(a, s);
  else launch_pair_bwd_tc<64, 128>(a, s);
  seg_partial_reduce(*a.plan, (const float*)a.partial, (int64_t)a.K1 * a.K2, a.out, s);
}

bool wgrad_tc_supported(const WgradArgs& a) {
  return a.a_dtype == BF16 && a.b_dtype == BF16 && (a.K1 == 64 || a.K1 == 128) && (a.K2 == 64 || a.K2 == 128);
}

void wgrad_tc(const WgradArgs& a, cudaStream_t s) {
  if (a.K1 == 64 && a.K2 == 64) launch_wgrad_tc<64, 64>(a, s);
  else if (a.K1 == 64 && a.K2 == 128) launch_wgrad_tc<64, 128>(a, s);
  else if (a.K1 == 128 && a.K2 == 64) launch_wgrad_tc<128, 64>(a, s);
  else launch_wgrad_tc<128, 128>(a, s);
}

bool gemm_tc_supported(const GemmArgs& a) {
  if (a.a_dtype != BF16 || a.b_dtype != BF16 || a.bt_scratch == nullptr) return false;
  if (a.K <= 0 || a.K % 64 != 0 || a.K > 8192) return false;
  const bool n_ok = a.N == 16 || a.N == 32 || a.N == 64 || a.N == 128 || (a.N % 256 == 0 && a.N <= 8192);
  if (!n_ok) return false;
  if (a.N > 256 && a.dotvec != nullptr) return false;  // the dot epilogue needs the whole row in one item
  if (a.red_ptr != nullptr && !fits_tc(a)) return false;
  return true;
}

void gemm_tc(const GemmArgs& a, cudaStream_t s) {
  // K-major bf16 image of the weights for the B operand
  int64_t total = (int64_t)a.num_w * a.K * a.N;
  bf16* Bt = static_cast<bf16*>(a.bt_scratch);
  launch("gemm_tc_prep_b", k_transpose_kmajor<bf16>, dim3(ceil_div(total, 256)), dim3(256), 0, s, (int64_t)a.num_w,
         a.K, a.N, static_cast<const bf16*>(a.B), a.transB, Bt);
  if (gemm_tma_enabled(a)) {
    gemm_tma(a, Bt, s);
    return;
  }
  if (use_ws(a)) {
    if (a.y_dtype == BF16) ws_by_n<bf16>(a, Bt, s); else ws_by_n<float>(a, Bt, s);
    return;
  }
  const int KB = a.K / 64;
  if (a.y_dtype == BF16) {
    if (KB == 1) by_n<bf16, 1>(a, Bt, s); else by_n<bf16, 2>(a, Bt, s);
  } else {
    if (KB == 1) by_n<float, 1>(a, Bt, s); else by_n<float, 2>(a, Bt, s);
  }
}

}  // namespace rgnn
