// A1 / A8 node and pair GEMMs on tcgen05 with TMA tile movement (bf16 operands, fp32 accumulation):
// the typed segment GEMM Y[row] = X[gather(row)] x W_w of the GEMM template Y[S] = X[G] x W[T]
// (§3.3.3; compact rows P:764-776), persistent and warp-specialized.
//
//   warps 4-7 producers: per 64-wide K block of an item (128-row tile x NT columns of one weight
//           segment) lane 0 of warp 4 arms the stage's mbarrier and issues the TMA loads -- B as one 2D box
//           of the K-major weight image and, for contiguous A, A as one 2D box of 128 rows -- 128B-swizzled
//           by the TMA unit into the canonical UMMA K-major layout; gathered A (X[pair_src]) is copied by
//           the 128 producer threads with cp.async into the same layout (a tile::gather4 TMA moves 4 x 128 B
//           per instruction from one thread: measured 3x slower for 128-byte rows), the next item's row
//           indices loaded while the current one is issued.
//   warp 8  MMA issuer (tcgen05.mma.cta_group::1.kind::f16, M = 128, N = NT, K = 16) into one of two
//           TMEM accumulators; tcgen05.commit frees the stage and publishes the accumulator.
//   warps 0-3 epilogue (TMEM lane quarters): tcgen05.ld, optional per-row dot (RGAT s_p = P_p . a_r,
//           P:962), pack to the output dtype into a 128B-swizzled staging box and one TMA 2D store
//           per 32 rows x 128 bytes (rows that end a segment mid-warp are stored by the lanes).
// The previous generation (gemm_tc.cu k_gemm_ws / k_gemm_tc) moves the same tiles with per-thread
// cp.async; this kernel replaces them for every GEMM without the fused per-source row reduction.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "ops.cuh"
#include "tc_ptx.cuh"

namespace rgnn {
namespace {
using namespace tc;

// ---------------------------------------------------------------- host: tensor maps
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// row-major [rows][cols] tensor of `esz`-byte elements, box {bcols, brows}, 128-byte swizzle
CUtensorMap make_map(const void* base, int esz, int64_t cols, int64_t rows, int bcols, int brows, bool l2_256) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(cols * esz)};
  cuuint32_t box[2] = {(cuuint32_t)bcols, (cuuint32_t)brows}, es[2] = {1, 1};
  const CUresult r = encode_fn()(&m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                 const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B,
                                 l2_256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  RGNN_CHECK(r == CUDA_SUCCESS, RGNN_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

// ---------------------------------------------------------------- kernel
template <int NT, class TY>
struct TmaCfg {
  static constexpr int NCOLS = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;
  static constexpr uint32_t A_BYTES = 128 * 128;
  static constexpr uint32_t B_BYTES = NT * 128;
  static constexpr uint32_t STAGE = A_BYTES + B_BYTES;
  static constexpr int RB = NT * (int)sizeof(TY);   // output row bytes of an item
  static constexpr int CB = RB < 128 ? RB : 128;    // staged row-chunk bytes
  static constexpr int CC = CB / (int)sizeof(TY);   // columns per chunk
  static constexpr int PC = CB / 16;                // 16-byte pieces per chunk row
  static constexpr bool TMA_Y = CB == 128;          // TMA store needs a full 128B-swizzle row
  static constexpr uint32_t STG = 32 * 128;         // one staging buffer of a warp (32 rows)
  static constexpr uint32_t STAGING = 4 * 2 * STG;  // 4 epilogue warps, double-buffered
  static constexpr int S_FIT = (int)((220 * 1024 - STAGING) / STAGE);
  static constexpr int S = S_FIT < 8 ? S_FIT : 8;
  static constexpr size_t SMEM = 1024 + (size_t)S * STAGE + STAGING + 256;
};

template <class TY, int NT, bool GATHER>
__global__ void __launch_bounds__(288, 1) k_gemm_tma(const __grid_constant__ CUtensorMap tmA,
                                                     const __grid_constant__ CUtensorMap tmB,
                                                     const __grid_constant__ CUtensorMap tmY,
                                                     const Tile* __restrict__ tiles, int ntiles, int nblk,
                                                     const bf16* __restrict__ A, const int32_t* __restrict__ gather,
                                                     int K, int ntot, TY* __restrict__ Y,
                                                     const float* __restrict__ dotvec, float* __restrict__ dotout) {
  using C = TmaCfg<NT, TY>;
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

  if (warp == 8) tmem_alloc<2 * C::NCOLS>(tslot);
  if (tid == 128) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (C::TMA_Y) tma_prefetch_desc(&tmY);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], GATHER ? 129 : 1);  // gathered: 128 producer threads + the TMA expect_tx arrival
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
    // ------------------------------------------------ producers
    // B (and A when contiguous) by TMA from lane 0 of warp 4; gathered A rows by the 128 producer threads
    // with cp.async (one group per stage, up to S - 1 in flight, released on the stage's full barrier once
    // landed and fenced for the async proxy), the next item's row indices loaded while this one is issued
    const int ptid = tid - 128, c = ptid & 7, r0 = ptid >> 3;  // rows r0 + 16 i, 16-byte chunk c
    int st = 0, pend = 0, old = 0;
    uint32_t ph = 0;
    int nidx[8], cur[8];
    auto load_idx = [&](int it) {
      const Tile t = tiles[it / nblk];
      const int nrows = t.row1 - t.row0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = r0 + 16 * i;
        nidx[i] = __ldg(gather + t.row0 + (r < nrows ? r : nrows - 1));
      }
    };
    if (GATHER && blockIdx.x < nitems) load_idx(blockIdx.x);
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int ti = it / nblk, nb = it - ti * nblk;
      const Tile t = tiles[ti];
      if (GATHER) {
#pragma unroll
        for (int i = 0; i < 8; ++i) cur[i] = nidx[i];
        if (it + (int)gridDim.x < nitems) load_idx(it + gridDim.x);
      }
      const int yb = t.w * ntot + nb * NT;
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&empty[st], ph ^ 1);
        const uint32_t sa = s_base + st * C::STAGE, sb = sa + C::A_BYTES;
        if (ptid == 0) {
          mbar_expect_tx(&full[st], GATHER ? C::B_BYTES : C::STAGE);
          if (!GATHER) tma_load_2d(sa, &tmA, kb * 64, t.row0, &full[st]);
          tma_load_2d(sb, &tmB, kb * 64, yb, &full[st]);
        }
        if (GATHER) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = r0 + 16 * i;
            cp_async16(sa + r * 128 + ((c ^ (r & 7)) << 4), A + (int64_t)cur[i] * K + kb * 64 + c * 8);
          }
          asm volatile("cp.async.commit_group;\n" ::: "memory");
          if (++pend == S - 1) {
            asm volatile("cp.async.wait_group %0;\n" ::"n"(S - 2) : "memory");
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_arrive(&full[old]);
            if (++old == S) old = 0;
            --pend;
          }
        }
        if (++st == S) { st = 0; ph ^= 1; }
      }
    }
    if (GATHER) {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      for (; pend > 0; --pend) {
        mbar_arrive(&full[old]);
        if (++old == S) old = 0;
      }
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
  } else {
    // ------------------------------------------------ epilogue (warps 0-3 = TMEM lane quarters)
    constexpr int NV = C::CC < 32 ? C::CC : 32;
    const int q = warp;
    uint8_t* stg0 = staging + q * 2 * C::STG;
    int acc = 0, buf = 0;
    uint32_t aph = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int ti = it / nblk, nb = it - ti * nblk;
      const Tile t = tiles[ti];
      const int nrows = t.row1 - t.row0;
      const int rows_here = min(32, nrows - q * 32);
      const int64_t row0 = t.row0 + (int64_t)q * 32;
      mbar_wait(&tfull[acc], aph);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t tb = tmem + acc * C::NCOLS + ((uint32_t)(q * 32) << 16);
      float dot = 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < NT; c0 += C::CC) {
        uint8_t* stg = stg0 + buf * C::STG;
        if (C::TMA_Y) {  // the store issued from this buffer two chunks ago has finished reading it
          if (lane == 0) tma_store_wait_read<1>();
          __syncwarp();
        }
#pragma unroll
        for (int s0 = 0; s0 < C::CC; s0 += 32) {
          float v[32];
          tmem_ld32(tb + c0 + s0, v);
          if (dotvec) {
#pragma unroll
            for (int i = 0; i < NV; ++i) dot = fmaf(v[i], __ldg(dotvec + (size_t)t.w * ntot + nb * NT + c0 + s0 + i), dot);
          }
          stage_vals<TY, NV, C::PC>(stg + lane * C::CB, lane, s0 * (int)sizeof(TY) / 16, v);
        }
        if (C::TMA_Y && rows_here == 32) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // staged rows -> async proxy
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmY, nb * NT + c0, (int)row0, smem_u32(stg));
            tma_store_commit();
          }
        } else {
          __syncwarp();
          uint8_t* ybase = reinterpret_cast<uint8_t*>(Y + row0 * ntot + (int64_t)nb * NT + c0);
          const int64_t ystride = (int64_t)ntot * sizeof(TY);
#pragma unroll
          for (int k = lane; k < 32 * C::PC; k += 32) {
            const int rr = k / C::PC, j = k % C::PC;
            if (rr < rows_here)
              *reinterpret_cast<uint4*>(ybase + rr * ystride + j * 16) =
                  *reinterpret_cast<const uint4*>(stg + rr * C::CB + ((j ^ (rr & (C::PC - 1))) << 4));
          }
          __syncwarp();
        }
        buf ^= 1;
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      mbar_arrive(&tempty[acc]);  // TMEM reads done: the MMA warp may reuse this accumulator
      if (dotvec && lane < rows_here) dotout[row0 + lane] = dot;
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
    if (C::TMA_Y && lane == 0) tma_store_wait<0>();
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 8) tmem_dealloc<2 * C::NCOLS>(tmem);
}

template <class TY, int NT>
void launch_tma(const GemmArgs& a, const bf16* Bt, cudaStream_t s) {
  using C = TmaCfg<NT, TY>;
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    RGNN_CUDA(cudaGetDevice(&dev));
    RGNN_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    RGNN_CUDA(cudaFuncSetAttribute(k_gemm_tma<TY, NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    RGNN_CUDA(cudaFuncSetAttribute(k_gemm_tma<TY, NT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  }
  const int nblk = a.N / NT;
  const int grid = std::min(a.ntiles * nblk, num_sms);
  // A: gathered rows come one at a time (box {64, 1}); the table's row count only bounds the map
  const int64_t a_rows = a.gather ? (a.a_rows > 0 ? a.a_rows : ((int64_t)1 << 31) - 1) : a.y_rows;
  const CUtensorMap tmA = make_map(a.A, 2, a.K, a_rows, 64, a.gather ? 1 : 128, a.gather == nullptr);
  const CUtensorMap tmB = make_map(Bt, 2, a.K, (int64_t)a.num_w * a.N, 64, NT, true);
  const CUtensorMap tmY = C::TMA_Y ? make_map(a.Y, (int)sizeof(TY), a.N, a.y_rows, C::CC, 32, true) : tmB;
  if (a.gather)
    launch(a.name, k_gemm_tma<TY, NT, true>, dim3(grid), dim3(288), C::SMEM, s, tmA, tmB, tmY, a.tiles, a.ntiles, nblk,
           static_cast<const bf16*>(a.A), a.gather, a.K, a.N, static_cast<TY*>(a.Y), a.dotvec, a.dotout);
  else
    launch(a.name, k_gemm_tma<TY, NT, false>, dim3(grid), dim3(288), C::SMEM, s, tmA, tmB, tmY, a.tiles, a.ntiles,
           nblk, static_cast<const bf16*>(a.A), a.gather, a.K, a.N, static_cast<TY*>(a.Y), a.dotvec, a.dotout);
}

template <class TY>
void tma_by_n(const GemmArgs& a, const bf16* Bt, cudaStream_t s) {
  switch (a.N < 256 ? a.N : 256) {
    case 16: launch_tma<TY, 16>(a, Bt, s); break;
    case 32: launch_tma<TY, 32>(a, Bt, s); break;
    case 64: launch_tma<TY, 64>(a, Bt, s); break;
    case 128: launch_tma<TY, 128>(a, Bt, s); break;
    case 256: launch_tma<TY, 256>(a, Bt, s); break;
    default: RGNN_FAIL(RGNN_ERR_UNSUPPORTED, "tcgen05 gemm: N");
  }
}

// ---------------------------------------------------------------- fused pair-side backward (A8), warp-specialized
// The fused kernel of gemm_tc.cu (k_pair_bwd_tc: one pass over a 2048-row weight-gradient tile of the pair
// gradient rows dP computes both Y = dP W_w^T and the tile's X[src]^T dP partial), persistent (one CTA per SM
// walks tiles blockIdx.x, + gridDim.x, ...) with the roles split:
//   warps 4-7  producers: per 128-row sub-tile the gathered X[src] rows by cp.async (zero-filled past the
//              tile end, so the rows a dP box reads beyond it contribute nothing to the weight gradient),
//              the next sub-tile's row indices loaded while this one is issued; lane 0 of warp 4 adds the
//              dP sub-tile as TMA 2D boxes (expect_tx) and, per tile, the K-major weight W_w into one of
//              two buffers (freed when the tile two back finished its MMAs).
//   warp 8     MMA issuer: D_w[j % 2] += dP^T X (both MN-major) and D_x[s % 2] = dP W^T (both K-major).
//   warps 0-3  epilogue: D_x[b] -> bf16 -> 128B-swizzled staging (two buffers) -> TMA 2D store per 32 rows;
//              at each tile end the D_w partial of that tile.
// S stages of (dP | X) sub-tiles are in flight; TMEM = 2 D_w + 2 D_x accumulators (256 columns).
template <int K1, int K2>
struct PbCfg {
  static constexpr int KB1 = K1 / 64, KB2 = K2 / 64;
  static constexpr uint32_t BLK = 128 * 128;                 // one 64-wide block of 128 rows
  static constexpr uint32_t STAGE = (KB1 + KB2) * BLK;       // [dP blocks | X blocks]
  static constexpr uint32_t WBLK = K1 * 128;                 // one 64-wide K block of the K1 weight rows
  static constexpr uint32_t WBYTES = KB2 * WBLK;
  static constexpr uint32_t STG = 32 * 128;                  // one staging buffer of an epilogue warp
  static constexpr uint32_t STAGING = 4 * 2 * STG;
  static constexpr int S_FIT = (int)((222 * 1024 - 2 * WBYTES - STAGING) / STAGE);
  static constexpr int S = S_FIT < 6 ? S_FIT : 6;
  static constexpr size_t SMEM = 1024 + (size_t)S * STAGE + 2 * WBYTES + STAGING + 512;
  static constexpr int NCOLS = 256;                          // 2 x D_w (K1) + 2 x D_x (K1)
};

template <int K1, int K2>
__global__ void __launch_bounds__(288, 1) k_pair_bwd_ws(const __grid_constant__ CUtensorMap tmP,
                                                        const __grid_constant__ CUtensorMap tmW,
                                                        const __grid_constant__ CUtensorMap tmY,
                                                        const Tile* __restrict__ tiles, int ntiles,
                                                        const bf16* __restrict__ A, const int32_t* __restrict__ gather,
                                                        bf16* __restrict__ Y, float* __restrict__ partial) {
  using C = PbCfg<K1, K2>;
  constexpr int S = C::S, KB1 = C::KB1, KB2 = C::KB2;
  constexpr uint32_t BLK = C::BLK, STAGE = C::STAGE, WBLK = C::WBLK;
  static_assert(S >= 2 && K1 == 64, "fused pair backward: K1 = 64");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t s_base = smem_u32(smem);
  const uint32_t s_w0 = s_base + S * STAGE;  // two weight buffers of WBYTES
  uint8_t* staging = smem + S * STAGE + 2 * C::WBYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + C::STAGING);
  uint64_t* empty = full + S;
  uint64_t* xready = empty + S;  // [2] D_x[b] written
  uint64_t* xempty = xready + 2; // [2] D_x[b] drained
  uint64_t* wready = xempty + 2; // [2] weight buffer b loaded
  uint64_t* wfree = wready + 2;  // [2] weight buffer b no longer read
  uint64_t* dready = wfree + 2;  // [2] D_w[b] complete
  uint64_t* dfree = dready + 2;  // [2] D_w[b] drained
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dfree + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == 8) tmem_alloc<C::NCOLS>(tslot);
  if (tid == 0) {
    tma_prefetch_desc(&tmP);
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmY);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 129);  // 128 producer threads + the TMA expect_tx arrival
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&xready[i], 1);
      mbar_init(&xempty[i], 128);
      mbar_init(&wready[i], 1);
      mbar_init(&wfree[i], 1);
      mbar_init(&dready[i], 1);
      mbar_init(&dfree[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp >= 4 && warp < 8) {
    // ------------------------------------------------ producers
    const int ptid = tid - 128, c = ptid & 7, r0 = ptid >> 3;  // rows r0 + 16 i, 16-byte chunk c
    int pend = 0, old = 0, g = 0;  // g: global sub-tile counter
    int nidx[8];
    auto load_idx = [&](const Tile& t, int sub) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = t.row0 + sub * 128 + r0 + 16 * i;
        nidx[i] = row < t.row1 ? __ldg(gather + row) : -1;
      }
    };
    auto drain = [&] {  // every issued group landed and released (nothing of an earlier tile left pending)
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      for (; pend > 0; --pend) {
        mbar_arrive(&full[old]);
        if (++old == S) old = 0;
      }
    };
    int jt = 0;
    for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++jt) {
      const Tile t = tiles[ti];
      const int nsub = (t.row1 - t.row0 + 127) / 128;
      // the weight buffer of tile jt is freed by the MMAs of tile jt - 2, which need this thread's pending
      // groups of earlier tiles: release them before anyone waits on it (short tiles at segment ends)
      if (jt >= 2) drain();
      if (ptid == 0) {  // this tile's weight into buffer jt % 2 once the tile two back stopped reading it
        const int wb = jt & 1;
        mbar_wait(&wfree[wb], ((jt >> 1) & 1) ^ 1);
        mbar_expect_tx(&wready[wb], C::WBYTES);
#pragma unroll
        for (int kb = 0; kb < KB2; ++kb) tma_load_2d(s_w0 + wb * C::WBYTES + kb * WBLK, &tmW, kb * 64, t.w * K1, &wready[wb]);
      }
      load_idx(t, 0);
      for (int sub = 0; sub < nsub; ++sub, ++g) {
        const int st = g % S;
        int cur[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) cur[i] = nidx[i];
        if (sub + 1 < nsub) load_idx(t, sub + 1);
        mbar_wait(&empty[st], ((g / S) & 1) ^ 1);
        const uint32_t sb = s_base + st * STAGE;
        if (ptid == 0) {
          mbar_expect_tx(&full[st], KB2 * BLK);
#pragma unroll
          for (int j = 0; j < KB2; ++j) tma_load_2d(sb + j * BLK, &tmP, j * 64, t.row0 + sub * 128, &full[st]);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = r0 + 16 * i;
          const bool ok = cur[i] >= 0;
          const uint32_t off = r * 128 + ((c ^ (r & 7)) << 4);
#pragma unroll
          for (int j = 0; j < KB1; ++j)
            cp_async16_zfill(sb + (KB2 + j) * BLK + off, A + (int64_t)(ok ? cur[i] : 0) * K1 + j * 64 + c * 8, ok);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        if (++pend == S - 1) {  // the oldest group landed: fence it for the async proxy, release its stage
          asm volatile("cp.async.wait_group %0;\n" ::"n"(S - 2) : "memory");
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          mbar_arrive(&full[old]);
          if (++old == S) old = 0;
          --pend;
        }
      }
    }
    drain();
  } else if (warp == 8) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc_w = umma_idesc_bf16_mn(K1), idesc_x = umma_idesc_bf16(K1);
      int g = 0, jt = 0;
      for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++jt) {
        const Tile t = tiles[ti];
        const int nsub = (t.row1 - t.row0 + 127) / 128, wb = jt & 1;
        const uint32_t s_w = s_w0 + wb * C::WBYTES;
        const uint32_t dw = tmem + wb * K1;  // D_w[jt % 2] at columns 0 / 64, D_x[b] at 128 / 192
        mbar_wait(&wready[wb], (jt >> 1) & 1);
        if (jt >= 2) mbar_wait(&dfree[wb], ((jt >> 1) - 1) & 1);  // the epilogue drained D_w[wb]
        for (int sub = 0; sub < nsub; ++sub, ++g) {
          const int st = g % S, b = g & 1;
          mbar_wait(&full[st], (g / S) & 1);
          if (g >= 2) mbar_wait(&xempty[b], ((g >> 1) - 1) & 1);  // the epilogue drained D_x[b]
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t sb = s_base + st * STAGE;
#pragma unroll
          for (int k = 0; k < 128 / 16; ++k) {
            const uint64_t da = umma_desc_mn_sw128(sb + k * 2048, KB2 == 2 ? BLK : 0);
            const uint64_t db = umma_desc_mn_sw128(sb + KB2 * BLK + k * 2048, BLK);
            umma_bf16(dw, da, db, idesc_w, (sub | k) ? 1u : 0u);
          }
#pragma unroll
          for (int kb = 0; kb < KB2; ++kb)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(tmem + 2 * K1 + b * K1, umma_desc_sw128(sb + kb * BLK + k * 32),
                        umma_desc_sw128(s_w + kb * WBLK + k * 32), idesc_x, (kb | k) ? 1u : 0u);
          umma_commit(&empty[st]);
          umma_commit(&xready[b]);
        }
        umma_commit(&dready[wb]);
        umma_commit(&wfree[wb]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ epilogue (warps 0-3 = TMEM lane quarters)
    int g = 0, jt = 0, buf = 0;
    for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++jt) {
      const Tile t = tiles[ti];
      const int nsub = (t.row1 - t.row0 + 127) / 128, wb = jt & 1;
      for (int sub = 0; sub < nsub; ++sub, ++g) {
        const int b = g & 1;
        uint8_t* stg = staging + (warp * 2 + buf) * C::STG;
        mbar_wait(&xready[b], (g >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (lane == 0) tma_store_wait_read<1>();  // the store issued from this buffer two rounds ago has read it
        __syncwarp();
        const int64_t row0 = (int64_t)t.row0 + sub * 128 + warp * 32;
        const int rows_here = min(32, (int)(t.row1 - row0));
#pragma unroll
        for (int c0 = 0; c0 < K1; c0 += 32) {
          float v[32];
          tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 2 * K1 + b * K1 + c0, v);
          stage_vals<bf16, 32, 8>(stg + lane * 128, lane, c0 * 2 / 16, v);
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        mbar_arrive(&xempty[b]);
        if (rows_here == 32) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmY, 0, (int)row0, smem_u32(stg));
            tma_store_commit();
          }
        } else {
          __syncwarp();
          uint8_t* ybase = reinterpret_cast<uint8_t*>(Y + row0 * K1);
#pragma unroll
          for (int k = lane; k < 32 * 8; k += 32) {
            const int rr = k / 8, j = k % 8;
            if (rr < rows_here)
              *reinterpret_cast<uint4*>(ybase + rr * 128 + j * 16) =
                  *reinterpret_cast<const uint4*>(stg + rr * 128 + ((j ^ (rr & 7)) << 4));
          }
          __syncwarp();
        }
        buf ^= 1;
      }
      // the tile's weight-gradient partial: lane m = k2 (rows 0..K2-1 of D_w), columns n = k1
      mbar_wait(&dready[wb], (jt >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      float* out = partial + (size_t)ti * K1 * K2;
      if (warp * 32 < K2) {
#pragma unroll
        for (int c0 = 0; c0 < K1; c0 += 32) {
          float v[32];
          tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + wb * K1 + c0, v);
          const int m = warp * 32 + lane;
#pragma unroll
          for (int i = 0; i < 32; ++i) out[(size_t)(c0 + i) * K2 + m] = v[i];
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      mbar_arrive(&dfree[wb]);
    }
    if (lane == 0) tma_store_wait<0>();
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 8) tmem_dealloc<C::NCOLS>(tmem);
}

template <int K1, int K2>
void launch_pair_bwd_ws(const PairBwdArgs& a, cudaStream_t s) {
  using C = PbCfg<K1, K2>;
  auto k = k_pair_bwd_ws<K1, K2>;
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    RGNN_CUDA(cudaGetDevice(&dev));
    RGNN_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    RGNN_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  }
  const CUtensorMap tmP = make_map(a.dP, 2, K2, a.rows, 64, 128, true);
  const CUtensorMap tmW = make_map(a.W, 2, K2, (int64_t)a.num_w * K1, 64, K1, true);  // W_w rows = K-major B of dX
  const CUtensorMap tmY = make_map(a.Y, 2, K1, a.rows, 64, 32, true);
  const int ntiles = a.plan->count;
  launch(a.name, k, dim3(std::min(ntiles, num_sms)), dim3(288), C::SMEM, s, tmP, tmW, tmY, a.plan->tiles, ntiles,
         static_cast<const bf16*>(a.X), a.gather, static_cast<bf16*>(a.Y), a.partial);
}

}  // namespace

// GEMMs without the fused per-source row reduction run here: contiguous A (TMA) always, gathered A (the
// producer warps' cp.async) when K > 128 -- at d = 64 the one-tile-per-CTA k_gemm_tc with ~9 CTAs per SM
// keeps more independent row gathers in flight (mag pair GEMM 0.242 vs 0.324 ms, wikikg2 0.849 vs 1.228 ms),
// from d = 512 this persistent pipeline is faster (D3 sweep, d = 1024: 962 vs 890 TFLOP/s).
// RGNN_TMA=0: never (cp.async generation for every GEMM); 2: contiguous A only; 3: every GEMM.
bool gemm_tma_enabled(const GemmArgs& a) {
  static const int mode = [] {
    const char* v = getenv("RGNN_TMA");
    return v ? atoi(v) : 1;
  }();
  if (mode == 0 || encode_fn() == nullptr) return false;
  if (a.gather != nullptr && (mode == 2 || (mode == 1 && a.K <= 128))) return false;
  if (a.red_ptr != nullptr || a.y_rows <= 0) return false;  // fused row reduction: k_gemm_tc only
  // TMA: 16-byte aligned bases and row strides
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return al(a.A) && al(a.Y) && (a.K * 2) % 16 == 0;
}

// RGNN_PAIR_WS=0: the two-role fused pair backward of gemm_tc.cu instead of the warp-specialized TMA one
bool pair_bwd_ws_enabled(const PairBwdArgs& a) {
  static const bool on = [] {
    const char* v = getenv("RGNN_PAIR_WS");
    return !(v && v[0] == '0');
  }();
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return on && encode_fn() != nullptr && a.rows > 0 && al(a.dP) && al(a.Y) && a.K1 == 64 && (a.K2 == 64 || a.K2 == 128);
}

void pair_bwd_ws(const PairBwdArgs& a, cudaStream_t s) {
  if (a.K2 == 64) launch_pair_bwd_ws<64, 64>(a, s);
  else launch_pair_bwd_ws<64, 128>(a, s);
}

void gemm_tma(const GemmArgs& a, const bf16* Bt, cudaStream_t s) {
  if (a.y_dtype == BF16) tma_by_n<bf16>(a, Bt, s);
  else tma_by_n<float>(a, Bt, s);
}

}  // namespace rgnn
