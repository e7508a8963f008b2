// C-ABI of the A1 primitive: the typed segment GEMM Y[S] = X[G] x W[T] (§3.3.3,
// algo:gemm_template P:901-918) on its own, over a caller segmentation (include/rgnn.h).
// The kernels are the layer's: k_gemm_ws / k_gemm_tc (tcgen05, bf16) and k_gemm_simt (f32).
#include <algorithm>
#include <cstring>
#include <vector>

#include "ops.cuh"

struct rgnn_segments_s {
  rgnn::Allocator alloc;
  int32_t nseg = 0;
  int64_t rows = 0;
  void* block = nullptr;          // device: tiles_tc | tiles_simt
  rgnn::Tile* tiles_tc = nullptr;  // 128-row tiles (tensor-core kernels)
  rgnn::Tile* tiles_simt = nullptr;  // 64-row tiles (SIMT kernel)
  int n_tc = 0, n_simt = 0;
  int32_t max_w = -1;
};

namespace rgnn {
namespace {

constexpr int TC_ROWS = 128, SIMT_ROWS = 64;

void make_tiles(const std::vector<int64_t>& ptr, const std::vector<int32_t>& w, int rows, std::vector<Tile>& out) {
  for (size_t i = 0; i + 1 < ptr.size(); ++i)
    for (int64_t r = ptr[i]; r < ptr[i + 1]; r += rows)
      out.push_back(Tile{(int32_t)r, (int32_t)std::min<int64_t>(r + rows, ptr[i + 1]), w[i], (int32_t)i});
}

}  // namespace
}  // namespace rgnn

using namespace rgnn;

extern "C" {

rgnn_status rgnn_segment_plan_create(int32_t num_segments, const int64_t* seg_ptr, const int32_t* seg_weight,
                                     rgnn_alloc_fn alloc, rgnn_free_fn free_fn, void* alloc_ctx, void* stream,
                                     rgnn_segments_t* out) {
  return guarded([&] {
    RGNN_CHECK(out && seg_ptr && num_segments >= 0, RGNN_ERR_INVALID_ARG, "NULL argument or negative segment count");
    *out = nullptr;
    RGNN_CHECK(seg_ptr[0] == 0, RGNN_ERR_INVALID_ARG, "seg_ptr[0] must be 0");
    std::vector<int64_t> ptr(seg_ptr, seg_ptr + num_segments + 1);
    std::vector<int32_t> w(num_segments);
    int32_t max_w = -1;
    for (int32_t i = 0; i < num_segments; ++i) {
      RGNN_CHECK(ptr[i + 1] >= ptr[i], RGNN_ERR_INVALID_ARG, "seg_ptr decreases at segment " + std::to_string(i));
      w[i] = seg_weight ? seg_weight[i] : i;
      RGNN_CHECK(w[i] >= 0, RGNN_ERR_INVALID_ARG, "negative weight index at segment " + std::to_string(i));
      max_w = std::max(max_w, w[i]);
    }
    RGNN_CHECK(ptr[num_segments] < (int64_t)INT32_MAX, RGNN_ERR_UNSUPPORTED, "more than 2^31-1 rows");
    std::vector<Tile> tc, simt;
    make_tiles(ptr, w, TC_ROWS, tc);
    make_tiles(ptr, w, SIMT_ROWS, simt);
    auto* p = new rgnn_segments_s();
    p->alloc = Allocator{alloc, free_fn, alloc_ctx};
    p->nseg = num_segments;
    p->rows = ptr[num_segments];
    p->n_tc = (int)tc.size();
    p->n_simt = (int)simt.size();
    p->max_w = max_w;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    try {
      const size_t bytes = std::max<size_t>(1, tc.size() + simt.size()) * sizeof(Tile);
      p->block = p->alloc.get(bytes, s);
      p->tiles_tc = static_cast<Tile*>(p->block);
      p->tiles_simt = p->tiles_tc + tc.size();
      std::vector<Tile> host(tc);
      host.insert(host.end(), simt.begin(), simt.end());
      if (!host.empty())
        RGNN_CUDA(cudaMemcpyAsync(p->block, host.data(), host.size() * sizeof(Tile), cudaMemcpyHostToDevice, s));
      RGNN_CUDA(cudaStreamSynchronize(s));  // `host` goes out of scope
    } catch (...) {
      if (p->block) p->alloc.put(p->block, s);
      delete p;
      throw;
    }
    *out = p;
  });
}

rgnn_status rgnn_segment_plan_destroy(rgnn_segments_t p) {
  return guarded([&] {
    if (!p) return;
    if (p->block) p->alloc.put(p->block, nullptr);
    delete p;
  });
}

rgnn_status rgnn_segment_gemm_workspace(rgnn_segments_t p, int32_t dtype, int32_t K, int32_t N, int32_t num_weights,
                                        size_t* scratch_bytes) {
  return guarded([&] {
    RGNN_CHECK(p && scratch_bytes, RGNN_ERR_INVALID_ARG, "NULL argument");
    RGNN_CHECK(K > 0 && N > 0 && num_weights > 0, RGNN_ERR_INVALID_ARG, "K, N and num_weights must be positive");
    *scratch_bytes = dtype == RGNN_BF16 ? (size_t)num_weights * K * N * sizeof(bf16) : 0;
  });
}

rgnn_status rgnn_segment_gemm(rgnn_segments_t p, int32_t dtype, const void* X, const int32_t* gather, int32_t K,
                              const void* W, int32_t num_weights, int32_t N, int32_t trans_w, void* Y, int32_t y_dtype,
                              void* scratch, size_t scratch_bytes, void* stream) {
  return guarded([&] {
    RGNN_CHECK(p && W && (Y || p->rows == 0), RGNN_ERR_INVALID_ARG, "NULL plan, W or Y");
    RGNN_CHECK(p->rows == 0 || X, RGNN_ERR_INVALID_ARG, "NULL X");
    RGNN_CHECK(dtype == RGNN_F32 || dtype == RGNN_BF16, RGNN_ERR_INVALID_ARG, "dtype");
    RGNN_CHECK(y_dtype == RGNN_F32 || (y_dtype == RGNN_BF16 && dtype == RGNN_BF16), RGNN_ERR_INVALID_ARG,
               "y_dtype must be F32, or BF16 with a BF16 dtype");
    RGNN_CHECK(num_weights > p->max_w, RGNN_ERR_INVALID_ARG, "the plan references weight " +
                                                                 std::to_string(p->max_w) + " >= num_weights");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    GemmArgs a;
    a.A = X;
    a.a_dtype = dtype;
    a.K = K;
    a.gather = gather;
    a.B = W;
    a.b_dtype = dtype;
    a.transB = trans_w != 0;
    a.Y = Y;
    a.y_dtype = y_dtype;
    a.N = N;
    a.num_w = num_weights;
    a.name = "segment_gemm";
    if (dtype == RGNN_BF16) {
      const size_t need = (size_t)num_weights * K * N * sizeof(bf16);
      RGNN_CHECK(scratch && scratch_bytes >= need, RGNN_ERR_INVALID_ARG, "scratch smaller than the workspace size");
      a.bt_scratch = scratch;
      a.tiles = p->tiles_tc;
      a.ntiles = p->n_tc;
      a.y_rows = p->rows;
      RGNN_CHECK(gemm_tc_supported(a), RGNN_ERR_UNSUPPORTED,
                 "bf16 segment GEMM: K must be a multiple of 64 (<= 8192), N one of 16/32/64/128 or a multiple of 256");
      gemm_tc(a, s);
    } else {
      RGNN_CHECK(K % 16 == 0 && (N == 16 || N == 32 || N == 64 || N == 128 || N == 256), RGNN_ERR_UNSUPPORTED,
                 "f32 segment GEMM: K must be a multiple of 16, N one of 16/32/64/128/256");
      a.tiles = p->tiles_simt;
      a.ntiles = p->n_simt;
      gemm_simt(a, s);
    }
  });
}

}  // extern "C"
