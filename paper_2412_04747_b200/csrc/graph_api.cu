// C-ABI graph entry points, RGCN edge norms and tile plans.
#include <algorithm>
#include <cstring>

#include "graph.cuh"

namespace rgnn {

void build_graph(rgnn_graph_s* g, const int32_t* src, const int32_t* dst, const int32_t* rel, int64_t E,
                 cudaStream_t s);

namespace {

// 1/c_{v,r} with c = |{e' in in(v) : rel e' = r}| (reading g1 'mean'): one value per CSR run of (dst, rel)
__global__ void k_norm_mean(int64_t UD, const int32_t* beg, const int32_t* cnt, float* csr_norm) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= UD) return;
  float v = 1.0f / (float)cnt[j];
  for (int32_t i = beg[j], e = beg[j] + cnt[j]; i < e; ++i) csr_norm[i] = v;
}

// 1/sqrt(d_out(src) d_in(dst)) (GCN A*)
__global__ void k_norm_sym(int64_t N, const int32_t* row_ptr, const int32_t* col_ptr, const int32_t* csr_src,
                           float* csr_norm) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= N) return;
  int32_t b = row_ptr[v], e = row_ptr[v + 1];
  float din = (float)(e - b);
  for (int32_t i = b; i < e; ++i) {
    int32_t u = csr_src[i];
    float dout = (float)(col_ptr[u + 1] - col_ptr[u]);
    csr_norm[i] = 1.0f / (sqrtf(dout) * sqrtf(din));
  }
}

__global__ void k_fill(int64_t n, float v, float* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = v;
}

__global__ void k_norm_custom(int64_t E, const int32_t* csr_eid, const int32_t* kept_eid, const float* custom,
                              float* csr_norm) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < E) csr_norm[i] = custom[kept_eid[csr_eid[i]]];
}

__global__ void k_gather_f(int64_t E, const int32_t* idx, const float* val, float* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < E) out[i] = val[idx[i]];
}

}  // namespace

void compute_norms(rgnn_graph_s* g, int kind, const float* custom, cudaStream_t s, float* csr_norm,
                   float* csc_norm) {
  const int TB = 256;
  const int64_t E = g->E;
  switch (kind) {
    case RGNN_NORM_MEAN:
      launch("norm_mean", k_norm_mean, dim3(ceil_div(g->UD, TB)), dim3(TB), 0, s, g->UD, g->dpair_csr_beg,
             g->dpair_cnt, csr_norm);
      break;
    case RGNN_NORM_SYM:
      launch("norm_sym", k_norm_sym, dim3(ceil_div(g->N, TB)), dim3(TB), 0, s, g->N, g->row_ptr,
             g->col_ptr_full ? g->col_ptr_full : g->col_ptr,
             g->csr_src, csr_norm);
      break;
    case RGNN_NORM_NONE:
      launch("norm_fill", k_fill, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, 1.0f, csr_norm);
      break;
    case RGNN_NORM_CUSTOM:
      RGNN_CHECK(custom != nullptr, RGNN_ERR_INVALID_ARG, "norm_kind CUSTOM needs weights.edge_norm");
      launch("norm_custom", k_norm_custom, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, g->csr_eid, g->kept_eid,
             custom, csr_norm);
      break;
    default:
      RGNN_FAIL(RGNN_ERR_INVALID_ARG, "unknown norm_kind");
  }
  launch("norm_to_csc", k_gather_f, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, g->csc2csr, csr_norm, csc_norm);
}

// Norms of the built-in kinds are cached in the graph; CUSTOM goes to the caller's buffers.
void graph_norms(rgnn_graph_s* g, int kind, const float* custom, cudaStream_t s, float** csr_norm,
                 float** csc_norm) {
  if (kind == RGNN_NORM_CUSTOM) {
    compute_norms(g, kind, custom, s, *csr_norm, *csc_norm);
    return;
  }
  auto it = g->norms.find(kind);
  if (it == g->norms.end()) {
    float* a = g->dev_f32(g->E, s);
    float* b = g->dev_f32(g->E, s);
    compute_norms(g, kind, nullptr, s, a, b);
    it = g->norms.emplace(kind, std::make_pair(a, b)).first;
  }
  *csr_norm = it->second.first;
  *csc_norm = it->second.second;
}

const Plan& get_plan(rgnn_graph_s* g, const std::string& key, const std::vector<int64_t>& seg_ptr,
                     const std::vector<int32_t>& w_of_seg, int rows, cudaStream_t s) {
  std::string k = key + "/" + std::to_string(rows);
  auto it = g->plans.find(k);
  if (it != g->plans.end()) return it->second;
  const int nseg = (int)seg_ptr.size() - 1;
  std::vector<Tile> tiles;
  std::vector<int32_t> ptr(1, 0), sw;
  for (int i = 0; i < nseg; ++i) {
    int32_t w = w_of_seg.empty() ? (int32_t)i : w_of_seg[i];
    for (int64_t r = seg_ptr[i]; w >= 0 && r < seg_ptr[i + 1]; r += rows)  // w < 0: a gap, no tiles
      tiles.push_back(Tile{(int32_t)r, (int32_t)std::min<int64_t>(r + rows, seg_ptr[i + 1]), w, (int32_t)i});
    ptr.push_back((int32_t)tiles.size());
    sw.push_back(w);
  }
  Plan p;
  p.count = (int32_t)tiles.size();
  p.nseg = nseg;
  // one device block: tiles | seg_tile_ptr | seg_w
  size_t tb = std::max<size_t>(1, tiles.size()) * sizeof(Tile);
  size_t pb = ptr.size() * sizeof(int32_t), wb = std::max<size_t>(1, sw.size()) * sizeof(int32_t);
  size_t pb_al = (pb + 15) & ~size_t(15);
  char* blk = reinterpret_cast<char*>(g->alloc.get(tb + pb_al + wb, s));
  g->owned.push_back(blk);
  g->owned_bytes += (int64_t)(tb + pb_al + wb);
  p.tiles = reinterpret_cast<Tile*>(blk);
  p.seg_tile_ptr = reinterpret_cast<int32_t*>(blk + tb);
  p.seg_w = reinterpret_cast<int32_t*>(blk + tb + pb_al);
  std::vector<char> host(tb + pb_al + wb, 0);
  if (!tiles.empty()) memcpy(host.data(), tiles.data(), tiles.size() * sizeof(Tile));
  memcpy(host.data() + tb, ptr.data(), pb);
  if (!sw.empty()) memcpy(host.data() + tb + pb_al, sw.data(), sw.size() * sizeof(int32_t));
  RGNN_CUDA(cudaMemcpyAsync(blk, host.data(), host.size(), cudaMemcpyHostToDevice, s));
  RGNN_CUDA(cudaStreamSynchronize(s));  // host staging goes out of scope; one-off per plan
  return g->plans.emplace(k, p).first->second;
}

}  // namespace rgnn

using namespace rgnn;

extern "C" {

rgnn_status rgnn_graph_build(int64_t num_nodes, int32_t num_node_types, const int64_t* node_type_ptr,
                             int32_t num_rels, int64_t num_edges, const int32_t* src, const int32_t* dst,
                             const int32_t* rel, int64_t dst_lo, int64_t dst_hi, rgnn_alloc_fn alloc,
                             rgnn_free_fn free_fn, void* alloc_ctx, void* stream, rgnn_graph_t* out) {
  rgnn_graph_opts opts{};
  opts.compact = 1;
  return rgnn_graph_build_opts(num_nodes, num_node_types, node_type_ptr, num_rels, num_edges, src, dst, rel, dst_lo,
                               dst_hi, &opts, alloc, free_fn, alloc_ctx, stream, out);
}

rgnn_status rgnn_graph_build_opts(int64_t num_nodes, int32_t num_node_types, const int64_t* node_type_ptr,
                                  int32_t num_rels, int64_t num_edges, const int32_t* src, const int32_t* dst,
                                  const int32_t* rel, int64_t dst_lo, int64_t dst_hi, const rgnn_graph_opts* opts,
                                  rgnn_alloc_fn alloc, rgnn_free_fn free_fn, void* alloc_ctx, void* stream,
                                  rgnn_graph_t* out) {
  return guarded([&] {
    RGNN_CHECK(opts != nullptr && (opts->compact == 0 || opts->compact == 1), RGNN_ERR_INVALID_ARG,
               "opts->compact must be 0 or 1");
    RGNN_CHECK(out != nullptr, RGNN_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    RGNN_CHECK(num_nodes >= 1 && num_node_types >= 1 && num_rels >= 1 && num_edges >= 0, RGNN_ERR_INVALID_ARG,
               "counts must be num_nodes>=1, num_node_types>=1, num_rels>=1, num_edges>=0");
    RGNN_CHECK(node_type_ptr != nullptr, RGNN_ERR_INVALID_ARG, "node_type_ptr is NULL");
    RGNN_CHECK(num_edges == 0 || (src && dst && rel), RGNN_ERR_INVALID_ARG, "src/dst/rel must be non-NULL");
    RGNN_CHECK((alloc == nullptr) == (free_fn == nullptr), RGNN_ERR_INVALID_ARG, "alloc and free_fn go together");
    RGNN_CHECK(num_edges < (int64_t(1) << 31) && num_nodes < (int64_t(1) << 31), RGNN_ERR_UNSUPPORTED,
               "num_edges and num_nodes must be < 2^31");
    RGNN_CHECK(0 <= dst_lo && dst_lo <= dst_hi && dst_hi <= num_nodes, RGNN_ERR_INVALID_ARG,
               "need 0 <= dst_lo <= dst_hi <= num_nodes");
    RGNN_CHECK(node_type_ptr[0] == 0 && node_type_ptr[num_node_types] == num_nodes, RGNN_ERR_INVALID_ARG,
               "node_type_ptr must start at 0 and end at num_nodes");
    for (int t = 0; t < num_node_types; ++t)
      RGNN_CHECK(node_type_ptr[t] <= node_type_ptr[t + 1], RGNN_ERR_INVALID_ARG, "node_type_ptr not monotone");
    auto* g = new rgnn_graph_s();
    g->alloc = Allocator{alloc, free_fn, alloc_ctx};
    g->N = num_nodes;
    g->T = num_node_types;
    g->R = num_rels;
    g->dst_lo = dst_lo;
    g->dst_hi = dst_hi;
    g->node_type_ptr.assign(node_type_ptr, node_type_ptr + num_node_types + 1);
    g->compact = opts->compact;
    try {
      build_graph(g, src, dst, rel, num_edges, static_cast<cudaStream_t>(stream));
    } catch (...) {
      rgnn_graph_destroy(g);
      throw;
    }
    *out = g;
  });
}

rgnn_status rgnn_graph_get_info(rgnn_graph_t g, rgnn_graph_info* o) {
  return guarded([&] {
    RGNN_CHECK(g && o, RGNN_ERR_INVALID_ARG, "NULL argument");
    o->num_nodes = g->N;
    o->num_edges = g->E;
    o->num_pairs = g->U;
    o->max_in_degree = g->max_in_deg;
    o->max_pair_degree = g->max_pair_deg;
    o->dst_lo = g->dst_lo;
    o->dst_hi = g->dst_hi;
    o->num_node_types = g->T;
    o->num_rels = g->R;
    o->device_bytes = g->owned_bytes;
    o->compaction_ratio = g->E == 0 ? 1.0 : (double)g->U / (double)g->E;
  });
}

static const int32_t* array_of(rgnn_graph_t g, rgnn_array w, int64_t* n) {
  switch (w) {
    case RGNN_ARR_ETYPE_PTR: *n = g->R + 1; return g->etype_ptr;
    case RGNN_ARR_ROW_PTR: *n = g->N + 1; return g->row_ptr;
    case RGNN_ARR_CSR_SRC: *n = g->E; return g->csr_src;
    case RGNN_ARR_CSR_REL: *n = g->E; return g->csr_rel;
    case RGNN_ARR_CSR_EID: *n = g->E; return g->csr_eid;
    case RGNN_ARR_COL_PTR: *n = g->N + 1; return g->col_ptr;
    case RGNN_ARR_CSC_DST: *n = g->E; return g->csc_dst;
    case RGNN_ARR_CSC_REL: *n = g->E; return g->csc_rel;
    case RGNN_ARR_CSC_EID: *n = g->E; return g->csc_eid;
    case RGNN_ARR_PAIR_REL_PTR: *n = g->R + 1; return g->pair_rel_ptr;
    case RGNN_ARR_PAIR_SRC: *n = g->U; return g->pair_src;
    case RGNN_ARR_EDGE_PAIR: *n = g->E; return g->edge_pair;
    case RGNN_ARR_CSR_PAIR: *n = g->E; return g->csr_pair;
    case RGNN_ARR_CSC_PAIR: *n = g->E; return g->csc_pair;
    default: RGNN_FAIL(RGNN_ERR_INVALID_ARG, "unknown rgnn_array");
  }
}

rgnn_status rgnn_graph_array_size(rgnn_graph_t g, rgnn_array which, int64_t* count) {
  return guarded([&] {
    RGNN_CHECK(g && count, RGNN_ERR_INVALID_ARG, "NULL argument");
    array_of(g, which, count);
  });
}

rgnn_status rgnn_graph_export(rgnn_graph_t g, rgnn_array which, void* dst_device, size_t bytes, void* stream) {
  return guarded([&] {
    RGNN_CHECK(g && dst_device, RGNN_ERR_INVALID_ARG, "NULL argument");
    int64_t n = 0;
    const int32_t* p = array_of(g, which, &n);
    RGNN_CHECK(bytes >= (size_t)n * sizeof(int32_t), RGNN_ERR_INVALID_ARG, "export buffer too small");
    if (n)
      RGNN_CUDA(cudaMemcpyAsync(dst_device, p, n * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                static_cast<cudaStream_t>(stream)));
  });
}

rgnn_status rgnn_graph_destroy(rgnn_graph_t g) {
  return guarded([&] {
    if (!g) return;
    cudaStream_t s = nullptr;
    for (void* p : g->owned) g->alloc.put(p, s);
    delete g;
  });
}

}  // extern "C"
