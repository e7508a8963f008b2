// A0 — graph build (C1 of §8(c)).
//
// From device COO (src, dst, rel) it builds, all on the GPU with stable radix
// sorts (CUB, CUDA toolkit) and flag/scan compaction:
//   etype_ptr, dst-CSR (key (dst, rel, src, eid)), src-CSC (key (src, rel, dst, eid)),
//   compact pairs = runs of (src, rel) in CSC order re-ranked by (rel, src)
//   ("one row per unique (edge type, source node) pair", §3.3.2),
//   edge_pair / csr_pair / csc_pair, the per-source pair list, the CSC->CSR map,
//   (rel, dst) runs for the RGAT destination-side gradient, and the (rel, src type)
//   sub-segments used by HGT's folded weights.
// Stability of the LSD radix sort makes the eid tie-break implicit: equal keys keep
// ascending edge order.  Host syncs: twice (after counting, after building).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>

#include "graph.cuh"

namespace rgnn {
namespace {

__global__ void k_validate(int64_t E, const int32_t* src, const int32_t* dst, const int32_t* rel, int64_t N,
                           int32_t R, int64_t dst_lo, int64_t dst_hi, unsigned long long* first_bad,
                           int32_t* keep_flag) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= E) return;
  int32_t s = src[e], d = dst[e], r = rel[e];
  bool ok = s >= 0 && s < N && d >= 0 && d < N && r >= 0 && r < R;
  if (!ok) atomicMin(first_bad, (unsigned long long)e);
  keep_flag[e] = ok && d >= dst_lo && d < dst_hi;
}

__global__ void k_gather3(int64_t E, const int32_t* idx, const int32_t* a, const int32_t* b, const int32_t* c,
                          int32_t* oa, int32_t* ob, int32_t* oc) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= E) return;
  int32_t j = idx[i];
  oa[i] = a[j]; ob[i] = b[j]; oc[i] = c[j];
}

__global__ void k_csr_single(int64_t E, const int32_t* csr_pair, const int32_t* pair_deg, uint8_t* single) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < E) single[i] = pair_deg[csr_pair[i]] == 1 ? 1 : 0;
}

__global__ void k_short_first(int64_t n, int4* items, const int32_t* idx) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int4 it = items[j];
  it.w = it.z > it.y ? -2 - idx[it.y] : -1;
  items[j] = it;
}

__global__ void k_iota(int64_t n, int32_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int32_t)i;
}

__global__ void k_key1(int64_t n, const int32_t* a, uint64_t* key) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) key[i] = (uint64_t)(uint32_t)a[i];
}

// key = (a << (wb + wc)) | (b << wc) | c
__global__ void k_make_key(int64_t E, const int32_t* a, const int32_t* b, const int32_t* c, int wb, int wc,
                           uint64_t* key) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= E) return;
  key[i] = ((uint64_t)(uint32_t)a[i] << (wb + wc)) | ((uint64_t)(uint32_t)b[i] << wc) | (uint64_t)(uint32_t)c[i];
}

__global__ void k_decode_key(int64_t E, const uint64_t* key, int wb, int wc, int32_t* a, int32_t* b, int32_t* c) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= E) return;
  uint64_t k = key[i];
  a[i] = (int32_t)(k >> (wb + wc));
  b[i] = (int32_t)((k >> wc) & ((1ull << wb) - 1));
  c[i] = (int32_t)(k & ((1ull << wc) - 1));
}

__global__ void k_histogram(int64_t E, const int32_t* v, int32_t* count) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < E) atomicAdd(&count[v[i]], 1);  // integer: order-independent result
}

// heads of runs of equal (a, b) in a sorted sequence (every position when `all`)
__global__ void k_run_heads(int64_t E, const int32_t* a, const int32_t* b, int32_t* flag, bool all) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= E) return;
  flag[i] = all || (i == 0) || a[i] != a[i - 1] || b[i] != b[i - 1];
}

__global__ void k_run_info(int64_t nruns, int64_t E, const int32_t* head_pos, const int32_t* a, const int32_t* b,
                           int nb_b, uint64_t* run_key, int32_t* run_len) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nruns) return;
  int32_t h = head_pos[j];
  int32_t nx = (j + 1 < nruns) ? head_pos[j + 1] : (int32_t)E;
  run_len[j] = nx - h;
  // run key sorted by (b, a): relation-major
  run_key[j] = ((uint64_t)(uint32_t)b[h] << nb_b) | (uint64_t)(uint32_t)a[h];
}

__global__ void k_scatter_rank(int64_t n, const int32_t* order, int32_t* rank_of) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < n) rank_of[order[p]] = (int32_t)p;
}

__global__ void k_pair_fields(int64_t n, const int32_t* order, const uint64_t* sorted_key, int nb,
                              const int32_t* head_pos, const int32_t* run_len, int32_t* node_of, int32_t* rel_of,
                              int32_t* beg, int32_t* deg) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  uint64_t k = sorted_key[p];
  node_of[p] = (int32_t)(k & ((1ull << nb) - 1));
  rel_of[p] = (int32_t)(k >> nb);
  int32_t j = order[p];
  beg[p] = head_pos[j];
  deg[p] = run_len[j];
}

// position -> run index (inclusive scan of heads - 1) -> pair rank
__global__ void k_pos_pair(int64_t E, const int32_t* run_incl, const int32_t* rank_of_run, int32_t* pos_pair) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < E) pos_pair[i] = rank_of_run[run_incl[i] - 1];
}

__global__ void k_scatter(int64_t E, const int32_t* idx, const int32_t* val, int32_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < E) out[idx[i]] = val[i];
}
__global__ void k_scatter_iota(int64_t E, const int32_t* idx, int32_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < E) out[idx[i]] = (int32_t)i;
}
__global__ void k_gather(int64_t E, const int32_t* idx, const int32_t* val, int32_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < E) out[i] = val[idx[i]];
}

__global__ void k_max_diff(int64_t n, const int32_t* ptr, unsigned long long* mx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) atomicMax(mx, (unsigned long long)(ptr[i + 1] - ptr[i]));
}
__global__ void k_max_val(int64_t n, const int32_t* v, unsigned long long* mx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) atomicMax(mx, (unsigned long long)v[i]);
}

// first pair index whose (rel, src) >= (r, node_type_ptr[t]) for every (r, t) and the end
__global__ void k_rt_bounds(int32_t R, int32_t T, const int64_t* ntp, int nb, const uint64_t* sorted_key, int64_t U,
                            int32_t* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > R * T) return;
  if (i == R * T) { out[i] = (int32_t)U; return; }
  int r = i / T, t = i % T;
  // addition, not OR: ntp[t] may equal N = 1 << nb (empty trailing type) and must carry into r + 1
  uint64_t target = ((uint64_t)r << nb) + (uint64_t)ntp[t];
  int64_t lo = 0, hi = U;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (sorted_key[mid] < target) lo = mid + 1; else hi = mid;
  }
  out[i] = (int32_t)lo;
}

int bits_for(int64_t n) {
  int b = 0;
  while ((int64_t(1) << b) < n) ++b;
  return std::max(b, 1);
}

const int TB = 256;

struct Tmp {  // temporaries freed at the end of the build
  const Allocator& a;
  cudaStream_t s;
  std::vector<void*> ptrs;
  Tmp(const Allocator& al, cudaStream_t st) : a(al), s(st) {}
  template <class T>
  T* get(size_t n) {
    void* p = a.get((n ? n : 1) * sizeof(T), s);
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~Tmp() {
    for (void* p : ptrs) a.put(p, s);
  }
};

void radix_pairs(Tmp& tmp, const uint64_t* kin, uint64_t* kout, const int32_t* vin, int32_t* vout, int64_t n,
                 int end_bit, cudaStream_t s) {
  if (n == 0) return;
  size_t bytes = 0;
  RGNN_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)n, 0, end_bit, s));
  void* t = tmp.get<char>(bytes);
  RGNN_CUDA(cub::DeviceRadixSort::SortPairs(t, bytes, kin, kout, vin, vout, (int)n, 0, end_bit, s));
  count_launch();
}

void excl_scan_counts(Tmp& tmp, int32_t* counts, int32_t* out, int64_t n, cudaStream_t s) {
  // out[0..n] = exclusive scan of counts[0..n-1] with out[n] = total
  size_t bytes = 0;
  RGNN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, counts, out, (int)(n + 1), s));
  void* t = tmp.get<char>(bytes);
  RGNN_CUDA(cub::DeviceScan::ExclusiveSum(t, bytes, counts, out, (int)(n + 1), s));
  count_launch();
}

void incl_scan(Tmp& tmp, const int32_t* in, int32_t* out, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  size_t bytes = 0;
  RGNN_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, (int)n, s));
  void* t = tmp.get<char>(bytes);
  RGNN_CUDA(cub::DeviceScan::InclusiveSum(t, bytes, in, out, (int)n, s));
  count_launch();
}

// compact positions i with flag[i] != 0 (in order); returns count through d_num
void select_flagged(Tmp& tmp, const int32_t* flags, int32_t* out, int32_t* d_num, int64_t n, cudaStream_t s) {
  if (n == 0) {
    RGNN_CUDA(cudaMemsetAsync(d_num, 0, sizeof(int32_t), s));
    return;
  }
  cub::CountingInputIterator<int32_t> it(0);
  size_t bytes = 0;
  RGNN_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, out, d_num, (int)n, s));
  void* t = tmp.get<char>(bytes);
  RGNN_CUDA(cub::DeviceSelect::Flagged(t, bytes, it, flags, out, d_num, (int)n, s));
  count_launch();
}

// histogram of v[0..n) into [0, nbins) and exclusive prefix (nbins+1 entries)
void hist_prefix(Tmp& tmp, const int32_t* v, int64_t n, int64_t nbins, int32_t* ptr_out, cudaStream_t s) {
  int32_t* cnt = tmp.get<int32_t>(nbins + 1);
  RGNN_CUDA(cudaMemsetAsync(cnt, 0, (nbins + 1) * sizeof(int32_t), s));
  launch("graph_histogram", k_histogram, dim3(ceil_div(n, TB)), dim3(TB), 0, s, n, v, cnt);
  excl_scan_counts(tmp, cnt, ptr_out, nbins, s);
}

}  // namespace

// Edge-balanced work list (graph.cuh WorkPlan) from per-id (begin, degree); one-off host pass.
void build_work_plan(rgnn_graph_s* g, const std::vector<int32_t>& beg, const std::vector<int32_t>& deg,
                     WorkPlan& wp, cudaStream_t s, int64_t id_lo = 0, int64_t id_hi = -1) {
  std::vector<int4> heavy, medium, light, splits;
  int64_t slots = 0;
  if (id_hi < 0) id_hi = (int64_t)beg.size();
  for (size_t id = (size_t)id_lo; id < (size_t)id_hi; ++id) {
    int32_t b = beg[id], e = beg[id] + deg[id];
    if (deg[id] > SPLIT_THRESH) {
      int32_t n = 0;
      for (int32_t c = b; c < e; c += SPLIT_CHUNK, ++n)
        heavy.push_back(make_int4((int)id, c, std::min(e, c + SPLIT_CHUNK), (int)(slots + n)));
      splits.push_back(make_int4((int)id, (int)slots, n, 0));
      slots += n;
    } else if (deg[id] > LIGHT_MAX) {
      medium.push_back(make_int4((int)id, b, e, -1));
    } else {
      light.push_back(make_int4((int)id, b, e, -1));
    }
  }
  // longest first within each class: medium rows start early (shorter tail), and neighbouring
  // light items (one warp = 32 / LPR of them) have similar lengths (little idle lane time)
  auto longer = [](const int4& a, const int4& b) { return (a.z - a.y) > (b.z - b.y); };
  std::stable_sort(medium.begin(), medium.end(), longer);
  std::stable_sort(light.begin(), light.end(), longer);
  wp.n_warp = (int64_t)(heavy.size() + medium.size());
  heavy.insert(heavy.end(), medium.begin(), medium.end());
  heavy.insert(heavy.end(), light.begin(), light.end());
  wp.n_items = (int64_t)heavy.size();
  wp.n_short = wp.n_items;  // light items are sorted longest first: the short ones are a suffix
  while (wp.n_short > wp.n_warp && heavy[wp.n_short - 1].z - heavy[wp.n_short - 1].y <= SHORT_MAX) --wp.n_short;
  wp.n_multi = wp.n_items;
  while (wp.n_multi > wp.n_warp && heavy[wp.n_multi - 1].z - heavy[wp.n_multi - 1].y <= 1) --wp.n_multi;
  wp.n_split = (int64_t)splits.size();
  wp.n_slots = slots;
  wp.items = reinterpret_cast<int4*>(g->dev_i32(4 * std::max<int64_t>(wp.n_items, 1), s));
  wp.splits = reinterpret_cast<int4*>(g->dev_i32(4 * std::max<int64_t>(wp.n_split, 1), s));
  if (wp.n_items)
    RGNN_CUDA(cudaMemcpyAsync(wp.items, heavy.data(), heavy.size() * sizeof(int4), cudaMemcpyHostToDevice, s));
  if (wp.n_split)
    RGNN_CUDA(cudaMemcpyAsync(wp.splits, splits.data(), splits.size() * sizeof(int4), cudaMemcpyHostToDevice, s));
  RGNN_CUDA(cudaStreamSynchronize(s));  // host staging goes out of scope
}

// Edge-stream chunks of the pair pass (graph.cuh WorkPlan::chunks) from the pairs in CSC order.
void build_stream_chunks(rgnn_graph_s* g, const std::vector<int32_t>& pb, const std::vector<int32_t>& pd,
                         WorkPlan& wp, cudaStream_t s) {
  const int64_t U = g->U;
  std::vector<int32_t> order(U);  // pairs by (src, rel) = CSC order
  if (U) RGNN_CUDA(cudaMemcpyAsync(order.data(), g->src_pairs, U * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  std::vector<int4> heavy(std::max<int64_t>(wp.n_warp, 0));
  if (wp.n_warp)
    RGNN_CUDA(cudaMemcpyAsync(heavy.data(), wp.items, wp.n_warp * sizeof(int4), cudaMemcpyDeviceToHost, s));
  RGNN_CUDA(cudaStreamSynchronize(s));
  for (int multi = 0; multi < 2; ++multi) {
    std::vector<int4> ch;
    for (const int4& it : heavy)
      if (it.w >= 0) ch.push_back(make_int4(it.y, it.z, it.w, 0));  // split chunks of heavy pairs (slots)
    int32_t cb = -1, ce = -1;
    auto close = [&] {
      if (cb >= 0 && ce > cb) ch.push_back(make_int4(cb, ce, -1, 0));
      cb = ce = -1;
    };
    for (int64_t j = 0; j < U; ++j) {
      const int32_t p = order[j], b = pb[p], n = pd[p];
      if (n > SPLIT_THRESH || (multi && n == 1)) {  // heavy (above) or resolved elsewhere: a gap
        close();
        continue;
      }
      if (n > STREAM_CHUNK) {
        close();
        ch.push_back(make_int4(b, b + n, -1, 0));
        continue;
      }
      if (cb < 0) cb = b;
      ce = b + n;
      if (ce - cb >= STREAM_CHUNK) close();
    }
    close();
    std::stable_sort(ch.begin() + (int64_t)std::count_if(heavy.begin(), heavy.end(), [](const int4& it) { return it.w >= 0; }),
                     ch.end(), [](const int4& a, const int4& b) { return a.y - a.x > b.y - b.x; });
    int4*& dst = multi ? wp.chunks_multi : wp.chunks;
    (multi ? wp.n_chunks_multi : wp.n_chunks) = (int64_t)ch.size();
    dst = reinterpret_cast<int4*>(g->dev_i32(4 * std::max<size_t>(ch.size(), 1), s));
    if (!ch.empty()) RGNN_CUDA(cudaMemcpyAsync(dst, ch.data(), ch.size() * sizeof(int4), cudaMemcpyHostToDevice, s));
    RGNN_CUDA(cudaStreamSynchronize(s));
  }
}

// Chunks of the long (rel, dst) runs (graph.cuh dpair_chunks / dpair_splits); one-off host pass.
void build_dpair_splits(rgnn_graph_s* g, cudaStream_t s) {
  const int64_t UD = g->UD;
  std::vector<int32_t> db(UD), dc(UD);
  if (UD) {
    RGNN_CUDA(cudaMemcpyAsync(db.data(), g->dpair_csr_beg, UD * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RGNN_CUDA(cudaMemcpyAsync(dc.data(), g->dpair_cnt, UD * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RGNN_CUDA(cudaStreamSynchronize(s));
  }
  std::vector<int4> chunks, splits;
  for (int64_t j = 0; j < UD; ++j) {
    if (dc[j] <= SPLIT_THRESH) continue;
    const int32_t b = db[j], e = db[j] + dc[j];
    int32_t n = 0;
    for (int32_t c = b; c < e; c += SPLIT_CHUNK, ++n)
      chunks.push_back(make_int4((int)j, c, std::min(e, c + SPLIT_CHUNK), (int)chunks.size()));
    splits.push_back(make_int4((int)j, (int)(chunks.size() - n), n, 0));
  }
  g->n_dpair_chunks = (int64_t)chunks.size();
  g->n_dpair_splits = (int64_t)splits.size();
  g->dpair_chunks = reinterpret_cast<int4*>(g->dev_i32(4 * std::max<size_t>(chunks.size(), 1), s));
  g->dpair_splits = reinterpret_cast<int4*>(g->dev_i32(4 * std::max<size_t>(splits.size(), 1), s));
  if (!chunks.empty())
    RGNN_CUDA(cudaMemcpyAsync(g->dpair_chunks, chunks.data(), chunks.size() * sizeof(int4), cudaMemcpyHostToDevice, s));
  if (!splits.empty())
    RGNN_CUDA(cudaMemcpyAsync(g->dpair_splits, splits.data(), splits.size() * sizeof(int4), cudaMemcpyHostToDevice, s));
  RGNN_CUDA(cudaStreamSynchronize(s));
}

void build_work_plans(rgnn_graph_s* g, cudaStream_t s) {
  const int64_t N = g->N, U = g->U;
  std::vector<int32_t> rp(N + 1), pb(U), pd(U);
  RGNN_CUDA(cudaMemcpyAsync(rp.data(), g->row_ptr, (N + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  if (U) {
    RGNN_CUDA(cudaMemcpyAsync(pb.data(), g->pair_csc_beg, U * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RGNN_CUDA(cudaMemcpyAsync(pd.data(), g->pair_deg, U * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  }
  RGNN_CUDA(cudaStreamSynchronize(s));
  // destination rows: only the owned range [dst_lo, dst_hi) (a partitioned build has no in-edges
  // elsewhere; its traversals must not touch the other ranks' output rows)
  const int64_t lo = g->dst_lo, hi = g->dst_hi;
  std::vector<int32_t> rb(N, 0), rd(N, 0);
  for (int64_t v = lo; v < hi; ++v) {
    rb[v] = rp[v];
    rd[v] = rp[v + 1] - rp[v];
  }
  build_work_plan(g, rb, rd, g->rows, s, lo, hi);
  build_work_plan(g, pb, pd, g->pairs, s);
  build_dpair_splits(g, s);
  build_stream_chunks(g, pb, pd, g->pairs, s);
  // short items carry their first edge's gather index (rows: csr_pair, pairs: csc_dst) as
  // w = -2 - index (negative: never a partial slot), saving the short kernels one dependent load
  const int64_t nr = g->rows.n_items - g->rows.n_short, np = g->pairs.n_items - g->pairs.n_short;
  launch("graph_short_first", k_short_first, dim3(std::max<unsigned>(ceil_div(nr, TB), 1)), dim3(TB), 0, s, nr,
         g->rows.items + g->rows.n_short, (const int32_t*)g->csr_pair);
  launch("graph_short_first", k_short_first, dim3(std::max<unsigned>(ceil_div(np, TB), 1)), dim3(TB), 0, s, np,
         g->pairs.items + g->pairs.n_short, (const int32_t*)g->csc_dst);
}

// The (rel, dst) pairs grouped by destination (ascending rel within a destination; stable sort of
// the (rel, dst)-ordered list by dst), built on first use by the RGAT path without reordering.
void ensure_dst_dpairs(rgnn_graph_s* g, cudaStream_t s) {
  if (g->dst_dpair_ptr) return;
  const int64_t UD = g->UD, N = g->N;
  Tmp tmp(g->alloc, s);
  int32_t* ptr = g->dev_i32(N + 1, s);
  int32_t* list = g->dev_i32(UD, s);
  hist_prefix(tmp, g->dpair_dst, UD, N, ptr, s);
  if (UD > 0) {
    uint64_t* kin = tmp.get<uint64_t>(UD);
    uint64_t* kout = tmp.get<uint64_t>(UD);
    int32_t* vin = tmp.get<int32_t>(UD);
    launch("graph_key", k_key1, dim3(ceil_div(UD, TB)), dim3(TB), 0, s, UD, (const int32_t*)g->dpair_dst, kin);
    launch("graph_iota", k_iota, dim3(ceil_div(UD, TB)), dim3(TB), 0, s, UD, vin);
    radix_pairs(tmp, kin, kout, vin, list, UD, bits_for(N), s);
  }
  RGNN_CUDA(cudaStreamSynchronize(s));  // temporaries are released when `tmp` goes out of scope
  g->dst_dpair_ptr = ptr;
  g->dst_dpairs = list;
}

// Active (relation, source type) combinations of the pairs (HGT A2 folds one weight per active
// combination only; with R*T combinations and one source type per relation most are empty).
void build_active_combos(rgnn_graph_s* g, cudaStream_t s) {
  const int R = g->R, T = g->T;
  std::vector<int32_t> act_rt, t_ptr(T + 1, 0), t_list, r_ptr(R + 1, 0);
  g->act_of_rt_h.assign((size_t)R * T, 0);
  for (int rt = 0; rt < R * T; ++rt)
    if (g->pair_rt_ptr_h[rt + 1] > g->pair_rt_ptr_h[rt]) {
      g->act_of_rt_h[rt] = (int32_t)act_rt.size();
      act_rt.push_back(rt);
      ++t_ptr[rt % T + 1];
      ++r_ptr[rt / T + 1];
    }
  for (int t = 0; t < T; ++t) t_ptr[t + 1] += t_ptr[t];
  for (int r = 0; r < R; ++r) r_ptr[r + 1] += r_ptr[r];
  t_list.resize(act_rt.size());
  std::vector<int32_t> fill(t_ptr.begin(), t_ptr.end() - 1);
  for (size_t a = 0; a < act_rt.size(); ++a) t_list[fill[act_rt[a] % T]++] = (int32_t)a;
  g->n_act = (int32_t)act_rt.size();
  const size_t na = std::max<size_t>(act_rt.size(), 1);
  std::vector<int32_t> host(2 * na + (T + 1) + (R + 1), 0);
  std::copy(act_rt.begin(), act_rt.end(), host.begin());
  std::copy(t_ptr.begin(), t_ptr.end(), host.begin() + na);
  std::copy(t_list.begin(), t_list.end(), host.begin() + na + T + 1);
  std::copy(r_ptr.begin(), r_ptr.end(), host.begin() + 2 * na + T + 1);
  int32_t* d = g->dev_i32(host.size(), s);
  g->act_rt = d;
  g->t_act_ptr = d + na;
  g->t_act = d + na + T + 1;
  g->r_act_ptr = d + 2 * na + T + 1;
  RGNN_CUDA(cudaMemcpyAsync(d, host.data(), host.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  RGNN_CUDA(cudaStreamSynchronize(s));  // `host` goes out of scope; one-off per graph
}

void build_graph(rgnn_graph_s* g, const int32_t* src_in, const int32_t* dst_in, const int32_t* rel_in,
                 int64_t E_in, cudaStream_t s) {
  const int64_t N = g->N;
  const int32_t R = g->R, T = g->T;
  Tmp tmp(g->alloc, s);

  // ---- validate + filter to the owned destination range
  unsigned long long* d_stats = tmp.get<unsigned long long>(4);
  unsigned long long init[4] = {~0ull, 0, 0, 0};
  RGNN_CUDA(cudaMemcpyAsync(d_stats, init, sizeof(init), cudaMemcpyHostToDevice, s));
  int32_t* keep = tmp.get<int32_t>(E_in);
  launch("graph_validate", k_validate, dim3(ceil_div(E_in, TB)), dim3(TB), 0, s, E_in, src_in, dst_in, rel_in, N, R,
         g->dst_lo, g->dst_hi, d_stats, keep);
  int32_t* kept = tmp.get<int32_t>(E_in);
  int32_t* d_num = tmp.get<int32_t>(4);
  select_flagged(tmp, keep, kept, d_num, E_in, s);
  unsigned long long h_bad = 0;
  int32_t h_kept = 0;
  RGNN_CUDA(cudaMemcpyAsync(&h_bad, d_stats, sizeof(h_bad), cudaMemcpyDeviceToHost, s));
  RGNN_CUDA(cudaMemcpyAsync(&h_kept, d_num, sizeof(h_kept), cudaMemcpyDeviceToHost, s));
  RGNN_CUDA(cudaStreamSynchronize(s));
  if (h_bad != ~0ull)
    RGNN_FAIL(RGNN_ERR_OUT_OF_RANGE, "node or relation id out of range at edge " + std::to_string(h_bad));
  const int64_t E = h_kept;
  g->E = E;
  // GCN 'sym' norms need every source's out-degree over the whole graph, not over
  // the kept (owned-destination) edges only
  if (g->dst_lo != 0 || g->dst_hi != N) {
    g->col_ptr_full = g->dev_i32(N + 1, s);
    hist_prefix(tmp, src_in, E_in, N, g->col_ptr_full, s);
  }

  int32_t* src = tmp.get<int32_t>(E);
  int32_t* dst = tmp.get<int32_t>(E);
  int32_t* rel = tmp.get<int32_t>(E);
  g->kept_eid = g->dev_i32(E, s);
  RGNN_CUDA(cudaMemcpyAsync(g->kept_eid, kept, E * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  launch("graph_gather", k_gather3, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, kept, src_in, dst_in, rel_in, src, dst,
         rel);

  const int nb = bits_for(N), rb = bits_for(R);
  g->nb = nb;
  g->rb = rb;
  RGNN_CHECK(2 * nb + rb <= 64, RGNN_ERR_UNSUPPORTED, "sort key wider than 64 bits (N or R too large)");

  int32_t* eid = tmp.get<int32_t>(E);
  launch("graph_iota", k_iota, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, eid);
  uint64_t* key = tmp.get<uint64_t>(E);
  uint64_t* key_sorted = tmp.get<uint64_t>(E);

  // ---- etype_ptr
  g->etype_ptr = g->dev_i32(R + 1, s);
  hist_prefix(tmp, rel, E, R, g->etype_ptr, s);

  // ---- dst-CSR: key (dst, rel, src), stable => eid ascending among equals
  g->csr_src = g->dev_i32(E, s);
  g->csr_rel = g->dev_i32(E, s);
  g->csr_eid = g->dev_i32(E, s);
  g->row_ptr = g->dev_i32(N + 1, s);
  int32_t* csr_dst = tmp.get<int32_t>(E);
  launch("graph_key", k_make_key, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, dst, rel, src, rb, nb, key);
  radix_pairs(tmp, key, key_sorted, eid, g->csr_eid, E, 2 * nb + rb, s);
  launch("graph_decode", k_decode_key, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, key_sorted, rb, nb, csr_dst,
         g->csr_rel, g->csr_src);
  hist_prefix(tmp, dst, E, N, g->row_ptr, s);

  // ---- src-CSC: key (src, rel, dst)
  g->csc_dst = g->dev_i32(E, s);
  g->csc_rel = g->dev_i32(E, s);
  g->csc_eid = g->dev_i32(E, s);
  g->col_ptr = g->dev_i32(N + 1, s);
  int32_t* csc_src = tmp.get<int32_t>(E);
  launch("graph_key", k_make_key, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, src, rel, dst, rb, nb, key);
  radix_pairs(tmp, key, key_sorted, eid, g->csc_eid, E, 2 * nb + rb, s);
  launch("graph_decode", k_decode_key, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, key_sorted, rb, nb, csc_src,
         g->csc_rel, g->csc_dst);
  hist_prefix(tmp, src, E, N, g->col_ptr, s);

  // ---- runs of (src, rel) in CSC order = compact pairs; runs of (dst, rel) in CSR order = dst pairs
  int32_t* flag = tmp.get<int32_t>(E);
  int32_t* head_pos = tmp.get<int32_t>(E);
  int32_t* dflag = tmp.get<int32_t>(E);
  int32_t* dhead_pos = tmp.get<int32_t>(E);
  // compact materialization: one pair per run of equal (src, rel); vanilla: one "pair" per edge
  launch("graph_heads", k_run_heads, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, csc_src, g->csc_rel, flag,
         !g->compact);
  select_flagged(tmp, flag, head_pos, d_num, E, s);
  launch("graph_heads", k_run_heads, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, csr_dst, g->csr_rel, dflag, false);
  select_flagged(tmp, dflag, dhead_pos, d_num + 1, E, s);
  int32_t h_counts[2] = {0, 0};
  RGNN_CUDA(cudaMemcpyAsync(h_counts, d_num, sizeof(h_counts), cudaMemcpyDeviceToHost, s));
  RGNN_CUDA(cudaStreamSynchronize(s));
  const int64_t U = h_counts[0], UD = h_counts[1];
  g->U = U;
  g->UD = UD;

  // pairs: sort runs by (rel, src)
  uint64_t* rkey = tmp.get<uint64_t>(U);
  uint64_t* rkey_sorted = tmp.get<uint64_t>(U);
  int32_t* rlen = tmp.get<int32_t>(U);
  int32_t* ridx = tmp.get<int32_t>(U);
  int32_t* order = tmp.get<int32_t>(U);
  int32_t* rank_of_run = tmp.get<int32_t>(U);
  int32_t* pair_rel = tmp.get<int32_t>(U);
  launch("graph_runs", k_run_info, dim3(ceil_div(U, TB)), dim3(TB), 0, s, U, E, head_pos, csc_src, g->csc_rel, nb,
         rkey, rlen);
  launch("graph_iota", k_iota, dim3(ceil_div(U, TB)), dim3(TB), 0, s, U, ridx);
  radix_pairs(tmp, rkey, rkey_sorted, ridx, order, U, nb + rb, s);
  launch("graph_rank", k_scatter_rank, dim3(ceil_div(U, TB)), dim3(TB), 0, s, U, order, rank_of_run);
  g->pair_src = g->dev_i32(U, s);
  g->pair_csc_beg = g->dev_i32(U, s);
  g->pair_deg = g->dev_i32(U, s);
  launch("graph_pairs", k_pair_fields, dim3(ceil_div(U, TB)), dim3(TB), 0, s, U, order, rkey_sorted, nb, head_pos,
         rlen, g->pair_src, pair_rel, g->pair_csc_beg, g->pair_deg);
  g->pair_rel_ptr = g->dev_i32(R + 1, s);
  hist_prefix(tmp, pair_rel, U, R, g->pair_rel_ptr, s);
  // per-source pair list: heads in CSC order are the pairs ordered by (src, rel)
  g->src_pairs = g->dev_i32(U, s);
  RGNN_CUDA(cudaMemcpyAsync(g->src_pairs, rank_of_run, U * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  g->src_pair_ptr = g->dev_i32(N + 1, s);
  hist_prefix(tmp, g->pair_src, U, N, g->src_pair_ptr, s);
  // csc_pair, edge_pair, csr_pair
  int32_t* run_incl = tmp.get<int32_t>(E);
  incl_scan(tmp, flag, run_incl, E, s);
  g->csc_pair = g->dev_i32(E, s);
  g->edge_pair = g->dev_i32(E, s);
  g->csr_pair = g->dev_i32(E, s);
  launch("graph_pos_pair", k_pos_pair, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, run_incl, rank_of_run, g->csc_pair);
  launch("graph_scatter", k_scatter, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, g->csc_eid, g->csc_pair, g->edge_pair);
  launch("graph_gather1", k_gather, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, g->csr_eid, g->edge_pair, g->csr_pair);
  g->csr_single = reinterpret_cast<uint8_t*>(g->dev_i32((E + 3) / 4, s));
  launch("graph_single", k_csr_single, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, (const int32_t*)g->csr_pair,
         (const int32_t*)g->pair_deg, g->csr_single);
  // csc2csr
  int32_t* csr_pos_of_eid = tmp.get<int32_t>(E);
  g->csc2csr = g->dev_i32(E, s);
  launch("graph_scatter_iota", k_scatter_iota, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, g->csr_eid, csr_pos_of_eid);
  launch("graph_gather1", k_gather, dim3(ceil_div(E, TB)), dim3(TB), 0, s, E, g->csc_eid, csr_pos_of_eid, g->csc2csr);

  // (rel, dst) pairs from CSR runs
  uint64_t* dkey = tmp.get<uint64_t>(UD);
  uint64_t* dkey_sorted = tmp.get<uint64_t>(UD);
  int32_t* dlen = tmp.get<int32_t>(UD);
  int32_t* didx = tmp.get<int32_t>(UD);
  int32_t* dorder = tmp.get<int32_t>(UD);
  int32_t* dpair_rel = tmp.get<int32_t>(UD);
  launch("graph_runs", k_run_info, dim3(ceil_div(UD, TB)), dim3(TB), 0, s, UD, E, dhead_pos, csr_dst, g->csr_rel, nb,
         dkey, dlen);
  launch("graph_iota", k_iota, dim3(ceil_div(UD, TB)), dim3(TB), 0, s, UD, didx);
  radix_pairs(tmp, dkey, dkey_sorted, didx, dorder, UD, nb + rb, s);
  g->dpair_dst = g->dev_i32(UD, s);
  g->dpair_csr_beg = g->dev_i32(UD, s);
  g->dpair_cnt = g->dev_i32(UD, s);
  launch("graph_pairs", k_pair_fields, dim3(ceil_div(UD, TB)), dim3(TB), 0, s, UD, dorder, dkey_sorted, nb, dhead_pos,
         dlen, g->dpair_dst, dpair_rel, g->dpair_csr_beg, g->dpair_cnt);
  int32_t* dpair_rel_ptr = tmp.get<int32_t>(R + 1);
  hist_prefix(tmp, dpair_rel, UD, R, dpair_rel_ptr, s);

  // (rel, src type) sub-segments of the pairs
  int64_t* d_ntp = tmp.get<int64_t>(T + 1);
  RGNN_CUDA(cudaMemcpyAsync(d_ntp, g->node_type_ptr.data(), (T + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  int32_t* rt = g->pair_rt_ptr = g->dev_i32((int64_t)R * T + 1, s);
  launch("graph_rt_bounds", k_rt_bounds, dim3(ceil_div((int64_t)R * T + 1, TB)), dim3(TB), 0, s, R, T, d_ntp, nb,
         rkey_sorted, U, rt);

  // stats
  launch("graph_maxdeg", k_max_diff, dim3(ceil_div(N, TB)), dim3(TB), 0, s, N, g->row_ptr, d_stats + 1);
  launch("graph_maxdeg", k_max_val, dim3(ceil_div(U, TB)), dim3(TB), 0, s, U, g->pair_deg, d_stats + 2);
  unsigned long long h_stats[4];
  g->pair_rel_ptr_h.resize(R + 1);
  g->dpair_rel_ptr_h.resize(R + 1);
  g->pair_rt_ptr_h.resize((size_t)R * T + 1);
  RGNN_CUDA(cudaMemcpyAsync(h_stats, d_stats, sizeof(h_stats), cudaMemcpyDeviceToHost, s));
  RGNN_CUDA(cudaMemcpyAsync(g->pair_rel_ptr_h.data(), g->pair_rel_ptr, (R + 1) * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, s));
  RGNN_CUDA(cudaMemcpyAsync(g->dpair_rel_ptr_h.data(), dpair_rel_ptr, (R + 1) * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, s));
  RGNN_CUDA(cudaMemcpyAsync(g->pair_rt_ptr_h.data(), rt, ((size_t)R * T + 1) * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, s));
  RGNN_CUDA(cudaStreamSynchronize(s));
  g->max_in_deg = (int64_t)h_stats[1];
  g->max_pair_deg = (int64_t)h_stats[2];
  build_active_combos(g, s);
  build_work_plans(g, s);
}

}  // namespace rgnn
