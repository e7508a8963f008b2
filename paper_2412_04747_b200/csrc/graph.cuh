// Internal layout of a built graph (rgnn_graph_t).  See DESIGN.md "Data layout in HBM".
#pragma once

#include <map>
#include <string>
#include <vector>

#include "common.cuh"

namespace rgnn {

// Work classes of destination rows and compact pairs (by their number of edges):
constexpr int SPLIT_THRESH = 1024;  // heavy: more edges than this -> chunks of SPLIT_CHUNK, one warp each,
constexpr int SPLIT_CHUNK = 512;    //        partial states merged afterwards
#ifndef RGNN_LIGHT_MAX
#define RGNN_LIGHT_MAX 64
#endif
constexpr int LIGHT_MAX = RGNN_LIGHT_MAX;  // light: at most this many edges -> one lane group each; else one warp
constexpr int SHORT_MAX = 4;        // short: light items with at most this many edges (a suffix of the sorted
                                    //        light list) -> KI items per lane group, gathered together

// Edge-balanced work list over "ids" (destination rows or pairs) whose edges are the
// contiguous range [begin, begin + deg) of the CSR (rows) or CSC (pairs).
struct WorkPlan {
  int4* items = nullptr;   // (id, edge begin, edge end, partial slot or -1)
  int64_t n_warp = 0;      // items [0, n_warp): heavy chunks then medium ids, one warp per item
  int64_t n_items = 0;     // items [n_warp, n_items): light ids, one lane group per item
  int64_t n_short = 0;     // items [n_short, n_items): short light ids (<= SHORT_MAX edges; n_warp <= n_short)
  int64_t n_multi = 0;     // items [n_multi, n_items) have exactly one edge (a suffix of the short ones)
  int4* splits = nullptr;  // (id, first slot, number of slots, 0) for every heavy id
  int64_t n_split = 0;
  int64_t n_slots = 0;
  // Edge-stream chunks (pairs only; the gather-ring kernels): contiguous CSC ranges (begin, end,
  // slot, 0) that start and end at id boundaries, about STREAM_CHUNK edges each (an id longer than
  // that alone; heavy ids as their split chunks with slots), longest first.  `_multi` leaves out
  // the single-edge ids (resolved by the destination-major pass when single_in_dst).
  int4* chunks = nullptr;
  int64_t n_chunks = 0;
  int4* chunks_multi = nullptr;
  int64_t n_chunks_multi = 0;
};
#ifndef RGNN_STREAM_CHUNK
#define RGNN_STREAM_CHUNK 48
#endif
constexpr int STREAM_CHUNK = RGNN_STREAM_CHUNK;

// A contiguous row range [row0, row1) of one segment (weight index w).
struct Tile {
  int32_t row0, row1, w, pad;
};

struct Plan {                      // cached per (segmentation, rows-per-tile)
  Tile* tiles = nullptr;           // device [count]; pad = segment id
  int32_t count = 0;
  int32_t nseg = 0;
  int32_t* seg_tile_ptr = nullptr;  // device [nseg+1]: tiles of segment i are [ptr[i], ptr[i+1])
  int32_t* seg_w = nullptr;         // device [nseg]: weight index of segment i
};

}  // namespace rgnn

struct rgnn_graph_s {
  rgnn::Allocator alloc;
  int64_t N = 0, E = 0, U = 0, UD = 0;  // nodes, kept edges, (rel,src) pairs, (rel,dst) pairs
  int32_t T = 0, R = 0;
  int64_t dst_lo = 0, dst_hi = 0;
  int64_t max_in_deg = 0, max_pair_deg = 0;
  int compact = 1;  // 1: rows per distinct (rel, src) pair; 0: one row per edge (vanilla materialization)
  int nb = 0, rb = 0;  // key bit widths

  std::vector<int64_t> node_type_ptr;    // host [T+1]
  std::vector<int32_t> pair_rel_ptr_h;   // host [R+1]
  std::vector<int32_t> pair_rt_ptr_h;    // host [R*T+1] : pairs sorted by (rel, src type)
  std::vector<int32_t> dpair_rel_ptr_h;  // host [R+1]
  std::vector<int32_t> pair_src_h;       // host [U], copied on first use by a chunked (multi-GPU) pair GEMM

  // device index arrays (int32)
  int32_t* etype_ptr = nullptr;  // [R+1]
  int32_t* row_ptr = nullptr;    // [N+1]
  int32_t* csr_src = nullptr;
  int32_t* csr_rel = nullptr;
  int32_t* csr_eid = nullptr;
  int32_t* csr_pair = nullptr;
  uint8_t* csr_single = nullptr;  // [E] 1 when the CSR entry's pair has exactly one edge
  int32_t* col_ptr = nullptr;  // [N+1]
  int32_t* col_ptr_full = nullptr;  // [N+1] out-degree prefix over ALL input edges (partitioned builds only)
  int32_t* csc_dst = nullptr;
  int32_t* csc_rel = nullptr;
  int32_t* csc_eid = nullptr;
  int32_t* csc_pair = nullptr;
  int32_t* csc2csr = nullptr;  // CSR position of each CSC entry
  int32_t* edge_pair = nullptr;
  int32_t* kept_eid = nullptr;       // [E] original edge id of each kept edge (partitioned builds)
  int32_t* pair_rel_ptr = nullptr;   // [R+1]
  int32_t* pair_rt_ptr = nullptr;    // [R*T+1] pairs by (rel, src type)
  // HGT A2 folds one weight per (r, t) combination that has pairs ("active"); a = 0..n_act-1 in rt order
  int32_t n_act = 0;
  std::vector<int32_t> act_of_rt_h;  // host [R*T]: active index, or 0 for an empty combination (no tiles)
  int32_t* act_rt = nullptr;         // [n_act] rt = r*T + t of each active combination
  int32_t* t_act_ptr = nullptr;      // [T+1] active combinations grouped by source type ...
  int32_t* t_act = nullptr;          // [n_act] ... (active indices, ascending r)
  int32_t* r_act_ptr = nullptr;      // [R+1] active indices of relation r are r_act_ptr[r] .. r_act_ptr[r+1]-1
  int32_t* pair_src = nullptr;       // [U]
  int32_t* pair_csc_beg = nullptr;   // [U] first CSC position of the pair's edges
  int32_t* pair_deg = nullptr;       // [U] number of edges of the pair
  int32_t* src_pair_ptr = nullptr;   // [N+1]
  int32_t* src_pairs = nullptr;      // [U] pairs ordered by (src, rel)
  int32_t* dpair_dst = nullptr;      // [UD] (rel,dst) pairs ordered by (rel, dst)
  int32_t* dpair_csr_beg = nullptr;  // [UD]
  int32_t* dpair_cnt = nullptr;      // [UD]
  // (rel, dst) runs longer than SPLIT_THRESH entries, for the deterministic two-level run sums (dpair_sum_w):
  // SPLIT_CHUNK-entry chunks (run, begin, end, slot) and per run (run, first slot, number of slots, 0)
  int4* dpair_chunks = nullptr;
  int64_t n_dpair_chunks = 0;
  int4* dpair_splits = nullptr;
  int64_t n_dpair_splits = 0;
  int32_t* dst_dpair_ptr = nullptr;  // [N+1] lazily (ensure_dst_dpairs): dpairs grouped by destination
  int32_t* dst_dpairs = nullptr;     // [UD]

  // edge-balanced work lists (skewed in-degrees and pair degrees), see rgnn::WorkPlan
  rgnn::WorkPlan rows;   // destination rows over the dst-CSR
  rgnn::WorkPlan pairs;  // compact pairs over the src-CSC

  // lazily computed RGCN norms (by kind): per CSR entry and per CSC entry
  std::map<int, std::pair<float*, float*>> norms;
  // cached tile plans
  std::map<std::string, rgnn::Plan> plans;
  std::vector<void*> owned;  // everything allocated through `alloc`
  int64_t owned_bytes = 0;   // their total size (rgnn_graph_info.device_bytes)

  int32_t* dev_i32(size_t n, cudaStream_t s) {
    void* p = alloc.get((n ? n : 1) * sizeof(int32_t), s);
    owned.push_back(p);
    owned_bytes += (int64_t)(n ? n : 1) * sizeof(int32_t);
    return static_cast<int32_t*>(p);
  }
  float* dev_f32(size_t n, cudaStream_t s) {
    void* p = alloc.get((n ? n : 1) * sizeof(float), s);
    owned.push_back(p);
    owned_bytes += (int64_t)(n ? n : 1) * sizeof(float);
    return static_cast<float*>(p);
  }
};

namespace rgnn {
// Segment offsets -> tiles of at most `rows` rows that never cross a segment.
// seg_ptr has nseg+1 entries; w_of_seg maps segment -> weight index (identity if empty).
const Plan& get_plan(rgnn_graph_s* g, const std::string& key, const std::vector<int64_t>& seg_ptr,
                     const std::vector<int32_t>& w_of_seg, int rows, cudaStream_t s);
void graph_norms(rgnn_graph_s* g, int kind, const float* custom, cudaStream_t s, float** csr_norm,
                 float** csc_norm);
void ensure_dst_dpairs(rgnn_graph_s* g, cudaStream_t s);
}  // namespace rgnn
