// Internal layout of a built graph (rgnn_graph_t).  See DESIGN.md "Data layout in HBM".
#pragma once

#include <map>
#include <string>
#include <vector>

#include "common.cuh"

namespace rgnn {

constexpr int SPLIT_THRESH = 1024;  // rows with more in-edges are split ...
constexpr int SPLIT_CHUNK = 512;    // ... into chunks of this many edges

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
  int nb = 0, rb = 0;  // key bit widths

  std::vector<int64_t> node_type_ptr;    // host [T+1]
  std::vector<int32_t> pair_rel_ptr_h;   // host [R+1]
  std::vector<int32_t> pair_rt_ptr_h;    // host [R*T+1] : pairs sorted by (rel, src type)
  std::vector<int32_t> dpair_rel_ptr_h;  // host [R+1]

  // device index arrays (int32)
  int32_t* etype_ptr = nullptr;  // [R+1]
  int32_t* row_ptr = nullptr;    // [N+1]
  int32_t* csr_src = nullptr;
  int32_t* csr_rel = nullptr;
  int32_t* csr_eid = nullptr;
  int32_t* csr_pair = nullptr;
  int32_t* col_ptr = nullptr;  // [N+1]
  int32_t* csc_dst = nullptr;
  int32_t* csc_rel = nullptr;
  int32_t* csc_eid = nullptr;
  int32_t* csc_pair = nullptr;
  int32_t* csc2csr = nullptr;  // CSR position of each CSC entry
  int32_t* edge_pair = nullptr;
  int32_t* kept_eid = nullptr;       // [E] original edge id of each kept edge (partitioned builds)
  int32_t* pair_rel_ptr = nullptr;   // [R+1]
  int32_t* pair_src = nullptr;       // [U]
  int32_t* pair_csc_beg = nullptr;   // [U] first CSC position of the pair's edges
  int32_t* pair_deg = nullptr;       // [U] number of edges of the pair
  int32_t* src_pair_ptr = nullptr;   // [N+1]
  int32_t* src_pairs = nullptr;      // [U] pairs ordered by (src, rel)
  int32_t* dpair_dst = nullptr;      // [UD] (rel,dst) pairs ordered by (rel, dst)
  int32_t* dpair_csr_beg = nullptr;  // [UD]
  int32_t* dpair_cnt = nullptr;      // [UD]

  // edge-balanced destination work list (skewed in-degrees): rows with more than
  // SPLIT_THRESH in-edges are cut into chunks of SPLIT_CHUNK edges, each a separate
  // warp item writing a partial state to slot w; heavy chunks are listed first.
  int4* row_items = nullptr;   // [n_items] (row, edge begin, edge end, slot or -1)
  int64_t n_items = 0;
  int4* split_rows = nullptr;  // [n_split] (row, first slot, number of slots, 0)
  int64_t n_split = 0, n_slots = 0;

  // lazily computed RGCN norms (by kind): per CSR entry and per CSC entry
  std::map<int, std::pair<float*, float*>> norms;
  // cached tile plans
  std::map<std::string, rgnn::Plan> plans;
  std::vector<void*> owned;  // everything allocated through `alloc`

  int32_t* dev_i32(size_t n, cudaStream_t s) {
    void* p = alloc.get((n ? n : 1) * sizeof(int32_t), s);
    owned.push_back(p);
    return static_cast<int32_t*>(p);
  }
  float* dev_f32(size_t n, cudaStream_t s) {
    void* p = alloc.get((n ? n : 1) * sizeof(float), s);
    owned.push_back(p);
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
}  // namespace rgnn
