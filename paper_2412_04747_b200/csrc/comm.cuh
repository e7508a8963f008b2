// Internal layout of a communicator (rgnn_comm_t) and the exchange steps the layer calls.
#pragma once

#include <utility>
#include <vector>

#include "common.cuh"

typedef struct ncclComm* ncclComm_t;

struct rgnn_comm_s {
  ncclComm_t nc = nullptr;
  int rank = 0, world = 1, device = 0;
  std::vector<int64_t> node_ptr;  // [world+1]: rank k owns node rows [node_ptr[k], node_ptr[k+1])
  cudaStream_t cs = nullptr;      // library-owned comm stream (high priority)
  std::vector<cudaEvent_t> chunk;  // [world]: row chunk k has arrived (forward all-gather)
  cudaEvent_t start = nullptr, done = nullptr;
};

namespace rgnn {
void comm_allgather_rows_begin(rgnn_comm_s* c, void* rows, size_t row_bytes, cudaStream_t s);
void comm_wait_chunk(rgnn_comm_s* c, int k, cudaStream_t s);
void comm_wait_all(rgnn_comm_s* c, cudaStream_t s);
void comm_reduce_grads(rgnn_comm_s* c, float* dX, int64_t d_in, const std::vector<std::pair<float*, size_t>>& dW,
                       cudaStream_t s);
void comm_join(rgnn_comm_s* c, cudaStream_t s);
}  // namespace rgnn
