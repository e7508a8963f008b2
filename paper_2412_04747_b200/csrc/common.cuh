// Shared internals of librgnn: status handling, allocation, launch + profiling,
// element-type helpers.  Not part of the ABI (see include/rgnn.h).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "rgnn.h"

#define RGNN_STR_(x) #x
#define RGNN_STR(x) RGNN_STR_(x)

namespace rgnn {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
void clear_error();

struct Error {
  rgnn_status st;
  std::string msg;
};

#define RGNN_FAIL(status, msg_expr)                                   \
  do {                                                                \
    throw ::rgnn::Error{(status), std::string(msg_expr)};             \
  } while (0)

#define RGNN_CUDA(call)                                                                        \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      RGNN_FAIL(RGNN_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));            \
  } while (0)

#define RGNN_CHECK(cond, status, msg_expr)  \
  do {                                      \
    if (!(cond)) RGNN_FAIL(status, msg_expr); \
  } while (0)

// Run `body` and convert exceptions to a status + thread-local message.
template <class F>
rgnn_status guarded(F&& body) {
  try {
    clear_error();
    body();
    return RGNN_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.st;
  } catch (const std::exception& e) {
    set_error(std::string("internal error: ") + e.what());
    return RGNN_ERR_INVALID_ARG;
  }
}

// ------------------------------------------------------------------ allocation
struct Allocator {
  rgnn_alloc_fn alloc = nullptr;
  rgnn_free_fn free_fn = nullptr;
  void* ctx = nullptr;
  void* get(size_t bytes, cudaStream_t s) const;
  void put(void* p, cudaStream_t s) const;
};

// Bump allocator over a caller buffer (workspaces); 256-byte alignment.
struct Arena {
  char* base = nullptr;
  size_t cap = 0;
  size_t off = 0;
  bool measure_only = false;
  template <class T>
  T* take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
    size_t at = off;
    off += bytes;
    if (measure_only) return nullptr;
    RGNN_CHECK(off <= cap, RGNN_ERR_INVALID_ARG, "workspace buffer too small");
    return reinterpret_cast<T*>(base + at);
  }
};

// ------------------------------------------------------------------ launches
// Every kernel launch goes through launch(); with profiling on, CUDA events
// bracket it on its stream (rgnn_profile_*).
void profile_begin(const char* name, cudaStream_t s, int* slot);
const char* intern(const std::string& name);  // stable C string for profile labels
void profile_end(int slot, cudaStream_t s);
void count_launch();

template <class Kernel, class... Args>
void launch(const char* name, Kernel k, dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
  int slot = -1;
  profile_begin(name, s, &slot);
  k<<<grid, block, smem, s>>>(args...);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) RGNN_FAIL(RGNN_ERR_CUDA, std::string("launch ") + name + ": " + cudaGetErrorString(e));
  count_launch();
  profile_end(slot, s);
}

inline unsigned ceil_div(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// Fork/join a per-thread side stream off `s` so two independent launches overlap (e.g. the
// warp-mode and group-mode halves of a traversal).  Capture-safe (events only).
cudaStream_t fork_side(cudaStream_t s);
void join_side(cudaStream_t s);

// ------------------------------------------------------------------ element types
typedef __nv_bfloat16 bf16;

template <class T> struct Vec;  // 16-byte vector of T
template <> struct Vec<float> { static constexpr int N = 4; };
template <> struct Vec<bf16> { static constexpr int N = 8; };

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(bf16 x) { return __bfloat162float(x); }
template <class T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

// Load 16 bytes (Vec<T>::N elements) as floats.  p must be 16-byte aligned.
__device__ __forceinline__ void load16(const float* p, float* out) {
  float4 v = __ldg(reinterpret_cast<const float4*>(p));
  out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
}
__device__ __forceinline__ void load16(const bf16* p, float* out) {
  uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    out[2 * i] = __uint_as_float(w[i] << 16);
    out[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
// Raw 16-byte loads (issue first, convert later, for memory-level parallelism).
__device__ __forceinline__ uint4 ldg16(const void* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
template <class T> __device__ __forceinline__ void cvt16(uint4 v, float* out);
template <> __device__ __forceinline__ void cvt16<float>(uint4 v, float* out) {
  out[0] = __uint_as_float(v.x); out[1] = __uint_as_float(v.y);
  out[2] = __uint_as_float(v.z); out[3] = __uint_as_float(v.w);
}
template <> __device__ __forceinline__ void cvt16<bf16>(uint4 v, float* out) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    out[2 * i] = __uint_as_float(w[i] << 16);
    out[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

__device__ __forceinline__ void store16(float* p, const float* v) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void store16(bf16* p, const float* v) {
  uint4 o;
  uint32_t* w = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  *reinterpret_cast<uint4*>(p) = o;
}

template <int WIDTH>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = WIDTH / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace rgnn
