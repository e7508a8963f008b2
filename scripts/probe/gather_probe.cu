// Random-row gather ceiling on B200: E gathers of ROW-byte rows from an N-row table (uniform random
// row ids), each row read by LPR = ROW/16 lanes with 16-byte loads and summed (so nothing is
// optimised away).  Reports useful GB/s = E * ROW / time.  Build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a gather_probe.cu -o gather_probe
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int ROW, int U>
__global__ void __launch_bounds__(256) k_gather(int64_t E, const int* __restrict__ idx, const uint4* __restrict__ tab,
                                                uint4* __restrict__ out) {
  constexpr int LPR = ROW / 16, EG = 32 / LPR;
  const int lane = threadIdx.x & 31, g = lane / LPR, c = lane % LPR;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int64_t base = (gw * EG + g) * U; base < E; base += nw * EG * U) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + u;
      const int64_t row = e < E ? __ldg(idx + e) : 0;
      r[u] = __ldg(tab + row * LPR + c);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x ^= r[u].x; acc.y += r[u].y; acc.z ^= r[u].z; acc.w += r[u].w; }
  }
  out[gw * 32 + lane] = acc;
}

template <int ROW, int U>
float run(int64_t E, const int* idx, const uint4* tab, uint4* out, int sms, int bps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  dim3 grid(sms * bps);
  k_gather<ROW, U><<<grid, 256>>>(E, idx, tab, out);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) k_gather<ROW, U><<<grid, 256>>>(E, idx, tab, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t E = 21111007;
  int* idx; uint4* tab; uint4* out;
  cudaMalloc(&idx, E * 4);
  cudaMalloc(&out, (size_t)sms * 32 * 256 * 16 * 8);
  const int64_t maxN = 20000000;
  cudaMalloc(&tab, maxN * 512);
  cudaMemset(tab, 1, maxN * 512);
  std::mt19937_64 rng(1);
  std::vector<int> h(E);
  for (int64_t N : {200000LL, 1939743LL, 20000000LL}) {
    for (auto& x : h) x = (int)(rng() % N);
    cudaMemcpy(idx, h.data(), E * 4, cudaMemcpyHostToDevice);
    for (int bps : {4, 8}) {
      float t1 = run<256, 1>(E, idx, tab, out, sms, bps);
      float t2 = run<256, 2>(E, idx, tab, out, sms, bps);
      float t4 = run<256, 4>(E, idx, tab, out, sms, bps);
      float t8 = run<256, 8>(E, idx, tab, out, sms, bps);
      float s4 = run<128, 4>(E, idx, tab, out, sms, bps);
      float w4 = run<512, 4>(E, idx, tab, out, sms, bps);
      printf("N=%lld (%.0f MB @256B) blocks/SM=%d  row256: U1 %.3f ms %.0f GB/s | U2 %.0f | U4 %.0f | U8 %.0f   row128 U4 %.0f GB/s   row512 U4 %.0f GB/s\n",
             (long long)N, N * 256 / 1e6, bps, t1, E * 256.0 / t1 / 1e6, E * 256.0 / t2 / 1e6, E * 256.0 / t4 / 1e6,
             E * 256.0 / t8 / 1e6, E * 128.0 / s4 / 1e6, E * 512.0 / w4 / 1e6);
    }
  }
  return 0;
}
