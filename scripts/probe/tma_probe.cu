// TMA semantics probe (sm_100a): tile::gather4 box shape and 128B swizzle placement, 2D tile load/store.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k_g4(const __grid_constant__ CUtensorMap tm, int r0, int r1, int r2, int r3, uint16_t* out, int bytes) {
  __shared__ __align__(1024) uint8_t buf[8192];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(buf), b = (uint32_t)__cvta_generic_to_shared(&bar);
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = 0xff;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes));
    asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      :: "r"(s), "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b) : "memory");
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(b) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(buf)[i];
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  const int R = 1000, C = 64;
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r) for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 64 + c);
  uint16_t *d, *o;
  cudaMalloc(&d, R * C * 2); cudaMalloc(&o, 2048 * 2);
  cudaMemcpy(d, h.data(), R * C * 2, cudaMemcpyHostToDevice);
  for (int box1 : {1, 4}) for (int sw : {0, 3}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R}, strides[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box1}, es[2] = {1, 1};
    CUresult rr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      sw == 3 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rr != CUDA_SUCCESS) { printf("box1=%d sw=%d encode error %d\n", box1, sw, (int)rr); continue; }
    cudaMemset(o, 0, 4096);
    k_g4<<<1, 128>>>(tm, 5, 17, 999, 3, o, 4 * 128);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint16_t> g(1024);
    cudaMemcpy(g.data(), o, 2048, cudaMemcpyDeviceToHost);
    printf("box1=%d swizzle=%s err=%s\n", box1, sw ? "128B" : "none", cudaGetErrorString(e));
    for (int r = 0; r < 5; ++r) {  // 16-byte chunk c of smem row r: first element -> (row, col)
      printf("  smem row %d:", r);
      for (int c = 0; c < 8; ++c) { uint16_t v = g[r * 64 + c * 8]; printf(" %s%d.%d", v == 0xffff ? "x" : "", v / 64, v % 64); }
      printf("\n");
    }
  }
  return 0;
}
