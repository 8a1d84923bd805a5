// Write bandwidth of TMA bulk-tensor stores by box shape, for the GEMM
// epilogue's per-warp store pattern: a [M x N] bf16 matrix (M = 8320, N = 3072:
// 51 MB, the FC1 forward's two outputs) written entirely by TMA stores of
//   narrow : 32 rows x 16 cols (32-B rows, SWIZZLE_32B)  = the current epilogue
//   wide   : 32 rows x 64 cols (128-B rows, SWIZZLE_128B)
// issued by one lane per warp from a per-warp smem buffer, 16 warps per CTA,
// one CTA per SM, each warp cycling through its blocks like the epilogue
// (wait_group.read before the buffer is rewritten).
// usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tsb tma_store_box.cu -lcuda && /tmp/tsb
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

constexpr int M = 8320, N = 3072;
template <int COLS>
__global__ void __launch_bounds__(512, 1) store_k(const __grid_constant__ CUtensorMap map, int nbuf) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int BYTES = 32 * COLS * 2;
  uint8_t* buf = sm + warp * BYTES * nbuf;
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
  const int bx = N / COLS, by = M / 32, blocks = bx * by;
  int k = 0;
  for (int b = blockIdx.x * 16 + warp; b < blocks; b += gridDim.x * 16, ++k) {
    const int slot = k % nbuf;
    if (lane == 0) {
      if (nbuf == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    }
    __syncwarp();
    // each lane writes its row's COLS*2 bytes (content irrelevant, layout = any swizzle)
    uint4* p = reinterpret_cast<uint4*>(buf + slot * BYTES + lane * COLS * 2);
#pragma unroll
    for (int j = 0; j < COLS * 2 / 16; ++j) p[j] = make_uint4(b, j, lane, 7);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                   ::"l"(reinterpret_cast<uint64_t>(&map)), "r"((b % bx) * COLS), "r"((b / bx) * 32),
                   "r"(sa + slot * BYTES) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  void* out; cudaMalloc(&out, (size_t)M * N * 2);
  char* flush; cudaMalloc(&flush, 512l << 20);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int cfg = 0; cfg < 4; ++cfg) {
    const bool wide = cfg & 1;
    const int nbuf = cfg < 2 ? 1 : 2;
    const int cols = wide ? 64 : 16;
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)N * 2};
    cuuint32_t box[2] = {(cuuint32_t)cols, 32};
    cuuint32_t es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, wide ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B,
        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = 16 * 32 * cols * 2 * nbuf;
    auto kern = wide ? store_k<64> : store_k<16>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(flush, rep, 512l << 20);   // evict (dirty) L2
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      kern<<<148, 512, smem>>>(map, nbuf);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-6s box 32x%-2d nbuf=%d: %7.2f us  %7.1f GB/s  (%s)\n", wide ? "wide" : "narrow", cols,
           nbuf, best * 1e3, (double)M * N * 2 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
