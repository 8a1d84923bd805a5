// Write-bandwidth probe for epilogue store patterns on a [M x N] bf16 matrix
// (M = 8320, N = 3072: 51 MB, the FC1 forward's two outputs).
//   sector : each warp instruction writes 16 rows x 32 B (the GEMM epilogue's
//            transposed 16-column blocks; 4 warps cover one 128-B line)
//   line   : each warp instruction writes 4 rows x 128 B (full lines)
//   linear : consecutive 16-B vectors (memset-like)
// usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sp store_pattern.cu && /tmp/sp
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

constexpr int M = 8320, N = 3072;   // bf16 elements
__global__ void sector_k(uint4* out) {
  // block = 16 warps; CTA tile 128 rows x 256 cols; warp w: quadrant q = w & 3 (32 rows),
  // group g = w >> 2 takes 16-col chunks g, g+4, g+8, g+12
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, q = warp & 3, g = warp >> 2;
  const int tiles_n = N / 256, tiles = (M / 128) * tiles_n;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int m0 = (t % (M / 128)) * 128, n0 = (t / (M / 128)) * 256;
    for (int c = 16 * g; c < 256; c += 64)
      for (int i = 0; i < 2; ++i) {
        const int row = m0 + q * 32 + i * 16 + (lane >> 1), col = n0 + c + (lane & 1) * 8;
        out[((long)row * N + col) / 8] = make_uint4(row, col, 1, 2);
      }
  }
}
__global__ void line_k(uint4* out) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, q = warp & 3, g = warp >> 2;
  const int tiles = (M / 128) * (N / 256);
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int m0 = (t % (M / 128)) * 128, n0 = (t / (M / 128)) * 256;
    // warp g owns cols [64g, 64g+64) of its quadrant's 32 rows: 8 instr x 4 rows x 128 B
    for (int i = 0; i < 8; ++i) {
      const int row = m0 + q * 32 + i * 4 + (lane >> 3), col = n0 + 64 * g + (lane & 7) * 8;
      out[((long)row * N + col) / 8] = make_uint4(row, col, 1, 2);
    }
  }
}
__global__ void linear_k(uint4* out, long n16) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n16; i += (long)gridDim.x * blockDim.x)
    out[i] = make_uint4(i, 0, 1, 2);
}
__global__ void read_k(const uint4* in, long n16, unsigned* sink) {
  unsigned acc = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n16; i += (long)gridDim.x * blockDim.x)
    acc ^= in[i].x;
  if (acc == 0x12345678u) *sink = acc;
}
int main(int argc, char** argv) {
  const bool read_flush = argc > 1;   // clean-L2 flush (a read) instead of a dirty memset
  uint4* out; cudaMalloc(&out, (size_t)M * N * 2);
  char* flush; cudaMalloc(&flush, 512l << 20); cudaMemset(flush, 1, 512l << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const double bytes = (double)M * N * 2;
  for (int k = 0; k < 3; ++k) {
    for (int rep = 0; rep < 3; ++rep) {
      if (read_flush) read_k<<<148 * 4, 512>>>((const uint4*)flush, (512l << 20) / 16, (unsigned*)out);
      else cudaMemset(flush, rep, 512l << 20);
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      if (k == 0) sector_k<<<148, 512>>>(out);
      else if (k == 1) line_k<<<148, 512>>>(out);
      else linear_k<<<148 * 4, 512>>>(out, (long)M * N / 8);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("%-7s %7.2f us  %7.1f GB/s\n", k == 0 ? "sector" : k == 1 ? "line" : "linear",
                           ms * 1e3, bytes / ms / 1e6);
    }
  }
  return 0;
}
