// tcgen05 GEMM placeholder (filled in by the tensor-core engine).
#include "common.cuh"
#include "kernels.cuh"
namespace ppll {
template <typename TO>
int launch_gemm_tc(int, int, int, const __nv_bfloat16*, long, bool, const __nv_bfloat16*, long,
                   bool, const Epilogue<TO>&, float*, size_t, cudaStream_t) {
  return PPLL_ERR_UNSUPPORTED;
}
template int launch_gemm_tc<float>(int, int, int, const __nv_bfloat16*, long, bool, const __nv_bfloat16*, long, bool, const Epilogue<float>&, float*, size_t, cudaStream_t);
template int launch_gemm_tc<__nv_bfloat16>(int, int, int, const __nv_bfloat16*, long, bool, const __nv_bfloat16*, long, bool, const Epilogue<__nv_bfloat16>&, float*, size_t, cudaStream_t);
}  // namespace ppll
