// Device primitives behind the reference's tape API (tensor.py:137-278):
// relu / bias_add / add / scale / sum_all forwards and the adjoints the
// device GradTape replays (tensor.py:153-198).  Not on the PPLL hot path —
// the stage step is one fused native call — but a training loop written
// against locopipe's GradTape / backward runs on the device through these.
// Every forward output is checked for non-finite values (tensor.py:41-43):
// a sticky flag the Python shim turns into NonFiniteError.
#include "common.cuh"
#include "kernels.cuh"

namespace ppll {

enum EwOp : int {
  kEwRelu = 0,      // out = max(a, 0)                    relu        tensor.py:153-157
  kEwReluBwd = 1,   // out = a * [b > 0]  (a = g, b = x)  relu adjoint (0 at 0)
  kEwBiasAdd = 2,   // out[r, c] = a[r, c] + b[c]         bias_add    tensor.py:170-180
  kEwAxpby = 3,     // out = alpha * a + b (b nullable)   add / scale / accumulate
  kEwBroadcast = 4, // out[i] = alpha * a[0]              sum_all adjoint tensor.py:194-198
};

template <typename T>
__global__ void __launch_bounds__(256)
ew_kernel(int op, long rows, long cols, const T* __restrict__ a, const T* __restrict__ b,
          float alpha, T* __restrict__ out, int* err) {
  pdl_entry();
  const long n = rows * cols;
  bool bad = false;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    float v;
    switch (op) {
      case kEwRelu: v = fmaxf(to_f(a[i]), 0.f); if (!isfinite(to_f(a[i]))) bad = true; break;
      case kEwReluBwd: v = to_f(b[i]) > 0.f ? to_f(a[i]) : 0.f; break;
      case kEwBiasAdd: v = to_f(a[i]) + to_f(b[i % cols]); break;
      case kEwAxpby: v = alpha * to_f(a[i]) + (b ? to_f(b[i]) : 0.f); break;
      default: v = alpha * to_f(a[0]); break;
    }
    bad |= !isfinite(v);
    DT<T>::st(out + i, v);
  }
  if (err && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, kErrParamNonFinite);
}

// sum of all n elements into *out (fp32), one block, fixed-order tree: deterministic
template <typename T>
__global__ void __launch_bounds__(1024) sum_all_kernel(long n, const T* __restrict__ x, float* out,
                                                       int* err) {
  pdl_entry();
  __shared__ double part[32];
  double s = 0.0;
  for (long i = threadIdx.x; i < n; i += blockDim.x) s += (double)to_f(x[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) {
      *out = (float)t;
      if (err && !isfinite((float)t)) atomicOr(err, kErrParamNonFinite);
    }
  }
}

}  // namespace ppll

using namespace ppll;

extern "C" int ppll_ew(int op, int64_t rows, int64_t cols, const void* a, const void* b,
                       float alpha, void* out, int dtype, int* err, void* stream) {
  if (op < kEwRelu || op > kEwBroadcast || rows < 0 || cols < 1 || !a || !out ||
      ((op == kEwReluBwd || op == kEwBiasAdd) && !b)) {
    set_error("ppll_ew: bad arguments (op %d)", op);
    return PPLL_ERR_ARG;
  }
  const long n = rows * cols;
  if (n == 0) return PPLL_OK;
  auto s = reinterpret_cast<cudaStream_t>(stream);
  const int blocks = (int)std::min<long>((n + 255) / 256, 148L * 8);
  if (dtype == PPLL_F32)
    launch_k(ew_kernel<float>, blocks, 256, 0, s, op, (long)rows, (long)cols, (const float*)a,
             (const float*)b, alpha, (float*)out, err);
  else
    launch_k(ew_kernel<__nv_bfloat16>, blocks, 256, 0, s, op, (long)rows, (long)cols,
             (const __nv_bfloat16*)a, (const __nv_bfloat16*)b, alpha, (__nv_bfloat16*)out, err);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

extern "C" int ppll_colsum(int rows, int cols, const void* g, float* out, int dtype, void* stream) {
  if (rows < 1 || cols < 1 || !g || !out) {
    set_error("ppll_colsum: bad arguments");
    return PPLL_ERR_ARG;
  }
  auto s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == PPLL_F32)
    return launch_colsum<float>(rows, cols, (const float*)g, cols, out, s, nullptr, 0);
  return launch_colsum<__nv_bfloat16>(rows, cols, (const __nv_bfloat16*)g, cols, out, s, nullptr, 0);
}

extern "C" int ppll_sum_all(int64_t n, const void* x, float* out, int dtype, int* err,
                            void* stream) {
  if (n < 1 || !x || !out) {
    set_error("ppll_sum_all: bad arguments");
    return PPLL_ERR_ARG;
  }
  auto s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == PPLL_F32)
    launch_k(sum_all_kernel<float>, 1, 1024, 0, s, (long)n, (const float*)x, out, err);
  else
    launch_k(sum_all_kernel<__nv_bfloat16>, 1, 1024, 0, s, (long)n, (const __nv_bfloat16*)x, out,
             err);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}
