// Shared device/host helpers for the PPLL B200 library (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/ppll.h"

#include <nvtx3/nvToolsExt.h>   // header-only; ranges are no-ops unless a tool attaches
namespace ppll {

// Sticky per-stage error word bits (checked asynchronously by the host;
// mapped to the reference's exception classes in the Python shim).
enum ErrBits : int {
  kErrLabel = PPLL_ERRBIT_LABEL,          // LabelOutOfRange   (tensor.py:216-219)
  kErrLossNonFinite = PPLL_ERRBIT_LOSS,   // NonFiniteError    (tensor.py:227)
  kErrParamNonFinite = PPLL_ERRBIT_PARAM, // NonFiniteError    (tensor.py:41-43)
  kErrStep = PPLL_ERRBIT_STEP,            // StepOutOfRange    (optim.py:41-42)
  kErrGradNonFinite = PPLL_ERRBIT_GRAD,   // NonFiniteError    (tensor.py:41-43, pre-update)
  kErrSync = PPLL_ERRBIT_SYNC,            // WorkerPanic       (a grid barrier watchdog fired)
};

void set_error(const char* fmt, ...);
const char* last_error();

#define PPLL_CUDA_CHECK(expr)                                                   \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) {                                                    \
      ::ppll::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,              \
                        cudaGetErrorString(_e));                                \
      return PPLL_ERR_CUDA;                                                     \
    }                                                                           \
  } while (0)

#define PPLL_LAUNCH_CHECK() PPLL_CUDA_CHECK(cudaGetLastError())

template <typename T> struct DT;
template <> struct DT<float> {
  static __device__ __forceinline__ float ld(const float* p) { return *p; }
  static __device__ __forceinline__ void st(float* p, float v) { *p = v; }
};
template <> struct DT<__nv_bfloat16> {
  static __device__ __forceinline__ float ld(const __nv_bfloat16* p) { return __bfloat162float(*p); }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
};

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

inline int ceil_div(long a, long b) { return (int)((a + b - 1) / b); }

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  Every kernel of the library is
// launched with programmatic stream serialisation and starts with
// pdl_entry(): it waits (griddepcontrol.wait) until its stream predecessor
// has completed and flushed, then immediately lets its own successor be
// scheduled (griddepcontrol.launch_dependents).  A successor's CTAs therefore
// launch and run their prologue (barrier init, TMEM allocation, tensor-map
// prefetch — placed before pdl_wait in the tcgen05 kernels) while the
// predecessor's last wave drains, instead of after it.  Inside CUDA graphs
// the attribute becomes a programmatic edge.  PPLL_PDL=0 disables it.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_entry() {
  pdl_wait();
  pdl_trigger();
}

extern thread_local int g_pdl;
// SM budget of the tcgen05 GEMM launches issued by this host thread (0 = the
// whole GPU): a stage step caps its data-gradient GEMMs / cluster weight
// gradients so the two streams' kernels can be resident side by side
extern thread_local int g_gemm_cap, g_wgrad_cap;
// 1 when the kernels this host thread launches own their GPU (one stage
// stream): full-GPU cooperative kernels (the grid-form fused BN) are allowed.
// A pipeline that puts several stage streams on one GPU sets 0 — a
// cooperative grid needs every SM at once and would serialise the streams.
extern thread_local int g_gpu_excl;

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace ppll

namespace ppll {
// Fork/join of a stage step's side stream (capturable: a CUDA graph records
// the event edges).  Without a side stream everything stays on the step's
// stream and the calls are no-ops.  The last event is reserved: if a step
// ever needs more events than the pool holds, the side work is joined and the
// rest of the step runs on the main stream (always correct, just serial).
// NVTX range for the host-side enqueue phases of a stage step (visible in ncu
// --nvtx / nsys timelines; free when no tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct SideFlow {
  cudaStream_t s, ss;
  cudaEvent_t* ev;
  int n = 0, cap;
  bool on() const { return ss != s; }
  bool reserve() {
    if (n < cap - 1) return true;
    if (on()) {
      cudaEventRecord(ev[cap - 1], ss);
      cudaStreamWaitEvent(s, ev[cap - 1], 0);
      ss = s;
    }
    return false;
  }
  void fork() {            // side work after everything enqueued on s so far
    if (!on() || !reserve()) return;
    cudaEventRecord(ev[n], s);
    cudaStreamWaitEvent(ss, ev[n++], 0);
  }
  cudaEvent_t mark() {     // completion of the side work enqueued so far
    if (!on() || !reserve()) return nullptr;
    cudaEventRecord(ev[n], ss);
    return ev[n++];
  }
  void join(cudaEvent_t e) {
    if (e) cudaStreamWaitEvent(s, e, 0);
  }
};
}  // namespace ppll
