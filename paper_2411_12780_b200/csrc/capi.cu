// extern "C" boundary (include/ppll.h) + linear-layer engine dispatch.
#include <stdarg.h>
#include <atomic>
#include <math.h>
#include <string.h>
#include <stdlib.h>
#include "common.cuh"
#include "kernels.cuh"

namespace ppll {

static thread_local char t_err[512] = {0};
static std::atomic<uint64_t> g_launches{0};
int g_gemm_engine = PPLL_GEMM_AUTO;
// per host thread: two pipelines driven from different threads each launch with
// their own setting (a process-wide flag could be flipped under a capture)
thread_local int g_pdl = getenv("PPLL_PDL") ? atoi(getenv("PPLL_PDL")) : 1;
thread_local int g_gemm_cap = 0, g_wgrad_cap = 0;
thread_local int g_gpu_excl = getenv("PPLL_GPU_EXCLUSIVE") ? atoi(getenv("PPLL_GPU_EXCLUSIVE")) : 1;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_err, sizeof(t_err), fmt, ap);
  va_end(ap);
}
const char* last_error() { return t_err; }
void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
using bf16 = __nv_bfloat16;

template <typename TO>
static Epilogue<TO> make_ep(const LinOpts& o, void* C, long ldc, int ncols) {
  Epilogue<TO> e;
  e.C = (TO*)C; e.ldc = ldc;
  e.C2 = (TO*)o.C2; e.ldc2 = o.ldc2;
  e.bias = o.bias; e.act = o.act;
  e.mask = (const TO*)o.mask; e.ldmask = o.ldmask;
  e.mask_mode = o.mask ? (o.mask_mode ? o.mask_mode : (int)kMaskRelu) : (int)kMaskNone;
  e.res = (const TO*)o.res; e.ldres = o.ldres;
  e.pre = (TO*)o.pre; e.ldpre = o.ldpre;
  epilogue_finalize(e, ncols);
  return e;
}

// ---- linear forward: Y = act(X·W + b [+ R]) ----------------------------------
int gemm_fwd(int M, int K, int N, const void* X, long ldx, const void* W, const LinOpts& o,
             void* Y, long ldy, int dtype, float* ws, size_t ws_elems, cudaStream_t s) {
  if (M < 0 || K < 1 || N < 1) { set_error("linear_fwd: bad shape %d %d %d", M, K, N); return PPLL_ERR_ARG; }
  if (M == 0) return PPLL_OK;
  if (dtype == PPLL_F32) {
    auto ep = make_ep<float>(o, Y, ldy, N);
    return launch_gemm_simt<float, float>(M, N, K, (const float*)X, ldx, 1, (const float*)W, N, 1,
                                          ep, ws, ws_elems, s);
  }
  auto ep = make_ep<bf16>(o, Y, ldy, N);
  if (g_gemm_engine != PPLL_GEMM_SIMT) {
    int r = launch_gemm_tc<bf16>(M, N, K, (const bf16*)X, ldx, true, (const bf16*)W, N, false, ep,
                                 ws, ws_elems, s);
    if (r != PPLL_ERR_UNSUPPORTED || g_gemm_engine == PPLL_GEMM_TCGEN05) return r;
  }
  return launch_gemm_simt<bf16, bf16>(M, N, K, (const bf16*)X, ldx, 1, (const bf16*)W, N, 1, ep,
                                      ws, ws_elems, s);
}

// ---- linear dgrad: dX = (dY·Wᵀ) ⊙ mask-function ------------------------------
int gemm_dgrad(int M, int K, int N, const void* dY, long lddy, const void* W, const LinOpts& o,
               void* dX, long lddx, int dtype, float* ws, size_t ws_elems, cudaStream_t s) {
  if (M < 0 || K < 1 || N < 1) { set_error("linear_dgrad: bad shape"); return PPLL_ERR_ARG; }
  if (M == 0) return PPLL_OK;
  if (dtype == PPLL_F32) {
    auto ep = make_ep<float>(o, dX, lddx, K);
    int r = launch_gemm_simt<float, float>(M, K, N, (const float*)dY, lddy, 1, (const float*)W, 1,
                                           N, ep, ws, ws_elems, s);
    if (r == PPLL_OK && o.db) r = launch_colsum<float>(M, K, (const float*)dX, (int)lddx, o.db, s, ws, ws_elems);
    return r;
  }
  auto ep = make_ep<bf16>(o, dX, lddx, K);
  if (g_gemm_engine != PPLL_GEMM_SIMT) {
    const bool fuse_cs = o.db && o.cs_ws && o.cs_ws_elems >= (size_t)ceil_div(M, 32) * K;
    if (fuse_cs) ep.cs_part = o.cs_ws;
    int r = launch_gemm_tc<bf16>(M, K, N, (const bf16*)dY, lddy, true, (const bf16*)W, N, true, ep,
                                 ws, ws_elems, s);
    if (r == PPLL_OK && o.db) {
      if (fuse_cs)   // Σ over the row-block partials (fixed order)
        return launch_colsum<float>(ceil_div(M, 32), K, o.cs_ws, K, o.db, s, ws, ws_elems);
      return launch_colsum<bf16>(M, K, (const bf16*)dX, (int)lddx, o.db, s, ws, ws_elems);
    }
    if (r != PPLL_ERR_UNSUPPORTED || g_gemm_engine == PPLL_GEMM_TCGEN05) return r;
    ep.cs_part = nullptr;
  }
  int r = launch_gemm_simt<bf16, bf16>(M, K, N, (const bf16*)dY, lddy, 1, (const bf16*)W, 1, N, ep,
                                       ws, ws_elems, s);
  if (r == PPLL_OK && o.db) r = launch_colsum<bf16>(M, K, (const bf16*)dX, (int)lddx, o.db, s, ws, ws_elems);
  return r;
}

int linear_fwd(int M, int K, int N, const void* X, int ldx, const void* W, const float* b,
               void* Y, int ldy, void* Y2, int ldy2, int relu, int dtype, float* ws,
               size_t ws_elems, cudaStream_t s) {
  LinOpts o;
  o.bias = b; o.act = relu ? kActRelu : kActNone; o.C2 = Y2; o.ldc2 = ldy2;
  return gemm_fwd(M, K, N, X, ldx, W, o, Y, ldy, dtype, ws, ws_elems, s);
}

int linear_dgrad(int M, int K, int N, const void* dY, int lddy, const void* W, const void* mask,
                 int ldmask, void* dX, int lddx, int dtype, float* ws, size_t ws_elems,
                 cudaStream_t s) {
  LinOpts o;
  o.mask = mask; o.ldmask = ldmask; o.mask_mode = mask ? kMaskRelu : kMaskNone;
  return gemm_dgrad(M, K, N, dY, lddy, W, o, dX, lddx, dtype, ws, ws_elems, s);
}

// ---- linear wgrad: dW = Xᵀ·dY (fp32), db = Σ_rows dY ------------------------
int linear_wgrad(int M, int K, int N, const void* X, int ldx, const void* dY, int lddy, float* dW,
                 float* db, int dtype, float* ws, size_t ws_elems, cudaStream_t s) {
  if (M < 0 || K < 1 || N < 1) { set_error("linear_wgrad: bad shape"); return PPLL_ERR_ARG; }
  Epilogue<float> ep;
  ep.C = dW; ep.ldc = N;
  epilogue_finalize(ep, N);
  int r;
  if (dtype == PPLL_F32) {
    r = launch_gemm_simt<float, float>(K, N, M, (const float*)X, 1, ldx, (const float*)dY, lddy, 1,
                                       ep, ws, ws_elems, s);
    if (r == PPLL_OK && db) r = launch_colsum<float>(M, N, (const float*)dY, lddy, db, s, ws, ws_elems);
    return r;
  }
  r = PPLL_ERR_UNSUPPORTED;
  if (g_gemm_engine != PPLL_GEMM_SIMT) {
    ep.colsum_b = db;   // the cluster split-K kernel can produce db alongside dW
    r = launch_gemm_tc<float>(K, N, M, (const bf16*)X, ldx, false, (const bf16*)dY, lddy, false, ep,
                              ws, ws_elems, s);
    ep.colsum_b = nullptr;
    if (r == kGemmColsumFused) return PPLL_OK;
    if (r != PPLL_OK && (r != PPLL_ERR_UNSUPPORTED || g_gemm_engine == PPLL_GEMM_TCGEN05)) return r;
  }
  if (r == PPLL_ERR_UNSUPPORTED)
    r = launch_gemm_simt<bf16, float>(K, N, M, (const bf16*)X, 1, ldx, (const bf16*)dY, lddy, 1, ep,
                                      ws, ws_elems, s);
  if (r == PPLL_OK && db) r = launch_colsum<bf16>(M, N, (const bf16*)dY, lddy, db, s, ws, ws_elems);
  return r;
}

}  // namespace ppll

using namespace ppll;

extern "C" {

int ppll_abi_version(void) { return PPLL_ABI_VERSION; }
const char* ppll_last_error(void) { return ppll::last_error(); }
uint64_t ppll_launch_count(void) { return g_launches.load(); }
// (profiling hook) the GEMM timeline buffer of PPLL_GEMM_TIMELINE, 148 x 4 x 4 u64
void* ppll_gemm_timeline(void) { return ppll::tc::timeline_buffer(); }
void ppll_set_gemm_engine(int engine) { g_gemm_engine = engine; }

int ppll_linear_fwd(int M, int K, int N, const void* X, int ldx, const void* W, const float* b,
                    void* Y, int ldy, void* Y2, int ldy2, int relu, int dtype, void* stream) {
  return linear_fwd(M, K, N, X, ldx, W, b, Y, ldy, Y2, ldy2, relu, dtype, nullptr, 0, S(stream));
}

int ppll_linear_dgrad(int M, int K, int N, const void* dY, int lddy, const void* W,
                      const void* mask, int ldmask, void* dX, int lddx, int dtype, void* stream) {
  return linear_dgrad(M, K, N, dY, lddy, W, mask, ldmask, dX, lddx, dtype, nullptr, 0, S(stream));
}

int ppll_linear_fwd_ex(int M, int K, int N, const void* X, int ldx, const void* W,
                       const float* b, const void* R, int ldr, int act, void* P, int ldp,
                       void* Y, int ldy, void* Y2, int ldy2, int dtype, void* stream) {
  if (act < kActNone || act > kActGeluD) { set_error("linear_fwd_ex: bad act %d", act); return PPLL_ERR_ARG; }
  LinOpts o;
  o.bias = b; o.res = R; o.ldres = ldr; o.act = act; o.pre = P; o.ldpre = ldp;
  o.C2 = Y2; o.ldc2 = ldy2;
  return gemm_fwd(M, K, N, X, ldx, W, o, Y, ldy, dtype, nullptr, 0, S(stream));
}

int ppll_linear_dgrad_ex(int M, int K, int N, const void* dY, int lddy, const void* W,
                         const void* mask, int ldmask, int mask_mode, void* dX, int lddx,
                         int dtype, void* stream) {
  if (mask_mode < kMaskNone || mask_mode > kMaskMul || (mask_mode != kMaskNone && !mask)) {
    set_error("linear_dgrad_ex: bad mask mode %d", mask_mode);
    return PPLL_ERR_ARG;
  }
  LinOpts o;
  o.mask = mask; o.ldmask = ldmask; o.mask_mode = mask ? mask_mode : kMaskNone;
  return gemm_dgrad(M, K, N, dY, lddy, W, o, dX, lddx, dtype, nullptr, 0, S(stream));
}

int ppll_linear_wgrad(int M, int K, int N, const void* X, int ldx, const void* dY, int lddy,
                      float* dW, float* db, int dtype, void* stream) {
  return linear_wgrad(M, K, N, X, ldx, dY, lddy, dW, db, dtype, nullptr, 0, S(stream));
}

int ppll_softmax_xent(int B, int C, const void* logits, int ldz, const int64_t* labels,
                      void* dlogits, int lddz, float* loss_hist, const int* step, int* err,
                      int dtype, void* stream) {
  if (B < 1 || C < 1) { set_error("softmax_xent needs a non-empty batch"); return PPLL_ERR_ARG; }
  if (dtype == PPLL_F32)
    return launch_softmax_xent<float>(B, C, (const float*)logits, ldz, labels, (float*)dlogits,
                                      lddz, loss_hist, step, err, S(stream));
  return launch_softmax_xent<bf16>(B, C, (const bf16*)logits, ldz, labels, (bf16*)dlogits, lddz,
                                   loss_hist, step, err, S(stream));
}

int ppll_nesterov_step(int64_t n, float* theta, float* v, const float* g, void* theta_lp,
                       const float* lr_table, int* step, int max_step, float lr_host, float mu,
                       float wd, int* err, void* stream) {
  if (n < 0) { set_error("nesterov: negative size"); return PPLL_ERR_ARG; }
  if (n == 0) return PPLL_OK;
  return launch_nesterov(n, theta, v, g, (bf16*)theta_lp, lr_table, step, max_step, lr_host, mu,
                         wd, err, S(stream));
}

int ppll_set_local_optimizer(const float* theta, int kind, float* m2, float beta1, float beta2,
                             float eps) {
  return set_local_optimizer(theta, kind, m2, beta1, beta2, eps);
}

double ppll_cosine_lr(int step, double lr0, double lr_min, int total_steps) {
  if (step < 0 || step > total_steps || total_steps < 1) return NAN;
  double span = lr0 - lr_min;
  return lr_min + 0.5 * span * (1.0 + cos(M_PI * (double)step / (double)total_steps));
}

int ppll_gather_rows(int n, int64_t width, const float* src, const int64_t* idx, void* dst,
                     int dst_dtype, const int64_t* labels_src, int64_t* labels_dst, void* stream) {
  if (n < 0 || width < 1 || !src || !idx || !dst || (labels_src && !labels_dst)) {
    set_error("gather_rows: invalid arguments");
    return PPLL_ERR_ARG;
  }
  return launch_gather_rows(n, width, src, idx, dst, dst_dtype, labels_src, labels_dst, S(stream));
}

int ppll_set_pdl(int on) {
  const int prev = g_pdl;
  g_pdl = on ? 1 : 0;
  return prev;
}

int ppll_set_gpu_exclusive(int on) {
  const int prev = g_gpu_excl;
  g_gpu_excl = on ? 1 : 0;
  return prev;
}

int ppll_events_elapsed(int n, const uint64_t* events, uint64_t ref, float* out_ms) {
  if (n < 0 || (n && (!events || !out_ms)) || !ref) {
    set_error("events_elapsed: invalid arguments");
    return PPLL_ERR_ARG;
  }
  for (int i = 0; i < n; ++i) {
    const cudaError_t e = cudaEventElapsedTime(
        &out_ms[i], reinterpret_cast<cudaEvent_t>(ref), reinterpret_cast<cudaEvent_t>(events[i]));
    if (e != cudaSuccess) {
      set_error("events_elapsed: %s", cudaGetErrorString(e));
      return PPLL_ERR_CUDA;
    }
  }
  return PPLL_OK;
}

int ppll_gather_rows_u8(int n, int64_t width, const uint8_t* src, const int64_t* idx, void* dst,
                        int dst_dtype, const int64_t* labels_src, int64_t* labels_dst,
                        void* stream) {
  if (n < 0 || width < 1 || !src || !idx || !dst || (labels_src && !labels_dst) ||
      (dst_dtype != PPLL_F32 && dst_dtype != PPLL_BF16)) {
    set_error("gather_rows_u8: invalid arguments");
    return PPLL_ERR_ARG;
  }
  return launch_gather_rows_u8(n, width, src, idx, dst, dst_dtype, labels_src, labels_dst,
                               S(stream));
}

int ppll_count_correct(int B, int C, const void* logits, int ldz, int dtype,
                       const int64_t* labels, unsigned long long* count, void* stream) {
  if (B < 0 || C < 1 || !logits || !labels || !count) {
    set_error("count_correct: invalid arguments");
    return PPLL_ERR_ARG;
  }
  return launch_count_correct(B, C, logits, ldz, dtype, labels, count, S(stream));
}

int ppll_cast(int64_t n, const void* src, int src_dtype, void* dst, int dst_dtype, void* stream) {
  return launch_cast(n, src, src_dtype, dst, dst_dtype, S(stream));
}

int ppll_ring_publish(int* ready_word, int seq, void* stream) {
  return launch_ring_publish(ready_word, seq, S(stream));
}
int ppll_ring_wait(const int* ready_word, int seq, void* stream) {
  return launch_ring_wait(ready_word, seq, S(stream));
}
int ppll_ring_release(int* credit_word, void* stream) {
  return launch_ring_release(credit_word, S(stream));
}
int ppll_ring_wait_credit(const int* credit_word, int need, void* stream) {
  return launch_ring_wait(credit_word, need, S(stream), 1);
}
void ppll_set_ring_timeout_ms(long long ms) { g_ring_timeout_ns = ms > 0 ? ms * 1000000LL : 0; }
int ppll_ring_stall(int* out4, int clear) { return ring_stall_read(out4, clear != 0); }

int ppll_ipc_get_handle(void* dev_ptr, void* handle_out) {
  cudaIpcMemHandle_t h;
  PPLL_CUDA_CHECK(cudaIpcGetMemHandle(&h, dev_ptr));
  memcpy(handle_out, &h, sizeof(h));
  return PPLL_OK;
}
int ppll_ipc_open_handle(const void* handle, void** dev_ptr_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  PPLL_CUDA_CHECK(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return PPLL_OK;
}
int ppll_ipc_close_handle(void* dev_ptr) {
  PPLL_CUDA_CHECK(cudaIpcCloseMemHandle(dev_ptr));
  return PPLL_OK;
}
int ppll_enable_peer(int peer_device) {
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) { cudaGetLastError(); return PPLL_OK; }
  PPLL_CUDA_CHECK(e);
  return PPLL_OK;
}
void* ppll_dev_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    set_error("cudaMalloc(%zu) failed", bytes);
    cudaGetLastError();
    return nullptr;
  }
  cudaMemset(p, 0, bytes);
  return p;
}
int ppll_dev_free(void* p) {
  PPLL_CUDA_CHECK(cudaFree(p));
  return PPLL_OK;
}
int ppll_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return PPLL_OK;
  PPLL_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, S(stream)));
  return PPLL_OK;
}
int ppll_stream_sync(void* stream) {
  PPLL_CUDA_CHECK(cudaStreamSynchronize(S(stream)));
  return PPLL_OK;
}

}  // extern "C"
