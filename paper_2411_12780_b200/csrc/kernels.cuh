// Internal launcher declarations shared by capi.cu / stage.cu / gemm_tc.cu.
#pragma once
#include "common.cuh"

namespace ppll {

void note_launch(int n = 1);

// GEMM epilogue: v -> (+bias[n]) -> relu? -> ⊙[mask>0] -> C (and C2).
template <typename TO>
struct Epilogue {
  TO* C = nullptr;
  long ldc = 0;
  TO* C2 = nullptr;       // optional dual store (fused ring push)
  long ldc2 = 0;
  const float* bias = nullptr;
  int relu = 0;
  const TO* mask = nullptr;
  long ldmask = 0;
  float* partial = nullptr;  // split-K workspace (internal)

  __device__ __forceinline__ void apply(int m, int n, float v) const {
    if (bias) v += bias[n];
    if (relu) v = fmaxf(v, 0.f);
    if (mask) v = (to_f(mask[(long)m * ldmask + n]) > 0.f) ? v : 0.f;
    DT<TO>::st(C + (long)m * ldc + n, v);
    if (C2) DT<TO>::st(C2 + (long)m * ldc2 + n, v);
  }
};

template <typename TI, typename TO>
int launch_gemm_simt(int M, int N, int K, const TI* A, long a_rs, long a_cs, const TI* B,
                     long b_rs, long b_cs, const Epilogue<TO>& ep, float* ws, size_t ws_elems,
                     cudaStream_t s);

// tcgen05 GEMM (gemm_tc.cu).  a_kmajor: A(m,k)=A[m*lda+k] else A[k*lda+m];
// b_kmajor: B(k,n)=B[n*ldb+k] else B[k*ldb+n].  Returns PPLL_ERR_UNSUPPORTED
// when the shape/alignment cannot use TMA (caller then uses the SIMT engine).
template <typename TO>
int launch_gemm_tc(int M, int N, int K, const __nv_bfloat16* A, long lda, bool a_kmajor,
                   const __nv_bfloat16* B, long ldb, bool b_kmajor, const Epilogue<TO>& ep,
                   float* ws, size_t ws_elems, cudaStream_t s);

template <typename TO>
int launch_splitk_reduce(int M, int N, int splits, const float* ws, const Epilogue<TO>& ep,
                         cudaStream_t s);

template <typename T>
int launch_colsum(int M, int N, const T* G, int ld, float* db, cudaStream_t s);

template <typename T>
int launch_softmax_xent(int B, int C, const T* z, int ldz, const int64_t* y, T* dz, int lddz,
                        float* loss_hist, const int* step, int* err, cudaStream_t s);

int launch_nesterov(long n, float* th, float* v, const float* g, __nv_bfloat16* th_lp,
                    const float* lr_table, int* step, int max_step, float lr_host, float mu,
                    float wd, int* err, cudaStream_t s);

int launch_cast(long n, const void* src, int sd, void* dst, int dd, cudaStream_t s);
int launch_ring_publish(int* w, int seq, cudaStream_t s);
int launch_ring_wait(const int* w, int seq, cudaStream_t s);
int launch_ring_release(int* w, cudaStream_t s);

// linear-layer ops used by both the C-ABI and the stage runtime
int linear_fwd(int M, int K, int N, const void* X, int ldx, const void* W, const float* b,
               void* Y, int ldy, void* Y2, int ldy2, int relu, int dtype, float* ws,
               size_t ws_elems, cudaStream_t s);
int linear_dgrad(int M, int K, int N, const void* dY, int lddy, const void* W, const void* mask,
                 int ldmask, void* dX, int lddx, int dtype, float* ws, size_t ws_elems,
                 cudaStream_t s);
int linear_wgrad(int M, int K, int N, const void* X, int ldx, const void* dY, int lddy, float* dW,
                 float* db, int dtype, float* ws, size_t ws_elems, cudaStream_t s);

extern int g_gemm_engine;

}  // namespace ppll
