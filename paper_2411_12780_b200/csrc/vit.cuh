// ViT kernel launchers (vit_kernels.cu), used by the ViT stage executor.
#pragma once
#include "common.cuh"

namespace ppll {

constexpr float kLnEps = 1e-5f;

template <typename T>
int launch_ln_fwd(int M, int D, const T* x, long ldx, const float* g, const float* b, T* y,
                  long ldy, float* mean, float* rstd, cudaStream_t s);
// dx may be null (only gamma/beta gradients wanted); part/dg/db may be null;
// dxsum (nullable) receives Σ_rows of the dx output — the bias gradient of the
// layer that produced dy's residual stream, fused (needs D % 128 == 0).
// part must hold ln_bwd_blocks(M) * 3 * D floats.
template <typename T>
int launch_ln_bwd(int M, int D, const T* dy, long lddy, const T* x, long ldx, const float* mean,
                  const float* rstd, const float* g, const T* dres, long ldres, T* dx, long lddx,
                  float* part, float* dg, float* db, cudaStream_t s, float* dxsum = nullptr,
                  struct LnDefer* defer = nullptr);
// Deferred LayerNorm parameter reductions: a stage's backward records each
// LN backward's per-block partials (dγ, dβ and the fused Σ-rows bias gradient)
// instead of reducing them right away, and one batched launch reduces them all
// before the optimizer (same fixed summation order: bitwise identical).
struct LnReduceTask {
  const float* part;
  float *o0, *o1, *o2;
  int nblk, D, NS, blk0;   // blk0: first block of this task in the batched grid
};
struct LnDefer {
  static constexpr int kMax = 24;
  LnReduceTask t[kMax];
  int n = 0, blocks = 0;
};
int launch_ln_reduce_deferred(const LnDefer& d, cudaStream_t s);
// LayerNorm backward fused into the data-gradient GEMM that feeds it
// (gemm_ln.cu, D = 384): dx = LN_bwd(dY·Wᵀ) (+ dres), column partials recorded
// in `defer`; PPLL_ERR_UNSUPPORTED outside its range.
int launch_gemm_ln_fwd(int M, int K, const __nv_bfloat16* A, const __nv_bfloat16* W,
                       const float* bias, const __nv_bfloat16* res, const float* g, const float* b,
                       __nv_bfloat16* x1, __nv_bfloat16* xn, float* mean, float* rstd,
                       cudaStream_t s);
int launch_gemm_ln_bwd(int M, int K, const __nv_bfloat16* dY, const __nv_bfloat16* W,
                       const __nv_bfloat16* x, const float* mean, const float* rstd,
                       const float* g, const __nv_bfloat16* dres, __nv_bfloat16* dx, float* part,
                       float* dg, float* db, float* dxsum, LnDefer* defer, cudaStream_t s);
int ln_bwd_blocks(int M);
template <typename T>
int launch_attn_fwd(int B, int Tn, int H, int dh, const T* qkv, T* o, float* lse, cudaStream_t s);
// attention of the cls query alone (head_dim 64): o [B, D] compact, lse [B·H];
// backward writes the full dqkv (zero Q rows past the cls row) and the
// per-image column sums of dqkv into bpart [B, 3D] (nullable)
template <typename T>
int launch_cls_attn_fwd(int B, int Tn, int H, const T* qkv, T* o, float* lse, cudaStream_t s);
template <typename T>
int launch_cls_attn_bwd(int B, int Tn, int H, const T* qkv, const T* o, const T* dout,
                        const float* lse, T* dqkv, float* bpart, cudaStream_t s);
template <typename T>
int launch_attn_bwd(int B, int Tn, int H, int dh, const T* qkv, const T* o, const T* dout,
                    const float* lse, T* dqkv, cudaStream_t s);
// tcgen05 attention (attn_tc.cu): bf16, head_dim 64, T <= 128
bool attn_tc_supported(int Tn, int dh);
int launch_attn_tc_fwd(int B, int Tn, int H, const __nv_bfloat16* qkv, __nv_bfloat16* o,
                       float* lse, cudaStream_t s);
// bias_part (nullable): [B, 3D] per-image column sums of dqkv (fused bias grad)
int launch_attn_tc_bwd(int B, int Tn, int H, const __nv_bfloat16* qkv, const __nv_bfloat16* o,
                       const __nv_bfloat16* dout, const float* lse, __nv_bfloat16* dqkv,
                       cudaStream_t s, float* bias_part = nullptr);
extern int g_attn_engine;   // 0 auto (tcgen05 when supported), 1 SIMT

template <typename T>
int launch_patchify(int B, int C, int HW, int p, const T* img, T* out, cudaStream_t s);
template <typename T>
int launch_embed(int B, int P, int D, const T* tok, const float* cls, const float* pos, T* x,
                 cudaStream_t s);
template <typename T>
int launch_embed_bwd(int B, int P, int D, const T* dx, T* dtok, float* dcls, float* dpos,
                     cudaStream_t s);
template <typename T>
int launch_scatter_cls(int B, int Tn, int D, const T* dz, T* dx, cudaStream_t s);

}  // namespace ppll
