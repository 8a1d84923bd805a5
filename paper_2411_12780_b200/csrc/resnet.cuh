// ResNet kernel launchers (resnet_kernels.cu), used by the ResNet stage executor.
#pragma once
#include "common.cuh"

namespace ppll {

constexpr float kBnEps = 1e-5f;

template <typename T>
int launch_im2col(int N, int H, int W, int C, int k, int stride, int Kp, const T* x, T* col,
                  cudaStream_t s);
template <typename T>
int launch_col2im(int N, int H, int W, int C, int k, int stride, int Kp, const T* dcol,
                  const T* dres, const T* mask, T* dx, cudaStream_t s);
int bn_chunks(int P);   // part buffers hold bn_chunks(P) * 3 * C floats
template <typename T>
int launch_bn_stats(int P, int C, const T* z, float* part, float* mean, float* rstd,
                    cudaStream_t s);
template <typename T>
int launch_bn_apply(long P, int C, const T* z, const float* mean, const float* rstd, const float* g,
                    const float* b, const T* z2, const float* mean2, const float* rstd2,
                    const float* g2, const float* b2, const T* res, int relu, T* y, cudaStream_t s);
template <typename T>
int launch_relu_mask(long n, const T* dout, const T* out, T* dy, cudaStream_t s);
template <typename T>
int launch_bn_bwd(int P, int C, const T* dy, const T* z, const float* mean, const float* rstd,
                  const float* g, float* part, float* dg, float* db, T* dz, cudaStream_t s);
// single-cluster fused BN (bn_cluster.cu, bf16 NHWC): statistics of z (and
// z2) + y = act(BN(z) [+ BN2(z2) | + res]) in one launch; backward from dout
// (masked by out > 0 when out != NULL; the masked dy stored when dy_store !=
// NULL) to dz (and dz2 of a second BN sharing dy).  PPLL_ERR_UNSUPPORTED when
// the shape / size is outside the fused kernel's range.
// Tensors past the single-cluster range use the GRID form when the caller
// provides its scratch (one co-resident CTA per SM, cooperative launch;
// per-CTA partials + a self-resetting barrier {arrivals, generation}, zeroed
// once; a watchdog sets kErrSync in *err instead of hanging).  One BnGrid per
// stream of concurrently running BN launches.
struct BnGrid {
  void* part;      // >= 148 * 128 float4
  unsigned* bar;   // 2 words, zero-initialised
  int* err;        // sticky error word (nullable)
};
int launch_bn_fwd_fused(int P, int C, const __nv_bfloat16* z, const float* g, const float* b,
                        float* mean, float* rstd, const __nv_bfloat16* z2, const float* g2,
                        const float* b2, float* mean2, float* rstd2, const __nv_bfloat16* res,
                        int relu, __nv_bfloat16* y, cudaStream_t s, const BnGrid* grid = nullptr);
int launch_bn_bwd_fused(int P, int C, const __nv_bfloat16* dout, const __nv_bfloat16* out,
                        __nv_bfloat16* dy_store, const __nv_bfloat16* z, const float* mean,
                        const float* rstd, const float* g, float* dg, float* db, __nv_bfloat16* dz,
                        const __nv_bfloat16* z2, const float* mean2, const float* rstd2,
                        const float* g2, float* dg2, float* db2, __nv_bfloat16* dz2,
                        cudaStream_t s, const BnGrid* grid = nullptr);
template <typename T>
int launch_gap(int N, int HW, int C, const T* x, T* out, cudaStream_t s);

template <typename TO> struct Epilogue;
// implicit-GEMM 3x3 / stride-1 convolution on tcgen05 (conv_tc.cu); dgrad =
// transposed convolution with the forward weights.  PPLL_ERR_UNSUPPORTED for
// shapes it does not cover.
int launch_conv3x3_tc(int N, int H, int W, int CI, int CO, const __nv_bfloat16* x,
                      const __nv_bfloat16* w, bool dgrad, const Epilogue<__nv_bfloat16>& ep,
                      cudaStream_t s);
template <typename T>
int launch_gap_bwd(int N, int HW, int C, const T* dp, T* dx, cudaStream_t s);
// implicit-GEMM weight gradient of the 3x3 / stride-1 convolution (conv_tc.cu):
// dw [9·CI, CO] fp32 (the GEMM weight layout) from x [N,H,W,CI] and dz [P,CO];
// ws: split-K partials (splits·9·CI·CO floats).  PPLL_ERR_UNSUPPORTED outside
// the kernel's shapes.
int launch_conv3x3_wgrad_tc(int N, int H, int W, int CI, int CO, const __nv_bfloat16* x,
                            const __nv_bfloat16* dz, float* dw, float* ws, size_t ws_elems,
                            cudaStream_t s);

}  // namespace ppll
