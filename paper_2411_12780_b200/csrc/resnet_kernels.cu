// Bandwidth-bound kernels of the ResNet local step (NHWC, sm_100a): im2col /
// col2im for the convolution-as-GEMM (the GEMM itself runs on the tcgen05
// engine), training-mode BatchNorm statistics / apply / backward with fixed-
// order (deterministic) reductions, the ReLU-mask, and global average pooling.
#include <math.h>
#include "common.cuh"
#include "kernels.cuh"
#include "resnet.cuh"

namespace ppll {

static int grid_for(long n, int threads = 256) {
  return (int)min((n + threads - 1) / threads, (long)148 * 16);
}

// ---------------------------------------------------------------------------
// im2col: x [N,H,W,C] -> col [N·Ho·Wo, Kp], column (r·k + s)·C + c, zero pad
// (spatial padding (k-1)/2 and columns >= k·k·C).  8-channel vectors when C%8==0.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void im2col_kernel(int N, int H, int W, int C, int k, int stride, int Ho, int Wo, int Kp,
                              const T* __restrict__ x, T* __restrict__ col) {
  pdl_entry();
  const int p = (k - 1) / 2;
  const long total = (long)N * Ho * Wo * Kp;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const int kk = (int)(idx % Kp);
    const long pix = idx / Kp;
    float v = 0.f;
    if (kk < k * k * C) {
      const int tap = kk / C, c = kk % C, r = tap / k, s = tap % k;
      const int wo = (int)(pix % Wo), ho = (int)((pix / Wo) % Ho), n = (int)(pix / ((long)Wo * Ho));
      const int h = ho * stride - p + r, w = wo * stride - p + s;
      if (h >= 0 && h < H && w >= 0 && w < W) v = to_f(x[(((long)n * H + h) * W + w) * C + c]);
    }
    DT<T>::st(col + idx, v);
  }
}

template <typename T>
__global__ void im2col_vec_kernel(int N, int H, int W, int C, int k, int stride, int Ho, int Wo,
                                  int Kp, const T* __restrict__ x, T* __restrict__ col) {
  pdl_entry();
  // one thread per 8-channel vector (16 B for bf16)
  const int p = (k - 1) / 2;
  const int C8 = C / 8, K8 = Kp / 8;
  const long total = (long)N * Ho * Wo * K8;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const int k8 = (int)(idx % K8);
    const long pix = idx / K8;
    uint4 v = make_uint4(0, 0, 0, 0);
    const int tap = k8 / C8, c8 = k8 % C8;
    if (tap < k * k) {
      const int r = tap / k, s = tap % k;
      const int wo = (int)(pix % Wo), ho = (int)((pix / Wo) % Ho), n = (int)(pix / ((long)Wo * Ho));
      const int h = ho * stride - p + r, w = wo * stride - p + s;
      if (h >= 0 && h < H && w >= 0 && w < W)
        v = *reinterpret_cast<const uint4*>(x + (((long)n * H + h) * W + w) * C + c8 * 8);
    }
    *reinterpret_cast<uint4*>(col + pix * Kp + (long)k8 * 8) = v;
  }
}

template <typename T>
int launch_im2col(int N, int H, int W, int C, int k, int stride, int Kp, const T* x, T* col,
                  cudaStream_t s) {
  const int p = (k - 1) / 2;
  const int Ho = (H + 2 * p - k) / stride + 1, Wo = (W + 2 * p - k) / stride + 1;
  if (sizeof(T) == 2 && C % 8 == 0 && Kp % 8 == 0) {
    const long n = (long)N * Ho * Wo * (Kp / 8);
    launch_k(im2col_vec_kernel<T>, grid_for(n), 256, 0, s, N, H, W, C, k, stride, Ho, Wo, Kp, x, col);
  } else {
    const long n = (long)N * Ho * Wo * Kp;
    launch_k(im2col_kernel<T>, grid_for(n), 256, 0, s, N, H, W, C, k, stride, Ho, Wo, Kp, x, col);
  }
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// ---------------------------------------------------------------------------
// col2im (gather): dx[n,h,w,c] = Σ_taps dcol[pix(n,ho,wo), tap·C + c]
//   (+ dres[n,h,w,c]) and optionally ⊙ [mask > 0] (the ReLU before the conv)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void col2im_kernel(int N, int H, int W, int C, int k, int stride, int Ho, int Wo, int Kp,
                              const T* __restrict__ dcol, const T* __restrict__ dres,
                              const T* __restrict__ mask, T* __restrict__ dx) {
  pdl_entry();
  const int p = (k - 1) / 2;
  const long total = (long)N * H * W * C;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const int c = (int)(idx % C);
    const long q = idx / C;
    const int w = (int)(q % W), h = (int)((q / W) % H), n = (int)(q / ((long)W * H));
    float acc = 0.f;
    for (int r = 0; r < k; ++r) {
      const int hh = h + p - r;
      if (hh < 0 || hh % stride) continue;
      const int ho = hh / stride;
      if (ho >= Ho) continue;
      for (int s2 = 0; s2 < k; ++s2) {
        const int ww = w + p - s2;
        if (ww < 0 || ww % stride) continue;
        const int wo = ww / stride;
        if (wo >= Wo) continue;
        acc += to_f(dcol[(((long)n * Ho + ho) * Wo + wo) * Kp + (r * k + s2) * C + c]);
      }
    }
    if (dres) acc += to_f(dres[idx]);
    if (mask && !(to_f(mask[idx]) > 0.f)) acc = 0.f;
    DT<T>::st(dx + idx, acc);
  }
}

// bf16, C % 8 == 0: one thread per (pixel, 8-channel group), 16-B gathers
__device__ __forceinline__ void acc8(float* a, uint4 q) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f = __bfloat1622float2(h[j]);
    a[2 * j] += f.x;
    a[2 * j + 1] += f.y;
  }
}
__global__ void col2im_vec_kernel(int N, int H, int W, int C, int k, int stride, int Ho, int Wo,
                                  int Kp, const __nv_bfloat16* __restrict__ dcol,
                                  const __nv_bfloat16* __restrict__ dres,
                                  const __nv_bfloat16* __restrict__ mask,
                                  __nv_bfloat16* __restrict__ dx) {
  pdl_entry();
  const int p = (k - 1) / 2, C8 = C / 8;
  const long total = (long)N * H * W * C8;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const int c8 = (int)(idx % C8);
    const long q = idx / C8;
    const int w = (int)(q % W), h = (int)((q / W) % H), n = (int)(q / ((long)W * H));
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int r = 0; r < k; ++r) {
      const int hh = h + p - r;
      if (hh < 0 || hh % stride) continue;
      const int ho = hh / stride;
      if (ho >= Ho) continue;
      for (int s2 = 0; s2 < k; ++s2) {
        const int ww = w + p - s2;
        if (ww < 0 || ww % stride) continue;
        const int wo = ww / stride;
        if (wo >= Wo) continue;
        acc8(a, *reinterpret_cast<const uint4*>(
                    dcol + (((long)n * Ho + ho) * Wo + wo) * Kp + (r * k + s2) * C + c8 * 8));
      }
    }
    const long o = q * C + c8 * 8;
    if (dres) acc8(a, *reinterpret_cast<const uint4*>(dres + o));
    if (mask) {
      const uint4 mq = *reinterpret_cast<const uint4*>(mask + o);
      const __nv_bfloat162* mh = reinterpret_cast<const __nv_bfloat162*>(&mq);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(mh[j]);
        if (!(f.x > 0.f)) a[2 * j] = 0.f;
        if (!(f.y > 0.f)) a[2 * j + 1] = 0.f;
      }
    }
    uint4 out;
    __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
    for (int j = 0; j < 4; ++j) oh[j] = __floats2bfloat162_rn(a[2 * j], a[2 * j + 1]);
    *reinterpret_cast<uint4*>(dx + o) = out;
  }
}

template <typename T>
int launch_col2im(int N, int H, int W, int C, int k, int stride, int Kp, const T* dcol,
                  const T* dres, const T* mask, T* dx, cudaStream_t s) {
  const int p = (k - 1) / 2;
  const int Ho = (H + 2 * p - k) / stride + 1, Wo = (W + 2 * p - k) / stride + 1;
  if constexpr (sizeof(T) == 2) {
    if (C % 8 == 0 && Kp % 8 == 0) {
      launch_k(col2im_vec_kernel, grid_for((long)N * H * W * C / 8), 256, 0, s, 
          N, H, W, C, k, stride, Ho, Wo, Kp, (const __nv_bfloat16*)dcol,
          (const __nv_bfloat16*)dres, (const __nv_bfloat16*)mask, (__nv_bfloat16*)dx);
      note_launch();
      PPLL_LAUNCH_CHECK();
      return PPLL_OK;
    }
  }
  launch_k(col2im_kernel<T>, grid_for((long)N * H * W * C), 256, 0, s, N, H, W, C, k, stride, Ho, Wo,
                                                                  Kp, dcol, dres, mask, dx);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// ---------------------------------------------------------------------------
// BatchNorm (training mode) over the P rows of a [P, C] NHWC activation.
// Statistics: per block, threads accumulate (count, mean, M2) with Welford
// over strided rows, merged in a fixed order (Chan); a second kernel merges
// the block partials in order -> mean, rstd.  Deterministic and stable.
// ---------------------------------------------------------------------------
struct Welford { float n, mean, m2; };
__device__ __forceinline__ Welford wf_merge(Welford a, Welford b) {
  if (b.n == 0.f) return a;
  if (a.n == 0.f) return b;
  const float n = a.n + b.n, d = b.mean - a.mean;
  return {n, a.mean + d * b.n / n, a.m2 + b.m2 + d * d * a.n * b.n / n};
}

// block (32 channels x 8 row-lanes); grid (C/32, chunks)
template <typename T>
__global__ void bn_stats_part_kernel(int P, int C, const T* __restrict__ z, int rpc,
                                     float* __restrict__ part) {
  pdl_entry();
  __shared__ Welford red[8][33];
  const int c = blockIdx.x * 32 + threadIdx.x;
  const int r0 = blockIdx.y * rpc, r1 = min(P, r0 + rpc);
  Welford w = {0.f, 0.f, 0.f};
  if (c < C)
    for (int r = r0 + threadIdx.y; r < r1; r += 8) {
      const float v = to_f(z[(long)r * C + c]);
      w.n += 1.f;
      const float d = v - w.mean;
      w.mean += d / w.n;
      w.m2 += d * (v - w.mean);
    }
  red[threadIdx.y][threadIdx.x] = w;
  __syncthreads();
  if (threadIdx.y == 0 && c < C) {
    Welford t = red[0][threadIdx.x];
    for (int k = 1; k < 8; ++k) t = wf_merge(t, red[k][threadIdx.x]);
    float* o = part + ((long)blockIdx.y * C + c) * 3;
    o[0] = t.n; o[1] = t.mean; o[2] = t.m2;
  }
}

// one warp per channel: lanes merge strided chunks, then a butterfly whose
// every merge is ordered (lower lane first) — identical on all lanes, and
// deterministic
__global__ void bn_stats_final_kernel(int chunks, int C, const float* __restrict__ part,
                                      float* __restrict__ mean, float* __restrict__ rstd) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= C) return;
  Welford t = {0.f, 0.f, 0.f};
  for (int k = lane; k < chunks; k += 32) {
    const float* o = part + ((long)k * C + c) * 3;
    t = wf_merge(t, Welford{o[0], o[1], o[2]});
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Welford u;
    u.n = __shfl_xor_sync(0xffffffffu, t.n, off);
    u.mean = __shfl_xor_sync(0xffffffffu, t.mean, off);
    u.m2 = __shfl_xor_sync(0xffffffffu, t.m2, off);
    t = (lane & off) ? wf_merge(u, t) : wf_merge(t, u);
  }
  if (lane == 0) {
    mean[c] = t.mean;
    rstd[c] = rsqrtf(t.m2 / fmaxf(t.n, 1.f) + kBnEps);
  }
}

int bn_chunks(int P) { return max(1, min(ceil_div(P, 256), 256)); }

template <typename T>
int launch_bn_stats(int P, int C, const T* z, float* part, float* mean, float* rstd,
                    cudaStream_t s) {
  const int chunks = bn_chunks(P);
  const int rpc = ceil_div(P, chunks);
  launch_k(bn_stats_part_kernel<T>, dim3(ceil_div(C, 32), chunks), dim3(32, 8), 0, s, P, C, z, rpc, part);
  note_launch();
  launch_k(bn_stats_final_kernel, ceil_div(C, 8), 256, 0, s, chunks, C, part, mean, rstd);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// y = act( (z - mean)·rstd·g + b  [+ (z2 - mean2)·rstd2·g2 + b2 | + res] )
template <typename T>
__global__ void bn_apply_kernel(long total, int C, const T* __restrict__ z, const float* __restrict__ mean,
                                const float* __restrict__ rstd, const float* __restrict__ g,
                                const float* __restrict__ b, const T* __restrict__ z2,
                                const float* __restrict__ mean2, const float* __restrict__ rstd2,
                                const float* __restrict__ g2, const float* __restrict__ b2,
                                const T* __restrict__ res, int relu, T* __restrict__ y) {
  pdl_entry();
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const int c = (int)(idx % C);
    float v = (to_f(z[idx]) - mean[c]) * rstd[c] * g[c] + b[c];
    if (z2) v += (to_f(z2[idx]) - mean2[c]) * rstd2[c] * g2[c] + b2[c];
    if (res) v += to_f(res[idx]);
    if (relu) v = fmaxf(v, 0.f);
    DT<T>::st(y + idx, v);
  }
}

template <typename T>
int launch_bn_apply(long P, int C, const T* z, const float* mean, const float* rstd, const float* g,
                    const float* b, const T* z2, const float* mean2, const float* rstd2,
                    const float* g2, const float* b2, const T* res, int relu, T* y, cudaStream_t s) {
  const long total = P * C;
  launch_k(bn_apply_kernel<T>, grid_for(total), 256, 0, s, total, C, z, mean, rstd, g, b, z2, mean2,
                                                     rstd2, g2, b2, res, relu, y);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// dy_eff = dout ⊙ [out > 0]  (materialised: feeds BN backward and the shortcut)
template <typename T>
__global__ void relu_mask_kernel(long total, const T* __restrict__ dout, const T* __restrict__ out,
                                 T* __restrict__ dy) {
  pdl_entry();
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x)
    DT<T>::st(dy + idx, to_f(out[idx]) > 0.f ? to_f(dout[idx]) : 0.f);
}

template <typename T>
int launch_relu_mask(long n, const T* dout, const T* out, T* dy, cudaStream_t s) {
  launch_k(relu_mask_kernel<T>, grid_for(n), 256, 0, s, n, dout, out, dy);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// BN backward part: per-chunk Σ dy·xhat, Σ dy (fixed order) -> part[chunk][2][C]
template <typename T>
__global__ void bn_bwd_part_kernel(int P, int C, const T* __restrict__ dy, const T* __restrict__ z,
                                   const float* __restrict__ mean, const float* __restrict__ rstd,
                                   int rpc, float* __restrict__ part) {
  pdl_entry();
  __shared__ float red[2][8][33];
  const int c = blockIdx.x * 32 + threadIdx.x;
  const int r0 = blockIdx.y * rpc, r1 = min(P, r0 + rpc);
  float sg = 0.f, sb = 0.f;
  if (c < C) {
    const float mu = mean[c], rs = rstd[c];
    for (int r = r0 + threadIdx.y; r < r1; r += 8) {
      const float d = to_f(dy[(long)r * C + c]);
      sg += d * (to_f(z[(long)r * C + c]) - mu) * rs;
      sb += d;
    }
  }
  red[0][threadIdx.y][threadIdx.x] = sg;
  red[1][threadIdx.y][threadIdx.x] = sb;
  __syncthreads();
  if (threadIdx.y == 0 && c < C) {
    float a = 0.f, b = 0.f;
    for (int k = 0; k < 8; ++k) {
      a += red[0][k][threadIdx.x];
      b += red[1][k][threadIdx.x];
    }
    part[((long)blockIdx.y * 2 + 0) * C + c] = a;
    part[((long)blockIdx.y * 2 + 1) * C + c] = b;
  }
}

// one warp per channel: lane-strided partial sums, fixed butterfly
__global__ void bn_bwd_final_kernel(int chunks, int C, const float* __restrict__ part,
                                    float* __restrict__ dg, float* __restrict__ db) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= C) return;
  float a = 0.f, b = 0.f;
  for (int k = lane; k < chunks; k += 32) {
    a += part[((long)k * 2 + 0) * C + c];
    b += part[((long)k * 2 + 1) * C + c];
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0) {
    dg[c] = a;
    db[c] = b;
  }
}

// dz = g·rstd/P · (P·dy − db − xhat·dg)
template <typename T>
__global__ void bn_bwd_dx_kernel(long total, int C, float invP, const T* __restrict__ dy,
                                 const T* __restrict__ z, const float* __restrict__ mean,
                                 const float* __restrict__ rstd, const float* __restrict__ g,
                                 const float* __restrict__ dg, const float* __restrict__ db,
                                 T* __restrict__ dz) {
  pdl_entry();
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const int c = (int)(idx % C);
    const float rs = rstd[c];
    const float xh = (to_f(z[idx]) - mean[c]) * rs;
    DT<T>::st(dz + idx, g[c] * rs * (to_f(dy[idx]) - (db[c] + xh * dg[c]) * invP));
  }
}

template <typename T>
int launch_bn_bwd(int P, int C, const T* dy, const T* z, const float* mean, const float* rstd,
                  const float* g, float* part, float* dg, float* db, T* dz, cudaStream_t s) {
  const int chunks = bn_chunks(P);
  const int rpc = ceil_div(P, chunks);
  launch_k(bn_bwd_part_kernel<T>, dim3(ceil_div(C, 32), chunks), dim3(32, 8), 0, s, P, C, dy, z, mean,
                                                                              rstd, rpc, part);
  note_launch();
  launch_k(bn_bwd_final_kernel, ceil_div(C, 8), 256, 0, s, chunks, C, part, dg, db);
  note_launch();
  const long total = (long)P * C;
  launch_k(bn_bwd_dx_kernel<T>, grid_for(total), 256, 0, s, total, C, 1.f / (float)P, dy, z, mean, rstd,
                                                      g, dg, db, dz);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// ---------------------------------------------------------------------------
// global average pool over H·W and its adjoint
// ---------------------------------------------------------------------------
template <typename T>
__global__ void gap_kernel(int N, int HW, int C, const T* __restrict__ x, T* __restrict__ out) {
  pdl_entry();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= N * C) return;
  const int n = idx / C, c = idx % C;
  float s = 0.f;
  for (int i = 0; i < HW; ++i) s += to_f(x[((long)n * HW + i) * C + c]);
  DT<T>::st(out + idx, s / (float)HW);
}

template <typename T>
__global__ void gap_bwd_kernel(int N, int HW, int C, const T* __restrict__ dp, T* __restrict__ dx) {
  pdl_entry();
  const long total = (long)N * HW * C;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const int c = (int)(idx % C);
    const int n = (int)(idx / ((long)HW * C));
    DT<T>::st(dx + idx, to_f(dp[(long)n * C + c]) / (float)HW);
  }
}

template <typename T>
int launch_gap(int N, int HW, int C, const T* x, T* out, cudaStream_t s) {
  launch_k(gap_kernel<T>, ceil_div(N * C, 256), 256, 0, s, N, HW, C, x, out);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}
template <typename T>
int launch_gap_bwd(int N, int HW, int C, const T* dp, T* dx, cudaStream_t s) {
  launch_k(gap_bwd_kernel<T>, grid_for((long)N * HW * C), 256, 0, s, N, HW, C, dp, dx);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

#define INST(T)                                                                                   \
  template int launch_im2col<T>(int, int, int, int, int, int, int, const T*, T*, cudaStream_t);  \
  template int launch_col2im<T>(int, int, int, int, int, int, int, const T*, const T*, const T*, \
                                T*, cudaStream_t);                                                \
  template int launch_bn_stats<T>(int, int, const T*, float*, float*, float*, cudaStream_t);     \
  template int launch_bn_apply<T>(long, int, const T*, const float*, const float*, const float*, \
                                  const float*, const T*, const float*, const float*,            \
                                  const float*, const float*, const T*, int, T*, cudaStream_t);  \
  template int launch_relu_mask<T>(long, const T*, const T*, T*, cudaStream_t);                 \
  template int launch_bn_bwd<T>(int, int, const T*, const T*, const float*, const float*,       \
                                const float*, float*, float*, float*, T*, cudaStream_t);         \
  template int launch_gap<T>(int, int, int, const T*, T*, cudaStream_t);                         \
  template int launch_gap_bwd<T>(int, int, int, const T*, T*, cudaStream_t);
INST(float)
INST(__nv_bfloat16)
#undef INST

}  // namespace ppll
