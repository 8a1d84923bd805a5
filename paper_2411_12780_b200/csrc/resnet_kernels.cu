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

// unsigned 32-bit division by a runtime constant: q = (umulhi(n, m) + n) >> s
// (valid for n < 2^31); replaces the 64-bit divisions of the index math
struct FastDiv {
  unsigned d, m, s;
  FastDiv() = default;
  explicit FastDiv(unsigned dv) : d(dv) {
    s = 0;
    while ((1u << s) < dv) ++s;
    m = (unsigned)((((unsigned long long)1 << 32) * ((1ull << s) - dv)) / dv + 1);
  }
  __device__ __forceinline__ unsigned div(unsigned n) const { return (__umulhi(n, m) + n) >> s; }
};

// ---------------------------------------------------------------------------
// im2col: x [N,H,W,C] -> col [N·Ho·Wo, Kp], column (r·k + s)·C + c, zero pad
// (spatial padding (k-1)/2 and columns >= k·k·C).  8-channel vectors when C%8==0.
// ---------------------------------------------------------------------------
// scalar form (C % 8 != 0, e.g. the 3-channel stem): one thread per 2-element
// pair of a column row, 32-bit fast-division index math
template <typename T>
__global__ void im2col_kernel(int total, int H, int W, int C, int k, int stride, int Kp,
                              FastDiv fKp, FastDiv fC, FastDiv fk, FastDiv fWo, FastDiv fHo,
                              const T* __restrict__ x, T* __restrict__ col) {
  pdl_entry();
  const int p = (k - 1) / 2;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += gridDim.x * blockDim.x) {
    const unsigned pix = fKp.div(idx), kk = idx - pix * fKp.d;
    float v = 0.f;
    if (kk < (unsigned)(k * k * C)) {
      const unsigned tap = fC.div(kk), c = kk - tap * fC.d;
      const unsigned r = fk.div(tap), sx = tap - r * fk.d;
      const unsigned q = fWo.div(pix), wo = pix - q * fWo.d;
      const unsigned n = fHo.div(q), ho = q - n * fHo.d;
      const int h = (int)ho * stride - p + (int)r, w = (int)wo * stride - p + (int)sx;
      if (h >= 0 && h < H && w >= 0 && w < W) v = to_f(x[(((long)n * H + h) * W + w) * C + c]);
    }
    DT<T>::st(col + idx, v);
  }
}

__global__ void im2col_vec_kernel(int total, int H, int W, int C, int k, int stride, int Kp,
                                  FastDiv fK8, FastDiv fC8, FastDiv fk, FastDiv fWo, FastDiv fHo,
                                  const __nv_bfloat16* __restrict__ x,
                                  __nv_bfloat16* __restrict__ col) {
  pdl_entry();
  // one thread per 8-channel vector (16 B); 32-bit fast-division index math
  const int p = (k - 1) / 2;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += gridDim.x * blockDim.x) {
    const unsigned pix = fK8.div(idx), k8 = idx - pix * fK8.d;
    const unsigned tap = fC8.div(k8), c8 = k8 - tap * fC8.d;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (tap < (unsigned)(k * k)) {
      const unsigned r = fk.div(tap), sx = tap - r * fk.d;
      const unsigned q = fWo.div(pix), wo = pix - q * fWo.d;
      const unsigned n = fHo.div(q), ho = q - n * fHo.d;
      const int h = (int)ho * stride - p + (int)r, w = (int)wo * stride - p + (int)sx;
      if (h >= 0 && h < H && w >= 0 && w < W)
        v = *reinterpret_cast<const uint4*>(x + (((long)n * H + h) * W + w) * C + c8 * 8);
    }
    *reinterpret_cast<uint4*>(col + (long)pix * Kp + (long)k8 * 8) = v;
  }
}

template <typename T>
int launch_im2col(int N, int H, int W, int C, int k, int stride, int Kp, const T* x, T* col,
                  cudaStream_t s) {
  const int p = (k - 1) / 2;
  const int Ho = (H + 2 * p - k) / stride + 1, Wo = (W + 2 * p - k) / stride + 1;
  const long nv = (long)N * Ho * Wo * (Kp / 8);
  if (sizeof(T) == 2 && C % 8 == 0 && Kp % 8 == 0 && nv < (1L << 31)) {
    launch_k(im2col_vec_kernel, grid_for(nv), 256, 0, s, (int)nv, H, W, C, k, stride, Kp,
             FastDiv(Kp / 8), FastDiv(C / 8), FastDiv(k), FastDiv(Wo), FastDiv(Ho),
             (const __nv_bfloat16*)x, (__nv_bfloat16*)col);
  } else {
    const long n = (long)N * Ho * Wo * Kp;
    if (n >= (1L << 31)) {
      set_error("im2col: %ld elements exceed the 32-bit index path", n);
      return PPLL_ERR_UNSUPPORTED;
    }
    launch_k(im2col_kernel<T>, grid_for(n), 256, 0, s, (int)n, H, W, C, k, stride, Kp,
             FastDiv(Kp), FastDiv(C), FastDiv(k), FastDiv(Wo), FastDiv(Ho), x, col);
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
__global__ void col2im_vec_kernel(int total, int H, int W, int C, int k, int stride, int Ho, int Wo,
                                  int Kp, FastDiv fC8, FastDiv fW, FastDiv fH,
                                  const __nv_bfloat16* __restrict__ dcol,
                                  const __nv_bfloat16* __restrict__ dres,
                                  const __nv_bfloat16* __restrict__ mask,
                                  __nv_bfloat16* __restrict__ dx) {
  pdl_entry();
  const int p = (k - 1) / 2;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += gridDim.x * blockDim.x) {
    const unsigned q = fC8.div(idx), c8 = idx - q * fC8.d;
    const unsigned q2 = fW.div(q), wq = q - q2 * fW.d;
    const unsigned n = fH.div(q2);
    const int h = (int)(q2 - n * fH.d);
    const int w = (int)wq;
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
    const long o = (long)q * C + c8 * 8;
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
    const long nv = (long)N * H * W * C / 8;
    if (C % 8 == 0 && Kp % 8 == 0 && nv < (1L << 31)) {
      launch_k(col2im_vec_kernel, grid_for(nv), 256, 0, s, (int)nv, H, W, C, k, stride, Ho, Wo, Kp,
               FastDiv(C / 8), FastDiv(W), FastDiv(H), (const __nv_bfloat16*)dcol,
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

// ---------------------------------------------------------------------------
// Vectorised NHWC forms (bf16, C % 8 == 0, 256 % (C/8) == 0): a thread owns
// one 16-B vector of 8 channels of a row; a 256-thread block covers
// RB = 256·8/C rows per pass, fully coalesced.  Statistics accumulate per
// thread as shifted sums (shift = the thread's first value, so the variance
// does not cancel), become Welford triples, and merge in a fixed smem tree
// (deterministic).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void unpack8(const uint4& q, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 t = __bfloat1622float2(h[e]);
    f[2 * e] = t.x;
    f[2 * e + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 q;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
  for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
  return q;
}
static bool bn_vec_ok(int C, const void* a, const void* b = nullptr, const void* c = nullptr) {
  auto al = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return C % 8 == 0 && C <= 256 && 256 % (C / 8) == 0 && al(a) && al(b) && al(c);
}
static int bn_vec_rpc(int P, int C) {
  const int RB = 256 / (C / 8);
  int rpc = max(RB * 8, ceil_div(P, bn_chunks(P)));
  return ceil_div(rpc, RB) * RB;
}

__global__ void __launch_bounds__(256)
bn_stats_part_vkernel(int P, int C, const __nv_bfloat16* __restrict__ z, int rpc,
                      float* __restrict__ part) {
  pdl_entry();
  __shared__ float red[256 * 8 * 3];          // [RB][C][3] Welford triples
  const int V = C / 8, RB = 256 / V, t = threadIdx.x, vc = t % V, ro = t / V;
  const int r0 = blockIdx.x * rpc, r1 = min(P, r0 + rpc);
  float K[8], sm[8], sq[8];
  int n = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) K[e] = sm[e] = sq[e] = 0.f;
  // four rows' loads in flight per thread before any is consumed (same
  // accumulation order as one row at a time)
  for (int rb = r0 + ro; rb < r1; rb += 4 * RB) {
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (rb + u * RB < r1) q[u] = *reinterpret_cast<const uint4*>(z + (long)(rb + u * RB) * C + vc * 8);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (rb + u * RB >= r1) break;
      float v[8];
      unpack8(q[u], v);
      if (n == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) K[e] = v[e];
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float d = v[e] - K[e];
        sm[e] += d;
        sq[e] = fmaf(d, d, sq[e]);
      }
      ++n;
    }
  }
  const float fn = (float)n;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    float* w = red + ((long)ro * C + vc * 8 + e) * 3;
    w[0] = fn;
    w[1] = n ? K[e] + sm[e] / fn : 0.f;
    w[2] = n ? fmaxf(sq[e] - sm[e] * sm[e] / fn, 0.f) : 0.f;
  }
  __syncthreads();
  for (int stride = RB / 2; stride >= 1; stride >>= 1) {
    for (int i = t; i < stride * C; i += 256) {
      float* a = red + (long)i * 3;
      const float* b = red + ((long)i + (long)stride * C) * 3;
      const Welford m = wf_merge(Welford{a[0], a[1], a[2]}, Welford{b[0], b[1], b[2]});
      a[0] = m.n; a[1] = m.mean; a[2] = m.m2;
    }
    __syncthreads();
  }
  for (int c = t; c < C; c += 256) {
    float* o = part + ((long)blockIdx.x * C + c) * 3;
    o[0] = red[c * 3]; o[1] = red[c * 3 + 1]; o[2] = red[c * 3 + 2];
  }
}

__global__ void __launch_bounds__(256)
bn_bwd_part_vkernel(int P, int C, const __nv_bfloat16* __restrict__ dy,
                    const __nv_bfloat16* __restrict__ z, const float* __restrict__ mean,
                    const float* __restrict__ rstd, int rpc, float* __restrict__ part) {
  pdl_entry();
  __shared__ float red[256 * 8 * 2];          // [RB][C][2]
  const int V = C / 8, RB = 256 / V, t = threadIdx.x, vc = t % V, ro = t / V;
  const int r0 = blockIdx.x * rpc, r1 = min(P, r0 + rpc);
  float mu[8], rs[8], sg[8], sb[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    mu[e] = mean[vc * 8 + e];
    rs[e] = rstd[vc * 8 + e];
    sg[e] = sb[e] = 0.f;
  }
  for (int rb = r0 + ro; rb < r1; rb += 4 * RB) {
    uint4 qd[4], qz[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (rb + u * RB < r1) {
        qd[u] = *reinterpret_cast<const uint4*>(dy + (long)(rb + u * RB) * C + vc * 8);
        qz[u] = *reinterpret_cast<const uint4*>(z + (long)(rb + u * RB) * C + vc * 8);
      }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (rb + u * RB >= r1) break;
      float d[8], x[8];
      unpack8(qd[u], d);
      unpack8(qz[u], x);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        sg[e] = fmaf(d[e], (x[e] - mu[e]) * rs[e], sg[e]);
        sb[e] += d[e];
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    red[((long)ro * C + vc * 8 + e) * 2] = sg[e];
    red[((long)ro * C + vc * 8 + e) * 2 + 1] = sb[e];
  }
  __syncthreads();
  for (int stride = RB / 2; stride >= 1; stride >>= 1) {
    for (int i = t; i < stride * C; i += 256) {
      red[(long)i * 2] += red[((long)i + (long)stride * C) * 2];
      red[(long)i * 2 + 1] += red[((long)i + (long)stride * C) * 2 + 1];
    }
    __syncthreads();
  }
  for (int c = t; c < C; c += 256) {
    part[((long)blockIdx.x * 2 + 0) * C + c] = red[c * 2];
    part[((long)blockIdx.x * 2 + 1) * C + c] = red[c * 2 + 1];
  }
}

// y = act(BN(z) [+ BN2(z2) | + res]), 8 channels per thread
__global__ void bn_apply_vkernel(long nvec, int C, const __nv_bfloat16* __restrict__ z,
                                 const float* __restrict__ mean, const float* __restrict__ rstd,
                                 const float* __restrict__ g, const float* __restrict__ b,
                                 const __nv_bfloat16* __restrict__ z2,
                                 const float* __restrict__ mean2, const float* __restrict__ rstd2,
                                 const float* __restrict__ g2, const float* __restrict__ b2,
                                 const __nv_bfloat16* __restrict__ res, int relu,
                                 __nv_bfloat16* __restrict__ y) {
  pdl_entry();
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nvec;
       i += (long)gridDim.x * blockDim.x) {
    const int c0 = (int)((i * 8) % C);
    float v[8], o[8];
    unpack8(reinterpret_cast<const uint4*>(z)[i], v);
#pragma unroll
    for (int e = 0; e < 8; ++e)
      o[e] = (v[e] - mean[c0 + e]) * rstd[c0 + e] * g[c0 + e] + b[c0 + e];
    if (z2) {
      unpack8(reinterpret_cast<const uint4*>(z2)[i], v);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        o[e] += (v[e] - mean2[c0 + e]) * rstd2[c0 + e] * g2[c0 + e] + b2[c0 + e];
    }
    if (res) {
      unpack8(reinterpret_cast<const uint4*>(res)[i], v);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] += v[e];
    }
    if (relu) {
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = fmaxf(o[e], 0.f);
    }
    reinterpret_cast<uint4*>(y)[i] = pack8(o);
  }
}

// dz = g·rstd/P · (P·dy − db − xhat·dg), 8 channels per thread
__global__ void bn_bwd_dx_vkernel(long nvec, int C, float invP, const __nv_bfloat16* __restrict__ dy,
                                  const __nv_bfloat16* __restrict__ z,
                                  const float* __restrict__ mean, const float* __restrict__ rstd,
                                  const float* __restrict__ g, const float* __restrict__ dg,
                                  const float* __restrict__ db, __nv_bfloat16* __restrict__ dz) {
  pdl_entry();
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nvec;
       i += (long)gridDim.x * blockDim.x) {
    const int c0 = (int)((i * 8) % C);
    float d[8], x[8], o[8];
    unpack8(reinterpret_cast<const uint4*>(dy)[i], d);
    unpack8(reinterpret_cast<const uint4*>(z)[i], x);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = c0 + e;
      const float rs = rstd[c];
      const float xh = (x[e] - mean[c]) * rs;
      o[e] = g[c] * rs * (d[e] - (db[c] + xh * dg[c]) * invP);
    }
    reinterpret_cast<uint4*>(dz)[i] = pack8(o);
  }
}

__global__ void relu_mask_vkernel(long nvec, const __nv_bfloat16* __restrict__ dout,
                                  const __nv_bfloat16* __restrict__ out,
                                  __nv_bfloat16* __restrict__ dy) {
  pdl_entry();
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nvec;
       i += (long)gridDim.x * blockDim.x) {
    float d[8], o[8];
    unpack8(reinterpret_cast<const uint4*>(dout)[i], d);
    unpack8(reinterpret_cast<const uint4*>(out)[i], o);
#pragma unroll
    for (int e = 0; e < 8; ++e) d[e] = o[e] > 0.f ? d[e] : 0.f;
    reinterpret_cast<uint4*>(dy)[i] = pack8(d);
  }
}



template <typename T>
int launch_bn_stats(int P, int C, const T* z, float* part, float* mean, float* rstd,
                    cudaStream_t s) {
  int chunks = bn_chunks(P);
  int rpc = ceil_div(P, chunks);
  if (sizeof(T) == 2 && bn_vec_ok(C, z)) {
    rpc = bn_vec_rpc(P, C);
    chunks = ceil_div(P, rpc);
    launch_k(bn_stats_part_vkernel, chunks, 256, 0, s, P, C, (const __nv_bfloat16*)z, rpc, part);
  } else {
    launch_k(bn_stats_part_kernel<T>, dim3(ceil_div(C, 32), chunks), dim3(32, 8), 0, s, P, C, z, rpc, part);
  }
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
  if (sizeof(T) == 2 && bn_vec_ok(C, z, z2, res) && bn_vec_ok(C, y))
    launch_k(bn_apply_vkernel, grid_for(total / 8), 256, 0, s, total / 8, C,
             (const __nv_bfloat16*)z, mean, rstd, g, b, (const __nv_bfloat16*)z2, mean2, rstd2, g2,
             b2, (const __nv_bfloat16*)res, relu, (__nv_bfloat16*)y);
  else
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
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (sizeof(T) == 2 && n % 8 == 0 && al(dout) && al(out) && al(dy))
    launch_k(relu_mask_vkernel, grid_for(n / 8), 256, 0, s, n / 8, (const __nv_bfloat16*)dout,
             (const __nv_bfloat16*)out, (__nv_bfloat16*)dy);
  else
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
  int chunks = bn_chunks(P);
  int rpc = ceil_div(P, chunks);
  const bool vec = sizeof(T) == 2 && bn_vec_ok(C, dy, z, dz);
  if (vec) {
    rpc = bn_vec_rpc(P, C);
    chunks = ceil_div(P, rpc);
    launch_k(bn_bwd_part_vkernel, chunks, 256, 0, s, P, C, (const __nv_bfloat16*)dy,
             (const __nv_bfloat16*)z, mean, rstd, rpc, part);
  } else {
    launch_k(bn_bwd_part_kernel<T>, dim3(ceil_div(C, 32), chunks), dim3(32, 8), 0, s, P, C, dy, z,
             mean, rstd, rpc, part);
  }
  note_launch();
  launch_k(bn_bwd_final_kernel, ceil_div(C, 8), 256, 0, s, chunks, C, part, dg, db);
  note_launch();
  const long total = (long)P * C;
  if (vec)
    launch_k(bn_bwd_dx_vkernel, grid_for(total / 8), 256, 0, s, total / 8, C, 1.f / (float)P,
             (const __nv_bfloat16*)dy, (const __nv_bfloat16*)z, mean, rstd, g, dg, db,
             (__nv_bfloat16*)dz);
  else
    launch_k(bn_bwd_dx_kernel<T>, grid_for(total), 256, 0, s, total, C, 1.f / (float)P, dy, z, mean,
             rstd, g, dg, db, dz);
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

// one block per image: 8-channel vectors x RB rows per pass, fixed smem tree
__global__ void __launch_bounds__(256)
gap_vkernel(int HW, int C, const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ out) {
  pdl_entry();
  __shared__ float red[256 * 8];
  const int V = C / 8, RB = 256 / V, t = threadIdx.x, vc = t % V, ro = t / V, n = blockIdx.x;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  for (int r = ro; r < HW; r += RB) {
    float v[8];
    unpack8(*reinterpret_cast<const uint4*>(x + ((long)n * HW + r) * C + vc * 8), v);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] += v[e];
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) red[ro * C + vc * 8 + e] = acc[e];
  __syncthreads();
  for (int stride = RB / 2; stride >= 1; stride >>= 1) {
    for (int i = t; i < stride * C; i += 256) red[i] += red[i + stride * C];
    __syncthreads();
  }
  for (int c = t; c < C; c += 256) out[(long)n * C + c] = __float2bfloat16_rn(red[c] / (float)HW);
}

template <typename T>
int launch_gap(int N, int HW, int C, const T* x, T* out, cudaStream_t s) {
  if (sizeof(T) == 2 && bn_vec_ok(C, x))
    launch_k(gap_vkernel, N, 256, 0, s, HW, C, (const __nv_bfloat16*)x, (__nv_bfloat16*)out);
  else
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
