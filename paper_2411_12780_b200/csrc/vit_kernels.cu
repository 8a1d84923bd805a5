// Bandwidth-bound / small-sequence kernels of the ViT local step (sm_100a):
// LayerNorm fwd/bwd (+ deterministic gamma/beta reductions), multi-head
// self-attention fwd/bwd for short sequences (T <= 160, head_dim 64), patch
// extraction and token-embedding assembly.  fp32 math, T in {float, bf16}.
// The GEMM-shaped work of the layer (QKV, projection, MLP) runs on the
// tcgen05 engine (gemm_tc.cu); see vit_stage.cu for the step schedule.
#include <math.h>
#include <stdlib.h>
#include "common.cuh"
#include "kernels.cuh"
#include "vit.cuh"

namespace ppll {

// ---------------------------------------------------------------------------
// 16-B vector row-segment helpers (N elements, 16-B aligned)
// ---------------------------------------------------------------------------
template <int N>
__device__ __forceinline__ void ldv(const __nv_bfloat16* p, float* o) {
#pragma unroll
  for (int i = 0; i < N / 8; ++i) {
    const uint4 q = reinterpret_cast<const uint4*>(p)[i];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(h[j]);
      o[8 * i + 2 * j] = f.x;
      o[8 * i + 2 * j + 1] = f.y;
    }
  }
}
template <int N>
__device__ __forceinline__ void ldv(const float* p, float* o) {
#pragma unroll
  for (int i = 0; i < N / 4; ++i) {
    const float4 q = reinterpret_cast<const float4*>(p)[i];
    o[4 * i] = q.x; o[4 * i + 1] = q.y; o[4 * i + 2] = q.z; o[4 * i + 3] = q.w;
  }
}
template <int N>
__device__ __forceinline__ void stv(__nv_bfloat16* p, const float* v) {
#pragma unroll
  for (int i = 0; i < N / 8; ++i) {
    uint4 q;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[8 * i + 2 * j], v[8 * i + 2 * j + 1]);
    reinterpret_cast<uint4*>(p)[i] = q;
  }
}
template <int N>
__device__ __forceinline__ void stv(float* p, const float* v) {
#pragma unroll
  for (int i = 0; i < N / 4; ++i)
    reinterpret_cast<float4*>(p)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}
__device__ __forceinline__ float half_sum(float v) {   // reduce over the 16 lanes of a half-warp
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// Vectorised LayerNorm (D = 16·EPL, EPL % 8 == 0): a half-warp per row, each
// lane owns EPL contiguous features moved as 16-B vectors.
// ---------------------------------------------------------------------------
template <typename T, int EPL>
__global__ void __launch_bounds__(256)
ln_fwd_vkernel(int M, const T* __restrict__ x, long ldx, const float* __restrict__ g,
               const float* __restrict__ b, T* __restrict__ y, long ldy, float* __restrict__ mean,
               float* __restrict__ rstd) {
  pdl_entry();
  constexpr int D = 16 * EPL;
  const int lane = threadIdx.x & 31, hl = lane & 15;
  const int row = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 2 + (lane >> 4);
  const bool live = row < M;
  const int c0 = hl * EPL;
  float v[EPL], gg[EPL], bb[EPL];
  if (live) ldv<EPL>(x + (long)row * ldx + c0, v);
  else {
#pragma unroll
    for (int i = 0; i < EPL; ++i) v[i] = 0.f;
  }
  // γ / β loads issued with the row's, not after the two reductions
  ldv<EPL>(g + c0, gg);
  ldv<EPL>(b + c0, bb);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < EPL; ++i) s += v[i];
  const float mu = half_sum(s) * (1.f / D);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    const float d = v[i] - mu;
    q += d * d;
  }
  const float rs = rsqrtf(half_sum(q) * (1.f / D) + kLnEps);
  if (!live) return;
#pragma unroll
  for (int i = 0; i < EPL; ++i) v[i] = (v[i] - mu) * rs * gg[i] + bb[i];
  stv<EPL>(y + (long)row * ldy + c0, v);
  if (hl == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

// backward; per-block column partials part[block][NS][D] with NS = 2 (dgamma,
// dbeta) or 3 (+ Σ rows of the dx output: the next bias gradient, fused).
// Persistent (one 256-thread block per SM, half-warp per row, rows strided by
// the grid) and software-pipelined: the next row's dy / x / residual vectors
// are in flight while the current row is reduced, so every SM keeps ~32 rows
// (~70 KB) of loads outstanding.
template <int N>
__device__ __forceinline__ void ldq(const __nv_bfloat16* p, uint4 (&q)[N / 8]) {
#pragma unroll
  for (int i = 0; i < N / 8; ++i) q[i] = reinterpret_cast<const uint4*>(p)[i];
}
template <int N>
__device__ __forceinline__ void unq(const uint4 (&q)[N / 8], float* o) {
#pragma unroll
  for (int i = 0; i < N / 8; ++i) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q[i]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(h[j]);
      o[8 * i + 2 * j] = f.x;
      o[8 * i + 2 * j + 1] = f.y;
    }
  }
}
template <int EPL, int NS, int LPR>
__global__ void __launch_bounds__(256, 1)
ln_bwd_vkernel(int M, const __nv_bfloat16* __restrict__ dy, long lddy,
               const __nv_bfloat16* __restrict__ x, long ldx, const float* __restrict__ mean,
               const float* __restrict__ rstd, const float* __restrict__ g,
               const __nv_bfloat16* __restrict__ dres, long ldres, __nv_bfloat16* __restrict__ dx,
               long lddx, float* __restrict__ part) {
  pdl_entry();
  // LPR lanes per row (16: two rows per warp; 32: one row per warp)
  constexpr int D = LPR * EPL, NQ = EPL / 8, RPW = 32 / LPR, RPB = 8 * RPW;
  // parameter-gradient accumulators live in shared memory, one [NS][D] slab
  // per row slot (registers go to the prefetch ring): [RPB][NS][D]
  extern __shared__ float accS[];
  const int lane = threadIdx.x & 31, hl = lane & (LPR - 1), w = threadIdx.x >> 5;
  const int c0 = hl * EPL;
  float* my = accS + (size_t)(RPW * w + (LPR == 16 ? (lane >> 4) : 0)) * NS * D + c0;
#pragma unroll
  for (int k = 0; k < NS; ++k)
#pragma unroll
    for (int i = 0; i < EPL; i += 4) *reinterpret_cast<float4*>(my + k * D + i) = make_float4(0.f, 0.f, 0.f, 0.f);
  // gamma staged in shared memory after the accumulator slabs
  float* gS = accS + (size_t)RPB * NS * D;
  for (int c = threadIdx.x; c < D; c += blockDim.x) gS[c] = g[c];
  __syncthreads();
  const float* gg = gS + c0;
  const int stride = gridDim.x * RPB;
  const int row0 = blockIdx.x * RPB + RPW * w + (LPR == 16 ? (lane >> 4) : 0);
  // PF-deep prefetch ring: rows row0 + (it + k)·stride for the next PF trips
  // are in flight while the current one is reduced (HBM latency hiding: one
  // block of 8 warps per SM, so bytes in flight come from depth, not warps)
  constexpr int PF = 2;
  uint4 qd[PF][NQ], qx[PF][NQ], qr[PF][NQ];
  float mu[PF], rs[PF];
#pragma unroll
  for (int k = 0; k < PF; ++k) {
    const int r = row0 + k * stride;
    mu[k] = rs[k] = 0.f;
    if (r < M) {
      ldq<EPL>(dy + (long)r * lddy + c0, qd[k]);
      ldq<EPL>(x + (long)r * ldx + c0, qx[k]);
      if (dres) ldq<EPL>(dres + (long)r * ldres + c0, qr[k]);
      mu[k] = mean[r];
      rs[k] = rstd[r];
    }
  }
  // every half-warp runs the same trip count (shuffles stay converged)
  const int trips = (M + stride - 1) / stride;
  for (int it0 = 0; it0 < trips; it0 += PF) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      if (it0 + k >= trips) break;
      const int crow = row0 + (it0 + k) * stride;
      const bool live = crow < M;
      float d[EPL], xh[EPL], o[EPL];
      if (live) {
        unq<EPL>(qd[k], d);
        unq<EPL>(qx[k], xh);
        if (dres) unq<EPL>(qr[k], o);
      } else {
#pragma unroll
        for (int i = 0; i < EPL; ++i) d[i] = xh[i] = o[i] = 0.f;
      }
      const float cmu = mu[k], crs = rs[k];
      const int nrow = crow + PF * stride;
      if (nrow < M) {   // refill this slot PF trips ahead
        ldq<EPL>(dy + (long)nrow * lddy + c0, qd[k]);
        ldq<EPL>(x + (long)nrow * ldx + c0, qx[k]);
        if (dres) ldq<EPL>(dres + (long)nrow * ldres + c0, qr[k]);
        mu[k] = mean[nrow];
        rs[k] = rstd[nrow];
      }
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        xh[i] = (xh[i] - cmu) * crs;
        const float dxh = d[i] * gg[i];
        s1 += dxh;
        s2 += dxh * xh[i];
      }
#pragma unroll
      for (int i = 0; i < EPL; i += 4) {
        float4 a = *reinterpret_cast<float4*>(my + i);
        float4 b = *reinterpret_cast<float4*>(my + D + i);
        a.x += d[i] * xh[i]; a.y += d[i + 1] * xh[i + 1];
        a.z += d[i + 2] * xh[i + 2]; a.w += d[i + 3] * xh[i + 3];
        b.x += d[i]; b.y += d[i + 1]; b.z += d[i + 2]; b.w += d[i + 3];
        *reinterpret_cast<float4*>(my + i) = a;
        *reinterpret_cast<float4*>(my + D + i) = b;
      }
      if (LPR == 16) {
        s1 = half_sum(s1) * (1.f / D);
        s2 = half_sum(s2) * (1.f / D);
      } else {
        s1 = warp_sum(s1) * (1.f / D);
        s2 = warp_sum(s2) * (1.f / D);
      }
      if (live) {
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const float t = crs * (d[i] * gg[i] - s1 - xh[i] * s2);
          o[i] = dres ? o[i] + t : t;
        }
        if (NS == 3) {
#pragma unroll
          for (int i = 0; i < EPL; i += 4) {
            float4 c = *reinterpret_cast<float4*>(my + 2 * D + i);
            c.x += o[i]; c.y += o[i + 1]; c.z += o[i + 2]; c.w += o[i + 3];
            *reinterpret_cast<float4*>(my + 2 * D + i) = c;
          }
        }
        if (dx) stv<EPL>(dx + (long)crow * lddx + c0, o);
      }
    }
  }
  if (!part) return;
  __syncthreads();
  // slots summed in a fixed order (deterministic)
  for (int c = threadIdx.x; c < NS * D; c += blockDim.x) {
    float t = 0.f;
#pragma unroll 4
    for (int k = 0; k < RPB; ++k) t += accS[(size_t)k * NS * D + c];
    part[(long)blockIdx.x * NS * D + c] = t;
  }
}
// LayerNorm backward, round-2 form (D = 32·CPL, CPL % 4 == 0, D <= 512): one
// warp per row, lane owns the 4-element groups at columns 4·lane + 128·k
// (8-B vectors, a warp moves 256 contiguous bytes per access); three rows'
// dy / x / residual loads in flight per warp before the first is reduced;
// the parameter-gradient sums (dγ, dβ and the fused Σ dx) accumulate in
// registers (the row loop is over the warp's own rows), then a fixed-order
// sum over the block's warps writes one [NS][D] partial per block.  Two
// 256-thread blocks per SM (≤ 128 registers): 16 warps x 3 rows ≈ 110 KB of
// loads in flight per SM, against 8 warps of 255-register threads before.
template <int CPL, int NS>
__global__ void __launch_bounds__(256, 2)
ln_bwd_w_kernel(int M, const __nv_bfloat16* __restrict__ dy, long lddy,
                const __nv_bfloat16* __restrict__ x, long ldx, const float* __restrict__ mean,
                const float* __restrict__ rstd, const float* __restrict__ g,
                const __nv_bfloat16* __restrict__ dres, long ldres, __nv_bfloat16* __restrict__ dx,
                long lddx, float* __restrict__ part) {
  pdl_entry();
  constexpr int D = 32 * CPL, NV = CPL / 4, PF = 3;
  extern __shared__ float gsm[];                     // gamma [D] | warp partials [8][NS][D]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c = threadIdx.x; c < D; c += 256) gsm[c] = g[c];
  __syncthreads();
  const int nw = gridDim.x * 8, gw = blockIdx.x * 8 + w;
  float acc[NS][CPL];
#pragma unroll
  for (int k = 0; k < NS; ++k)
#pragma unroll
    for (int i = 0; i < CPL; ++i) acc[k][i] = 0.f;
  uint2 qd[PF][NV], qx[PF][NV], qr[PF][NV];
  float mu[PF], rs[PF];
  auto load = [&](int slot, int row) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int c = 4 * lane + 128 * v;
      qd[slot][v] = *reinterpret_cast<const uint2*>(dy + (long)row * lddy + c);
      qx[slot][v] = *reinterpret_cast<const uint2*>(x + (long)row * ldx + c);
      if (dres) qr[slot][v] = *reinterpret_cast<const uint2*>(dres + (long)row * ldres + c);
    }
    mu[slot] = mean[row];
    rs[slot] = rstd[row];
  };
#pragma unroll
  for (int k = 0; k < PF; ++k)
    if (gw + k * nw < M) load(k, gw + k * nw);
  for (int row = gw, it = 0; row < M; row += nw, ++it) {
    const int slot = it % PF;
    float d[CPL], xh[CPL], o[CPL];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qd[slot][v].x));
      const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qd[slot][v].y));
      d[4 * v] = a.x; d[4 * v + 1] = a.y; d[4 * v + 2] = b.x; d[4 * v + 3] = b.y;
      const float2 e = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qx[slot][v].x));
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qx[slot][v].y));
      xh[4 * v] = e.x; xh[4 * v + 1] = e.y; xh[4 * v + 2] = f.x; xh[4 * v + 3] = f.y;
      if (dres) {
        const float2 p = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qr[slot][v].x));
        const float2 q = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qr[slot][v].y));
        o[4 * v] = p.x; o[4 * v + 1] = p.y; o[4 * v + 2] = q.x; o[4 * v + 3] = q.y;
      }
    }
    const float cmu = mu[slot], crs = rs[slot];
    if (row + PF * nw < M) load(slot, row + PF * nw);   // refill this slot PF rows ahead
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = 4 * v + j;
        xh[i] = (xh[i] - cmu) * crs;
        const float dxh = d[i] * gsm[4 * lane + 128 * v + j];
        s1 += dxh;
        s2 += dxh * xh[i];
        acc[0][i] += d[i] * xh[i];
        acc[1][i] += d[i];
      }
    s1 = warp_sum(s1) * (1.f / D);
    s2 = warp_sum(s2) * (1.f / D);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      float t[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = 4 * v + j;
        const float u = crs * (d[i] * gsm[4 * lane + 128 * v + j] - s1 - xh[i] * s2);
        t[j] = dres ? o[i] + u : u;
        if (NS == 3) acc[NS - 1][i] += t[j];
      }
      if (dx) {
        __nv_bfloat162 h0 = __floats2bfloat162_rn(t[0], t[1]), h1 = __floats2bfloat162_rn(t[2], t[3]);
        uint2 q;
        q.x = *reinterpret_cast<uint32_t*>(&h0);
        q.y = *reinterpret_cast<uint32_t*>(&h1);
        *reinterpret_cast<uint2*>(dx + (long)row * lddx + 4 * lane + 128 * v) = q;
      }
    }
  }
  if (!part) return;
  // block partial: the 8 warps' sums in fixed order
  float* wp = gsm + D;
#pragma unroll
  for (int k = 0; k < NS; ++k)
#pragma unroll
    for (int v = 0; v < NV; ++v)
      *reinterpret_cast<float4*>(wp + ((long)w * NS + k) * D + 4 * lane + 128 * v) =
          make_float4(acc[k][4 * v], acc[k][4 * v + 1], acc[k][4 * v + 2], acc[k][4 * v + 3]);
  __syncthreads();
  for (int c = threadIdx.x; c < NS * D; c += 256) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += wp[(long)k * NS * D + c];
    part[(long)blockIdx.x * NS * D + c] = t;
  }
}

template <int EPL, int NS, int LPR>
static void launch_ln_bwd_v(int nblk, cudaStream_t s, int M, const __nv_bfloat16* dy, long lddy,
                            const __nv_bfloat16* x, long ldx, const float* mean,
                            const float* rstd, const float* g, const __nv_bfloat16* dres,
                            long ldres, __nv_bfloat16* dx, long lddx, float* part) {
  constexpr int smem = (8 * (32 / LPR) * NS + 1) * LPR * EPL * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ln_bwd_vkernel<EPL, NS, LPR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    attr = true;
  }
  launch_k(ln_bwd_vkernel<EPL, NS, LPR>, nblk, 256, smem, s, M, dy, lddy, x, ldx, mean, rstd, g,
           dres, ldres, dx, lddx, part);
}

// ---------------------------------------------------------------------------
// LayerNorm forward: one warp per row, D <= 1024 (D % 32 == 0).
// y = (x - mean) * rstd * g + b ; stores mean/rstd for the backward.
// ---------------------------------------------------------------------------
template <typename T, int VPL>
__global__ void __launch_bounds__(256)
ln_fwd_kernel(int M, int D, const T* __restrict__ x, long ldx, const float* __restrict__ g,
              const float* __restrict__ b, T* __restrict__ y, long ldy, float* __restrict__ mean,
              float* __restrict__ rstd) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= M) return;
  const T* xr = x + (long)row * ldx;
  float v[VPL];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = lane + 32 * i;
    v[i] = c < D ? to_f(xr[c]) : 0.f;
    s += v[i];
  }
  const float mu = warp_sum(s) / (float)D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = lane + 32 * i;
    const float d = c < D ? v[i] - mu : 0.f;
    q += d * d;
  }
  const float rs = rsqrtf(warp_sum(q) / (float)D + kLnEps);
  T* yr = y + (long)row * ldy;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = lane + 32 * i;
    if (c < D) DT<T>::st(yr + c, (v[i] - mu) * rs * g[c] + b[c]);
  }
  if (lane == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

// ---------------------------------------------------------------------------
// LayerNorm backward: warp per row; dx = rstd·(dxh − mean(dxh) − xh·mean(dxh·xh))
// (+ dres, the residual-stream gradient, fused).  Per-block partial sums of
// dg = Σ dy·xh and db = Σ dy go to part[block][2][D] (fixed order).
// ---------------------------------------------------------------------------
template <typename T, int VPL>
__global__ void __launch_bounds__(256)
ln_bwd_kernel(int M, int D, const T* __restrict__ dy, long lddy, const T* __restrict__ x, long ldx,
              const float* __restrict__ mean, const float* __restrict__ rstd,
              const float* __restrict__ g, const T* __restrict__ dres, long ldres,
              T* __restrict__ dx, long lddx, float* __restrict__ part, int rows_per_block) {
  pdl_entry();
  __shared__ float red[2][32 * VPL];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float pg[VPL], pb[VPL];
#pragma unroll
  for (int i = 0; i < VPL; ++i) pg[i] = pb[i] = 0.f;
  const int r0 = blockIdx.x * rows_per_block;
  const int r1 = min(M, r0 + rows_per_block);
  for (int row = r0 + w; row < r1; row += 8) {
    const T* dyr = dy + (long)row * lddy;
    const T* xr = x + (long)row * ldx;
    const float mu = mean[row], rs = rstd[row];
    float xh[VPL], dxh[VPL];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = lane + 32 * i;
      if (c < D) {
        const float d = to_f(dyr[c]);
        xh[i] = (to_f(xr[c]) - mu) * rs;
        dxh[i] = d * g[c];
        pg[i] += d * xh[i];
        pb[i] += d;
      } else {
        xh[i] = dxh[i] = 0.f;
      }
      s1 += dxh[i];
      s2 += dxh[i] * xh[i];
    }
    s1 = warp_sum(s1) / (float)D;
    s2 = warp_sum(s2) / (float)D;
    if (dx) {
      T* dxr = dx + (long)row * lddx;
      const T* rr = dres ? dres + (long)row * ldres : nullptr;
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = lane + 32 * i;
        if (c < D) {
          float o = rs * (dxh[i] - s1 - xh[i] * s2);
          if (rr) o += to_f(rr[c]);
          DT<T>::st(dxr + c, o);
        }
      }
    }
  }
  if (part) {
    // warps accumulate in a fixed order (warp 0, 1, ..., 7): deterministic
    for (int k = 0; k < 8; ++k) {
      if (w == k) {
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          const int c = lane + 32 * i;
          red[0][c] = (k == 0 ? 0.f : red[0][c]) + pg[i];
          red[1][c] = (k == 0 ? 0.f : red[1][c]) + pb[i];
        }
      }
      __syncthreads();
    }
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
      part[((long)blockIdx.x * 2 + 0) * D + c] = red[0][c];
      part[((long)blockIdx.x * 2 + 1) * D + c] = red[1][c];
    }
  }
}

// part is [nblk][NS·D]; block (32 cols x 8 lanes), fixed-order combination;
// stat k of column c goes to out[k][c] (dgamma, dbeta, Σ dx)
__global__ void __launch_bounds__(1024)
ln_param_reduce_kernel(int nblk, int D, int NS, const float* __restrict__ part,
                       float* __restrict__ o0, float* __restrict__ o1, float* __restrict__ o2) {
  pdl_entry();
  __shared__ float red[32][33];
  const int c = blockIdx.x * 32 + threadIdx.x;   // column of the [nblk, NS·D] matrix
  float s = 0.f;
  if (c < NS * D) {
#pragma unroll 4
    for (int k = threadIdx.y; k < nblk; k += 32) s += part[(long)k * NS * D + c];
  }
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && c < NS * D) {
    float t = 0.f;
#pragma unroll
    for (int r = 0; r < 32; ++r) t += red[r][threadIdx.x];
    const int k = c / D, cc = c % D;
    float* o = k == 0 ? o0 : (k == 1 ? o1 : o2);
    if (o) o[cc] = t;
  }
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
template <typename T>
static bool vec_ok(int D, long ld) { return D % 128 == 0 && D <= 1024 && (ld * (long)sizeof(T)) % 16 == 0; }

template <typename T>
int launch_ln_fwd(int M, int D, const T* x, long ldx, const float* g, const float* b, T* y,
                  long ldy, float* mean, float* rstd, cudaStream_t s) {
  if (D % 32 || D > 1024) { set_error("layernorm: D=%d unsupported", D); return PPLL_ERR_ARG; }
  if (vec_ok<T>(D, ldx) && vec_ok<T>(D, ldy) && aligned16(x) && aligned16(y) && aligned16(g) &&
      aligned16(b)) {
    const int blocks = ceil_div(M, 16);     // 8 warps x 2 rows
    switch (D / 16) {
#define LNF(E) case E: launch_k(ln_fwd_vkernel<T, E>, blocks, 256, 0, s, M, x, ldx, g, b, y, ldy, mean, rstd); break;
      LNF(8) LNF(16) LNF(24) LNF(32) LNF(40) LNF(48) LNF(56) LNF(64)
#undef LNF
    }
  } else {
    const int blocks = ceil_div(M, 8);
    if (D <= 384)
      launch_k(ln_fwd_kernel<T, 12>, blocks, 256, 0, s, M, D, x, ldx, g, b, y, ldy, mean, rstd);
    else if (D <= 768)
      launch_k(ln_fwd_kernel<T, 24>, blocks, 256, 0, s, M, D, x, ldx, g, b, y, ldy, mean, rstd);
    else
      launch_k(ln_fwd_kernel<T, 32>, blocks, 256, 0, s, M, D, x, ldx, g, b, y, ldy, mean, rstd);
  }
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// ~2 rows per warp: enough rows in flight to cover DRAM latency, few partials
// vector path: persistent, one block per SM (16 rows per block per trip);
// scalar path: ~2 rows per warp
int ln_bwd_blocks(int M) { return M < 148 * 8 ? ceil_div(M, 8) : min(ceil_div(M, 16), 148 * 2); }
static int ln_bwd_vblocks(int M, int rpb) { return min(ceil_div(M, rpb), 148); }

// batched form of ln_param_reduce_kernel over the deferred tasks of a stage
// backward: block b belongs to the task whose [blk0, blk0 + ceil(NS·D/32)) holds
// it; per column the same fixed-order sum
__global__ void __launch_bounds__(1024)
ln_param_reduce_batch_kernel(const __grid_constant__ LnDefer d) {
  pdl_entry();
  __shared__ float red[32][33];
  int k = 0;
  while (k + 1 < d.n && (int)blockIdx.x >= d.t[k + 1].blk0) ++k;
  const LnReduceTask& t = d.t[k];
  const int NS = t.NS, D = t.D;
  const int c = ((int)blockIdx.x - t.blk0) * 32 + threadIdx.x;
  float s = 0.f;
  if (c < NS * D) {
#pragma unroll 4
    for (int j = threadIdx.y; j < t.nblk; j += 32) s += t.part[(long)j * NS * D + c];
  }
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && c < NS * D) {
    float u = 0.f;
#pragma unroll
    for (int r = 0; r < 32; ++r) u += red[r][threadIdx.x];
    const int kk = c / D, cc = c % D;
    float* o = kk == 0 ? t.o0 : (kk == 1 ? t.o1 : t.o2);
    if (o) o[cc] = u;
  }
}

int launch_ln_reduce_deferred(const LnDefer& d, cudaStream_t s) {
  if (d.n == 0) return PPLL_OK;
  launch_k(ln_param_reduce_batch_kernel, d.blocks, dim3(32, 32), 0, s, d);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

template <typename T>
int launch_ln_bwd(int M, int D, const T* dy, long lddy, const T* x, long ldx, const float* mean,
                  const float* rstd, const float* g, const T* dres, long ldres, T* dx, long lddx,
                  float* part, float* dg, float* db, cudaStream_t s, float* dxsum, LnDefer* defer) {
  if (D % 32 || D > 1024) { set_error("layernorm: D=%d unsupported", D); return PPLL_ERR_ARG; }
  int nblk = ln_bwd_blocks(M);
  const int rpb = ceil_div(M, nblk);
  const bool vec = sizeof(T) == 2 && (D == 128 || D == 256 || D == 384 || D == 512 || D == 768) &&
                   vec_ok<T>(D, lddy) && vec_ok<T>(D, ldx) && (!dres || vec_ok<T>(D, ldres)) &&
                   (!dx || vec_ok<T>(D, lddx)) && aligned16(dy) && aligned16(x) &&
                   (!dres || aligned16(dres)) && (!dx || aligned16(dx)) && aligned16(g);
  int NS = 2;
  // round-2 warp-per-row form for D = 128 .. 512 (PPLL_LN_BWD_W=0: the
  // half-warp form below)
  static const int w_env = getenv("PPLL_LN_BWD_W") ? atoi(getenv("PPLL_LN_BWD_W")) : 1;
  if (vec && w_env && (D == 128 || D == 256 || D == 384 || D == 512)) {
    NS = dxsum ? 3 : 2;
    nblk = ln_bwd_blocks(M);   // <= 296 (two blocks per SM); the partial buffers hold this many
    using B16 = __nv_bfloat16;
    const B16 *dyb = (const B16*)dy, *xb = (const B16*)x, *rb = (const B16*)dres;
    B16* dxb = (B16*)dx;
#define LNW(CPLV, NSV)                                                                          \
    {                                                                                           \
      auto kern = ln_bwd_w_kernel<CPLV, NSV>;                                                   \
      const int smem = (32 * CPLV + 8 * NSV * 32 * CPLV) * 4;                                   \
      static bool attr = false;                                                                 \
      if (!attr) {                                                                              \
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);          \
        attr = true;                                                                            \
      }                                                                                         \
      launch_k(kern, nblk, 256, smem, s, M, dyb, lddy, xb, ldx, mean, rstd, g, rb, ldres, dxb,  \
               lddx, part);                                                                     \
    }
    if (NS == 3) {
      switch (D) { case 128: LNW(4, 3) break; case 256: LNW(8, 3) break;
                   case 384: LNW(12, 3) break; default: LNW(16, 3) break; }
    } else {
      switch (D) { case 128: LNW(4, 2) break; case 256: LNW(8, 2) break;
                   case 384: LNW(12, 2) break; default: LNW(16, 2) break; }
    }
#undef LNW
  } else if (vec) {
    NS = dxsum ? 3 : 2;
    nblk = ln_bwd_vblocks(M, D == 768 || D == 512 ? 8 : 16);
    using B16 = __nv_bfloat16;
    const B16 *dyb = (const B16*)dy, *xb = (const B16*)x, *rb = (const B16*)dres;
    B16* dxb = (B16*)dx;
#define LNB(E, NSV, L) launch_ln_bwd_v<E, NSV, L>(nblk, s, M, dyb, lddy, xb, ldx, mean, rstd, g, rb, ldres, dxb, lddx, part)
#define LNB_ALL(NSV)                          \
    switch (D) {                              \
      case 128: LNB(8, NSV, 16); break;       \
      case 256: LNB(16, NSV, 16); break;      \
      case 384: LNB(24, NSV, 16); break;      \
      case 512: LNB(16, NSV, 32); break;      \
      default: LNB(24, NSV, 32); break;       \
    }
    if (NS == 3) {
      LNB_ALL(3)
    } else {
      LNB_ALL(2)
    }
#undef LNB_ALL
#undef LNB
  } else {
    if (dxsum && !dx) { set_error("layernorm: bias sum needs the dx output"); return PPLL_ERR_ARG; }
    if (D <= 384)
      launch_k(ln_bwd_kernel<T, 12>, nblk, 256, 0, s, M, D, dy, lddy, x, ldx, mean, rstd, g, dres, ldres, dx, lddx, part, rpb);
    else if (D <= 768)
      launch_k(ln_bwd_kernel<T, 24>, nblk, 256, 0, s, M, D, dy, lddy, x, ldx, mean, rstd, g, dres, ldres, dx, lddx, part, rpb);
    else
      launch_k(ln_bwd_kernel<T, 32>, nblk, 256, 0, s, M, D, dy, lddy, x, ldx, mean, rstd, g, dres, ldres, dx, lddx, part, rpb);
  }
  note_launch();
  PPLL_LAUNCH_CHECK();
  if (part && (dg || (vec && dxsum)) && defer && defer->n < LnDefer::kMax) {
    LnReduceTask& t = defer->t[defer->n++];
    t = LnReduceTask{part, dg, db, vec ? dxsum : nullptr, nblk, D, NS, defer->blocks};
    defer->blocks += ceil_div(NS * D, 32);
  } else if (part && (dg || (vec && dxsum))) {
    launch_k(ln_param_reduce_kernel, ceil_div(NS * D, 32), dim3(32, 32), 0, s, nblk, D, NS, part, dg, db,
                                                                        vec ? dxsum : nullptr);
    note_launch();
    PPLL_LAUNCH_CHECK();
  }
  if (!vec && dxsum)   // wide rows: the bias sum as a separate column reduction
    return launch_colsum<T>(M, D, dx, (int)lddx, dxsum, s, nullptr, 0);
  return PPLL_OK;
}

// ---------------------------------------------------------------------------
// Multi-head self-attention, short sequences: one CTA per (batch, head),
// Q/K/V/S resident in shared memory, fp32 math.
// qkv rows: [q (H*dh) | k | v], row b*T + t; o rows: b*T + t, head h at h*dh.
// ---------------------------------------------------------------------------
constexpr int kDh = 64;
constexpr int kLd = kDh + 1;

__host__ __device__ inline size_t attn_fwd_smem(int T) {
  return sizeof(float) * (3 * (size_t)T * kLd + (size_t)T * (T + 1));
}
__host__ __device__ inline size_t attn_bwd_smem(int T) {
  return sizeof(float) * (4 * (size_t)T * kLd + (size_t)T * (T + 1) + (size_t)T);
}

template <typename T>
__device__ __forceinline__ void load_head(float* dst, const T* src, int Tn, long ld, int col0) {
  for (int idx = threadIdx.x; idx < Tn * kDh; idx += blockDim.x) {
    const int t = idx / kDh, d = idx % kDh;
    dst[t * kLd + d] = to_f(src[(long)t * ld + col0 + d]);
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
attn_fwd_kernel(int Tn, int H, const T* __restrict__ qkv, T* __restrict__ o, float* __restrict__ lse,
                float scale) {
  pdl_entry();
  extern __shared__ float sm[];
  float* Q = sm;
  float* Kk = Q + Tn * kLd;
  float* V = Kk + Tn * kLd;
  float* S = V + Tn * kLd;
  const int b = blockIdx.x / H, h = blockIdx.x % H;
  const int D = H * kDh;
  const long ld = 3L * D;
  const T* base = qkv + (long)b * Tn * ld;
  load_head(Q, base, Tn, ld, h * kDh);
  load_head(Kk, base, Tn, ld, D + h * kDh);
  load_head(V, base, Tn, ld, 2 * D + h * kDh);
  __syncthreads();
  const int ldS = Tn + 1;
  for (int idx = threadIdx.x; idx < Tn * Tn; idx += blockDim.x) {
    const int i = idx / Tn, j = idx % Tn;
    const float* qi = Q + i * kLd;
    const float* kj = Kk + j * kLd;
    float acc = 0.f;
#pragma unroll 16
    for (int d = 0; d < kDh; ++d) acc = fmaf(qi[d], kj[d], acc);
    S[i * ldS + j] = acc * scale;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = w; i < Tn; i += nw) {
    float* si = S + i * ldS;
    float mx = -INFINITY;
    for (int j = lane; j < Tn; j += 32) mx = fmaxf(mx, si[j]);
    mx = warp_max(mx);
    float se = 0.f;
    for (int j = lane; j < Tn; j += 32) {
      const float e = __expf(si[j] - mx);
      si[j] = e;
      se += e;
    }
    se = warp_sum(se);
    const float inv = 1.f / se;
    for (int j = lane; j < Tn; j += 32) si[j] *= inv;
    if (lane == 0) lse[(long)blockIdx.x * Tn + i] = mx + logf(se);
  }
  __syncthreads();
  T* ob = o + (long)b * Tn * D + h * kDh;
  for (int idx = threadIdx.x; idx < Tn * kDh; idx += blockDim.x) {
    const int i = idx / kDh, d = idx % kDh;
    const float* pi = S + i * ldS;
    float acc = 0.f;
    for (int j = 0; j < Tn; ++j) acc = fmaf(pi[j], V[j * kLd + d], acc);
    DT<T>::st(ob + (long)i * D + d, acc);
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
attn_bwd_kernel(int Tn, int H, const T* __restrict__ qkv, const T* __restrict__ o,
                const T* __restrict__ dout, const float* __restrict__ lse, T* __restrict__ dqkv,
                float scale) {
  pdl_entry();
  extern __shared__ float sm[];
  float* Q = sm;
  float* Kk = Q + Tn * kLd;
  float* V = Kk + Tn * kLd;
  float* dO = V + Tn * kLd;
  float* S = dO + Tn * kLd;
  float* Di = S + Tn * (Tn + 1);
  const int b = blockIdx.x / H, h = blockIdx.x % H;
  const int D = H * kDh;
  const long ld = 3L * D;
  const T* base = qkv + (long)b * Tn * ld;
  load_head(Q, base, Tn, ld, h * kDh);
  load_head(Kk, base, Tn, ld, D + h * kDh);
  load_head(V, base, Tn, ld, 2 * D + h * kDh);
  load_head(dO, dout + (long)b * Tn * D, Tn, D, h * kDh);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // D_i = rowsum(dO ⊙ O)
  const T* ob = o + (long)b * Tn * D + h * kDh;
  __syncthreads();
  for (int i = w; i < Tn; i += nw) {
    float acc = 0.f;
    for (int d = lane; d < kDh; d += 32) acc += dO[i * kLd + d] * to_f(ob[(long)i * D + d]);
    acc = warp_sum(acc);
    if (lane == 0) Di[i] = acc;
  }
  // P = exp(scale·QKᵀ − lse)
  const int ldS = Tn + 1;
  const float* lrow = lse + (long)blockIdx.x * Tn;
  for (int idx = threadIdx.x; idx < Tn * Tn; idx += blockDim.x) {
    const int i = idx / Tn, j = idx % Tn;
    const float* qi = Q + i * kLd;
    const float* kj = Kk + j * kLd;
    float acc = 0.f;
#pragma unroll 16
    for (int d = 0; d < kDh; ++d) acc = fmaf(qi[d], kj[d], acc);
    S[i * ldS + j] = __expf(acc * scale - lrow[i]);
  }
  __syncthreads();
  T* dq = dqkv + (long)b * Tn * ld + h * kDh;
  T* dk = dq + D;
  T* dv = dq + 2 * D;
  // dV = Pᵀ dO
  for (int idx = threadIdx.x; idx < Tn * kDh; idx += blockDim.x) {
    const int j = idx / kDh, d = idx % kDh;
    float acc = 0.f;
    for (int i = 0; i < Tn; ++i) acc = fmaf(S[i * ldS + j], dO[i * kLd + d], acc);
    DT<T>::st(dv + (long)j * ld + d, acc);
  }
  __syncthreads();
  // dS = P ⊙ (dO Vᵀ − D_i), in place
  for (int idx = threadIdx.x; idx < Tn * Tn; idx += blockDim.x) {
    const int i = idx / Tn, j = idx % Tn;
    const float* gi = dO + i * kLd;
    const float* vj = V + j * kLd;
    float acc = 0.f;
#pragma unroll 16
    for (int d = 0; d < kDh; ++d) acc = fmaf(gi[d], vj[d], acc);
    S[i * ldS + j] = S[i * ldS + j] * (acc - Di[i]);
  }
  __syncthreads();
  // dQ = scale · dS K ; dK = scale · dSᵀ Q
  for (int idx = threadIdx.x; idx < Tn * kDh; idx += blockDim.x) {
    const int i = idx / kDh, d = idx % kDh;
    float aq = 0.f, ak = 0.f;
    for (int j = 0; j < Tn; ++j) {
      aq = fmaf(S[i * ldS + j], Kk[j * kLd + d], aq);
      ak = fmaf(S[j * ldS + i], Q[j * kLd + d], ak);
    }
    DT<T>::st(dq + (long)i * ld + d, aq * scale);
    DT<T>::st(dk + (long)i * ld + d, ak * scale);
  }
}

template <typename T>
int launch_attn_fwd(int B, int Tn, int H, int dh, const T* qkv, T* o, float* lse, cudaStream_t s) {
  if (dh != kDh) { set_error("attention: head_dim %d unsupported (64)", dh); return PPLL_ERR_ARG; }
  const size_t smem = attn_fwd_smem(Tn);
  if (smem > 220 * 1024) { set_error("attention: T=%d too long", Tn); return PPLL_ERR_ARG; }
  static bool set = false;
  if (!set) {
    PPLL_CUDA_CHECK(cudaFuncSetAttribute(attn_fwd_kernel<T>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    set = true;
  }
  launch_k(attn_fwd_kernel<T>, B * H, 256, smem, s, Tn, H, qkv, o, lse, 1.0f / sqrtf((float)dh));
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

template <typename T>
int launch_attn_bwd(int B, int Tn, int H, int dh, const T* qkv, const T* o, const T* dout,
                    const float* lse, T* dqkv, cudaStream_t s) {
  if (dh != kDh) { set_error("attention: head_dim %d unsupported (64)", dh); return PPLL_ERR_ARG; }
  const size_t smem = attn_bwd_smem(Tn);
  if (smem > 220 * 1024) { set_error("attention: T=%d too long", Tn); return PPLL_ERR_ARG; }
  static bool set = false;
  if (!set) {
    PPLL_CUDA_CHECK(cudaFuncSetAttribute(attn_bwd_kernel<T>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    set = true;
  }
  launch_k(attn_bwd_kernel<T>, B * H, 256, smem, s, Tn, H, qkv, o, dout, lse, dqkv,
                                              1.0f / sqrtf((float)dh));
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// ---------------------------------------------------------------------------
// patches + token assembly
// ---------------------------------------------------------------------------
// img [B, C, HW, HW] -> out [B*P, C*p*p], inner order (c, py, px), patches row-major
template <typename T>
__global__ void patchify_kernel(int B, int C, int HW, int p, const T* __restrict__ img,
                                T* __restrict__ out) {
  pdl_entry();
  const int np = HW / p, P = np * np, pd = C * p * p;
  const long total = (long)B * P * pd;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const int e = (int)(idx % pd);
    const long bp = idx / pd;
    const int pi = (int)(bp % P), b = (int)(bp / P);
    const int c = e / (p * p), r = e % (p * p), py = r / p, px = r % p;
    const int yy = (pi / np) * p + py, xx = (pi % np) * p + px;
    out[idx] = img[(((long)b * C + c) * HW + yy) * HW + xx];
  }
}

// x[b,0,:] = cls + pos[0]; x[b,1+i,:] = tok[b,i,:] + pos[1+i]
// (VEC: 8 consecutive features per thread as 16-B bf16 vectors, D % 8 == 0)
template <typename T, int VEC>
__global__ void embed_kernel(int B, int P, int D, const T* __restrict__ tok,
                             const float* __restrict__ cls, const float* __restrict__ pos,
                             T* __restrict__ x) {
  pdl_entry();
  const int Tn = P + 1;
  const long total = (long)B * Tn * D / VEC;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const long e0 = idx * VEC;
    const int d = (int)(e0 % D);
    const long bt = e0 / D;
    const int t = (int)(bt % Tn), b = (int)(bt / Tn);
    float v[VEC];
    if (t == 0) {
#pragma unroll
      for (int i = 0; i < VEC; ++i) v[i] = cls[d + i];
    } else if constexpr (VEC == 8) {
      ldv<8>(tok + ((long)b * P + t - 1) * D + d, v);
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) v[i] = to_f(tok[((long)b * P + t - 1) * D + d + i]);
    }
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] += pos[(long)t * D + d + i];
    if constexpr (VEC == 8) {
      stv<8>(x + e0, v);
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) DT<T>::st(x + e0 + i, v[i]);
    }
  }
}

// dtok[b,i,:] = dx[b,1+i,:]; dcls = Σ_b dx[b,0,:]; dpos[t,:] = Σ_b dx[b,t,:]
// block (32 features x 8 batch groups) per token position, fixed-order
// combination of the 8 partial sums (deterministic)
template <typename T>
__global__ void __launch_bounds__(256)
embed_bwd_kernel(int B, int P, int D, const T* __restrict__ dx, T* __restrict__ dtok,
                 float* __restrict__ dcls, float* __restrict__ dpos) {
  pdl_entry();
  __shared__ float red[8][33];
  const int Tn = P + 1;
  const int d = blockIdx.x * 32 + threadIdx.x, t = blockIdx.y, g = threadIdx.y;
  float s = 0.f;
  if (d < D) {
    for (int b = g; b < B; b += 8) {
      const float v = to_f(dx[((long)b * Tn + t) * D + d]);
      s += v;
      if (t > 0) DT<T>::st(dtok + ((long)b * P + t - 1) * D + d, v);
    }
  }
  red[g][threadIdx.x] = s;
  __syncthreads();
  if (g == 0 && d < D) {
    float tot = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) tot += red[q][threadIdx.x];
    dpos[(long)t * D + d] = tot;
    if (t == 0) dcls[d] = tot;
  }
}

// dx = 0 except the cls rows: dx[b,0,:] = dcls_rows[b,:] (head backward)
template <typename T, int VEC>
__global__ void scatter_cls_kernel(int B, int Tn, int D, const T* __restrict__ dz,
                                   T* __restrict__ dx) {
  pdl_entry();
  const long total = (long)B * Tn * D / VEC;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const long e0 = idx * VEC;
    const int d = (int)(e0 % D);
    const long bt = e0 / D;
    const int t = (int)(bt % Tn), b = (int)(bt / Tn);
    if constexpr (VEC == 8) {
      uint4 q = make_uint4(0u, 0u, 0u, 0u);
      if (t == 0) q = *reinterpret_cast<const uint4*>(dz + (long)b * D + d);
      *reinterpret_cast<uint4*>(dx + e0) = q;
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i)
        DT<T>::st(dx + e0 + i, t == 0 ? to_f(dz[(long)b * D + d + i]) : 0.f);
    }
  }
}

static int grid_for(long n) { return (int)min((n + 255) / 256, (long)148 * 16); }

template <typename T>
int launch_patchify(int B, int C, int HW, int p, const T* img, T* out, cudaStream_t s) {
  const long n = (long)B * (HW / p) * (HW / p) * C * p * p;
  launch_k(patchify_kernel<T>, grid_for(n), 256, 0, s, B, C, HW, p, img, out);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}
template <typename T>
int launch_embed(int B, int P, int D, const T* tok, const float* cls, const float* pos, T* x,
                 cudaStream_t s) {
  const bool v8 = sizeof(T) == 2 && D % 8 == 0 && ((uintptr_t)tok & 15) == 0 && ((uintptr_t)x & 15) == 0;
  if (v8)
    launch_k(embed_kernel<T, 8>, grid_for((long)B * (P + 1) * D / 8), 256, 0, s, B, P, D, tok, cls, pos, x);
  else
    launch_k(embed_kernel<T, 1>, grid_for((long)B * (P + 1) * D), 256, 0, s, B, P, D, tok, cls, pos, x);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}
template <typename T>
int launch_embed_bwd(int B, int P, int D, const T* dx, T* dtok, float* dcls, float* dpos,
                     cudaStream_t s) {
  launch_k(embed_bwd_kernel<T>, dim3(ceil_div(D, 32), P + 1), dim3(32, 8), 0, s, B, P, D, dx, dtok, dcls, dpos);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}
// ---------------------------------------------------------------------------
// Attention of the cls query alone (the cls-only top layer of a stage, see
// vit_stage.cu): per (image, head) one block —
//   forward   s_j = scale·q₀·k_j, p = softmax(s), o₀ = Σ_j p_j v_j, lse₀;
//   backward  with dO non-zero on the cls row only: dP_j = dO₀·v_j,
//             Dsum = dO₀·o₀, dS_j = p_j (dP_j − Dsum),
//             dV_j = p_j dO₀, dK_j = scale·dS_j q₀, dQ₀ = scale·Σ_j dS_j k_j,
//             dQ_j = 0 (j > 0); per-image column sums of dqkv into bpart.
// fp32 arithmetic from T inputs; head_dim 64; any T.  Phase 1: thread = key
// (dot products over the 64 dims, 16-B loads); phase 2: thread = (dim, key
// half), fixed-order combination of the halves.
// ---------------------------------------------------------------------------
constexpr int kClsThreads = 128;

// dot product of a 64-element row with q (shared memory), eight lanes per row:
// lane g of the group loads dims [8g, 8g + 8) as one 16-B (bf16) vector — the
// group reads the row as one coalesced 128-B segment — and the group sums over
// xor shuffles (offsets 1, 2, 4); every lane of the group returns the sum
template <typename T>
__device__ __forceinline__ float dot64_g8(const T* __restrict__ row, const float* q, int g) {
  float v[8];
  ldv<8>(row + 8 * g, v);
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc = fmaf(v[i], q[8 * g + i], acc);
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

__device__ __forceinline__ float block_max128(float v, float* red) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  const float r = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  __syncthreads();
  return r;
}
__device__ __forceinline__ float block_sum128(float v, float* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  const float r = (red[0] + red[1]) + (red[2] + red[3]);
  __syncthreads();
  return r;
}

template <typename T>
__global__ void __launch_bounds__(kClsThreads)
cls_attn_fwd_kernel(int Tn, int H, const T* __restrict__ qkv, T* __restrict__ o,
                    float* __restrict__ lse, float scale) {
  pdl_entry();
  extern __shared__ float csm[];
  float* q = csm;              // [64]
  float* p = q + 64;           // [Tn]
  float* red = p + Tn;         // [4]
  float* half = red + 4;       // [64]
  const int bh = blockIdx.x, b = bh / H, h = bh % H, t = threadIdx.x;
  const int D = H * 64, D3 = 3 * D;
  const T* base = qkv + (long)b * Tn * D3;
  if (t < 64) q[t] = to_f(base[h * 64 + t]) * scale;
  __syncthreads();
  float mx = -INFINITY;
  {
    const int g = t & 7, kr = t >> 3;   // 16 keys per pass, eight lanes each
    for (int j0 = 0; j0 < Tn; j0 += kClsThreads / 8) {
      const int j = j0 + kr;
      const float sj = dot64_g8(base + (long)min(j, Tn - 1) * D3 + D + h * 64, q, g);
      if (j < Tn) {
        if (g == 0) p[j] = sj;
        mx = fmaxf(mx, sj);
      }
    }
  }
  mx = block_max128(mx, red);   // (barrier inside: p complete)
  float sum = 0.f;
  for (int j = t; j < Tn; j += kClsThreads) {
    const float e = __expf(p[j] - mx);
    p[j] = e;
    sum += e;
  }
  sum = block_sum128(sum, red);   // (barrier inside: p complete)
  const float inv = 1.f / sum;
  const int d = t & 63, hf = t >> 6;
  const int jm = (Tn + 1) / 2, j0 = hf ? jm : 0, j1 = hf ? Tn : jm;
  float acc = 0.f;
  for (int j = j0; j < j1; ++j) acc = fmaf(p[j], to_f(base[(long)j * D3 + 2 * D + h * 64 + d]), acc);
  if (hf) half[d] = acc;
  __syncthreads();
  if (!hf) {
    DT<T>::st(o + (long)b * D + h * 64 + d, (acc + half[d]) * inv);
    if (d == 0) lse[bh] = mx + logf(sum);
  }
}

template <typename T>
__global__ void __launch_bounds__(kClsThreads)
cls_attn_bwd_kernel(int Tn, int H, const T* __restrict__ qkv, const T* __restrict__ o,
                    const T* __restrict__ dout, const float* __restrict__ lse,
                    T* __restrict__ dqkv, float* __restrict__ bpart, float scale) {
  pdl_entry();
  extern __shared__ float csm[];
  float* q = csm;               // [64]  scale·q₀
  float* g = q + 64;            // [64]  dO₀
  float* p = g + 64;            // [Tn]
  float* ds = p + Tn;           // [Tn]
  float* red = ds + Tn;         // [4]
  float* hq = red + 4;          // [64] second-half partials: dQ
  float* hk = hq + 64;          // [64] Σ dK
  float* hv = hk + 64;          // [64] Σ dV
  const int bh = blockIdx.x, b = bh / H, h = bh % H, t = threadIdx.x;
  const int D = H * 64, D3 = 3 * D;
  const T* base = qkv + (long)b * Tn * D3;
  float dsum = 0.f;
  if (t < 64) {
    q[t] = to_f(base[h * 64 + t]) * scale;
    const float gd = to_f(dout[(long)b * D + h * 64 + t]);
    g[t] = gd;
    dsum = gd * to_f(o[(long)b * D + h * 64 + t]);
  }
  dsum = block_sum128(dsum, red);   // Dsum = dO₀·o₀ (barrier inside: q, g complete)
  const float l0 = lse[bh];
  {
    const int gl = t & 7, kq = t >> 3;   // 16 keys per pass, eight lanes each
    for (int j0 = 0; j0 < Tn; j0 += kClsThreads / 8) {
      const int j = j0 + kq;
      const T* kr = base + (long)min(j, Tn - 1) * D3 + D + h * 64;
      const float pj = __expf(dot64_g8(kr, q, gl) - l0);
      const float dpj = dot64_g8(kr + D, g, gl);   // v_j (the V block is D further on)
      if (j < Tn && gl == 0) {
        p[j] = pj;
        ds[j] = pj * (dpj - dsum);
      }
    }
  }
  __syncthreads();
  const int d = t & 63, hf = t >> 6;
  const int jm = (Tn + 1) / 2, j0 = hf ? jm : 0, j1 = hf ? Tn : jm;
  const float qd = q[d], gd = g[d];   // q already carries the scale
  float aq = 0.f, ak = 0.f, av = 0.f;
  for (int j = j0; j < j1; ++j) {
    T* row = dqkv + ((long)b * Tn + j) * D3 + h * 64 + d;
    const float kd = to_f(base[(long)j * D3 + D + h * 64 + d]);
    aq = fmaf(ds[j], kd, aq);
    const float dk = ds[j] * qd, dv = p[j] * gd;
    ak += dk;
    av += dv;
    if (j > 0) DT<T>::st(row, 0.f);
    DT<T>::st(row + D, dk);
    DT<T>::st(row + 2 * D, dv);
  }
  if (hf) { hq[d] = aq; hk[d] = ak; hv[d] = av; }
  __syncthreads();
  if (!hf) {
    const float dq = (aq + hq[d]) * scale;
    DT<T>::st(dqkv + (long)b * Tn * D3 + h * 64 + d, dq);
    if (bpart) {
      float* bp = bpart + (long)b * D3 + h * 64 + d;
      bp[0] = dq;
      bp[D] = ak + hk[d];
      bp[2 * D] = av + hv[d];
    }
  }
}

template <typename T>
int launch_cls_attn_fwd(int B, int Tn, int H, const T* qkv, T* o, float* lse, cudaStream_t s) {
  const size_t smem = sizeof(float) * (64 + Tn + 4 + 64);
  launch_k(cls_attn_fwd_kernel<T>, B * H, kClsThreads, smem, s, Tn, H, qkv, o, lse, 0.125f);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}
template <typename T>
int launch_cls_attn_bwd(int B, int Tn, int H, const T* qkv, const T* o, const T* dout,
                        const float* lse, T* dqkv, float* bpart, cudaStream_t s) {
  const size_t smem = sizeof(float) * (128 + 2 * Tn + 4 + 192);
  launch_k(cls_attn_bwd_kernel<T>, B * H, kClsThreads, smem, s, Tn, H, qkv, o, dout, lse, dqkv,
           bpart, 0.125f);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}
template int launch_cls_attn_fwd<float>(int, int, int, const float*, float*, float*, cudaStream_t);
template int launch_cls_attn_fwd<__nv_bfloat16>(int, int, int, const __nv_bfloat16*, __nv_bfloat16*, float*, cudaStream_t);
template int launch_cls_attn_bwd<float>(int, int, int, const float*, const float*, const float*, const float*, float*, float*, cudaStream_t);
template int launch_cls_attn_bwd<__nv_bfloat16>(int, int, int, const __nv_bfloat16*, const __nv_bfloat16*, const __nv_bfloat16*, const float*, __nv_bfloat16*, float*, cudaStream_t);

template <typename T>
int launch_scatter_cls(int B, int Tn, int D, const T* dz, T* dx, cudaStream_t s) {
  const bool v8 = sizeof(T) == 2 && D % 8 == 0 && ((uintptr_t)dz & 15) == 0 && ((uintptr_t)dx & 15) == 0;
  if (v8)
    launch_k(scatter_cls_kernel<T, 8>, grid_for((long)B * Tn * D / 8), 256, 0, s, B, Tn, D, dz, dx);
  else
    launch_k(scatter_cls_kernel<T, 1>, grid_for((long)B * Tn * D), 256, 0, s, B, Tn, D, dz, dx);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

#define INST(T)                                                                                  \
  template int launch_ln_fwd<T>(int, int, const T*, long, const float*, const float*, T*, long,  \
                                float*, float*, cudaStream_t);                                   \
  template int launch_ln_bwd<T>(int, int, const T*, long, const T*, long, const float*,          \
                                const float*, const float*, const T*, long, T*, long, float*,    \
                                float*, float*, cudaStream_t, float*, LnDefer*);                 \
  template int launch_attn_fwd<T>(int, int, int, int, const T*, T*, float*, cudaStream_t);      \
  template int launch_attn_bwd<T>(int, int, int, int, const T*, const T*, const T*,             \
                                  const float*, T*, cudaStream_t);                               \
  template int launch_patchify<T>(int, int, int, int, const T*, T*, cudaStream_t);              \
  template int launch_embed<T>(int, int, int, const T*, const float*, const float*, T*,          \
                               cudaStream_t);                                                    \
  template int launch_embed_bwd<T>(int, int, int, const T*, T*, float*, float*, cudaStream_t);  \
  template int launch_scatter_cls<T>(int, int, int, const T*, T*, cudaStream_t);
INST(float)
INST(__nv_bfloat16)
#undef INST

}  // namespace ppll
