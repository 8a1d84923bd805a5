// Bandwidth-bound and SIMT kernels of the PPLL local step (sm_100a).
//
//  * gemm_simt      — fp32-accumulate SIMT GEMM with fused bias/ReLU/mask/dual
//                     store epilogue.  It is the fp32 parity engine and the
//                     engine for skinny shapes (class-count N, tiny K) that
//                     cannot fill a 128-row tcgen05 tile.
//  * colsum         — bias gradient Σ_rows dY (tensor.py:179), deterministic.
//  * softmax_xent   — fused mean-CE forward + adjoint (tensor.py:201-234).
//  * nesterov_step  — multi-tensor (flat buffer) Nesterov-SGD (optim.py:71-89).
//  * ring kernels   — release/acquire flag words for the stage-boundary ring.
#include <math.h>
#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

#include <mutex>
#include <unordered_map>

namespace ppll {

// ------------------------------------------------------------------------
// SIMT GEMM: C(m,n) = Σ_k A(m,k)·B(k,n), generic strides.
// A(m,k) = A[m*a_rs + k*a_cs];  B(k,n) = B[k*b_rs + n*b_cs].
// 64x64x16 tiles, 256 threads, 4x4 outputs per thread.
// ------------------------------------------------------------------------
constexpr int SB_M = 64, SB_N = 64, SB_K = 16;

template <typename TI, typename TO>
__global__ void __launch_bounds__(256)
gemm_simt_kernel(int M, int N, int K, const TI* __restrict__ A, long a_rs, long a_cs,
                 const TI* __restrict__ Bm, long b_rs, long b_cs, Epilogue<TO> ep, int k_per_split) {
  pdl_entry();
  __shared__ float As[SB_K][SB_M + 4];
  __shared__ float Bs[SB_K][SB_N + 4];
  const int t = threadIdx.x;
  const int m0 = blockIdx.y * SB_M, n0 = blockIdx.x * SB_N;
  const int kbeg = blockIdx.z * k_per_split;
  const int kend = min(K, kbeg + k_per_split);
  const int ty = t / 16, tx = t % 16;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  const bool a_kc = (a_cs == 1);   // A is k-contiguous (row-major [M,K])
  const bool b_nc = (b_cs == 1);   // B is n-contiguous (row-major [K,N])
  for (int k0 = kbeg; k0 < kend; k0 += SB_K) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int mm, kk;
      if (a_kc) { kk = t % 16; mm = t / 16 + 16 * i; }
      else      { mm = t % 64; kk = t / 64 + 4 * i; }
      int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < kend) ? to_f(A[(long)gm * a_rs + (long)gk * a_cs]) : 0.f;
      int nn, kb;
      if (b_nc) { nn = t % 64; kb = t / 64 + 4 * i; }
      else      { kb = t % 16; nn = t / 16 + 16 * i; }
      int gn = n0 + nn, gkb = k0 + kb;
      Bs[kb][nn] = (gn < N && gkb < kend) ? to_f(Bm[(long)gkb * b_rs + (long)gn * b_cs]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SB_K; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int gm = m0 + ty + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gn = n0 + tx + 16 * j;
      if (gn >= N) continue;
      if (ep.partial) {  // split-K partial: raw fp32 into the workspace slice
        ep.partial[((long)blockIdx.z * M + gm) * N + gn] = acc[i][j];
      } else {
        ep.apply(gm, gn, acc[i][j]);
      }
    }
  }
}

// split-K reduction + epilogue: C = epilogue(Σ_s partial[s])
template <typename TO>
__global__ void splitk_reduce_kernel(int M, int N, int splits, const float* __restrict__ part,
                                     Epilogue<TO> ep) {
  pdl_entry();
  long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  long total = (long)M * N;
  for (; idx < total; idx += (long)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += part[(long)z * total + idx];
    ep.apply((int)(idx / N), (int)(idx % N), s);
  }
}

// Skinny shapes (classifier N <= 32, or reduction K <= 32): the 64x64 tile
// would idle most of its lanes, so use
//  * row-warp: one warp per output row, lanes split K, NP accumulators,
//    butterfly reduction (A k-contiguous, N <= 32);
//  * col-warp: lanes own 32 consecutive output rows (A m-contiguous), the 8
//    warps split K, fixed-order reduction across warps (N <= 32);
//  * dot: one thread per output element, the coalesced operand dimension
//    mapped to the fastest thread index.
// Both warp forms stage B (the K x N classifier weights / upstream gradient)
// in shared memory in chunks of 4096 / NP rows (16 KB), so the inner loop
// streams only A.

// Stage a [kc x NP] chunk of B (rows k0.., columns >= N zero) in shared
// memory; every thread has eight independent loads in flight before it stores
// (one memory latency per eight elements instead of one per element).
template <int NP, int LD, typename TI>
__device__ __forceinline__ void stage_b(float* bs, const TI* __restrict__ Bm, int k0, int kc, int N,
                                        long b_rs, long b_cs) {
  const int total = kc * NP;
  for (int i0 = threadIdx.x; i0 < total; i0 += 8 * blockDim.x) {
    float t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x, kk = i / NP, n = i % NP;
      t[u] = (i < total && n < N) ? to_f(Bm[(long)(k0 + kk) * b_rs + (long)n * b_cs]) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < total) bs[(i / NP) * LD + i % NP] = t[u];
    }
  }
}

template <typename TI, typename TO, int NP>
__global__ void __launch_bounds__(256)
gemm_rowwarp_kernel(int M, int N, int K, const TI* __restrict__ A, long a_rs,
                    const TI* __restrict__ Bm, long b_rs, long b_cs, Epilogue<TO> ep) {
  pdl_entry();
  constexpr int kSkK = 4096 / NP;
  constexpr int LD = NP + 1;   // lanes read different K rows: odd stride, no bank conflicts
  __shared__ float bs[kSkK * LD];
  const int lane = threadIdx.x & 31;
  const int m = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const bool live = m < M;
  float acc[NP];
#pragma unroll
  for (int n = 0; n < NP; ++n) acc[n] = 0.f;
  const TI* ar = A + (long)(live ? m : 0) * a_rs;
  constexpr int kJ = kSkK / 32;
  for (int k0 = 0; k0 < K; k0 += kSkK) {
    const int kc = min(kSkK, K - k0);
    // the row's A chunk is loaded before the B staging so both latencies overlap
    float av[kJ];
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int kk = lane + 32 * j;
      av[j] = (live && kk < kc) ? to_f(ar[k0 + kk]) : 0.f;
    }
    __syncthreads();
    stage_b<NP, LD>(bs, Bm, k0, kc, N, b_rs, b_cs);
    __syncthreads();
    if (live) {
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        const int kk = lane + 32 * j;
        if (kk < kc) {
          const float* br = bs + kk * LD;
#pragma unroll
          for (int n = 0; n < NP; ++n) acc[n] = fmaf(av[j], br[n], acc[n]);
        }
      }
    }
  }
  if (!live) return;
#pragma unroll
  for (int n = 0; n < NP; ++n) acc[n] = warp_sum(acc[n]);
#pragma unroll
  for (int n = 0; n < NP; ++n)
    if (n < N && lane == n) ep.apply(m, n, acc[n]);
}

template <typename TI, typename TO, int NP>
__global__ void __launch_bounds__(256)
gemm_colwarp_kernel(int M, int N, int K, const TI* __restrict__ A, long a_cs,
                    const TI* __restrict__ Bm, long b_rs, long b_cs, Epilogue<TO> ep) {
  pdl_entry();
  constexpr int kSkK = 4096 / NP;
  __shared__ float bs[kSkK * NP];
  __shared__ float red[8][8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int m = blockIdx.x * 32 + lane;
  const bool live = m < M;
  float acc[NP];
#pragma unroll
  for (int n = 0; n < NP; ++n) acc[n] = 0.f;
  for (int k0 = 0; k0 < K; k0 += kSkK) {
    const int kc = min(kSkK, K - k0);
    __syncthreads();
    stage_b<NP, NP>(bs, Bm, k0, kc, N, b_rs, b_cs);
    __syncthreads();
    if (live) {
      // A elements of four K rows loaded before they are consumed (same order)
      for (int kb = w; kb < kc; kb += 32) {
        float a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          a[u] = kb + 8 * u < kc ? to_f(A[(long)(k0 + kb + 8 * u) * a_cs + m]) : 0.f;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (kb + 8 * u >= kc) break;
          const float* br = bs + (kb + 8 * u) * NP;
#pragma unroll
          for (int n = 0; n < NP; ++n) acc[n] = fmaf(a[u], br[n], acc[n]);
        }
      }
    }
  }
  // fixed-order reduction over the 8 K-slices, eight output columns at a time
#pragma unroll
  for (int n0 = 0; n0 < NP; n0 += 8) {
    __syncthreads();
#pragma unroll
    for (int n = 0; n < 8; ++n) red[w][n][lane] = acc[n0 + n];
    __syncthreads();
    if (w == 0 && live) {
      for (int n = 0; n < 8 && n0 + n < N; ++n) {
        float t = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) t += red[q][n][lane];
        ep.apply(m, n0 + n, t);
      }
    }
  }
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(256)
gemm_dot_kernel(int M, int N, int K, const TI* __restrict__ A, long a_rs, long a_cs,
                const TI* __restrict__ Bm, long b_rs, long b_cs, Epilogue<TO> ep, int m_fast) {
  pdl_entry();
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long)M * N) return;
  const int m = m_fast ? (int)(idx % M) : (int)(idx / N);
  const int n = m_fast ? (int)(idx / M) : (int)(idx % N);
  const TI* ar = A + (long)m * a_rs;
  const TI* bc = Bm + (long)n * b_cs;
  float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;   // 4 independent chains (ILP)
  int k = 0;
  for (; k + 4 <= K; k += 4) {
    acc0 = fmaf(to_f(ar[(long)k * a_cs]), to_f(bc[(long)k * b_rs]), acc0);
    acc1 = fmaf(to_f(ar[(long)(k + 1) * a_cs]), to_f(bc[(long)(k + 1) * b_rs]), acc1);
    acc2 = fmaf(to_f(ar[(long)(k + 2) * a_cs]), to_f(bc[(long)(k + 2) * b_rs]), acc2);
    acc3 = fmaf(to_f(ar[(long)(k + 3) * a_cs]), to_f(bc[(long)(k + 3) * b_rs]), acc3);
  }
  for (; k < K; ++k) acc0 = fmaf(to_f(ar[(long)k * a_cs]), to_f(bc[(long)k * b_rs]), acc0);
  ep.apply(m, n, (acc0 + acc1) + (acc2 + acc3));
}

template <typename TI, typename TO>
int launch_gemm_simt(int M, int N, int K, const TI* A, long a_rs, long a_cs, const TI* B,
                     long b_rs, long b_cs, const Epilogue<TO>& ep, float* ws, size_t ws_elems,
                     cudaStream_t s) {
  if (N <= 32 && a_cs == 1 && K >= 64) {
    Epilogue<TO> e = ep;
    e.partial = nullptr;
    if (N <= 16)
      launch_k(gemm_rowwarp_kernel<TI, TO, 16>, ceil_div(M, 8), 256, 0, s, M, N, K, A, a_rs, B, b_rs, b_cs, e);
    else
      launch_k(gemm_rowwarp_kernel<TI, TO, 32>, ceil_div(M, 8), 256, 0, s, M, N, K, A, a_rs, B, b_rs, b_cs, e);
    note_launch();
    PPLL_LAUNCH_CHECK();
    return PPLL_OK;
  }
  if (N <= 32 && a_rs == 1 && K >= 64) {
    Epilogue<TO> e = ep;
    e.partial = nullptr;
    if (N <= 16)
      launch_k(gemm_colwarp_kernel<TI, TO, 16>, ceil_div(M, 32), 256, 0, s, M, N, K, A, a_cs, B, b_rs, b_cs, e);
    else
      launch_k(gemm_colwarp_kernel<TI, TO, 32>, ceil_div(M, 32), 256, 0, s, M, N, K, A, a_cs, B, b_rs, b_cs, e);
    note_launch();
    PPLL_LAUNCH_CHECK();
    return PPLL_OK;
  }
  if (N <= 32 || K <= 32) {
    Epilogue<TO> e = ep;
    e.partial = nullptr;
    // fastest thread index along the dimension whose streamed operand is contiguous:
    // m when A is m-contiguous and N is small (its B element is then a warp broadcast)
    const int m_fast = (a_rs == 1 && (b_cs != 1 || N <= 32)) ? 1 : 0;
    launch_k(gemm_dot_kernel<TI, TO>, ceil_div((long)M * N, 256), 256, 0, s, M, N, K, A, a_rs, a_cs, B,
                                                                         b_rs, b_cs, e, m_fast);
    note_launch();
    PPLL_LAUNCH_CHECK();
    return PPLL_OK;
  }
  dim3 grid(ceil_div(N, SB_N), ceil_div(M, SB_M), 1);
  int tiles = grid.x * grid.y;
  int splits = 1;
  // split K when the tile grid cannot fill the 148 SMs and K is deep
  if (ws && tiles < 74 && K >= 512) {
    splits = 148 / tiles;
    splits = min(splits, K / 128);
    while (splits > 1 && (size_t)splits * M * N > ws_elems) --splits;
    if (splits < 1) splits = 1;
  }
  int kps = ((K + splits - 1) / splits + SB_K - 1) / SB_K * SB_K;
  splits = ceil_div(K, kps);
  grid.z = splits;
  if (splits == 1) {
    Epilogue<TO> e = ep;
    e.partial = nullptr;
    launch_k(gemm_simt_kernel<TI, TO>, grid, 256, 0, s, M, N, K, A, a_rs, a_cs, B, b_rs, b_cs, e, K);
    note_launch();
  } else {
    Epilogue<TO> e = ep;
    e.partial = ws;
    launch_k(gemm_simt_kernel<TI, TO>, grid, 256, 0, s, M, N, K, A, a_rs, a_cs, B, b_rs, b_cs, e, kps);
    note_launch();
    Epilogue<TO> r = ep;
    r.partial = nullptr;
    int blocks = min(ceil_div((long)M * N, 256), 148 * 8);
    launch_k(splitk_reduce_kernel<TO>, blocks, 256, 0, s, M, N, splits, ws, r);
    note_launch();
  }
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// split-K reduction with the splits spread over 8 thread rows: block (32
// outputs x 8 split groups); each thread sums splits g, g+8, ... in order,
// then a fixed-order combination of the 8 partials (deterministic)
template <typename TO>
__global__ void __launch_bounds__(256)
splitk_reduce2_kernel(int M, int N, int splits, const float* __restrict__ part, Epilogue<TO> ep) {
  pdl_entry();
  __shared__ float red[8][33];
  const long total = (long)M * N;
  const long idx = (long)blockIdx.x * 32 + threadIdx.x;
  float s = 0.f;
  if (idx < total)
    for (int z = threadIdx.y; z < splits; z += 8) s += part[(long)z * total + idx];
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && idx < total) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][threadIdx.x];
    ep.apply((int)(idx / N), (int)(idx % N), t);
  }
}

template <typename TO>
int launch_splitk_reduce(int M, int N, int splits, const float* ws, const Epilogue<TO>& ep,
                         cudaStream_t s) {
  Epilogue<TO> r = ep;
  r.partial = nullptr;
  const long total = (long)M * N;
  if (splits >= 16 && total <= 148L * 8 * 256) {
    // few outputs, many splits (conv weight gradients): parallel over the splits
    launch_k(splitk_reduce2_kernel<TO>, ceil_div(total, 32), dim3(32, 8), 0, s, M, N, splits, ws, r);
  } else {
    int blocks = min(ceil_div(total, 256), 148 * 8);
    launch_k(splitk_reduce_kernel<TO>, blocks, 256, 0, s, M, N, splits, ws, r);
  }
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}
template int launch_splitk_reduce<float>(int, int, int, const float*, const Epilogue<float>&, cudaStream_t);
template int launch_splitk_reduce<__nv_bfloat16>(int, int, int, const float*, const Epilogue<__nv_bfloat16>&, cudaStream_t);

template int launch_gemm_simt<float, float>(int, int, int, const float*, long, long, const float*, long, long, const Epilogue<float>&, float*, size_t, cudaStream_t);
template int launch_gemm_simt<__nv_bfloat16, __nv_bfloat16>(int, int, int, const __nv_bfloat16*, long, long, const __nv_bfloat16*, long, long, const Epilogue<__nv_bfloat16>&, float*, size_t, cudaStream_t);
template int launch_gemm_simt<__nv_bfloat16, float>(int, int, int, const __nv_bfloat16*, long, long, const __nv_bfloat16*, long, long, const Epilogue<float>&, float*, size_t, cudaStream_t);

// ------------------------------------------------------------------------
// bias gradient: db[n] = Σ_m G[m*ld + n]   (fixed summation order)
// ------------------------------------------------------------------------
// Pass 1: block (32 cols x 8 row lanes) sums rows [chunk*rpc, (chunk+1)*rpc)
// of 32 columns; the 8 lanes combine in a fixed order -> out[chunk][n].
// Pass 2 (only when several chunks): out[n] = Σ_chunk part[chunk][n] in order.
template <typename T>
__global__ void colsum_kernel(int M, int N, const T* __restrict__ G, long ld, int rpc,
                              float* __restrict__ out) {
  pdl_entry();
  __shared__ float red[8][33];
  const int n = blockIdx.x * 32 + threadIdx.x;
  const int r0 = blockIdx.y * rpc, r1 = min(M, r0 + rpc);
  float s = 0.f;
  if (n < N) {
#pragma unroll 4
    for (int m = r0 + threadIdx.y; m < r1; m += 8) s += to_f(G[(long)m * ld + n]);
  }
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && n < N) {
    float t = 0.f;
#pragma unroll
    for (int r = 0; r < 8; ++r) t += red[r][threadIdx.x];
    out[(long)blockIdx.y * N + n] = t;
  }
}

template <typename T>
int launch_colsum(int M, int N, const T* G, int ld, float* db, cudaStream_t s, float* ws,
                  size_t ws_elems) {
  int chunks = 1;
  if (ws && M > 512) {
    chunks = min(ceil_div(M, 64), 256);
    while (chunks > 1 && (size_t)chunks * N > ws_elems) chunks /= 2;
  }
  const int rpc = ceil_div(M, chunks);
  chunks = ceil_div(M, rpc);
  if (chunks <= 1) {
    launch_k(colsum_kernel<T>, dim3(ceil_div(N, 32), 1), dim3(32, 8), 0, s, M, N, G, ld, M, db);
    note_launch();
  } else {
    launch_k(colsum_kernel<T>, dim3(ceil_div(N, 32), chunks), dim3(32, 8), 0, s, M, N, G, ld, rpc, ws);
    note_launch();
    launch_k(colsum_kernel<float>, dim3(ceil_div(N, 32), 1), dim3(32, 8), 0, s, chunks, N, ws, N,
                                                                           chunks, db);
    note_launch();
  }
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}
template int launch_colsum<float>(int, int, const float*, int, float*, cudaStream_t, float*, size_t);
template int launch_colsum<__nv_bfloat16>(int, int, const __nv_bfloat16*, int, float*, cudaStream_t, float*, size_t);

// ------------------------------------------------------------------------
// softmax cross-entropy, fused forward + adjoint (tensor.py:201-234).
// One block; warp w handles rows w, w+nw, ...; per-row losses are summed in a
// fixed order in double so the scalar is deterministic.
// ------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(1024)
softmax_xent_kernel(int B, int C, const T* __restrict__ z, int ldz, const int64_t* __restrict__ y,
                    T* __restrict__ dz, int lddz, float* loss_hist, const int* step, int* err) {
  pdl_entry();
  extern __shared__ float row_loss[];
  // a half-warp per row (16 lanes stride the classes): two rows per warp in
  // flight; every half-warp runs the same trip count so shuffles stay converged
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int sl = lane & 15, seg = lane >> 4;
  const float invB = 1.0f / (float)B;
  const int trips = (B + 2 * nw - 1) / (2 * nw);
  for (int it = 0; it < trips; ++it) {
    const int r = (it * nw + w) * 2 + seg;
    const bool live = r < B;
    const T* zr = z + (long)(live ? r : 0) * ldz;
    const long lab = live ? y[r] : 0;
    const bool bad = (lab < 0 || lab >= C);
    float mx = -INFINITY;
    for (int c = sl; c < C; c += 16) mx = fmaxf(mx, to_f(zr[c]));
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float se = 0.f, zl = 0.f;
    for (int c = sl; c < C; c += 16) {
      const float v = to_f(zr[c]);
      se += __expf(v - mx);
      if (c == lab) zl = v;
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      se += __shfl_xor_sync(0xffffffffu, se, o);
      zl += __shfl_xor_sync(0xffffffffu, zl, o);
    }
    if (!live) continue;
    const float inv = 1.0f / se;
    T* dr = dz + (long)r * lddz;
    for (int c = sl; c < C; c += 16) {
      const float p = __expf(to_f(zr[c]) - mx) * inv;
      DT<T>::st(dr + c, bad ? 0.f : (p - (c == lab ? 1.f : 0.f)) * invB);
    }
    if (sl == 0) {
      row_loss[r] = bad ? 0.f : -((zl - mx) - logf(se));
      if (bad && err) atomicOr(err, kErrLabel);
    }
  }
  __syncthreads();
  if (w == 0) {   // fixed-order reduction: lane-strided partials, then a fixed tree
    double s = 0.0;
    for (int r = lane; r < B; r += 32) s += (double)row_loss[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const float loss = (float)(s / (double)B);
      loss_hist[step ? *step : 0] = loss;
      if (!isfinite(loss) && err) atomicOr(err, kErrLossNonFinite);
    }
  }
}

template <typename T>
int launch_softmax_xent(int B, int C, const T* z, int ldz, const int64_t* y, T* dz, int lddz,
                        float* loss_hist, const int* step, int* err, cudaStream_t s) {
  int threads = B >= 32 ? 1024 : 32 * B;
  size_t smem = sizeof(float) * (size_t)B;
  if (smem > 48 * 1024) {
    set_error("softmax_xent: batch %d too large", B);
    return PPLL_ERR_ARG;
  }
  launch_k(softmax_xent_kernel<T>, 1, threads, smem, s, B, C, z, ldz, y, dz, lddz, loss_hist, step, err);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}
template int launch_softmax_xent<float>(int, int, const float*, int, const int64_t*, float*, int, float*, const int*, int*, cudaStream_t);
template int launch_softmax_xent<__nv_bfloat16>(int, int, const __nv_bfloat16*, int, const int64_t*, __nv_bfloat16*, int, float*, const int*, int*, cudaStream_t);

// ------------------------------------------------------------------------
// Fused classifier head of a local step (blocks.py:280-285 for the head's
// Linear + softmax_xent, tensor.py:137-150 / 201-234), one warp per row:
//   logits = z·W + b            (the rowwarp GEMM's arithmetic and order:
//                                lane-strided K, fmaf, xor-tree warp sum)
//   loss, dlog = softmax_xent   (the softmax_xent kernel's arithmetic on the
//                                stored logits; same fixed-order batch mean)
//   dz = dlog·Wᵀ                (the gemm_dot kernel's four FMA chains)
// so logits, dlog, dz and the loss are bitwise what the three separate
// launches produce, with two launches and their dependent latencies off the
// critical path of every stage step.  One 8-CTA cluster (rows split over the
// CTAs, 16 warps each): every CTA stages W [K, C] (the reference's (fan_in,
// fan_out) layout) in shared memory as fp32 [K][NP+1] with 16-B loads while
// its warps' row loads (all of a row's lane-strided elements, issued at once)
// are in flight; the row losses stay in each CTA's shared memory and rank 0
// gathers them over DSMEM in the fixed order of the batch mean.
// ------------------------------------------------------------------------
constexpr int kHeadCluster = 8, kHeadWarps = 16, kHeadMaxT = 24;   // K <= 768 in registers


template <typename T, int NP>
__global__ void __launch_bounds__(kHeadWarps * 32)
head_xent_kernel(int B, int K, int C, const T* __restrict__ z, int ldz, const T* __restrict__ W,
                 const float* __restrict__ bias, const int64_t* __restrict__ y,
                 T* __restrict__ logits, T* __restrict__ dlog, T* __restrict__ dz, int lddz,
                 float* loss_hist, const int* step, int* err) {
  constexpr int LD = NP + 1;
  extern __shared__ float hsm[];
  const int rank = (int)(blockIdx.x % kHeadCluster);
  const int rpc = (B + kHeadCluster - 1) / kHeadCluster;   // rows of this CTA: [rank·rpc, +rpc)
  float* ws = hsm;                                          // [K][LD]
  float* row_loss = ws + (size_t)K * LD;                    // [rpc]
  T* rowbuf = reinterpret_cast<T*>(row_loss + rpc);         // per warp: logits[32] | dlog[32]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r0 = rank * rpc, r1 = min(B, r0 + rpc);
  pdl_entry();
  // first row of this warp: every lane-strided element loaded before W is staged
  int r = r0 + w;
  float av[kHeadMaxT];
  auto load_row = [&](int row) {
    const T* zr = z + (long)row * ldz;
#pragma unroll
    for (int t = 0; t < kHeadMaxT; ++t) {
      const int k = lane + 32 * t;
      av[t] = (row < r1 && k < K) ? to_f(zr[k]) : 0.f;
    }
  };
  load_row(r);
  // W [K, C] contiguous: 16-B vectors when aligned, scattered into [K][LD]
  const long nW = (long)K * C;
  constexpr int V = 16 / sizeof(T);
  if ((reinterpret_cast<uintptr_t>(W) & 15) == 0 && nW % V == 0) {
    for (long v = threadIdx.x; v < nW / V; v += blockDim.x) {
      const uint4 q = reinterpret_cast<const uint4*>(W)[v];
      const T* e = reinterpret_cast<const T*>(&q);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const long idx = v * V + i;
        ws[(idx / C) * LD + idx % C] = to_f(e[i]);
      }
    }
  } else {
    for (long idx = threadIdx.x; idx < nW; idx += blockDim.x) ws[(idx / C) * LD + idx % C] = to_f(W[idx]);
  }
  if (C < NP)
    for (int i = threadIdx.x; i < K * (NP - C); i += blockDim.x)
      ws[(i / (NP - C)) * LD + C + i % (NP - C)] = 0.f;
  __syncthreads();
  T* lg = rowbuf + w * 64;
  T* dl = lg + 32;
  const float invB = 1.0f / (float)B;
  const int sl = lane & 15, seg = lane >> 4;
  for (; r < r1; r += kHeadWarps) {
    // ---- logits row r ----
    float acc[NP];
#pragma unroll
    for (int n = 0; n < NP; ++n) acc[n] = 0.f;
#pragma unroll
    for (int t = 0; t < kHeadMaxT; ++t) {
      const int k = lane + 32 * t;
      if (k < K) {
        const float* br = ws + k * LD;
#pragma unroll
        for (int n = 0; n < NP; ++n) acc[n] = fmaf(av[t], br[n], acc[n]);
      }
    }
    for (int k = lane + 32 * kHeadMaxT; k < K; k += 32) {   // K > 768: the rest streamed
      const float a = to_f(z[(long)r * ldz + k]);
      const float* br = ws + k * LD;
#pragma unroll
      for (int n = 0; n < NP; ++n) acc[n] = fmaf(a, br[n], acc[n]);
    }
    if (r + kHeadWarps < r1) load_row(r + kHeadWarps);   // next row's loads under this row's math
#pragma unroll
    for (int n = 0; n < NP; ++n) acc[n] = warp_sum(acc[n]);
    float mine = 0.f;
#pragma unroll
    for (int n = 0; n < NP; ++n)
      if (lane == n) mine = acc[n];
    if (lane < C) {
      float v = mine;
      if (bias) v += bias[lane];
      DT<T>::st(lg + lane, v);
      DT<T>::st(logits + (long)r * C + lane, v);
    }
    __syncwarp();
    // ---- softmax_xent on the stored row (half-warp arithmetic of softmax_xent_kernel;
    //      both halves evaluate the row, the lower half writes) ----
    const long lab = y[r];
    const bool bad = (lab < 0 || lab >= C);
    float mx = -INFINITY;
    for (int c = sl; c < C; c += 16) mx = fmaxf(mx, to_f(lg[c]));
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float se = 0.f, zl = 0.f;
    for (int c = sl; c < C; c += 16) {
      const float v = to_f(lg[c]);
      se += __expf(v - mx);
      if (c == lab) zl = v;
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      se += __shfl_xor_sync(0xffffffffu, se, o);
      zl += __shfl_xor_sync(0xffffffffu, zl, o);
    }
    const float inv = 1.0f / se;
    if (seg == 0) {
      for (int c = sl; c < C; c += 16) {
        const float p = __expf(to_f(lg[c]) - mx) * inv;
        const float g = bad ? 0.f : (p - (c == lab ? 1.f : 0.f)) * invB;
        DT<T>::st(dl + c, g);
        DT<T>::st(dlog + (long)r * C + c, g);
      }
      if (sl == 0) {
        row_loss[r - r0] = bad ? 0.f : -((zl - mx) - logf(se));
        if (bad && err) atomicOr(err, kErrLabel);
      }
    }
    __syncwarp();
    // ---- dz row r = dlog[r]·Wᵀ (gemm_dot's chains: k ≡ 0,1,2,3 mod 4) ----
    T* dzr = dz + (long)r * lddz;
    for (int n = lane; n < K; n += 32) {
      const float* wr = ws + n * LD;
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
      int k = 0;
      for (; k + 4 <= C; k += 4) {
        a0 = fmaf(to_f(dl[k]), wr[k], a0);
        a1 = fmaf(to_f(dl[k + 1]), wr[k + 1], a1);
        a2 = fmaf(to_f(dl[k + 2]), wr[k + 2], a2);
        a3 = fmaf(to_f(dl[k + 3]), wr[k + 3], a3);
      }
      for (; k < C; ++k) a0 = fmaf(to_f(dl[k]), wr[k], a0);
      DT<T>::st(dzr + n, (a0 + a1) + (a2 + a3));
    }
    __syncwarp();
  }
  ptx::cluster_sync();   // every CTA's row losses are in its shared memory
  if (rank == 0 && w == 0) {   // the softmax_xent kernel's fixed-order batch mean
    double s = 0.0;
    for (int q = lane; q < B; q += 32) s += (double)ptx::ld_dsmem_f32(ptx::smem_u32(row_loss + q % rpc), q / rpc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const float loss = (float)(s / (double)B);
      loss_hist[step ? *step : 0] = loss;
      if (!isfinite(loss) && err) atomicOr(err, kErrLossNonFinite);
    }
  }
  ptx::cluster_sync();   // peers keep their shared memory until rank 0 has read it
}

static size_t head_xent_smem(int B, int K, int np, size_t esz) {
  const int rpc = (B + kHeadCluster - 1) / kHeadCluster;
  return sizeof(float) * ((size_t)K * (np + 1) + (size_t)rpc) + kHeadWarps * 64 * esz;
}

bool head_xent_fusable(int B, int K, int C, size_t esz) {
  static const int on = getenv("PPLL_HEAD_FUSED") ? atoi(getenv("PPLL_HEAD_FUSED")) : 1;
  return on && C >= 1 && C <= 32 && K >= 64 && B >= 1 &&
         head_xent_smem(B, K, C <= 16 ? 16 : 32, esz) <= 200 * 1024;
}

template <typename T, int NP>
static int head_xent_go(int B, int K, int C, const T* z, int ldz, const T* W, const float* bias,
                        const int64_t* y, T* logits, T* dlog, T* dz, int lddz, float* loss_hist,
                        const int* step, int* err, cudaStream_t s) {
  auto kern = head_xent_kernel<T, NP>;
  static bool set = false;
  if (!set) {
    PPLL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kHeadCluster);
  cfg.blockDim = dim3(kHeadWarps * 32);
  cfg.dynamicSmemBytes = head_xent_smem(B, K, NP, sizeof(T));
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kHeadCluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  PPLL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, B, K, C, z, ldz, W, bias, y, logits, dlog, dz,
                                     lddz, loss_hist, step, err));
  return PPLL_OK;
}

template <typename T>
int launch_head_xent(int B, int K, int C, const T* z, int ldz, const T* W, const float* bias,
                     const int64_t* y, T* logits, T* dlog, T* dz, int lddz, float* loss_hist,
                     const int* step, int* err, cudaStream_t s) {
  if (!head_xent_fusable(B, K, C, sizeof(T))) return PPLL_ERR_UNSUPPORTED;
  const int r = C <= 16 ? head_xent_go<T, 16>(B, K, C, z, ldz, W, bias, y, logits, dlog, dz, lddz,
                                              loss_hist, step, err, s)
                        : head_xent_go<T, 32>(B, K, C, z, ldz, W, bias, y, logits, dlog, dz, lddz,
                                              loss_hist, step, err, s);
  if (r) return r;
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}
template int launch_head_xent<float>(int, int, int, const float*, int, const float*, const float*, const int64_t*, float*, float*, float*, int, float*, const int*, int*, cudaStream_t);
template int launch_head_xent<__nv_bfloat16>(int, int, int, const __nv_bfloat16*, int, const __nv_bfloat16*, const float*, const int64_t*, __nv_bfloat16*, __nv_bfloat16*, __nv_bfloat16*, int, float*, const int*, int*, cudaStream_t);

// ------------------------------------------------------------------------
// Nesterov-SGD over one flat buffer (optim.py:81-88):
//   g' = g + wd·θ ; v = μv + g' ; θ -= lr·(g' + μv)
// 20 B/param algorithmic (read θ,v,g; write θ,v) + 2 B for the bf16 shadow.
// The last block to finish advances the device step counter (optim.py:89).
// ------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
nesterov_kernel(long n, float* __restrict__ th, float* __restrict__ v, const float* __restrict__ g,
                __nv_bfloat16* __restrict__ th_lp, const float* __restrict__ lr_table, int* step,
                int max_step, float lr_host, float mu, float wd, int* err, unsigned int* done,
                int advance) {
  pdl_entry();
  __shared__ int s_skip;
  __shared__ float s_lr;
  if (threadIdx.x == 0) {
    int e = err ? *(volatile int*)err : 0;
    int st = step ? *(volatile int*)step : 0;
    int skip = (e & (kErrLabel | kErrLossNonFinite | kErrGradNonFinite)) ? 1 : 0;
    if (step && (st < 0 || st > max_step)) {
      skip = 1;
      if (err) atomicOr(err, kErrStep);
    }
    s_skip = skip;
    s_lr = step ? lr_table[min(max(st, 0), max_step)] : lr_host;
  }
  __syncthreads();
  bool bad = false;
  if (!s_skip) {
    const float lr = s_lr;
    long n4 = n / 4;
    float4* th4 = reinterpret_cast<float4*>(th);
    float4* v4 = reinterpret_cast<float4*>(v);
    const float4* g4 = reinterpret_cast<const float4*>(g);
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
      float4 t = th4[i], vv = v4[i], gg = g4[i];
      float gp;
#define NEST(c)                                  \
      gp = fmaf(wd, t.c, gg.c);                  \
      vv.c = fmaf(mu, vv.c, gp);                 \
      t.c = t.c - lr * fmaf(mu, vv.c, gp);       \
      bad |= !isfinite(t.c);
      NEST(x) NEST(y) NEST(z) NEST(w)
#undef NEST
      th4[i] = t;
      v4[i] = vv;
      if (th_lp) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(t.x, t.y);
        __nv_bfloat162 hi = __floats2bfloat162_rn(t.z, t.w);
        reinterpret_cast<__nv_bfloat162*>(th_lp)[2 * i] = lo;
        reinterpret_cast<__nv_bfloat162*>(th_lp)[2 * i + 1] = hi;
      }
    }
    for (long i = n4 * 4 + (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
      float t = th[i], gp = fmaf(wd, t, g[i]);
      float vv = fmaf(mu, v[i], gp);
      t = t - lr * fmaf(mu, vv, gp);
      th[i] = t;
      v[i] = vv;
      if (th_lp) th_lp[i] = __float2bfloat16_rn(t);
      bad |= !isfinite(t);
    }
  }
  if (bad && err) atomicOr(err, kErrParamNonFinite);
  if (step && advance) {
    // last block advances the step counter after every block has read it
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      unsigned int prev = atomicAdd(done, 1u);
      if (prev == gridDim.x - 1) {
        if (!s_skip) atomicAdd(step, 1);
        *done = 0u;
        __threadfence();
      }
    }
  }
}

// All-or-nothing guard in front of the update: the reference raises
// NonFiniteError inside the forward/backward (tensor.py:41-43, called from
// every primitive) BEFORE sgd_nesterov_step runs, so a non-finite value never
// reaches the parameters.  The device step cannot raise mid-graph; instead one
// pass over the gradient sets PPLL_ERRBIT_GRAD and the Nesterov kernel skips
// the whole update (a NaN input can be squashed by ReLU = fmaxf on the way to
// the loss, but it always reaches dW = Xᵀ·G).
__global__ void __launch_bounds__(256)
grad_finite_kernel(long n, const float* __restrict__ g, int* err) {
  pdl_entry();
  bool bad = false;
  const long n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    const float4 q = g4[i];
    bad |= !(isfinite(q.x) & isfinite(q.y) & isfinite(q.z) & isfinite(q.w));
  }
  for (long i = n4 * 4 + (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    bad |= !isfinite(g[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, kErrGradNonFinite);
}

// ------------------------------------------------------------------------
// AdamW over one flat buffer — the "local SGD/Adam update" of north_star.
// The reference has only Nesterov (optim.py:71-89); the Adam variant follows
// torch.optim.AdamW (decoupled weight decay, bias-corrected moments):
//   θ -= lr·wd·θ ; m = β1·m + (1-β1)·g ; v = β2·v + (1-β2)·g²
//   θ -= lr · (m / (1-β1^t)) / (sqrt(v / (1-β2^t)) + eps),  t = step + 1
// with the same device step counter, cosine-LR table, all-or-nothing skip and
// step advance as nesterov_kernel.  28 B/param (+2 for the bf16 shadow).
// ------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
adamw_kernel(long n, float* __restrict__ th, float* __restrict__ m1, float* __restrict__ m2,
             const float* __restrict__ g, __nv_bfloat16* __restrict__ th_lp,
             const float* __restrict__ lr_table, int* step, int max_step, float lr_host,
             float beta1, float beta2, float eps, float wd, int* err, unsigned int* done,
             int advance) {
  pdl_entry();
  __shared__ int s_skip;
  __shared__ float s_lr, s_c1, s_c2;
  if (threadIdx.x == 0) {
    int e = err ? *(volatile int*)err : 0;
    int st = step ? *(volatile int*)step : 0;
    int skip = (e & (kErrLabel | kErrLossNonFinite | kErrGradNonFinite)) ? 1 : 0;
    if (step && (st < 0 || st > max_step)) {
      skip = 1;
      if (err) atomicOr(err, kErrStep);
    }
    s_skip = skip;
    s_lr = step ? lr_table[min(max(st, 0), max_step)] : lr_host;
    const float t = (float)(max(st, 0) + 1);
    s_c1 = 1.0f / (1.0f - powf(beta1, t));
    s_c2 = 1.0f / (1.0f - powf(beta2, t));
  }
  __syncthreads();
  bool bad = false;
  if (!s_skip) {
    const float lr = s_lr, c1 = s_c1, c2 = s_c2, decay = 1.0f - s_lr * wd;
    const float ob1 = 1.0f - beta1, ob2 = 1.0f - beta2;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
      const float gi = g[i];
      const float a = fmaf(beta1, m1[i], ob1 * gi);
      const float b = fmaf(beta2, m2[i], ob2 * gi * gi);
      const float t = th[i] * decay - lr * (a * c1) / (sqrtf(b * c2) + eps);
      m1[i] = a;
      m2[i] = b;
      th[i] = t;
      if (th_lp) th_lp[i] = __float2bfloat16_rn(t);
      bad |= !isfinite(t);
    }
  }
  if (bad && err) atomicOr(err, kErrParamNonFinite);
  if (step && advance) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      unsigned int prev = atomicAdd(done, 1u);
      if (prev == gridDim.x - 1) {
        if (!s_skip) atomicAdd(step, 1);
        *done = 0u;
        __threadfence();
      }
    }
  }
}

// Per-flat-buffer optimizer choice: a stage whose θ buffer was registered
// with ppll_set_local_optimizer(AdamW) is updated by adamw_kernel wherever
// the stage executors call launch_nesterov (one switch for all families).
struct AdamCfg { float* m2; float beta1, beta2, eps; };
static std::mutex g_opt_mu;
static std::unordered_map<const float*, AdamCfg> g_opt;

int set_local_optimizer(const float* theta, int kind, float* m2, float beta1, float beta2,
                        float eps) {
  std::lock_guard<std::mutex> lk(g_opt_mu);
  if (kind == 0) {
    g_opt.erase(theta);
    return PPLL_OK;
  }
  if (kind != 1 || !m2 || !(beta1 >= 0.f && beta1 < 1.f) || !(beta2 >= 0.f && beta2 < 1.f) ||
      !(eps > 0.f)) {
    set_error("set_local_optimizer: bad arguments");
    return PPLL_ERR_ARG;
  }
  g_opt[theta] = AdamCfg{m2, beta1, beta2, eps};
  return PPLL_OK;
}

static bool adam_for(const float* theta, AdamCfg* out) {
  std::lock_guard<std::mutex> lk(g_opt_mu);
  auto it = g_opt.find(theta);
  if (it == g_opt.end()) return false;
  *out = it->second;
  return true;
}

int launch_nesterov(long n, float* th, float* v, const float* g, __nv_bfloat16* th_lp,
                    const float* lr_table, int* step, int max_step, float lr_host, float mu,
                    float wd, int* err, cudaStream_t s, bool advance) {
  if (n <= 0 && !advance) return PPLL_OK;
  long n4 = (n + 3) / 4;
  int blocks = (int)min((n4 + 255) / 256, (long)148 * 4);
  if (blocks < 1) blocks = 1;
  if ((reinterpret_cast<uintptr_t>(th) | reinterpret_cast<uintptr_t>(v) |
       reinterpret_cast<uintptr_t>(g)) & 15) {
    set_error("nesterov: flat buffers must be 16-byte aligned");
    return PPLL_ERR_ARG;
  }
  // step points to two int32 words: [step_count, block-completion scratch]
  unsigned int* done = step ? reinterpret_cast<unsigned int*>(step + 1) : nullptr;
  if (err && step && n > 0) {
    launch_k(grad_finite_kernel, blocks, 256, 0, s, n, g, err);
    note_launch();
    PPLL_LAUNCH_CHECK();
  }
  AdamCfg ad;
  if (adam_for(th, &ad))
    launch_k(adamw_kernel, blocks, 256, 0, s, n, th, v, ad.m2, g, th_lp, lr_table, step, max_step,
             lr_host, ad.beta1, ad.beta2, ad.eps, wd, err, done, advance ? 1 : 0);
  else
    launch_k(nesterov_kernel, blocks, 256, 0, s, n, th, v, g, th_lp, lr_table, step, max_step,
             lr_host, mu, wd, err, done, advance ? 1 : 0);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// ------------------------------------------------------------------------
// casts
// ------------------------------------------------------------------------
template <typename TS, typename TD>
__global__ void cast_kernel(long n, const TS* __restrict__ s, TD* __restrict__ d) {
  pdl_entry();
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    DT<TD>::st(d + i, to_f(s[i]));
}

int launch_cast(long n, const void* src, int sd, void* dst, int dd, cudaStream_t s) {
  int blocks = (int)min((n + 255) / 256, (long)148 * 8);
  if (blocks < 1) return PPLL_OK;
  if (sd == PPLL_F32 && dd == PPLL_BF16)
    launch_k(cast_kernel<float, __nv_bfloat16>, blocks, 256, 0, s, n, (const float*)src, (__nv_bfloat16*)dst);
  else if (sd == PPLL_BF16 && dd == PPLL_F32)
    launch_k(cast_kernel<__nv_bfloat16, float>, blocks, 256, 0, s, n, (const __nv_bfloat16*)src, (float*)dst);
  else if (sd == PPLL_F32 && dd == PPLL_F32)
    launch_k(cast_kernel<float, float>, blocks, 256, 0, s, n, (const float*)src, (float*)dst);
  else
    launch_k(cast_kernel<__nv_bfloat16, __nv_bfloat16>, blocks, 256, 0, s, n, (const __nv_bfloat16*)src, (__nv_bfloat16*)dst);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// ReLU adjoint alone (tensor.py:156): out = g * [act > 0] (subgradient 0 at 0)
template <typename T>
__global__ void relu_mask_kernel(long n, const T* __restrict__ g, const T* __restrict__ act,
                                 T* __restrict__ out) {
  pdl_entry();
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    DT<T>::st(out + i, to_f(act[i]) > 0.f ? to_f(g[i]) : 0.f);
}

int launch_relu_mask(long n, const void* g, const void* act, void* out, int dtype, cudaStream_t s) {
  int blocks = (int)min((n + 255) / 256, (long)148 * 8);
  if (blocks < 1) return PPLL_OK;
  if (dtype == PPLL_F32)
    launch_k(relu_mask_kernel<float>, blocks, 256, 0, s, n, (const float*)g, (const float*)act, (float*)out);
  else
    launch_k(relu_mask_kernel<__nv_bfloat16>, blocks, 256, 0, s, n, (const __nv_bfloat16*)g, (const __nv_bfloat16*)act,
                                            (__nv_bfloat16*)out);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// ------------------------------------------------------------------------
// data path: HBM-resident dataset -> batch (data.py:107-179 order on device)
// ------------------------------------------------------------------------
// dst[r, :] = cast(src[idx[r], :]); one warp per row, 16-B vectors when the
// row width allows (fp32 source, fp32 or bf16 destination).
template <typename TD>
__global__ void gather_rows_kernel(int n, long width, const float* __restrict__ src,
                                   const int64_t* __restrict__ idx, TD* __restrict__ dst,
                                   const int64_t* __restrict__ ysrc, int64_t* __restrict__ ydst,
                                   int vec) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n) return;
  const long row = idx[r];
  const float* s = src + row * width;
  TD* d = dst + (long)r * width;
  if (ysrc && lane == 0) ydst[r] = ysrc[row];
  if (vec) {
    for (long c = 4 * lane; c < width; c += 128) {
      const float4 v = *reinterpret_cast<const float4*>(s + c);
      if constexpr (sizeof(TD) == 4) {
        *reinterpret_cast<float4*>(d + c) = v;
      } else {
        __nv_bfloat162 h[2] = {__floats2bfloat162_rn(v.x, v.y), __floats2bfloat162_rn(v.z, v.w)};
        *reinterpret_cast<uint2*>(d + c) = *reinterpret_cast<uint2*>(h);
      }
    }
  } else {
    for (long c = lane; c < width; c += 32) DT<TD>::st(d + c, s[c]);
  }
}

int launch_gather_rows(int n, long width, const float* src, const int64_t* idx, void* dst,
                       int dst_dtype, const int64_t* ysrc, int64_t* ydst, cudaStream_t s) {
  if (n <= 0) return PPLL_OK;
  const int vec = (width % 4) == 0 && ((uintptr_t)src & 15) == 0 &&
                  ((uintptr_t)dst & (dst_dtype == PPLL_F32 ? 15 : 7)) == 0;
  const int blocks = (n + 7) / 8;
  if (dst_dtype == PPLL_F32)
    launch_k(gather_rows_kernel<float>, blocks, 256, 0, s, n, width, src, idx, (float*)dst, ysrc, ydst,
                                                     vec);
  else
    launch_k(gather_rows_kernel<__nv_bfloat16>, blocks, 256, 0, s, n, width, src, idx,
                                                             (__nv_bfloat16*)dst, ysrc, ydst, vec);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// IDX pixels kept in HBM as the file's bytes (1 B/feature, a quarter of fp32):
// one warp per row, 16 pixels per lane-load, value = byte / 255 with IEEE
// division (load_idx scales to [0,1], data.py:137-139), fused bf16 cast
template <typename TD>
__global__ void gather_rows_u8_kernel(int n, long width, const uint8_t* __restrict__ src,
                                      const int64_t* __restrict__ idx, TD* __restrict__ dst,
                                      const int64_t* __restrict__ ysrc, int64_t* __restrict__ ydst,
                                      int vec) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n) return;
  const long row = idx[r];
  const uint8_t* s = src + row * width;
  TD* d = dst + (long)r * width;
  if (ysrc && lane == 0) ydst[r] = ysrc[row];
  if (vec) {
    for (long c = 16 * lane; c < width; c += 512) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(s + c));
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float f[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) f[b] = __fdiv_rn((float)((w[q] >> (8 * b)) & 0xffu), 255.f);
        if constexpr (sizeof(TD) == 4) {
          *reinterpret_cast<float4*>(d + c + 4 * q) = make_float4(f[0], f[1], f[2], f[3]);
        } else {
          __nv_bfloat162 h[2] = {__floats2bfloat162_rn(f[0], f[1]), __floats2bfloat162_rn(f[2], f[3])};
          *reinterpret_cast<uint2*>(d + c + 4 * q) = *reinterpret_cast<uint2*>(h);
        }
      }
    }
  } else {
    for (long c = lane; c < width; c += 32) DT<TD>::st(d + c, __fdiv_rn((float)s[c], 255.f));
  }
}

int launch_gather_rows_u8(int n, long width, const uint8_t* src, const int64_t* idx, void* dst,
                          int dst_dtype, const int64_t* ysrc, int64_t* ydst, cudaStream_t s) {
  if (n <= 0) return PPLL_OK;
  const int vec = (width % 16) == 0 && ((uintptr_t)src & 15) == 0 &&
                  ((uintptr_t)dst & (dst_dtype == PPLL_F32 ? 15 : 7)) == 0;
  const int blocks = (n + 7) / 8;
  if (dst_dtype == PPLL_F32)
    launch_k(gather_rows_u8_kernel<float>, blocks, 256, 0, s, n, width, src, idx, (float*)dst,
             ysrc, ydst, vec);
  else
    launch_k(gather_rows_u8_kernel<__nv_bfloat16>, blocks, 256, 0, s, n, width, src, idx,
             (__nv_bfloat16*)dst, ysrc, ydst, vec);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// evaluate (harness.py:121-131): count rows whose argmax (first maximum, like
// numpy) equals the label; integer atomics, so the count is exact
template <typename T>
__global__ void count_correct_kernel(int B, int C, const T* __restrict__ z, long ldz,
                                     const int64_t* __restrict__ y, unsigned long long* count) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= B) return;
  float best = -INFINITY;
  int arg = 0x7fffffff;
  for (int c = lane; c < C; c += 32) {
    const float v = to_f(z[(long)r * ldz + c]);
    if (v > best || (v == best && c < arg) || (v != v && arg == 0x7fffffff)) { best = v; arg = c; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
    if (ob > best || (ob == best && oa < arg)) { best = ob; arg = oa; }
  }
  if (lane == 0 && (long long)arg == y[r]) atomicAdd(count, 1ull);
}

int launch_count_correct(int B, int C, const void* z, long ldz, int dtype, const int64_t* y,
                         unsigned long long* count, cudaStream_t s) {
  if (B <= 0) return PPLL_OK;
  const int blocks = (B + 7) / 8;
  if (dtype == PPLL_F32)
    launch_k(count_correct_kernel<float>, blocks, 256, 0, s, B, C, (const float*)z, ldz, y, count);
  else
    launch_k(count_correct_kernel<__nv_bfloat16>, blocks, 256, 0, s, B, C, (const __nv_bfloat16*)z, ldz, y, count);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// ------------------------------------------------------------------------
// ring flag words (runtime.py:88-115 push/pop/close semantics on device)
// ------------------------------------------------------------------------
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

__global__ void ring_publish_kernel(int* w, int seq) {
  pdl_entry();
  __threadfence_system();
  st_release_sys(w, seq);
}
// Watchdog (SURVEY §5 "host watchdog on flag progress"): a wait that sees no
// progress for `timeout_ns` (%globaltimer) gives up instead of hanging the GPU,
// and records {stalled, wanted, seen, kind} once in g_ring_stall, which the
// host reads with ppll_ring_stall() and maps to WorkerPanic.  kind: 0 = ready
// flag (pop), 1 = credit (backpressure).
__device__ int g_ring_stall[4];
__global__ void ring_wait_kernel(const int* w, int seq, long long timeout_ns, int kind) {
  pdl_entry();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  int v;
  while ((v = ld_acquire_sys(w)) < seq) {
    __nanosleep(64);
    if (timeout_ns > 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if ((long long)(t - t0) > timeout_ns) {
        if (atomicCAS(&g_ring_stall[0], 0, 1) == 0) {
          g_ring_stall[1] = seq;
          g_ring_stall[2] = v;
          g_ring_stall[3] = kind;
        }
        break;
      }
    }
  }
  __threadfence_system();
}
long long g_ring_timeout_ns = getenv("PPLL_RING_TIMEOUT_MS")
                                  ? (long long)atoll(getenv("PPLL_RING_TIMEOUT_MS")) * 1000000LL
                                  : 30000000000LL;
__global__ void ring_release_kernel(int* w) {
  pdl_entry();
  __threadfence_system();
  atomicAdd_system(w, 1);
}

int launch_ring_publish(int* w, int seq, cudaStream_t s) {
  launch_k(ring_publish_kernel, 1, 1, 0, s, w, seq);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}
int launch_ring_wait(const int* w, int seq, cudaStream_t s, int kind) {
  launch_k(ring_wait_kernel, 1, 1, 0, s, w, seq, g_ring_timeout_ns, kind);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}
int launch_ring_release(int* w, cudaStream_t s) {
  launch_k(ring_release_kernel, 1, 1, 0, s, w);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

int ring_stall_read(int* out4, bool clear) {
  int h[4];
  PPLL_CUDA_CHECK(cudaMemcpyFromSymbol(h, g_ring_stall, sizeof(h)));
  if (out4) memcpy(out4, h, sizeof(h));
  if (clear && h[0]) {
    const int z[4] = {0, 0, 0, 0};
    PPLL_CUDA_CHECK(cudaMemcpyToSymbol(g_ring_stall, z, sizeof(z)));
  }
  return h[0];
}

}  // namespace ppll
