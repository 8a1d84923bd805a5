// Single-cluster fused training-mode BatchNorm for NHWC bf16 activations
// (the ResNet stage's conv → BN → [+BN' | +res] → ReLU and its adjoint).
//
// The unfused path is three launches per forward BN (partial statistics →
// merge → apply) and four per backward BN (ReLU mask → partial sums → merge →
// dx); on the CIFAR shapes (0.5-8 MB per tensor) each is a few µs of launch
// and tail latency around well under a µs of traffic.  Here ONE launch of one
// thread-block cluster (8 or 16 CTAs, one per SM) does the whole BN:
//
//   1. each CTA streams its contiguous row slice of the inputs through a
//      shared-memory ring with bulk async copies (cp.async.bulk, up to
//      ~150 KB in flight per SM) and accumulates per-thread statistics
//      (forward: shifted sums → Welford triples; backward: Σ dy·x̂, Σ dy with
//      the ReLU mask applied on the fly);
//   2. warp butterflies (ordered merges), a fixed-order sum over warps, then
//      every CTA merges the CS per-CTA partials read over distributed shared
//      memory in rank order — the same arithmetic in every CTA, so all CTAs
//      hold identical statistics; rank 0 publishes mean / rstd (forward) or
//      dγ / dβ (backward);
//   3. each CTA re-reads its slice (an L2 hit: the tensor was just streamed)
//      and writes y = act(BN(z) [+ BN'(z') | + res]) or
//      dz = γ·rstd·(dy − (dβ + x̂·dγ)/P) (and dz' for the shortcut BN, and the
//      masked dy when the identity shortcut needs it).
//
// Deterministic (fixed merge orders, no atomics).  Reference semantics: the
// batch-statistics BN of oracle/resnet_oracle.py (the reference itself has no
// BN — SURVEY §8 ResNet extension row).
#include <cuda.h>
#include <stdlib.h>
#include <mutex>
#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"
#include "resnet.cuh"

namespace ppll {
namespace tc { unsigned long long* timeline_buffer(); }
namespace bnc {
using namespace ptx;

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxC = 128;           // V = C/8 <= 16 vectors per row
constexpr int kRing = 176 * 1024;    // bulk-copy ring
constexpr int kMaxSlots = 22;
constexpr int kWredOff = kRing;                              // [kWarps][kMaxC] float4
constexpr int kCpartOff = kWredOff + kWarps * kMaxC * 16;    // [kMaxC] float4
constexpr int kCoefOff = kCpartOff + kMaxC * 16;             // [8][kMaxC] float
constexpr int kBarOff = kCoefOff + 8 * kMaxC * 4;            // 4 x kMaxSlots mbarriers
constexpr int kSmem = kBarOff + 4 * kMaxSlots * 8 + 1024;    // + alignment slack

struct FwdArgs {
  int P, C;
  const __nv_bfloat16* z;
  const float *g, *b;
  float *mean, *rstd;
  const __nv_bfloat16* z2;            // optional second BN (projection shortcut)
  const float *g2, *b2;
  float *mean2, *rstd2;
  const __nv_bfloat16* res;           // optional identity residual
  int relu;
  __nv_bfloat16* y;
  unsigned long long* tl;             // PPLL_BN_TIMELINE probe: per CTA 8 %globaltimer stamps
  float4* gpart;                      // grid form: per-CTA partials [grid][C]
  unsigned* gbar;                     // grid form: {arrivals, generation}
  int* err;                           // grid form: sticky error word (watchdog: kErrSync)
  int ncl;                            // split form: cluster partials written by launch A
};

struct BwdArgs {
  int P, C;
  float invP;
  const __nv_bfloat16* dout;          // gradient w.r.t. the (post-activation) output
  const __nv_bfloat16* out;           // optional: dy = dout ⊙ [out > 0]
  __nv_bfloat16* dy_store;            // optional: the masked dy (identity-shortcut gradient)
  const __nv_bfloat16* z;
  const float *mean, *rstd, *g;
  float *dg, *db;
  __nv_bfloat16* dz;
  const __nv_bfloat16* z2;            // optional second BN sharing dy (projection shortcut)
  const float *mean2, *rstd2, *g2;
  float *dg2, *db2;
  __nv_bfloat16* dz2;
  unsigned long long* tl;
  float4* gpart;
  unsigned* gbar;
  int* err;
  int ncl;
};

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// bf16x2 -> fp32x2 (exact) and back (round to nearest even)
__device__ __forceinline__ float2 up2(uint32_t u) {
  return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
}
__device__ __forceinline__ uint32_t dn2(float2 v) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(v.x, v.y);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t relu2(uint32_t u) {
  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&u);
  h = __hmax2(h, __float2bfloat162_rn(0.f));
  return *reinterpret_cast<uint32_t*>(&h);
}
// bf16x2 lanes of d kept where the matching lane of o is > 0 (else +0)
__device__ __forceinline__ uint32_t mask_pos2(uint32_t d, uint32_t o) {
  const __nv_bfloat162 ho = *reinterpret_cast<const __nv_bfloat162*>(&o);
  return d & __hgt2_mask(ho, __float2bfloat162_rn(0.f));
}
__device__ __forceinline__ uint32_t w32(const uint4& q, int p) {
  return p == 0 ? q.x : p == 1 ? q.y : p == 2 ? q.z : q.w;
}

#define BN_TL(k) \
  if (a.tl && threadIdx.x == 0) a.tl[blockIdx.x * 8 + (k)] = gtimer();

// A CTA's contiguous row slice of NT tensors (same byte range in each)
// streamed through the shared-memory ring in chunks: slot = NT pieces of
// PIECE bytes filled by bulk async copies (one elected thread issues,
// completion on full[slot]); each warp releases a slot on empty[slot] once
// done, and the issuing thread refills it.  When every chunk fits in the ring
// at once (`resident`), nothing is refilled and the slice stays in shared
// memory for a second pass.
template <int NT>
struct Ring {
  static constexpr int PIECE = NT == 1 ? 16384 : 8192;
  static constexpr int SLOT = NT * PIECE;
  static constexpr int NS = (kRing / SLOT) < kMaxSlots ? (kRing / SLOT) : kMaxSlots;
  uint8_t* base;
  uint64_t *full, *empty;
  const uint8_t* src[NT];
  long bytes, nch;
  __device__ static bool fits(long bytes) { return (bytes + PIECE - 1) / PIECE <= NS; }
  __device__ void init(uint8_t* b, uint64_t* bars, long nbytes) {
    base = b;
    full = bars;
    empty = bars + kMaxSlots;
    bytes = nbytes;
    nch = (bytes + PIECE - 1) / PIECE;
  }
  __device__ void issue(long i) const {
    const int sl = (int)(i % NS);
    const uint32_t nb = (uint32_t)min((long)PIECE, bytes - i * PIECE);
    mbar_expect_tx(&full[sl], NT * nb);
#pragma unroll
    for (int k = 0; k < NT; ++k)
      bulk_g2s(smem_u32(base + sl * SLOT + k * PIECE), src[k] + i * PIECE, nb, &full[sl]);
  }
  __device__ void start() const {
    if (threadIdx.x == 0)
      for (long i = 0; i < NS && i < nch; ++i) issue(i);
  }
  __device__ const uint8_t* wait(long i) const {
    mbar_wait(&full[i % NS], (uint32_t)((i / NS) & 1));
    return base + (i % NS) * SLOT;
  }
  __device__ const uint8_t* slot(long i) const { return base + (i % NS) * SLOT; }
  __device__ int nvec(long i) const { return (int)(min((long)PIECE, bytes - i * PIECE) / 16); }
  __device__ void release(long i) const {
    if (i + NS >= nch) return;            // never refilled
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[i % NS]);
    if (threadIdx.x == 0) {
      mbar_wait(&empty[i % NS], (uint32_t)((i / NS) & 1));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + NS);
    }
  }
};

__device__ __forceinline__ void init_bars(uint64_t* bars) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4 * kMaxSlots; ++i) mbar_init(&bars[i], (i / kMaxSlots) & 1 ? kWarps : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

// Σ over the lanes of a warp that hold the same channel vector (lane ≡ vc mod
// V): xor butterfly, commutative adds (every lane ends with the same value)
__device__ __forceinline__ float lanes_sum(float v, int V) {
  for (int off = V; off < 32; off <<= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}


// ---- cross-CTA merge of the per-channel partials (cpart[c], c < C) ----------
// CLUSTER: read the CS peers' partials over DSMEM in rank order.
// GRID (cooperative launch, every CTA co-resident): publish the partial to
// global memory, meet at a self-resetting grid barrier (arrival count +
// generation word; a watchdog gives up after ~0.5 s and raises the flag word
// instead of hanging), then sum the grid's partials in a fixed decomposition
// (512/C strided groups in ascending CTA order, groups combined in order).
__device__ __forceinline__ void grid_barrier(unsigned* bar, int* err) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar + 1;
    const unsigned g = *vgen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      const unsigned long long t0 = gtimer();
      while (*vgen == g) {
        if (gtimer() - t0 > 500000000ull) {
          if (err) atomicOr(err, kErrSync);
          break;
        }
      }
    }
    __threadfence();
  }
  __syncthreads();
}
template <bool GRID>
__device__ __forceinline__ float4 merge_partials(const float4* cpart, float4* scratch, int C,
                                                 float4* gpart, unsigned* gbar, int* err,
                                                 unsigned long long* tl = nullptr) {
  const int t = threadIdx.x;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if constexpr (!GRID) {
    cluster_sync();   // every CTA's partial sums are in its shared memory
    if (tl && t == 0) tl[blockIdx.x * 8 + 7] = gtimer();
    if (t < C) {
      const int CS = (int)cluster_nctarank();
      const uint32_t la = smem_u32(&cpart[t]);
      float4 q[16];
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r < CS) q[r] = ld_dsmem_f4(la, (uint32_t)r);
      acc = q[0];
#pragma unroll
      for (int r = 1; r < 16; ++r)
        if (r < CS) { acc.x += q[r].x; acc.y += q[r].y; acc.z += q[r].z; acc.w += q[r].w; }
    }
  } else {
    if (t < C) gpart[(long)blockIdx.x * C + t] = cpart[t];
    __threadfence();
    grid_barrier(gbar, err);
    const int G = kThreads / C, g = t / C, c = t % C;
    float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (g < G)
      for (int r0 = g; r0 < (int)gridDim.x; r0 += 8 * G) {   // eight loads in flight
        float4 q[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int r = r0 + u * G;
          q[u] = r < (int)gridDim.x ? __ldcg(&gpart[(long)r * C + c]) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) { s4.x += q[u].x; s4.y += q[u].y; s4.z += q[u].z; s4.w += q[u].w; }
      }
    if (g < G) scratch[g * C + c] = s4;
    __syncthreads();
    if (t < C) {
      acc = scratch[t];
      for (int k = 1; k < G; ++k) {
        const float4 q = scratch[k * C + t];
        acc.x += q.x; acc.y += q.y; acc.z += q.z; acc.w += q.w;
      }
    }
  }
  return acc;
}

// SPLIT form (stage streams sharing the GPU, tensors past the one-cluster
// range): launch A (SPLIT = 1) = statistics over the whole grid, merged per
// 8-CTA cluster over DSMEM, rank 0 writing the cluster's partial to
// gpart[cluster]; launch B (SPLIT = 2, plain grid) = every CTA sums the ncl
// cluster partials in ascending order, then applies.  No grid barrier (the
// kernel boundary orders A before B), two launches instead of three / four.
__device__ __forceinline__ float4 split_partial_out(const float4* cpart, int C, float4* gpart) {
  const float4 acc = merge_partials<false>(cpart, nullptr, C, nullptr, nullptr, nullptr);
  if (threadIdx.x < C && cluster_ctarank() == 0)
    gpart[(long)(blockIdx.x / cluster_nctarank()) * C + threadIdx.x] = acc;
  return acc;
}
__device__ __forceinline__ float4 split_partial_in(int C, const float4* gpart, int ncl) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (threadIdx.x < C)
    for (int k = 0; k < ncl; ++k) {
      const float4 q = __ldcg(&gpart[(long)k * C + threadIdx.x]);
      acc.x += q.x; acc.y += q.y; acc.z += q.z; acc.w += q.w;
    }
  return acc;
}

// ---------------------------------------------------------------------------
// forward: per channel, with one shift K = z[0, c] for the whole cluster,
//   S1 = Σ (z − K), S2 = Σ (z − K)²   (plain fixed-order sums, no divisions)
//   mean = K + S1/P, var = S2/P − (S1/P)², rstd = 1/sqrt(var + eps)
//   y = act( z·s + t  [+ z2·s2 + t2 | + res] ),  s = γ·rstd, t = β − mean·s
// RESIDENT: the whole slice (incl. res) fits in the ring: one HBM read.
// ---------------------------------------------------------------------------
template <bool TWO, bool RES, bool RESIDENT, bool GRID = false, int SPLIT = 0>
__global__ void __launch_bounds__(kThreads, 1) bn_fwd_cluster_kernel(const __grid_constant__ FwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  float4* wred = reinterpret_cast<float4*>(smem + kWredOff);
  float4* cpart = reinterpret_cast<float4*>(smem + kCpartOff);
  float* coef = reinterpret_cast<float*>(smem + kCoefOff);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int C = a.C, V = C >> 3, vc = t % V;
  // row slice of this CTA: over the cluster (one-cluster form) or over the grid
  const int CS = (GRID || SPLIT) ? (int)gridDim.x : (int)cluster_nctarank();
  const int rank = (GRID || SPLIT) ? (int)blockIdx.x : (int)cluster_ctarank();
  const int rpc = (a.P + CS - 1) / CS;
  const int r0 = min(a.P, rank * rpc), r1 = min(a.P, r0 + rpc);
  const long bytes = (long)(r1 - r0) * C * 2, o = (long)r0 * C;
  init_bars(bars);
  BN_TL(0)
  pdl_entry();
  BN_TL(1)

  constexpr int NT1 = 1 + (TWO ? 1 : 0) + (RES && RESIDENT ? 1 : 0);
  static_assert(SPLIT != 2 || !RESIDENT, "the apply-only launch streams its slice");
  Ring<NT1> r1g;
  r1g.init(smem, bars, bytes);
  r1g.src[0] = reinterpret_cast<const uint8_t*>(a.z + o);
  if constexpr (TWO) r1g.src[1] = reinterpret_cast<const uint8_t*>(a.z2 + o);
  if constexpr (RES && RESIDENT) r1g.src[NT1 - 1] = reinterpret_cast<const uint8_t*>(a.res + o);
  if constexpr (SPLIT != 2) r1g.start();

  // the cluster-wide shift: row 0 of the tensor (a sample of every channel)
  float2 nk[4], s1[4], s2[4], nk2[4], u1[4], u2[4];
  {
    const uint4 q = reinterpret_cast<const uint4*>(a.z)[vc];
    const uint4 q2 = TWO ? reinterpret_cast<const uint4*>(a.z2)[vc] : q;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const float2 k = up2(w32(q, p)), k2 = up2(w32(q2, p));
      nk[p] = make_float2(-k.x, -k.y);
      nk2[p] = make_float2(-k2.x, -k2.y);
      s1[p] = s2[p] = u1[p] = u2[p] = make_float2(0.f, 0.f);
    }
  }
  for (long i = 0; i < (SPLIT == 2 ? 0 : r1g.nch); ++i) {
    const uint8_t* sl = r1g.wait(i);
    const int nv = r1g.nvec(i);
    for (int v = t; v < nv; v += kThreads) {
      const uint4 q = reinterpret_cast<const uint4*>(sl)[v];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const float2 d = __fadd2_rn(up2(w32(q, p)), nk[p]);
        s1[p] = __fadd2_rn(s1[p], d);
        s2[p] = __ffma2_rn(d, d, s2[p]);
      }
      if constexpr (TWO) {
        const uint4 q2 = reinterpret_cast<const uint4*>(sl + Ring<NT1>::PIECE)[v];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const float2 d = __fadd2_rn(up2(w32(q2, p)), nk2[p]);
          u1[p] = __fadd2_rn(u1[p], d);
          u2[p] = __ffma2_rn(d, d, u2[p]);
        }
      }
    }
    if constexpr (!RESIDENT) r1g.release(i);
  }
  BN_TL(2)
  // this thread's channel (t < C) parameters, loaded while the merges run
  float pg = 0.f, pb = 0.f, pg2 = 0.f, pb2 = 0.f, pk = 0.f, pk2 = 0.f;
  if (t < C) {
    pg = a.g[t];
    pb = a.b[t];
    pk = __bfloat162float(a.z[t]);
    if (TWO) {
      pg2 = a.g2[t];
      pb2 = a.b2[t];
      pk2 = __bfloat162float(a.z2[t]);
    }
  }
  // threads -> warp -> CTA (fixed order over warps)
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const float a0 = lanes_sum(s1[p].x, V), a1 = lanes_sum(s1[p].y, V);
    const float b0 = lanes_sum(s2[p].x, V), b1 = lanes_sum(s2[p].y, V);
    float c0 = 0.f, c1 = 0.f, d0 = 0.f, d1 = 0.f;
    if (TWO) {
      c0 = lanes_sum(u1[p].x, V); c1 = lanes_sum(u1[p].y, V);
      d0 = lanes_sum(u2[p].x, V); d1 = lanes_sum(u2[p].y, V);
    }
    if (lane < V) {
      wred[warp * kMaxC + vc * 8 + 2 * p] = make_float4(a0, b0, c0, d0);
      wred[warp * kMaxC + vc * 8 + 2 * p + 1] = make_float4(a1, b1, c1, d1);
    }
  }
  __syncthreads();
  if (t < C) {
    float4 sacc = wred[t];
    for (int k = 1; k < kWarps; ++k) {
      const float4 q = wred[k * kMaxC + t];
      sacc.x += q.x; sacc.y += q.y; sacc.z += q.z; sacc.w += q.w;
    }
    cpart[t] = sacc;
  }
  BN_TL(3)
  float4 sacc;
  if constexpr (SPLIT == 1) {
    split_partial_out(cpart, C, a.gpart);
    cluster_arrive();
    cluster_wait();
    return;
  } else if constexpr (SPLIT == 2) {
    sacc = split_partial_in(C, a.gpart, a.ncl);
  } else {
    sacc = merge_partials<GRID>(cpart, wred, C, a.gpart, a.gbar, a.err, a.tl);
  }
  if (t < C) {
    const float invP = 1.f / (float)a.P;
    {
      const float m1 = sacc.x * invP;
      const float mean = pk + m1;
      const float rstd = rsqrtf(fmaxf(fmaf(-m1, m1, sacc.y * invP), 0.f) + kBnEps);
      const float sc = rstd * pg;
      coef[t] = sc;
      coef[kMaxC + t] = fmaf(-mean, sc, pb);
      if (rank == 0) { a.mean[t] = mean; a.rstd[t] = rstd; }
    }
    if (TWO) {
      const float m1 = sacc.z * invP;
      const float mean = pk2 + m1;
      const float rstd = rsqrtf(fmaxf(fmaf(-m1, m1, sacc.w * invP), 0.f) + kBnEps);
      const float sc = rstd * pg2;
      coef[2 * kMaxC + t] = sc;
      coef[3 * kMaxC + t] = fmaf(-mean, sc, pb2);
      if (rank == 0) { a.mean2[t] = mean; a.rstd2[t] = rstd; }
    }
  }
  if constexpr (!GRID && !SPLIT) cluster_arrive();   // done reading the peers' partials
  __syncthreads();
  BN_TL(4)

  float2 sc[4], sh[4], sc2[4], sh2[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int c = vc * 8 + 2 * p;
    sc[p] = make_float2(coef[c], coef[c + 1]);
    sh[p] = make_float2(coef[kMaxC + c], coef[kMaxC + c + 1]);
    sc2[p] = TWO ? make_float2(coef[2 * kMaxC + c], coef[2 * kMaxC + c + 1]) : sc[p];
    sh2[p] = TWO ? make_float2(coef[3 * kMaxC + c], coef[3 * kMaxC + c + 1]) : sh[p];
  }
  uint4* y4 = reinterpret_cast<uint4*>(a.y + o);
  constexpr int NT3 = 1 + (TWO ? 1 : 0) + (RES ? 1 : 0);
  auto apply = [&](const uint8_t* sl, int piece, int nv, long v0) {
    for (int v = t; v < nv; v += kThreads) {
      const uint4 q = reinterpret_cast<const uint4*>(sl)[v];
      uint4 q2, qr;
      if (TWO) q2 = reinterpret_cast<const uint4*>(sl + piece)[v];
      if (RES) qr = reinterpret_cast<const uint4*>(sl + (NT3 - 1) * piece)[v];
      uint32_t w[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        float2 y = __ffma2_rn(up2(w32(q, p)), sc[p], sh[p]);
        if (TWO) y = __fadd2_rn(y, __ffma2_rn(up2(w32(q2, p)), sc2[p], sh2[p]));
        if (RES) y = __fadd2_rn(y, up2(w32(qr, p)));
        w[p] = a.relu ? relu2(dn2(y)) : dn2(y);
      }
      y4[v0 + v] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  };
  if constexpr (RESIDENT) {
    for (long i = 0; i < r1g.nch; ++i)
      apply(r1g.slot(i), Ring<NT1>::PIECE, r1g.nvec(i), i * (Ring<NT1>::PIECE / 16));
  } else {
    Ring<NT3> r3;
    r3.init(smem, bars + 2 * kMaxSlots, bytes);
    r3.src[0] = reinterpret_cast<const uint8_t*>(a.z + o);
    if constexpr (TWO) r3.src[1] = reinterpret_cast<const uint8_t*>(a.z2 + o);
    if constexpr (RES) r3.src[NT3 - 1] = reinterpret_cast<const uint8_t*>(a.res + o);
    r3.start();
    for (long i = 0; i < r3.nch; ++i) {
      apply(r3.wait(i), Ring<NT3>::PIECE, r3.nvec(i), i * (Ring<NT3>::PIECE / 16));
      r3.release(i);
    }
  }
  BN_TL(5)
  if constexpr (!GRID && !SPLIT) cluster_wait();   // no CTA leaves while a peer may still read its partial
  BN_TL(6)
}

// ---------------------------------------------------------------------------
// backward: dy = dout [⊙ (out > 0)];  dγ = Σ dy·x̂, dβ = Σ dy (cluster-merged);
//   dz = γ·rstd·(dy − (dβ + x̂·dγ)/P) = A·dy + B·z + D   [dz2 likewise]
// ---------------------------------------------------------------------------
template <bool MASK, bool TWO, bool RESIDENT, bool GRID = false, int SPLIT = 0>
__global__ void __launch_bounds__(kThreads, 1) bn_bwd_cluster_kernel(const __grid_constant__ BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  float4* wred = reinterpret_cast<float4*>(smem + kWredOff);
  float4* cpart = reinterpret_cast<float4*>(smem + kCpartOff);
  float* coef = reinterpret_cast<float*>(smem + kCoefOff);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int C = a.C, V = C >> 3, vc = t % V;
  const int CS = (GRID || SPLIT) ? (int)gridDim.x : (int)cluster_nctarank();
  const int rank = (GRID || SPLIT) ? (int)blockIdx.x : (int)cluster_ctarank();
  const int rpc = (a.P + CS - 1) / CS;
  const int r0 = min(a.P, rank * rpc), r1 = min(a.P, r0 + rpc);
  const long bytes = (long)(r1 - r0) * C * 2, o = (long)r0 * C;
  init_bars(bars);
  BN_TL(0)
  pdl_entry();
  BN_TL(1)

  constexpr int NT = 2 + (MASK ? 1 : 0) + (TWO ? 1 : 0);
  constexpr int kOut = 1, kZ = MASK ? 2 : 1, kZ2 = kZ + 1;
  Ring<NT> rg;
  rg.init(smem, bars, bytes);
  rg.src[0] = reinterpret_cast<const uint8_t*>(a.dout + o);
  if constexpr (MASK) rg.src[kOut] = reinterpret_cast<const uint8_t*>(a.out + o);
  rg.src[kZ] = reinterpret_cast<const uint8_t*>(a.z + o);
  if constexpr (TWO) rg.src[kZ2] = reinterpret_cast<const uint8_t*>(a.z2 + o);
  static_assert(SPLIT != 2 || !RESIDENT, "the apply-only launch streams its slice");
  if constexpr (SPLIT != 2) rg.start();

  // x̂ = z·rstd − mean·rstd
  float2 rs[4], nm[4], rs2[4], nm2[4], sg[4], sb[4], sg2[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int c = vc * 8 + 2 * p;
    rs[p] = make_float2(a.rstd[c], a.rstd[c + 1]);
    nm[p] = make_float2(-a.mean[c] * rs[p].x, -a.mean[c + 1] * rs[p].y);
    rs2[p] = TWO ? make_float2(a.rstd2[c], a.rstd2[c + 1]) : rs[p];
    nm2[p] = TWO ? make_float2(-a.mean2[c] * rs2[p].x, -a.mean2[c + 1] * rs2[p].y) : nm[p];
    sg[p] = sb[p] = sg2[p] = make_float2(0.f, 0.f);
  }
  for (long i = 0; i < (SPLIT == 2 ? 0 : rg.nch); ++i) {
    const uint8_t* sl = rg.wait(i);
    const int nv = rg.nvec(i);
    for (int v = t; v < nv; v += kThreads) {
      const uint4 qd = reinterpret_cast<const uint4*>(sl)[v];
      const uint4 qz = reinterpret_cast<const uint4*>(sl + kZ * Ring<NT>::PIECE)[v];
      uint4 qo, q2;
      if (MASK) qo = reinterpret_cast<const uint4*>(sl + kOut * Ring<NT>::PIECE)[v];
      if (TWO) q2 = reinterpret_cast<const uint4*>(sl + kZ2 * Ring<NT>::PIECE)[v];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const uint32_t dw = MASK ? mask_pos2(w32(qd, p), w32(qo, p)) : w32(qd, p);
        const float2 d = up2(dw);
        const float2 xh = __ffma2_rn(up2(w32(qz, p)), rs[p], nm[p]);
        sg[p] = __ffma2_rn(d, xh, sg[p]);
        sb[p] = __fadd2_rn(sb[p], d);
        if (TWO) sg2[p] = __ffma2_rn(d, __ffma2_rn(up2(w32(q2, p)), rs2[p], nm2[p]), sg2[p]);
      }
    }
    if constexpr (!RESIDENT) rg.release(i);
  }
  BN_TL(2)
  float pr = 0.f, pg = 0.f, pm = 0.f, pr2 = 0.f, pg2 = 0.f, pm2 = 0.f;
  if (t < C) {
    pr = a.rstd[t];
    pg = a.g[t];
    pm = a.mean[t];
    if (TWO) {
      pr2 = a.rstd2[t];
      pg2 = a.g2[t];
      pm2 = a.mean2[t];
    }
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const float a0 = lanes_sum(sg[p].x, V), a1 = lanes_sum(sg[p].y, V);
    const float b0 = lanes_sum(sb[p].x, V), b1 = lanes_sum(sb[p].y, V);
    float c0 = 0.f, c1 = 0.f;
    if (TWO) { c0 = lanes_sum(sg2[p].x, V); c1 = lanes_sum(sg2[p].y, V); }
    if (lane < V) {
      wred[warp * kMaxC + vc * 8 + 2 * p] = make_float4(a0, b0, c0, 0.f);
      wred[warp * kMaxC + vc * 8 + 2 * p + 1] = make_float4(a1, b1, c1, 0.f);
    }
  }
  __syncthreads();
  if (t < C) {
    float4 sacc = wred[t];
    for (int k = 1; k < kWarps; ++k) {
      const float4 q = wred[k * kMaxC + t];
      sacc.x += q.x; sacc.y += q.y; sacc.z += q.z;
    }
    cpart[t] = sacc;
  }
  BN_TL(3)
  float4 sacc;
  if constexpr (SPLIT == 1) {
    split_partial_out(cpart, C, a.gpart);
    cluster_arrive();
    cluster_wait();
    return;
  } else if constexpr (SPLIT == 2) {
    sacc = split_partial_in(C, a.gpart, a.ncl);
  } else {
    sacc = merge_partials<GRID>(cpart, wred, C, a.gpart, a.gbar, a.err);
  }
  if (t < C) {
    // dz = k1·(dy − db/P − x̂·dg/P) = A·dy + B·z + D
    const float k1 = pg * pr;
    const float Bc = -k1 * pr * sacc.x * a.invP;
    coef[t] = k1;
    coef[kMaxC + t] = Bc;
    coef[2 * kMaxC + t] = -k1 * sacc.y * a.invP - Bc * pm;
    if (TWO) {
      const float j1 = pg2 * pr2;
      const float B2 = -j1 * pr2 * sacc.z * a.invP;
      coef[3 * kMaxC + t] = j1;
      coef[4 * kMaxC + t] = B2;
      coef[5 * kMaxC + t] = -j1 * sacc.y * a.invP - B2 * pm2;
    }
    if (rank == 0) {
      a.dg[t] = sacc.x;
      a.db[t] = sacc.y;
      if (TWO) {
        a.dg2[t] = sacc.z;
        a.db2[t] = sacc.y;
      }
    }
  }
  if constexpr (!GRID && !SPLIT) cluster_arrive();
  __syncthreads();
  BN_TL(4)

  float2 A[4], Bv[4], D[4], A2[4], B2[4], D2[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int c = vc * 8 + 2 * p;
    A[p] = make_float2(coef[c], coef[c + 1]);
    Bv[p] = make_float2(coef[kMaxC + c], coef[kMaxC + c + 1]);
    D[p] = make_float2(coef[2 * kMaxC + c], coef[2 * kMaxC + c + 1]);
    A2[p] = TWO ? make_float2(coef[3 * kMaxC + c], coef[3 * kMaxC + c + 1]) : A[p];
    B2[p] = TWO ? make_float2(coef[4 * kMaxC + c], coef[4 * kMaxC + c + 1]) : Bv[p];
    D2[p] = TWO ? make_float2(coef[5 * kMaxC + c], coef[5 * kMaxC + c + 1]) : D[p];
  }
  uint4* dz4 = reinterpret_cast<uint4*>(a.dz + o);
  uint4* dz24 = TWO ? reinterpret_cast<uint4*>(a.dz2 + o) : nullptr;
  uint4* dy4 = a.dy_store ? reinterpret_cast<uint4*>(a.dy_store + o) : nullptr;
  auto apply = [&](const uint8_t* sl, int nv, long v0) {
    for (int v = t; v < nv; v += kThreads) {
      const uint4 qd = reinterpret_cast<const uint4*>(sl)[v];
      const uint4 qz = reinterpret_cast<const uint4*>(sl + kZ * Ring<NT>::PIECE)[v];
      uint4 qo, q2;
      if (MASK) qo = reinterpret_cast<const uint4*>(sl + kOut * Ring<NT>::PIECE)[v];
      if (TWO) q2 = reinterpret_cast<const uint4*>(sl + kZ2 * Ring<NT>::PIECE)[v];
      uint32_t wd[4], w1[4], w2[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        wd[p] = MASK ? mask_pos2(w32(qd, p), w32(qo, p)) : w32(qd, p);
        const float2 d = up2(wd[p]);
        w1[p] = dn2(__ffma2_rn(A[p], d, __ffma2_rn(Bv[p], up2(w32(qz, p)), D[p])));
        if (TWO) w2[p] = dn2(__ffma2_rn(A2[p], d, __ffma2_rn(B2[p], up2(w32(q2, p)), D2[p])));
      }
      dz4[v0 + v] = make_uint4(w1[0], w1[1], w1[2], w1[3]);
      if (TWO) dz24[v0 + v] = make_uint4(w2[0], w2[1], w2[2], w2[3]);
      if (MASK && dy4) dy4[v0 + v] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    }
  };
  if constexpr (RESIDENT) {
    for (long i = 0; i < rg.nch; ++i) apply(rg.slot(i), rg.nvec(i), i * (Ring<NT>::PIECE / 16));
  } else {
    Ring<NT> r3 = rg;
    r3.init(smem, bars + 2 * kMaxSlots, bytes);
    r3.start();
    for (long i = 0; i < r3.nch; ++i) {
      apply(r3.wait(i), r3.nvec(i), i * (Ring<NT>::PIECE / 16));
      r3.release(i);
    }
  }
  BN_TL(5)
  if constexpr (!GRID && !SPLIT) cluster_wait();
  BN_TL(6)
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
static unsigned long long* bn_tl() {
  static const int on = getenv("PPLL_BN_TIMELINE") ? 1 : 0;
  return on ? tc::timeline_buffer() : nullptr;
}

// largest usable cluster size (16 needs the non-portable attribute and a GPC
// with 16 free SMs; 8 is portable), queried once per kernel
template <typename K>
static int cluster_size_for(K kern) {
  static const int env = getenv("PPLL_BN_CS") ? atoi(getenv("PPLL_BN_CS")) : 0;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem) != cudaSuccess ||
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  for (int cs : {16, 8, 4}) {
    if (env && cs != env) continue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0) return cs;
    cudaGetLastError();
  }
  return 0;
}

// grid form: every CTA co-resident (cooperative launch), one CTA per SM
template <typename K, typename A>
static int launch_grid(K kern, const A& args, cudaStream_t s) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  static const void* keys[32];
  static int vals[32];
  static int n = 0;
  int grid = -1;
  for (int i = 0; i < n; ++i)
    if (keys[i] == (const void*)kern) grid = vals[i];
  if (grid < 0) {
    int occ = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, kSmem) != cudaSuccess) {
      cudaGetLastError();
      occ = 0;
    }
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = occ > 0 ? sms : 0;   // one CTA per SM (the ring takes ~200 KB)
    if (n < 32) { keys[n] = (const void*)kern; vals[n++] = grid; }
  }
  if (grid <= 0) return PPLL_ERR_UNSUPPORTED;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  PPLL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, args));
  note_launch();
  return PPLL_OK;
}

template <typename K, typename A>
static int launch_cluster(K kern, int cs, const A& args, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  PPLL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, args));
  note_launch();
  return PPLL_OK;
}

// the fused path covers bf16 NHWC with C % 8 == 0, C <= 128, 512 % (C/8) == 0
// and 16-B aligned tensors.  One cluster streams at ~50 GB/s per SM (~0.8
// TB/s for 16 SMs) against the unfused kernels' ~4 µs per dependent launch,
// so it is used where it is measured faster (tools/ab_bn.sh): forward up to
// PPLL_BN_FWD_MAX_MB (default 2.5) MB per tensor, backward up to
// PPLL_BN_BWD_MAX_MB (default 1.2).
static int fused_mode(long P, int C, bool bwd, bool grid_ok) {
  static const int off = getenv("PPLL_BN_FUSED") ? !atoi(getenv("PPLL_BN_FUSED")) : 0;
  static const double fwd_mb = getenv("PPLL_BN_FWD_MAX_MB") ? atof(getenv("PPLL_BN_FWD_MAX_MB")) : 2.5;
  static const double bwd_mb = getenv("PPLL_BN_BWD_MAX_MB") ? atof(getenv("PPLL_BN_BWD_MAX_MB")) : 1.2;
  static const double grid_mb = getenv("PPLL_BN_GRID_MAX_MB") ? atof(getenv("PPLL_BN_GRID_MAX_MB")) : 64.0;
  if (off || C % 8 || C > kMaxC || kThreads % (C / 8) || P < 1 || P > (1L << 30) / C) return 0;
  // a stage that owns its GPU: the full-GPU grid form beats the 16-SM cluster
  // form above ~1 MB (ResNet-32 stage steps 472 -> 462 / 392 -> 376 µs with the
  // forward threshold at 1.0 MB, tools/prof_gaps.py; 0.5 MB and below slower)
  static const double excl_mb = getenv("PPLL_BN_EXCL_MAX_MB") ? atof(getenv("PPLL_BN_EXCL_MAX_MB")) : 1.0;
  const double mb = (double)P * C * 2 / 1048576.0;
  // (explicit PPLL_BN_FWD_MAX_MB / PPLL_BN_BWD_MAX_MB keep the old thresholds)
  static const bool thr_env = getenv("PPLL_BN_FWD_MAX_MB") || getenv("PPLL_BN_BWD_MAX_MB");
  if (!thr_env && g_gpu_excl && grid_ok && mb > excl_mb && mb <= grid_mb) return 2;
  // split form off by default: its 144 one-per-SM CTAs (~200 KB smem) crowd out the other
  // stage streams — ResNet-32 pipeline 132.8k -> 111.3k img/s (PPLL_BN_SPLIT=1 enables)
  static const int split_on = getenv("PPLL_BN_SPLIT") ? atoi(getenv("PPLL_BN_SPLIT")) : 0;
  if (mb <= (bwd ? bwd_mb : fwd_mb)) return 1;
  if (!grid_ok || mb > grid_mb) return 0;
  return g_gpu_excl ? 2 : (split_on ? 3 : 0);
}

// cluster size + launch of one kernel instantiation; `resident` picks the
// form that keeps the slice in shared memory (decided from the slice size)
// (cached per kernel: the smem / cluster attributes are per function)
template <typename K>
static int cluster_size_cached(K kern) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  static const void* keys[32];
  static int vals[32];
  static int n = 0;
  for (int i = 0; i < n; ++i)
    if (keys[i] == (const void*)kern) return vals[i];
  const int cs = cluster_size_for(kern);
  if (n < 32) { keys[n] = (const void*)kern; vals[n++] = cs; }
  return cs;
}
template <int NT, typename K, typename A>
static int run_fused(K kern_stream, K kern_resident, long P, int C, const A& args, cudaStream_t s) {
  const int cs = cluster_size_cached(kern_stream);
  const int cs_r = cluster_size_cached(kern_resident);
  if (!cs || !cs_r) return PPLL_ERR_UNSUPPORTED;
  const long slice = (P + cs_r - 1) / cs_r * C * 2;
  const bool res = (slice + Ring<NT>::PIECE - 1) / Ring<NT>::PIECE <= Ring<NT>::NS;
  return res ? launch_cluster(kern_resident, cs_r, args, s) : launch_cluster(kern_stream, cs, args, s);
}
// split form: launch A = 8-CTA clusters over the grid (statistics, one partial
// per cluster), launch B = a plain grid that merges them and applies
template <typename K, typename A>
static int run_split(K kern_a, K kern_b, A args, cudaStream_t s) {
  constexpr int kCl = 8, kNcl = 18;   // 144 CTAs: one per SM, whole clusters
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  static const void* keys[32];
  static int n = 0;
  bool seen = false;
  for (int i = 0; i < n; ++i) seen |= keys[i] == (const void*)kern_a;
  if (!seen) {
    if (cudaFuncSetAttribute(kern_a, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem) != cudaSuccess ||
        cudaFuncSetAttribute(kern_b, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem) != cudaSuccess) {
      cudaGetLastError();
      return PPLL_ERR_UNSUPPORTED;
    }
    if (n < 32) keys[n++] = (const void*)kern_a;
  }
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kCl * kNcl);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = g_pdl;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    PPLL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern_a, args));
    note_launch();
  }
  args.ncl = kNcl;
  launch_k(kern_b, kCl * kNcl, kThreads, kSmem, s, args);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

template <int NT, typename K, typename A>
static int run_grid(K kern_stream, K kern_resident, long P, int C, const A& args, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long slice = (P + sms - 1) / sms * C * 2;
  const bool res = (slice + Ring<NT>::PIECE - 1) / Ring<NT>::PIECE <= Ring<NT>::NS;
  return launch_grid(res ? kern_resident : kern_stream, args, s);
}

}  // namespace bnc

int launch_bn_fwd_fused(int P, int C, const __nv_bfloat16* z, const float* g, const float* b,
                        float* mean, float* rstd, const __nv_bfloat16* z2, const float* g2,
                        const float* b2, float* mean2, float* rstd2, const __nv_bfloat16* res,
                        int relu, __nv_bfloat16* y, cudaStream_t s, const BnGrid* grid) {
  using namespace bnc;
  const int mode = fused_mode(P, C, false, grid && grid->part && grid->bar);
  if (!mode || !aligned16(z) || !aligned16(z2) || !aligned16(res) || !aligned16(y))
    return PPLL_ERR_UNSUPPORTED;
  if (z2 && res) return PPLL_ERR_UNSUPPORTED;
  FwdArgs a{P, C, z, g, b, mean, rstd, z2, g2, b2, mean2, rstd2, res, relu, y, bn_tl(),
            mode >= 2 ? (float4*)grid->part : nullptr, mode == 2 ? grid->bar : nullptr,
            mode == 2 ? grid->err : nullptr, 0};
#define PPLL_BN_FWD(NT_, T_, R_)                                                                 \
  return mode == 3 ? run_split(bn_fwd_cluster_kernel<T_, R_, false, false, 1>,                   \
                               bn_fwd_cluster_kernel<T_, R_, false, false, 2>, a, s)             \
       : mode == 2 ? run_grid<NT_>(bn_fwd_cluster_kernel<T_, R_, false, true>,                   \
                                   bn_fwd_cluster_kernel<T_, R_, true, true>, P, C, a, s)        \
                   : run_fused<NT_>(bn_fwd_cluster_kernel<T_, R_, false>,                        \
                                    bn_fwd_cluster_kernel<T_, R_, true>, P, C, a, s);
  if (z2) { PPLL_BN_FWD(2, true, false) }
  if (res) { PPLL_BN_FWD(2, false, true) }
  PPLL_BN_FWD(1, false, false)
#undef PPLL_BN_FWD
}

int launch_bn_bwd_fused(int P, int C, const __nv_bfloat16* dout, const __nv_bfloat16* out,
                        __nv_bfloat16* dy_store, const __nv_bfloat16* z, const float* mean,
                        const float* rstd, const float* g, float* dg, float* db, __nv_bfloat16* dz,
                        const __nv_bfloat16* z2, const float* mean2, const float* rstd2,
                        const float* g2, float* dg2, float* db2, __nv_bfloat16* dz2,
                        cudaStream_t s, const BnGrid* grid) {
  using namespace bnc;
  const int mode = fused_mode(P, C, true, grid && grid->part && grid->bar);
  if (!mode || !aligned16(dout) || !aligned16(out) || !aligned16(dy_store) || !aligned16(z) ||
      !aligned16(dz) || !aligned16(z2) || !aligned16(dz2))
    return PPLL_ERR_UNSUPPORTED;
  BwdArgs a{P, C, 1.f / (float)P, dout, out, out ? dy_store : nullptr, z, mean, rstd, g, dg, db, dz,
            z2, mean2, rstd2, g2, dg2, db2, dz2, bn_tl(),
            mode >= 2 ? (float4*)grid->part : nullptr, mode == 2 ? grid->bar : nullptr,
            mode == 2 ? grid->err : nullptr, 0};
#define PPLL_BN_BWD(NT_, M_, T_)                                                                 \
  return mode == 3 ? run_split(bn_bwd_cluster_kernel<M_, T_, false, false, 1>,                   \
                               bn_bwd_cluster_kernel<M_, T_, false, false, 2>, a, s)             \
       : mode == 2 ? run_grid<NT_>(bn_bwd_cluster_kernel<M_, T_, false, true>,                   \
                                   bn_bwd_cluster_kernel<M_, T_, true, true>, P, C, a, s)        \
                   : run_fused<NT_>(bn_bwd_cluster_kernel<M_, T_, false>,                        \
                                    bn_bwd_cluster_kernel<M_, T_, true>, P, C, a, s);
  if (out && z2) { PPLL_BN_BWD(4, true, true) }
  if (out) { PPLL_BN_BWD(3, true, false) }
  if (z2) { PPLL_BN_BWD(3, false, true) }
  PPLL_BN_BWD(2, false, false)
#undef PPLL_BN_BWD
}

}  // namespace ppll
