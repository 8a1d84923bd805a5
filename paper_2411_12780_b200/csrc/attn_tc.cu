// Multi-head self-attention on tcgen05 tensor cores for short ViT sequences
// (T <= 128 tokens, head_dim 64): one CTA per (image, head).
//
// Forward   S = Q·Kᵀ (TMEM) → row softmax in registers (thread = query row,
//           keys >= T masked) → P (bf16) written to shared memory in the
//           128-B-swizzled K-major layout → O = P·V (TMEM) → bf16 rows out;
//           lse = max + log Σ kept for the backward.
// Backward  S = Q·Kᵀ and dP = dO·Vᵀ (TMEM) → P = exp(scale·S − lse),
//           dS = P ⊙ (dP − rowsum(dO ⊙ O)) → P, dS to shared memory (the
//           same buffer serves as K-major A for dQ = dS·K and, read
//           MN-major, as Pᵀ / dSᵀ for dV = Pᵀ·dO and dK = dSᵀ·Q) → three
//           MMAs into TMEM → dQ, dK, dV rows into the fused qkv gradient.
// Q, K, V, dO tiles arrive by TMA (128-B swizzle) straight from the
// [tokens, 3·D] qkv activations; rows past the image (next image / OOB
// zeros) are neutralised by the key mask and by zero P / dS rows.
#include <cuda.h>
#include <stdlib.h>
#include <cudaTypedefs.h>
#include "common.cuh"
#include "kernels.cuh"
#include "vit.cuh"
#include "ptx.cuh"

namespace ppll {
namespace tc { unsigned long long* timeline_buffer(); }
namespace atc {

constexpr int kDh = 64;

using namespace ptx;
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return umma_desc_sw128(saddr, lbo, sbo);
}
__device__ __forceinline__ uint32_t idesc(int M, int N, bool a_mn, bool b_mn) {
  return umma_idesc_bf16(M, N, a_mn, b_mn);
}
__device__ __forceinline__ void ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  tmem_ld16(taddr, r);
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// K-major operand from a [128 rows][128 keys] bf16 buffer stored as two 64-key
// swizzled atoms (16 KB each): K step j covers keys 16j..16j+15
__device__ __forceinline__ uint64_t kmaj_keys(uint32_t base, int j) {
  return desc(base + (uint32_t)((j >> 2) * 16384 + (j & 3) * 32), 16, 1024);
}
// the same buffer read MN-major (rows = K dim, 64-element MN chunks 16 KB apart)
__device__ __forceinline__ uint64_t mnmaj_rows(uint32_t base, int j) {
  return desc(base + (uint32_t)(j * 2048), 16384, 1024);
}
// K-major tile loaded by TMA: rows of 128 B (64 elements), K step j (16 elements)
__device__ __forceinline__ uint64_t kmaj_tile(uint32_t base, int j) {
  return desc(base + (uint32_t)(j * 32), 16, 1024);
}
// MN-major tile loaded by TMA: rows = K dim, one 64-element MN chunk
__device__ __forceinline__ uint64_t mnmaj_tile(uint32_t base, int j) {
  return desc(base + (uint32_t)(j * 2048), 8192, 1024);
}

// write keys [16c, 16c+16) of row r into the two-atom swizzled buffer
__device__ __forceinline__ void store_chunk16(uint8_t* buf, int r, int c16, const float* v) {
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    uint4 q;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[8 * hh + 2 * e], v[8 * hh + 2 * e + 1]);
    const int c = 2 * c16 + hh;            // 8-key chunk index 0..15
    const int atom = c >> 3, cc = c & 7;
    *reinterpret_cast<uint4*>(buf + atom * 16384 + r * 128 + ((cc ^ (r & 7)) << 4)) = q;
  }
}

// write keys [8c, 8c+8) of row r (one 16-B chunk) into the two-atom buffer
__device__ __forceinline__ void store_chunk8(uint8_t* buf, int r, int c, const float* v) {
  uint4 q;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
  for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
  const int atom = c >> 3, cc = c & 7;
  *reinterpret_cast<uint4*>(buf + atom * 16384 + r * 128 + ((cc ^ (r & 7)) << 4)) = q;
}

struct Maps {
  CUtensorMap qkv128;   // box {64, 128} over [tokens, 3D]
  CUtensorMap qkvK;     // box {64, NK}
  CUtensorMap do128;    // box {64, 128} over [tokens, D]
};

// ------------------------------------------------------------------ forward
__global__ void __launch_bounds__(128, 4)
attn_tc_fwd_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                   int Tn, int H, int NK, __nv_bfloat16* __restrict__ o, float* __restrict__ lse,
                   float scale) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base0 = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + ((1024 - (base0 & 1023)) & 1023);
  // ~53 KB and 128 TMEM columns so four CTAs share an SM: P's first 64-key
  // atom overwrites Q (dead once S = Q·Kᵀ has retired), K and V hold only
  // their NK rows, and O = P·V reuses the S columns after they are read.
  const int kbytes = (NK * 128 + 1023) & ~1023;
  // NK <= 64 (e.g. ViT-B/16 at 96x96, T = 37): P is one 64-key atom (it
  // overwrites Q exactly) and S / O fit 64 TMEM columns, so ~30 KB of smem
  // and 64 columns per CTA: more CTAs per SM than the 128-key layout
  const bool small = NK <= 64;
  const uint32_t tcols = small ? 64u : 128u;
  uint8_t* sQ = sm;                 // 16 KB
  uint8_t* sP = sm;                 // [Q | keys 64..127 atom]: 16 KB or 32 KB
  uint8_t* sK = sm + (small ? 16384 : 32768);   // NK*128 B (<= 16 KB)
  uint8_t* sV = sK + kbytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + kbytes);   // [0]=tma [1]=mma
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int b = blockIdx.x / H, h = blockIdx.x % H;
  const int D = H * kDh;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
        smem_u32(tslot)), "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = *tslot;
  // prologue (barriers, TMEM, tensor-map prefetch) overlaps the predecessor's tail
  pdl_entry();
  const int row0 = b * Tn;
  if (tid == 0) {
    mbar_expect_tx(&bar[0], 16384 + 2 * NK * 128);
    tma_load_2d(&mq, &bar[0], sQ, h * kDh, row0);
    tma_load_2d(&mk, &bar[0], sK, D + h * kDh, row0);
    tma_load_2d(&mk, &bar[0], sV, 2 * D + h * kDh, row0);
    mbar_wait(&bar[0], 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t id = idesc(128, NK, false, false);
    const uint32_t aq = smem_u32(sQ), ak = smem_u32(sK);
#pragma unroll
    for (int j = 0; j < kDh / 16; ++j) mma_bf16(tm, kmaj_tile(aq, j), kmaj_tile(ak, j), id, j > 0);
    mma_commit(&bar[1]);
  }
  mbar_wait(&bar[1], 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // softmax: thread = query row (TMEM lane); keys in chunks of 16.  Warps whose
  // 32 rows are all past Tn skip it (their P rows only feed O rows that are
  // never stored), and P columns >= NK are never read by the P·V MMA.
  const int r = tid;
  const uint32_t lane_base = tm + ((uint32_t)(warp * 32) << 16);
  const bool live = r < Tn;
  float sum = 0.f, mx = -INFINITY;
  if (warp * 32 < Tn) {
    for (int c = 0; c < NK; c += 16) {
      float v[16];
      ld16(lane_base + c, v);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (c + i < Tn) mx = fmaxf(mx, v[i] * scale);
    }
    for (int c = 0; c < NK; c += 16) {
      float v[16];
      ld16(lane_base + c, v);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float e = (live && c + i < Tn) ? __expf(v[i] * scale - mx) : 0.f;
        v[i] = e;
        sum += e;
      }
      store_chunk16(sP, r, c >> 4, v);        // unnormalised; O is divided by the sum
    }
    if (live) lse[(long)blockIdx.x * Tn + r] = mx + logf(sum);
  }
  const float inv = live ? 1.f / sum : 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t id = idesc(128, kDh, false, true);
    const uint32_t ap = smem_u32(sP), av = smem_u32(sV);
    for (int j = 0; j < NK / 16; ++j) mma_bf16(tm, kmaj_keys(ap, j), mnmaj_tile(av, j), id, j > 0);
    mma_commit(&bar[1]);
  }
  mbar_wait(&bar[1], 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float ov[64];
#pragma unroll
  for (int c = 0; c < 64; c += 16) ld16(lane_base + c, ov + c);
  if (live) {
    float v32[32];
    __nv_bfloat16* dst = o + (long)(row0 + r) * D + h * kDh;
#pragma unroll
    for (int i = 0; i < 32; ++i) v32[i] = ov[i] * inv;
    st_row32<__nv_bfloat16>(dst, true, 32, v32);
#pragma unroll
    for (int i = 0; i < 32; ++i) v32[i] = ov[32 + i] * inv;
    st_row32<__nv_bfloat16>(dst + 32, true, 32, v32);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(tcols));
  }
}

// ----------------------------------------------------------------- backward
// Warp transpose-reduce of 32 per-lane values: lane L ends with the warp-wide
// sum of column L (five halving rounds, fixed order).
__device__ __forceinline__ float warp_colsum32(const float (&v)[32], int lane) {
  float a[16];
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float keep = hi ? v[j + 16] : v[j], send = hi ? v[j] : v[j + 16];
      a[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
  }
  float b[8];
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float keep = hi ? a[j + 8] : a[j], send = hi ? a[j] : a[j + 8];
      b[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
  }
  float c[4];
  {
    const bool hi = lane & 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float keep = hi ? b[j + 4] : b[j], send = hi ? b[j] : b[j + 4];
      c[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
  }
  float d[2];
  {
    const bool hi = lane & 2;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float keep = hi ? c[j + 2] : c[j], send = hi ? c[j] : c[j + 2];
      d[j] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
  }
  const bool hi = lane & 1;
  return (hi ? d[1] : d[0]) + __shfl_xor_sync(0xffffffffu, hi ? d[0] : d[1], 1);
}

// 256 threads: two warps per TMEM lane quadrant (warps w and w + 4 own the
// same 32 query / key rows) split the columns of every per-row phase — the
// D_i dot product, the P / dS chunks, the dQ / dK / dV read-out and stores and
// the fused bias sums — so each row's serial work is halved and an SM holds
// 16 warps (two CTAs) to hide the TMA / MMA / TMEM latencies.
//
// Persistent over (image, head) items (grid = resident CTAs): as soon as the
// last MMAs of item i (dV, dK, dQ) retire, every input buffer is dead and the
// TMA loads of item i+1 are issued, so they land while item i's epilogue
// (TMEM read-out, dQKV stores, bias sums) runs; TMEM, barriers and tensor-map
// prefetches are set up once per CTA instead of once per item.
constexpr int kBwdThreads = 256;
__global__ void __launch_bounds__(kBwdThreads, 2)
attn_tc_bwd_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                   const __grid_constant__ CUtensorMap mdo, const __grid_constant__ CUtensorMap mo,
                   int Tn, int H, int NK, int items,
                   const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                   const float* __restrict__ lse, __nv_bfloat16* __restrict__ dqkv, float scale,
                   float* __restrict__ bias_part, unsigned long long* __restrict__ tl) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base0 = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + ((1024 - (base0 & 1023)) & 1023);
  // timeline probe (PPLL_ATTN_TIMELINE): per CTA and item (first 4), %globaltimer
  // at: item start, inputs landed, S/dP retired, P/dS stored, dV/dK/dQ retired, done
#define ATL(k) \
  if (tl && tid == 0 && it < 4) tl[((long)blockIdx.x * 4 + it) * 8 + (k)] = gtimer();
  // ~109 KB so two CTAs share an SM: K holds only its NK rows, and V (dead
  // once dP = dO·Vᵀ has retired) lives in dS's second 64-key atom, which is
  // written only after that MMA completes.
  const int kbytes = (NK * 128 + 1023) & ~1023;
  uint8_t* sQ = sm;                 // 16 KB (128 q rows)
  uint8_t* sK = sQ + 16384;         // NK rows
  uint8_t* sdO = sK + kbytes;       // 16 KB
  uint8_t* sP = sdO + 16384;        // 32 KB
  uint8_t* sdS = sP + 32768;        // 32 KB
  uint8_t* sV = sdS + 16384;        // NK rows, aliases dS keys 64..127
  uint64_t* bar = reinterpret_cast<uint64_t*>(sdS + 32768);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  float* scr = reinterpret_cast<float*>(sdS + 32768 + 64);   // [2][128] D_i halves
  float* red = scr + 256;                                     // [3][8 warps][32] bias-sum scratch
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int half = warp >> 2;
  const int D = H * kDh;
  const int NQ = NK;   // query rows that matter: Tn rounded up to the MMA K step (16)
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mq)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mk)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mdo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mo)) : "memory");
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = *tslot;
  // prologue (barriers, TMEM, tensor-map prefetch) overlaps the predecessor's tail
  pdl_entry();
  // TMEM columns: S [0,128), dP [128,256); later dV [0,64), dK [64,128), dQ [128,192)
  // O arrives by TMA too, into the P buffer (P is written only after the
  // D_i pass below has read O and every thread has passed a barrier)
  uint8_t* sO = sP;
  auto load_item = [&](int w) {    // thread 0: the five input tiles of item w
    const int row = (w / H) * Tn, hh = w % H;
    mbar_expect_tx(&bar[0], 3 * 16384 + 2 * NK * 128);
    tma_load_2d(&mq, &bar[0], sQ, hh * kDh, row);
    tma_load_2d(&mk, &bar[0], sK, D + hh * kDh, row);
    tma_load_2d(&mk, &bar[0], sV, 2 * D + hh * kDh, row);
    tma_load_2d(&mdo, &bar[0], sdO, hh * kDh, row);
    tma_load_2d(&mo, &bar[0], sO, hh * kDh, row);
  };
  if (tid == 0 && (int)blockIdx.x < items) load_item(blockIdx.x);
  const int r = (warp & 3) * 32 + lane;
  const bool live = r < Tn;
  const uint32_t lane_base = tm + ((uint32_t)((warp & 3) * 32) << 16);
  const long ld = 3L * D;
  int it = 0;
  for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
    const int b = w / H, h = w % H;
    const int row0 = b * Tn;
    ATL(0)
    if (tid == 0) {
      mbar_wait(&bar[0], it & 1);
      ATL(1)
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t id = idesc(128, NK, false, false);
      const uint32_t aq = smem_u32(sQ), ak = smem_u32(sK), av = smem_u32(sV), ad = smem_u32(sdO);
#pragma unroll
      for (int j = 0; j < kDh / 16; ++j) mma_bf16(tm, kmaj_tile(aq, j), kmaj_tile(ak, j), id, j > 0);
#pragma unroll
      for (int j = 0; j < kDh / 16; ++j) mma_bf16(tm + 128, kmaj_tile(ad, j), kmaj_tile(av, j), id, j > 0);
      mma_commit(&bar[1]);
    }
    // D_i = rowsum(dO ⊙ O) from the swizzled smem tiles while the MMAs run;
    // each half of the CTA sums 32 of the 64 columns (four 16-B chunks), the
    // halves are added in fixed order
    const float lr = live ? lse[(long)w * Tn + r] : 0.f;
    mbar_wait(&bar[0], it & 1);
    {
      float part = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int off = r * 128 + (((4 * half + j) ^ (r & 7)) << 4);
        const uint4 qo = *reinterpret_cast<const uint4*>(sO + off);
        const uint4 qd = *reinterpret_cast<const uint4*>(sdO + off);
        const __nv_bfloat162* ho = reinterpret_cast<const __nv_bfloat162*>(&qo);
        const __nv_bfloat162* hd = reinterpret_cast<const __nv_bfloat162*>(&qd);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 a = __bfloat1622float2(ho[e]), g = __bfloat1622float2(hd[e]);
          part = fmaf(a.x, g.x, part);
          part = fmaf(a.y, g.y, part);
        }
      }
      scr[half * 128 + r] = live ? part : 0.f;
    }
    __syncthreads();
    const float Di = scr[r] + scr[128 + r];
    mbar_wait(&bar[1], 0);
    ATL(2)
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // P / dS chunks of 16 keys, interleaved between the halves; two chunks'
    // TMEM loads in flight per wait (the loop is TMEM-latency bound)
    // P / dS in 8-key chunks, alternating between the two halves (balanced for
    // any NK), TMEM loads two chunks deep.  Only rows < NQ of P / dS are read
    // by the dV / dK MMAs (K = queries < NQ) and only keys < NK by dQ; rows >=
    // NQ feed only dQ rows that are never stored, key columns >= NK only dV /
    // dK rows that are never stored — those regions are left unwritten (rows
    // in [Tn, NQ) are written as 0).
    if ((warp & 3) * 32 < NQ) {
      auto ld8 = [&](int k, uint32_t (&rp)[8], uint32_t (&rd)[8]) {
        tmem_ld8_nw(lane_base + 8 * k, rp);
        tmem_ld8_nw(lane_base + 128 + 8 * k, rd);
      };
      auto pds = [&](int k, const uint32_t (&rp)[8], const uint32_t (&rd)[8]) {
        float p[8], ds[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float pv = (live && 8 * k + i < Tn) ? __expf(__uint_as_float(rp[i]) * scale - lr) : 0.f;
          ds[i] = pv * (__uint_as_float(rd[i]) - Di);
          p[i] = pv;
        }
        store_chunk8(sP, r, k, p);
        store_chunk8(sdS, r, k, ds);
      };
      const int n8 = NK / 8;
      uint32_t ap[8], ad[8], bp[8], bd[8];
      int k = half;
      if (k < n8) ld8(k, ap, ad);
      if (k + 2 < n8) ld8(k + 2, bp, bd);
      tmem_wait_ld();
      for (; k < n8; k += 4) {
        pds(k, ap, ad);
        if (k + 4 < n8) ld8(k + 4, ap, ad);
        if (k + 2 < n8) pds(k + 2, bp, bd);
        if (k + 6 < n8) ld8(k + 6, bp, bd);
        tmem_wait_ld();
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    ATL(3)
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t ap = smem_u32(sP), as = smem_u32(sdS);
      const uint32_t aq = smem_u32(sQ), ak = smem_u32(sK), ad = smem_u32(sdO);
      const uint32_t id_mn = idesc(128, kDh, true, true);
      // dV = Pᵀ·dO  (M = keys, K = queries < NQ: P / dS rows past Tn are 0)
      for (int j = 0; j < NQ / 16; ++j) mma_bf16(tm + 0, mnmaj_rows(ap, j), mnmaj_tile(ad, j), id_mn, j > 0);
      // dK = dSᵀ·Q
      for (int j = 0; j < NQ / 16; ++j) mma_bf16(tm + 64, mnmaj_rows(as, j), mnmaj_tile(aq, j), id_mn, j > 0);
      // dQ = dS·K   (M = queries, K = keys)
      const uint32_t id_k = idesc(128, kDh, false, true);
      for (int j = 0; j < NK / 16; ++j) mma_bf16(tm + 128, kmaj_keys(as, j), mnmaj_tile(ak, j), id_k, j > 0);
      mma_commit(&bar[1]);
      // every input (and P / dS) is dead once these MMAs retire: the next
      // item's tiles stream in under this item's epilogue
      mbar_wait(&bar[1], 1);
      ATL(4)
      const int wn = w + (int)gridDim.x;
      if (wn < items) load_item(wn);
    }
    mbar_wait(&bar[1], 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // lane r holds: dV[key r], dK[key r], dQ[query r]; this half: columns 32·half ..
    // (TMEM loads two parts deep: the next part's columns are in flight while
    // the current part is scaled and stored)
    {
      auto tld = [&](int part, uint32_t (&ra)[16], uint32_t (&rb)[16]) {
        const uint32_t col = (part == 0 ? 0u : (part == 1 ? 64u : 128u)) + 32u * half;
        tmem_ld16_nw(lane_base + col, ra);
        tmem_ld16_nw(lane_base + col + 16, rb);
      };
      auto emit = [&](int part, const uint32_t (&ra)[16], const uint32_t (&rb)[16]) {
        float v[32];
        const float sc = part == 0 ? 1.f : scale;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v[i] = live ? __uint_as_float(ra[i]) * sc : 0.f;
          v[16 + i] = live ? __uint_as_float(rb[i]) * sc : 0.f;
        }
        const int off = (part == 0 ? 2 * D : (part == 1 ? D : 0)) + h * kDh + 32 * half;
        if (live) st_row32<__nv_bfloat16>(dqkv + (long)(row0 + r) * ld + off, true, 32, v);
        // fused bias gradient: Σ over this image's rows of the 32 columns, as a
        // warp transpose-reduce (lane = column); the four row quadrants are
        // summed in fixed order below
        if (bias_part) red[(part * 8 + warp) * 32 + lane] = warp_colsum32(v, lane);
      };
      if ((warp & 3) * 32 < Tn) {   // quadrants with no live row skip the read-out
        uint32_t a0[16], b0[16], a1[16], b1[16];
        tld(0, a0, b0);
        tld(1, a1, b1);
        tmem_wait_ld();
        emit(0, a0, b0);
        tld(2, a0, b0);
        emit(1, a1, b1);
        tmem_wait_ld();
        emit(2, a0, b0);
      } else if (bias_part) {
#pragma unroll
        for (int part = 0; part < 3; ++part) red[(part * 8 + warp) * 32 + lane] = 0.f;
      }
    }
    if (bias_part) {
      __syncthreads();
      if (warp == 0 || warp == 4) {
        const int w0 = warp;   // quadrants w0 .. w0 + 3 of this half
#pragma unroll
        for (int part = 0; part < 3; ++part) {
          const float* rr = red + part * 256;
          const int off = (part == 0 ? 2 * D : (part == 1 ? D : 0)) + h * kDh + 32 * half;
          bias_part[(long)b * ld + off + lane] =
              ((rr[w0 * 32 + lane] + rr[(w0 + 1) * 32 + lane]) + rr[(w0 + 2) * 32 + lane]) +
              rr[(w0 + 3) * 32 + lane];
        }
      }
    }
    // TMEM read-out done before the next item's MMAs overwrite the columns
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    ATL(5)
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
#undef ATL
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static bool map2d(CUtensorMap* m, const void* ptr, long inner, long outer, long ld, int box_rows) {
  auto enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr int kFwdSmem = 16384 * 2 + 32768 + 1024 + 64;   // upper bound (NK = 128)
inline int fwd_smem(int NK) {
  return (NK <= 64 ? 16384 : 32768) + 2 * ((NK * 128 + 1023) & ~1023) + 1024 + 64;
}
constexpr int kBwdSmem = 16384 * 3 + 32768 * 2 + 1024 + 64 + 4096;   // upper bound (NK = 128)
inline int bwd_smem(int NK) {
  return 16384 * 2 + ((NK * 128 + 1023) & ~1023) + 32768 * 2 + 1024 + 64 + 4096;
}

}  // namespace atc

int g_attn_engine = 0;

bool attn_tc_supported(int Tn, int dh) { return dh == 64 && Tn >= 1 && Tn <= 128; }

int launch_attn_tc_fwd(int B, int Tn, int H, const __nv_bfloat16* qkv, __nv_bfloat16* o,
                       float* lse, cudaStream_t s) {
  using namespace atc;
  const int D = H * kDh, NK = (Tn + 15) / 16 * 16;
  CUtensorMap mq, mk;
  if (!map2d(&mq, qkv, 3L * D, (long)B * Tn, 3L * D, 128) ||
      !map2d(&mk, qkv, 3L * D, (long)B * Tn, 3L * D, NK)) {
    set_error("attention: tensor map encode failed");
    return PPLL_ERR_CUDA;
  }
  static bool set = false;
  if (!set) {
    PPLL_CUDA_CHECK(cudaFuncSetAttribute(attn_tc_fwd_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem));
    set = true;
  }
  launch_k(attn_tc_fwd_kernel, B * H, 128, fwd_smem(NK), s, mq, mk, Tn, H, NK, o, lse,
                                                  1.0f / sqrtf((float)kDh));
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

int launch_attn_tc_bwd(int B, int Tn, int H, const __nv_bfloat16* qkv, const __nv_bfloat16* o,
                       const __nv_bfloat16* dout, const float* lse, __nv_bfloat16* dqkv,
                       cudaStream_t s, float* bias_part) {
  using namespace atc;
  const int D = H * kDh, NK = (Tn + 15) / 16 * 16;
  CUtensorMap mq, mk, md, mo;
  if (!map2d(&mq, qkv, 3L * D, (long)B * Tn, 3L * D, 128) ||
      !map2d(&mk, qkv, 3L * D, (long)B * Tn, 3L * D, NK) ||
      !map2d(&md, dout, (long)D, (long)B * Tn, (long)D, 128) ||
      !map2d(&mo, o, (long)D, (long)B * Tn, (long)D, 128)) {
    set_error("attention: tensor map encode failed");
    return PPLL_ERR_CUDA;
  }
  static bool set = false;
  if (!set) {
    PPLL_CUDA_CHECK(cudaFuncSetAttribute(attn_tc_bwd_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem));
    set = true;
  }
  // persistent: one CTA per resident slot (two per SM), items round-robin
  // resident CTAs per SM from the shared-memory footprint (228 KB per SM, 1 KB
  // reserved per CTA; registers and TMEM (256 columns) allow two)
  int per_sm = 233472 / (bwd_smem(NK) + 1024);
  per_sm = per_sm < 1 ? 1 : (per_sm > 2 ? 2 : per_sm);
  static const int env_grid = getenv("PPLL_ATTN_BWD_GRID") ? atoi(getenv("PPLL_ATTN_BWD_GRID")) : 0;
  const int items = B * H;
  int grid = env_grid > 0 ? env_grid : 148 * per_sm;
  if (grid > items) grid = items;
  static unsigned long long* tl =
      getenv("PPLL_ATTN_TIMELINE") ? tc::timeline_buffer() : nullptr;
  launch_k(attn_tc_bwd_kernel, grid, kBwdThreads, bwd_smem(NK), s, mq, mk, md, mo, Tn, H, NK,
           items, o, dout, lse, dqkv, 1.0f / sqrtf((float)kDh), bias_part, tl);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

}  // namespace ppll

extern "C" void ppll_set_attn_engine(int engine) { ppll::g_attn_engine = engine; }

extern "C" int ppll_attn_fwd_bf16(int B, int T, int H, const void* qkv, void* o, float* lse,
                                  void* stream) {
  if (B < 1 || H < 1 || !ppll::attn_tc_supported(T, 64) || !qkv || !o || !lse) {
    ppll::set_error("ppll_attn_fwd_bf16: unsupported arguments (B=%d T=%d H=%d)", B, T, H);
    return PPLL_ERR_ARG;
  }
  return ppll::launch_attn_tc_fwd(B, T, H, (const __nv_bfloat16*)qkv, (__nv_bfloat16*)o, lse,
                                  (cudaStream_t)stream);
}

extern "C" int ppll_attn_bwd_bf16(int B, int T, int H, const void* qkv, const void* o,
                                  const void* dout, const float* lse, void* dqkv,
                                  float* bias_part, void* stream) {
  if (B < 1 || H < 1 || !ppll::attn_tc_supported(T, 64) || !qkv || !o || !dout || !lse || !dqkv) {
    ppll::set_error("ppll_attn_bwd_bf16: unsupported arguments (B=%d T=%d H=%d)", B, T, H);
    return PPLL_ERR_ARG;
  }
  return ppll::launch_attn_tc_bwd(B, T, H, (const __nv_bfloat16*)qkv, (const __nv_bfloat16*)o,
                                  (const __nv_bfloat16*)dout, lse, (__nv_bfloat16*)dqkv,
                                  (cudaStream_t)stream, bias_part);
}
