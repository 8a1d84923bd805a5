// LayerNorm backward fused into the epilogue of the GEMM that produces its
// input gradient (the ViT layer's FC1 and QKV data gradients, D = 384):
//
//   dxn = dY · Wᵀ                       (tcgen05, fp32 in TMEM, never stored)
//   dx  = rstd·(γ·dxn − mean_row(γ·dxn) − x̂·mean_row(γ·dxn·x̂)) + dres
//   dγ += Σ_rows dxn·x̂,  dβ += Σ_rows dxn,  Σ_rows dx  (next bias gradient)
//
// One CTA per 128-row tile and the WHOLE row (N = 384 = two N = 192 MMAs per
// K step into TMEM columns [0,192) / [192,384)), so the epilogue has complete
// rows: pass 1 reads the accumulator chunk by chunk with x̂ for the two row
// sums (the four warps sharing a TMEM lane quadrant meet at a named barrier),
// pass 2 re-reads it, writes dx and folds the three column sums (warp
// transpose-reduce, fixed quadrant order) into one per-CTA partial that the
// stage's deferred LN reduction sums (vit_kernels.cu).  Replaces the GEMM's
// dxn store + the LN-backward kernel's re-read of it (12.8 MB and one launch
// per LayerNorm) — tensor.py:137-150 matmul adjoint + the LN adjoint of the
// ViT extension (oracle/vit_oracle.py).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>
#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"
#include "vit.cuh"

namespace ppll {
namespace tc { unsigned long long* timeline_buffer(); }
namespace gln {
using namespace ptx;

// A 2-CTA cluster owns a 128-row tile: CTA rank h computes columns
// [192h, 192h + 192) (one N = 192 MMA per K step) and the two CTAs exchange
// their halves of the row sums over DSMEM — 130 CTAs for M = 8320 instead of 65.
constexpr int BM = 128, BK = 64, D = 384, NH = 192;
constexpr int kEpiWarps = 16, kThreads = 64 + 32 * kEpiWarps;
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;            // 16 KB
constexpr int BH_BYTES = NH * BK * 2;           // 24 KB (this CTA's N half)
constexpr int STAGE = A_BYTES + BH_BYTES;       // 40 KB
constexpr int kGamOff = STAGES * STAGE;         // γ of this half [NH] f32
constexpr int kRedOff = kGamOff + NH * 4;       // [2][4][BM] f32 quadrant row partial sums
constexpr int kRowOff = kRedOff + 2 * 4 * BM * 4;     // [2][BM] this CTA's row sums (DSMEM)
constexpr int kCpartOff = kRowOff + 2 * BM * 4;       // [4 quadrants][3][NH] f32
constexpr int kBarOff = kCpartOff + 4 * 3 * NH * 4;
constexpr int kSmem = kBarOff + 256 + 1024;

struct Args {
  int M, K;
  const __nv_bfloat16* x;      // LN input [M, D]
  const float *mean, *rstd;    // [M]
  const float* g;              // γ [D]
  const __nv_bfloat16* dres;   // residual gradient added to dx [M, D] (nullable)
  __nv_bfloat16* dx;           // [M, D] (nullable: parameter gradients only)
  float* part;                 // [gridDim][3][D] per-CTA column partials
  unsigned long long* tl;      // PPLL_GEMM_LN_TIMELINE: per CTA 8 %globaltimer stamps
};
#define GLN_TL(k) \
  if (a.tl && threadIdx.x == 64) a.tl[blockIdx.x * 8 + (k)] = gtimer();

// warp transpose-reduce of 32 per-lane values: lane L ends with Σ_lanes v[L]
__device__ __forceinline__ float colsum32(const float (&v)[32], int lane) {
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

__global__ void __launch_bounds__(kThreads, 1)
gemm_ln_bwd_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_r,
                   const __grid_constant__ Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  float* gam = reinterpret_cast<float*>(smem + kGamOff);
  float* red = reinterpret_cast<float*>(smem + kRedOff);
  float* rows_s = reinterpret_cast<float*>(smem + kRowOff);
  float* cpart = reinterpret_cast<float*>(smem + kCpartOff);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kBarOff);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* xfull = tfull + 1;     // x / dres tiles landed in the (freed) operand ring
  uint64_t* xch = xfull + 1;       // the peer half's row sums are ready (remote arrive)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xch + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int half = (int)cluster_ctarank(), tile = blockIdx.x / 2;
  const int m0 = tile * BM, n0 = half * NH;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(xfull, 1);
    mbar_init(xch, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();   // the peer's barriers are initialised before any remote arrive
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_entry();
  GLN_TL(0)

  const int nkb = a.K / BK;
  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % STAGES;
        mbar_wait(&empty[st], ((kb / STAGES) & 1) ^ 1);
        uint8_t* sa = smem + st * STAGE;
        mbar_expect_tx(&full[st], STAGE);
        tma_load_2d(&map_a, &full[st], sa, kb * BK, m0);
        tma_load_2d(&map_b, &full[st], sa + A_BYTES, kb * BK, n0);
      }
      // every MMA retired => the ring is free: this half's x and dres columns
      // (three 64-column SW128 boxes each, 48 KB per tensor) arrive in it
      mbar_wait(tfull, 0);
      mbar_expect_tx(xfull, (a.dres ? 2 : 1) * BM * NH * 2);
      for (int b = 0; b < NH / 64; ++b) {
        tma_load_2d(&map_x, xfull, smem + b * 16384, n0 + 64 * b, m0);
        if (a.dres) tma_load_2d(&map_r, xfull, smem + 3 * 16384 + b * 16384, n0 + 64 * b, m0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(BM, NH, false, false);
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % STAGES;
        mbar_wait(&full[st], (kb / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sa = smem_u32(smem + st * STAGE);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          mma_bf16(tmem, umma_desc_sw128(sa + k * 32, 16, 1024),
                   umma_desc_sw128(sa + A_BYTES + k * 32, 16, 1024), idesc, (kb | k) ? 1u : 0u);
        mma_commit(&empty[st]);
      }
      mma_commit(tfull);
    }
    __syncwarp();
  } else {
    // ---------------------------- LN-backward epilogue ----------------------------
    const int q = warp & 3, grp = (warp - 2) >> 2;       // lane quadrant, column group
    const int r = q * 32 + lane, row = m0 + r;
    const bool live = row < a.M;
    const float mu = live ? a.mean[row] : 0.f, rs = live ? a.rstd[row] : 0.f;
    for (int c = threadIdx.x - 64; c < NH; c += 32 * kEpiWarps) gam[c] = a.g[n0 + c];
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
    mbar_wait(tfull, 0);
    GLN_TL(1)
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16);
    mbar_wait(xfull, 0);
    GLN_TL(2)
    // 16 columns c.. (of this half) of this thread's row from a swizzled [128][64] box set
    auto ld16s = [&](int tensor, int c, float (&v)[16]) {
      const uint8_t* box = smem + (tensor * 3 + c / 64) * 16384 + r * 128;
      const int j0 = (c % 64) / 8;
      const uint4 q0 = *reinterpret_cast<const uint4*>(box + (((j0) ^ (r & 7)) << 4));
      const uint4 q1 = *reinterpret_cast<const uint4*>(box + (((j0 + 1) ^ (r & 7)) << 4));
      const __nv_bfloat162* h0 = reinterpret_cast<const __nv_bfloat162*>(&q0);
      const __nv_bfloat162* h1 = reinterpret_cast<const __nv_bfloat162*>(&q1);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 x0 = __bfloat1622float2(h0[e]), x1 = __bfloat1622float2(h1[e]);
        v[2 * e] = x0.x; v[2 * e + 1] = x0.y; v[8 + 2 * e] = x1.x; v[8 + 2 * e + 1] = x1.y;
      }
    };
    // pass 1: this warp's three 16-column chunks -> partial row sums
    float s1 = 0.f, s2 = 0.f;
#pragma unroll 1
    for (int j = 0; j < 3; ++j) {
      const int c = 16 * grp + 64 * j;
      uint32_t u[16];
      tmem_ld16(tbase + (uint32_t)c, u);
      float x[16];
      ld16s(0, c, x);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float dxh = __uint_as_float(u[i]) * gam[c + i];
        s1 += dxh;
        s2 += dxh * ((x[i] - mu) * rs);
      }
    }
    red[(0 * 4 + grp) * BM + r] = s1;
    red[(1 * 4 + grp) * BM + r] = s2;
    asm volatile("bar.sync %0, 128;" ::"r"(2 + q) : "memory");   // the quadrant's four warps
    // this half's row sums -> shared memory; the peer reads them over DSMEM
    if (grp == 0) {
      rows_s[r] = ((red[0 * BM + r] + red[1 * BM + r]) + red[2 * BM + r]) + red[3 * BM + r];
      rows_s[BM + r] = ((red[4 * BM + r] + red[5 * BM + r]) + red[6 * BM + r]) + red[7 * BM + r];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
    if (threadIdx.x == 64) mbar_arrive_cluster(mapa_shared(smem_u32(xch), (uint32_t)(half ^ 1)));
    asm volatile(
        "{\n\t.reg .pred p;\n\tXW_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra XW_%=;\n\t}" ::"r"(smem_u32(xch))
        : "memory");
    GLN_TL(3)
    float p1, p2;   // the peer half's sums of this row
    {
      const uint32_t ra = mapa_shared(smem_u32(rows_s + r), (uint32_t)(half ^ 1));
      asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(p1) : "r"(ra) : "memory");
      asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(p2) : "r"(ra + 4 * BM) : "memory");
    }
    const float o1 = rows_s[r], o2 = rows_s[BM + r];
    // fixed order: columns [0,192) first
    const float m1 = (half == 0 ? o1 + p1 : p1 + o1) * (1.f / D);
    const float m2 = (half == 0 ? o2 + p2 : p2 + o2) * (1.f / D);
    // pass 2: dx, and the column sums dγ (dxn·x̂), dβ (dxn), Σ dx
    __nv_bfloat16* orow = a.dx ? a.dx + (long)row * D + n0 : nullptr;
    float* cp = cpart + (long)q * 3 * NH;
#pragma unroll 1
    for (int j = 0; j < 3; ++j) {
      const int c = 16 * grp + 64 * j;
      uint32_t u[16];
      tmem_ld16(tbase + (uint32_t)c, u);
      float x[16], rv[16];
      ld16s(0, c, x);
      if (a.dres) {
        ld16s(1, c, rv);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) rv[i] = 0.f;
      }
      float va[32], vd[32], o[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float dy = live ? __uint_as_float(u[i]) : 0.f;
        const float xh = (x[i] - mu) * rs;
        o[i] = rs * (dy * gam[c + i] - m1 - xh * m2) + rv[i];
        va[i] = dy * xh;          // dγ
        va[16 + i] = dy;          // dβ
        vd[i] = live ? o[i] : 0.f;
        vd[16 + i] = 0.f;
      }
      if (orow && live) {
        uint4 q0, q1;
        __nv_bfloat162* h0 = reinterpret_cast<__nv_bfloat162*>(&q0);
        __nv_bfloat162* h1 = reinterpret_cast<__nv_bfloat162*>(&q1);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          h0[e] = __floats2bfloat162_rn(o[2 * e], o[2 * e + 1]);
          h1[e] = __floats2bfloat162_rn(o[8 + 2 * e], o[8 + 2 * e + 1]);
        }
        reinterpret_cast<uint4*>(orow + c)[0] = q0;
        reinterpret_cast<uint4*>(orow + c)[1] = q1;
      }
      const float sa = colsum32(va, lane), sd = colsum32(vd, lane);
      if (lane < 16) {
        cp[0 * NH + c + lane] = sa;          // dγ chunk
        cp[2 * NH + c + lane] = sd;          // Σ dx chunk
      } else {
        cp[1 * NH + c + lane - 16] = sa;     // dβ chunk
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
    GLN_TL(4)
    // this half's columns of the tile's partial: the four lane quadrants in fixed order
    for (int i = threadIdx.x - 64; i < 3 * NH; i += 32 * kEpiWarps) {
      const int st = i / NH, c = i % NH;
      a.part[((long)tile * 3 + st) * D + n0 + c] =
          ((cpart[i] + cpart[3 * NH + i]) + cpart[6 * NH + i]) + cpart[9 * NH + i];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();   // the peer has read this CTA's row sums
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------
// Forward counterpart: x1 = res + A·W + bias and xn = LN(x1) (the ViT proj
// GEMM followed by LN2), one 2-CTA cluster per 128-row tile, N half per CTA
// (W read MN-major, as the forward GEMMs do).  The residual columns arrive by
// TMA in the freed ring; the epilogue keeps its 48 values per row in registers:
// pass A stores x1 (bf16) and sums its rounded values, the halves exchange the
// row sums (DSMEM) -> mean; pass B sums (x1 − mean)², second exchange -> rstd;
// pass C stores xn.  Same two-pass statistics as ln_fwd_vkernel.
// ---------------------------------------------------------------------------
struct FwdArgs {
  int M, K;
  const float* bias;            // [D]
  const float *g, *b;           // LN γ, β [D]
  __nv_bfloat16 *x1, *xn;       // [M, D]
  float *mean, *rstd;           // [M]
};

__global__ void __launch_bounds__(kThreads, 1)
gemm_ln_fwd_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_r, const __grid_constant__ FwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  float* prm = reinterpret_cast<float*>(smem + kGamOff);       // reuses γ slot: [3][NH] below
  float* red = reinterpret_cast<float*>(smem + kRedOff);       // [4][BM]
  float* rows_s = reinterpret_cast<float*>(smem + kRowOff);    // [2][BM]: mean / var partials
  float* pb = reinterpret_cast<float*>(smem + kCpartOff);      // bias, γ, β of this half [3][NH]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kBarOff);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* xfull = tfull + 1;
  uint64_t* xch = xfull + 1;       // [2] the peer's mean / variance partials are ready
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xch + 2);
  (void)prm;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int half = (int)cluster_ctarank(), tile = blockIdx.x / 2;
  const int m0 = tile * BM, n0 = half * NH;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(xfull, 1);
    mbar_init(&xch[0], 1);
    mbar_init(&xch[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_entry();
  const int nkb = a.K / BK;
  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % STAGES;
        mbar_wait(&empty[st], ((kb / STAGES) & 1) ^ 1);
        uint8_t* sa = smem + st * STAGE;
        mbar_expect_tx(&full[st], STAGE);
        tma_load_2d(&map_a, &full[st], sa, kb * BK, m0);
#pragma unroll
        for (int i = 0; i < NH / 64; ++i)   // W [K, N] MN-major: 64-column boxes 8 KB apart
          tma_load_2d(&map_b, &full[st], sa + A_BYTES + i * 8192, n0 + 64 * i, kb * BK);
      }
      mbar_wait(tfull, 0);
      mbar_expect_tx(xfull, BM * NH * 2);
      for (int b = 0; b < NH / 64; ++b)
        tma_load_2d(&map_r, xfull, smem + b * 16384, n0 + 64 * b, m0);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(BM, NH, false, true);
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % STAGES;
        mbar_wait(&full[st], (kb / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sa = smem_u32(smem + st * STAGE);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          mma_bf16(tmem, umma_desc_sw128(sa + k * 32, 16, 1024),
                   umma_desc_sw128(sa + A_BYTES + k * 2048, 8192, 1024), idesc,
                   (kb | k) ? 1u : 0u);
        mma_commit(&empty[st]);
      }
      mma_commit(tfull);
    }
    __syncwarp();
  } else {
    const int q = warp & 3, grp = (warp - 2) >> 2;
    const int r = q * 32 + lane, row = m0 + r;
    const bool live = row < a.M;
    for (int c = threadIdx.x - 64; c < NH; c += 32 * kEpiWarps) {
      pb[c] = a.bias[n0 + c];
      pb[NH + c] = a.g[n0 + c];
      pb[2 * NH + c] = a.b[n0 + c];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
    mbar_wait(tfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16);
    mbar_wait(xfull, 0);
    auto st16 = [&](__nv_bfloat16* dst, const float (&o)[16]) {
      uint4 q0, q1;
      __nv_bfloat162* h0 = reinterpret_cast<__nv_bfloat162*>(&q0);
      __nv_bfloat162* h1 = reinterpret_cast<__nv_bfloat162*>(&q1);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        h0[e] = __floats2bfloat162_rn(o[2 * e], o[2 * e + 1]);
        h1[e] = __floats2bfloat162_rn(o[8 + 2 * e], o[8 + 2 * e + 1]);
      }
      reinterpret_cast<uint4*>(dst)[0] = q0;
      reinterpret_cast<uint4*>(dst)[1] = q1;
    };
    // row-sum exchange k (0: Σ x1, 1: Σ (x1 − mean)²) with the peer half
    auto exchange = [&](float part, int k) -> float {
      red[grp * BM + r] = part;
      asm volatile("bar.sync %0, 128;" ::"r"(2 + q) : "memory");
      if (grp == 0)
        rows_s[k * BM + r] = ((red[r] + red[BM + r]) + red[2 * BM + r]) + red[3 * BM + r];
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      if (threadIdx.x == 64) mbar_arrive_cluster(mapa_shared(smem_u32(&xch[k]), (uint32_t)(half ^ 1)));
      asm volatile(
          "{\n\t.reg .pred p;\n\tXF_%=:\n\t"
          "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], 0;\n\t"
          "@!p bra XF_%=;\n\t}" ::"r"(smem_u32(&xch[k]))
          : "memory");
      float peer;
      const uint32_t ra = mapa_shared(smem_u32(rows_s + k * BM + r), (uint32_t)(half ^ 1));
      asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(peer) : "r"(ra) : "memory");
      const float own = rows_s[k * BM + r];
      return half == 0 ? own + peer : peer + own;
    };
    float v[3][16];
    float s1 = 0.f;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int c = 16 * grp + 64 * j;
      uint32_t u[16];
      tmem_ld16(tbase + (uint32_t)c, u);
      const uint8_t* box = smem + (c / 64) * 16384 + r * 128;
      const int j0 = (c % 64) / 8;
      const uint4 q0 = *reinterpret_cast<const uint4*>(box + ((j0 ^ (r & 7)) << 4));
      const uint4 q1 = *reinterpret_cast<const uint4*>(box + (((j0 + 1) ^ (r & 7)) << 4));
      const __nv_bfloat162* h0 = reinterpret_cast<const __nv_bfloat162*>(&q0);
      const __nv_bfloat162* h1 = reinterpret_cast<const __nv_bfloat162*>(&q1);
      float o[16];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 r0 = __bfloat1622float2(h0[e]), r1 = __bfloat1622float2(h1[e]);
        o[2 * e] = __uint_as_float(u[2 * e]) + pb[c + 2 * e] + r0.x;
        o[2 * e + 1] = __uint_as_float(u[2 * e + 1]) + pb[c + 2 * e + 1] + r0.y;
        o[8 + 2 * e] = __uint_as_float(u[8 + 2 * e]) + pb[c + 8 + 2 * e] + r1.x;
        o[8 + 2 * e + 1] = __uint_as_float(u[8 + 2 * e + 1]) + pb[c + 8 + 2 * e + 1] + r1.y;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {   // the statistics see the stored (rounded) x1
        v[j][i] = __bfloat162float(__float2bfloat16_rn(o[i]));
        s1 += live ? v[j][i] : 0.f;
      }
      if (live) st16(a.x1 + (long)row * D + n0 + c, o);
    }
    const float mean = exchange(s1, 0) * (1.f / D);
    float s2 = 0.f;
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float d = v[j][i] - mean;
        s2 += live ? d * d : 0.f;
      }
    const float rstd = rsqrtf(exchange(s2, 1) * (1.f / D) + kLnEps);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int c = 16 * grp + 64 * j;
      float o[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i] = (v[j][i] - mean) * rstd * pb[NH + c + i] + pb[2 * NH + c + i];
      if (live) st16(a.xn + (long)row * D + n0 + c, o);
    }
    if (live && half == 0 && grp == 0) {
      a.mean[row] = mean;
      a.rstd[row] = rstd;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
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
// 2-D K-major bf16 operand map: inner extent K (contiguous), `rows` rows of
// pitch ld elements, box {64, box_rows}, 128-B swizzle
static bool kmap(CUtensorMap* m, const void* p, long K, long rows, long ld, int box_rows) {
  auto enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace gln

// dx = LN_backward(dY · Wᵀ) for D = 384 (bf16): dY [M, K] (ld K), W [384, K]
// (the linear weight [in, out] = [D, K], ld K), x / dres / dx [M, 384].
// The per-CTA column partials go to `part` ([ceil(M/128)][3][384]) and are
// recorded in `defer` for the stage's batched reduction into dg, db and
// dxsum (each nullable).  PPLL_ERR_UNSUPPORTED outside the fused shape range
// (the caller keeps GEMM + LN-backward kernel).
int launch_gemm_ln_bwd(int M, int K, const __nv_bfloat16* dY, const __nv_bfloat16* W,
                       const __nv_bfloat16* x, const float* mean, const float* rstd,
                       const float* g, const __nv_bfloat16* dres, __nv_bfloat16* dx, float* part,
                       float* dg, float* db, float* dxsum, LnDefer* defer, cudaStream_t s) {
  using namespace gln;
  static const int on = getenv("PPLL_GEMM_LN") ? atoi(getenv("PPLL_GEMM_LN")) : 1;
  if (!on || M < 1 || K % BK || K < BK || !defer || defer->n >= LnDefer::kMax || !part)
    return PPLL_ERR_UNSUPPORTED;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al(dY) || !al(W) || !al(x) || !al(dres) || !al(dx)) return PPLL_ERR_UNSUPPORTED;
  CUtensorMap ma, mb, mx, mr;
  if (!kmap(&ma, dY, K, M, K, BM) || !kmap(&mb, W, K, D, K, NH) || !kmap(&mx, x, D, M, D, BM))
    return PPLL_ERR_UNSUPPORTED;
  if (dres ? !kmap(&mr, dres, D, M, D, BM) : false) return PPLL_ERR_UNSUPPORTED;
  if (!dres) mr = mx;
  static bool attr = false;
  if (!attr) {
    PPLL_CUDA_CHECK(cudaFuncSetAttribute(gemm_ln_bwd_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr = true;
  }
  const int tiles = (M + BM - 1) / BM, grid = tiles;
  static unsigned long long* tl =
      getenv("PPLL_GEMM_LN_TIMELINE") ? tc::timeline_buffer() : nullptr;
  Args a{M, K, x, mean, rstd, g, dres, dx, part, tl};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * tiles);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  PPLL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, gemm_ln_bwd_kernel, ma, mb, mx, mr, a));
  note_launch();
  LnReduceTask& t = defer->t[defer->n++];
  t = LnReduceTask{part, dg, db, dxsum, grid, D, 3, defer->blocks};
  defer->blocks += (3 * D + 31) / 32;
  return PPLL_OK;
}

}  // namespace ppll

namespace ppll {
// x1 = res + A·W + bias, xn = LN(x1)·γ + β with mean / rstd per row (bf16,
// D = 384): A [M, K] (ld K), W [K, 384] (ld 384), res / x1 / xn [M, 384].
// PPLL_ERR_UNSUPPORTED outside the fused range.
int launch_gemm_ln_fwd(int M, int K, const __nv_bfloat16* A, const __nv_bfloat16* W,
                       const float* bias, const __nv_bfloat16* res, const float* g, const float* b,
                       __nv_bfloat16* x1, __nv_bfloat16* xn, float* mean, float* rstd,
                       cudaStream_t s) {
  using namespace gln;
  // off by default: measured ViT-S pipeline 55.0k -> 54.1k img/s (the 148-CTA proj GEMM + LN
  // kernel beat the 130-CTA fused form with its two DSMEM exchanges); PPLL_GEMM_LN_FWD=1 enables
  static const int on = getenv("PPLL_GEMM_LN_FWD") ? atoi(getenv("PPLL_GEMM_LN_FWD")) : 0;
  if (!on || M < 1 || K % BK || K < BK || !bias || !res) return PPLL_ERR_UNSUPPORTED;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al(A) || !al(W) || !al(res) || !al(x1) || !al(xn)) return PPLL_ERR_UNSUPPORTED;
  CUtensorMap ma, mb, mr;
  if (!kmap(&ma, A, K, M, K, BM) || !kmap(&mb, W, D, K, D, 64) || !kmap(&mr, res, D, M, D, BM))
    return PPLL_ERR_UNSUPPORTED;
  static bool attr = false;
  if (!attr) {
    PPLL_CUDA_CHECK(cudaFuncSetAttribute(gemm_ln_fwd_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr = true;
  }
  const int tiles = (M + BM - 1) / BM;
  FwdArgs a{M, K, bias, g, b, x1, xn, mean, rstd};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * tiles);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  PPLL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, gemm_ln_fwd_kernel, ma, mb, mr, a));
  note_launch();
  return PPLL_OK;
}
}  // namespace ppll
