// Implicit-GEMM 3x3 convolution (stride 1, pad 1, NHWC bf16) on tcgen05
// tensor cores for the ResNet stages — no im2col matrix.
//
//   out[p, co] = Σ_tap Σ_ci  x[p + off(tap), ci] · Wtap[co, ci]
//
// Output tile = 128 consecutive pixels (whole image rows: 128 / W rows, or
// 128 / (H·W) images for 8x8 maps).  For every tap the TMA engine fetches the
// shifted input window as ONE 4-D box {CI, W, rows, images} of the NHWC
// tensor: out-of-range rows / columns (the zero padding) come back as zeros,
// and the box lands in shared memory as a K-major [128 pixels x CI] tile in
// the swizzle mode matching its 32/64/128-B rows.  The nine tap tiles of a
// pixel tile are nine k-blocks of K = CI; the 3x3 weights (≤ 73 KB) are
// staged once per CTA as nine K-major [CO x CI] tiles in the same swizzle.
// Persistent CTAs, warp roles as in gemm_tc.cu (TMA producer, MMA issuer,
// 16 epilogue warps over double-buffered TMEM accumulators, the GEMM
// engine's generic fused epilogue).
//
// The input gradient of the same convolution is this kernel applied to dZ
// with the taps mirrored and the weights transposed (transposed convolution,
// stride 1): `dgrad` selects that weight view, so the dZ·Wᵀ GEMM and the
// col2im gather of the explicit path disappear (its residual-add and ReLU
// mask ride in the epilogue).
#include <cuda.h>
#include <stdlib.h>
#include <cudaTypedefs.h>
#include "common.cuh"
#include "kernels.cuh"
#include "resnet.cuh"
#include "ptx.cuh"

namespace ppll {
namespace cv {

constexpr int kNumSMs = 148;
// epilogue warps: 4 per 16 output channels (one 16-column chunk per TMEM lane
// quadrant and warp), so small-CO convolutions fit several CTAs per SM
template <int CO> constexpr int epi_warps() { return 4 * (CO / 16); }
template <int CO> constexpr int conv_threads() { return 64 + 32 * epi_warps<CO>(); }

using namespace ptx;

// K-major operand descriptor for rows of RB = 32/64/128 bytes (SW32/64/128):
// 8-row swizzle atoms of 8·RB bytes (SBO), K advanced by +32 B per K=16 step
template <int RB>
__device__ __forceinline__ uint64_t kdesc(uint32_t saddr) {
  constexpr uint64_t layout = RB == 128 ? 2 : (RB == 64 ? 4 : 6);
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;                            // LBO (unused for swizzled K-major)
  d |= (uint64_t)(((8 * RB) >> 4) & 0x3FFF) << 32;   // SBO
  d |= (uint64_t)1 << 46;                            // descriptor version (sm_100)
  d |= layout << 61;
  return d;
}
// the byte offset of 16-B chunk j of row r in a K-major swizzled tile (the
// pattern TMA writes and UMMA reads for SW32 / SW64 / SW128)
template <int RB>
__device__ __forceinline__ int swz(int r, int j) {
  const int f = RB == 128 ? (r & 7) : (RB == 64 ? ((r >> 1) & 3) : ((r >> 2) & 1));
  return r * RB + ((j ^ f) * 16);
}
// MN-major swizzled operand descriptor: 8-row K groups of 8·RB bytes (SBO),
// MN atoms of RB bytes' worth of elements `lbo` bytes apart
template <int RB>
__device__ __forceinline__ uint64_t mndesc(uint32_t saddr, uint32_t lbo) {
  constexpr uint64_t layout = RB == 128 ? 2 : (RB == 64 ? 4 : 6);
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(((8 * RB) >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= layout << 61;
  return d;
}

// CLUSTER form (one thread-block cluster of CS CTAs, no workspace): each CTA
// dumps its TMEM partial into its idle operand ring, the cluster synchronises
// once and CTA r sums rows [r·R, r·R + R) of dW over the CS partials through
// distributed shared memory in rank order, writing dW directly.  Uses CS SMs
// for the whole weight gradient — the form for stage streams sharing a GPU
// (one launch, ~1/9 of the SM-time of the wide form + reduction).
// HALO: a pixel tile covers whole rows of ONE image (W >= 16); instead of nine
// shifted 128-pixel windows the producer loads three column-shifted copies
// (dx = -1, 0, +1) of the tile's rows plus one halo row above and below, and
// tap (dy, dx) is copy dx read from row dy + 1 on: a constant row offset of
// W·RB bytes, a whole number of swizzle atoms.  Same MMA sequence (bitwise
// identical result), 2-3x fewer TMA rows and shared-memory bytes per tile, so
// more tiles are in flight.
template <int CI, int CO, bool HALO = false>
struct ConvSmem {
  static constexpr int RB = CI * 2;                  // A / B row bytes (K = CI)
  // one slot: a 128-pixel tap window, or (HALO) one shifted copy of up to
  // 192 pixels ((rows + 2)·W: 6 x 32 or 10 x 16)
  static constexpr int A_BYTES = (HALO ? 192 : 128) * RB;
  static constexpr int W_BYTES = 9 * CO * RB;        // nine [CO x CI] weight tiles
  // tap slots (two pixel tiles below CI = 64) / HALO copy slots (four tiles
  // at CI = 16, three at 32, two at 64)
#ifndef PPLL_CONV_HALO_TILES
#define PPLL_CONV_HALO_TILES 4
#endif
  // HALO: copy slots for PPLL_CONV_HALO_TILES pixel tiles at CI = 16 (fewer at 32 / 64)
  static constexpr int STAGES = HALO ? (CI == 64 ? 4 : (CI == 32 ? 9 : 3 * PPLL_CONV_HALO_TILES)) : (CI == 64 ? 6 : 18);
  static constexpr int STG = epi_warps<CO>() * 1024;
  static constexpr int TOTAL = STAGES * A_BYTES + W_BYTES + STG + 1024 /*align*/ + (2 * STAGES + 8) * 8 /*barriers*/;
  static constexpr uint32_t TMEM_COLS = 2 * CO <= 32 ? 32 : (2 * CO <= 64 ? 64 : 128);
};

// W (global, bf16) is the GEMM weight [k·k·Cin (padded), Cout], row (tap·Cin + ci).
// fwd:   Wtap[co][ci] = W[(tap·CI + ci)·CO + co]             (CI = Cin, CO = Cout)
// dgrad: Wtap[co][ci] = W[((8 − tap)·CO + co)·CI + ci]       (CI = Cout, CO = Cin)
// Forward weights: W rows (tap·CI + ci) hold co contiguous — exactly an
// MN-major B operand (N = co contiguous, K = ci), so the nine [CI x CO] tap
// tiles arrive by TMA (box {CO, CI}, swizzle of their 2·CO-byte rows) and the
// MMA reads them MN-major: no transpose (it was ~1-2 µs of a 64->64 launch).
template <int CI, int CO, bool HALO>
__global__ void __launch_bounds__(conv_threads<CO>(), 1)
conv3x3_tc_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap wmap,
                  const __nv_bfloat16* __restrict__ wg,
                  int dgrad, int wtma, int P, int H, int Wd, int rows, int imgs,
                  Epilogue<__nv_bfloat16> ep) {
  using L = ConvSmem<CI, CO, HALO>;
  constexpr int S = L::STAGES, RB = L::RB;
  constexpr int kEpiWarps = epi_warps<CO>(), kThreads = conv_threads<CO>();
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (base & 1023)) & 1023);
  uint8_t* sw = smem + S * L::A_BYTES;               // weight tiles
  uint8_t* stg_all = sw + L::W_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg_all + L::STG);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint64_t* wbar = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wbar + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles = P / 128;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps);
    }
    mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();   // every thread sees the initialised barriers (wbar is waited on below)
  pdl_entry();   // the weights below are written by the predecessor (optimizer step)
  // stage the nine weight tiles, K-major and swizzled like the TMA'd A tiles,
  // reading the global weight rows as 16-B vectors
  // weights by TMA: issued here, awaited only by the MMA issuer, so the first
  // activation windows stream in alongside them
  if (dgrad && wtma) {   // Wtap[co][ci] = W row (8 - tap)·CO + co: K-major tiles
    if (threadIdx.x == 0) {
      mbar_expect_tx(wbar, 9 * CI * CO * 2);
      for (int tap = 0; tap < 9; ++tap)
        tma_load_2d(&wmap, wbar, sw + tap * CO * RB, 0, (8 - tap) * CO);
    }
  } else if (dgrad) {   // Wtap[co][ci..ci+7] is contiguous in W
    for (int i = threadIdx.x; i < 9 * CO * (CI / 8); i += kThreads) {
      const int j = i % (CI / 8), co = (i / (CI / 8)) % CO, tap = i / (CI / 8) / CO;
      const uint4 q = *reinterpret_cast<const uint4*>(wg + ((long)(8 - tap) * CO + co) * CI + 8 * j);
      *reinterpret_cast<uint4*>(sw + tap * CO * RB + swz<RB>(co, j)) = q;
    }
  } else if (wtma) {   // W row (tap, ci) holds co contiguous: nine MN-major [CI x CO] tiles
    if (threadIdx.x == 0) {
      mbar_expect_tx(wbar, 9 * CI * CO * 2);
      for (int tap = 0; tap < 9; ++tap) tma_load_2d(&wmap, wbar, sw + tap * CO * RB, 0, tap * CI);
    }
  } else {       // (PPLL_CONV_WTMA=0) transpose into K-major [co][ci] through the idle ring
    static_assert(9 * CI * CO * 2 <= S * L::A_BYTES, "weight transpose buffer");
    uint4* tmp4 = reinterpret_cast<uint4*>(smem);
    for (int i = threadIdx.x; i < 9 * CI * CO / 8; i += kThreads)
      tmp4[i] = reinterpret_cast<const uint4*>(wg)[i];
    __syncthreads();
    const __nv_bfloat16* tmp = reinterpret_cast<const __nv_bfloat16*>(smem);
    for (int i = threadIdx.x; i < 9 * CO * (CI / 8); i += kThreads) {
      const int co = i % CO, j = (i / CO) % (CI / 8), tap = i / CO / (CI / 8);
      uint4 q;
      __nv_bfloat16* e = reinterpret_cast<__nv_bfloat16*>(&q);
#pragma unroll
      for (int t = 0; t < 8; ++t) e[t] = tmp[((long)tap * CI + 8 * j + t) * CO + co];
      *reinterpret_cast<uint4*>(sw + tap * CO * RB + swz<RB>(co, j)) = q;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int HWp = H * Wd;

  if (warp == 0) {
    // ------------------------- TMA producer -------------------------
    if (lane == 0) {
      int kb = 0;
      const uint32_t copy_bytes = (uint32_t)((rows + 2) * Wd * RB);
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int p0 = t * 128, n0 = p0 / HWp, h0 = (p0 % HWp) / Wd;
        if constexpr (HALO) {   // three column-shifted copies with a halo row each side
          for (int dx = 0; dx < 3; ++dx, ++kb) {
            const int st = kb % S;
            mbar_wait(&empty[st], ((kb / S) & 1) ^ 1);
            mbar_expect_tx(&full[st], copy_bytes);
            tma_load_4d(&xmap, &full[st], smem + st * L::A_BYTES, 0, dx - 1, h0 - 1, n0);
          }
          continue;
        }
        for (int tap = 0; tap < 9; ++tap, ++kb) {
          const int st = kb % S;
          mbar_wait(&empty[st], ((kb / S) & 1) ^ 1);
          mbar_expect_tx(&full[st], L::A_BYTES);
          tma_load_4d(&xmap, &full[st], smem + st * L::A_BYTES, 0, tap % 3 - 1, h0 + tap / 3 - 1,
                      n0);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------- MMA issuer ---------------------------
    // forward: B (weights) MN-major; input gradient: B K-major
    const bool bmn = !dgrad && wtma;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (bmn ? (1u << 16) : 0u) |
                           ((uint32_t)(CO >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    auto bdesc = [&](uint32_t sb, int k) {
      return bmn ? mndesc<2 * CO>(sb + k * 16 * 2 * CO, CI * 2 * CO) : kdesc<RB>(sb + 32 * k);
    };
    if (lane == 0) {
      if (wtma) mbar_wait(wbar, 0);   // the weight tiles have landed
      int kb = 0, it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if constexpr (HALO) {
          for (int dx = 0; dx < 3; ++dx) mbar_wait(&full[(kb + dx) % S], ((kb + dx) / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          for (int tap = 0; tap < 9; ++tap) {
            const int st = (kb + tap % 3) % S;
            const uint32_t sa = smem_u32(smem + st * L::A_BYTES) + (uint32_t)((tap / 3) * Wd * RB);
            const uint32_t sb = smem_u32(sw + tap * CO * RB);
#pragma unroll
            for (int k = 0; k < CI / 16; ++k)
              mma_bf16(tmem + (uint32_t)(acc * CO), kdesc<RB>(sa + 32 * k), bdesc(sb, k),
                       idesc, (tap | k) ? 1u : 0u);
          }
          for (int dx = 0; dx < 3; ++dx) mma_commit(&empty[(kb + dx) % S]);
          kb += 3;
          mma_commit(&tfull[acc]);
          continue;
        }
        for (int tap = 0; tap < 9; ++tap, ++kb) {
          const int st = kb % S;
          mbar_wait(&full[st], (kb / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(smem + st * L::A_BYTES);
          const uint32_t sb = smem_u32(sw + tap * CO * RB);
#pragma unroll
          for (int k = 0; k < CI / 16; ++k)
            mma_bf16(tmem + (uint32_t)(acc * CO), kdesc<RB>(sa + 32 * k), bdesc(sb, k),
                     idesc, (tap | k) ? 1u : 0u);
          mma_commit(&empty[st]);
        }
        mma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------- epilogue -----------------------------
    const int q = warp & 3, grp = (warp - 2) >> 2;
    uint8_t* stg = stg_all + (warp - 2) * 1024;
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int acc = it & 1, m0 = t * 128;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = m0 + q * 32 + lane;
#pragma unroll 1
      for (int c = 16 * grp; c < CO; c += 64) {
        float ra[16], ka[16];
        if (row < P) ep.load_aux16(row, c, ra, ka);
        uint32_t r[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * CO + c), r);
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
        ep.finish_block16(m0 + q * 32, P, c, v, ra, ka, nullptr, stg, lane);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(L::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// Implicit-GEMM weight gradient of the same 3x3 / stride-1 convolution:
//
//   dW[tap·CI + ci, co] = Σ_p x[p + off(tap), ci] · dZ[p, co]
//
// K = pixels.  Per 128-pixel chunk the producer fetches the nine shifted input
// windows exactly like the forward (one 4-D TMA box per tap, zero padding from
// out-of-range boxes) into nine consecutive [128 px x CI] slots, plus the
// [128 px x CO] dZ tile.  Read MN-major (rows = pixels = K, CI contiguous),
// consecutive tap slots are consecutive MN atoms (descriptor LBO = slot
// stride), so ONE M = 128 MMA covers 128 / CI taps: rows m = tap·CI + ci of
// the accumulator are the rows of dW in the GEMM weight layout.  N = CO (dZ
// tile, MN-major), K step = 16 pixels.  M-tiles past the ninth tap read the
// next slots (other data, never-stored accumulator rows).  Each CTA sums its
// chunks in TMEM and writes one fp32 partial [9·CI, CO]; the fixed-order
// split-K reduction (splitk_reduce) sums the partials — deterministic, no
// im2col matrix (which was P·9·CI bf16: 38 MB for a 32x32x16 layer at B=128).
// ---------------------------------------------------------------------------
// HALO (chunks of whole rows of one image, CI <= 32): the chunk's input is
// three column-shifted copies (dx = -1, 0, +1) of its rows plus a halo row on
// each side, as in the forward; M-tile dx stacks the taps dy = -1, 0, +1 of
// copy dx along M at a stride of one image row (LBO = W·RB, whole swizzle
// atoms), the remaining 128/CI − 3 atoms of the tile read further rows and
// their (discarded) dW rows are never stored.  3·(rows + 2)/rows instead of
// 9 windows of TMA rows per chunk, so twice as many chunks are in flight.
template <int CI, int CO, bool HALO = false>
struct WgSmem {
  static constexpr int RB = CI * 2, RBO = CO * 2;
  static constexpr int SLOT = (HALO ? 192 : 128) * RB;      // a tap window / a shifted copy
  static constexpr int TAPS_PER_M = 128 / CI;               // taps (atoms) per M = 128 tile
  static constexpr int MT = HALO ? 3 : (9 + TAPS_PER_M - 1) / TAPS_PER_M;
  static constexpr int DZ = 128 * RBO;
  static constexpr int BUF = (HALO ? 3 : 9) * SLOT + DZ;    // one chunk
  static constexpr int NB = HALO ? (204800 / BUF < 8 ? 204800 / BUF : 8)
                                : (CI == 16 ? 4 : (CI == 32 ? 2 : 1));
  // the last M-tile reads up to MT·TAPS_PER_M − 9 slots past a buffer's ninth;
  // (HALO) copy dx = +1 of the last buffer read up to TAPS_PER_M − 1 rows (≤ 8 KB
  // at W·RB ≤ 1 KB) plus a window past its start
  static constexpr int PAD = HALO ? 8192 : (MT * TAPS_PER_M - 9) * SLOT;
  static constexpr int TOTAL = NB * BUF + PAD + 1024 + 256;
  static constexpr uint32_t TMEM_COLS = MT * CO <= 32 ? 32 : (MT * CO <= 64 ? 64 : (MT * CO <= 128 ? 128 : (MT * CO <= 256 ? 256 : 512)));
};

template <int CI, int CO, bool CLUSTER = false, bool HALO = false>
__global__ void __launch_bounds__(192, 1)
conv3x3_wgrad_tc_kernel(const __grid_constant__ CUtensorMap xmap,
                        const __grid_constant__ CUtensorMap dzmap, int P, int H, int Wd,
                        float* __restrict__ part) {
  using L = WgSmem<CI, CO, HALO>;
  constexpr int NB = L::NB, RB = L::RB, RBO = L::RBO, MT = L::MT;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (base & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NB * L::BUF + L::PAD);
  uint64_t* empty = full + NB;
  uint64_t* done = empty + NB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int chunks = P / 128;
  // contiguous chunk range of this split (fixed assignment: deterministic)
  const int per = (chunks + gridDim.x - 1) / gridDim.x;
  const int c0 = blockIdx.x * per, c1 = min(chunks, c0 + per);

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&dzmap)) : "memory");
    for (int i = 0; i < NB; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_entry();
  const int HWp = H * Wd;

  if (warp == 0) {
    if (lane == 0) {
      int kb = 0;
      for (int c = c0; c < c1; ++c, ++kb) {
        const int b = kb % NB;
        mbar_wait(&empty[b], ((kb / NB) & 1) ^ 1);
        uint8_t* buf = smem + b * L::BUF;
        const int p0 = c * 128, n0 = p0 / HWp, h0 = (p0 % HWp) / Wd;
        if constexpr (HALO) {
          mbar_expect_tx(&full[b], 3 * (128 + 2 * Wd) * RB + L::DZ);
          for (int dx = 0; dx < 3; ++dx)
            tma_load_4d(&xmap, &full[b], buf + dx * L::SLOT, 0, dx - 1, h0 - 1, n0);
          tma_load_2d(&dzmap, &full[b], buf + 3 * L::SLOT, 0, p0);
          continue;
        }
        mbar_expect_tx(&full[b], 9 * L::SLOT + L::DZ);
        for (int tap = 0; tap < 9; ++tap)
          tma_load_4d(&xmap, &full[b], buf + tap * L::SLOT, 0, tap % 3 - 1, h0 + tap / 3 - 1, n0);
        tma_load_2d(&dzmap, &full[b], buf + 9 * L::SLOT, 0, p0);
      }
    }
  } else if (warp == 1) {
    // M = 128 rows (tap, ci), N = CO, both operands MN-major
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                           ((uint32_t)(CO >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (lane == 0) {
      int kb = 0;
      for (int c = c0; c < c1; ++c, ++kb) {
        const int b = kb % NB;
        mbar_wait(&full[b], (kb / NB) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sbuf = smem_u32(smem + b * L::BUF);
        const uint32_t sdz = sbuf + (HALO ? 3 : 9) * L::SLOT;
        // M-tile stride between taps: a window (SLOT) / an image row (HALO)
        const uint32_t lbo = HALO ? (uint32_t)(Wd * RB) : (uint32_t)L::SLOT;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const uint32_t sa = sbuf + (uint32_t)(mt * (HALO ? 1 : L::TAPS_PER_M) * L::SLOT);
#pragma unroll
          for (int k = 0; k < 8; ++k)   // 16 pixels per MMA = two 8-row groups
            mma_bf16(tmem + (uint32_t)(mt * CO), mndesc<RB>(sa + k * 16 * RB, lbo),
                     mndesc<RBO>(sdz + k * 16 * RBO, 128 * RBO), idesc,
                     (c > c0 || k > 0) ? 1u : 0u);
        }
        mma_commit(&empty[b]);
      }
      mma_commit(done);
    }
    __syncwarp();
  } else {
    // warps 2..5: one TMEM lane quadrant each; row r of M-tile mt is dW row mt·128 + r
    const int q = warp & 3;
    if (c1 > c0) {
      mbar_wait(done, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    // the wide form writes its partial to the workspace; the cluster form to
    // its own (now idle) operand ring, row-major [9·CI][CO]
    float* dst = CLUSTER ? reinterpret_cast<float*>(smem) : part + (long)blockIdx.x * 9 * CI * CO;
#pragma unroll 1
    for (int mt = 0; mt < MT; ++mt) {
      // dW row (tap·CI + ci) of TMEM lane q·32 + lane: HALO tile dx holds tap
      // (dy, dx) = atom dy (< 3), ci at lane % CI
      const int lr = q * 32 + lane;
      const int row = HALO ? ((lr / CI) < 3 ? ((lr / CI) * 3 + mt) * CI + lr % CI : 1 << 20)
                           : mt * 128 + lr;
#pragma unroll 1
      for (int cc = 0; cc < CO; cc += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(mt * CO + cc), r);
        if (row < 9 * CI) {
          float4* o = reinterpret_cast<float4*>(dst + (long)row * CO + cc);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            o[j] = c1 > c0 ? make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                         __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
  }
  if constexpr (CLUSTER) {
    // ---- distributed reduction: CTA `rank` owns rows [rank·R, rank·R + R) ----
    static_assert(9 * CI * CO * 4 <= L::NB * L::BUF + L::PAD, "partial must fit the ring");
    cluster_sync();
    const int CS = (int)cluster_nctarank(), rank = (int)cluster_ctarank();
    const int R = (9 * CI + CS - 1) / CS;
    const int r0 = rank * R, r1 = min(9 * CI, r0 + R);
    constexpr int C4 = CO / 4;
    const uint32_t base_s = smem_u32(smem);
    for (int idx = threadIdx.x; idx < (r1 - r0) * C4; idx += 192) {
      const int row = r0 + idx / C4, c4 = idx % C4;
      const uint32_t a = base_s + (uint32_t)((row * CO + 4 * c4) * 4);
      float4 acc = ld_dsmem_f4(a, 0);
      for (int src = 1; src < CS; ++src) {
        const float4 t = ld_dsmem_f4(a, (uint32_t)src);
        acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
      }
      reinterpret_cast<float4*>(part)[(long)row * C4 + c4] = acc;   // part = dW here
    }
    cluster_sync();   // peers may still read this CTA's partial until here
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(L::TMEM_COLS));
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

template <int CI, int CO, bool HALO>
static int run(const CUtensorMap& xm, const CUtensorMap& wm, const __nv_bfloat16* w, int dgrad,
               int P, int H, int Wd, int rows, int imgs, const Epilogue<__nv_bfloat16>& ep,
               cudaStream_t s) {
  auto kern = conv3x3_tc_kernel<CI, CO, HALO>;
  constexpr int smem = ConvSmem<CI, CO, HALO>::TOTAL;
  static bool attr = false;
  if (!attr) {
    PPLL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const int tiles = P / 128;
  int per_sm = 1;
  PPLL_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, conv_threads<CO>(),
                                                                smem));
  const int grid = tiles < kNumSMs * per_sm ? tiles : kNumSMs * (per_sm > 0 ? per_sm : 1);
  static const int wtma = getenv("PPLL_CONV_WTMA") ? atoi(getenv("PPLL_CONV_WTMA")) : 1;
  launch_k(kern, grid, conv_threads<CO>(), smem, s, xm, wm, w, dgrad, wtma, P, H, Wd, rows, imgs, ep);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

}  // namespace cv

// out = conv3x3(x) (stride 1, pad 1) with CI input / CO output channels, NHWC
// bf16; `dgrad` = the transposed convolution of the forward weights (input
// gradient).  Returns PPLL_ERR_UNSUPPORTED for shapes the kernel does not
// cover (the caller keeps the explicit im2col path).
int launch_conv3x3_tc(int N, int H, int W, int CI, int CO, const __nv_bfloat16* x,
                      const __nv_bfloat16* w, bool dgrad, const Epilogue<__nv_bfloat16>& ep,
                      cudaStream_t s) {
  using namespace cv;
  const long P = (long)N * H * W;
  if (CI % 16 || CO % 16 || CI > 64 || CO > 64 || P % 128) return PPLL_ERR_UNSUPPORTED;
  int rows, imgs;
  if (W > 128 || 128 % W) return PPLL_ERR_UNSUPPORTED;
  if (128 / W <= H) {
    rows = 128 / W;
    imgs = 1;
    if (H % rows) return PPLL_ERR_UNSUPPORTED;
  } else {
    if (128 % (H * W)) return PPLL_ERR_UNSUPPORTED;
    rows = H;
    imgs = 128 / (H * W);
  }
  if (((uintptr_t)x & 15) || ((uintptr_t)w & 15)) return PPLL_ERR_UNSUPPORTED;
  auto enc = encoder();
  if (!enc) return PPLL_ERR_UNSUPPORTED;
  CUtensorMap xm;
  cuuint64_t dims[4] = {(cuuint64_t)CI, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[3] = {(cuuint64_t)CI * 2, (cuuint64_t)W * CI * 2, (cuuint64_t)H * W * CI * 2};
  // whole rows of one image per tile: the halo form (three shifted copies)
  static const int halo_env = getenv("PPLL_CONV_HALO") ? atoi(getenv("PPLL_CONV_HALO")) : 1;
  const bool halo = halo_env && imgs == 1 && (rows + 2) * W <= 192;
  cuuint32_t box[4] = {(cuuint32_t)CI, (cuuint32_t)W, (cuuint32_t)(halo ? rows + 2 : rows),
                       (cuuint32_t)imgs};
  cuuint32_t es[4] = {1, 1, 1, 1};
  const CUtensorMapSwizzle sz = CI == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : (CI == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  if (enc(&xm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<__nv_bfloat16*>(x), dims, strides,
          box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return PPLL_ERR_UNSUPPORTED;
  // forward weights as MN-major B tiles: W viewed as [9·CI rows][CO], box {CO, CI};
  // input gradient: W viewed as [9·CO rows][CI] (CI = the forward's Cout), box
  // {CI, CO}, landing K-major like the activation tiles
  CUtensorMap wm = xm;
  if (dgrad) {
    cuuint64_t dims[2] = {(cuuint64_t)CI, (cuuint64_t)(9 * CO)};
    cuuint64_t strides[1] = {(cuuint64_t)CI * 2};
    cuuint32_t box[2] = {(cuuint32_t)CI, (cuuint32_t)CO};
    cuuint32_t es2[2] = {1, 1};
    const CUtensorMapSwizzle wsz = CI == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                   : (CI == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
    if (enc(&wm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(w), dims, strides,
            box, es2, CU_TENSOR_MAP_INTERLEAVE_NONE, wsz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return PPLL_ERR_UNSUPPORTED;
  } else {
    cuuint64_t dims[2] = {(cuuint64_t)CO, (cuuint64_t)(9 * CI)};
    cuuint64_t strides[1] = {(cuuint64_t)CO * 2};
    cuuint32_t box[2] = {(cuuint32_t)CO, (cuuint32_t)CI};
    cuuint32_t es2[2] = {1, 1};
    const CUtensorMapSwizzle wsz = CO == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                   : (CO == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
    if (enc(&wm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(w), dims, strides,
            box, es2, CU_TENSOR_MAP_INTERLEAVE_NONE, wsz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return PPLL_ERR_UNSUPPORTED;
  }
  Epilogue<__nv_bfloat16> e = ep;
  const int d = dgrad ? 1 : 0, Pi = (int)P;
#define CONV_CASE(A, B)                                                             \
  if (CI == A && CO == B)                                                           \
    return halo ? run<A, B, true>(xm, wm, w, d, Pi, H, W, rows, imgs, e, s)         \
                : run<A, B, false>(xm, wm, w, d, Pi, H, W, rows, imgs, e, s);
  CONV_CASE(16, 16) CONV_CASE(32, 32) CONV_CASE(64, 64)
  CONV_CASE(16, 32) CONV_CASE(32, 16) CONV_CASE(32, 64) CONV_CASE(64, 32)
#undef CONV_CASE
  return PPLL_ERR_UNSUPPORTED;
}

// dW[9·CI, CO] (fp32, the GEMM weight layout) of conv3x3(x) given dZ [P, CO]:
// implicit-GEMM partials (conv3x3_wgrad_tc_kernel) + the fixed-order split-K
// reduction.  ws must hold splits·9·CI·CO floats.  PPLL_ERR_UNSUPPORTED for
// shapes outside the kernel (the caller keeps im2col + GEMM).
int launch_conv3x3_wgrad_tc(int N, int H, int W, int CI, int CO, const __nv_bfloat16* x,
                            const __nv_bfloat16* dz, float* dw, float* ws, size_t ws_elems,
                            cudaStream_t s) {
  using namespace cv;
  static const int off = getenv("PPLL_CONV_WGRAD_IMPLICIT") ? !atoi(getenv("PPLL_CONV_WGRAD_IMPLICIT")) : 0;
  if (off) return PPLL_ERR_UNSUPPORTED;
  const long P = (long)N * H * W;
  if (CI % 16 || CO % 16 || CI > 64 || CO > 64 || P % 128 || !ws) return PPLL_ERR_UNSUPPORTED;
  int rows, imgs;
  if (W > 128 || 128 % W) return PPLL_ERR_UNSUPPORTED;
  if (128 / W <= H) {
    rows = 128 / W;
    imgs = 1;
    if (H % rows) return PPLL_ERR_UNSUPPORTED;
  } else {
    if (128 % (H * W)) return PPLL_ERR_UNSUPPORTED;
    rows = H;
    imgs = 128 / (H * W);
  }
  if (((uintptr_t)x & 15) || ((uintptr_t)dz & 15) || ((uintptr_t)dw & 15)) return PPLL_ERR_UNSUPPORTED;
  auto enc = encoder();
  if (!enc) return PPLL_ERR_UNSUPPORTED;
  // whole rows of one image per chunk: the halo form (PPLL_CONV_WGRAD_HALO=0 never,
  // 1 where it measured faster, 2 always)
  // (read per call: the parity tests switch it)
  const char* halo_s = getenv("PPLL_CONV_WGRAD_HALO");
  const int halo_env = halo_s ? atoi(halo_s) : 1;
  // Measured (tools/ab_wgrad_halo.sh): faster in the wide form (16->16 15.0 -> 13.5 us,
  // 32->32 11.2 -> 10.5 us) and the one-cluster form at CI = 32; the one-cluster
  // 16->16 form is held by its MMA count (24 vs 16 per chunk: 48.8 -> 57 us)
  static const int wcl_env = getenv("PPLL_CONV_WGRAD_CLUSTER") ? atoi(getenv("PPLL_CONV_WGRAD_CLUSTER")) : -1;
  const bool will_cluster = wcl_env >= 0 ? wcl_env != 0 : !g_gpu_excl;
  const bool halo = CI <= 32 && imgs == 1 && (rows + 2) * W <= 192 && W >= 16 &&
                    (halo_env == 2 || (halo_env == 1 && (!will_cluster || CI == 32)));
  CUtensorMap xm, dm;
  {
    cuuint64_t dims[4] = {(cuuint64_t)CI, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)CI * 2, (cuuint64_t)W * CI * 2, (cuuint64_t)H * W * CI * 2};
    cuuint32_t box[4] = {(cuuint32_t)CI, (cuuint32_t)W, (cuuint32_t)(halo ? rows + 2 : rows),
                         (cuuint32_t)imgs};
    cuuint32_t es[4] = {1, 1, 1, 1};
    const CUtensorMapSwizzle sz = CI == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : (CI == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
    if (enc(&xm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<__nv_bfloat16*>(x), dims, strides,
            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return PPLL_ERR_UNSUPPORTED;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)CO, (cuuint64_t)P};
    cuuint64_t strides[1] = {(cuuint64_t)CO * 2};
    cuuint32_t box[2] = {(cuuint32_t)CO, 128};
    cuuint32_t es[2] = {1, 1};
    const CUtensorMapSwizzle sz = CO == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : (CO == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
    if (enc(&dm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(dz), dims, strides,
            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return PPLL_ERR_UNSUPPORTED;
  }
  // splits: at least two chunks per CTA where the CTA double-buffers its
  // chunks (CI < 64), one otherwise; the partials must fit the workspace
  const int chunks = (int)(P / 128);
  static const int minc_env = getenv("PPLL_CONV_WGRAD_MINC") ? atoi(getenv("PPLL_CONV_WGRAD_MINC")) : 0;
  const int minc = minc_env > 0 ? minc_env : (CI == 64 ? 1 : 2);
  int splits = chunks / minc < kNumSMs ? chunks / minc : kNumSMs;
  if (splits < 1) splits = 1;
  while (splits > 1 && (size_t)splits * 9 * CI * CO > ws_elems) --splits;
  if ((size_t)splits * 9 * CI * CO > ws_elems) return PPLL_ERR_UNSUPPORTED;
  const int per = (chunks + splits - 1) / splits;
  splits = (chunks + per - 1) / per;   // every split owns >= 1 chunk
  const int Pi = (int)P;
  // stage streams sharing the GPU (g_gpu_excl == 0): one cluster, in-kernel
  // DSMEM reduction, dW written directly (PPLL_CONV_WGRAD_CLUSTER=0|1 forces)
  const bool cl = will_cluster;
  if (cl) {
#define WGC_CASE(A, B, HL)                                                                   \
    if (CI == A && CO == B && halo == HL) {                                                  \
      auto kern = conv3x3_wgrad_tc_kernel<A, B, true, HL>;                                   \
      constexpr int smem = WgSmem<A, B, HL>::TOTAL;                                          \
      static int cs = -1;                                                                    \
      if (cs < 0) {                                                                          \
        cs = 0;                                                                              \
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == \
                cudaSuccess &&                                                               \
            cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == \
                cudaSuccess) {                                                               \
          for (int c : {16, 8}) {                                                            \
            cudaLaunchConfig_t q = {};                                                       \
            q.gridDim = dim3(c); q.blockDim = dim3(192); q.dynamicSmemBytes = smem;          \
            cudaLaunchAttribute qa[1];                                                       \
            qa[0].id = cudaLaunchAttributeClusterDimension;                                  \
            qa[0].val.clusterDim.x = c; qa[0].val.clusterDim.y = 1; qa[0].val.clusterDim.z = 1; \
            q.attrs = qa; q.numAttrs = 1;                                                    \
            int nc = 0;                                                                      \
            if (cudaOccupancyMaxActiveClusters(&nc, kern, &q) == cudaSuccess && nc > 0) { cs = c; break; } \
            cudaGetLastError();                                                              \
          }                                                                                  \
        } else {                                                                             \
          cudaGetLastError();                                                                \
        }                                                                                    \
      }                                                                                      \
      if (cs > 0 && chunks >= cs) {                                                          \
        cudaLaunchConfig_t cfg = {};                                                         \
        cfg.gridDim = dim3(cs); cfg.blockDim = dim3(192); cfg.dynamicSmemBytes = smem;       \
        cfg.stream = s;                                                                      \
        cudaLaunchAttribute at[2];                                                           \
        at[0].id = cudaLaunchAttributeClusterDimension;                                      \
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; \
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;                       \
        at[1].val.programmaticStreamSerializationAllowed = g_pdl;                            \
        cfg.attrs = at; cfg.numAttrs = 2;                                                    \
        PPLL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, xm, dm, Pi, H, W, dw));               \
        note_launch();                                                                       \
        return PPLL_OK;                                                                      \
      }                                                                                      \
    }
    WGC_CASE(16, 16, true) WGC_CASE(32, 32, true) WGC_CASE(16, 32, true) WGC_CASE(32, 16, true)
    WGC_CASE(32, 64, true)
    WGC_CASE(16, 16, false) WGC_CASE(32, 32, false) WGC_CASE(64, 64, false) WGC_CASE(16, 32, false)
    WGC_CASE(32, 16, false) WGC_CASE(32, 64, false) WGC_CASE(64, 32, false)
#undef WGC_CASE
  }
#define WG_CASE(A, B, HL)                                                                    \
  if (CI == A && CO == B && halo == HL) {                                                    \
    auto kern = conv3x3_wgrad_tc_kernel<A, B, false, HL>;                                    \
    constexpr int smem = WgSmem<A, B, HL>::TOTAL;                                            \
    static bool attr = false;                                                                \
    if (!attr) {                                                                             \
      PPLL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
      attr = true;                                                                           \
    }                                                                                        \
    launch_k(kern, splits, 192, smem, s, xm, dm, Pi, H, W, ws);                              \
    note_launch();                                                                           \
    PPLL_LAUNCH_CHECK();                                                                     \
  } else
  WG_CASE(16, 16, true) WG_CASE(32, 32, true) WG_CASE(16, 32, true) WG_CASE(32, 16, true)
  WG_CASE(32, 64, true)
  WG_CASE(16, 16, false) WG_CASE(32, 32, false) WG_CASE(64, 64, false) WG_CASE(16, 32, false)
  WG_CASE(32, 16, false) WG_CASE(32, 64, false) WG_CASE(64, 32, false) { return PPLL_ERR_UNSUPPORTED; }
#undef WG_CASE
  Epilogue<float> e;
  e.C = dw;
  e.ldc = CO;
  epilogue_finalize(e, CO);
  return launch_splitk_reduce<float>(9 * CI, CO, splits, ws, e, s);
}

}  // namespace ppll

extern "C" int ppll_conv3x3_bf16_ex(int N, int H, int W, int Cin, int Cout, const void* x,
                                    const void* w, void* y, int dgrad, const void* res,
                                    const void* mask, void* stream) {
  using namespace ppll;
  Epilogue<__nv_bfloat16> e;
  const int co = dgrad ? Cin : Cout, ci = dgrad ? Cout : Cin;
  e.C = (__nv_bfloat16*)y;
  e.ldc = co;
  e.res = (const __nv_bfloat16*)res;
  e.ldres = co;
  e.mask = (const __nv_bfloat16*)mask;
  e.ldmask = co;
  e.mask_mode = mask ? kMaskRelu : kMaskNone;
  epilogue_finalize(e, co);
  return launch_conv3x3_tc(N, H, W, ci, co, (const __nv_bfloat16*)x, (const __nv_bfloat16*)w,
                           dgrad != 0, e, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int ppll_conv3x3_bf16(int N, int H, int W, int Cin, int Cout, const void* x,
                                 const void* w, void* y, int dgrad, void* stream) {
  return ppll_conv3x3_bf16_ex(N, H, W, Cin, Cout, x, w, y, dgrad, nullptr, nullptr, stream);
}

// dW (fp32 [9·Cin, Cout], the GEMM weight layout) of the 3x3 / stride-1 conv
// of x [N,H,W,Cin] given dz = dLoss/dconv-output [N·H·W, Cout]; ws: split-K
// partials (ppll_conv3x3_wgrad_ws_floats)
extern "C" long ppll_conv3x3_wgrad_ws_floats(int N, int H, int W, int Cin, int Cout) {
  (void)N; (void)H; (void)W;
  return 148L * 9 * Cin * Cout;
}
extern "C" int ppll_conv3x3_wgrad_bf16(int N, int H, int W, int Cin, int Cout, const void* x,
                                       const void* dz, float* dw, float* ws, long ws_floats,
                                       void* stream) {
  using namespace ppll;
  if (N < 1 || H < 1 || W < 1 || !x || !dz || !dw || !ws || ws_floats < 1) {
    set_error("ppll_conv3x3_wgrad_bf16: invalid arguments");
    return PPLL_ERR_ARG;
  }
  return launch_conv3x3_wgrad_tc(N, H, W, Cin, Cout, (const __nv_bfloat16*)x,
                                 (const __nv_bfloat16*)dz, dw, ws, (size_t)ws_floats,
                                 reinterpret_cast<cudaStream_t>(stream));
}
