// tcgen05 + TMA + TMEM GEMM for sm_100a (the tensor-core engine of the
// linear-layer fwd / dgrad / wgrad ops, tensor.py:137-150 adjoints).
//
//   C[M,N] = Σ_k A(m,k)·B(k,n)   bf16 operands, fp32 accumulation in TMEM.
//
// Persistent kernel: one CTA per SM walks a static schedule of work items
// (128 x BN output tiles, optionally split along K).  Warp roles (576 thr):
//   warp 0      TMA producer (one elected lane): A/B k-blocks of 64 into a
//               kStages-deep shared-memory ring (mbarrier full/empty);
//   warp 1      TMEM allocator + MMA issuer (one elected lane): 4 x
//               tcgen05.mma (M=128, N=BN, K=16) per k-block, tcgen05.commit
//               frees the smem slot; accumulators are DOUBLE-BUFFERED in
//               TMEM (2 x BN columns) so tile i+1's MMAs overlap tile i's
//               epilogue;
//   warps 2..17 epilogue (four warps per TMEM lane quadrant, interleaved
//               16-column chunks): tcgen05.ld 32x32b.x16 (one accumulator row per
//               thread) → fused bias / residual / pre-activation store /
//               ReLU|GELU / ReLU-mask|GELU-gradient / dual store (the ring
//               push); each warp's 32x16 block is transposed through a 1-KB
//               smem buffer so stores cover 16 rows x 32 B (full sectors); or fp32
//               split-K partials reduced afterwards in fixed split order
//               (deterministic) by splitk_reduce_kernel with the same epilogue.
// Operand layouts (128-byte swizzled, TMA box inner extent 64 elements):
//   K-major  box {64 (K), rows};  UMMA desc SBO = 1024 B, K step +32 B.
//   MN-major boxes {64 (MN), 64 (K)} every 8 KB along MN;  UMMA desc
//            LBO = 8 KB (MN-chunk stride), SBO = 1024 B, K step +2048 B.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>
#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace ppll {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kEpiWarps = 16;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kNumSMs = 148;

using namespace ptx;

template <int BN>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 2;     // 16 KB
  static constexpr int B_BYTES = (BN < 64 ? 64 : BN) * BK * 2;  // MN-major boxes are 64 wide
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN >= 256) ? 4 : (BN >= 192 ? 4 : 6);
  static constexpr int EPI = 2 * BN * 4;          // bias slice per accumulator buffer
  static constexpr int STG = kEpiWarps * 1024;    // per-warp store-transpose buffers
  static constexpr int TOTAL = STAGES * STAGE + EPI + STG + 1024 /*align*/ + 512 /*barriers, work ring*/;
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 128) ? 128 : (2 * BN <= 256 ? 256 : 512);
};

struct Sched {
  // TMA store maps of the outputs C and pre (valid when tma_st): the kernel
  // takes Sched as a __grid_constant__ parameter so the maps live in param space
  CUtensorMap st_c, st_p;
  int tma_st;
  int drain_full;   // PPLL_GEMM_DRAIN_FULL=1: wait for the bulk stores' writes at exit
  int clc;          // dynamic tile scheduling (grid = items, CLC try_cancel work stealing)
  int mt, nt, tiles, splits, kps, items;
  int probe;   // profiling probe (PPLL_GEMM_PROBE): 1 = skip the epilogue math/stores,
              // 2 = bias+GELU math only, 3 = stores only (interior tiles)
  // timeline probe (PPLL_GEMM_TIMELINE): per CTA and tile, %globaltimer at
  // MMA start / MMA done (tfull observed) / epilogue done, 4 tiles max
  unsigned long long* tl;
};

// Dynamic tile scheduling (Sched::clc): the grid has one CTA per work item;
// a running CTA first takes its own item, then steals the items of CTAs the
// hardware has not launched yet with clusterlaunchcontrol.try_cancel — so when
// other streams' kernels hold some SMs, the CTAs that do run take more tiles
// instead of leaving a static 1/148 share to CTAs that start late.  The TMA
// producer thread owns the sequence and hands each item id to the MMA and
// epilogue warps through a 4-deep shared-memory ring (full / empty mbarriers).
__device__ __forceinline__ void clc_try_cancel(uint32_t resp, uint64_t* bar) {
  asm volatile(
      "clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];"
      ::"r"(resp), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ int clc_decode(uint32_t resp) {
  uint32_t x = 0, valid = 0;
  asm volatile(
      "{\n\t.reg .pred p1;\n\t.reg .b128 r;\n\t"
      "ld.shared.b128 r, [%2];\n\t"
      "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p1, r;\n\t"
      "selp.u32 %1, 1, 0, p1;\n\t"
      "@p1 clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %0, r;\n\t}"
      : "=r"(x), "=r"(valid)
      : "r"(resp)
      : "memory");
  return valid ? (int)x : -1;
}
constexpr int kWorkRing = 4;

// MC: CTA pair (cta_group::2, 2-CTA cluster): the pair computes one 256 x BN
// tile — each CTA loads its 128 rows of A and BN/2 rows of B, the leader
// (rank 0) issues M=256 MMAs over both CTAs' smem, each CTA's TMEM holds its
// 128 accumulator rows and its epilogue stores them.  Per SM, a k-block moves
// 16 KB + BN·64 B instead of 16 KB + BN·128 B (the L2->smem fill bound of the
// single-CTA kernel).
// (m-tiles 2p, 2p+1, same n-tile) and shares the B operand — each CTA fetches
// half of every B k-block and multicasts it to both, halving B's L2->SM
// traffic; a slot is refilled only when both CTAs' MMAs have consumed it
// (empty barriers count the two CTAs' multicast commits).
template <typename TO, bool A_K, bool B_K, int BN, int F, bool MC = false>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               int M, int N, int K, const __grid_constant__ Sched sc, Epilogue<TO> ep,
               float* part) {
  using L = Smem<BN>;
  constexpr int S = L::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (base & 1023)) & 1023);
  float* bias_s = reinterpret_cast<float*>(smem + S * L::STAGE);
  uint8_t* stg_all = smem + S * L::STAGE + L::EPI;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg_all + L::STG);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;      // [2]
  uint64_t* tempty = tfull + 2;     // [2]
  uint64_t* wfull = tempty + 2;     // [kWorkRing] dynamic-schedule work ring
  uint64_t* wempty = wfull + kWorkRing;
  uint64_t* clc_bar = wempty + kWorkRing;
  int* wq = reinterpret_cast<int*>(clc_bar + 1);                   // [kWorkRing]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wq + kWorkRing);
  uint8_t* clc_resp = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(tmem_slot) + 16 + 15) & ~uintptr_t(15));   // 16-B aligned
  const bool clc = !MC && sc.clc;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], MC ? 2 * kEpiWarps : kEpiWarps);   // pair: both CTAs' warps
    }
    for (int i = 0; i < kWorkRing; ++i) {
      mbar_init(&wfull[i], 1);
      mbar_init(&wempty[i], 1 + kEpiWarps);                     // MMA warp + epilogue warps
    }
    mbar_init(clc_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  // work decomposition: MC clusters walk pair-tiles, the CTA rank picks the row
  const int rank = MC ? (int)cluster_ctarank() : 0;
  const int wid0 = MC ? (int)blockIdx.x / 2 : (int)blockIdx.x;
  const int wstride = MC ? (int)gridDim.x / 2 : (int)gridDim.x;
  const int mtw = MC ? (sc.mt + 1) / 2 : sc.mt;          // m-tiles (pairs) per n column
  const int tiles_w = mtw * sc.nt;
  const int items_w = MC ? tiles_w : sc.items;
  if constexpr (MC) cluster_sync();   // peers' barriers initialised before any remote use
  if (warp == 1) {
    if constexpr (MC) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(L::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(L::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // prologue (barriers, TMEM, tensor-map prefetch) overlaps the predecessor's tail
  pdl_entry();

  if (warp == 0) {
    // ------------------------- TMA producer -------------------------
    if (lane == 0) {
      int kb_total = 0;
      int w = wid0;
      for (int n = 0;; ++n) {
        if (clc) {   // publish this item (or the end) to the MMA / epilogue warps
          const int ws = n % kWorkRing;
          mbar_wait(&wempty[ws], ((n / kWorkRing) & 1) ^ 1);
          wq[ws] = w;
          mbar_arrive(&wfull[ws]);
          if (w < 0) break;
          // ask for the next item while this one's operands stream in
          mbar_expect_tx(clc_bar, 16);
          clc_try_cancel(smem_u32(clc_resp), clc_bar);
        } else {
          if (n > 0) w += wstride;
          if (w >= items_w) break;
        }
        const int tile = w % tiles_w, z = MC ? 0 : w / sc.tiles;
        const int m0 = ((tile % mtw) * (MC ? 2 : 1) + rank) * BM, n0 = (tile / mtw) * BN;
        const int kbeg = z * sc.kps, kend = min(K, kbeg + sc.kps);
        for (int k0 = kbeg; k0 < kend; k0 += BK, ++kb_total) {
          const int st = kb_total % S;
          mbar_wait(&empty[st], ((kb_total / S) & 1) ^ 1);
          uint8_t* sa = smem + st * L::STAGE;
          uint8_t* sb = sa + L::A_BYTES;
          if constexpr (MC) {
            // both CTAs' loads complete on the leader's barrier; only the
            // leader arrives (with the pair's byte count)
            const uint32_t lb = mapa_shared(smem_u32(&full[st]), 0);
            if (rank == 0) mbar_expect_tx(&full[st], 2 * (L::A_BYTES + (BN / 2) * BK * 2));
            if (A_K) {
              tma_load_2d_cg2(&map_a, lb, sa, k0, m0);
            } else {
#pragma unroll
              for (int i = 0; i < BM / 64; ++i)
                tma_load_2d_cg2(&map_a, lb, sa + i * 8192, m0 + 64 * i, k0);
            }
            const int nb = n0 + rank * (BN / 2);
            if (B_K) {
              tma_load_2d_cg2(&map_b, lb, sb, k0, nb);
            } else {
#pragma unroll
              for (int i = 0; i < BN / 128; ++i)
                tma_load_2d_cg2(&map_b, lb, sb + i * 8192, nb + 64 * i, k0);
            }
            continue;
          }
          mbar_expect_tx(&full[st], L::A_BYTES + (B_K ? BN * BK * 2 : L::B_BYTES));
          if (A_K) {
            tma_load_2d(&map_a, &full[st], sa, k0, m0);
          } else {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i)
              tma_load_2d(&map_a, &full[st], sa + i * 8192, m0 + 64 * i, k0);
          }
          if (B_K) {
            tma_load_2d(&map_b, &full[st], sb, k0, n0);
          } else {
#pragma unroll
            for (int i = 0; i < (BN + 63) / 64; ++i)
              tma_load_2d(&map_b, &full[st], sb + i * 8192, n0 + 64 * i, k0);
          }
        }
        if (clc) {
          mbar_wait(clc_bar, n & 1);
          w = clc_decode(smem_u32(clc_resp));
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------- MMA issuer ---------------------------
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((A_K ? 0u : 1u) << 15) |
                           ((B_K ? 0u : 1u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)((MC ? 2 * BM : BM) >> 4) << 24);
    if (lane == 0 && rank == 0) {   // pair: the leader issues for both CTAs
      int kb_total = 0, it = 0;
      int w = wid0;
      for (int n = 0;; ++n, ++it) {
        if (clc) {
          const int ws = n % kWorkRing;
          mbar_wait(&wfull[ws], (n / kWorkRing) & 1);
          w = wq[ws];
          mbar_arrive(&wempty[ws]);
          if (w < 0) break;
        } else {
          if (n > 0) w += wstride;
          if (w >= items_w) break;
        }
        const int z = MC ? 0 : w / sc.tiles;
        const int kbeg = z * sc.kps, kend = min(K, kbeg + sc.kps);
        const int acc = it & 1;
        const uint32_t dtm = tmem + (uint32_t)(acc * BN);
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (sc.tl && it < 4) sc.tl[(blockIdx.x * 4 + it) * 4 + 0] = gtimer();
        int first = 1;
        for (int k0 = kbeg; k0 < kend; k0 += BK, ++kb_total) {
          const int st = kb_total % S;
          mbar_wait(&full[st], (kb_total / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(smem + st * L::STAGE);
          const uint32_t sb = sa + L::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_K ? umma_desc_sw128(sa + k * 32, 16, 1024)
                                    : umma_desc_sw128(sa + k * 2048, 8192, 1024);
            const uint64_t bd = B_K ? umma_desc_sw128(sb + k * 32, 16, 1024)
                                    : umma_desc_sw128(sb + k * 2048, 8192, 1024);
            if constexpr (MC) mma_bf16_cg2(dtm, ad, bd, idesc, first ? 0u : 1u);
            else mma_bf16(dtm, ad, bd, idesc, first ? 0u : 1u);
            first = 0;
          }
          if constexpr (MC) mma_commit_cg2(&empty[st], (uint16_t)3);   // both CTAs' slot
          else mma_commit(&empty[st]);
        }
        if constexpr (MC) mma_commit_cg2(&tfull[acc], (uint16_t)3);
        else mma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------- epilogue -----------------------------
    // thread = one accumulator row; kEpiWarps/4 warps per TMEM lane quadrant
    // take interleaved 16-column chunks (more warps in flight per scheduler
    // hide the TMEM-load / MUFU / store latencies of the fused epilogue)
    constexpr int NG = kEpiWarps / 4;
    const int q = warp & 3;                    // TMEM lane quadrant of this warp
    const int grp = (warp - 2) >> 2;
    uint8_t* stg = stg_all + (warp - 2) * 1024;
    int it = 0;
    int w = wid0;
    for (int n = 0;; ++n, ++it) {
      if (clc) {
        const int ws = n % kWorkRing;
        mbar_wait(&wfull[ws], (n / kWorkRing) & 1);
        w = wq[ws];
        __syncwarp();
        if (lane == 0) mbar_arrive(&wempty[ws]);
        if (w < 0) break;
      } else {
        if (n > 0) w += wstride;
        if (w >= items_w) break;
      }
      const int tile = w % tiles_w, z = MC ? 0 : w / sc.tiles;
      const int m0 = ((tile % mtw) * (MC ? 2 : 1) + rank) * BM, n0 = (tile / mtw) * BN;
      const int acc = it & 1;
      const bool split = sc.splits > 1;
      float* bs = bias_s + acc * BN;
      if (!split && ep.bias) {
        // stage this tile's bias slice in shared memory (epilogue warps only)
        for (int t = threadIdx.x - 64; t < BN; t += 32 * kEpiWarps)
          bs[t] = (n0 + t < N) ? __ldg(ep.bias + n0 + t) : 0.f;
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      }
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (sc.tl && it < 4 && warp == 2 && lane == 0) sc.tl[(blockIdx.x * 4 + it) * 4 + 1] = gtimer();
      const int row = m0 + q * 32 + lane;
      const bool live = row < M;
      // interior tiles store without bounds tests (uniform per tile)
      const bool full = F != kEFGeneric && ep.vec && m0 + BM <= M && n0 + BN <= N;
      const bool tst = F != kEFGeneric && sc.tma_st;
      // residual / mask blocks (bf16 specialised forms) are fetched one chunk
      // ahead: chunk c+1's global loads are in flight while chunk c computes
      constexpr bool kAhead = Epilogue<TO>::template kBlockAux<F>;
      uint4 nqr[2], nqk[2];
      if (kAhead && !split && !sc.probe && 16 * grp < BN && n0 + 16 * grp < N)
        ep.template aux_issue<F>(m0 + q * 32, M, n0 + 16 * grp, nqr, nqk, lane);
#pragma unroll 1
      for (int c = 16 * grp; c < BN && n0 + c < N; c += 16 * NG) {
        float ra[16], ka[16];
        uint4 qr[2], qk[2];
        // residual / mask loads are issued before the TMEM load so they overlap it
        if (!split && !sc.probe) {
          if constexpr (kAhead) {
#pragma unroll
            for (int j = 0; j < 2; ++j) { qr[j] = nqr[j]; qk[j] = nqk[j]; }
            const int cn = c + 16 * NG;
            if (cn < BN && n0 + cn < N)
              ep.template aux_issue<F>(m0 + q * 32, M, n0 + cn, nqr, nqk, lane);
          } else {
            ep.template aux_issue<F>(m0 + q * 32, M, n0 + c, qr, qk, lane);
          }
          if (live) ep.template load_aux16_t<F>(row, n0 + c, ra, ka);
        }
        uint32_t r[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c), r);
        if (!split && !sc.probe) {
          // aux_finish transposes through stg: the last bulk store must have read it
          if (tst && (F & (kEFRes | kEFMaskRelu | kEFMaskMul)) != 0) {
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
          }
          ep.template aux_finish<F>(qr, qk, ra, ka, stg, lane);
        }
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
        if (split)
          warp_store_block16<float>(part + (long)z * M * N, N, nullptr, 0, m0 + q * 32, M, n0 + c,
                                    N, (N % 4) == 0, v, stg, lane);
        else if (!sc.probe) {
          if (tst)
            ep.template finish_block16_t<F, true, true>(m0 + q * 32, M, n0 + c, v, ra, ka, bs + c,
                                                        stg, lane, &sc.st_c, &sc.st_p);
          else if (full)
            ep.template finish_block16_t<F, true>(m0 + q * 32, M, n0 + c, v, ra, ka, bs + c, stg,
                                                  lane);
          else
            ep.template finish_block16_t<F>(m0 + q * 32, M, n0 + c, v, ra, ka, bs + c, stg, lane);
        }
        else if (sc.probe == 2) {           // math only (bias + GELU pair), no stores
          float d[16], acc_s = 0.f;
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            v[i] += bs[c + i]; v[i + 1] += bs[c + i + 1];
            gelu_tanh2(v[i], v[i + 1], d[i], d[i + 1]);
            acc_s += v[i] + v[i + 1] + d[i] + d[i + 1];
          }
          if (live && acc_s == 12345.f) ep.C[0] = (TO)acc_s;
        } else if (sc.probe == 3) {         // stores only (both outputs, no math)
          warp_store_block16<TO, true>(ep.C, ep.ldc, nullptr, 0, m0 + q * 32, M, n0 + c, N, true,
                                       v, stg, lane);
          if (ep.pre)
            warp_store_block16<TO, true>(ep.pre, ep.ldpre, nullptr, 0, m0 + q * 32, M, n0 + c, N,
                                         true, v, stg, lane);
        } else if (live && v[0] == 12345.f)   // keep the TMEM load live in probe mode
          ep.C[0] = v[1];
      }
      // accumulator buffer drained: hand it back to the MMA warp
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if constexpr (MC) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
        else mbar_arrive(&tempty[acc]);
      }
      if (sc.tl && it < 4 && lane == 0) atomicMax(&sc.tl[(blockIdx.x * 4 + it) * 4 + 2], gtimer());
    }
    if (F != kEFGeneric && sc.tma_st) tma_store_drain(lane, sc.drain_full);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  // the leader's last commits land on the peer's barriers and the peer's
  // epilogue arrives on the leader's: both stay alive until here
  if constexpr (MC) cluster_sync();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (MC)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(L::TMEM_COLS));
    else
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(L::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// Cluster split-K (one output tile per cluster, one K slice per CTA).
// The CS CTAs of a thread-block cluster each accumulate a K slice of the
// same 128 x BN tile in TMEM; the partial is dumped into the CTA's own
// (now idle) operand ring as fp32 [128][BN] (16-B chunks XOR-swizzled by
// row), the cluster synchronises once, and CTA r reduces rows
// [r·R, r·R + R) over all CS partials through distributed shared memory in
// fixed rank order (deterministic) and stores them with coalesced 16-B
// vectors.  Replaces the fp32 HBM workspace + splitk_reduce pass for the
// weight-gradient GEMMs (long K = tokens, small M x N).  Plain epilogue.
// ---------------------------------------------------------------------------
template <typename TO, bool A_K, bool B_K, int BN>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tc_cluster_kernel(const __grid_constant__ CUtensorMap map_a,
                       const __grid_constant__ CUtensorMap map_b, int M, int N, int K, int mt,
                       int kps, TO* __restrict__ C, long ldc, int vec, float* __restrict__ db,
                       unsigned long long* __restrict__ tl) {
  using L = Smem<BN>;
  constexpr int S = L::STAGES;
  static_assert(S * L::STAGE >= BM * BN * 4, "reduction buffer must fit in the operand ring");
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (base & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * L::STAGE + L::EPI + L::STG);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 2);
  float* red = reinterpret_cast<float*>(smem);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int CS = (int)cluster_nctarank(), rank = (int)cluster_ctarank();
  const int tile = blockIdx.x / CS;
  const int m0 = (tile % mt) * BM, n0 = (tile / mt) * BN;
  const int kbeg = rank * kps, kend = min(K, kbeg + kps);
  // fused bias gradient db[n] = Σ_k B(k, n) (the Σ rows of dY of a weight
  // gradient): the idle epilogue warps of the m-tile-0 clusters sum each B
  // k-block from shared memory while the MMAs run (MN-major B only)
  const bool do_cs = !B_K && db != nullptr && (tile % mt) == 0;
  float* cs_red = reinterpret_cast<float*>(smem + S * L::STAGE + L::EPI);   // STG area
  float* cs_part = reinterpret_cast<float*>(smem + S * L::STAGE);           // EPI area

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], do_cs ? 1 + kEpiWarps : 1);
    }
    mbar_init(&tfull[0], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  constexpr uint32_t kCols = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // prologue (barriers, TMEM, tensor-map prefetch) overlaps the predecessor's tail
  pdl_entry();
  // timeline probe (PPLL_GEMM_TIMELINE): per CTA, %globaltimer at start / first
  // operands landed / mainloop done / partial dumped + cluster barrier /
  // reduction done / exit
  if (tl && threadIdx.x == 0) tl[blockIdx.x * 8 + 0] = gtimer();

  if (warp == 0) {
    if (lane == 0) {
      int kb = 0;
      for (int k0 = kbeg; k0 < kend; k0 += BK, ++kb) {
        const int st = kb % S;
        mbar_wait(&empty[st], ((kb / S) & 1) ^ 1);
        uint8_t* sa = smem + st * L::STAGE;
        uint8_t* sb = sa + L::A_BYTES;
        mbar_expect_tx(&full[st], L::A_BYTES + (B_K ? BN * BK * 2 : L::B_BYTES));
        if (A_K) {
          tma_load_2d(&map_a, &full[st], sa, k0, m0);
        } else {
#pragma unroll
          for (int i = 0; i < BM / 64; ++i)
            tma_load_2d(&map_a, &full[st], sa + i * 8192, m0 + 64 * i, k0);
        }
        if (B_K) {
          tma_load_2d(&map_b, &full[st], sb, k0, n0);
        } else {
#pragma unroll
          for (int i = 0; i < (BN + 63) / 64; ++i)
            tma_load_2d(&map_b, &full[st], sb + i * 8192, n0 + 64 * i, k0);
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((A_K ? 0u : 1u) << 15) |
                           ((B_K ? 0u : 1u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
    if (lane == 0) {
      int kb = 0, first = 1;
      for (int k0 = kbeg; k0 < kend; k0 += BK, ++kb) {
        const int st = kb % S;
        mbar_wait(&full[st], (kb / S) & 1);
        if (tl && kb == 0) tl[blockIdx.x * 8 + 1] = gtimer();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sa = smem_u32(smem + st * L::STAGE);
        const uint32_t sb = sa + L::A_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t ad = A_K ? umma_desc_sw128(sa + k * 32, 16, 1024)
                                  : umma_desc_sw128(sa + k * 2048, 8192, 1024);
          const uint64_t bd = B_K ? umma_desc_sw128(sb + k * 32, 16, 1024)
                                  : umma_desc_sw128(sb + k * 2048, 8192, 1024);
          mma_bf16(tmem, ad, bd, idesc, first ? 0u : 1u);
          first = 0;
        }
        mma_commit(&empty[st]);
      }
      mma_commit(&tfull[0]);
    }
    __syncwarp();
  } else {
    if (do_cs) {
      // thread t: 8-column chunk ch = t % NCH of the B tile, rows rg, rg + RG, ...
      constexpr int NCH = BN / 8, RG = (32 * kEpiWarps) / NCH;
      const int t = threadIdx.x - 64, ch = t % NCH, rg = t / NCH;
      float acc[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = 0.f;
      int kb = 0;
      for (int k0 = kbeg; k0 < kend; k0 += BK, ++kb) {
        const int st = kb % S;
        mbar_wait(&full[st], (kb / S) & 1);
        if (rg < RG) {
          const uint8_t* sb = smem + st * L::STAGE + L::A_BYTES + (ch >> 3) * 8192;
          const int c16 = ch & 7;
          for (int r = rg; r < BK; r += RG) {
            const uint4 q = *reinterpret_cast<const uint4*>(sb + r * 128 + ((c16 ^ (r & 7)) * 16));
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(h[e]);
              acc[2 * e] += f.x;
              acc[2 * e + 1] += f.y;
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);   // this warp is done with the slot
      }
      if (rg < RG) {
#pragma unroll
        for (int e = 0; e < 8; ++e) cs_red[rg * BN + ch * 8 + e] = acc[e];
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      for (int c = t; c < BN; c += 32 * kEpiWarps) {
        float v = 0.f;
        for (int g = 0; g < RG; ++g) v += cs_red[g * BN + c];      // fixed order
        cs_part[c] = v;
      }
    }
    // all MMAs retired => every operand slot has been consumed: the ring is
    // free and becomes this CTA's fp32 partial tile
    const int q = warp & 3, grp = (warp - 2) >> 2;
    mbar_wait(&tfull[0], 0);
    if (tl && warp == 2 && lane == 0) tl[blockIdx.x * 8 + 2] = gtimer();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int r = q * 32 + lane;
    float* row = red + (long)r * BN;
#pragma unroll 1
    for (int c = 32 * grp; c < BN; c += 32 * (kEpiWarps / 4)) {
      uint32_t v[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int ch = (c >> 2) + j;                       // 16-B chunk index in the row
        const int sw = (ch & ~7) | ((ch ^ r) & 7);
        *reinterpret_cast<uint4*>(row + 4 * sw) = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  if (tl && threadIdx.x == 0) tl[blockIdx.x * 8 + 3] = gtimer();
  // ---- distributed reduction: this CTA owns rows [rank·R, rank·R + R) ----
  {
    const int R = (BM + CS - 1) / CS;
    const int r0 = rank * R, r1 = min(BM, r0 + R);
    constexpr int C4 = BN / 4;
    const uint32_t red_addr = smem_u32(red);
    for (int idx = threadIdx.x; idx < (r1 - r0) * C4; idx += kThreads) {
      const int r = r0 + idx / C4, ch = idx % C4;
      const int sw = (ch & ~7) | ((ch ^ r) & 7);
      const uint32_t a = red_addr + (uint32_t)((r * BN + 4 * sw) * 4);
      float4 acc = ld_dsmem_f4(a, 0);
      for (int src = 1; src < CS; ++src) {
        const float4 t = ld_dsmem_f4(a, (uint32_t)src);
        acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
      }
      const int grow = m0 + r, gcol = n0 + 4 * ch;
      if (grow < M && gcol < N) {
        TO* dst = C + (long)grow * ldc + gcol;
        const float e[4] = {acc.x, acc.y, acc.z, acc.w};
        if (vec && gcol + 4 <= N) {
          if constexpr (sizeof(TO) == 4) {
            *reinterpret_cast<float4*>(dst) = acc;
          } else {
            __nv_bfloat162 h[2] = {__floats2bfloat162_rn(acc.x, acc.y), __floats2bfloat162_rn(acc.z, acc.w)};
            *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<uint2*>(h);
          }
        } else {
          for (int t = 0; t < 4 && gcol + t < N; ++t) DT<TO>::st(dst + t, e[t]);
        }
      }
    }
  }
  if (do_cs && rank == 0) {   // Σ of the K-slice column sums in fixed rank order
    const uint32_t cs_addr = smem_u32(cs_part);
    for (int c = threadIdx.x; c < BN / 4; c += kThreads) {
      float4 acc = ld_dsmem_f4(cs_addr + 16 * c, 0);
      for (int src = 1; src < CS; ++src) {
        const float4 t = ld_dsmem_f4(cs_addr + 16 * c, (uint32_t)src);
        acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
      }
      const float e[4] = {acc.x, acc.y, acc.z, acc.w};
      for (int j = 0; j < 4; ++j)
        if (n0 + 4 * c + j < N) db[n0 + 4 * c + j] = e[j];
    }
  }
  if (tl && threadIdx.x == 0) tl[blockIdx.x * 8 + 4] = gtimer();
  cluster_sync();   // peers may still be reading this CTA's partial until here
  if (tl && threadIdx.x == 0) tl[blockIdx.x * 8 + 5] = gtimer();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static unsigned long long* cluster_tl();
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 map: inner extent `inner` (contiguous), outer extent `outer`, row
// pitch `ld` elements, box {64, box_outer}, 128-B swizzle, OOB -> zero.
static bool make_map(CUtensorMap* map, const void* ptr, long inner, long outer, long ld,
                     int box_outer) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 2-D output map for the epilogue's TMA stores: box {32 B, 32 rows} (one
// warp's 32-row x 16-column block, or 8 fp32 columns), 32-B swizzle (the
// layout warp_store_tma16 writes), dims {N, M} so ragged edges are clipped.
template <typename TO>
static bool make_store_map(CUtensorMap* map, const void* ptr, long n, long m, long ld) {
  auto enc = get_encode();
  if (!enc || !ptr) return false;
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * sizeof(TO))};
  cuuint32_t box[2] = {(cuuint32_t)(32 / sizeof(TO)), 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, sizeof(TO) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                        : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                   2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <typename TO, bool A_K, bool B_K, int BN, int F>
static int run(const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K, const Sched& sc,
               const Epilogue<TO>& ep, float* part, cudaStream_t s) {
  auto kern = gemm_tc_kernel<TO, A_K, B_K, BN, F>;
  constexpr int smem = Smem<BN>::TOTAL;
  static bool attr_set = false;
  if (!attr_set) {
    PPLL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set = true;
  }
  const int lim = (g_gemm_cap > 0 && g_gemm_cap < kNumSMs) ? g_gemm_cap : kNumSMs;
  // dynamic scheduling: one CTA per item, running CTAs steal unlaunched ones
  const int grid = sc.clc ? sc.items : (sc.items < lim ? sc.items : lim);
  launch_k(kern, grid, kThreads, smem, s, ma, mb, M, N, K, sc, ep, part);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

// CTA-pair launch (2-CTA clusters, cta_group::2; see gemm_tc_kernel MC)
template <typename TO, bool A_K, bool B_K, int BN, int F>
static int run_mc(const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K,
                  const Sched& sc, const Epilogue<TO>& ep, cudaStream_t s) {
  auto kern = gemm_tc_kernel<TO, A_K, B_K, BN, F, true>;
  constexpr int smem = Smem<BN>::TOTAL;
  static bool attr_set = false;
  if (!attr_set) {
    PPLL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set = true;
  }
  const int pairs = ((sc.mt + 1) / 2) * sc.nt;
  const int grid = 2 * (pairs < kNumSMs / 2 ? pairs : kNumSMs / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
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
  float* part = nullptr;
  PPLL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, ma, mb, M, N, K, sc, ep, part));
  note_launch();
  return PPLL_OK;
}
template <typename TO, bool A_K, bool B_K, int F>
static int dispatch_mc(int bn, const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K,
                       const Sched& sc, const Epilogue<TO>& ep, cudaStream_t s) {
  switch (bn) {
    case 256: return run_mc<TO, A_K, B_K, 256, F>(ma, mb, M, N, K, sc, ep, s);
    case 192: return run_mc<TO, A_K, B_K, 192, F>(ma, mb, M, N, K, sc, ep, s);
    default: return run_mc<TO, A_K, B_K, 128, F>(ma, mb, M, N, K, sc, ep, s);
  }
}
// specialised epilogues with multicast (bf16 outputs, no split-K, BN >= 128)
template <typename TO, bool A_K, bool B_K>
static int dispatch_f_mc(int f, int bn, const CUtensorMap& ma, const CUtensorMap& mb, int M,
                         int N, int K, const Sched& sc, const Epilogue<TO>& ep, cudaStream_t s) {
  if constexpr (A_K && !B_K && sizeof(TO) == 2) {
    switch (f) {
      case 0: return dispatch_mc<TO, A_K, B_K, 0>(bn, ma, mb, M, N, K, sc, ep, s);
      case kEFBias: return dispatch_mc<TO, A_K, B_K, kEFBias>(bn, ma, mb, M, N, K, sc, ep, s);
      case kEFBias | kEFRes:
        return dispatch_mc<TO, A_K, B_K, kEFBias | kEFRes>(bn, ma, mb, M, N, K, sc, ep, s);
      case kEFBias | kEFGeluD:
        return dispatch_mc<TO, A_K, B_K, kEFBias | kEFGeluD>(bn, ma, mb, M, N, K, sc, ep, s);
      case kEFBias | kEFRelu:
        return dispatch_mc<TO, A_K, B_K, kEFBias | kEFRelu>(bn, ma, mb, M, N, K, sc, ep, s);
      default: break;
    }
  } else if constexpr (A_K && B_K && sizeof(TO) == 2) {
    switch (f) {
      case 0: return dispatch_mc<TO, A_K, B_K, 0>(bn, ma, mb, M, N, K, sc, ep, s);
      case kEFMaskRelu: return dispatch_mc<TO, A_K, B_K, kEFMaskRelu>(bn, ma, mb, M, N, K, sc, ep, s);
      case kEFMaskMul: return dispatch_mc<TO, A_K, B_K, kEFMaskMul>(bn, ma, mb, M, N, K, sc, ep, s);
      default: break;
    }
  }
  return PPLL_ERR_UNSUPPORTED;
}

template <typename TO, bool A_K, bool B_K, int F>
static int dispatch_bn(int bn, const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K,
                       const Sched& sc, const Epilogue<TO>& ep, float* part, cudaStream_t s) {
  switch (bn) {
    case 256: return run<TO, A_K, B_K, 256, F>(ma, mb, M, N, K, sc, ep, part, s);
    case 192: return run<TO, A_K, B_K, 192, F>(ma, mb, M, N, K, sc, ep, part, s);
    case 128: return run<TO, A_K, B_K, 128, F>(ma, mb, M, N, K, sc, ep, part, s);
    case 64: return run<TO, A_K, B_K, 64, F>(ma, mb, M, N, K, sc, ep, part, s);
    case 32: return run<TO, A_K, B_K, 32, kEFGeneric>(ma, mb, M, N, K, sc, ep, part, s);
    default: return run<TO, A_K, B_K, 16, kEFGeneric>(ma, mb, M, N, K, sc, ep, part, s);
  }
}

// epilogue specialisations instantiated per operand layout (bf16 outputs):
//   forward (A K-major, W MN-major): bias | bias+res | bias+GELU' | plain | bias+ReLU
//   dgrad   (both K-major)         : plain | ReLU mask | stored-derivative mask
template <typename TO, bool A_K, bool B_K>
static int dispatch_f(int f, int bn, const CUtensorMap& ma, const CUtensorMap& mb, int M, int N,
                      int K, const Sched& sc, const Epilogue<TO>& ep, float* part,
                      cudaStream_t s) {
  if (sc.splits > 1 || sizeof(TO) == 4)   // fp32 partials / fp32 outputs: generic
    return dispatch_bn<TO, A_K, B_K, kEFGeneric>(bn, ma, mb, M, N, K, sc, ep, part, s);
  if constexpr (A_K && !B_K) {
    switch (f) {
      case 0: return dispatch_bn<TO, A_K, B_K, 0>(bn, ma, mb, M, N, K, sc, ep, part, s);
      case kEFBias: return dispatch_bn<TO, A_K, B_K, kEFBias>(bn, ma, mb, M, N, K, sc, ep, part, s);
      case kEFBias | kEFRes:
        return dispatch_bn<TO, A_K, B_K, kEFBias | kEFRes>(bn, ma, mb, M, N, K, sc, ep, part, s);
      case kEFBias | kEFGeluD:
        return dispatch_bn<TO, A_K, B_K, kEFBias | kEFGeluD>(bn, ma, mb, M, N, K, sc, ep, part, s);
      case kEFBias | kEFRelu:
        return dispatch_bn<TO, A_K, B_K, kEFBias | kEFRelu>(bn, ma, mb, M, N, K, sc, ep, part, s);
      default: break;
    }
  } else if constexpr (A_K && B_K) {
    switch (f) {
      case 0: return dispatch_bn<TO, A_K, B_K, 0>(bn, ma, mb, M, N, K, sc, ep, part, s);
      case kEFMaskRelu:
        return dispatch_bn<TO, A_K, B_K, kEFMaskRelu>(bn, ma, mb, M, N, K, sc, ep, part, s);
      case kEFMaskMul:
        return dispatch_bn<TO, A_K, B_K, kEFMaskMul>(bn, ma, mb, M, N, K, sc, ep, part, s);
      default: break;
    }
  }
  return dispatch_bn<TO, A_K, B_K, kEFGeneric>(bn, ma, mb, M, N, K, sc, ep, part, s);
}

// ---- cluster split-K launcher ----------------------------------------------
template <typename TO, bool A_K, bool B_K, int BN>
static cudaLaunchConfig_t cluster_cfg(int grid, int cs, cudaStream_t s, cudaLaunchAttribute* at) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Smem<BN>::TOTAL;
  cfg.stream = s;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cfg;
}
template <typename TO, bool A_K, bool B_K, int BN>
static bool cluster_attr_init() {
  static bool done = false, ok = false;
  if (!done) {
    done = true;
    ok = cudaFuncSetAttribute(gemm_tc_cluster_kernel<TO, A_K, B_K, BN>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<BN>::TOTAL) ==
         cudaSuccess;
  }
  return ok;
}
// how many clusters of `cs` CTAs fit on the GPU at once (GPC packing), cached
template <typename TO, bool A_K, bool B_K, int BN>
static int cluster_capacity(int cs) {
  static int cap[9] = {-1, -1, -1, -1, -1, -1, -1, -1, -1};
  if (cs < 1 || cs > 8) return 0;
  if (cap[cs] < 0) {
    cap[cs] = 0;
    if (cluster_attr_init<TO, A_K, B_K, BN>()) {
      cudaLaunchAttribute at[2];
      cudaLaunchConfig_t cfg = cluster_cfg<TO, A_K, B_K, BN>(cs * kNumSMs, cs, 0, at);
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, gemm_tc_cluster_kernel<TO, A_K, B_K, BN>, &cfg) ==
          cudaSuccess)
        cap[cs] = n;
      else
        cudaGetLastError();
    }
  }
  return cap[cs];
}
template <typename TO, bool A_K, bool B_K, int BN>
static int run_cluster(const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K, int mt,
                       int tiles, int cs, int kps, TO* C, long ldc, int vec, float* db,
                       cudaStream_t s) {
  if (!cluster_attr_init<TO, A_K, B_K, BN>()) {
    set_error("gemm_tc_cluster_kernel: smem attribute");
    return PPLL_ERR_CUDA;
  }
  cudaLaunchAttribute at[2];
  cudaLaunchConfig_t cfg = cluster_cfg<TO, A_K, B_K, BN>(tiles * cs, cs, s, at);
  PPLL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, gemm_tc_cluster_kernel<TO, A_K, B_K, BN>, ma, mb, M, N,
                                     K, mt, kps, C, ldc, vec, db, cluster_tl()));
  note_launch();
  return PPLL_OK;
}
template <typename TO, bool A_K, bool B_K>
static int cluster_capacity_bn(int bn, int cs) {
  switch (bn) {
    case 256: return cluster_capacity<TO, A_K, B_K, 256>(cs);
    case 192: return cluster_capacity<TO, A_K, B_K, 192>(cs);
    case 128: return cluster_capacity<TO, A_K, B_K, 128>(cs);
    default: return cluster_capacity<TO, A_K, B_K, 64>(cs);
  }
}
template <typename TO, bool A_K, bool B_K>
static int dispatch_cluster(int bn, const CUtensorMap& ma, const CUtensorMap& mb, int M, int N,
                            int K, int mt, int tiles, int cs, int kps, TO* C, long ldc, int vec,
                            float* db, cudaStream_t s) {
  switch (bn) {
    case 256: return run_cluster<TO, A_K, B_K, 256>(ma, mb, M, N, K, mt, tiles, cs, kps, C, ldc, vec, db, s);
    case 192: return run_cluster<TO, A_K, B_K, 192>(ma, mb, M, N, K, mt, tiles, cs, kps, C, ldc, vec, db, s);
    case 128: return run_cluster<TO, A_K, B_K, 128>(ma, mb, M, N, K, mt, tiles, cs, kps, C, ldc, vec, db, s);
    default: return run_cluster<TO, A_K, B_K, 64>(ma, mb, M, N, K, mt, tiles, cs, kps, C, ldc, vec, db, s);
  }
}
template <typename TO>
static int capacity_any(bool ak, bool bk, int bn, int cs) {
  if (ak && !bk) return cluster_capacity_bn<TO, true, false>(bn, cs);
  if (ak && bk) return cluster_capacity_bn<TO, true, true>(bn, cs);
  if (!ak && !bk) return cluster_capacity_bn<TO, false, false>(bn, cs);
  return cluster_capacity_bn<TO, false, true>(bn, cs);
}

unsigned long long* timeline_buffer();
static unsigned long long* cluster_tl() {
  static const int on = getenv("PPLL_GEMM_TIMELINE") ? 1 : 0;
  return on ? timeline_buffer() : nullptr;
}
unsigned long long* timeline_buffer() {
  static unsigned long long* buf = nullptr;
  if (!buf && cudaMalloc(&buf, 65536 * 8) != cudaSuccess) buf = nullptr;   // 64 Ki stamps
  return buf;
}

// per-k-block (BK=64) mainloop cycles of a 128 x c tile: max(tensor floor,
// operand bytes (A 4 KB + B c·32 B per K=16) streamed L2 -> smem at ~80 B/cycle/SM)
static inline double kblock_cycles(int c) { return 4.0 * fmax(c / 2.0, (4096.0 + 32.0 * c) / 80.0); }

}  // namespace tc

template <typename TO>
int launch_gemm_tc(int M, int N, int K, const __nv_bfloat16* A, long lda, bool a_kmajor,
                   const __nv_bfloat16* B, long ldb, bool b_kmajor, const Epilogue<TO>& ep,
                   float* ws, size_t ws_elems, cudaStream_t s) {
  using namespace tc;
  // shapes a 128-row tensor-core tile cannot use efficiently go to the SIMT engine
  if (N < 16 || K < 16 || M < 1) return PPLL_ERR_UNSUPPORTED;
  if (((uintptr_t)A & 15) || ((uintptr_t)B & 15) || (lda * 2) % 16 || (ldb * 2) % 16)
    return PPLL_ERR_UNSUPPORTED;
  const int mt = ceil_div(M, BM);
  // Pick (tile width, K splits) with a small cost model (seconds):
  //   MMA    : waves x 128·BN·K/splits MACs at the per-SM tcgen05 rate
  //   epilog : 128·BN·bytes per item at ~150 GB/s per SM (one exposed, the
  //            rest overlap the next item's MMAs through the TMEM double buffer)
  //   split-K: partial write + read + reduce launch
  const double mac_rate = 1.5e15 / 2 / kNumSMs;          // MAC/s per SM (bf16, sustained)
  const double out_b = (double)sizeof(TO);
  int bn = 64, splits = 1;
  double best = -1;
  const int cands[6] = {256, 192, 128, 64, 32, 16};
  for (int i = 0; i < 6; ++i) {
    const int c = cands[i];
    if (c < 64 && N > c) continue;       // narrow tiles only as the single column tile
    const long tiles = (long)mt * ceil_div(N, c);
    int sp = 1;
    if (ws && !ep.cs_part && tiles * 2 <= kNumSMs && K >= 8 * BK) {
      sp = (int)(kNumSMs / tiles);
      if (sp > K / (4 * BK)) sp = K / (4 * BK);
      while (sp > 1 && (size_t)sp * M * N > ws_elems) --sp;
      if (sp < 1) sp = 1;
    }
    const long items = tiles * sp;
    const double waves = (double)((items + kNumSMs - 1) / kNumSMs);
    // per K=16 step: max(tensor floor 128·N/256 cycles, operand bytes (A 4 KB + B N·32 B)
    // streamed L2 -> smem at ~80 B/cycle/SM (measured: 128-wide tiles reach ~55 % of the
    // tensor peak, 256-wide ~82 %) — narrow tiles re-read A and are bandwidth bound
    const double cyc16 = fmax(c / 2.0, (4096.0 + 32.0 * c) / 80.0);
    const double t_mma = (double)ceil_div(K, 16 * sp) * cyc16 / 1.9e9;
    (void)mac_rate;
    const double t_epi = 128.0 * c * (sp > 1 ? 4.0 : out_b) / 150e9;
    double cost = waves * (t_mma > t_epi ? t_mma : t_epi) + t_epi;
    if (sp > 1) cost += (double)(sp + 1) * M * N * 4 / 5e12 + 2e-6;
    if (best < 0 || cost < best) { best = cost; bn = c; splits = sp; }
  }
  // Cluster split-K (plain epilogue only): one tile per cluster of cs CTAs,
  // partials reduced through DSMEM.  Cost: waves over the GPC-packed cluster
  // capacity x (K/cs mainloop + partial dump + distributed reduction).
  static const int force_cl = getenv("PPLL_GEMM_CLUSTER") ? atoi(getenv("PPLL_GEMM_CLUSTER")) : -1;
  const bool plain = !ep.bias && ep.act == kActNone && ep.mask_mode == kMaskNone && !ep.res &&
                     !ep.pre && !ep.C2;
  int cl_bn = 0, cl_cs = 0;
  static const double dsmem_bpc = getenv("PPLL_DSMEM_BPC") ? atof(getenv("PPLL_DSMEM_BPC")) : 24.0;
  // (experiment, PPLL_WGRAD_SHARED_CS=k) with stage streams sharing the GPU,
  // fix the K-split of the cluster weight gradients at k: fewer SMs for longer,
  // ~1/3 of the SM-time of the 6-8-way split.  Measured: ViT-S pipeline
  // 53.1k -> 47.3k (k=2) / 48.0k (k=3) / 45.0k (k=4) img/s — the longer
  // side-stream gradients delay each stage's update more than the freed SMs
  // help the other streams — so it is off by default.
  static const int shared_cs = getenv("PPLL_WGRAD_SHARED_CS") ? atoi(getenv("PPLL_WGRAD_SHARED_CS")) : 0;
  const int cs_fixed = (!g_gpu_excl && shared_cs >= 2) ? shared_cs : 0;
  if (plain && force_cl != 0 && K >= 8 * BK) {
    double cl_best = -1;
    const int cb[4] = {256, 192, 128, 64};
    for (int i = 0; i < 4; ++i) {
      const int c = cb[i];
      if (c > 64 && N <= c / 2) continue;
      const long tiles = (long)mt * ceil_div(N, c);
      for (int cs = cs_fixed ? cs_fixed : 2; cs <= (cs_fixed ? cs_fixed : 8); ++cs) {
        if (K < cs * 4 * BK) break;
        int cap = capacity_any<TO>(a_kmajor, b_kmajor, c, cs);
        if (g_wgrad_cap > 0 && cap > g_wgrad_cap / cs) cap = g_wgrad_cap / cs;
        if (cap <= 0) continue;
        const double waves = (double)((tiles + cap - 1) / cap);
        const double kb = (double)ceil_div(K, cs * BK);
        // partial dump (st.shared, ~128 B/cycle) + the distributed reduction: every
        // CTA reads one fp32 tile's worth over DSMEM, (cs-1)/cs of it remote
        const double t_red = 128.0 * c * 4 * (cs - 1) / cs / dsmem_bpc + 128.0 * c * 4 / 128.0;
        const double cost = waves * ((kb * kblock_cycles(c) + t_red) / 1.9e9 + 1.5e-6);
        if (cl_best < 0 || cost < cl_best) { cl_best = cost; cl_bn = c; cl_cs = cs; }
      }
    }
    if (cl_bn && (force_cl == 1 || cs_fixed || cl_best < best)) {
      bn = cl_bn;
    } else {
      cl_bn = 0;
    }
  }
  // (profiling) force the tile width: PPLL_GEMM_BN=64|128|192|256
  static const int force_bn = getenv("PPLL_GEMM_BN") ? atoi(getenv("PPLL_GEMM_BN")) : 0;
  if (force_bn && !cl_bn && (force_bn == 64 || force_bn == 128 || force_bn == 192 ||
                             force_bn == 256)) {
    bn = force_bn;
    splits = 1;
  }
  Sched sc;
  sc.tma_st = 0;
  static const int drain_full = getenv("PPLL_GEMM_DRAIN_FULL") ? atoi(getenv("PPLL_GEMM_DRAIN_FULL")) : 0;
  sc.drain_full = drain_full;
  static const int clc_env = getenv("PPLL_GEMM_CLC") ? atoi(getenv("PPLL_GEMM_CLC")) : 1;
  sc.clc = clc_env && g_gemm_cap == 0;
  sc.mt = mt;
  sc.nt = ceil_div(N, bn);
  sc.tiles = sc.mt * sc.nt;
  sc.kps = ceil_div(ceil_div(K, cl_bn ? cl_cs : splits), BK) * BK;
  sc.splits = ceil_div(K, sc.kps);
  sc.items = sc.tiles * sc.splits;
  static const int probe = getenv("PPLL_GEMM_PROBE") ? atoi(getenv("PPLL_GEMM_PROBE")) : 0;
  sc.probe = probe;
  static const int tl_on = getenv("PPLL_GEMM_TIMELINE") ? 1 : 0;
  sc.tl = tl_on ? timeline_buffer() : nullptr;
  // 2-CTA multicast of B: specialised bf16 epilogues, no split, >= 2 m-tiles
  // CTA pair (cta_group::2, M = 256 per MMA, B split across the pair), opt-in
  // (PPLL_GEMM_MC=1).  Measured (tools/gemm_one.py): 8192^3 1306 -> 1359 TF/s (82 % of
  // the measured peak); the ViT layer shapes gain nothing (ViT-S dgrads 4-5 % slower:
  // halving the per-SM B bytes did not shorten their ~580-cycle k-blocks, so those are
  // not smem-fill bound) and lose half the SMs when pair tiles do not fill the GPU
  // (ViT-B FC1 dgrad 23 -> 36 us).
  static const int force_mc = getenv("PPLL_GEMM_MC") ? atoi(getenv("PPLL_GEMM_MC")) : 0;
  const int fl = epi_flags(ep);
  const bool mc = force_mc != 0 && !cl_bn && sc.splits == 1 && sizeof(TO) == 2 && a_kmajor &&
                  bn >= 128 && mt >= 2 && fl != kEFGeneric && (b_kmajor || bn % 128 == 0) &&
                  (b_kmajor ? (fl == 0 || fl == kEFMaskRelu || fl == kEFMaskMul)
                            : (fl == 0 || fl == kEFBias || fl == (kEFBias | kEFRes) ||
                               fl == (kEFBias | kEFGeluD) || fl == (kEFBias | kEFRelu)));
  static const int verbose = getenv("PPLL_GEMM_VERBOSE") ? atoi(getenv("PPLL_GEMM_VERBOSE")) : 0;
  if (verbose)
    fprintf(stderr, "[gemm_tc] M=%d N=%d K=%d %s%s bn=%d tiles=%d splits=%d cluster=%d mc=%d "
            "flags=%d\n", M, N, K, a_kmajor ? "A:K" : "A:MN", b_kmajor ? " B:K" : " B:MN", bn,
            sc.tiles, sc.splits, cl_bn ? sc.splits : 0, (int)mc, fl);
  CUtensorMap ma, mb;
  bool ok = a_kmajor ? make_map(&ma, A, K, M, lda, BM) : make_map(&ma, A, M, K, lda, 64);
  ok = ok && (b_kmajor ? make_map(&mb, B, K, N, ldb, mc ? bn / 2 : bn)
                       : make_map(&mb, B, N, K, ldb, 64));
  if (!ok) return PPLL_ERR_UNSUPPORTED;
  // epilogue stores through the TMA engine (PPLL_GEMM_TMA_STORE=0: st.global)
  static const int tma_env = getenv("PPLL_GEMM_TMA_STORE") ? atoi(getenv("PPLL_GEMM_TMA_STORE")) : 1;
  if (tma_env && !cl_bn && sc.splits == 1 && fl != kEFGeneric && !ep.C2 && !ep.cs_part &&
      ep.vec && !sc.probe)
    sc.tma_st = make_store_map<TO>(&sc.st_c, ep.C, N, M, ep.ldc) &&
                (!(fl & kEFGeluD) || make_store_map<TO>(&sc.st_p, ep.pre, N, M, ep.ldpre));
  if (mc) {
    Epilogue<TO> e = ep;
    e.partial = nullptr;
    const int r = b_kmajor ? dispatch_f_mc<TO, true, true>(fl, bn, ma, mb, M, N, K, sc, e, s)
                           : dispatch_f_mc<TO, true, false>(fl, bn, ma, mb, M, N, K, sc, e, s);
    if (r != PPLL_ERR_UNSUPPORTED) return r;
    // (unsupported combination: rebuild the B map for the plain path)
    if (b_kmajor && !make_map(&mb, B, K, N, ldb, bn)) return PPLL_ERR_UNSUPPORTED;
  }
  if (cl_bn) {
    const int cs = sc.splits;   // every CTA of the cluster owns >= 1 k-block
    Epilogue<TO> e = ep;
    // fused bias column sums of the MN-major B operand (weight gradients)
    float* db = (!b_kmajor && ep.colsum_b) ? ep.colsum_b : nullptr;
    int r;
    if (a_kmajor && !b_kmajor)
      r = dispatch_cluster<TO, true, false>(bn, ma, mb, M, N, K, mt, sc.tiles, cs, sc.kps, e.C, e.ldc, e.vec, db, s);
    else if (a_kmajor && b_kmajor)
      r = dispatch_cluster<TO, true, true>(bn, ma, mb, M, N, K, mt, sc.tiles, cs, sc.kps, e.C, e.ldc, e.vec, nullptr, s);
    else if (!a_kmajor && !b_kmajor)
      r = dispatch_cluster<TO, false, false>(bn, ma, mb, M, N, K, mt, sc.tiles, cs, sc.kps, e.C, e.ldc, e.vec, db, s);
    else
      r = dispatch_cluster<TO, false, true>(bn, ma, mb, M, N, K, mt, sc.tiles, cs, sc.kps, e.C, e.ldc, e.vec, nullptr, s);
    return (r == PPLL_OK && db) ? kGemmColsumFused : r;
  }
  Epilogue<TO> e = ep;
  e.partial = nullptr;
  float* part = sc.splits > 1 ? ws : nullptr;
  int r;
  const int f = epi_flags(e);

  if (a_kmajor && !b_kmajor) r = dispatch_f<TO, true, false>(f, bn, ma, mb, M, N, K, sc, e, part, s);
  else if (a_kmajor && b_kmajor) r = dispatch_f<TO, true, true>(f, bn, ma, mb, M, N, K, sc, e, part, s);
  else if (!a_kmajor && !b_kmajor) r = dispatch_f<TO, false, false>(f, bn, ma, mb, M, N, K, sc, e, part, s);
  else r = dispatch_f<TO, false, true>(f, bn, ma, mb, M, N, K, sc, e, part, s);
  if (r || sc.splits == 1) return r;
  // deterministic split-K reduction (fixed split order) + the fused epilogue
  return launch_splitk_reduce<TO>(M, N, sc.splits, ws, ep, s);
}

template int launch_gemm_tc<float>(int, int, int, const __nv_bfloat16*, long, bool, const __nv_bfloat16*, long, bool, const Epilogue<float>&, float*, size_t, cudaStream_t);
template int launch_gemm_tc<__nv_bfloat16>(int, int, int, const __nv_bfloat16*, long, bool, const __nv_bfloat16*, long, bool, const Epilogue<__nv_bfloat16>&, float*, size_t, cudaStream_t);

}  // namespace ppll
