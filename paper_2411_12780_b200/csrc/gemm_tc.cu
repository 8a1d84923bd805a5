// tcgen05 + TMA + TMEM GEMM for sm_100a (the tensor-core engine of the
// linear-layer fwd / dgrad / wgrad ops, tensor.py:137-150 adjoints).
//
//   C[M,N] = Σ_k A(m,k)·B(k,n)   bf16 operands, fp32 accumulation in TMEM.
//
// One CTA computes a 128 x BN tile (UMMA M=128, N=BN, K=16 per instruction,
// cta_group::1).  Warp roles (192 threads):
//   warp 0      TMA producer (one elected lane): A/B k-blocks of 64 into a
//               kStages-deep smem ring, mbarrier full/empty handshake;
//   warp 1      TMEM allocator + MMA issuer (one elected lane): 4 x
//               tcgen05.mma per k-block, tcgen05.commit frees the smem slot;
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 (one accumulator row per
//               thread), fused bias / ReLU / ReLU-mask / dual store (the ring
//               push) or raw fp32 split-K partials.
// Operand layouts (all 128-byte swizzled, TMA box inner extent 64 elements):
//   K-major  (A: X[M,K], dY[M,N];  B: W[K_in,N_out] seen as N x K in dgrad):
//            box {64 (K), rows}; UMMA desc SBO = 1024 B, K advance +32 B.
//   MN-major (A: Xᵀ in wgrad;  B: W in fwd, dY in wgrad):
//            boxes {64 (MN), 64 (K)} stacked along MN every 8 KB;
//            UMMA desc LBO = 8 KB (MN chunk stride), SBO = 1024 B (8-row K
//            group stride), K advance +2048 B (16 rows of 128 B).
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"
#include "kernels.cuh"

namespace ppll {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;            // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int BN>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 2;     // 16 KB
  static constexpr int B_BYTES = BN * BK * 2;     // BN * 128 B
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN >= 256) ? 4 : 6;
  static constexpr int TOTAL = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/;
};

template <typename TO, bool A_K, bool B_K, int BN>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               int M, int N, int K, int k_per_split, Epilogue<TO> ep) {
  using L = Smem<BN>;
  constexpr int S = L::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (base & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * L::STAGE);
  uint64_t* empty = full + S;
  uint64_t* tmem_full = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kbeg = blockIdx.z * k_per_split;
  const int kend = min(K, kbeg + k_per_split);
  const int nkb = (kend - kbeg + BK - 1) / BK;
  constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------- TMA producer -------------------------
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % S;
        const uint32_t round = kb / S;
        mbar_wait(&empty[st], (round & 1) ^ 1);
        uint8_t* sa = smem + st * L::STAGE;
        uint8_t* sb = sa + L::A_BYTES;
        const int k0 = kbeg + kb * BK;
        mbar_expect_tx(&full[st], L::STAGE);
        if (A_K) {
          tma_load_2d(&map_a, &full[st], sa, k0, m0);
        } else {
#pragma unroll
          for (int i = 0; i < BM / 64; ++i) tma_load_2d(&map_a, &full[st], sa + i * 8192, m0 + 64 * i, k0);
        }
        if (B_K) {
          tma_load_2d(&map_b, &full[st], sb, k0, n0);
        } else {
#pragma unroll
          for (int i = 0; i < BN / 64; ++i) tma_load_2d(&map_b, &full[st], sb + i * 8192, n0 + 64 * i, k0);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------- MMA issuer ---------------------------
    // instruction descriptor: D=f32, A=B=bf16, majors, N>>3, M>>4
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((A_K ? 0u : 1u) << 15) |
                           ((B_K ? 0u : 1u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % S;
        const uint32_t round = kb / S;
        mbar_wait(&full[st], round & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sa = smem_u32(smem + st * L::STAGE);
        const uint32_t sb = sa + L::A_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t ad = A_K ? make_desc(sa + k * 32, 16, 1024) : make_desc(sa + k * 2048, 8192, 1024);
          const uint64_t bd = B_K ? make_desc(sb + k * 32, 16, 1024) : make_desc(sb + k * 2048, 8192, 1024);
          mma_bf16(tmem, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
        }
        mma_commit(&empty[st]);
      }
      mma_commit(tmem_full);
    }
    __syncwarp();
  } else {
    // ------------------------- epilogue -----------------------------
    const int q = warp & 3;                 // TMEM lane quadrant of this warp
    const int row = m0 + q * 32 + lane;
    if (lane == 0) mbar_wait(tmem_full, 0);
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c, r);
      if (row < M) {
        const int nb = n0 + c;
        if (ep.partial) {
          float* dst = ep.partial + ((long)blockIdx.z * M + row) * N + nb;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (nb + i < N) dst[i] = __uint_as_float(r[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (nb + i < N) ep.apply(row, nb + i, __uint_as_float(r[i]));
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
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

template <typename TO, bool A_K, bool B_K, int BN>
static int run(const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K, int splits,
               int kps, const Epilogue<TO>& ep, cudaStream_t s) {
  auto kern = gemm_tc_kernel<TO, A_K, B_K, BN>;
  constexpr int smem = Smem<BN>::TOTAL;
  static bool attr_set = false;
  if (!attr_set) {
    PPLL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set = true;
  }
  dim3 grid(ceil_div(N, BN), ceil_div(M, BM), splits);
  kern<<<grid, kThreads, smem, s>>>(ma, mb, M, N, K, kps, ep);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

template <typename TO, bool A_K, bool B_K>
static int dispatch_bn(int bn, const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K,
                       int splits, int kps, const Epilogue<TO>& ep, cudaStream_t s) {
  if (bn == 256) return run<TO, A_K, B_K, 256>(ma, mb, M, N, K, splits, kps, ep, s);
  if (bn == 128) return run<TO, A_K, B_K, 128>(ma, mb, M, N, K, splits, kps, ep, s);
  return run<TO, A_K, B_K, 64>(ma, mb, M, N, K, splits, kps, ep, s);
}

}  // namespace tc

template <typename TO>
int launch_gemm_tc(int M, int N, int K, const __nv_bfloat16* A, long lda, bool a_kmajor,
                   const __nv_bfloat16* B, long ldb, bool b_kmajor, const Epilogue<TO>& ep,
                   float* ws, size_t ws_elems, cudaStream_t s) {
  using namespace tc;
  // shapes the tensor-core tile cannot use efficiently go to the SIMT engine
  if (N < 32 || K < 16 || M < 1) return PPLL_ERR_UNSUPPORTED;
  if (((uintptr_t)A & 15) || ((uintptr_t)B & 15) || (lda * 2) % 16 || (ldb * 2) % 16)
    return PPLL_ERR_UNSUPPORTED;
  // tile width: widest that still gives >= ~1 wave of CTAs
  const int mt = ceil_div(M, BM);
  int bn = 256;
  while (bn > 64 && (long)mt * ceil_div(N, bn) < 120) bn >>= 1;
  const int tiles = mt * ceil_div(N, bn);
  int splits = 1;
  if (ws && tiles < 100 && K >= 4 * BK) {
    splits = min(148 / tiles, K / (2 * BK));
    while (splits > 1 && (size_t)splits * M * N > ws_elems) --splits;
    if (splits < 1) splits = 1;
  }
  int kps = ceil_div(ceil_div(K, splits), BK) * BK;
  splits = ceil_div(K, kps);

  CUtensorMap ma, mb;
  bool ok = a_kmajor ? make_map(&ma, A, K, M, lda, BM) : make_map(&ma, A, M, K, lda, 64);
  ok = ok && (b_kmajor ? make_map(&mb, B, K, N, ldb, bn) : make_map(&mb, B, N, K, ldb, 64));
  if (!ok) return PPLL_ERR_UNSUPPORTED;

  Epilogue<TO> e = ep;
  e.partial = splits > 1 ? ws : nullptr;
  int r;
  if (a_kmajor && !b_kmajor) r = dispatch_bn<TO, true, false>(bn, ma, mb, M, N, K, splits, kps, e, s);
  else if (a_kmajor && b_kmajor) r = dispatch_bn<TO, true, true>(bn, ma, mb, M, N, K, splits, kps, e, s);
  else if (!a_kmajor && !b_kmajor) r = dispatch_bn<TO, false, false>(bn, ma, mb, M, N, K, splits, kps, e, s);
  else r = dispatch_bn<TO, false, true>(bn, ma, mb, M, N, K, splits, kps, e, s);
  if (r || splits == 1) return r;
  return launch_splitk_reduce<TO>(M, N, splits, ws, ep, s);
}

template int launch_gemm_tc<float>(int, int, int, const __nv_bfloat16*, long, bool, const __nv_bfloat16*, long, bool, const Epilogue<float>&, float*, size_t, cudaStream_t);
template int launch_gemm_tc<__nv_bfloat16>(int, int, int, const __nv_bfloat16*, long, bool, const __nv_bfloat16*, long, bool, const Epilogue<__nv_bfloat16>&, float*, size_t, cudaStream_t);

}  // namespace ppll
