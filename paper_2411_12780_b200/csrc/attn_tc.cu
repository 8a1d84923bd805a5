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
#include <cudaTypedefs.h>
#include "common.cuh"
#include "kernels.cuh"
#include "vit.cuh"
#include "ptx.cuh"

namespace ppll {
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

// Warp transpose-reduce of 64 per-lane values: after 5 halving rounds lane L
// holds the warp-wide sums of columns col_of_lane(L) and col_of_lane(L) + 1.
__device__ __forceinline__ int col_of_lane(int L) {
  return ((L >> 4) & 1) * 32 + ((L >> 3) & 1) * 16 + ((L >> 2) & 1) * 8 + ((L >> 1) & 1) * 4 +
         (L & 1) * 2;
}
__device__ __forceinline__ float2 warp_colsum64(const float (&v)[64], int lane) {
  float a[32];
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float keep = hi ? v[j + 32] : v[j], send = hi ? v[j] : v[j + 32];
      a[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
  }
  float b[16];
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float keep = hi ? a[j + 16] : a[j], send = hi ? a[j] : a[j + 16];
      b[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
  }
  float c[8];
  {
    const bool hi = lane & 4;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float keep = hi ? b[j + 8] : b[j], send = hi ? b[j] : b[j + 8];
      c[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
  }
  float d[4];
  {
    const bool hi = lane & 2;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float keep = hi ? c[j + 4] : c[j], send = hi ? c[j] : c[j + 4];
      d[j] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
  }
  const bool hi = lane & 1;
  const float k0 = hi ? d[2] : d[0], s0 = hi ? d[0] : d[2];
  const float k1 = hi ? d[3] : d[1], s1 = hi ? d[1] : d[3];
  return make_float2(k0 + __shfl_xor_sync(0xffffffffu, s0, 1),
                     k1 + __shfl_xor_sync(0xffffffffu, s1, 1));
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
  // softmax: thread = query row (TMEM lane); keys in chunks of 16
  const int r = tid;
  const uint32_t lane_base = tm + ((uint32_t)(warp * 32) << 16);
  float mx = -INFINITY;
  for (int c = 0; c < NK; c += 16) {
    float v[16];
    ld16(lane_base + c, v);
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (c + i < Tn) mx = fmaxf(mx, v[i] * scale);
  }
  float sum = 0.f;
  const bool live = r < Tn;
  const int pkeys = small ? 64 : 128;   // P columns written (zeros past NK)
  for (int c = 0; c < pkeys; c += 16) {
    float v[16];
    if (c < NK) ld16(lane_base + c, v);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float e = (live && c + i < Tn) ? __expf(v[i] * scale - mx) : 0.f;
      v[i] = e;
      sum += e;
    }
    store_chunk16(sP, r, c >> 4, v);        // unnormalised; O is divided by the sum
  }
  if (live) lse[(long)blockIdx.x * Tn + r] = mx + logf(sum);
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
__global__ void __launch_bounds__(128, 2)
attn_tc_bwd_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                   const __grid_constant__ CUtensorMap mdo, int Tn, int H, int NK,
                   const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                   const float* __restrict__ lse, __nv_bfloat16* __restrict__ dqkv, float scale,
                   float* __restrict__ bias_part) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base0 = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + ((1024 - (base0 & 1023)) & 1023);
  // ~107 KB so two CTAs share an SM: K holds only its NK rows, and V (dead
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
  const int row0 = b * Tn;
  // TMEM columns: S [0,128), dP [128,256); later dV [0,64), dK [64,128), dQ [128,192)
  if (tid == 0) {
    mbar_expect_tx(&bar[0], 2 * 16384 + 2 * NK * 128);
    tma_load_2d(&mq, &bar[0], sQ, h * kDh, row0);
    tma_load_2d(&mk, &bar[0], sK, D + h * kDh, row0);
    tma_load_2d(&mk, &bar[0], sV, 2 * D + h * kDh, row0);
    tma_load_2d(&mdo, &bar[0], sdO, h * kDh, row0);
    mbar_wait(&bar[0], 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t id = idesc(128, NK, false, false);
    const uint32_t aq = smem_u32(sQ), ak = smem_u32(sK), av = smem_u32(sV), ad = smem_u32(sdO);
#pragma unroll
    for (int j = 0; j < kDh / 16; ++j) mma_bf16(tm, kmaj_tile(aq, j), kmaj_tile(ak, j), id, j > 0);
#pragma unroll
    for (int j = 0; j < kDh / 16; ++j) mma_bf16(tm + 128, kmaj_tile(ad, j), kmaj_tile(av, j), id, j > 0);
    mma_commit(&bar[1]);
  }
  // D_i = rowsum(dO ⊙ O) from global rows while the MMAs run
  const int r = tid;
  float Di = 0.f;
  if (r < Tn) {
    const __nv_bfloat16* orow = o + (long)(row0 + r) * D + h * kDh;
    const __nv_bfloat16* grow = dout + (long)(row0 + r) * D + h * kDh;
    float a[32], g[32];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      ld_row32<__nv_bfloat16>(orow + 32 * half, true, 32, a);
      ld_row32<__nv_bfloat16>(grow + 32 * half, true, 32, g);
#pragma unroll
      for (int i = 0; i < 32; ++i) Di = fmaf(a[i], g[i], Di);
    }
  }
  const float lr = r < Tn ? lse[(long)blockIdx.x * Tn + r] : 0.f;
  mbar_wait(&bar[1], 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t lane_base = tm + ((uint32_t)(warp * 32) << 16);
  const bool live = r < Tn;
  for (int c = 0; c < 128; c += 16) {
    float p[16], ds[16];
    if (c < NK) {
      ld16(lane_base + c, p);
      ld16(lane_base + 128 + c, ds);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float pv = (live && c + i < Tn) ? __expf(p[i] * scale - lr) : 0.f;
      ds[i] = pv * (ds[i] - Di);
      p[i] = pv;
    }
    store_chunk16(sP, r, c >> 4, p);
    store_chunk16(sdS, r, c >> 4, ds);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t ap = smem_u32(sP), as = smem_u32(sdS);
    const uint32_t aq = smem_u32(sQ), ak = smem_u32(sK), ad = smem_u32(sdO);
    const uint32_t id_mn = idesc(128, kDh, true, true);
    // dV = Pᵀ·dO  (M = keys, K = queries)
    for (int j = 0; j < 8; ++j) mma_bf16(tm + 0, mnmaj_rows(ap, j), mnmaj_tile(ad, j), id_mn, j > 0);
    // dK = dSᵀ·Q
    for (int j = 0; j < 8; ++j) mma_bf16(tm + 64, mnmaj_rows(as, j), mnmaj_tile(aq, j), id_mn, j > 0);
    // dQ = dS·K   (M = queries, K = keys)
    const uint32_t id_k = idesc(128, kDh, false, true);
    for (int j = 0; j < NK / 16; ++j) mma_bf16(tm + 128, kmaj_keys(as, j), mnmaj_tile(ak, j), id_k, j > 0);
    mma_commit(&bar[1]);
  }
  mbar_wait(&bar[1], 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const long ld = 3L * D;
  float v[64];
  // lane r holds: dV[key r], dK[key r], dQ[query r]
#pragma unroll
  for (int part = 0; part < 3; ++part) {
    const uint32_t col = part == 0 ? 0u : (part == 1 ? 64u : 128u);
#pragma unroll
    for (int c = 0; c < 64; c += 16) ld16(lane_base + col + c, v + c);
    const float sc = part == 0 ? 1.f : scale;
    const int off = part == 0 ? 2 * D : (part == 1 ? D : 0);
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = r < Tn ? v[i] * sc : 0.f;
    if (r < Tn) {
      __nv_bfloat16* dst = dqkv + (long)(row0 + r) * ld + off + h * kDh;
      float v32[32];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v32[i] = v[32 * hh + i];
        st_row32<__nv_bfloat16>(dst + 32 * hh, true, 32, v32);
      }
    }
    if (bias_part) {
      // fused bias gradient: Σ over this image's rows of the 64 columns, as a
      // warp transpose-reduce (lane keeps 2 columns) then a fixed-order sum of
      // the 4 warps; partial row b of a [batch, 3D] matrix
      float2 cs = warp_colsum64(v, r & 31);
      float* red = reinterpret_cast<float*>(sP);
      const int cb = col_of_lane(r & 31);
      red[warp * 64 + cb] = cs.x;
      red[warp * 64 + cb + 1] = cs.y;
      __syncthreads();
      if (tid < 64)
        bias_part[(long)b * ld + off + h * kDh + tid] =
            ((red[tid] + red[64 + tid]) + red[128 + tid]) + red[192 + tid];
      __syncthreads();
    }
  }
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
constexpr int kBwdSmem = 16384 * 3 + 32768 * 2 + 1024 + 64;   // upper bound (NK = 128)
inline int bwd_smem(int NK) { return 16384 * 2 + ((NK * 128 + 1023) & ~1023) + 32768 * 2 + 1024 + 64; }

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
  CUtensorMap mq, mk, md;
  if (!map2d(&mq, qkv, 3L * D, (long)B * Tn, 3L * D, 128) ||
      !map2d(&mk, qkv, 3L * D, (long)B * Tn, 3L * D, NK) ||
      !map2d(&md, dout, (long)D, (long)B * Tn, (long)D, 128)) {
    set_error("attention: tensor map encode failed");
    return PPLL_ERR_CUDA;
  }
  static bool set = false;
  if (!set) {
    PPLL_CUDA_CHECK(cudaFuncSetAttribute(attn_tc_bwd_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem));
    set = true;
  }
  launch_k(attn_tc_bwd_kernel, B * H, 128, bwd_smem(NK), s, mq, mk, md, Tn, H, NK, o, dout, lse, dqkv,
                                                  1.0f / sqrtf((float)kDh), bias_part);
  note_launch();
  PPLL_LAUNCH_CHECK();
  return PPLL_OK;
}

}  // namespace ppll

extern "C" void ppll_set_attn_engine(int engine) { ppll::g_attn_engine = engine; }
