// Internal launcher declarations shared by capi.cu / stage.cu / gemm_tc.cu.
#pragma once
#include "common.cuh"

namespace ppll {

void note_launch(int n = 1);

// kActGeluD: GELU whose `pre` output receives gelu'(pre-activation) instead of
// the pre-activation itself, so the backward multiplies (kMaskMul) instead of
// re-evaluating erf/exp in the dgrad epilogue.
enum Act : int { kActNone = 0, kActRelu = 1, kActGelu = 2, kActGeluD = 3 };
enum MaskMode : int { kMaskNone = 0, kMaskRelu = 1, kMaskGeluGrad = 2, kMaskMul = 3 };

// Exact-erf GELU and its derivative sharing one exponential:
//   erf(z) = 1 - t·P(t)·e^{-z²}, t = 1/(1 + p|z|)   (Abramowitz-Stegun 7.1.26,
//   |error| <= 1.5e-7, i.e. fp32-level for the GELU),  z = x/√2,
//   gelu = x·Φ(x),  gelu' = Φ(x) + x·φ(x),  φ(x) = e^{-z²}/√(2π).
// Two MUFU ops (rcp, ex2; approx.ftz: ~1 ulp, no range fix-ups) + 13 FP ops.
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void gelu_both(float x, float& g, float& d) {
  const float t = rcp_approx(fmaf(0.3275911f * 0.70710678118654752f, fabsf(x), 1.f));
  float p = fmaf(t, 1.061405429f, -1.453152027f);
  p = fmaf(t, p, 1.421413741f);
  p = fmaf(t, p, -0.284496736f);
  p = fmaf(t, p, 0.254829592f);
  p *= t;
  const float e = ex2_approx(x * x * -0.72134752044448170f);   // e^{-x²/2}
  const float h = 0.5f * fmaf(-p, e, 1.f);                       // erf(|z|)/2
  const float cdf = x >= 0.f ? 0.5f + h : 0.5f - h;
  g = x * cdf;
  d = fmaf(x, 0.3989422804014327f * e, cdf);
}

// Packed fp32x2 arithmetic (sm_100 FFMA2 / FMUL2 / FADD2: two lanes per
// instruction) for the epilogue's per-element math.
struct f2 { float x, y; };
__device__ __forceinline__ f2 ffma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
__device__ __forceinline__ f2 fmul2(f2 a, f2 b) {
  f2 r;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ f2 fadd2(f2 a, f2 b) {
  f2 r;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ f2 splat2(float c) { return f2{c, c}; }
// gelu_both on two elements: the polynomial and the products run packed,
// rcp / ex2 stay scalar MUFU ops.
__device__ __forceinline__ void gelu_both2(float& x0, float& x1, float& d0, float& d1) {
  const f2 x{x0, x1};
  const f2 ax{fabsf(x0), fabsf(x1)};
  const f2 den = ffma2(splat2(0.3275911f * 0.70710678118654752f), ax, splat2(1.f));
  const f2 t{rcp_approx(den.x), rcp_approx(den.y)};
  f2 p = ffma2(t, splat2(1.061405429f), splat2(-1.453152027f));
  p = ffma2(t, p, splat2(1.421413741f));
  p = ffma2(t, p, splat2(-0.284496736f));
  p = ffma2(t, p, splat2(0.254829592f));
  p = fmul2(p, t);
  const f2 q = fmul2(fmul2(x, x), splat2(-0.72134752044448170f));
  const f2 e{ex2_approx(q.x), ex2_approx(q.y)};
  const f2 h = ffma2(fmul2(p, e), splat2(-0.5f), splat2(0.5f));      // erf(|z|)/2
  const f2 hs{copysignf(h.x, x0), copysignf(h.y, x1)};
  const f2 cdf = fadd2(hs, splat2(0.5f));
  const f2 g = fmul2(x, cdf);
  const f2 d = ffma2(x, fmul2(e, splat2(0.3989422804014327f)), cdf);
  x0 = g.x; x1 = g.y; d0 = d.x; d1 = d.y;
}
__device__ __forceinline__ float gelu_f(float x) {        // exact (erf) GELU
  float g, d;
  gelu_both(x, g, d);
  return g;
}
__device__ __forceinline__ float gelu_grad_f(float x) {   // d/dx gelu(x)
  float g, d;
  gelu_both(x, g, d);
  return d;
}

template <typename T>
__device__ __forceinline__ void ld_row32(const T* p, bool vec, int valid, float (&o)[32]);
template <>
__device__ __forceinline__ void ld_row32<float>(const float* p, bool vec, int valid, float (&o)[32]) {
  if (vec && valid == 32) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 q = reinterpret_cast<const float4*>(p)[i];
      o[4 * i] = q.x; o[4 * i + 1] = q.y; o[4 * i + 2] = q.z; o[4 * i + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] = i < valid ? p[i] : 0.f;
  }
}
template <>
__device__ __forceinline__ void ld_row32<__nv_bfloat16>(const __nv_bfloat16* p, bool vec, int valid,
                                                        float (&o)[32]) {
  if (vec && valid == 32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 q = reinterpret_cast<const uint4*>(p)[i];
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        o[8 * i + 2 * j] = f.x;
        o[8 * i + 2 * j + 1] = f.y;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] = i < valid ? __bfloat162float(p[i]) : 0.f;
  }
}
// NV consecutive elements (NV % 8 == 0), 16-B vectors when `vec` and all valid
template <int NV>
__device__ __forceinline__ void ld_rowN(const float* p, bool vec, int valid, float (&o)[NV]) {
  if (vec && valid == NV) {
#pragma unroll
    for (int i = 0; i < NV / 4; ++i) {
      const float4 q = reinterpret_cast<const float4*>(p)[i];
      o[4 * i] = q.x; o[4 * i + 1] = q.y; o[4 * i + 2] = q.z; o[4 * i + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < NV; ++i) o[i] = i < valid ? p[i] : 0.f;
  }
}
template <int NV>
__device__ __forceinline__ void ld_rowN(const __nv_bfloat16* p, bool vec, int valid, float (&o)[NV]) {
  if (vec && valid == NV) {
#pragma unroll
    for (int i = 0; i < NV / 8; ++i) {
      const uint4 q = reinterpret_cast<const uint4*>(p)[i];
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        o[8 * i + 2 * j] = f.x;
        o[8 * i + 2 * j + 1] = f.y;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < NV; ++i) o[i] = i < valid ? __bfloat162float(p[i]) : 0.f;
  }
}

template <typename T>
__device__ __forceinline__ void st_row32(T* p, bool vec, int valid, const float (&v)[32]);
template <>
__device__ __forceinline__ void st_row32<float>(float* p, bool vec, int valid, const float (&v)[32]) {
  if (vec && valid == 32) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      reinterpret_cast<float4*>(p)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < valid) p[i] = v[i];
  }
}
template <>
__device__ __forceinline__ void st_row32<__nv_bfloat16>(__nv_bfloat16* p, bool vec, int valid,
                                                        const float (&v)[32]) {
  if (vec && valid == 32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint4 q;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
      for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[8 * i + 2 * j], v[8 * i + 2 * j + 1]);
      reinterpret_cast<uint4*>(p)[i] = q;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < valid) p[i] = __float2bfloat16_rn(v[i]);
  }
}

// Coalesced store of a warp's 32x32 output block (thread = one row, 32
// consecutive columns in registers, as tcgen05.ld 32x32b delivers them).
// The block is transposed through a 2-KB per-warp shared-memory buffer (rows
// of 64 B, 16-B chunks XOR-swizzled by (row>>1)&3 so both the row-wise writes
// and the column-wise reads are bank-conflict free), then each store
// instruction covers 8 rows x 64 contiguous bytes (full 32-B sectors) instead
// of 32 rows x 16 B.  fp32 goes in two 16-column halves.  Up to two outputs
// (the dual store of the ring push) share one transpose.
// `csum` (optional): this 32-row block's column sums of the stored (rounded)
// values, rows >= M excluded, written as one partial row csum[n0 .. n0+31]
// (a fused bias-gradient Σ_rows; reduced over the row blocks afterwards).
template <typename TO, bool kFull = false>
__device__ __forceinline__ void warp_store_block32(TO* out, long ld, TO* out2, long ld2, int row0,
                                                   int M, int n0, int N, bool vec,
                                                   const float (&v)[32], uint8_t* stg, int lane,
                                                   float* csum = nullptr) {
  constexpr int kEl = 16 / (int)sizeof(TO);          // elements per 16-B chunk
  constexpr int kPasses = sizeof(TO) == 4 ? 2 : 1;   // 64-B row slices per 32 columns
  constexpr int kCols = 32 / kPasses;                // columns per pass
#pragma unroll
  for (int p = 0; p < kPasses; ++p) {
    // write: this lane's row, 4 chunks of 16 B
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint4 q;
      if constexpr (sizeof(TO) == 4) {
        q = make_uint4(__float_as_uint(v[p * kCols + 4 * j]), __float_as_uint(v[p * kCols + 4 * j + 1]),
                       __float_as_uint(v[p * kCols + 4 * j + 2]), __float_as_uint(v[p * kCols + 4 * j + 3]));
      } else {
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          h[e] = __floats2bfloat162_rn(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
      }
      const int sj = j ^ ((lane >> 1) & 3);
      *reinterpret_cast<uint4*>(stg + lane * 64 + sj * 16) = q;
    }
    __syncwarp();
    // read: 8 rows x 4 chunks per instruction, 4 instructions
    float cs[kEl];
#pragma unroll
    for (int e = 0; e < kEl; ++e) cs[e] = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = i * 8 + (lane >> 2), c = lane & 3;
      const uint4 q = *reinterpret_cast<const uint4*>(stg + r * 64 + ((c ^ ((r >> 1) & 3)) * 16));
      const int row = row0 + r;
      const int col = n0 + p * kCols + c * kEl;
      if (csum && (kFull || row < M)) {
        const TO* e = reinterpret_cast<const TO*>(&q);
#pragma unroll
        for (int t = 0; t < kEl; ++t) cs[t] += to_f(e[t]);
      }
      if constexpr (kFull) {
        *reinterpret_cast<uint4*>(out + (long)row * ld + col) = q;
        if (out2) *reinterpret_cast<uint4*>(out2 + (long)row * ld2 + col) = q;
      } else if (row < M && col < N) {
        if (vec && col + kEl <= N) {
          *reinterpret_cast<uint4*>(out + (long)row * ld + col) = q;
          if (out2) *reinterpret_cast<uint4*>(out2 + (long)row * ld2 + col) = q;
        } else {
          const TO* e = reinterpret_cast<const TO*>(&q);
          for (int t = 0; t < kEl && col + t < N; ++t) {
            out[(long)row * ld + col + t] = e[t];
            if (out2) out2[(long)row * ld2 + col + t] = e[t];
          }
        }
      }
    }
    if (csum && row0 < M) {   // lanes with equal (lane & 3) hold the same columns
#pragma unroll
      for (int t = 0; t < kEl; ++t) {
        cs[t] += __shfl_xor_sync(0xffffffffu, cs[t], 4);
        cs[t] += __shfl_xor_sync(0xffffffffu, cs[t], 8);
        cs[t] += __shfl_xor_sync(0xffffffffu, cs[t], 16);
      }
      const int col = n0 + p * kCols + (lane & 3) * kEl;
      if (lane < 4) {
        for (int t = 0; t < kEl; ++t)
          if (col + t < N) csum[col + t] = cs[t];
      }
    }
    __syncwarp();
  }
}

// The same 32-row x 16-column block written by the TMA engine: the lanes put
// it into the warp's 1-KB buffer in the 32-B-swizzled layout of a
// {32 B, 32 rows} box (rows of 32 B, 16-B halves swapped on every other group
// of four rows: conflict-free STS.128), then one lane issues a bulk tensor
// store.  Rows >= M / columns >= N are clipped by the tensor map, so ragged
// tiles need no tests.  Before the buffer is rewritten the previous bulk store
// must have finished READING it (wait_group.read); global completion is
// awaited once at kernel exit (tma_store_drain).
template <typename TO>
__device__ __forceinline__ void warp_store_tma16(const void* map, int row0, int n0,
                                                 const float (&v)[16], uint8_t* stg, int lane) {
  constexpr int kPasses = sizeof(TO) == 4 ? 2 : 1;
  constexpr int kCols = 16 / kPasses;
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(stg));
#pragma unroll
  for (int p = 0; p < kPasses; ++p) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      uint4 q;
      if constexpr (sizeof(TO) == 4) {
        q = make_uint4(__float_as_uint(v[p * kCols + 4 * j]), __float_as_uint(v[p * kCols + 4 * j + 1]),
                       __float_as_uint(v[p * kCols + 4 * j + 2]), __float_as_uint(v[p * kCols + 4 * j + 3]));
      } else {
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          h[e] = __floats2bfloat162_rn(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
      }
      const int sj = j ^ ((lane >> 2) & 1);
      *reinterpret_cast<uint4*>(stg + lane * 32 + sj * 16) = q;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile(
          "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
              reinterpret_cast<uint64_t>(map)),
          "r"(n0 + p * kCols), "r"(row0), "r"(sa)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
}
// at exit only the shared-memory source must have been read (the CTA's smem
// is released); the global writes complete with the grid, before any
// dependent grid passes griddepcontrol.wait or the stream moves on
// (PPLL_GEMM_DRAIN_FULL=1 restores the full wait_group 0)
__device__ __forceinline__ void tma_store_drain(int lane, int full = 0) {
  if (lane == 0) {
    if (full) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncwarp();
}

// Coalesced store of a warp's 32-row x 16-column block (thread = one row, 16
// consecutive columns in registers, as tcgen05.ld 32x32b.x16 delivers them),
// transposed through a 1-KB per-warp buffer: rows of 32 B (two 16-B chunks,
// swapped on every other group of four rows so both the row-wise writes and
// the column-wise reads are bank-conflict free); each store instruction then
// covers 16 rows x 32 contiguous bytes (one full sector per row).  fp32 goes
// in two 8-column passes.  `csum` as in warp_store_block32.
// kFull: the block lies inside [M, N] and `vec` holds — no bounds tests.
template <typename TO, bool kFull = false>
__device__ __forceinline__ void warp_store_block16(TO* out, long ld, TO* out2, long ld2, int row0,
                                                   int M, int n0, int N, bool vec,
                                                   const float (&v)[16], uint8_t* stg, int lane,
                                                   float* csum = nullptr) {
  constexpr int kEl = 16 / (int)sizeof(TO);          // elements per 16-B chunk
  constexpr int kPasses = sizeof(TO) == 4 ? 2 : 1;   // 32-B row slices per 16 columns
  constexpr int kCols = 16 / kPasses;                // columns per pass
#pragma unroll
  for (int p = 0; p < kPasses; ++p) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      uint4 q;
      if constexpr (sizeof(TO) == 4) {
        q = make_uint4(__float_as_uint(v[p * kCols + 4 * j]), __float_as_uint(v[p * kCols + 4 * j + 1]),
                       __float_as_uint(v[p * kCols + 4 * j + 2]), __float_as_uint(v[p * kCols + 4 * j + 3]));
      } else {
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          h[e] = __floats2bfloat162_rn(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
      }
      const int sj = j ^ ((lane >> 2) & 1);
      *reinterpret_cast<uint4*>(stg + lane * 32 + sj * 16) = q;
    }
    __syncwarp();
    float cs[kEl];
#pragma unroll
    for (int e = 0; e < kEl; ++e) cs[e] = 0.f;
    // both shared-memory reads before any global store: the stores then do
    // not serialise on the reused source registers
    uint4 qs[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int r = i * 16 + (lane >> 1), c = lane & 1;
      qs[i] = *reinterpret_cast<const uint4*>(stg + r * 32 + ((c ^ ((r >> 2) & 1)) * 16));
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int r = i * 16 + (lane >> 1), c = lane & 1;
      const uint4 q = qs[i];
      const int row = row0 + r;
      const int col = n0 + p * kCols + c * kEl;
      if (csum && (kFull || row < M)) {
        const TO* e = reinterpret_cast<const TO*>(&q);
#pragma unroll
        for (int t = 0; t < kEl; ++t) cs[t] += to_f(e[t]);
      }
      if constexpr (kFull) {
        *reinterpret_cast<uint4*>(out + (long)row * ld + col) = q;
        if (out2) *reinterpret_cast<uint4*>(out2 + (long)row * ld2 + col) = q;
      } else if (row < M && col < N) {
        if (vec && col + kEl <= N) {
          *reinterpret_cast<uint4*>(out + (long)row * ld + col) = q;
          if (out2) *reinterpret_cast<uint4*>(out2 + (long)row * ld2 + col) = q;
        } else {
          const TO* e = reinterpret_cast<const TO*>(&q);
          for (int t = 0; t < kEl && col + t < N; ++t) {
            out[(long)row * ld + col + t] = e[t];
            if (out2) out2[(long)row * ld2 + col + t] = e[t];
          }
        }
      }
    }
    if (csum && row0 < M) {   // lanes with equal (lane & 1) hold the same columns
#pragma unroll
      for (int t = 0; t < kEl; ++t) {
        cs[t] += __shfl_xor_sync(0xffffffffu, cs[t], 2);
        cs[t] += __shfl_xor_sync(0xffffffffu, cs[t], 4);
        cs[t] += __shfl_xor_sync(0xffffffffu, cs[t], 8);
        cs[t] += __shfl_xor_sync(0xffffffffu, cs[t], 16);
      }
      const int col = n0 + p * kCols + (lane & 1) * kEl;
      if (lane < 2) {
        for (int t = 0; t < kEl; ++t)
          if (col + t < N) csum[col + t] = cs[t];
      }
    }
    __syncwarp();
  }
}

// Coalesced load of a warp's 32-row x 16-column bf16 block into thread-row
// registers (the inverse of warp_store_block16): issue() puts 16 rows x 32 B
// per instruction in flight (full sectors), finish() transposes them through
// the same 1-KB swizzled buffer so lane r holds row r's 16 values.
__device__ __forceinline__ void blk16_issue(const __nv_bfloat16* src, long ld, int row0, int M,
                                            int n0, int N, bool vec, uint4 (&q)[2], int lane) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = i * 16 + (lane >> 1), c = lane & 1;
    const int row = row0 + r, col = n0 + c * 8;
    q[i] = make_uint4(0u, 0u, 0u, 0u);
    if (row < M && col < N) {
      const __nv_bfloat16* p = src + (long)row * ld + col;
      if (vec && col + 8 <= N) {
        q[i] = *reinterpret_cast<const uint4*>(p);
      } else {
        __nv_bfloat16* e = reinterpret_cast<__nv_bfloat16*>(&q[i]);
        for (int t = 0; t < 8 && col + t < N; ++t) e[t] = p[t];
      }
    }
  }
}
__device__ __forceinline__ void blk16_finish(const uint4 (&q)[2], float (&k)[16], uint8_t* stg,
                                             int lane) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = i * 16 + (lane >> 1), c = lane & 1;
    *reinterpret_cast<uint4*>(stg + r * 32 + ((c ^ ((r >> 2) & 1)) * 16)) = q[i];
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const uint4 t = *reinterpret_cast<const uint4*>(stg + lane * 32 + ((j ^ ((lane >> 2) & 1)) * 16));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&t);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      k[8 * j + 2 * e] = f.x;
      k[8 * j + 2 * e + 1] = f.y;
    }
  }
  __syncwarp();
}

// bf16-output GELU pair on the tanh form (one MUFU tanh per element, packed
// FP32x2 arithmetic):  u = √(2/π)(x + 0.044715x³),  gelu = ½x(1 + tanh u),
// gelu' = ½(1 + t) + ½x(1 − t²)·√(2/π)(1 + 0.134145x²).  Its distance to the
// erf GELU (≤ 5e-4 absolute, tanh.approx included) is far below the bf16
// resolution of the stored activations; fp32 outputs keep gelu_both2 (erf).
__device__ __forceinline__ float tanh_approx(float x) {
  float r;
  asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void gelu_tanh2(float& x0, float& x1, float& d0, float& d1) {
  const f2 x{x0, x1};
  const f2 x2 = fmul2(x, x);
  const f2 p = ffma2(x2, splat2(0.0356774081363001f), splat2(0.7978845608028654f));
  const f2 u = fmul2(x, p);
  const f2 t{tanh_approx(u.x), tanh_approx(u.y)};
  const f2 hx = fmul2(x, splat2(0.5f));
  const f2 g = ffma2(hx, t, hx);
  const f2 omt = ffma2(t, f2{-t.x, -t.y}, splat2(1.f));
  const f2 q = ffma2(x2, splat2(0.1070322244089003f), splat2(0.7978845608028654f));
  const f2 d = ffma2(fmul2(hx, omt), q, ffma2(t, splat2(0.5f), splat2(0.5f)));
  x0 = g.x; x1 = g.y; d0 = d.x; d1 = d.y;
}

// Compile-time epilogue specialisations of the tcgen05 engine (the runtime
// flag tests of the generic form cost ~40% of the epilogue's instructions).
enum EpiF : int {
  kEFBias = 1, kEFRes = 2, kEFRelu = 4, kEFGeluD = 8, kEFMaskRelu = 16, kEFMaskMul = 32,
  kEFGeneric = 1 << 10
};

// GEMM epilogue:
//   v -> (+bias[n]) -> (+R[m,n]) -> [store pre-activation P] -> act (ReLU|GELU)
//     -> ReLU mask (v·[mask>0]) | GELU gradient (v·gelu'(mask)) | v·mask -> C (and C2)
//   (act GeluD: P receives gelu'(pre-activation) instead)
// `vec` = every pointer 16-B aligned and every leading dimension a multiple of
// 16 B, so 32-column row segments move as 16-B vectors.
template <typename TO>
struct Epilogue {
  TO* C = nullptr;
  long ldc = 0;
  TO* C2 = nullptr;       // optional dual store (fused ring push)
  long ldc2 = 0;
  const float* bias = nullptr;
  int act = kActNone;
  const TO* mask = nullptr;
  long ldmask = 0;
  int mask_mode = kMaskNone;
  const TO* res = nullptr;   // residual added before the activation
  long ldres = 0;
  TO* pre = nullptr;         // pre-activation store (GELU backward)
  long ldpre = 0;
  int ncols = 0;             // N (for row-segment bounds)
  int vec = 0;
  float* partial = nullptr;  // split-K workspace (internal)
  float* cs_part = nullptr;  // fused column sums: [ceil(M/32)][ncols] partial rows (or null)
  float* colsum_b = nullptr; // weight-gradient GEMMs: Σ_k B(k, n) (bias gradient), if fused

  __device__ __forceinline__ float act_f(float v) const {
    if (act == kActRelu) return fmaxf(v, 0.f);
    if (act == kActGelu || act == kActGeluD) return gelu_f(v);
    return v;
  }
  __device__ __forceinline__ void apply(int m, int n, float v) const {
    if (bias) v += bias[n];
    if (res) v += to_f(res[(long)m * ldres + n]);
    if (pre) DT<TO>::st(pre + (long)m * ldpre + n, act == kActGeluD ? gelu_grad_f(v) : v);
    v = act_f(v);
    if (mask_mode == kMaskRelu) v = (to_f(mask[(long)m * ldmask + n]) > 0.f) ? v : 0.f;
    else if (mask_mode == kMaskGeluGrad) v *= gelu_grad_f(to_f(mask[(long)m * ldmask + n]));
    else if (mask_mode == kMaskMul) v *= to_f(mask[(long)m * ldmask + n]);
    DT<TO>::st(C + (long)m * ldc + n, v);
    if (C2) DT<TO>::st(C2 + (long)m * ldc2 + n, v);
  }
  // Split form used by the tensor-core epilogue: issue the residual / mask row
  // loads first (they overlap the TMEM load), then finish with the bias taken
  // from a shared-memory copy of the tile's bias slice.
  __device__ __forceinline__ void load_aux32(int m, int n0, float (&r)[32], float (&k)[32]) const {
    const int valid = min(32, ncols - n0);
    if (res) ld_row32<TO>(res + (long)m * ldres + n0, vec != 0, valid, r);
    if (mask_mode != kMaskNone) ld_row32<TO>(mask + (long)m * ldmask + n0, vec != 0, valid, k);
  }
  // activation (with the GeluD derivative written into d) and mask, in place
  // activation (with the GeluD derivative written into d) and mask, in place.
  // One GELU evaluation per element: on v (act GELU/GeluD) or on the mask
  // (GELU-gradient mask); the two are never combined (host-checked).
  template <int NV>
  __device__ __forceinline__ void act_mask(float (&v)[NV], const float (&k)[NV],
                                           float (&d)[NV]) const {
    const bool ga = act == kActGelu || act == kActGeluD;
    if (ga) {
#pragma unroll
      for (int i = 0; i < NV; i += 2) gelu_both2(v[i], v[i + 1], d[i], d[i + 1]);
    } else if (mask_mode == kMaskGeluGrad) {
#pragma unroll
      for (int i = 0; i < NV; i += 2) {
        float g0 = k[i], g1 = k[i + 1];
        gelu_both2(g0, g1, d[i], d[i + 1]);
        const f2 r = fmul2(f2{v[i], v[i + 1]}, f2{d[i], d[i + 1]});
        v[i] = r.x; v[i + 1] = r.y;
      }
    } else if (act == kActRelu) {
#pragma unroll
      for (int i = 0; i < NV; ++i) v[i] = fmaxf(v[i], 0.f);
    }
    if (mask_mode == kMaskRelu) {
#pragma unroll
      for (int i = 0; i < NV; ++i) v[i] = k[i] > 0.f ? v[i] : 0.f;
    } else if (mask_mode == kMaskMul) {
#pragma unroll
      for (int i = 0; i < NV; i += 2) {
        const f2 r = fmul2(f2{v[i], v[i + 1]}, f2{k[i], k[i + 1]});
        v[i] = r.x; v[i + 1] = r.y;
      }
    }
  }
  // Warp-cooperative epilogue of a 32-row x 32-column block (rows
  // row0..row0+31, one per lane; rows >= M are computed but not stored):
  // every store goes through warp_store_block32.  `r` (the residual) is dead
  // after the add and is reused for the GeluD derivative.
  __device__ __forceinline__ void finish_block32(int row0, int M, int n0, float (&v)[32],
                                                 float (&r)[32], const float (&k)[32],
                                                 const float* bias_s, uint8_t* stg,
                                                 int lane) const {
    const bool vv = vec != 0;
    if (bias) {
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const float2 bb = *reinterpret_cast<const float2*>(bias_s + i);
        const f2 t = fadd2(f2{v[i], v[i + 1]}, f2{bb.x, bb.y});
        v[i] = t.x; v[i + 1] = t.y;
      }
    }
    if (res) {
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const f2 t = fadd2(f2{v[i], v[i + 1]}, f2{r[i], r[i + 1]});
        v[i] = t.x; v[i + 1] = t.y;
      }
    }
    if (pre && act != kActGeluD)
      warp_store_block32<TO>(pre, ldpre, nullptr, 0, row0, M, n0, ncols, vv, v, stg, lane);
    act_mask<32>(v, k, r);
    if (pre && act == kActGeluD)
      warp_store_block32<TO>(pre, ldpre, nullptr, 0, row0, M, n0, ncols, vv, r, stg, lane);
    warp_store_block32<TO>(C, ldc, C2, ldc2, row0, M, n0, ncols, vv, v, stg, lane,
                           cs_part ? cs_part + (long)(row0 >> 5) * ncols : nullptr);
  }

  // 16-column forms used by the tcgen05 engine (tcgen05.ld 32x32b.x16 chunks)
  __device__ __forceinline__ void load_aux16(int m, int n0, float (&r)[16], float (&k)[16]) const {
    const int valid = min(16, ncols - n0);
    if (res) ld_rowN<16>(res + (long)m * ldres + n0, vec != 0, valid, r);
    if (mask_mode != kMaskNone) ld_rowN<16>(mask + (long)m * ldmask + n0, vec != 0, valid, k);
  }
  __device__ __forceinline__ void finish_block16(int row0, int M, int n0, float (&v)[16],
                                                 float (&r)[16], const float (&k)[16],
                                                 const float* bias_s, uint8_t* stg,
                                                 int lane) const {
    const bool vv = vec != 0;
    if (bias) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const float2 bb = *reinterpret_cast<const float2*>(bias_s + i);
        const f2 t = fadd2(f2{v[i], v[i + 1]}, f2{bb.x, bb.y});
        v[i] = t.x; v[i + 1] = t.y;
      }
    }
    if (res) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const f2 t = fadd2(f2{v[i], v[i + 1]}, f2{r[i], r[i + 1]});
        v[i] = t.x; v[i + 1] = t.y;
      }
    }
    if (pre && act != kActGeluD)
      warp_store_block16<TO>(pre, ldpre, nullptr, 0, row0, M, n0, ncols, vv, v, stg, lane);
    act_mask<16>(v, k, r);
    if (pre && act == kActGeluD)
      warp_store_block16<TO>(pre, ldpre, nullptr, 0, row0, M, n0, ncols, vv, r, stg, lane);
    warp_store_block16<TO>(C, ldc, C2, ldc2, row0, M, n0, ncols, vv, v, stg, lane,
                           cs_part ? cs_part + (long)(row0 >> 5) * ncols : nullptr);
  }

  // specialised forms (F = EpiF bits, or kEFGeneric -> the runtime forms);
  // C2 (ring push) and cs_part (fused column sums) stay runtime options
  // bf16 specialisations: coalesced block loads issued before the TMEM load
  // (aux_issue) and transposed into thread rows after it (aux_finish)
  template <int F>
  static constexpr bool kBlockAux = F != kEFGeneric && sizeof(TO) == 2 &&
                                    (F & (kEFRes | kEFMaskRelu | kEFMaskMul)) != 0;
  template <int F>
  __device__ __forceinline__ void aux_issue(int row0, int M, int n0, uint4 (&qr)[2],
                                            uint4 (&qk)[2], int lane) const {
    if constexpr (kBlockAux<F>) {
      if constexpr ((F & kEFRes) != 0)
        blk16_issue(reinterpret_cast<const __nv_bfloat16*>(res), ldres, row0, M, n0, ncols,
                    vec != 0, qr, lane);
      if constexpr ((F & (kEFMaskRelu | kEFMaskMul)) != 0)
        blk16_issue(reinterpret_cast<const __nv_bfloat16*>(mask), ldmask, row0, M, n0, ncols,
                    vec != 0, qk, lane);
    }
  }
  template <int F>
  __device__ __forceinline__ void aux_finish(const uint4 (&qr)[2], const uint4 (&qk)[2],
                                             float (&r)[16], float (&k)[16], uint8_t* stg,
                                             int lane) const {
    if constexpr (kBlockAux<F>) {
      if constexpr ((F & kEFRes) != 0) blk16_finish(qr, r, stg, lane);
      if constexpr ((F & (kEFMaskRelu | kEFMaskMul)) != 0) blk16_finish(qk, k, stg, lane);
    }
  }
  template <int F>
  __device__ __forceinline__ void load_aux16_t(int m, int n0, float (&r)[16], float (&k)[16]) const {
    if constexpr (F == kEFGeneric) {
      load_aux16(m, n0, r, k);
    } else if constexpr (!kBlockAux<F>) {
      const int valid = min(16, ncols - n0);
      if constexpr ((F & kEFRes) != 0) ld_rowN<16>(res + (long)m * ldres + n0, vec != 0, valid, r);
      if constexpr ((F & (kEFMaskRelu | kEFMaskMul)) != 0)
        ld_rowN<16>(mask + (long)m * ldmask + n0, vec != 0, valid, k);
    }
  }
  // kFull: interior tile, unchecked stores; kTma: TMA bulk stores through the
  // maps tm_c (C) and tm_p (pre)
  template <int F, bool kFull = false, bool kTma = false>
  __device__ __forceinline__ void finish_block16_t(int row0, int M, int n0, float (&v)[16],
                                                   float (&r)[16], const float (&k)[16],
                                                   const float* bias_s, uint8_t* stg,
                                                   int lane, const void* tm_c = nullptr,
                                                   const void* tm_p = nullptr) const {
    if constexpr (F == kEFGeneric) {
      finish_block16(row0, M, n0, v, r, k, bias_s, stg, lane);
    } else {
      const bool vv = vec != 0;
      if constexpr ((F & kEFBias) != 0) {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const float2 bb = *reinterpret_cast<const float2*>(bias_s + i);
          const f2 t = fadd2(f2{v[i], v[i + 1]}, f2{bb.x, bb.y});
          v[i] = t.x; v[i + 1] = t.y;
        }
      }
      if constexpr ((F & kEFRes) != 0) {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const f2 t = fadd2(f2{v[i], v[i + 1]}, f2{r[i], r[i + 1]});
          v[i] = t.x; v[i + 1] = t.y;
        }
      }
      if constexpr ((F & kEFGeluD) != 0) {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          if constexpr (sizeof(TO) == 2) gelu_tanh2(v[i], v[i + 1], r[i], r[i + 1]);
          else gelu_both2(v[i], v[i + 1], r[i], r[i + 1]);
        }
        if constexpr (kTma) warp_store_tma16<TO>(tm_p, row0, n0, r, stg, lane);
        else warp_store_block16<TO, kFull>(pre, ldpre, nullptr, 0, row0, M, n0, ncols, vv, r, stg,
                                           lane);
      }
      if constexpr ((F & kEFRelu) != 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
      }
      if constexpr ((F & kEFMaskRelu) != 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = k[i] > 0.f ? v[i] : 0.f;
      }
      if constexpr ((F & kEFMaskMul) != 0) {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const f2 t = fmul2(f2{v[i], v[i + 1]}, f2{k[i], k[i + 1]});
          v[i] = t.x; v[i + 1] = t.y;
        }
      }
      if constexpr (kTma) warp_store_tma16<TO>(tm_c, row0, n0, v, stg, lane);
      else warp_store_block16<TO, kFull>(C, ldc, C2, ldc2, row0, M, n0, ncols, vv, v, stg, lane,
                                         cs_part ? cs_part + (long)(row0 >> 5) * ncols : nullptr);
    }
  }

  // 32 consecutive columns n0..n0+31 of row m (n0 % 32 == 0)
  __device__ __forceinline__ void apply_row32(int m, int n0, float (&v)[32]) const {
    const int valid = min(32, ncols - n0);
    const bool vv = vec != 0;
    if (bias) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += (i < valid) ? __ldg(bias + n0 + i) : 0.f;
    }
    if (res) {
      float r[32];
      ld_row32<TO>(res + (long)m * ldres + n0, vv, valid, r);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += r[i];
    }
    if (pre && act != kActGeluD) st_row32<TO>(pre + (long)m * ldpre + n0, vv, valid, v);
    float k[32], d[32];
    if (mask_mode != kMaskNone) ld_row32<TO>(mask + (long)m * ldmask + n0, vv, valid, k);
    act_mask<32>(v, k, d);
    if (pre && act == kActGeluD) st_row32<TO>(pre + (long)m * ldpre + n0, vv, valid, d);
    st_row32<TO>(C + (long)m * ldc + n0, vv, valid, v);
    if (C2) st_row32<TO>(C2 + (long)m * ldc2 + n0, vv, valid, v);
  }
};

// host: the compile-time epilogue specialisation matching `e` (or kEFGeneric)
template <typename TO>
inline int epi_flags(const Epilogue<TO>& e) {
  int f = 0;
  if (e.bias) f |= kEFBias;
  if (e.res) f |= kEFRes;
  if (e.act == kActRelu) f |= kEFRelu;
  else if (e.act == kActGeluD && e.pre) f |= kEFGeluD;
  else if (e.act != kActNone) return kEFGeneric;
  if (e.pre && e.act != kActGeluD) return kEFGeneric;
  if (e.mask_mode == kMaskRelu) f |= kEFMaskRelu;
  else if (e.mask_mode == kMaskMul) f |= kEFMaskMul;
  else if (e.mask_mode != kMaskNone) return kEFGeneric;
  return f;
}

// host: decide the vector flag from pointer alignment and leading dimensions
template <typename TO>
inline void epilogue_finalize(Epilogue<TO>& e, int ncols) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  auto ldok = [](long ld) { return (ld * (long)sizeof(TO)) % 16 == 0; };
  e.ncols = ncols;
  bool v = al(e.C) && ldok(e.ldc);
  if (e.C2) v = v && al(e.C2) && ldok(e.ldc2);
  if (e.mask) v = v && al(e.mask) && ldok(e.ldmask);
  if (e.res) v = v && al(e.res) && ldok(e.ldres);
  if (e.pre) v = v && al(e.pre) && ldok(e.ldpre);
  e.vec = v ? 1 : 0;
}

template <typename TI, typename TO>
int launch_gemm_simt(int M, int N, int K, const TI* A, long a_rs, long a_cs, const TI* B,
                     long b_rs, long b_cs, const Epilogue<TO>& ep, float* ws, size_t ws_elems,
                     cudaStream_t s);

namespace tc {
unsigned long long* timeline_buffer();   // PPLL_GEMM_TIMELINE probe (gemm_tc.cu)
}

// launch_gemm_tc return value when Epilogue::colsum_b was produced in-kernel
constexpr int kGemmColsumFused = 1000;

// tcgen05 GEMM (gemm_tc.cu).  a_kmajor: A(m,k)=A[m*lda+k] else A[k*lda+m];
// b_kmajor: B(k,n)=B[n*ldb+k] else B[k*ldb+n].  Returns PPLL_ERR_UNSUPPORTED
// when the shape/alignment cannot use TMA (caller then uses the SIMT engine).
template <typename TO>
int launch_gemm_tc(int M, int N, int K, const __nv_bfloat16* A, long lda, bool a_kmajor,
                   const __nv_bfloat16* B, long ldb, bool b_kmajor, const Epilogue<TO>& ep,
                   float* ws, size_t ws_elems, cudaStream_t s);

template <typename TO>
int launch_splitk_reduce(int M, int N, int splits, const float* ws, const Epilogue<TO>& ep,
                         cudaStream_t s);

template <typename T>
int launch_colsum(int M, int N, const T* G, int ld, float* db, cudaStream_t s, float* ws = nullptr,
                  size_t ws_elems = 0);

template <typename T>
int launch_softmax_xent(int B, int C, const T* z, int ldz, const int64_t* y, T* dz, int lddz,
                        float* loss_hist, const int* step, int* err, cudaStream_t s);

// fused classifier head of a local step: logits = z·W + b, softmax_xent
// (loss, dlog) and dz = dlog·Wᵀ in one launch, bitwise equal to the three
// separate kernels; PPLL_ERR_UNSUPPORTED outside C <= 32, K >= 64
bool head_xent_fusable(int B, int K, int C, size_t esz);
template <typename T>
int launch_head_xent(int B, int K, int C, const T* z, int ldz, const T* W, const float* bias,
                     const int64_t* y, T* logits, T* dlog, T* dz, int lddz, float* loss_hist,
                     const int* step, int* err, cudaStream_t s);

// advance = false: update only (the step counter is advanced by the step's
// last launch, after every range has read it)
int set_local_optimizer(const float* theta, int kind, float* m2, float beta1, float beta2,
                        float eps);
int launch_nesterov(long n, float* th, float* v, const float* g, __nv_bfloat16* th_lp,
                    const float* lr_table, int* step, int max_step, float lr_host, float mu,
                    float wd, int* err, cudaStream_t s, bool advance = true);

int launch_cast(long n, const void* src, int sd, void* dst, int dd, cudaStream_t s);
int launch_gather_rows(int n, long width, const float* src, const int64_t* idx, void* dst,
                       int dst_dtype, const int64_t* ysrc, int64_t* ydst, cudaStream_t s);
int launch_gather_rows_u8(int n, long width, const uint8_t* src, const int64_t* idx, void* dst,
                          int dst_dtype, const int64_t* ysrc, int64_t* ydst, cudaStream_t s);
int launch_count_correct(int B, int C, const void* z, long ldz, int dtype, const int64_t* y,
                         unsigned long long* count, cudaStream_t s);
int launch_relu_mask(long n, const void* g, const void* act, void* out, int dtype, cudaStream_t s);
int launch_ring_publish(int* w, int seq, cudaStream_t s);
int launch_ring_wait(const int* w, int seq, cudaStream_t s, int kind = 0);
// ring-wait watchdog: timeout of every later wait (ns; <= 0 disables) and the
// first recorded stall {stalled, wanted, seen, kind}
extern long long g_ring_timeout_ns;
int ring_stall_read(int* out4, bool clear);
int launch_ring_release(int* w, cudaStream_t s);

// Host-side description of a fused linear epilogue (see Epilogue).
struct LinOpts {
  const float* bias = nullptr;
  int act = kActNone;
  const void* mask = nullptr;
  long ldmask = 0;
  int mask_mode = kMaskNone;
  const void* res = nullptr;
  long ldres = 0;
  void* pre = nullptr;
  long ldpre = 0;
  void* C2 = nullptr;
  long ldc2 = 0;
  // fused bias gradient db = Σ_rows(output) (tcgen05 engine: per-32-row-block
  // column partials in cs_ws [ceil(M/32) x ncols], then one small reduction)
  float* db = nullptr;
  float* cs_ws = nullptr;
  size_t cs_ws_elems = 0;
};
int gemm_fwd(int M, int K, int N, const void* X, long ldx, const void* W, const LinOpts& o,
             void* Y, long ldy, int dtype, float* ws, size_t ws_elems, cudaStream_t s);
int gemm_dgrad(int M, int K, int N, const void* dY, long lddy, const void* W, const LinOpts& o,
               void* dX, long lddx, int dtype, float* ws, size_t ws_elems, cudaStream_t s);

// linear-layer ops used by both the C-ABI and the stage runtime
int linear_fwd(int M, int K, int N, const void* X, int ldx, const void* W, const float* b,
               void* Y, int ldy, void* Y2, int ldy2, int relu, int dtype, float* ws,
               size_t ws_elems, cudaStream_t s);
int linear_dgrad(int M, int K, int N, const void* dY, int lddy, const void* W, const void* mask,
                 int ldmask, void* dX, int lddx, int dtype, float* ws, size_t ws_elems,
                 cudaStream_t s);
int linear_wgrad(int M, int K, int N, const void* X, int ldx, const void* dY, int lddy, float* dW,
                 float* db, int dtype, float* ws, size_t ws_elems, cudaStream_t s);

extern int g_gemm_engine;

}  // namespace ppll
