// C-ABI for the normalisation kernels of the extension families (SURVEY §8b
// lists layernorm_{fwd,bwd} and bn_{fwd,bwd} below the boundary): the same
// launchers the ViT / ResNet stage executors call, exposed with plain
// pointers + sizes so they can be tested against torch and timed alone.  The
// reference has no normalisation layers (its blocks are MLPs, blocks.py:240-255).
#include <algorithm>
#include "common.cuh"
#include "kernels.cuh"
#include "resnet.cuh"
#include "vit.cuh"

using namespace ppll;

extern "C" {

long ppll_layernorm_bwd_ws_floats(int M, int D) {
  return (long)std::max(ln_bwd_blocks(M), 148) * 3 * D;
}

int ppll_layernorm_fwd(int M, int D, const void* x, long ldx, const float* g, const float* b,
                       void* y, long ldy, float* mean, float* rstd, int dtype, void* stream) {
  if (M < 1 || !x || !g || !b || !y || !mean || !rstd) {
    set_error("ppll_layernorm_fwd: invalid arguments");
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == PPLL_F32)
    return launch_ln_fwd<float>(M, D, (const float*)x, ldx, g, b, (float*)y, ldy, mean, rstd, s);
  return launch_ln_fwd<__nv_bfloat16>(M, D, (const __nv_bfloat16*)x, ldx, g, b,
                                      (__nv_bfloat16*)y, ldy, mean, rstd, s);
}

int ppll_layernorm_bwd(int M, int D, const void* dy, long lddy, const void* x, long ldx,
                       const float* mean, const float* rstd, const float* g, const void* dres,
                       long ldres, void* dx, long lddx, float* dg, float* db, float* dxsum,
                       float* ws, long ws_floats, int dtype, void* stream) {
  if (M < 1 || !dy || !x || !mean || !rstd || !g || !ws ||
      ws_floats < ppll_layernorm_bwd_ws_floats(M, D)) {
    set_error("ppll_layernorm_bwd: invalid arguments (workspace needs %ld floats)",
              ppll_layernorm_bwd_ws_floats(M, D));
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == PPLL_F32)
    return launch_ln_bwd<float>(M, D, (const float*)dy, lddy, (const float*)x, ldx, mean, rstd, g,
                                (const float*)dres, ldres, (float*)dx, lddx, ws, dg, db, s, dxsum);
  using B16 = __nv_bfloat16;
  return launch_ln_bwd<B16>(M, D, (const B16*)dy, lddy, (const B16*)x, ldx, mean, rstd, g,
                            (const B16*)dres, ldres, (B16*)dx, lddx, ws, dg, db, s, dxsum);
}

// scratch of the grid-form fused BN for the C-ABI entry points (one set per
// process: these entry points are not meant for concurrent streams)
static const BnGrid* capi_bn_grid() {
  static BnGrid g{nullptr, nullptr, nullptr};
  static bool init = false;
  if (!init) {
    init = true;
    void* p = nullptr;
    unsigned* b = nullptr;
    if (cudaMalloc(&p, 256 * 128 * 16) == cudaSuccess && cudaMalloc(&b, 256) == cudaSuccess &&
        cudaMemset(b, 0, 256) == cudaSuccess) {
      g.part = p;
      g.bar = b;
    } else {
      cudaGetLastError();
    }
  }
  return g.part ? &g : nullptr;
}

long ppll_batchnorm_ws_floats(int P, int C) { return (long)bn_chunks(P) * 3 * C; }

// train-mode BatchNorm over the rows of an NHWC [P, C] tensor: batch
// statistics (biased variance, eps 1e-5) into mean / rstd, then
// y = act((z - mean)·rstd·g + b [+ res]); relu != 0 applies ReLU
int ppll_batchnorm_fwd(int P, int C, const void* z, const float* g, const float* b,
                       const void* res, int relu, void* y, float* mean, float* rstd, float* ws,
                       long ws_floats, int dtype, void* stream) {
  if (P < 1 || C < 1 || !z || !g || !b || !y || !mean || !rstd || !ws ||
      ws_floats < ppll_batchnorm_ws_floats(P, C)) {
    set_error("ppll_batchnorm_fwd: invalid arguments");
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int r;
  if (dtype == PPLL_F32) {
    r = launch_bn_stats<float>(P, C, (const float*)z, ws, mean, rstd, s);
    if (r) return r;
    return launch_bn_apply<float>(P, C, (const float*)z, mean, rstd, g, b, nullptr, nullptr,
                                  nullptr, nullptr, nullptr, (const float*)res, relu, (float*)y, s);
  }
  using B16 = __nv_bfloat16;
  // one fused launch where it applies (bn_cluster.cu: one cluster, or the
  // whole GPU for large tensors), else stats + apply
  r = launch_bn_fwd_fused(P, C, (const B16*)z, g, b, mean, rstd, nullptr, nullptr, nullptr,
                          nullptr, nullptr, (const B16*)res, relu, (B16*)y, s, capi_bn_grid());
  if (r != PPLL_ERR_UNSUPPORTED) return r;
  r = launch_bn_stats<B16>(P, C, (const B16*)z, ws, mean, rstd, s);
  if (r) return r;
  return launch_bn_apply<B16>(P, C, (const B16*)z, mean, rstd, g, b, nullptr, nullptr, nullptr,
                              nullptr, nullptr, (const B16*)res, relu, (B16*)y, s);
}

// given dy = dLoss/dBN-output: dg, db and dz = dLoss/dz
int ppll_batchnorm_bwd(int P, int C, const void* dy, const void* z, const float* mean,
                       const float* rstd, const float* g, float* dg, float* db, void* dz,
                       float* ws, long ws_floats, int dtype, void* stream) {
  if (P < 1 || C < 1 || !dy || !z || !mean || !rstd || !g || !dg || !db || !dz || !ws ||
      ws_floats < ppll_batchnorm_ws_floats(P, C)) {
    set_error("ppll_batchnorm_bwd: invalid arguments");
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == PPLL_F32)
    return launch_bn_bwd<float>(P, C, (const float*)dy, (const float*)z, mean, rstd, g, ws, dg, db,
                                (float*)dz, s);
  using B16 = __nv_bfloat16;
  const int r = launch_bn_bwd_fused(P, C, (const B16*)dy, nullptr, nullptr, (const B16*)z, mean,
                                    rstd, g, dg, db, (B16*)dz, nullptr, nullptr, nullptr, nullptr,
                                    nullptr, nullptr, nullptr, s, capi_bn_grid());
  if (r != PPLL_ERR_UNSUPPORTED) return r;
  return launch_bn_bwd<B16>(P, C, (const B16*)dy, (const B16*)z, mean, rstd, g, ws, dg, db,
                            (B16*)dz, s);
}

}  // extern "C"
