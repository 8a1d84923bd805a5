// Native executor of one ViT local-learning stage (the PPLL local step,
// blocks.py:266-289 semantics, applied to pre-LN transformer blocks):
//
//   [patchify → patch GEMM → +cls/+pos]            (stage 0 only)
//   block layers   : LN1 → QKV GEMM → MHSA → proj GEMM(+res) → LN2 →
//                    FC1 GEMM(+GELU, pre-act kept) → FC2 GEMM(+res)
//                    (the last block layer's FC2 epilogue dual-stores x_out,
//                     i.e. the push, with PRE-update parameters)
//   aux layers     : same layer type, N_l = aux_depth(l, d', n) of them
//   head           : LN on the cls rows → classifier GEMM → softmax-CE
//   backward       : reverse of the above; no gradient into the detached
//                    stage input (the first LN1 backward only produces its
//                    gamma/beta gradients)
//   update         : one Nesterov launch over the flat parameter buffer.
//
// Every tensor is [rows, features] row-major with rows = batch·tokens; the
// per-layer activations needed by the backward are kept in a workspace sized
// once for max_batch.
#include <algorithm>
#include <type_traits>
#include <vector>
#include "common.cuh"
#include "kernels.cuh"
#include "vit.cuh"

namespace {
enum { kLn1g, kLn1b, kWqkv, kBqkv, kWo, kBo, kLn2g, kLn2b, kW1, kB1, kW2, kB2, kLayerParams };
struct LayerBufs {
  char *xn1, *qkv, *o, *x1, *xn2, *u, *h, *x2;
  float *mean1, *rstd1, *mean2, *rstd2, *lse;
};
}  // namespace

struct ppll_vit_stage {
  int Bmax, T, D, H, F, C, n_block, n_aux, has_patch, img_c, img_hw, patch;
  int dtype;
  size_t esz;
  std::vector<int64_t> off;          // [patch 4][12 per layer][head 4]
  int64_t n_params;
  float *theta, *grad, *mom;
  void* theta_lp;
  const float* lr_table;
  int* step;
  int max_step;
  float* loss_hist;
  int* err;
  float mu, wd;
  std::vector<LayerBufs> L;
  char *patches = nullptr, *tok = nullptr, *x0 = nullptr;
  char *zc = nullptr, *logits = nullptr, *dlog = nullptr, *dz = nullptr, *dzc = nullptr;
  float *meanf = nullptr, *rstdf = nullptr;
  char *dxa = nullptr, *dxb = nullptr, *dxc = nullptr, *dbig = nullptr, *dxn = nullptr,
       *dqkv = nullptr, *dO = nullptr, *dtok = nullptr;
  float* ln_part = nullptr;
  float* ln_parts = nullptr;   // [2·layers + 1][ln_slab] deferred LN partials
  size_t ln_slab = 0;
  float* cs_part = nullptr;       // fused bias-gradient column partials [ceil(M/32), F]
  size_t cs_part_elems = 0;
  float* attn_bpart = nullptr;
  float* ws = nullptr;
  size_t ws_elems = 0;
  // weight gradients run on a side stream (off the dgrad critical path), with
  // their own split-K workspace; events fork/join it to the step's stream
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> ev;
  float* ws2 = nullptr;
  std::vector<void*> allocs;
  // the last forward ran its top layer on the cls rows only (see vit_forward)
  bool cls_top = false;

  int layers() const { return n_block + n_aux; }
  int64_t po(int layer, int k) const { return off[4 + layer * kLayerParams + k]; }
  int64_t ho(int k) const { return off[4 + layers() * kLayerParams + k]; }
  const void* W(int64_t o) const {
    return dtype == PPLL_F32 ? (const void*)(theta + o)
                             : (const void*)(reinterpret_cast<const __nv_bfloat16*>(theta_lp) + o);
  }
  const float* P(int64_t o) const { return theta + o; }
  float* G(int64_t o) const { return grad + o; }
  char* alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, (bytes + 255) / 256 * 256) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    return reinterpret_cast<char*>(p);
  }
};

using namespace ppll;

// attention engine: tcgen05 for bf16 with T <= 128, SIMT kernels otherwise
template <typename TT>
static int attn_fwd_any(int B, int T, int H, int dh, const TT* qkv, TT* o, float* lse,
                        cudaStream_t s) {
  if constexpr (std::is_same<TT, __nv_bfloat16>::value) {
    if (g_attn_engine == 0 && attn_tc_supported(T, dh))
      return launch_attn_tc_fwd(B, T, H, qkv, o, lse, s);
  }
  return launch_attn_fwd<TT>(B, T, H, dh, qkv, o, lse, s);
}
// also produces dbqkv = Σ rows of dqkv (fused into the tcgen05 kernel, or a
// separate column reduction for the SIMT kernels)
template <typename TT>
static int attn_bwd_any(int B, int T, int H, int dh, const TT* qkv, const TT* o, const TT* dout,
                        const float* lse, TT* dqkv, float* dbqkv, float* bpart, float* ws,
                        size_t ws_elems, cudaStream_t s) {
  const int D3 = 3 * H * dh;
  if constexpr (std::is_same<TT, __nv_bfloat16>::value) {
    if (g_attn_engine == 0 && attn_tc_supported(T, dh)) {
      int r = launch_attn_tc_bwd(B, T, H, qkv, o, dout, lse, dqkv, s, bpart);
      if (r) return r;
      return launch_colsum<float>(B, D3, bpart, D3, dbqkv, s, ws, ws_elems);
    }
  }
  int r = launch_attn_bwd<TT>(B, T, H, dh, qkv, o, dout, lse, dqkv, s);
  if (r) return r;
  return launch_colsum<TT>(B * T, D3, dqkv, D3, dbqkv, s, ws, ws_elems);
}

template <typename TT>
static int vit_forward(ppll_vit_stage* st, int B, const void* x_in, void* x_out, bool head,
                       cudaStream_t s, int nl = -1, bool defer_logits = false) {
  NvtxRange nv("ppll.vit.forward");
  if (nl < 0) nl = st->layers();
  const int T = st->T, D = st->D, F = st->F, H = st->H;
  const int M = B * T;
  const TT* xcur = reinterpret_cast<const TT*>(x_in);
  int r;
  // Top layer on the cls rows only: when the stage's last layer feeds nothing
  // but the head (an aux stack's last layer, or the final stage's last block
  // layer — not a layer whose output is pushed), only its cls rows reach the
  // loss.  Its LN1 / QKV / attention still run over every token (the cls
  // query attends to all keys and values), but the proj, LN2, FC1 and FC2
  // work — and their backward — is needed for the B cls rows alone; the other
  // rows' contributions to the loss and to every gradient are exactly zero:
  // the same math for everything the step produces (the cls-query attention
  // rounds in fp32 where the tcgen05 tiles round P to bf16), ~80 % of the
  // layer's GEMM work gone.  PPLL_VIT_CLS_TOP=0 runs the layer over all rows.
  static const int cls_env = getenv("PPLL_VIT_CLS_TOP") ? atoi(getenv("PPLL_VIT_CLS_TOP")) : 1;
  const bool cls_top = cls_env && head && nl >= 1 && !(nl - 1 == st->n_block - 1 && x_out);
  st->cls_top = cls_top;
  if (st->has_patch) {
    const int P = T - 1, pd = st->img_c * st->patch * st->patch;
    r = launch_patchify<TT>(B, st->img_c, st->img_hw, st->patch, (const TT*)x_in, (TT*)st->patches, s);
    if (r) return r;
    LinOpts o;
    o.bias = st->P(st->off[1]);
    r = gemm_fwd(B * P, pd, D, st->patches, pd, st->W(st->off[0]), o, st->tok, D, st->dtype, st->ws,
                 st->ws_elems, s);
    if (r) return r;
    r = launch_embed<TT>(B, P, D, (const TT*)st->tok, st->P(st->off[2]), st->P(st->off[3]),
                         (TT*)st->x0, s);
    if (r) return r;
    xcur = (const TT*)st->x0;
  }
  for (int l = 0; l < nl; ++l) {
    LayerBufs& b = st->L[l];
    r = launch_ln_fwd<TT>(M, D, xcur, D, st->P(st->po(l, kLn1g)), st->P(st->po(l, kLn1b)),
                          (TT*)b.xn1, D, b.mean1, b.rstd1, s);
    if (r) return r;
    LinOpts o1;
    o1.bias = st->P(st->po(l, kBqkv));
    r = gemm_fwd(M, D, 3 * D, b.xn1, D, st->W(st->po(l, kWqkv)), o1, b.qkv, 3 * D, st->dtype,
                 st->ws, st->ws_elems, s);
    if (r) return r;
    if (cls_top && l == nl - 1) {
      // cls rows only: the cls query's attention (o, lse compact: B rows /
      // B·H entries), then proj (+ the residual's cls rows, row stride T·D),
      // LN2, FC1, FC2 on B compact rows
      r = launch_cls_attn_fwd<TT>(B, T, H, (const TT*)b.qkv, (TT*)b.o, b.lse, s);
      if (r) return r;
      LinOpts o2;
      o2.bias = st->P(st->po(l, kBo));
      o2.res = xcur;
      o2.ldres = (long)T * D;
      r = gemm_fwd(B, D, D, b.o, D, st->W(st->po(l, kWo)), o2, b.x1, D, st->dtype, st->ws,
                   st->ws_elems, s);
      if (r) return r;
      r = launch_ln_fwd<TT>(B, D, (const TT*)b.x1, D, st->P(st->po(l, kLn2g)),
                            st->P(st->po(l, kLn2b)), (TT*)b.xn2, D, b.mean2, b.rstd2, s);
      if (r) return r;
      LinOpts o3;
      o3.bias = st->P(st->po(l, kB1));
      o3.act = kActGeluD;
      o3.pre = b.u;
      o3.ldpre = F;
      r = gemm_fwd(B, D, F, b.xn2, D, st->W(st->po(l, kW1)), o3, b.h, F, st->dtype, st->ws,
                   st->ws_elems, s);
      if (r) return r;
      LinOpts o4;
      o4.bias = st->P(st->po(l, kB2));
      o4.res = b.x1;
      o4.ldres = D;
      r = gemm_fwd(B, F, D, b.h, F, st->W(st->po(l, kW2)), o4, b.x2, D, st->dtype, st->ws,
                   st->ws_elems, s);
      if (r) return r;
      xcur = (const TT*)b.x2;
      continue;
    }
    r = attn_fwd_any<TT>(B, T, H, D / H, (const TT*)b.qkv, (TT*)b.o, b.lse, s);
    if (r) return r;
    // proj (+bias, +residual) -> x1 and LN2 -> xn2: one fused launch for bf16
    // D = 384 (gemm_ln.cu), else the GEMM with its residual epilogue + LN kernel
    r = PPLL_ERR_UNSUPPORTED;
    if (st->dtype == PPLL_BF16 && D == 384)
      r = launch_gemm_ln_fwd(M, D, (const __nv_bfloat16*)b.o,
                             (const __nv_bfloat16*)st->W(st->po(l, kWo)), st->P(st->po(l, kBo)),
                             (const __nv_bfloat16*)xcur, st->P(st->po(l, kLn2g)),
                             st->P(st->po(l, kLn2b)), (__nv_bfloat16*)b.x1, (__nv_bfloat16*)b.xn2,
                             b.mean2, b.rstd2, s);
    if (r != PPLL_OK && r != PPLL_ERR_UNSUPPORTED) return r;
    if (r == PPLL_ERR_UNSUPPORTED) {
      LinOpts o2;
      o2.bias = st->P(st->po(l, kBo));
      o2.res = xcur;
      o2.ldres = D;
      r = gemm_fwd(M, D, D, b.o, D, st->W(st->po(l, kWo)), o2, b.x1, D, st->dtype, st->ws,
                   st->ws_elems, s);
      if (r) return r;
      r = launch_ln_fwd<TT>(M, D, (const TT*)b.x1, D, st->P(st->po(l, kLn2g)),
                            st->P(st->po(l, kLn2b)), (TT*)b.xn2, D, b.mean2, b.rstd2, s);
      if (r) return r;
    }
    LinOpts o3;
    o3.bias = st->P(st->po(l, kB1));
    o3.act = kActGeluD;   // b.u <- gelu'(pre-activation)
    o3.pre = b.u;
    o3.ldpre = F;
    r = gemm_fwd(M, D, F, b.xn2, D, st->W(st->po(l, kW1)), o3, b.h, F, st->dtype, st->ws,
                 st->ws_elems, s);
    if (r) return r;
    LinOpts o4;
    o4.bias = st->P(st->po(l, kB2));
    o4.res = b.x1;
    o4.ldres = D;
    if (l == st->n_block - 1 && x_out) {   // fused push of the block output
      o4.C2 = x_out;
      o4.ldc2 = D;
    }
    r = gemm_fwd(M, F, D, b.h, F, st->W(st->po(l, kW2)), o4, b.x2, D, st->dtype, st->ws,
                 st->ws_elems, s);
    if (r) return r;
    xcur = (const TT*)b.x2;
  }
  if (!head) return PPLL_OK;
  // head: LayerNorm on the cls rows (row stride T·D; compact after a cls-only
  // top layer) + classifier
  r = launch_ln_fwd<TT>(B, D, xcur, cls_top ? (long)D : (long)T * D, st->P(st->ho(0)),
                        st->P(st->ho(1)), (TT*)st->zc, D, st->meanf, st->rstdf, s);
  if (r) return r;
  // a backward follows (local step / E2E final stage): the fused head kernel
  // computes the logits there, together with the loss and dz
  if (defer_logits && head_xent_fusable(B, D, st->C, st->esz)) return PPLL_OK;
  LinOpts oh;
  oh.bias = st->P(st->ho(3));
  return gemm_fwd(B, D, st->C, st->zc, D, st->W(st->ho(2)), oh, st->logits, st->C, st->dtype,
                  st->ws, st->ws_elems, s);
}

// Backward of the stage's first `nl` layers (+ head when `labels`), then the
// patch embedding on stage 0.  The gradient entering the top layer's output is
// either the task / aux loss through the head (labels != NULL) or `g_out`
// (dLoss/d(block output) from the next stage: E2E / naive PP).  `g_in`
// receives dLoss/d(stage input) (NULL: detached input, blocks.py:277-278).
// Every weight gradient has landed on `s` when this returns.
template <typename TT>
static int vit_backward(ppll_vit_stage* st, int B, const void* x_in, const int64_t* labels,
                        const void* g_out, void* g_in, int nl, cudaStream_t s) {
  NvtxRange nv("ppll.vit.backward");
  const int T = st->T, D = st->D, F = st->F, H = st->H, C = st->C;
  const int M = B * T;
  static const bool side_on = !(getenv("PPLL_SIDE_WGRAD") && atoi(getenv("PPLL_SIDE_WGRAD")) == 0);
  SideFlow sf{s, (side_on && st->side) ? st->side : s, st->ev.data(), 0, (int)st->ev.size()};
  float* wsw = sf.on() ? st->ws2 : st->ws;   // the weight gradients' workspace
  int r;
  LinOpts none;
  // LN parameter (and fused bias) reductions are deferred to one batched
  // launch at the end of the backward; each LN backward gets its own slab
  LnDefer dfr;
  int nslab = 0;
  // SM budgets (experiment, PPLL_DGRAD_CAP / PPLL_WGRAD_CAP): with the weight
  // gradients on the side stream, cap the data-gradient chain's GEMM grid and
  // the cluster wgrads' footprint so both streams' kernels can co-reside
  static const int dcap = getenv("PPLL_DGRAD_CAP") ? atoi(getenv("PPLL_DGRAD_CAP")) : 0;
  static const int wcap = getenv("PPLL_WGRAD_CAP") ? atoi(getenv("PPLL_WGRAD_CAP")) : 0;
  struct CapScope {
    int g0, w0;
    CapScope(bool on, int d, int w) : g0(g_gemm_cap), w0(g_wgrad_cap) {
      if (on) { g_gemm_cap = d; g_wgrad_cap = w; }
    }
    ~CapScope() { g_gemm_cap = g0; g_wgrad_cap = w0; }
  } caps(sf.on(), dcap, wcap);
  auto slab = [&]() { return st->ln_parts + st->ln_slab * (size_t)(nslab++); };
  const bool cls_top = labels && st->cls_top;   // the forward's choice
  if (labels) {
    // logits + softmax_xent + dz in one launch (the forward deferred the logits)
    const bool fused = head_xent_fusable(B, D, C, st->esz);
    if (fused) {
      r = launch_head_xent<TT>(B, D, C, (const TT*)st->zc, D, (const TT*)st->W(st->ho(2)),
                               st->P(st->ho(3)), labels, (TT*)st->logits, (TT*)st->dlog,
                               (TT*)st->dz, D, st->loss_hist, st->step, st->err, s);
    } else {
      r = launch_softmax_xent<TT>(B, C, (const TT*)st->logits, C, labels, (TT*)st->dlog, C,
                                  st->loss_hist, st->step, st->err, s);
    }
    if (r) return r;
    const TT* xlast = (const TT*)st->L[nl - 1].x2;
    // ---- head backward ----
    sf.fork();
    r = linear_wgrad(B, D, C, st->zc, D, st->dlog, C, st->G(st->ho(2)), st->G(st->ho(3)),
                     st->dtype, wsw, st->ws_elems, sf.ss);
    if (r) return r;
    if (!fused) {
      r = gemm_dgrad(B, D, C, st->dlog, C, st->W(st->ho(2)), none, st->dz, D, st->dtype, st->ws,
                     st->ws_elems, s);
      if (r) return r;
    }
    // cls-only top layer: the head's input gradient IS the top layer's
    // (compact, B rows) output gradient; else it is scattered to the cls rows
    char* dhead = cls_top ? st->dxa : st->dzc;
    r = launch_ln_bwd<TT>(B, D, (const TT*)st->dz, D, xlast, cls_top ? (long)D : (long)T * D,
                          st->meanf, st->rstdf, st->P(st->ho(0)), nullptr, 0, (TT*)dhead, D,
                          slab(), st->G(st->ho(0)), st->G(st->ho(1)), s, nullptr, &dfr);
    if (r) return r;
    if (!cls_top) {
      r = launch_scatter_cls<TT>(B, T, D, (const TT*)st->dzc, (TT*)st->dxa, s);
      if (r) return r;
    }
    // db2 of the top layer = Σ rows of its output gradient: only the cls rows
    // are non-zero (Σ of dz over the batch)
    r = launch_colsum<TT>(B, D, (const TT*)dhead, D, st->G(st->po(nl - 1, kB2)), s, st->ws,
                          st->ws_elems);
    if (r) return r;
  } else {
    PPLL_CUDA_CHECK(cudaMemcpyAsync(st->dxa, g_out, (size_t)M * D * st->esz,
                                    cudaMemcpyDeviceToDevice, s));
    r = launch_colsum<TT>(M, D, (const TT*)st->dxa, D, st->G(st->po(nl - 1, kB2)), s, st->ws,
                          st->ws_elems);
    if (r) return r;
  }
  // ---- layers, last first ----
  char* dx2 = st->dxa;   // gradient w.r.t. the current layer's output
  char* dx1 = st->dxb;
  char* dxn_out = st->dxc;
  // side-stream completion of the previous (higher) layer's weight gradients:
  // the main stream waits on them before overwriting the buffers they read
  cudaEvent_t e_w2 = nullptr, e_w1 = nullptr, e_wo = nullptr, e_wqkv = nullptr;
  for (int l = nl - 1; l >= 0; --l) {
    LayerBufs& b = st->L[l];
    const void* xin_l = l > 0 ? (const void*)st->L[l - 1].x2
                              : (st->has_patch ? (const void*)st->x0 : x_in);
    // (db2 of layer l < top: fused into the LN1 backward of layer l+1)
    // cls-only top layer: FC2 / FC1 / LN2 / proj over the B compact cls rows
    const bool cls = cls_top && l == nl - 1;
    const int Mr = cls ? B : M;
    sf.fork();
    r = linear_wgrad(Mr, F, D, b.h, F, dx2, D, st->G(st->po(l, kW2)), nullptr, st->dtype, wsw,
                     st->ws_elems, sf.ss);
    if (r) return r;
    const cudaEvent_t n_w2 = sf.mark();
    sf.join(e_w1);   // dbig is still read by the layer above's W1 gradient
    LinOpts og;
    og.mask = b.u;
    og.ldmask = F;
    og.mask_mode = kMaskMul;
    r = gemm_dgrad(Mr, F, D, dx2, D, st->W(st->po(l, kW2)), og, st->dbig, F, st->dtype, st->ws,
                   st->ws_elems, s);
    if (r) return r;
    // db1 = Σ rows dU: summed from the dU tiles in smem by the cluster wgrad
    sf.fork();
    r = linear_wgrad(Mr, D, F, b.xn2, D, st->dbig, F, st->G(st->po(l, kW1)), st->G(st->po(l, kB1)),
                     st->dtype, wsw, st->ws_elems, sf.ss);
    if (r) return r;
    e_w1 = sf.mark();
    // FC1 data gradient + LN2 backward (+ residual) -> dx1, with dbo = Σ rows
    // dx1: one fused launch for bf16 D = 384 (gemm_ln.cu), else GEMM + LN kernel
    sf.join(e_wo);   // dx1 is still read by the layer above's Wo gradient
    r = PPLL_ERR_UNSUPPORTED;
    float* part2 = slab();   // this LayerNorm's partial slab (fused or not)
    // cls-only: the compact dx1 goes to dzc (free after the head), then is
    // scattered to the cls rows of dx1 (the residual input of the LN1 backward)
    char* dx1w = cls ? st->dzc : dx1;
    if (st->dtype == PPLL_BF16 && D == 384)
      r = launch_gemm_ln_bwd(Mr, F, (const __nv_bfloat16*)st->dbig,
                             (const __nv_bfloat16*)st->W(st->po(l, kW1)),
                             (const __nv_bfloat16*)b.x1, b.mean2, b.rstd2, st->P(st->po(l, kLn2g)),
                             (const __nv_bfloat16*)dx2, (__nv_bfloat16*)dx1w, part2,
                             st->G(st->po(l, kLn2g)), st->G(st->po(l, kLn2b)),
                             st->G(st->po(l, kBo)), &dfr, s);
    if (r != PPLL_OK && r != PPLL_ERR_UNSUPPORTED) return r;
    if (r == PPLL_ERR_UNSUPPORTED) {
      r = gemm_dgrad(Mr, D, F, st->dbig, F, st->W(st->po(l, kW1)), none, st->dxn, D, st->dtype,
                     st->ws, st->ws_elems, s);
      if (r) return r;
      r = launch_ln_bwd<TT>(Mr, D, (const TT*)st->dxn, D, (const TT*)b.x1, D, b.mean2, b.rstd2,
                            st->P(st->po(l, kLn2g)), (const TT*)dx2, D, (TT*)dx1w, D, part2,
                            st->G(st->po(l, kLn2g)), st->G(st->po(l, kLn2b)), s,
                            st->G(st->po(l, kBo)), &dfr);
      if (r) return r;
    }
    sf.fork();
    r = linear_wgrad(Mr, D, D, b.o, D, dx1w, D, st->G(st->po(l, kWo)), nullptr,
                     st->dtype, wsw, st->ws_elems, sf.ss);
    if (r) return r;
    e_wo = sf.mark();
    r = gemm_dgrad(Mr, D, D, dx1w, D, st->W(st->po(l, kWo)), none, cls ? st->dz : st->dO, D,
                   st->dtype, st->ws, st->ws_elems, s);
    if (r) return r;
    if (cls) {   // the residual gradient: zero except on the cls rows
      r = launch_scatter_cls<TT>(B, T, D, (const TT*)st->dzc, (TT*)dx1, s);
      if (r) return r;
    }
    sf.join(e_wqkv);   // dqkv is still read by the layer above's Wqkv gradient
    if (cls) {   // dO is non-zero on the cls rows only (compact in st->dz)
      r = launch_cls_attn_bwd<TT>(B, T, H, (const TT*)b.qkv, (const TT*)b.o, (const TT*)st->dz,
                                  b.lse, (TT*)st->dqkv, st->attn_bpart, s);
      if (r) return r;
      r = launch_colsum<float>(B, 3 * D, st->attn_bpart, 3 * D, st->G(st->po(l, kBqkv)), s,
                               st->ws, st->ws_elems);
    } else {
      r = attn_bwd_any<TT>(B, T, H, D / H, (const TT*)b.qkv, (const TT*)b.o, (const TT*)st->dO,
                           b.lse, (TT*)st->dqkv, st->G(st->po(l, kBqkv)), st->attn_bpart, st->ws,
                           st->ws_elems, s);
    }
    if (r) return r;
    sf.fork();
    r = linear_wgrad(M, D, 3 * D, b.xn1, D, st->dqkv, 3 * D, st->G(st->po(l, kWqkv)), nullptr,
                     st->dtype, wsw, st->ws_elems, sf.ss);
    if (r) return r;
    e_wqkv = sf.mark();
    // QKV data gradient + LN1 backward (+ residual) -> gradient of the layer
    // input; no gradient into the detached stage input (blocks.py:277-278).
    // Its row sum is the bias gradient db2 of the layer below (fused).
    const bool need_dx = l > 0 || st->has_patch || g_in;
    // the stage input's gradient goes straight to g_in (no patch embedding below)
    TT* dx_dst = (l == 0 && !st->has_patch) ? (TT*)g_in : (TT*)dxn_out;
    sf.join(e_w2);   // dxn_out was the layer above's dx2, read by its W2 gradient
    e_w2 = n_w2;
    r = PPLL_ERR_UNSUPPORTED;
    float* part1 = slab();
    if (st->dtype == PPLL_BF16 && D == 384)
      r = launch_gemm_ln_bwd(M, 3 * D, (const __nv_bfloat16*)st->dqkv,
                             (const __nv_bfloat16*)st->W(st->po(l, kWqkv)),
                             (const __nv_bfloat16*)xin_l, b.mean1, b.rstd1, st->P(st->po(l, kLn1g)),
                             (const __nv_bfloat16*)dx1, need_dx ? (__nv_bfloat16*)dx_dst : nullptr,
                             part1, st->G(st->po(l, kLn1g)), st->G(st->po(l, kLn1b)),
                             l > 0 ? st->G(st->po(l - 1, kB2)) : nullptr, &dfr, s);
    if (r != PPLL_OK && r != PPLL_ERR_UNSUPPORTED) return r;
    if (r == PPLL_ERR_UNSUPPORTED) {
      r = gemm_dgrad(M, D, 3 * D, st->dqkv, 3 * D, st->W(st->po(l, kWqkv)), none, st->dxn, D,
                     st->dtype, st->ws, st->ws_elems, s);
      if (r) return r;
      r = launch_ln_bwd<TT>(M, D, (const TT*)st->dxn, D, (const TT*)xin_l, D, b.mean1, b.rstd1,
                            st->P(st->po(l, kLn1g)), (const TT*)dx1, D,
                            need_dx ? dx_dst : nullptr, D, part1,
                            st->G(st->po(l, kLn1g)), st->G(st->po(l, kLn1b)), s,
                            l > 0 ? st->G(st->po(l - 1, kB2)) : nullptr, &dfr);
      if (r) return r;
    }
    char* t = dx2;
    dx2 = dxn_out;
    dxn_out = t;
  }
  if (st->has_patch) {
    const int P = T - 1, pd = st->img_c * st->patch * st->patch;
    r = launch_embed_bwd<TT>(B, P, D, (const TT*)dx2, (TT*)st->dtok, st->G(st->off[2]),
                             st->G(st->off[3]), s);
    if (r) return r;
    r = linear_wgrad(B * P, pd, D, st->patches, pd, st->dtok, D, st->G(st->off[0]),
                     st->G(st->off[1]), st->dtype, st->ws, st->ws_elems, s);
    if (r) return r;
  }
  r = launch_ln_reduce_deferred(dfr, s);
  if (r) return r;
  // every weight gradient has landed before the optimizer reads them
  sf.join(sf.mark());
  return PPLL_OK;
}

// optimizer over the first `n` elements of the flat parameter buffer
static int vit_update(ppll_vit_stage* st, int64_t n, cudaStream_t s) {
  NvtxRange nv("ppll.vit.update");
  return launch_nesterov(n, st->theta, st->mom, st->grad,
                         reinterpret_cast<__nv_bfloat16*>(st->theta_lp), st->lr_table, st->step,
                         st->max_step, 0.f, st->mu, st->wd, st->err, s);
}

// one PPLL local step: forward (block + aux + head, the last block epilogue
// dual-stores the push), local loss, backward with no gradient into the
// detached input, update of every stage parameter
template <typename TT>
static int vit_step(ppll_vit_stage* st, int B, const void* x_in, const int64_t* labels,
                    void* x_out, cudaStream_t s) {
  int r = vit_forward<TT>(st, B, x_in, x_out, true, s, -1, true);
  if (r) return r;
  r = vit_backward<TT>(st, B, x_in, labels, nullptr, nullptr, st->layers(), s);
  if (r) return r;
  return vit_update(st, st->n_params, s);
}

extern "C" {

ppll_vit_stage* ppll_vit_stage_create(const int* cfg, const int64_t* offsets, int64_t n_params,
                                      int dtype, float* theta, float* grad, float* mom,
                                      void* theta_lp, const float* lr_table, int* step,
                                      int max_step, float* loss_hist, int* err, float mu, float wd) {
  ppll_vit_stage* st = new ppll_vit_stage();
  st->Bmax = cfg[0]; st->T = cfg[1]; st->D = cfg[2]; st->H = cfg[3]; st->F = cfg[4];
  st->C = cfg[5]; st->n_block = cfg[6]; st->n_aux = cfg[7]; st->has_patch = cfg[8];
  st->img_c = cfg[9]; st->img_hw = cfg[10]; st->patch = cfg[11];
  if (st->Bmax < 1 || st->T < 1 || st->D % 32 || st->D % st->H || st->D / st->H != 64 ||
      st->n_block < 1 || (dtype != PPLL_F32 && dtype != PPLL_BF16) ||
      (dtype == PPLL_BF16 && !theta_lp)) {
    set_error("ppll_vit_stage_create: unsupported configuration (D=%d H=%d)", st->D, st->H);
    delete st;
    return nullptr;
  }
  st->dtype = dtype;
  st->esz = dtype == PPLL_F32 ? 4 : 2;
  st->off.assign(offsets, offsets + 4 + (st->n_block + st->n_aux) * kLayerParams + 4);
  st->n_params = n_params;
  st->theta = theta; st->grad = grad; st->mom = mom; st->theta_lp = theta_lp;
  st->lr_table = lr_table; st->step = step; st->max_step = max_step;
  st->loss_hist = loss_hist; st->err = err; st->mu = mu; st->wd = wd;
  const size_t M = (size_t)st->Bmax * st->T, D = st->D, F = st->F, e = st->esz;
  bool ok = true;
  auto A = [&](size_t bytes) { char* p = st->alloc(bytes); ok = ok && p; return p; };
  for (int l = 0; l < st->layers(); ++l) {
    LayerBufs b;
    b.xn1 = A(M * D * e); b.qkv = A(M * 3 * D * e); b.o = A(M * D * e); b.x1 = A(M * D * e);
    b.xn2 = A(M * D * e); b.u = A(M * F * e); b.h = A(M * F * e); b.x2 = A(M * D * e);
    b.mean1 = (float*)A(M * 4); b.rstd1 = (float*)A(M * 4);
    b.mean2 = (float*)A(M * 4); b.rstd2 = (float*)A(M * 4);
    b.lse = (float*)A((size_t)st->Bmax * st->H * st->T * 4);
    st->L.push_back(b);
  }
  if (st->has_patch) {
    const size_t P = st->T - 1, pd = (size_t)st->img_c * st->patch * st->patch;
    st->patches = A(st->Bmax * P * pd * e);
    st->tok = A(st->Bmax * P * D * e);
    st->x0 = A(M * D * e);
    st->dtok = A(st->Bmax * P * D * e);
  }
  st->zc = A(st->Bmax * D * e);
  st->logits = A((size_t)st->Bmax * st->C * e);
  st->dlog = A((size_t)st->Bmax * st->C * e);
  st->dz = A(st->Bmax * D * e);
  st->dzc = A(st->Bmax * D * e);
  st->meanf = (float*)A(st->Bmax * 4);
  st->rstdf = (float*)A(st->Bmax * 4);
  st->dxa = A(M * D * e); st->dxb = A(M * D * e); st->dxc = A(M * D * e);
  st->dbig = A(M * F * e); st->dxn = A(M * D * e); st->dqkv = A(M * 3 * D * e);
  st->dO = A(M * D * e);
  st->ln_part = (float*)A((size_t)ln_bwd_blocks((int)M) * 3 * D * 4);
  // deferred LN reductions: one partial slab per LN backward of a step
  // (head LN + two per layer), reduced in one batched launch before the update
  // one slab holds the partials of either LN backward form: the persistent
  // kernel's blocks or the fused GEMM + LN kernel's 128-row tiles (more than
  // the former past ~37k rows, e.g. ViT-S at batch 1024)
  st->ln_slab = (size_t)std::max(ln_bwd_blocks((int)M), (int)((M + 127) / 128)) * 3 * D;
  st->ln_parts = (float*)A(st->ln_slab * (2 * st->L.size() + 1) * 4);
  st->cs_part_elems = (size_t)ceil_div((long)M, 32) * st->F;
  st->cs_part = (float*)A(st->cs_part_elems * 4);
  st->attn_bpart = (float*)A((size_t)st->Bmax * 3 * D * 4);
  // split-K workspace: 16 partial copies of the largest weight gradient
  st->ws_elems = 16 * (size_t)D * (F > 3 * D ? F : 3 * D);
  st->ws = (float*)A(st->ws_elems * 4);
  st->ws2 = (float*)A(st->ws_elems * 4);
  if (cudaStreamCreateWithFlags(&st->side, cudaStreamNonBlocking) != cudaSuccess) {
    st->side = nullptr;
    cudaGetLastError();
  } else {
    st->ev.resize(8 * (size_t)st->layers() + 8);
    for (auto& e : st->ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) ok = false;
  }
  if (!ok) {
    set_error("ppll_vit_stage_create: out of device memory");
    ppll_vit_stage_destroy(st);
    return nullptr;
  }
  return st;
}

void ppll_vit_stage_destroy(ppll_vit_stage* st) {
  if (!st) return;
  for (cudaEvent_t e : st->ev)
    if (e) cudaEventDestroy(e);
  if (st->side) cudaStreamDestroy(st->side);
  for (void* p : st->allocs) cudaFree(p);
  delete st;
}

int ppll_vit_stage_step(ppll_vit_stage* st, int B, const void* x_in, const int64_t* labels,
                        void* x_out, void* stream) {
  if (!st || B < 1 || B > st->Bmax || !x_in || !labels) {
    set_error("ppll_vit_stage_step: invalid arguments (B=%d)", B);
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (st->dtype == PPLL_F32) return vit_step<float>(st, B, x_in, labels, x_out, s);
  return vit_step<__nv_bfloat16>(st, B, x_in, labels, x_out, s);
}

int ppll_vit_stage_forward(ppll_vit_stage* st, int B, const void* x_in, void* h_out,
                           void* logits, void* stream) {
  if (!st || B < 1 || B > st->Bmax) {
    set_error("ppll_vit_stage_forward: invalid arguments");
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int r = st->dtype == PPLL_F32 ? vit_forward<float>(st, B, x_in, h_out, logits != nullptr, s)
                                : vit_forward<__nv_bfloat16>(st, B, x_in, h_out, logits != nullptr, s);
  if (r || !logits) return r;
  PPLL_CUDA_CHECK(cudaMemcpyAsync(logits, st->logits, (size_t)B * st->C * st->esz,
                                  cudaMemcpyDeviceToDevice, s));
  return PPLL_OK;
}

// ---- the paper's baselines: E2E / naive PP (runtime.py:248-284, 359-382) ----
// Block forward only (aux layers and aux head unused).  h_out != NULL: the
// block output is stored there (a non-final stage); h_out == NULL: the final
// stage, whose block ends in the task head (LN on the cls row + classifier).
int ppll_vit_stage_block_forward(ppll_vit_stage* st, int B, const void* x_in, void* h_out,
                                 void* stream) {
  if (!st || B < 1 || B > st->Bmax || !x_in || (!h_out && st->n_aux)) {
    set_error("ppll_vit_stage_block_forward: invalid arguments (B=%d)", B);
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool head = h_out == nullptr;
  return st->dtype == PPLL_F32
             ? vit_forward<float>(st, B, x_in, h_out, head, s, st->n_block, true)
             : vit_forward<__nv_bfloat16>(st, B, x_in, h_out, head, s, st->n_block, true);
}

// Backward through the block from dLoss/d(block output) `g_out`, or — final
// stage, labels != NULL — from the task loss; dLoss/d(block input) into
// `g_in` (NULL for stage 0); then the optimizer over the BLOCK parameters only
// (patch embedding + block layers; + the task head on the final stage).  The
// step counter advances.
int ppll_vit_stage_block_backward(ppll_vit_stage* st, int B, const void* x_in, const void* g_out,
                                  const int64_t* labels, void* g_in, void* stream) {
  if (!st || B < 1 || B > st->Bmax || !x_in || (!g_out && !labels) || (labels && st->n_aux)) {
    set_error("ppll_vit_stage_block_backward: invalid arguments (B=%d)", B);
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t nb = labels ? st->n_params
                            : (st->n_aux ? st->po(st->n_block, 0) : st->ho(0));
  int r = st->dtype == PPLL_F32
              ? vit_backward<float>(st, B, x_in, labels, g_out, g_in, st->n_block, s)
              : vit_backward<__nv_bfloat16>(st, B, x_in, labels, g_out, g_in, st->n_block, s);
  if (r) return r;
  return vit_update(st, nb, s);
}

}  // extern "C"
