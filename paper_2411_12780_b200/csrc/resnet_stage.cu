// Native executor of one ResNet local-learning stage (the PPLL local step,
// blocks.py:266-289 semantics, applied to CIFAR basic blocks; parity vs
// oracle/resnet_oracle.py):
//
//   [stem conv3x3 + BN + ReLU]                         (stage 0 only)
//   blocks : conv3x3(stride) → BN → ReLU → conv3x3 → BN  (+ shortcut: identity
//            or conv1x1(stride) → BN) → add → ReLU; the last block's apply
//            kernel also stores the push (x_out, PRE-update parameters)
//   aux    : N_l × [conv3x3 → BN → ReLU] at the boundary resolution
//   head   : global average pool → linear → softmax-CE
//   backward in reverse (no gradient into the detached stage input), then one
//   Nesterov launch over the flat parameter buffer.
//
// NHWC activations; a convolution is im2col (kept for the weight gradient) ·
// W[k·k·Cin(padded to Kp), Cout] on the tcgen05 GEMM engine; its input
// gradient is (dZ · Wᵀ) → col2im.  BatchNorm uses batch statistics (training
// mode) with deterministic Welford / fixed-order reductions.
#include <stdlib.h>
#include <algorithm>
#include <vector>
#include "common.cuh"
#include "kernels.cuh"
#include "resnet.cuh"

namespace {
struct ConvBN {            // conv (+ its BN) activations kept for the backward
  int cin, cout, k, stride, h_in, h_out, kp;
  char *col, *z;
  float *mean, *rstd;
  const void* x_in = nullptr;   // conv input (implicit path: im2col deferred to the wgrad)
  bool implicit = false;        // forward ran as the implicit-GEMM kernel
};
struct Block {
  ConvBN c1, c2;
  bool has_sc;
  ConvBN sc;
  char *a1, *out;
  int64_t off[9];          // w1 g1 b1 w2 g2 b2 ws gs bs
};
struct Aux {
  ConvBN c;
  char* out;
  int64_t off[3];
};
}  // namespace

struct ppll_resnet_stage {
  int Bmax, img_c, img_hw, classes, has_stem, n_blk, n_aux, dtype;
  size_t esz;
  int64_t n_params;
  float *theta, *grad, *mom;
  void* theta_lp;
  const float* lr_table;
  int* step;
  int max_step;
  float* loss_hist;
  int* err;
  float mu, wd;
  ConvBN stem;
  char* stem_out = nullptr;
  int64_t stem_off[3];
  std::vector<Block> blocks;
  std::vector<Aux> aux;
  int64_t head_off[2];
  int c_out = 0, h_out = 0;
  char *pooled = nullptr, *logits = nullptr, *dlog = nullptr, *dp = nullptr;
  char *dsum = nullptr, *dz = nullptr, *dy = nullptr, *dcol = nullptr, *dxa = nullptr,
       *dxb = nullptr, *dtmp = nullptr;
  float* bn_part = nullptr;
  ppll::BnGrid bng{nullptr, nullptr, nullptr};   // scratch of the grid-form fused BN (main stream)
  float* ws = nullptr;
  size_t ws_elems = 0;
  // weight gradients (im2col + GEMM) on a side stream; the BN-backward output
  // dz is double-buffered so the next conv's BN backward need not wait for
  // the previous conv's weight gradient
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> ev;
  float* ws2 = nullptr;
  char* dz2 = nullptr;
  std::vector<void*> allocs;

  char* alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, (bytes + 255) / 256 * 256) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    return reinterpret_cast<char*>(p);
  }
  const void* W(int64_t o) const {
    return dtype == PPLL_F32 ? (const void*)(theta + o)
                             : (const void*)(reinterpret_cast<const __nv_bfloat16*>(theta_lp) + o);
  }
  const float* P(int64_t o) const { return theta + o; }
  float* G(int64_t o) const { return grad + o; }
};

using namespace ppll;

static int kp_of(int k, int cin) { return (k * k * cin + 7) / 8 * 8; }

static bool make_conv(ppll_resnet_stage* st, ConvBN& c, int cin, int cout, int k, int stride,
                      int h_in) {
  c.cin = cin; c.cout = cout; c.k = k; c.stride = stride; c.h_in = h_in;
  c.h_out = (h_in + 2 * ((k - 1) / 2) - k) / stride + 1;
  c.kp = kp_of(k, cin);
  const size_t P = (size_t)st->Bmax * c.h_out * c.h_out;
  c.col = st->alloc(P * c.kp * st->esz);
  c.z = st->alloc(P * cout * st->esz);
  c.mean = (float*)st->alloc(cout * 4);
  c.rstd = (float*)st->alloc(cout * 4);
  return c.col && c.z && c.mean && c.rstd;
}

static bool use_implicit(const ppll_resnet_stage* st, const ConvBN& c) {
  static const int off = getenv("PPLL_CONV_IMPLICIT") ? !atoi(getenv("PPLL_CONV_IMPLICIT")) : 0;
  return !off && st->dtype == PPLL_BF16 && c.k == 3 && c.stride == 1;
}

// conv; returns z in c.z (BN follows in bn_act).  3x3 stride-1 convolutions
// run as the implicit-GEMM kernel (conv_tc.cu, TMA gathers the shifted
// windows); the rest as im2col · W on the GEMM engine
template <typename TT>
static int conv_fwd(ppll_resnet_stage* st, ConvBN& c, int B, const void* x, int64_t w_off,
                    cudaStream_t s) {
  const int P = B * c.h_out * c.h_out;
  int r = PPLL_ERR_UNSUPPORTED;
  c.implicit = false;
  c.x_in = x;
  if (use_implicit(st, c)) {
    Epilogue<__nv_bfloat16> e;
    e.C = (__nv_bfloat16*)c.z;
    e.ldc = c.cout;
    epilogue_finalize(e, c.cout);
    r = launch_conv3x3_tc(B, c.h_in, c.h_in, c.cin, c.cout, (const __nv_bfloat16*)x,
                          (const __nv_bfloat16*)st->W(w_off), false, e, s);
    if (r != PPLL_OK && r != PPLL_ERR_UNSUPPORTED) return r;
    c.implicit = r == PPLL_OK;
  }
  if (!c.implicit) {
    r = launch_im2col<TT>(B, c.h_in, c.h_in, c.cin, c.k, c.stride, c.kp, (const TT*)x,
                          (TT*)c.col, s);
    if (r) return r;
    LinOpts o;
    r = gemm_fwd(P, c.kp, c.cout, c.col, c.kp, st->W(w_off), o, c.z, c.cout, st->dtype, st->ws,
                 st->ws_elems, s);
  }
  return r;
}

// y = ReLU(BN(c.z) [+ BN2(c2.z) | + res]) with batch statistics (into c.mean /
// c.rstd): one single-cluster launch for bf16 (bn_cluster.cu), else the
// statistics kernels of each BN + the apply kernel.  g/b (g2/b2): parameter
// offsets of the affine terms.
template <typename TT>
static int bn_act(ppll_resnet_stage* st, int P, ConvBN& c, int64_t g, int64_t b, ConvBN* c2,
                  int64_t g2, int64_t b2, const void* res, void* y, cudaStream_t s) {
  if (st->dtype == PPLL_BF16) {
    const int r = launch_bn_fwd_fused(
        P, c.cout, (const __nv_bfloat16*)c.z, st->P(g), st->P(b), c.mean, c.rstd,
        c2 ? (const __nv_bfloat16*)c2->z : nullptr, c2 ? st->P(g2) : nullptr,
        c2 ? st->P(b2) : nullptr, c2 ? c2->mean : nullptr, c2 ? c2->rstd : nullptr,
        (const __nv_bfloat16*)res, 1, (__nv_bfloat16*)y, s, &st->bng);
    if (r != PPLL_ERR_UNSUPPORTED) return r;
  }
  int r = launch_bn_stats<TT>(P, c.cout, (const TT*)c.z, st->bn_part, c.mean, c.rstd, s);
  if (r) return r;
  if (c2) {
    r = launch_bn_stats<TT>(P, c2->cout, (const TT*)c2->z, st->bn_part, c2->mean, c2->rstd, s);
    if (r) return r;
  }
  return launch_bn_apply<TT>(P, c.cout, (const TT*)c.z, c.mean, c.rstd, st->P(g), st->P(b),
                             c2 ? (const TT*)c2->z : nullptr, c2 ? c2->mean : nullptr,
                             c2 ? c2->rstd : nullptr, c2 ? st->P(g2) : nullptr,
                             c2 ? st->P(b2) : nullptr, (const TT*)res, 1, (TT*)y, s);
}

// side-stream state of one backward pass: BN-backward outputs alternate
// between the two dz buffers; dz_done[i] = completion of the weight gradient
// that last read dz[i]
struct BwdSide {
  SideFlow sf;
  char* dz[2];
  cudaEvent_t dz_done[2] = {nullptr, nullptr};
  int k = 0;
  float* wsw;
  int take() {                   // next dz buffer, once its last reader is done
    const int slot = k++ & 1;
    sf.join(dz_done[slot]);
    return slot;
  }
};

// BatchNorm backward of c (and of c2, which shares dy — the projection
// shortcut): dy = dout ⊙ [out > 0] when out != NULL (the ReLU after the add),
// else dout; dγ/dβ into the gradient buffer, dz (dz2).  bf16: one fused
// cluster launch (the masked dy stored only when keep_dy); else ReLU mask into
// `scratch` + the three-kernel BN backward per BN.
template <typename TT>
static int bn_bwd(ppll_resnet_stage* st, int P, ConvBN& c, int64_t g, int64_t b, ConvBN* c2,
                  int64_t g2, int64_t b2, const void* dout, const void* out, char* scratch,
                  bool keep_dy, char* dz, char* dz2, cudaStream_t s) {
  if (st->dtype == PPLL_BF16) {
    const int r = launch_bn_bwd_fused(
        P, c.cout, (const __nv_bfloat16*)dout, (const __nv_bfloat16*)out,
        keep_dy ? (__nv_bfloat16*)scratch : nullptr, (const __nv_bfloat16*)c.z, c.mean, c.rstd,
        st->P(g), st->G(g), st->G(b), (__nv_bfloat16*)dz,
        c2 ? (const __nv_bfloat16*)c2->z : nullptr, c2 ? c2->mean : nullptr,
        c2 ? c2->rstd : nullptr, c2 ? st->P(g2) : nullptr, c2 ? st->G(g2) : nullptr,
        c2 ? st->G(b2) : nullptr, (__nv_bfloat16*)dz2, s, &st->bng);
    if (r != PPLL_ERR_UNSUPPORTED) return r;
  }
  const void* dy = dout;
  int r;
  if (out) {
    r = launch_relu_mask<TT>((long)P * c.cout, (const TT*)dout, (const TT*)out, (TT*)scratch, s);
    if (r) return r;
    dy = scratch;
  }
  r = launch_bn_bwd<TT>(P, c.cout, (const TT*)dy, (const TT*)c.z, c.mean, c.rstd, st->P(g),
                        st->bn_part, st->G(g), st->G(b), (TT*)dz, s);
  if (r || !c2) return r;
  return launch_bn_bwd<TT>(P, c2->cout, (const TT*)dy, (const TT*)c2->z, c2->mean, c2->rstd,
                           st->P(g2), st->bn_part, st->G(g2), st->G(b2), (TT*)dz2, s);
}

// given dz (gradient w.r.t. the conv output, in bs.dz[slot]): the weight
// gradient on the side stream and (if dx) the input gradient (+dres, ⊙mask):
// the transposed implicit convolution, or col2im(dZ·Wᵀ)
template <typename TT>
static int conv_bwd(ppll_resnet_stage* st, ConvBN& c, int B, int slot, int64_t w_off, void* dx,
                    const void* dres, const void* mask, cudaStream_t s, BwdSide& bs) {
  const int P = B * c.h_out * c.h_out;
  char* dz = bs.dz[slot];
  bs.sf.fork();
  int r = PPLL_ERR_UNSUPPORTED;
  if (c.implicit) {
    // implicit-GEMM weight gradient: tap windows gathered by TMA, no im2col
    r = launch_conv3x3_wgrad_tc(B, c.h_in, c.h_in, c.cin, c.cout,
                                (const __nv_bfloat16*)c.x_in, (const __nv_bfloat16*)dz,
                                st->G(w_off), bs.wsw, st->ws_elems, bs.sf.ss);
    if (r != PPLL_OK && r != PPLL_ERR_UNSUPPORTED) return r;
    if (r == PPLL_ERR_UNSUPPORTED) {   // the GEMM still contracts over the im2col'd input
      r = launch_im2col<TT>(B, c.h_in, c.h_in, c.cin, c.k, c.stride, c.kp, (const TT*)c.x_in,
                            (TT*)c.col, bs.sf.ss);
      if (r) return r;
      r = PPLL_ERR_UNSUPPORTED;
    }
  }
  if (r == PPLL_ERR_UNSUPPORTED) {
    r = linear_wgrad(P, c.kp, c.cout, c.col, c.kp, dz, c.cout, st->G(w_off), nullptr,
                     st->dtype, bs.wsw, st->ws_elems, bs.sf.ss);
    if (r) return r;
  }
  bs.dz_done[slot] = bs.sf.mark();
  if (!dx) return r;
  if (c.implicit) {
    Epilogue<__nv_bfloat16> e;
    e.C = (__nv_bfloat16*)dx;
    e.ldc = c.cin;
    e.res = (const __nv_bfloat16*)dres;
    e.ldres = c.cin;
    e.mask = (const __nv_bfloat16*)mask;
    e.ldmask = c.cin;
    e.mask_mode = mask ? kMaskRelu : kMaskNone;
    epilogue_finalize(e, c.cin);
    r = launch_conv3x3_tc(B, c.h_out, c.h_out, c.cout, c.cin, (const __nv_bfloat16*)dz,
                          (const __nv_bfloat16*)st->W(w_off), true, e, s);
    if (r != PPLL_ERR_UNSUPPORTED) return r;
  }
  LinOpts none;
  r = gemm_dgrad(P, c.kp, c.cout, dz, c.cout, st->W(w_off), none, st->dcol, c.kp, st->dtype,
                 st->ws, st->ws_elems, s);
  if (r) return r;
  return launch_col2im<TT>(B, c.h_in, c.h_in, c.cin, c.k, c.stride, c.kp, (const TT*)st->dcol,
                           (const TT*)dres, (const TT*)mask, (TT*)dx, s);
}

template <typename TT>
static int res_forward(ppll_resnet_stage* st, int B, const void* x_in, void* x_out, bool head,
                       cudaStream_t s, bool with_aux = true, bool defer_logits = false) {
  NvtxRange nv("ppll.resnet.forward");
  const void* x = x_in;
  int r;
  if (st->has_stem) {
    ConvBN& c = st->stem;
    r = conv_fwd<TT>(st, c, B, x, st->stem_off[0], s);
    if (r) return r;
    r = bn_act<TT>(st, B * c.h_out * c.h_out, c, st->stem_off[1], st->stem_off[2], nullptr, 0, 0,
                   nullptr, st->stem_out, s);
    if (r) return r;
    x = st->stem_out;
  }
  for (size_t i = 0; i < st->blocks.size(); ++i) {
    Block& b = st->blocks[i];
    const int P = B * b.c1.h_out * b.c1.h_out;
    r = conv_fwd<TT>(st, b.c1, B, x, b.off[0], s);
    if (r) return r;
    r = bn_act<TT>(st, P, b.c1, b.off[1], b.off[2], nullptr, 0, 0, nullptr, b.a1, s);
    if (r) return r;
    r = conv_fwd<TT>(st, b.c2, B, b.a1, b.off[3], s);
    if (r) return r;
    if (b.has_sc) {
      r = conv_fwd<TT>(st, b.sc, B, x, b.off[6], s);
      if (r) return r;
      r = bn_act<TT>(st, P, b.c2, b.off[4], b.off[5], &b.sc, b.off[7], b.off[8], nullptr, b.out, s);
    } else {
      r = bn_act<TT>(st, P, b.c2, b.off[4], b.off[5], nullptr, 0, 0, x, b.out, s);
    }
    if (r) return r;
    x = b.out;
  }
  const long Pout = (long)B * st->h_out * st->h_out;
  if (x_out)   // the push: the block output (pre-update parameters)
    PPLL_CUDA_CHECK(cudaMemcpyAsync(x_out, x, Pout * st->c_out * st->esz, cudaMemcpyDeviceToDevice, s));
  if (!head) return PPLL_OK;
  for (auto& a : st->aux) {
    if (!with_aux) break;
    r = conv_fwd<TT>(st, a.c, B, x, a.off[0], s);
    if (r) return r;
    r = bn_act<TT>(st, (int)Pout, a.c, a.off[1], a.off[2], nullptr, 0, 0, nullptr, a.out, s);
    if (r) return r;
    x = a.out;
  }
  r = launch_gap<TT>(B, st->h_out * st->h_out, st->c_out, (const TT*)x, (TT*)st->pooled, s);
  if (r) return r;
  // a backward follows: the fused head kernel computes the logits there
  if (defer_logits && head_xent_fusable(B, st->c_out, st->classes, st->esz)) return PPLL_OK;
  LinOpts oh;
  oh.bias = st->P(st->head_off[1]);
  return gemm_fwd(B, st->c_out, st->classes, st->pooled, st->c_out, st->W(st->head_off[0]), oh,
                  st->logits, st->classes, st->dtype, st->ws, st->ws_elems, s);
}

// Backward from the loss through the head (labels != NULL; aux layers when
// `with_aux`) or from `g_out` = dLoss/d(block output), through the blocks and
// the stem; dLoss/d(stage input) into `g_in` (NULL: detached input).  Every
// weight gradient has landed on `s` when this returns.
template <typename TT>
static int res_backward(ppll_resnet_stage* st, int B, const int64_t* labels, const void* g_out,
                        void* g_in, bool with_aux, cudaStream_t s) {
  NvtxRange nv("ppll.resnet.backward");
  const int C = st->c_out, HW = st->h_out * st->h_out;
  int r;
  static const bool side_on = !(getenv("PPLL_SIDE_WGRAD") && atoi(getenv("PPLL_SIDE_WGRAD")) == 0);
  const bool side = side_on && st->side && st->dz2;
  BwdSide bs{SideFlow{s, side ? st->side : s, st->ev.data(), 0, (int)st->ev.size()},
             {st->dz, side ? st->dz2 : st->dz}};
  bs.wsw = side ? st->ws2 : st->ws;
  // without a side stream both "buffers" alias: the projection shortcut's two
  // BN gradients then need distinct storage
  char* dz_sc_alias = side ? nullptr : st->dtmp;
  char* dx = st->dxa;
  char* dx_next = st->dxb;
  if (!labels) {
    PPLL_CUDA_CHECK(cudaMemcpyAsync(dx, g_out, (size_t)B * HW * C * st->esz,
                                    cudaMemcpyDeviceToDevice, s));
  } else {
    const bool fused = head_xent_fusable(B, C, st->classes, st->esz);
    if (fused) {   // logits + softmax_xent + dp in one launch (the forward deferred the logits)
      r = launch_head_xent<TT>(B, C, st->classes, (const TT*)st->pooled, C,
                               (const TT*)st->W(st->head_off[0]), st->P(st->head_off[1]), labels,
                               (TT*)st->logits, (TT*)st->dlog, (TT*)st->dp, C, st->loss_hist,
                               st->step, st->err, s);
    } else {
      r = launch_softmax_xent<TT>(B, st->classes, (const TT*)st->logits, st->classes, labels,
                                  (TT*)st->dlog, st->classes, st->loss_hist, st->step, st->err, s);
    }
    if (r) return r;
    // head
    bs.sf.fork();
    r = linear_wgrad(B, C, st->classes, st->pooled, C, st->dlog, st->classes,
                     st->G(st->head_off[0]), st->G(st->head_off[1]), st->dtype, bs.wsw,
                     st->ws_elems, bs.sf.ss);
    if (r) return r;
    LinOpts none;
    if (!fused) {
      r = gemm_dgrad(B, C, st->classes, st->dlog, st->classes, st->W(st->head_off[0]), none,
                     st->dp, C, st->dtype, st->ws, st->ws_elems, s);
      if (r) return r;
    }
    r = launch_gap_bwd<TT>(B, HW, C, (const TT*)st->dp, (TT*)dx, s);
    if (r) return r;
  }
  // aux layers, last first (gradient w.r.t. each aux conv-BN-ReLU output)
  for (int i = with_aux ? (int)st->aux.size() - 1 : -1; i >= 0; --i) {
    Aux& a = st->aux[i];
    const int sl = bs.take();
    r = bn_bwd<TT>(st, B * HW, a.c, a.off[1], a.off[2], nullptr, 0, 0, dx, a.out, st->dy, false,
                   bs.dz[sl], nullptr, s);
    if (r) return r;
    r = conv_bwd<TT>(st, a.c, B, sl, a.off[0], dx_next, nullptr, nullptr, s, bs);
    if (r) return r;
    char* t = dx; dx = dx_next; dx_next = t;
  }
  // blocks, last first
  for (int i = (int)st->blocks.size() - 1; i >= 0; --i) {
    Block& b = st->blocks[i];
    const int P = B * b.c1.h_out * b.c1.h_out;
    const bool need_dx = i > 0 || st->has_stem || g_in;
    // the stage input's gradient goes straight to g_in (no stem below)
    char* dx_dst = (i == 0 && !st->has_stem) ? (char*)g_in : dx_next;
    const void* dres = nullptr;
    if (b.has_sc) {
      // BN2 and the shortcut BN share dy = dx ⊙ [out > 0]: one backward launch
      const int sa = bs.take();
      int sb = bs.take();
      char* dz_sc = dz_sc_alias ? dz_sc_alias : bs.dz[sb];
      r = bn_bwd<TT>(st, P, b.c2, b.off[4], b.off[5], &b.sc, b.off[7], b.off[8], dx, b.out,
                     st->dsum, false, bs.dz[sa], dz_sc, s);
      if (r) return r;
      // conv2: input gradient masked by the ReLU that produced a1 -> dy
      r = conv_bwd<TT>(st, b.c2, B, sa, b.off[3], st->dy, nullptr, b.a1, s, bs);
      if (r) return r;
      if (dz_sc_alias) {   // single stream: dz_sc lives in dtmp, copy it into the slot
        PPLL_CUDA_CHECK(cudaMemcpyAsync(bs.dz[sb], dz_sc, (size_t)P * b.sc.cout * st->esz,
                                        cudaMemcpyDeviceToDevice, s));
      }
      r = conv_bwd<TT>(st, b.sc, B, sb, b.off[6], need_dx ? st->dtmp : nullptr, nullptr, nullptr,
                       s, bs);
      if (r) return r;
      dres = st->dtmp;
    } else {
      const int sa = bs.take();
      r = bn_bwd<TT>(st, P, b.c2, b.off[4], b.off[5], nullptr, 0, 0, dx, b.out, st->dsum, true,
                     bs.dz[sa], nullptr, s);
      if (r) return r;
      r = conv_bwd<TT>(st, b.c2, B, sa, b.off[3], st->dy, nullptr, b.a1, s, bs);
      if (r) return r;
      dres = st->dsum;
    }
    // conv1 (+ shortcut / identity gradient) -> gradient of the block input
    const int s1 = bs.take();
    r = bn_bwd<TT>(st, P, b.c1, b.off[1], b.off[2], nullptr, 0, 0, st->dy, nullptr, nullptr,
                   false, bs.dz[s1], nullptr, s);
    if (r) return r;
    r = conv_bwd<TT>(st, b.c1, B, s1, b.off[0], need_dx ? dx_dst : nullptr, dres, nullptr, s, bs);
    if (r) return r;
    char* t = dx; dx = dx_next; dx_next = t;
  }
  if (st->has_stem) {
    ConvBN& c = st->stem;
    const int sl = bs.take();
    r = bn_bwd<TT>(st, B * c.h_out * c.h_out, c, st->stem_off[1], st->stem_off[2], nullptr, 0, 0,
                   dx, st->stem_out, st->dy, false, bs.dz[sl], nullptr, s);
    if (r) return r;
    r = conv_bwd<TT>(st, c, B, sl, st->stem_off[0], nullptr, nullptr, nullptr, s, bs);
    if (r) return r;
  }
  bs.sf.join(bs.sf.mark());   // every weight gradient has landed
  return PPLL_OK;
}

// optimizer over the first `n` elements of the flat parameter buffer
static int res_update(ppll_resnet_stage* st, int64_t n, cudaStream_t s) {
  NvtxRange nv("ppll.resnet.update");
  return launch_nesterov(n, st->theta, st->mom, st->grad,
                         reinterpret_cast<__nv_bfloat16*>(st->theta_lp), st->lr_table, st->step,
                         st->max_step, 0.f, st->mu, st->wd, st->err, s);
}

template <typename TT>
static int res_step(ppll_resnet_stage* st, int B, const void* x_in, const int64_t* labels,
                    void* x_out, cudaStream_t s) {
  int r = res_forward<TT>(st, B, x_in, x_out, true, s, true, true);
  if (r) return r;
  r = res_backward<TT>(st, B, labels, nullptr, nullptr, true, s);
  if (r) return r;
  return res_update(st, st->n_params, s);
}

extern "C" {

// cfg = {max_batch, img_channels, img_size, classes, has_stem, n_blocks, n_aux, stem_cout}
// geo = 4 ints per block {cin, cout, stride, h_in}; out_geo = {C_out, H_out}
// offsets = stem(3) + 9 per block (ws/gs/bs = -1 without shortcut) + 3 per aux + head(2)
ppll_resnet_stage* ppll_resnet_stage_create(const int* cfg, const int* geo, const int* out_geo,
                                            const int64_t* offsets, int64_t n_params, int dtype,
                                            float* theta, float* grad, float* mom, void* theta_lp,
                                            const float* lr_table, int* step, int max_step,
                                            float* loss_hist, int* err, float mu, float wd) {
  ppll_resnet_stage* st = new ppll_resnet_stage();
  st->Bmax = cfg[0]; st->img_c = cfg[1]; st->img_hw = cfg[2]; st->classes = cfg[3];
  st->has_stem = cfg[4]; st->n_blk = cfg[5]; st->n_aux = cfg[6];
  const int stem_cout = cfg[7];
  st->dtype = dtype;
  st->esz = dtype == PPLL_F32 ? 4 : 2;
  st->n_params = n_params;
  st->theta = theta; st->grad = grad; st->mom = mom; st->theta_lp = theta_lp;
  st->lr_table = lr_table; st->step = step; st->max_step = max_step;
  st->loss_hist = loss_hist; st->err = err; st->mu = mu; st->wd = wd;
  st->c_out = out_geo[0]; st->h_out = out_geo[1];
  if ((dtype != PPLL_F32 && dtype != PPLL_BF16) || (dtype == PPLL_BF16 && !theta_lp) ||
      st->Bmax < 1 || (!st->has_stem && st->n_blk < 1)) {
    set_error("ppll_resnet_stage_create: invalid configuration");
    delete st;
    return nullptr;
  }
  bool ok = true;
  int o = 0;
  size_t maxPC = 0, maxPK = 0, maxC = 16;
  auto track = [&](const ConvBN& c) {
    const size_t P = (size_t)st->Bmax * c.h_out * c.h_out;
    const size_t Pin = (size_t)st->Bmax * c.h_in * c.h_in;
    maxPC = std::max(maxPC, std::max(P * c.cout, Pin * c.cin));
    maxPK = std::max(maxPK, P * c.kp);
    maxC = std::max(maxC, (size_t)c.cout);
  };
  if (st->has_stem) {
    ok = ok && make_conv(st, st->stem, st->img_c, stem_cout, 3, 1, st->img_hw);
    st->stem_out = st->alloc((size_t)st->Bmax * st->img_hw * st->img_hw * stem_cout * st->esz);
    ok = ok && st->stem_out;
    track(st->stem);
  }
  for (int i = 0; i < 3; ++i) st->stem_off[i] = offsets[o++];
  for (int i = 0; i < st->n_blk; ++i) {
    Block b{};
    const int cin = geo[4 * i], cout = geo[4 * i + 1], stride = geo[4 * i + 2], h = geo[4 * i + 3];
    ok = ok && make_conv(st, b.c1, cin, cout, 3, stride, h);
    ok = ok && make_conv(st, b.c2, cout, cout, 3, 1, b.c1.h_out);
    b.has_sc = stride != 1 || cin != cout;
    if (b.has_sc) ok = ok && make_conv(st, b.sc, cin, cout, 1, stride, h);
    const size_t P = (size_t)st->Bmax * b.c1.h_out * b.c1.h_out;
    b.a1 = st->alloc(P * cout * st->esz);
    b.out = st->alloc(P * cout * st->esz);
    ok = ok && b.a1 && b.out;
    for (int k = 0; k < 9; ++k) b.off[k] = offsets[o++];
    track(b.c1); track(b.c2);
    if (b.has_sc) track(b.sc);
    st->blocks.push_back(b);
  }
  for (int i = 0; i < st->n_aux; ++i) {
    Aux a{};
    ok = ok && make_conv(st, a.c, st->c_out, st->c_out, 3, 1, st->h_out);
    a.out = st->alloc((size_t)st->Bmax * st->h_out * st->h_out * st->c_out * st->esz);
    ok = ok && a.out;
    for (int k = 0; k < 3; ++k) a.off[k] = offsets[o++];
    track(a.c);
    st->aux.push_back(a);
  }
  st->head_off[0] = offsets[o++];
  st->head_off[1] = offsets[o++];
  const size_t e = st->esz;
  st->pooled = st->alloc((size_t)st->Bmax * st->c_out * e);
  st->logits = st->alloc((size_t)st->Bmax * st->classes * e);
  st->dlog = st->alloc((size_t)st->Bmax * st->classes * e);
  st->dp = st->alloc((size_t)st->Bmax * st->c_out * e);
  st->dsum = st->alloc(maxPC * e); st->dz = st->alloc(maxPC * e); st->dy = st->alloc(maxPC * e);
  st->dxa = st->alloc(maxPC * e); st->dxb = st->alloc(maxPC * e); st->dtmp = st->alloc(maxPC * e);
  st->dcol = st->alloc(maxPK * e);
  st->bn_part = (float*)st->alloc((size_t)256 * 3 * maxC * 4);     // bn_chunks() <= 256
  st->bng.part = st->alloc((size_t)256 * 128 * 16);
  st->bng.bar = (unsigned*)st->alloc(256);
  st->bng.err = st->err;
  if (st->bng.bar) cudaMemset(st->bng.bar, 0, 256);
  // split-K partials of the largest weight gradient ([9·C, C]) for up to 160 splits
  st->ws_elems = std::max((size_t)1 << 22, (size_t)160 * 9 * maxC * maxC);
  st->ws = (float*)st->alloc(st->ws_elems * 4);
  ok = ok && st->pooled && st->logits && st->dlog && st->dp && st->dsum && st->dz && st->dy &&
       st->dxa && st->dxb && st->dtmp && st->dcol && st->bn_part && st->ws;
  st->ws2 = (float*)st->alloc(st->ws_elems * 4);
  st->dz2 = st->alloc(maxPC * e);
  ok = ok && st->ws2 && st->dz2;
  if (ok && cudaStreamCreateWithFlags(&st->side, cudaStreamNonBlocking) == cudaSuccess) {
    int convs = 2 + (st->has_stem ? 1 : 0) + (int)st->aux.size();
    for (const Block& b : st->blocks) convs += b.has_sc ? 3 : 2;
    st->ev.resize(2 * (size_t)convs + 8);
    for (auto& ev : st->ev)
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) ok = false;
  } else {
    st->side = nullptr;
    cudaGetLastError();
  }
  if (!ok) {
    set_error("ppll_resnet_stage_create: out of device memory");
    ppll_resnet_stage_destroy(st);
    return nullptr;
  }
  return st;
}

void ppll_resnet_stage_destroy(ppll_resnet_stage* st) {
  if (!st) return;
  for (cudaEvent_t ev : st->ev)
    if (ev) cudaEventDestroy(ev);
  if (st->side) cudaStreamDestroy(st->side);
  for (void* p : st->allocs) cudaFree(p);
  delete st;
}

int ppll_resnet_stage_step(ppll_resnet_stage* st, int B, const void* x_in, const int64_t* labels,
                           void* x_out, void* stream) {
  if (!st || B < 1 || B > st->Bmax || !x_in || !labels) {
    set_error("ppll_resnet_stage_step: invalid arguments (B=%d)", B);
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (st->dtype == PPLL_F32) return res_step<float>(st, B, x_in, labels, x_out, s);
  return res_step<__nv_bfloat16>(st, B, x_in, labels, x_out, s);
}

int ppll_resnet_stage_forward(ppll_resnet_stage* st, int B, const void* x_in, void* h_out,
                              void* logits, void* stream) {
  if (!st || B < 1 || B > st->Bmax) {
    set_error("ppll_resnet_stage_forward: invalid arguments");
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int r = st->dtype == PPLL_F32
              ? res_forward<float>(st, B, x_in, h_out, logits != nullptr, s)
              : res_forward<__nv_bfloat16>(st, B, x_in, h_out, logits != nullptr, s);
  if (r || !logits) return r;
  PPLL_CUDA_CHECK(cudaMemcpyAsync(logits, st->logits, (size_t)B * st->classes * st->esz,
                                  cudaMemcpyDeviceToDevice, s));
  return PPLL_OK;
}

// ---- the paper's baselines: E2E / naive PP (runtime.py:248-284, 359-382) ----
// Block forward only (aux convs and aux classifier unused): h_out != NULL
// receives the block output (non-final stage); h_out == NULL is the final
// stage, whose block ends in the task head (GAP + classifier).
int ppll_resnet_stage_block_forward(ppll_resnet_stage* st, int B, const void* x_in, void* h_out,
                                    void* stream) {
  if (!st || B < 1 || B > st->Bmax || !x_in || (!h_out && st->n_aux)) {
    set_error("ppll_resnet_stage_block_forward: invalid arguments (B=%d)", B);
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool head = h_out == nullptr;
  return st->dtype == PPLL_F32 ? res_forward<float>(st, B, x_in, h_out, head, s, false, true)
                               : res_forward<__nv_bfloat16>(st, B, x_in, h_out, head, s, false, true);
}

// Backward through the block from `g_out` = dLoss/d(block output), or — final
// stage, labels != NULL — from the task loss; dLoss/d(block input) into g_in
// (NULL for stage 0); then the optimizer over the BLOCK parameters only (stem
// + basic blocks; + the task head on the final stage).  The step advances.
int ppll_resnet_stage_block_backward(ppll_resnet_stage* st, int B, const void* x_in,
                                     const void* g_out, const int64_t* labels, void* g_in,
                                     void* stream) {
  if (!st || B < 1 || B > st->Bmax || !x_in || (!g_out && !labels) || (labels && st->n_aux)) {
    set_error("ppll_resnet_stage_block_backward: invalid arguments (B=%d)", B);
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t nb = labels ? st->n_params
                            : (st->aux.empty() ? st->head_off[0] : st->aux[0].off[0]);
  int r = st->dtype == PPLL_F32 ? res_backward<float>(st, B, labels, g_out, g_in, false, s)
                                : res_backward<__nv_bfloat16>(st, B, labels, g_out, g_in, false, s);
  if (r) return r;
  return res_update(st, nb, s);
}

}  // extern "C"
