/*
 * ppll.h — C-ABI of the B200-native PPLL (arXiv 2411.12780) local-learning
 * hot path.  Plain pointers, sizes and an opaque CUDA stream handle; no torch
 * types.  Every entry point is stream-ordered and never synchronises the host
 * unless its name says so.
 *
 * The reference (locopipe, /root/reference/pkg/src/locopipe) is pure Python,
 * so "the reference's FFI" is its Python API; each function below names the
 * reference symbol (file:line) whose semantics it implements.  The Python
 * mirror in paper_2411_12780_b200/ binds these via ctypes.
 *
 * dtype codes: PPLL_F32 (parity mode, SIMT fp32 GEMMs) and PPLL_BF16
 * (performance mode: bf16 operands on tcgen05 tensor cores, fp32 accumulate,
 * fp32 master weights/momenta).  Return value: PPLL_OK or a PPLL_ERR_* code;
 * ppll_last_error() describes the last failure on the calling thread.
 */
#ifndef PPLL_H_
#define PPLL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PPLL_ABI_VERSION 1

enum {
  PPLL_OK = 0,
  PPLL_ERR_ARG = 1,       /* DimensionMismatch / ValueError (errors.py:14-15)  */
  PPLL_ERR_CUDA = 2,      /* CUDA runtime failure                              */
  PPLL_ERR_UNSUPPORTED = 3,
  PPLL_ERR_CLOSED = 4,    /* PushAfterClose (errors.py:70-71)                  */
  PPLL_ERR_TIMEOUT = 5
};

enum { PPLL_F32 = 0, PPLL_BF16 = 1 };

/* sticky device error-word bits (one int32 per stage) */
#define PPLL_ERRBIT_LABEL 1   /* LabelOutOfRange  tensor.py:216-219 */
#define PPLL_ERRBIT_LOSS 2    /* NonFiniteError   tensor.py:227     */
#define PPLL_ERRBIT_PARAM 4   /* NonFiniteError   tensor.py:41-43   */
#define PPLL_ERRBIT_STEP 8    /* StepOutOfRange   optim.py:41-42    */
#define PPLL_ERRBIT_GRAD 16   /* NonFiniteError   tensor.py:41-43: a non-finite gradient;
                                 the update is skipped (all-or-nothing) */
#define PPLL_ERRBIT_SYNC 32   /* a device-side grid barrier gave up (watchdog): the stage's
                                 results are invalid — a worker failure, WorkerPanic
                                 (runtime.py:383-386) */

/* GEMM engine selection for the bf16 path (PPLL_GEMM_AUTO picks tcgen05 when
 * the shape/alignment allows, else the SIMT kernel for skinny shapes). */
enum { PPLL_GEMM_AUTO = 0, PPLL_GEMM_SIMT = 1, PPLL_GEMM_TCGEN05 = 2 };

int ppll_abi_version(void);
const char* ppll_last_error(void);
/* number of kernels this library launched since load (process-wide counter) */
uint64_t ppll_launch_count(void);
void ppll_set_gemm_engine(int engine);
/* ViT attention engine: 0 = tcgen05 when supported (bf16, T <= 128), 1 = SIMT */
void ppll_set_attn_engine(int engine);
/* Multi-head self-attention of the ViT blocks (no reference counterpart; the
 * reference's blocks are MLPs): qkv [B*T, 3*H*64] bf16 (q | k | v column
 * blocks), o [B*T, H*64] bf16, lse [B*H*T] fp32 (row log-sum-exp kept for the
 * backward).  Backward: dqkv [B*T, 3*H*64] from dout; bias_part (optional,
 * fp32 [B, 3*H*64]) receives the per-image column sums of dqkv (the qkv bias
 * gradient before the sum over images).  tcgen05 kernels, T <= 128. */
int ppll_attn_fwd_bf16(int B, int T, int H, const void* qkv, void* o, float* lse, void* stream);
int ppll_attn_bwd_bf16(int B, int T, int H, const void* qkv, const void* o, const void* dout,
                       const float* lse, void* dqkv, float* bias_part, void* stream);
/* profiling hook: device buffer of the GEMM timeline probe (PPLL_GEMM_TIMELINE
 * set): 148 CTAs x 4 tiles x {MMA start, MMA done, epilogue done, -} u64 ns */
void* ppll_gemm_timeline(void);

/* ---- primitive ops: tensor.py ------------------------------------------ */

/* Y[M,N] = relu?(X[M,K] · W[K,N] + b[N]); W is stored (in,out) row-major as in
 * blocks.py:193.  Optional Y2 receives an identical copy (the fused push of a
 * block's output into a ring slot, runtime.py:349-353).
 * Replaces matmul tensor.py:137-150, bias_add :170-180, relu :153-157. */
int ppll_linear_fwd(int M, int K, int N, const void* X, int ldx, const void* W,
                    const float* b, void* Y, int ldy, void* Y2, int ldy2,
                    int relu, int dtype, void* stream);

/* dX[M,K] = (dY[M,N] · Wᵀ) ⊙ [mask > 0]  (mask NULL: no mask).
 * Replaces the matmul adjoint dA = g·Bᵀ (tensor.py:148) and the ReLU adjoint
 * g·(x>0) (tensor.py:156-157; subgradient 0 at 0). */
int ppll_linear_dgrad(int M, int K, int N, const void* dY, int lddy, const void* W,
                      const void* mask, int ldmask, void* dX, int lddx, int dtype,
                      void* stream);

/* dW[K,N] = Xᵀ·dY (fp32), db[N] = Σ_rows dY (fp32; NULL to skip).
 * Replaces the matmul adjoint dB = Aᵀ·g (tensor.py:149) and the bias_add
 * adjoint g.sum(axis=0) (tensor.py:179). */
int ppll_linear_wgrad(int M, int K, int N, const void* X, int ldx, const void* dY,
                      int lddy, float* dW, float* db, int dtype, void* stream);

/* Tape primitives (the device GradTape of tensor.py; not the fused hot path).
 * op 0 relu      out = max(a, 0)                 replaces relu      tensor.py:153-157
 * op 1 relu_bwd  out = a · [b > 0] (g, x)        its adjoint (subgradient 0 at 0)
 * op 2 bias_add  out[r,c] = a[r,c] + b[c]        replaces bias_add  tensor.py:170-180
 * op 3 axpby     out = alpha·a + b (b nullable)  add :160-167, scale :183-191, _accumulate :128-132
 * op 4 broadcast out[i] = alpha·a[0]             sum_all adjoint    tensor.py:194-198
 * a/b/out are [rows, cols] of `dtype`; a non-finite output sets
 * PPLL_ERRBIT_PARAM in *err (nullable) — _ensure_finite, tensor.py:41-43. */
int ppll_ew(int op, int64_t rows, int64_t cols, const void* a, const void* b, float alpha,
            void* out, int dtype, int* err, void* stream);
/* out[c] = Σ_r g[r, c] in fp32 (the bias_add adjoint g.sum(axis=0), tensor.py:179) */
int ppll_colsum(int rows, int cols, const void* g, float* out, int dtype, void* stream);
/* *out = Σ x (fp32 result, fixed-order reduction): sum_all, tensor.py:194-198 */
int ppll_sum_all(int64_t n, const void* x, float* out, int dtype, int* err, void* stream);

/* Extended fused epilogues (the transformer-layer forms; same engines):
 *   fwd:   Y = act(X·W + b [+ R]);  act 0 none, 1 ReLU, 2 GELU(erf),
 *          3 GELU with P <- gelu'(pre-activation);  for act 0..2 P (optional)
 *          receives the pre-activation.  Y2 (optional) is an identical copy.
 *   dgrad: dX = (dY·Wᵀ) ∘ f(mask);  mask_mode 1 [mask>0], 2 gelu'(mask),
 *          3 mask (a stored derivative).
 * Replace the same tensor.py:137-180 ops plus the extension families' GELU /
 * residual fusions (no reference counterpart). */
int ppll_linear_fwd_ex(int M, int K, int N, const void* X, int ldx, const void* W,
                       const float* b, const void* R, int ldr, int act, void* P, int ldp,
                       void* Y, int ldy, void* Y2, int ldy2, int dtype, void* stream);
int ppll_linear_dgrad_ex(int M, int K, int N, const void* dY, int lddy, const void* W,
                         const void* mask, int ldmask, int mask_mode, void* dX, int lddx,
                         int dtype, void* stream);

/* Fused mean softmax cross-entropy forward + adjoint (tensor.py:201-234):
 * loss = mean_b −log softmax(z_b)[y_b] (max-subtracted), dz = (softmax −
 * onehot)/B.  The scalar loss is written to loss_hist[*step] (step may be
 * NULL → index 0).  Out-of-range labels set PPLL_ERRBIT_LABEL, a non-finite
 * loss sets PPLL_ERRBIT_LOSS in *err (err may be NULL). */
int ppll_softmax_xent(int B, int C, const void* logits, int ldz, const int64_t* labels,
                      void* dlogits, int lddz, float* loss_hist, const int* step,
                      int* err, int dtype, void* stream);

/* ---- optimizer: optim.py ----------------------------------------------- */

/* One Nesterov-SGD step over a flat parameter buffer (optim.py:71-89):
 *   g' = g + wd·θ;  v = μ·v + g';  θ −= lr·(g' + μ·v)
 * lr = lr_table[*step] when step != NULL (device-resident cosine table,
 * CUDA-graph safe), else lr_host.  When step != NULL the kernel's last block
 * advances *step by one (OptimizerState.step_count += 1, optim.py:89) and sets
 * PPLL_ERRBIT_STEP if *step > max_step.  theta_lp (nullable) receives a bf16
 * shadow copy of the updated θ for the tensor-core path. */
int ppll_nesterov_step(int64_t n, float* theta, float* v, const float* g, void* theta_lp,
                       const float* lr_table, int* step, int max_step, float lr_host,
                       float mu, float wd, int* err, void* stream);

/* The local optimizer of the stage whose flat parameter buffer is `theta`:
 * kind 0 = Nesterov-SGD (the reference's, optim.py:71-89; the default),
 * kind 1 = AdamW (north_star's "local SGD/Adam update"; no reference
 * counterpart — torch.optim.AdamW semantics: decoupled weight decay
 * θ -= lr·wd·θ, bias-corrected moments, t = step + 1).  m2 (second moment,
 * same length as theta) is owned by the caller; the first moment is the
 * buffer passed as `v`.  Every later update of that buffer — the fused stage
 * steps and ppll_nesterov_step — applies the registered rule. */
int ppll_set_local_optimizer(const float* theta, int kind, float* m2, float beta1, float beta2,
                             float eps);

/* cosine_lr (optim.py:39-44), fp64 on the host; returns NaN if out of range */
double ppll_cosine_lr(int step, double lr0, double lr_min, int total_steps);

/* element conversion helpers (fp32 <-> bf16), n elements */
/* Implicit-GEMM 3x3 convolution, stride 1, pad 1, NHWC bf16 (tcgen05, TMA
 * gathers the shifted windows — no im2col matrix).  w is the GEMM weight
 * [9·Cin, Cout] (row tap·Cin + ci, tap = 3r + s).  dgrad = 0: y[N,H,W,Cout] =
 * conv(x[N,H,W,Cin]); dgrad = 1: y[N,H,W,Cin] = the input gradient for
 * x = dZ[N,H,W,Cout] (transposed convolution).  Cin, Cout ∈ {16, 32, 64},
 * N·H·W % 128 == 0; PPLL_ERR_UNSUPPORTED otherwise.  The ResNet stages'
 * stride-1 convolutions (the extension family; no reference counterpart). */
int ppll_conv3x3_bf16(int N, int H, int W, int Cin, int Cout, const void* x, const void* w,
                      void* y, int dgrad, void* stream);
/* The same convolution with the ResNet stage's fused epilogue:
 * y = (conv + res) ⊙ [mask > 0] — res (same shape as y) and mask (the
 * producing ReLU's output, same shape as y) may be NULL.  With dgrad = 1 this
 * is the basic block's input-gradient epilogue: the shortcut gradient added
 * and the previous ReLU's mask applied (blocks.py's backward of relu(bn(conv))
 * + residual; resnet_stage.cu conv_bn_bwd). */
int ppll_conv3x3_bf16_ex(int N, int H, int W, int Cin, int Cout, const void* x, const void* w,
                         void* y, int dgrad, const void* res, const void* mask, void* stream);
/* Weight gradient of the same convolution as an implicit GEMM (the matmul
 * adjoint dW = Xᵀ·dY of tensor.py:145-150 with X the im2col'd input, which is
 * never materialised): dw [9·Cin, Cout] fp32 (the GEMM weight layout) from
 * x [N,H,W,Cin] and dz = dLoss/dconv-output [N·H·W, Cout]; ws holds the
 * split-K partials (at least ppll_conv3x3_wgrad_ws_floats floats).  Fixed-
 * order reduction (deterministic).  Same shape range as ppll_conv3x3_bf16. */
long ppll_conv3x3_wgrad_ws_floats(int N, int H, int W, int Cin, int Cout);
int ppll_conv3x3_wgrad_bf16(int N, int H, int W, int Cin, int Cout, const void* x, const void* dz,
                            float* dw, float* ws, long ws_floats, void* stream);

/* ---- data path / evaluation -------------------------------------------- */
/* dst[r,:] = cast(src[idx[r],:]) for r < n (fp32 rows of `width` features,
 * dst fp32 or bf16), and labels_dst[r] = labels_src[idx[r]] when given: the
 * batch assembly of BatchIterator.__next__ (data.py:169-173) from an
 * HBM-resident dataset. */
int ppll_gather_rows(int n, int64_t width, const float* src, const int64_t* idx, void* dst,
                     int dst_dtype, const int64_t* labels_src, int64_t* labels_dst, void* stream);
/* Programmatic dependent launch on (1) / off (0) for kernels the CALLING
 * THREAD launches (or captures into graphs) from now on; returns that
 * thread's previous setting.  On by default (PPLL_PDL=0 in the environment
 * turns it off). */
int ppll_set_pdl(int on);
/* 1 (default; PPLL_GPU_EXCLUSIVE=0 in the environment flips it): the stage
 * steps the CALLING THREAD launches own their GPU, so full-GPU cooperative
 * kernels (the grid form of the fused BatchNorm) may be used; 0: several stage
 * streams share the GPU (the single-GPU pipeline) and only kernels that leave
 * SMs to the other streams are launched.  Returns the previous setting. */
int ppll_set_gpu_exclusive(int on);
/* out_ms[i] = milliseconds from event `ref` to events[i] (cudaEvent_t
 * handles, all recorded and complete): the per-step timestamps behind
 * EpochMetrics busy / wall time (runtime.py:340-354, 383-406), read in one
 * call instead of one driver round trip per event. */
int ppll_events_elapsed(int n, const uint64_t* events, uint64_t ref, float* out_ms);
/* Same gather from a dataset held as the IDX file's pixel bytes (uint8):
 * dst[r,c] = src[idx[r],c] / 255 (IEEE division, then the dst cast) — the
 * [0,1] scaling of load_idx (data.py:137-139) applied per batch on the
 * device, so the resident dataset costs 1 B per feature. */
int ppll_gather_rows_u8(int n, int64_t width, const uint8_t* src, const int64_t* idx, void* dst,
                        int dst_dtype, const int64_t* labels_src, int64_t* labels_dst,
                        void* stream);
/* *count += #{r < B : argmax_c logits[r,c] == labels[r]} (first maximum, as
 * numpy's argmax): the accuracy count of evaluate (harness.py:121-131). */
int ppll_count_correct(int B, int C, const void* logits, int ldz, int dtype,
                       const int64_t* labels, unsigned long long* count, void* stream);

int ppll_cast(int64_t n, const void* src, int src_dtype, void* dst, int dst_dtype, void* stream);

/* ---- one local step of a stage: blocks.py:266-289 ----------------------- */

typedef struct ppll_stage ppll_stage;

/* Layers 0..n_block-1 are the block, n_block..n_layers-1 the aux head
 * (blocks.py:147-187).  param_offsets[2*i] / [2*i+1] are the element offsets
 * of W_i / b_i inside the flat fp32 buffers theta/grad/mom (and theta_lp, bf16,
 * same offsets).  The stage keeps device scratch of its own (activations and
 * two gradient ping-pong buffers for max_batch rows). */
ppll_stage* ppll_stage_create(int n_layers, int n_block, const int* in_w, const int* out_w,
                              const int* relu_after, const int64_t* param_offsets,
                              int64_t n_params, int max_batch, int dtype, float* theta,
                              float* grad, float* mom, void* theta_lp, const float* lr_table,
                              int* step, int max_step, float* loss_hist, int* err, float mu,
                              float wd);
void ppll_stage_destroy(ppll_stage* st);

/* The whole PPLL local step, stream-ordered, no host sync:
 * block forward (last epilogue also stores into x_out = the push, which
 * reflects PRE-update params, blocks.py:279-283) → aux forward → softmax-CE →
 * backward (no dX for the detached block input, blocks.py:277-278) →
 * cosine-LR Nesterov over every stage param (blocks.py:287-288). */
int ppll_stage_step(ppll_stage* st, int B, const void* x_in, const int64_t* labels,
                    void* x_out, void* stream);

/* forward only (block_forward / aux_forward, blocks.py:249-263): writes the
 * block output to h_out and, if logits != NULL, the local logits. */
int ppll_stage_forward(ppll_stage* st, int B, const void* x_in, void* h_out, void* logits,
                       void* stream);

/* The paper's comparison baselines, E2E and naive PP (runtime.py:248-284,
 * 294-408 with ppll=False, 423-465): block-only forward keeping activations;
 * block backward from dLoss/d(block output) g_out (or, final stage, from the
 * task loss on the block output when labels != NULL; loss recorded like a
 * local step), writing dLoss/d(block input) into g_in (NULL: untracked
 * input), then the Nesterov step over the block parameters only. */
int ppll_stage_block_forward(ppll_stage* st, int B, const void* x_in, void* h_out, void* stream);
int ppll_stage_block_backward(ppll_stage* st, int B, const void* x_in, const void* g_out,
                              const int64_t* labels, void* g_in, void* stream);

/* ---- one local step of a ViT stage (same step semantics, blocks.py:266-289,
 * applied to pre-LN transformer blocks; no reference implementation exists —
 * parity is pinned to oracle/vit_oracle.py) -------------------------------
 * cfg[12] = {max_batch, tokens, dim, heads, mlp, classes, n_block_layers,
 *            n_aux_layers, has_patch_embed, img_channels, img_size, patch}
 * offsets = [wpe, bpe, cls, pos] (stage 0; ignored otherwise)
 *         + 12 per transformer layer (ln1_g, ln1_b, wqkv, bqkv, wo, bo, ln2_g,
 *           ln2_b, w1, b1, w2, b2), block layers then aux layers
 *         + [lnf_g, lnf_b, wh, bh] (aux head, or the task head on the final stage)
 * Activations are [batch*tokens, dim] row-major; stage 0 takes images
 * [batch, C, H, W] in the activation dtype. */
typedef struct ppll_vit_stage ppll_vit_stage;
ppll_vit_stage* ppll_vit_stage_create(const int* cfg, const int64_t* offsets, int64_t n_params,
                                      int dtype, float* theta, float* grad, float* mom,
                                      void* theta_lp, const float* lr_table, int* step,
                                      int max_step, float* loss_hist, int* err, float mu,
                                      float wd);
void ppll_vit_stage_destroy(ppll_vit_stage* st);
int ppll_vit_stage_step(ppll_vit_stage* st, int B, const void* x_in, const int64_t* labels,
                        void* x_out, void* stream);
int ppll_vit_stage_forward(ppll_vit_stage* st, int B, const void* x_in, void* h_out,
                           void* logits, void* stream);
/* The paper's E2E / naive-PP baselines for the ViT family (reference
 * runtime.py:248-284 E2E, :359-382 NaivePP; the reference's own blocks are
 * MLPs): block forward only (h_out != NULL: non-final stage, output stored
 * there; h_out == NULL: final stage, block + task head), and backward from
 * g_out = dLoss/d(block output) or, on the final stage, from the task loss
 * (labels), with dLoss/d(block input) into g_in (NULL on stage 0), then the
 * optimizer over the block parameters only. */
int ppll_vit_stage_block_forward(ppll_vit_stage* st, int B, const void* x_in, void* h_out,
                                 void* stream);
int ppll_vit_stage_block_backward(ppll_vit_stage* st, int B, const void* x_in, const void* g_out,
                                  const int64_t* labels, void* g_in, void* stream);

/* ---- one local step of a ResNet stage (CIFAR basic blocks, NHWC; no
 * reference implementation — parity pinned to oracle/resnet_oracle.py) ----
 * cfg[8]  = {max_batch, img_channels, img_size, classes, has_stem, n_blocks,
 *            n_aux_convs, stem_cout}
 * geo     = 4 ints per block {cin, cout, stride, h_in}; out_geo = {C, H} of
 *           the stage output (aux convs and the head run at this size)
 * offsets = stem {w, bn_g, bn_b} (ignored without stem) + 9 per block
 *           {w1, g1, b1, w2, g2, b2, ws, gs, bs} (-1 without a shortcut conv)
 *           + 3 per aux conv {w, g, b} + head {w, b}.  Conv weights are
 *           [round_up(k·k·Cin, 8), Cout] row-major (tap-major rows). */
typedef struct ppll_resnet_stage ppll_resnet_stage;
ppll_resnet_stage* ppll_resnet_stage_create(const int* cfg, const int* geo, const int* out_geo,
                                            const int64_t* offsets, int64_t n_params, int dtype,
                                            float* theta, float* grad, float* mom, void* theta_lp,
                                            const float* lr_table, int* step, int max_step,
                                            float* loss_hist, int* err, float mu, float wd);
void ppll_resnet_stage_destroy(ppll_resnet_stage* st);
int ppll_resnet_stage_step(ppll_resnet_stage* st, int B, const void* x_in, const int64_t* labels,
                           void* x_out, void* stream);
int ppll_resnet_stage_forward(ppll_resnet_stage* st, int B, const void* x_in, void* h_out,
                              void* logits, void* stream);
/* E2E / naive-PP baselines for the ResNet family (same contract as the ViT
 * pair above; runtime.py:248-284, 359-382). */
int ppll_resnet_stage_block_forward(ppll_resnet_stage* st, int B, const void* x_in, void* h_out,
                                    void* stream);
int ppll_resnet_stage_block_backward(ppll_resnet_stage* st, int B, const void* x_in,
                                     const void* g_out, const int64_t* labels, void* g_in,
                                     void* stream);

/* ---- stage-boundary ring (runtime.py:52-120 StageBuffer) ----------------
 * Device-resident flag words for an SPSC ring of `capacity` slots.  ready[i]
 * holds the sequence number (batch_id+1) published into slot i; credit holds
 * the number of slots the consumer has released.  Publication is a
 * release-store at system scope after the slot payload; waits are acquire
 * spins on the device (no host round trip), usable inside CUDA graphs and
 * across NVLink peers (flags may live in peer memory mapped via CUDA IPC). */
int ppll_ring_publish(int* ready_word, int seq, void* stream);
int ppll_ring_wait(const int* ready_word, int seq, void* stream);
int ppll_ring_release(int* credit_word, void* stream);
int ppll_ring_wait_credit(const int* credit_word, int need, void* stream);
/* ---- normalisation kernels of the extension families (no reference: its
 * blocks are MLPs, blocks.py:240-255; SURVEY §8b lists them below the
 * boundary).  Row-major [rows, features], dtype PPLL_F32 or PPLL_BF16;
 * statistics, gamma / beta and their gradients are fp32.
 * LayerNorm (eps 1e-5): mean / rstd per row.  Backward: dx (nullable) =
 * LN-backward(dy) [+ dres]; dg / db (nullable) the gamma / beta gradients;
 * dxsum (nullable) = Σ_rows dx (the fused bias gradient of the layer below);
 * ws: ppll_layernorm_bwd_ws_floats(M, D) floats.
 * BatchNorm (train mode, biased variance, eps 1e-5) over the rows of an NHWC
 * [P, C] tensor: forward = batch statistics + apply (+ res, + ReLU);
 * backward from dy to dz with dg / db; ws: ppll_batchnorm_ws_floats(P, C). */
long ppll_layernorm_bwd_ws_floats(int M, int D);
int ppll_layernorm_fwd(int M, int D, const void* x, long ldx, const float* g, const float* b,
                       void* y, long ldy, float* mean, float* rstd, int dtype, void* stream);
int ppll_layernorm_bwd(int M, int D, const void* dy, long lddy, const void* x, long ldx,
                       const float* mean, const float* rstd, const float* g, const void* dres,
                       long ldres, void* dx, long lddx, float* dg, float* db, float* dxsum,
                       float* ws, long ws_floats, int dtype, void* stream);
long ppll_batchnorm_ws_floats(int P, int C);
int ppll_batchnorm_fwd(int P, int C, const void* z, const float* g, const float* b,
                       const void* res, int relu, void* y, float* mean, float* rstd, float* ws,
                       long ws_floats, int dtype, void* stream);
int ppll_batchnorm_bwd(int P, int C, const void* dy, const void* z, const float* mean,
                       const float* rstd, const float* g, float* dg, float* db, void* dz,
                       float* ws, long ws_floats, int dtype, void* stream);

/* Ring watchdog (no reference counterpart: the reference's threaded queues
 * poll a stop flag, runtime.py:411-418): a wait that sees no progress for the
 * timeout (default 30 s, PPLL_RING_TIMEOUT_MS; <= 0 disables) gives up instead
 * of hanging the GPU and records the first stall.  ppll_ring_stall returns
 * 1 if a wait timed out, with out4 = {1, wanted, seen, kind (0 ready, 1
 * credit)}; clear != 0 re-arms it. */
void ppll_set_ring_timeout_ms(long long ms);
int ppll_ring_stall(int* out4, int clear);

/* ---- P2P / IPC plumbing for the multi-GPU ring -------------------------- */
int ppll_ipc_get_handle(void* dev_ptr, void* handle_out /* 64 bytes */);
int ppll_ipc_open_handle(const void* handle /* 64 bytes */, void** dev_ptr_out);
int ppll_ipc_close_handle(void* dev_ptr);
int ppll_enable_peer(int peer_device);

/* stream-ordered byte copy between any two device pointers (incl. IPC-mapped
 * peer memory): the labels travelling with a pushed batch (runtime.py:353) */
int ppll_copy_async(void* dst, const void* src, size_t bytes, void* stream);

/* runtime-owned device memory (ring slots/flags; IPC-exportable) */
void* ppll_dev_alloc(size_t bytes);   /* zero-filled; NULL on failure */
int ppll_dev_free(void* dev_ptr);

/* synchronising helpers (host waits) */
int ppll_stream_sync(void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PPLL_H_ */
