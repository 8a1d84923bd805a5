// Native per-stage executor: one PPLL local step (blocks.py:266-289) issued as
// a fixed, stream-ordered kernel sequence with no host synchronisation, so it
// can be captured into a CUDA graph per (stage, ring slot).
//
// Memory layout (all device-resident, sized once at create time):
//   theta/grad/mom : flat fp32 buffers of every stage parameter, W_i as
//                    [in, out] row-major like blocks.py:193, 256-B aligned
//                    offsets; the Nesterov step is ONE launch over them.
//   theta_lp       : bf16 shadow of theta written by the Nesterov kernel
//                    (tensor-core operands in PPLL_BF16 mode).
//   act            : per-layer outputs [max_batch, out_w[i]] (kept for the
//                    backward ReLU masks and weight gradients).
//   g0/g1          : gradient ping-pong [max_batch, max_width].
//   ws             : split-K workspace.
#include <vector>
#include "common.cuh"
#include "kernels.cuh"

struct ppll_stage {
  int n_layers = 0, n_block = 0, dtype = PPLL_F32, max_batch = 0;
  std::vector<int> in_w, out_w, relu;
  std::vector<int64_t> off;
  int64_t n_params = 0;
  float *theta = nullptr, *grad = nullptr, *mom = nullptr;
  void* theta_lp = nullptr;
  const float* lr_table = nullptr;
  int* step = nullptr;
  int max_step = 0;
  float* loss_hist = nullptr;
  int* err = nullptr;
  float mu = 0.9f, wd = 1e-4f;
  char* act = nullptr;
  std::vector<size_t> act_off;   // bytes
  char* g0 = nullptr;
  char* g1 = nullptr;
  char* g2 = nullptr;             // third gradient buffer (side-stream weight gradients)
  float* ws = nullptr;
  size_t ws_elems = 0;
  // weight gradients on a side stream, each layer's concurrent with its dgrad
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> ev;
  float* ws2 = nullptr;
  size_t esz = 4;

  void* act_ptr(int i) const { return act + act_off[i]; }
  const void* w_ptr(int i) const {
    if (dtype == PPLL_F32) return theta + off[2 * i];
    return reinterpret_cast<const __nv_bfloat16*>(theta_lp) + off[2 * i];
  }
  const float* b_ptr(int i) const { return theta + off[2 * i + 1]; }
};

using namespace ppll;

extern "C" {

ppll_stage* ppll_stage_create(int n_layers, int n_block, const int* in_w, const int* out_w,
                              const int* relu_after, const int64_t* param_offsets,
                              int64_t n_params, int max_batch, int dtype, float* theta,
                              float* grad, float* mom, void* theta_lp, const float* lr_table,
                              int* step, int max_step, float* loss_hist, int* err, float mu,
                              float wd) {
  if (n_layers < 1 || n_block < 1 || n_block > n_layers || max_batch < 1 ||
      (dtype != PPLL_F32 && dtype != PPLL_BF16) || !theta || !grad || !mom ||
      (dtype == PPLL_BF16 && !theta_lp)) {
    set_error("ppll_stage_create: invalid arguments");
    return nullptr;
  }
  for (int i = 0; i + 1 < n_layers; ++i)
    if (out_w[i] != in_w[i + 1]) {
      set_error("ppll_stage_create: layer %d width %d != layer %d input %d", i, out_w[i], i + 1,
                in_w[i + 1]);
      return nullptr;
    }
  ppll_stage* st = new ppll_stage();
  st->n_layers = n_layers;
  st->n_block = n_block;
  st->dtype = dtype;
  st->max_batch = max_batch;
  st->in_w.assign(in_w, in_w + n_layers);
  st->out_w.assign(out_w, out_w + n_layers);
  st->relu.assign(relu_after, relu_after + n_layers);
  st->off.assign(param_offsets, param_offsets + 2 * n_layers);
  st->n_params = n_params;
  st->theta = theta; st->grad = grad; st->mom = mom; st->theta_lp = theta_lp;
  st->lr_table = lr_table; st->step = step; st->max_step = max_step;
  st->loss_hist = loss_hist; st->err = err; st->mu = mu; st->wd = wd;
  st->esz = dtype == PPLL_F32 ? 4 : 2;
  size_t bytes = 0;
  int maxw = in_w[0];
  for (int i = 0; i < n_layers; ++i) {
    st->act_off.push_back(bytes);
    size_t b = (size_t)max_batch * out_w[i] * st->esz;
    bytes += (b + 255) / 256 * 256;
    maxw = out_w[i] > maxw ? out_w[i] : maxw;
    maxw = in_w[i] > maxw ? in_w[i] : maxw;
  }
  size_t gbytes = ((size_t)max_batch * maxw * st->esz + 255) / 256 * 256;
  // split-K workspace: enough for 16 partial copies of the largest weight grad
  size_t maxwn = 0;
  for (int i = 0; i < n_layers; ++i) {
    size_t a = (size_t)in_w[i] * out_w[i], c = (size_t)max_batch * (in_w[i] > out_w[i] ? in_w[i] : out_w[i]);
    maxwn = a > maxwn ? a : maxwn;
    maxwn = c > maxwn ? c : maxwn;
  }
  st->ws_elems = 16 * maxwn;
  if (cudaMalloc(&st->act, bytes) != cudaSuccess || cudaMalloc(&st->g0, gbytes) != cudaSuccess ||
      cudaMalloc(&st->g1, gbytes) != cudaSuccess ||
      cudaMalloc(&st->ws, st->ws_elems * sizeof(float)) != cudaSuccess) {
    cudaGetLastError();
    set_error("ppll_stage_create: out of device memory");
    ppll_stage_destroy(st);
    return nullptr;
  }
  // split-K tickets live at the end of the workspace and must start at zero
  cudaMemset(st->ws, 0, st->ws_elems * sizeof(float));
  if (cudaMalloc(&st->g2, gbytes) == cudaSuccess &&
      cudaMalloc(&st->ws2, st->ws_elems * sizeof(float)) == cudaSuccess &&
      cudaStreamCreateWithFlags(&st->side, cudaStreamNonBlocking) == cudaSuccess) {
    cudaMemset(st->ws2, 0, st->ws_elems * sizeof(float));
    st->ev.resize(2 * (size_t)n_layers + 4);
    for (auto& e : st->ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) e = nullptr;
    for (auto e : st->ev)
      if (!e) { st->ev.clear(); break; }
  }
  cudaGetLastError();
  if (st->ev.empty() && st->side) { cudaStreamDestroy(st->side); st->side = nullptr; }
  return st;
}

void ppll_stage_destroy(ppll_stage* st) {
  if (!st) return;
  if (st->act) cudaFree(st->act);
  if (st->g0) cudaFree(st->g0);
  if (st->g1) cudaFree(st->g1);
  if (st->g2) cudaFree(st->g2);
  if (st->ws) cudaFree(st->ws);
  if (st->ws2) cudaFree(st->ws2);
  for (cudaEvent_t e : st->ev)
    if (e) cudaEventDestroy(e);
  if (st->side) cudaStreamDestroy(st->side);
  delete st;
}

static int forward_layers(ppll_stage* st, int B, const void* x_in, void* x_out, cudaStream_t s) {
  for (int i = 0; i < st->n_layers; ++i) {
    const void* in = i == 0 ? x_in : st->act_ptr(i - 1);
    void* dual = (i == st->n_block - 1) ? x_out : nullptr;
    int r = linear_fwd(B, st->in_w[i], st->out_w[i], in, st->in_w[i], st->w_ptr(i), st->b_ptr(i),
                       st->act_ptr(i), st->out_w[i], dual, st->out_w[i], st->relu[i], st->dtype,
                       st->ws, st->ws_elems, s);
    if (r) return r;
  }
  return PPLL_OK;
}

int ppll_stage_step(ppll_stage* st, int B, const void* x_in, const int64_t* labels, void* x_out,
                    void* stream) {
  NvtxRange nv("ppll.mlp.step");
  if (!st || B < 1 || B > st->max_batch || !x_in || !labels) {
    set_error("ppll_stage_step: invalid arguments (B=%d)", B);
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // 1. block + aux forward; the last block epilogue dual-stores the push
  int r = forward_layers(st, B, x_in, x_out, s);
  if (r) return r;
  // 2. local loss and its adjoint
  const int L = st->n_layers - 1;
  const int C = st->out_w[L];
  if (st->dtype == PPLL_F32)
    r = launch_softmax_xent<float>(B, C, (const float*)st->act_ptr(L), C, labels, (float*)st->g0,
                                   C, st->loss_hist, st->step, st->err, s);
  else
    r = launch_softmax_xent<__nv_bfloat16>(B, C, (const __nv_bfloat16*)st->act_ptr(L), C, labels,
                                           (__nv_bfloat16*)st->g0, C, st->loss_hist, st->step,
                                           st->err, s);
  if (r) return r;
  // 3. backward, last layer first; no dX for the detached block input.  The
  // weight gradient of layer i runs on the side stream beside its dgrad; the
  // layer gradients rotate over three buffers, and a dgrad waits for the
  // weight gradient that last read the buffer it overwrites.
  static const bool side_on = !(getenv("PPLL_SIDE_WGRAD") && atoi(getenv("PPLL_SIDE_WGRAD")) == 0);
  const bool side = side_on && st->side && st->g2;
  SideFlow sf{s, side ? st->side : s, st->ev.data(), 0, (int)st->ev.size()};
  char* buf[3] = {st->g0, st->g1, side ? st->g2 : st->g0};
  cudaEvent_t read_done[3] = {nullptr, nullptr, nullptr};
  int cur = 0;
  for (int i = L; i >= 0; --i) {
    const void* in = i == 0 ? x_in : st->act_ptr(i - 1);
    sf.fork();
    r = linear_wgrad(B, st->in_w[i], st->out_w[i], in, st->in_w[i], buf[cur], st->out_w[i],
                     st->grad + st->off[2 * i], st->grad + st->off[2 * i + 1], st->dtype,
                     sf.on() ? st->ws2 : st->ws, st->ws_elems, sf.ss);
    if (r) return r;
    read_done[cur] = sf.mark();
    if (i > 0) {
      const int nxt = side ? (cur + 1) % 3 : 1 - cur;
      sf.join(read_done[nxt]);
      const void* mask = st->relu[i - 1] ? st->act_ptr(i - 1) : nullptr;
      r = linear_dgrad(B, st->in_w[i], st->out_w[i], buf[cur], st->out_w[i], st->w_ptr(i), mask,
                       st->in_w[i], buf[nxt], st->in_w[i], st->dtype, st->ws, st->ws_elems, s);
      if (r) return r;
      cur = nxt;
    }
  }
  sf.join(sf.mark());   // every weight gradient has landed
  // 4. cosine-LR Nesterov over all stage params (block + aux), one launch
  return launch_nesterov(st->n_params, st->theta, st->mom, st->grad,
                         reinterpret_cast<__nv_bfloat16*>(st->theta_lp), st->lr_table, st->step,
                         st->max_step, 0.f, st->mu, st->wd, st->err, s);
}

int ppll_stage_forward(ppll_stage* st, int B, const void* x_in, void* h_out, void* logits,
                       void* stream) {
  if (!st || B < 1 || B > st->max_batch) {
    set_error("ppll_stage_forward: invalid arguments");
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int r = forward_layers(st, B, x_in, h_out, s);
  if (r) return r;
  if (logits) {
    const int L = st->n_layers - 1;
    PPLL_CUDA_CHECK(cudaMemcpyAsync(logits, st->act_ptr(L), (size_t)B * st->out_w[L] * st->esz,
                                    cudaMemcpyDeviceToDevice, s));
  }
  return PPLL_OK;
}

// ---- the paper's baselines: E2E / naive PP (runtime.py:248-284, 359-382) ----
// Block forward only (aux heads unused), activations kept for the backward.
int ppll_stage_block_forward(ppll_stage* st, int B, const void* x_in, void* h_out, void* stream) {
  if (!st || B < 1 || B > st->max_batch || !x_in) {
    set_error("ppll_stage_block_forward: invalid arguments (B=%d)", B);
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  for (int i = 0; i < st->n_block; ++i) {
    const void* in = i == 0 ? x_in : st->act_ptr(i - 1);
    void* dual = (i == st->n_block - 1) ? h_out : nullptr;
    int r = linear_fwd(B, st->in_w[i], st->out_w[i], in, st->in_w[i], st->w_ptr(i), st->b_ptr(i),
                       st->act_ptr(i), st->out_w[i], dual, st->out_w[i], st->relu[i], st->dtype,
                       st->ws, st->ws_elems, s);
    if (r) return r;
  }
  return PPLL_OK;
}

// Backward through the block from dLoss/d(block output) `g_out` (after the
// block's last ReLU), or — final stage, labels != NULL — from the task loss
// on the block output; dLoss/d(block input) into `g_in` (NULL for stage 0,
// whose input is the untracked data); then Nesterov over the BLOCK
// parameters only (runtime.py:280-281, 378-380).  The step counter advances.
int ppll_stage_block_backward(ppll_stage* st, int B, const void* x_in, const void* g_out,
                              const int64_t* labels, void* g_in, void* stream) {
  if (!st || B < 1 || B > st->max_batch || !x_in || (!g_out && !labels)) {
    set_error("ppll_stage_block_backward: invalid arguments (B=%d)", B);
    return PPLL_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int L = st->n_block - 1;
  const int C = st->out_w[L];
  int r;
  char* G = st->g0;
  char* Gn = st->g1;
  if (labels) {
    if (st->dtype == PPLL_F32)
      r = launch_softmax_xent<float>(B, C, (const float*)st->act_ptr(L), C, labels, (float*)G, C,
                                     st->loss_hist, st->step, st->err, s);
    else
      r = launch_softmax_xent<__nv_bfloat16>(B, C, (const __nv_bfloat16*)st->act_ptr(L), C, labels,
                                             (__nv_bfloat16*)G, C, st->loss_hist, st->step,
                                             st->err, s);
  } else if (st->relu[L]) {
    r = launch_relu_mask((long)B * C, g_out, st->act_ptr(L), G, st->dtype, s);
  } else {
    r = launch_cast((long)B * C, g_out, st->dtype, G, st->dtype, s);
  }
  if (r) return r;
  for (int i = L; i >= 0; --i) {
    const void* in = i == 0 ? x_in : st->act_ptr(i - 1);
    r = linear_wgrad(B, st->in_w[i], st->out_w[i], in, st->in_w[i], G, st->out_w[i],
                     st->grad + st->off[2 * i], st->grad + st->off[2 * i + 1], st->dtype, st->ws,
                     st->ws_elems, s);
    if (r) return r;
    if (i > 0 || g_in) {
      const void* mask = (i > 0 && st->relu[i - 1]) ? st->act_ptr(i - 1) : nullptr;
      void* dst = i > 0 ? (void*)Gn : g_in;
      r = linear_dgrad(B, st->in_w[i], st->out_w[i], G, st->out_w[i], st->w_ptr(i), mask,
                       st->in_w[i], dst, st->in_w[i], st->dtype, st->ws, st->ws_elems, s);
      if (r) return r;
      char* t = G; G = Gn; Gn = t;
    }
  }
  const int64_t nb = st->n_block < st->n_layers ? st->off[2 * st->n_block] : st->n_params;
  return launch_nesterov(nb, st->theta, st->mom, st->grad,
                         reinterpret_cast<__nv_bfloat16*>(st->theta_lp), st->lr_table, st->step,
                         st->max_step, 0.f, st->mu, st->wd, st->err, s);
}

}  // extern "C"
