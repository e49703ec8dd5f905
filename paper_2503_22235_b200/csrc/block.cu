// K2-K5 chain of one processor block as single C-ABI calls (SURVEY.md §8b `wm3_block_fwd`): the host-side
// orchestration of the 7 launches of attention.py:146-184 lives in the library, so a caller binds one function
// per block (and one ctypes call replaces seven on the Python side).
//
//   wm3_block_qkv   LN1 -> QKV GEMM (+bias, rotary) into the band's K/V grid     (attention.py:163-171)
//   wm3_block_rest  NA -> O-proj (+bias, +x) -> LN2 -> W1 (+bias, GELU) -> W2 (+bias, +x)  (:173-184)
//   wm3_block_fwd   both, for a band without halos (single GPU) or with halos filled by the fused epilogue
// The halo exchange of a band with NCCL neighbours goes between the two halves.
//
// With folded weights (w_qkv_f != NULL) the two LayerNorms are not separate launches (wm3_ln_fold_t): the
// residual epilogues (O-proj, W2) also write the fp16 copy of the updated stream into ws->hn and its row
// statistics into ws->stats, and the QKV / W1 GEMMs consume them with gain-scaled weights.  A block is then
// 5 GEMM / attention launches plus two tiny row-statistics launches (wm3_ln_fold_finalize); the first block of
// a chain (geom x_prepped = 0) starts with wm3_ln_fold_prep.
#include <cmath>

#include "launch.h"
#include "../../include/wm3.h"

using namespace wm3;

static int ln_parts(const wm3_block_weights_t* w) {
  const int bn = (w->np >= 256) ? 256 : 128;  // column tile of the residual GEMMs (gemm.cu linear_impl)
  return 2 * ((w->np + bn - 1) / bn);
}

static int check_block(const float* x, const wm3_block_weights_t* w, const wm3_block_ws_t* ws,
                       const wm3_block_geom_t* g) {
  if (x == nullptr || w == nullptr || ws == nullptr || g == nullptr) return set_error("wm3_block: null argument");
  if (w->hidden <= 0 || w->heads <= 0 || w->dh <= 0 || (w->dhp != 64 && w->dhp != 128) || w->kp < w->hidden ||
      w->np < w->hidden || w->nm <= 0)
    return set_error("wm3_block: bad weight geometry (hidden %d heads %d dh %d dhp %d)", w->hidden, w->heads, w->dh,
                     w->dhp);
  if (g->batch < 1 || g->depth < 1 || g->rows < 1 || g->cols < 1 || g->rows_global < g->rows)
    return set_error("wm3_block: bad geometry");
  if (w->w_qkv_f != nullptr && (ws->stats == nullptr || ws->row_stats == nullptr || w->c_qkv == nullptr || w->d_qkv == nullptr ||
                                w->w_1_f == nullptr || w->c_1 == nullptr || w->d_1 == nullptr || ln_parts(w) > WM3_LN_SLOTS))
    return set_error("wm3_block: folded LayerNorm needs w_1_f, c_*, d_* and ws stats (hidden <= %d)",
                     WM3_LN_SLOTS / 2 * 256);
  return 0;
}

static wm3_ln_fold_t fold_consumer(const wm3_block_ws_t* ws, const float* c) {
  wm3_ln_fold_t f{};
  f.row_stats = ws->row_stats;
  f.fold_c = c;
  return f;
}

static wm3_ln_fold_t fold_producer(const wm3_block_weights_t* w, const wm3_block_ws_t* ws) {
  wm3_ln_fold_t f{};
  f.xh_out = ws->hn;
  f.ld_xh = w->kp;
  f.stats_out = ws->stats;
  return f;
}

extern "C" int wm3_block_qkv(const float* x, const wm3_block_weights_t* w, const wm3_block_ws_t* ws,
                             const wm3_block_geom_t* g, const wm3_rope_t* rope, const wm3_halo_t* halo,
                             void* stream) {
  if (check_block(x, w, ws, g)) return -1;
  const int t = g->batch * g->depth * g->rows * g->cols;
  const int rows_ext = g->halo_lo + g->rows + g->halo_hi;
  const int qkv_n = 3 * w->heads * w->dhp;
  const int plane = g->rows * g->cols;
  if (w->w_qkv_f != nullptr) {
    if (!g->x_prepped && wm3_ln_fold_prep(x, w->hidden, t, w->hidden, ws->hn, w->kp, 1e-6f, ws->row_stats, stream))
      return -1;
    const wm3_ln_fold_t f = fold_consumer(ws, w->c_qkv);
    return wm3_linear_fold(ws->hn, w->kp, w->w_qkv_f, w->kp, t, qkv_n, w->kp, WM3_EPI_QKV_ROPE, ws->qkv, qkv_n, qkv_n,
                           w->d_qkv, rope, g->batch * g->depth, plane, static_cast<long long>(rows_ext) * g->cols,
                           g->halo_lo * g->cols, halo, &f, stream);
  }
  if (wm3_layernorm_bf16(x, w->hidden, t, w->hidden, w->ln1_g, w->ln1_b, 1e-6f, ws->hn, w->kp, stream)) return -1;
  if (halo != nullptr)
    return wm3_linear_planes_halo(ws->hn, w->kp, w->w_qkv, w->kp, t, qkv_n, w->kp, WM3_EPI_QKV_ROPE, ws->qkv, qkv_n,
                                  qkv_n, w->b_qkv, rope, g->batch * g->depth, plane,
                                  static_cast<long long>(rows_ext) * g->cols, g->halo_lo * g->cols, halo, stream);
  return wm3_linear_planes(ws->hn, w->kp, w->w_qkv, w->kp, t, qkv_n, w->kp, WM3_EPI_QKV_ROPE, ws->qkv, qkv_n, qkv_n,
                           w->b_qkv, rope, g->batch * g->depth, plane, static_cast<long long>(rows_ext) * g->cols,
                           g->halo_lo * g->cols, stream);
}

extern "C" int wm3_block_na_rows(const wm3_block_weights_t* w, const wm3_block_ws_t* ws, const wm3_block_geom_t* g,
                                 int q_lo, int q_rows, void* stream) {
  if (w == nullptr || ws == nullptr || g == nullptr) return set_error("wm3_block_na_rows: null argument");
  const int hd = w->heads * w->dhp;
  return wm3_natten_fwd_rows(ws->qkv, 3 * hd, ws->ctx, hd, g->batch, g->depth, g->rows, g->cols, g->rows_global,
                             g->row0, g->halo_lo, g->halo_hi, w->heads, w->dhp, g->wd, g->wh, g->ww,
                             1.0f / std::sqrt(static_cast<float>(w->dh)), q_lo, q_rows, stream);
}

extern "C" int wm3_block_rest(float* x, const wm3_block_weights_t* w, const wm3_block_ws_t* ws,
                              const wm3_block_geom_t* g, void* stream) {
  if (check_block(x, w, ws, g)) return -1;
  if (wm3_block_na_rows(w, ws, g, g->row0, g->rows, stream)) return -1;
  return wm3_block_out(x, w, ws, g, stream);
}

extern "C" int wm3_block_out(float* x, const wm3_block_weights_t* w, const wm3_block_ws_t* ws,
                             const wm3_block_geom_t* g, void* stream) {
  if (check_block(x, w, ws, g)) return -1;
  const int t = g->batch * g->depth * g->rows * g->cols;
  const int hd = w->heads * w->dhp;
  if (w->w_qkv_f != nullptr) {
    const wm3_ln_fold_t prod = fold_producer(w, ws), cons = fold_consumer(ws, w->c_1);
    if (wm3_linear_fold(ws->ctx, hd, w->w_o, hd, t, w->np, hd, WM3_EPI_BIAS_RESID_F32, x, w->hidden, w->hidden,
                        w->b_o, nullptr, 1, t, t, 0, nullptr, &prod, stream))
      return -1;
    if (wm3_ln_fold_finalize(ws->stats, ln_parts(w), w->hidden, 1e-6f, t, ws->row_stats, stream)) return -1;
    if (wm3_linear_fold(ws->hn, w->kp, w->w_1_f, w->kp, t, w->nm, w->kp, WM3_EPI_BIAS_GELU_BF16, ws->mid, w->nm,
                        w->nm, w->d_1, nullptr, 1, t, t, 0, nullptr, &cons, stream))
      return -1;
    // W2 leaves xh / row statistics of the block's output for the next block's QKV GEMM
    if (wm3_linear_fold(ws->mid, w->nm, w->w_2, w->nm, t, w->np, w->nm, WM3_EPI_BIAS_RESID_F32, x, w->hidden,
                        w->hidden, w->b_2, nullptr, 1, t, t, 0, nullptr, &prod, stream))
      return -1;
    return wm3_ln_fold_finalize(ws->stats, ln_parts(w), w->hidden, 1e-6f, t, ws->row_stats, stream);
  }
  if (wm3_linear(ws->ctx, hd, w->w_o, hd, t, w->np, hd, WM3_EPI_BIAS_RESID_F32, x, w->hidden, w->hidden, w->b_o,
                 nullptr, stream))
    return -1;
  if (wm3_layernorm_bf16(x, w->hidden, t, w->hidden, w->ln2_g, w->ln2_b, 1e-6f, ws->hn, w->kp, stream)) return -1;
  if (wm3_linear(ws->hn, w->kp, w->w_1, w->kp, t, w->nm, w->kp, WM3_EPI_BIAS_GELU_BF16, ws->mid, w->nm, w->nm, w->b_1,
                 nullptr, stream))
    return -1;
  return wm3_linear(ws->mid, w->nm, w->w_2, w->nm, t, w->np, w->nm, WM3_EPI_BIAS_RESID_F32, x, w->hidden, w->hidden,
                    w->b_2, nullptr, stream);
}

extern "C" int wm3_block_fwd(float* x, const wm3_block_weights_t* w, const wm3_block_ws_t* ws,
                             const wm3_block_geom_t* g, const wm3_rope_t* rope, void* stream) {
  if (wm3_block_qkv(x, w, ws, g, rope, nullptr, stream)) return -1;
  return wm3_block_rest(x, w, ws, g, stream);
}
