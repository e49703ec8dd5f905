/*
 * wm3.h — C ABI of the B200-native WeatherMesh-3 forecast hot path (libwm3.so).
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t passed as void*.
 * Nothing here throws: each call returns 0 on success or a nonzero status, with a message
 * available from wm3_last_error() (thread-local).  Validation that the reference performs
 * in Python (ConfigError, gridcast/errors.py:4-5) stays in the Python host layer and runs
 * before any of these are called; a nonzero status here is a launch/device fault
 * ("compute" category in the reference CLI, gridcast/cli.py:456-463).
 *
 * Operand type.  Every `void*` tensor-core operand below (GEMM A / B, LayerNorm outputs, the q/k/v grid, ctx,
 * MLP activations, conv activations and weights) is a 16-bit float of ONE type for the whole library, chosen at
 * build time: IEEE fp16 in the default build (measured 8-10x lower forecast error than bf16),
 * bf16 when built with -DWM3_OPERAND_BF16.  wm3_operand_dtype() reports it; bind it before feeding data.
 * Names carrying "bf16" (wm3_layernorm_bf16, WM3_EPI_BIAS_BF16, WM3_EPI_BIAS_GELU_BF16) are historical and
 * mean "the 16-bit operand type".  Accumulation is fp32 (TMEM); the residual stream / latent is fp32.
 *
 * Reference interfaces replaced (paths relative to the reference package pkg/src/gridcast):
 *   wm3_neighbor_table      grid.py:96-130       bump_starts + neighborhood (bit-exact int64 export)
 *   wm3_layernorm_bf16      autodiff.py:400-424  layernorm, eps 1e-6, biased variance (16-bit operand out)
 *   wm3_linear              attention.py:142-143 _linear = matmul(x, W) + b, with fused epilogues:
 *                             WM3_EPI_BIAS_BF16       (plain linear, 16-bit operand out)
 *                             WM3_EPI_BIAS_GELU_BF16  attention.py:182  gelu(hn2 W1 + b1), erf form to 2.5e-5
 *                             WM3_EPI_BIAS_RESID_F32  attention.py:179,183  x += ctx Wo + bo / mid W2 + b2
 *                             WM3_EPI_QKV_ROPE        attention.py:167-171  q,k,v + bias, rotary on q,k
 *                             WM3_EPI_F32             raw fp32 accumulator (tests)
 *                             WM3_EPI_GELU_GRAD_F32   autodiff.py:372-382  out = acc / scale * gelu'(out + bias),
 *                                                     in place over the stored pre-activation (wm3_linear_gelu_grad)
 *   wm3_natten_fwd          attention.py:173-178 gather + q k^T/sqrt(dh) + softmax + @V, fused
 *   wm3_block_fwd           attention.py:146-184 the whole block (7 launches) in one call
 *   wm3_conv  WM3_CONV_S1/S2  model.py:296-301 + autodiff.py:677-713  3x3, row zero pad, col wrap, stride 1/2
 *   wm3_conv  WM3_CONV_T2     model.py:317-325 + autodiff.py:716-764  4x4 stride-2 transposed (exact adjoint)
 *   wm3_fields_to_nhwc / wm3_tokens_to_nhwc   model.py:332-337, 350-360  relayouts feeding the pyramids
 *   wm3_sq_err_rows / wm3_zonal_power          evaluation.py:37-75         verification metrics
 */
#ifndef WM3_H
#define WM3_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  WM3_EPI_F32 = 0,
  WM3_EPI_BIAS_BF16 = 1,
  WM3_EPI_BIAS_GELU_BF16 = 2,
  WM3_EPI_BIAS_RESID_F32 = 3,
  WM3_EPI_QKV_ROPE = 4,
  WM3_EPI_GELU_GRAD_F32 = 5,
};

/* Rotary description for WM3_EPI_QKV_ROPE (attention.py:48-92).  Output columns are laid out
 * [3][heads][dhp]; within a q/k head, rotation pair j (reference columns j, j + dh/2) sits at the
 * adjacent columns (2j, 2j + 1), j < dh/2 (a permutation shared by q and k leaves q.k unchanged).
 * The phases factor by axis: pairs j < split (depth, then row pairs) depend on the token's (depth plane,
 * global row) only, pairs j >= split (column pairs) on its column only.
 *   dr:  [depth * rows][128] fp32, row d * rows + h = cos[64] then sin[64] of band row h of plane d
 *        (32-byte aligned; entries of column pairs and of pairs >= dh/2 are (1, 0));
 *   col: [2][64][cols] fp32, pair-major cos then sin of every column (entries of pairs < split are (1, 0)).
 * rows, cols: the band's token extents; period = depth * rows * cols tokens per latent: GEMM row r is token
 * r % period, so a batch of ensemble members shares the tables. */
typedef struct {
  const float* dr;
  const float* col;
  int heads, dhp;
  int rows, cols;
  int period;
  int split;
} wm3_rope_t;

const char* wm3_last_error(void);
int wm3_version(void);
int wm3_sm_count(void);
/* The 16-bit operand type of this build: WM3_DTYPE_F16 (default) or WM3_DTYPE_BF16 (-DWM3_OPERAND_BF16). */
enum { WM3_DTYPE_F16 = 1, WM3_DTYPE_BF16 = 2 };
int wm3_operand_dtype(void);

/* (T, K) int64 neighbor table of a (depth,rows,cols) box; rows [row0, row0+nrows) of a grid with
 * global extent `rows`.  Row-major K order kd*wh*ww + kh*ww + kw (grid.py:124-127). */
int wm3_neighbor_table(int depth, int rows, int cols, int wd, int wh, int ww, int row0, int nrows,
                       int64_t* out, void* stream);

/* out[m, 0:ldo] = operand(layernorm(x[m, 0:n]) * gain + bias), zero in [n, ldo) (operand = wm3_operand_dtype). */
int wm3_layernorm_bf16(const float* x, int ldx, int m, int n, const float* gain, const float* bias,
                       float eps, void* out_bf16, int ldo, void* stream);

/* C[M, N] = A[M, K] (16-bit operand, row pitch lda) * B[N, K]^T (16-bit operand, row pitch ldb) + epilogue.
 * out: 16-bit operand or f32 depending on epi; ldo in elements; n_valid columns are stored. */
int wm3_linear(const void* a, int lda, const void* b, int ldb, int m, int n, int k, int epi,
               void* out, int ldo, int n_valid, const float* bias, const wm3_rope_t* rope, void* stream);

/* As wm3_linear, with the m GEMM rows split into `planes` planes of plane_rows rows each; plane p row r
 * is stored at row row_off + p * plane_stride + r of `out` (M-tiles never straddle planes).  This writes a
 * latitude band's q/k/v into the K/V grid of wm3_natten_fwd, leaving halo rows between depth planes. */
int wm3_linear_planes(const void* a, int lda, const void* b, int ldb, int m, int n, int k, int epi,
                      void* out, int ldo, int n_valid, const float* bias, const wm3_rope_t* rope,
                      int planes, int plane_rows, long long plane_stride, int row_off, void* stream);

/* Fused halo exchange for latitude bands (the QKV GEMM epilogue stores a band's boundary K/V rows straight
 * into the neighbouring ranks' K/V grids over NVLink peer memory; no separate collective).
 * For GEMM plane p and plane-row r (band row * cols + col) with column block n >= col_lo:
 *   r <  n_up           -> up[(p * up_plane_stride + up_row_off + r) * ld + n]
 *   r >= plane_rows - n_dn -> dn[(p * dn_plane_stride + dn_row_off + r - (plane_rows - n_dn)) * ld + n]
 * up / dn may be null (no neighbour).  Pointers are peer-mapped device addresses (CUDA IPC); the stores are
 * followed by a system-scope fence in the kernel, and wm3_halo_signal / wm3_halo_wait order them against the
 * neighbours' attention kernels (monotonic epoch flags, one int32 per direction and purpose). */
typedef struct {
  void* up;
  void* dn;
  int n_up, n_dn;                  /* plane-rows sent to each neighbour */
  long long up_plane_stride, dn_plane_stride;
  long long up_row_off, dn_row_off;
  int ld;                          /* destination row pitch (elements) */
  int col_lo;                      /* first column sent (K and V sections only) */
} wm3_halo_t;

int wm3_linear_planes_halo(const void* a, int lda, const void* b, int ldb, int m, int n, int k, int epi, void* out,
                           int ldo, int n_valid, const float* bias, const wm3_rope_t* rope, int planes,
                           int plane_rows, long long plane_stride, int row_off, const wm3_halo_t* halo,
                           void* stream);
/* Release-store `epoch` to each non-null peer flag (system scope), after a system fence. */
int wm3_halo_signal(int* peer_flag_a, int* peer_flag_b, int epoch, void* stream);
/* Spin (acquire, system scope) until each of the n local flags is >= epoch; traps after ~10 s. */
int wm3_halo_wait(const int* flags, int n, int epoch, void* stream);

/* LayerNorm folded into the GEMMs around it (attention.py:163-165, 180-181).  A residual GEMM
 * (WM3_EPI_BIAS_RESID_F32) acting as producer also writes an fp16 copy of the updated stream (xh_out, columns
 * < n_valid; pad columns untouched) and per row partial (sum, sum of squares) pairs into
 * stats_out[row][slot][2] (slot = 2 * column tile + epilogue group, every slot < 2 * ceil(n / tile) written);
 * wm3_ln_fold_finalize turns them into row_stats[row] = (rstd, rstd * mean) (biased variance, eps).  The next
 * GEMM, as consumer, takes A = xh with weights pre-scaled by the LN gain and applies
 * rstd * acc - rstd * mean * fold_c[col] + bias[col] before its own epilogue (bias = b + beta . W). */
#define WM3_LN_SLOTS 16
typedef struct {
  void* xh_out;
  int ld_xh;
  float* stats_out;
  const float* row_stats;
  const float* fold_c;
} wm3_ln_fold_t;
/* wm3_linear_planes_halo with an optional LayerNorm fold (producer and / or consumer side); halo may be NULL. */
int wm3_linear_fold(const void* a, int lda, const void* b, int ldb, int m, int n, int k, int epi, void* out, int ldo,
                    int n_valid, const float* bias, const wm3_rope_t* rope, int planes, int plane_rows,
                    long long plane_stride, int row_off, const wm3_halo_t* halo, const wm3_ln_fold_t* fold,
                    void* stream);
/* Producer partials (the first `parts` pairs of each row) -> row_stats[m][2] = (rstd, rstd * mean) over n. */
int wm3_ln_fold_finalize(const float* stats, int parts, int n, float eps, int m, float* row_stats, void* stream);
/* Start of a folded chain: xh = fp16(x) (columns >= n of each xh row zeroed) and row_stats of x. */
int wm3_ln_fold_prep(const float* x, int ldx, int m, int n, void* xh, int ld_xh, float eps, float* row_stats,
                     void* stream);

/* One processor block (attention.py:146-184) as library calls: x (T, hidden) fp32 in place, T = batch * depth *
 * rows * cols band tokens.  Weights in the device layout the Python layer prepares (blocks.prepare_block:
 * K-major fp16, q/k rotary pairs interleaved, heads padded to dhp); workspace buffers: hn (T, kp), the K/V grid
 * qkv ([batch * depth][halo_lo + rows + halo_hi][cols][3 * heads * dhp]), ctx (T, heads * dhp), mid (T, nm). */
typedef struct {
  const float *ln1_g, *ln1_b;
  const void* w_qkv;
  const float* b_qkv;
  const void* w_o;
  const float* b_o;
  const float *ln2_g, *ln2_b;
  const void* w_1;
  const float* b_1;
  const void* w_2;
  const float* b_2;
  int hidden, heads, dh, dhp, kp, np, nm;
  /* LayerNorm folded into the QKV and W1 GEMMs (wm3_ln_fold_t); NULL w_qkv_f = separate LayerNorm launches.
   * w_qkv_f / w_1_f: w_qkv / w_1 with every input column k scaled by ln1 / ln2 gain[k] (fp16); c_*: per
   * output column sum over k of those fp16 weights; d_*: bias + sum_k ln bias[k] * W[col][k]. */
  const void* w_qkv_f;
  const float *c_qkv, *d_qkv;
  const void* w_1_f;
  const float *c_1, *d_1;
} wm3_block_weights_t;
typedef struct {
  void *hn, *qkv, *ctx, *mid;
  float* stats;     /* [T][WM3_LN_SLOTS][2] LayerNorm partial sums (folded path); hn then holds fp16(x) */
  float* row_stats; /* [T][2] (rstd, rstd * mean) of x (folded path) */
} wm3_block_ws_t;
typedef struct {
  int batch, depth, rows, cols;    /* local band extents (batch = ensemble members) */
  int rows_global, row0, halo_lo, halo_hi;
  int wd, wh, ww;                  /* attention window */
  int x_prepped;                   /* folded LayerNorm: ws hn / stats already describe x (written by the
                                      previous block's W2 epilogue); 0 = compute them first */
} wm3_block_geom_t;
/* LN1 + QKV (+rotary) into the K/V grid; with halo != NULL the epilogue also fills the neighbours' halos. */
int wm3_block_qkv(const float* x, const wm3_block_weights_t* w, const wm3_block_ws_t* ws, const wm3_block_geom_t* g,
                  const wm3_rope_t* rope, const wm3_halo_t* halo, void* stream);
/* NA -> O-proj + residual -> LN2 -> W1 + GELU -> W2 + residual (halo rows of the K/V grid must be filled). */
int wm3_block_rest(float* x, const wm3_block_weights_t* w, const wm3_block_ws_t* ws, const wm3_block_geom_t* g,
                   void* stream);
/* The two halves of wm3_block_rest, for overlapping the halo exchange with attention: NA of the global query
 * rows [q_lo, q_lo + q_rows) of the band into ws->ctx (wm3_natten_fwd_rows; rows whose windows stay inside the
 * band need no halo), then everything after NA once every row's ctx is written. */
int wm3_block_na_rows(const wm3_block_weights_t* w, const wm3_block_ws_t* ws, const wm3_block_geom_t* g, int q_lo,
                      int q_rows, void* stream);
int wm3_block_out(float* x, const wm3_block_weights_t* w, const wm3_block_ws_t* ws, const wm3_block_geom_t* g,
                  void* stream);
/* Both halves (a band without halos, or halos filled by the fused epilogue). */
int wm3_block_fwd(float* x, const wm3_block_weights_t* w, const wm3_block_ws_t* ws, const wm3_block_geom_t* g,
                  const wm3_rope_t* rope, void* stream);

/* Fused 3D neighborhood attention forward, over `batch` independent latents (ensemble members).
 * qkv: 16-bit operand K/V grid [batch * depth][rows_ext][cols][ldqkv] (member b owns depth planes [b * depth, (b + 1) * depth);
 *      windows never cross members), token channels [3][heads][dhp]; rows_ext =
 *      halo_lo + rows + halo_hi: the local band rows [row0, row0 + rows) of a grid with global row extent
 *      rows_global, plus halo rows received from the neighbouring bands.  Longitude wrap is handled inside
 *      the kernel (a wrapping key patch is fetched as two TMA boxes).
 * out: 16-bit operand [batch * depth * rows * cols][ldo] (member-major, local token order), channels [heads][dhp].
 * scale = 1/sqrt(dh).  The window mask is applied inside the QK^T MMA from key-bias images that the library
 * builds once per device and geometry (on `stream`, at first use) and caches for the process. */
int wm3_natten_fwd(const void* qkv, int ldqkv, void* out, int ldo, int batch, int depth, int rows, int cols,
                   int rows_global, int row0, int halo_lo, int halo_hi, int heads, int dhp, int wd,
                   int wh, int ww, float scale, void* stream);
/* wm3_natten_fwd restricted to the queries of global rows [q_lo, q_lo + q_rows) (inside the band); other rows of
 * `out` are untouched.  Query tiles are aligned to global rows and a query's key chunks do not depend on the
 * launch, so any split of the band's rows over several launches writes bitwise the bytes of one launch (and of
 * the single-GPU launch): rows whose windows stay inside the band can run while the halo rows are in flight. */
int wm3_natten_fwd_rows(const void* qkv, int ldqkv, void* out, int ldo, int batch, int depth, int rows, int cols,
                        int rows_global, int row0, int halo_lo, int halo_hi, int heads, int dhp, int wd, int wh,
                        int ww, float scale, int q_lo, int q_rows, void* stream);

/* Implicit-GEMM convolutions of the encoder / decoder pyramids (model.py:296-325, autodiff.py:585-764).
 * Activations are 16-bit operand NHWC with a 1-pixel halo, [imgs][H + 2][W + 2][Cp] (Cp % 64 == 0): zero halo rows,
 * halo columns = opposite edge (longitude wrap).  Modes:
 *   WM3_CONV_S1  3x3 stride 1       w: [cout_pad][9][cinp]      (tap = kh * 3 + kw)
 *   WM3_CONV_S2  3x3 stride 2       w: [cout_pad][9][cinp]
 *   WM3_CONV_T2  4x4 stride 2 transposed (adjoint geometry), as 4 output-parity classes of 2x2 taps:
 *                w: [4 = 2a + b][cout_pad][4 = 2tr + tc][cinp] = W[cin][cout][3 - a - 2tr][3 - b - 2tc]
 * cout_pad = cout rounded up to wm3_conv_bn(cout).  Epilogue: + bias, optional exact GELU, optional
 * residual (16-bit NHWC, same layout as the output), then one of
 *   WM3_CONV_OUT_NHWC    16-bit padded NHWC (pitch out_cp), wrap columns written too
 *   WM3_CONV_OUT_TOKENS  fp32 tokens [img][H][W][cout] (the latent, model.py:350-354)
 *   WM3_CONV_OUT_FIELD   fp32 NCHW: out[img * img_stride + (c / chan_div) * a_stride + (c % chan_div) * p_stride
 *                        + h * W + w] (surface / atmos fields with the level unfold of model.py:340-347). */
enum { WM3_CONV_S1 = 0, WM3_CONV_S2 = 1, WM3_CONV_T2 = 2 };
enum { WM3_CONV_OUT_NHWC = 0, WM3_CONV_OUT_TOKENS = 1, WM3_CONV_OUT_FIELD = 2 };
int wm3_conv_bn(int cout);
int wm3_conv(int mode, const void* in, int imgs, int hin, int win, int cinp, const void* w, int cout,
             const float* bias, int act_gelu, const void* resid, int resid_cp, int out_kind, void* out, int out_cp,
             long long img_stride, long long a_stride, long long p_stride, int chan_div, void* stream);
/* fp32 fields -> padded NHWC: channel c of image i at src[i * img_stride + (c / chan_div) * a_stride
 * + (c % chan_div) * p_stride + h * W + w] (level fold of model.py:332-337).  If `overflow` is non-null, *overflow
 * is OR-ed with 1 when any input value is outside the operand type's finite range (|x| > 65504 for fp16) or is
 * not finite; the caller zeroes it first and checks it after the launch. */
int wm3_fields_to_nhwc(const float* src, long long img_stride, long long a_stride, long long p_stride, int chan_div,
                       int imgs, int channels, int h, int w, int cp, void* dst, int* overflow, void* stream);
/* fp32 tokens [img][H][W][channels] -> padded NHWC (model.py:357-360). */
int wm3_tokens_to_nhwc(const float* tokens, int imgs, int h, int w, int channels, int cp, void* dst, void* stream);

/* Verification metrics (evaluation.py:37-190), float64 accumulation, deterministic order.
 * Fields are [imgs][rows][cols] of dtype 0 = float32 or 1 = float64; with k > 1 the field is the mean of k
 * ensemble members spaced member_stride elements apart (the leading-k ensemble mean of ensemble_curve).
 *   wm3_sq_err_rows:  partial[t * rows + r] = w_rows[r] * sum_c (a - b)^2 (latitude_rmse, evaluation.py:37-52)
 *   wm3_zonal_power:  out[img][r][m], m <= cols / 2, mean-square zonal power (zonal_power, evaluation.py:59-75) */
int wm3_sq_err_rows(int dtype, const void* a, long long member_stride, int k, const void* b, const double* w_rows,
                    int times, int rows, int cols, double* partial, void* stream);
int wm3_zonal_power(int dtype, const void* field, long long member_stride, int k, int imgs, int rows, int cols,
                    double* out, void* stream);

/* Reverse mode of one processor block (autodiff.py backward rules; orchestrated by
 * paper_2503_22235_b200/backward.py, which runs the weight / input gradient GEMMs on wm3_linear).  Deterministic
 * (fixed summation orders), so recomputed segments reproduce their gradients bitwise.  Gradient tensors are fp32;
 * before a GEMM they are cast to the 16-bit operand with a power-of-two scale 2^(14 - ceil(log2 max|g|)) held on
 * the device (amax_bits = the float bits of max|g|, written by wm3_bw_amax), and every consumer of a GEMM result
 * divides it back out (NULL amax_bits = scale 1).
 *   wm3_bw_amax       *amax_bits = bits of max |x| over rows x cols (pitch ld)
 *   wm3_bw_cast       dst = operand(src * scale), row-major [rows][ldd] or transposed [cols][ldd] (zero padded);
 *                     src fp32 (src_f32 = 1) or 16-bit operand
 *   wm3_bw_colsum     out[c] = sum_r src[r][c] (* src2[r][c]) / scale, fixed order (partial: ceil(rows/256) * cols)
 *   wm3_bw_gelu       out = g / scale * gelu'(a + bias) (exact-erf GELU, autodiff.py:372-382)
 *   wm3_bw_gelu_fwd   out = operand(GELU(a + bias)) exactly as the W1 GEMM epilogue computes it (the forward's
 *                     activation, bitwise, from the stored fp32 pre-activation; cols, lda, ldo multiples of 8)
 *   wm3_bw_colsum_amax  one pass: colsum[c] = sum_r v[r][c] (wm3_bw_colsum's order) and *amax_bits = bits of
 *                     max |v|, v = g; with a != NULL, v = g / scale(in_scale_bits) * gelu'(a + bias) is also
 *                     stored to out (the GELU backward, its bias gradient and the next operand scale at once)
 *   wm3_bw_layernorm  gx = LayerNorm-backward(x, gamma, g / scale) (+ add); gxh = g / scale * xhat; gsc = g / scale
 *                     (autodiff.py:400-424: mean, biased variance, eps); gsc may be NULL; gx_amax (or NULL): atomicMax
 *                     of max |gx| (the producer leaves the next cast's scale: no separate amax pass)
 *   wm3_bw_cast_colsum  one pass: dst = operand(src * scale(amax_bits)) [rows][ldd] (columns >= cols zero) and
 *                     colsum[c] = sum_r src[r][c] (fixed order; partial: ceil(rows / 256) * cols floats)
 *   wm3_bw_natten     attention backward over the neighbor table nbr [T][K] (grid.py K order) of the 16-bit qkv
 *                     [T][3][heads][dhp] (rotated q, k): the q gradient per query, the k / v gradients per key from
 *                     the inverse neighbor list (inv_off [T + 1], inv_ent [(t, k)] sorted by t); P, dS
 *                     [T][heads][K] and work [T][heads][2K] scratch; gout [T][3][heads][dhp] fp32
 *   wm3_bw_rope_q     wm3_bw_rope on the q section only (the tensor-core attention backward rotates dK itself);
 *                     amax (or NULL): atomicMax of the rotated values' max |.|
 *   wm3_bw_rope       in place on the q / k sections of gout: the transpose of the rotary rotation (cos / sin
 *                     [T][dhp / 2] of the interleaved pairs) */
int wm3_bw_amax(const float* x, int rows, int cols, int ld, unsigned* amax_bits, void* stream);
int wm3_bw_cast(const void* src, int src_f32, int rows, int cols, int lds, void* dst, int ldd, int transpose,
                const unsigned* amax_bits, void* stream);
int wm3_bw_colsum(const float* src, const float* src2, int rows, int cols, int ld, const unsigned* amax_bits,
                  float* partial, float* out, void* stream);
int wm3_bw_gelu(const float* g, int ldg, const float* a, int lda, const float* bias, int rows, int cols,
                const unsigned* amax_bits, float* out, int ldo, void* stream);
int wm3_bw_gelu_fwd(const float* a, int lda, const float* bias, int rows, int cols, void* out, int ldo, void* stream);
int wm3_bw_colsum_amax(const float* g, int ldg, const float* a, int lda, const float* bias,
                       const unsigned* in_scale_bits, int rows, int cols, float* out, int ldo, float* partial,
                       float* colsum, unsigned* amax_bits, void* stream);
int wm3_bw_layernorm(const float* x, int ldx, int rows, int n, float eps, const float* gamma, const float* g, int ldg,
                     const unsigned* amax_bits, const float* add, float* gx, float* gxh, float* gsc, unsigned* gx_amax,
                     void* stream);
int wm3_bw_natten(const void* qkv, int ldq, const int64_t* nbr, const int* inv_off, const int* inv_ent, int T, int K,
                  int heads, int dhp, float scale, const float* gctx, int ldc, const unsigned* amax_bits, float* P,
                  float* dS, float* work, float* gout, int ldg, void* stream);
int wm3_bw_rope_q(float* g, int ldg, int T, int heads, int dhp, const float* cos_t, const float* sin_t, unsigned* amax,
                  void* stream);
int wm3_bw_cast_colsum(const float* src, int rows, int cols, int lds, void* dst, int ldd, const unsigned* amax_bits,
                       float* partial, float* colsum, void* stream);
int wm3_bw_rope(float* g, int ldg, int T, int heads, int dhp, const float* cos_t, const float* sin_t, void* stream);

/* The MLP's GELU backward fused into the gradient GEMM (autodiff.py:372-382 after the W2 matmul VJP :350):
 * preact_inout [m][n] fp32 holds the W1 pre-activation without bias on entry and
 * (A . B^T) / scale(amax_bits) * gelu'(preact + bias) on exit (the residual epilogue's in-place read-then-write);
 * out_amax_bits (or NULL): atomicMax of the result's max |.| (zeroed by the caller). */
int wm3_linear_gelu_grad(const void* a, int lda, const void* b, int ldb, int m, int n, int k, float* preact_inout,
                         int ldo, const float* bias, const unsigned* amax_bits, unsigned* out_amax_bits, void* stream);

/* C[m][n] (fp32) = sum_t A[t][m] B[t][n] with A [k][m], B [k][n] row-major 16-bit (the backward's weight gradients
 * over the token axis, autodiff.py:350 matmul VJP): MN-major tcgen05 operands, no transposed copies; m, n multiples
 * of 64. */
int wm3_linear_tn(const void* a, int lda, const void* b, int ldb, int m, int n, int k, float* out, int ldo,
                  void* stream);
/* wm3_linear_tn with the K range split over CTA pairs when the output has too few 256 x 256 tiles to fill the GPU
 * (the split count minimises tile waves per split, <= 16, >= 8 k-blocks per split, sp * m * n <= scratch_floats):
 * per-split fp32 partials in scratch, then summed in split order (deterministic).  NULL scratch = no split. */
int wm3_linear_tn_split(const void* a, int lda, const void* b, int ldb, int m, int n, int k, float* out, int ldo,
                        float* scratch, size_t scratch_floats, void* stream);
/* the split count wm3_linear_tn_split picks for m x n x k with unlimited scratch (size the scratch as count * m * n
 * floats; 1 = no split, no scratch needed) */
int wm3_linear_tn_split_count(int m, int n, int k);

/* Attention backward on the tensor cores (replaces wm3_bw_natten when wm3_natten_bwd_info reports support: head
 * dim padded to 128, window mask in the MMA).  Same reference rules (attention.py:173-178 through autodiff.py's
 * matmul / softmax / take VJPs); full domain, one member.
 *   wm3_natten_fwd_lse     the forward (wm3_natten_fwd) also writing lse [T][heads] (log2-domain log-sum-exp)
 *   wm3_bw_na_prep         dO (fp16, [T][heads * dhp]) = gctx * sigma with sigma a power of two keeping
 *                          |dO . v| <= 2^13; factors[2] = (scale / (sigma s), 1 / (sigma s)), s = gctx's grad
 *                          scale (amax bits); maxima[2] scratch
 *   wm3_natten_bwd_info    tiles and per-tile chunk slots of the geometry; supported = 1 if the tcgen05 path applies
 *   wm3_natten_slot_table  int32 [tiles][maxch][128]: key token of every chunk slot (-1: none), for the CSR
 *                          (csr_off [T + 1], csr_ent = (tile * maxch + chunk) * 128 + slot, by token, fixed order)
 *   wm3_natten_bwd         dQ into gqkv's q section, dK / dV (the CSR-ordered sum of per-chunk partials, partial =
 *                          [tiles * heads][maxch][2][2][64][128] fp32 scratch) into its k / v sections (fp32);
 *                          with rope_cos / rope_sin ([T][dhp / 2] pair tables, or both NULL) dK leaves through the
 *                          transpose of the rotary rotation (dQ then takes wm3_bw_rope_q); kv_amax (or NULL):
 *                          atomicMax of max |dK|, |dV| */
int wm3_natten_fwd_lse(const void* qkv, int ldqkv, void* out, int ldo, int depth, int rows, int cols, int heads, int dhp,
                       int wd, int wh, int ww, float scale, float* lse, void* stream);
int wm3_bw_na_prep(const void* qkv, int ldq, int T, int heads, int dhp, const float* gctx, int ldc,
                   const unsigned* gscale_bits, float scale, void* dout, int ldd, unsigned* maxima, float* factors,
                   void* stream);
int wm3_natten_bwd_info(int depth, int rows, int cols, int heads, int dhp, int wd, int wh, int ww, int* ntiles,
                        int* maxch, int* supported, void* stream);
int wm3_natten_slot_table(int depth, int rows, int cols, int heads, int dhp, int wd, int wh, int ww, int32_t* table,
                          void* stream);
int wm3_natten_bwd(const void* qkv, int ldqkv, const void* dout, int ldd, const void* o, int ldo, const float* lse,
                   float* gqkv, int ldg, float* partial, const int32_t* csr_off, const int32_t* csr_ent,
                   const float* factors, const float* rope_cos, const float* rope_sin, unsigned* kv_amax, int depth,
                   int rows, int cols, int heads, int dhp, int wd, int wh, int ww, float scale, void* stream);

/* Debug export of the kernel's own window arithmetic: per token, the (start_d, start_h, col_off)
 * it uses; int32 [T][3]. */
int wm3_natten_windows(int depth, int rows, int cols, int rows_global, int row0, int wd, int wh, int ww,
                       int32_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* WM3_H */
