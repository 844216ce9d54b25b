/* pscwin.h — C ABI of libpscwin.so, the B200 (sm_100a) PSCWin layer of HRSAM (arXiv 2407.02109).
 *
 * Citations: P:Lx = PAPER.md line x (section / equation alongside); Qn = reading n in DESIGN.md "Readings".
 *
 * Conventions for every call below
 *   - Tensor pointers are DEVICE pointers unless the argument says "host". They are row-major, contiguous,
 *     16-byte aligned (TMA requirement; violations return PSCWIN_ERR_ALIGN) and owned by the caller.
 *     The library never allocates device memory inside these calls; scratch comes from a caller-provided
 *     workspace sized by the matching *_workspace_bytes() function.
 *   - `stream` is a cudaStream_t passed as void*. Calls enqueue work on it and return immediately;
 *     argument/contract validation is synchronous. A launch failure returns PSCWIN_ERR_CUDA; a fault inside a
 *     kernel surfaces later through pscwin_last_async_error() or the next call.
 *   - No exceptions or C++ types cross the boundary. Calls are reentrant and may run concurrently on different
 *     host threads and streams: the library's only state is a cached SM count, per-(device, kernel)
 *     shared-memory attributes set once under a lock, and helper streams / fork-join events that are private to
 *     each host thread and device (thread_local; e.g. the side stream of the pad work). The A/B tuning knobs
 *     (PSCWIN_* environment variables) are read once per process.
 *   - dtype PSCWIN_BF16 (the product path): activations and GEMM weights are bf16; LayerNorm parameters, biases,
 *     conv, dt_proj, A_log, D_skip are f32; accumulation and the scan state are f32. PSCWIN_F32 (everything f32,
 *     the 1e-4 correctness path of DESIGN.md §6b) is accepted by the partition / merge / layer-norm calls, the
 *     attention, cycle-scan and whole-layer calls; the multi-scale, band and encoder-end calls require BF16
 *     (PSCWIN_ERR_UNSUPPORTED otherwise).
 *   - Head width d = C / heads must be 32 or 64 (tcgen05 tiles of the attention kernels); d = 128 is a contract
 *     limit of this library (PSCWIN_ERR_UNSUPPORTED): ViT-B / HRSAM use d = 64.
 */
#ifndef PSCWIN_H_
#define PSCWIN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PSCWIN_OK = 0,
  PSCWIN_ERR_SHAPE = 1,       /* non-positive or inconsistent sizes */
  PSCWIN_ERR_CONTRACT = 2,    /* violates the layer's definition (see each call) */
  PSCWIN_ERR_ALIGN = 3,       /* pointer not 16-byte aligned */
  PSCWIN_ERR_WORKSPACE = 4,   /* workspace missing or too small */
  PSCWIN_ERR_CUDA = 5,        /* CUDA launch / driver error */
  PSCWIN_ERR_UNSUPPORTED = 6, /* valid per the paper but not implemented on this path (e.g. d_head 128) */
  PSCWIN_ERR_NCCL = 7,        /* an NCCL call failed, an asynchronous communicator error is pending, or the
                                 communicator was aborted (pscwin_nccl_comm_check / _abort) */
  PSCWIN_ERR_TIMEOUT = 8      /* pscwin_nccl_wait: the stream did not drain within the deadline (comm aborted) */
} pscwin_status;

typedef enum { PSCWIN_BF16 = 0, PSCWIN_F32 = 1 } pscwin_dtype;
/* Q5: LEARNABLE = the paper's Pad Swin (pad slots hold the projected learnable token p);
 *     MASKED = pad keys get -inf logits (= vanilla shifted windows of different sizes). */
typedef enum { PSCWIN_PAD_LEARNABLE = 0, PSCWIN_PAD_MASKED = 1 } pscwin_pad_mode;
/* Q13: order in which the cycle scan walks the token grid (row-major raster by default). */
typedef enum { PSCWIN_SCAN_ROW_MAJOR = 0, PSCWIN_SCAN_COL_MAJOR = 1, PSCWIN_SCAN_WINDOW_MAJOR = 2 } pscwin_scan_order;
/* Q11: B_bar rule. ZOH = Eq. 3 B_bar = (e^{Delta A} - 1)/A * B;  EULER = Delta * B. */
typedef enum { PSCWIN_BBAR_ZOH = 0, PSCWIN_BBAR_EULER = 1 } pscwin_bbar_mode;

/* One PSCWin layer. Token grid H x W = image / 16. */
typedef struct {
  int32_t B, H, W, C, heads;          /* d_head = C / heads; d_head in {32, 64} on this path          */
  int32_t window;                     /* w; power of two in [4, 128] (w = H = W: global attention) */
  int32_t shift_x, shift_y;           /* in [0, w); (0,0) = plain window attention (Q7)          */
  int32_t pad_mode;                   /* pscwin_pad_mode                                                */
  int32_t rope;                       /* 0 off, 1 axial 2-D RoPE base 10000 on q,k (Q6)         */
  int32_t cycle_scan;                 /* 1: run the cycle-scan module before attention     */
  int32_t ssm_state;                  /* N (32); N <= 64                                        */
  int32_t ssm_expand;                 /* E, D = E*C (Mamba default 2, Q9)                              */
  int32_t ssm_dt_rank;                /* R; 0 => ceil(C/16)                                              */
  int32_t ssm_conv;                   /* causal depthwise conv width k (Mamba default 4, Q9)            */
  int32_t scan_order;                 /* pscwin_scan_order of the cycle scan (window-major: H, W % window == 0) */
  int32_t bbar_mode;                  /* pscwin_bbar_mode                                               */
  int32_t dtype;                      /* pscwin_dtype                                                   */
  float ln_eps;                       /* LayerNorm eps (Q15: 1e-6)                                      */
  int32_t mlp_hidden;                 /* FFN sub-layer hidden width (768 x 4; reading Q21); 0 = none.
                                         A multiple of 64. x += GELU(LN2(x) W_fc1^T + b_fc1) W_fc2^T + b_fc2 */
} pscwin_layer_desc;

/* Weights of one layer. Linear weights are nn.Linear-style [out, in], bf16 (dtype BF16).
 * Attention (a4-a7): ln1_g, ln1_b [C] f32; w_qkv [3C, C]; b_qkv [3C] f32 (Q = rows [0,C), K = [C,2C),
 * V = [2C,3C), head-contiguous, Q3); pad [C] = learnable pad token p; w_o [C, C]; b_o [C] f32.
 * Cycle scan (a1-a3, Mamba-1 block, Q9): lns_g, lns_b [C] f32; w_in [2D, C] (x-branch rows [0,D), z rows
 * [D,2D)); conv_w [D, k] f32; conv_b [D] f32; w_x [R+2N, D] (delta_low, B, C); w_dt [D, R] f32; b_dt [D] f32;
 * a_log [D, N] f32 (A = -exp(a_log)); d_skip [D] f32; w_out [C, D].
 * FFN (mlp_hidden = Hd > 0): ln2_g, ln2_b [C] f32; w_fc1 [Hd, C]; b_fc1 [Hd] f32; w_fc2 [C, Hd]; b_fc2 [C] f32.
 * Unused pointers may be NULL. */
typedef struct {
  const void *ln1_g, *ln1_b, *w_qkv, *b_qkv, *pad, *w_o, *b_o;
  const void *lns_g, *lns_b, *w_in, *conv_w, *conv_b, *w_x, *w_dt, *b_dt, *w_out;
  const float *a_log, *d_skip;
  const void *ln2_g, *ln2_b, *w_fc1, *b_fc1, *w_fc2, *b_fc2;
} pscwin_layer_weights;

/* ------------------------------------------------------------------------------------------------ info */
const char* pscwin_version(void);
const char* pscwin_status_string(int status);
/* Returns PSCWIN_ERR_CUDA if an asynchronous kernel fault is pending on the device (cudaGetLastError /
 * cudaPeekAtLastError), else PSCWIN_OK. */
int pscwin_last_async_error(void);

/* ------------------------------------------------------------------------------- a5: window geometry */
/* Number of windows per image. Plain (sx = sy = 0): H, W must be divisible by w else
 * ERR_CONTRACT. Shifted: pad left/top = (w - s) mod w (Q7), right/bottom minimal. */
int pscwin_window_count(int32_t H, int32_t W, int32_t window, int32_t shift_x, int32_t shift_y,
                        int32_t* n_windows /* host, out */);
/* Host-side index map (App. C): for destination slot s = win*w*w + iy*w + ix (windows
 * row-major over (wy,wx), Q4) the source token y*W + x, or 0xFFFFFFFF (PAD) outside the grid.
 * host_map must hold n_windows*w*w entries. Pure host computation; no GPU needed. */
int pscwin_index_map(int32_t H, int32_t W, int32_t window, int32_t shift_x, int32_t shift_y, uint32_t* host_map);

/* Plain window partition F -> F_w: x [B,H,W,Cx] -> out [B*nW, w*w, Cx]. Bit-exact copy. */
int pscwin_window_partition(const void* x, int32_t B, int32_t H, int32_t W, int32_t Cx, int32_t window,
                            int32_t dtype, void* out, void* stream);
/* Padding-shifted partition: out [B*nWp, w*w, Cx]; pad slots receive pad_row [Cx]
 * (required: ERR_CONTRACT if NULL and the layout has pad slots). Bit-exact copy. */
int pscwin_shifted_pad_partition(const void* x, const void* pad_row, int32_t B, int32_t H, int32_t W, int32_t Cx,
                                 int32_t window, int32_t shift_x, int32_t shift_y, int32_t dtype, void* out,
                                 void* stream);
/* Merge / crop / un-shift ("paddings are discarded"): out[b,y,x] = win[b, window(y,x), slot(y,x)]
 * (+ residual[b,y,x] when residual != NULL, added in f32 and rounded once). win [B*nW, w*w, Cx]. */
int pscwin_window_merge(const void* win, int32_t B, int32_t H, int32_t W, int32_t Cx, int32_t window,
                        int32_t shift_x, int32_t shift_y, const void* residual, int32_t dtype, void* out,
                        void* stream);

/* ---------------------------------------------------------------------------------- step entry points */
/* LayerNorm over the last axis (Q15): out = (x - mean)/sqrt(var + eps) * g + b. x, out [rows, C]. */
int pscwin_layer_norm(const void* x, int64_t rows, int32_t C, const float* g, const float* b, float eps,
                      int32_t dtype, void* out, void* stream);
/* out[M, N] = A[M, K] . Wt[N, K]^T (+ bias[N]) (+ residual[M, N]); bf16 in, f32 accumulate on tcgen05,
 * out bf16 (out_f32 = 0) or f32 (out_f32 = 1, no residual). K % 8 == 0. (Projection step of a1/a3/a4/a7.) */
int pscwin_linear(const void* A, int64_t M, int32_t K, const void* Wt, int32_t N, const float* bias,
                  const void* residual, int32_t out_f32, void* out, void* stream);
/* a4: u = LN1(x); qkv = u W_qkv^T + b_qkv with 2-D RoPE applied to q and k at each token's grid coordinate
 * (Q6) -> qkv [B,H,W,3C] bf16; qkv_pad = p W_qkv^T + b_qkv [3C] f32 (unrotated).
 * Workspace: pscwin_workspace_bytes(desc). */
int pscwin_qkv_project(const pscwin_layer_desc* desc, const pscwin_layer_weights* wts, const void* x, void* qkv,
                       float* qkv_pad, void* workspace, size_t ws_bytes, void* stream);
/* a5 + a6 + crop: window attention core. qkv [B,H,W,3C] bf16 (q,k already rotated), qkv_pad [3C] f32
 * (required for shifted LEARNABLE layers, else may be NULL) -> O [B,H,W,C] bf16, heads contiguous.
 * Softmax over all w^2 slots (LEARNABLE) or over real slots only (MASKED). Pad query rows never written.
 * Workspace: pscwin_workspace_bytes(desc). */
int pscwin_window_attention(const pscwin_layer_desc* desc, const void* qkv, const float* qkv_pad, void* O,
                            void* workspace, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------------ a2: the cycle scan */
typedef struct {
  int32_t B, H, W;             /* L = H*W tokens per image, walked in scan_order                        */
  int32_t D, N, R, conv_k;     /* channels, SSM state (N <= 64), dt rank, conv width (L >= conv_k - 1)   */
  int32_t scan_order, bbar_mode, dtype;
  int32_t window;              /* WINDOW_MAJOR block size (H, W divisible by it); ignored by other orders */
} pscwin_scan_desc;
/* Cycle scan: per image the token sequence (in scan order) is repeated three times, the Mamba
 * selective SSM (block internals Q9) scans the 3L sequence, the three output segments are summed:
 *   v = SiLU(causal_conv(xin)) over the cycled sequence (copy 1 sees zero history, copies 2-3 the tail, Q10)
 *   (delta_low, B, C) = v W_x^T;  Delta = softplus(delta_low W_dt^T + b_dt);  A = -exp(a_log)
 *   h_j = exp(Delta A) h_{j-1} + B_bar v_j (Eq. 3-4);  y_j = C_j . h_j + d_skip * v_j
 *   out_t = sum_{c=0..2} y_{cL+t} * SiLU(z_t)   (no gate when z == NULL)
 * xin, z, out [B, L, D] bf16 in grid (row-major token) order; the recurrence walks the tokens in scan_order
 * (ROW_MAJOR raster, COL_MAJOR raster of the transpose, WINDOW_MAJOR windows in raster order with a raster
 * inside each window; reading Q13) — non-raster orders gather into scan order and scatter the result back. Computed exactly (up to rounding) by a
 * two-pass chunked closed form. Workspace: pscwin_scan_workspace_bytes. */
int pscwin_cycle_scan(const pscwin_scan_desc* desc, const void* xin, const void* z, const float* conv_w,
                      const float* conv_b, const void* w_x, const float* w_dt, const float* b_dt,
                      const float* a_log, const float* d_skip, void* out, void* workspace, size_t ws_bytes,
                      void* stream);
size_t pscwin_scan_workspace_bytes(const pscwin_scan_desc* desc);
/* Instrumentation: the chunk length (tokens) the bf16 two-pass scan would use for desc on the current device
 * (chosen from the pass-2 occupancy so the chunk x channel-block CTAs fill the SMs); 0 for an invalid desc or the
 * F32 path. Lets a caller account the carry's bytes (chunks x D x (N + 1) floats per image). */
int32_t pscwin_scan_chunk_length(const pscwin_scan_desc* desc);

/* ----------------------------------------------------------------------------------- the whole layer */
/* One PSCWin layer: [cycle-scan module: x += (cycle_scan(in_proj(LN_s(x)))) W_out^T] then
 * x_out = x + window_attention(qkv_project(x)) W_o^T + b_o, then [FFN sub-layer when mlp_hidden > 0:
 * x_out += GELU(LN2(x_out) W_fc1^T + b_fc1) W_fc2^T + b_fc2]. x_in, x_out [B,H,W,C] bf16; x_out may alias
 * x_in. Workspace: pscwin_workspace_bytes(desc). */
size_t pscwin_workspace_bytes(const pscwin_layer_desc* desc);
int pscwin_forward(const pscwin_layer_desc* desc, const pscwin_layer_weights* wts, const void* x_in, void* x_out,
                   void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- HRSAM++ multi-scale */
/* PAPER.md §3.4 "Multi-scale Fusion": the token grids of several input scales are concatenated
 * into one sequence ("patchified and concatenated ... (HW + H_sW_s)/16^2"). Window attention runs on
 * every scale's own grid ("tokens from the same scale remain contiguous", block-diagonal over windows; no window
 * spans two scales); the cycle-scan module runs SINGLE-SCALE ("splits the tokens by scale, scan each scale's
 * tokens separately") or MULTI-SCALE ("directly performs the SSM across the tokens from all the scales").
 * Packing (reading Q20): scale outermost — scale s occupies packed rows [B*off_s, B*off_{s+1}) as a
 * [B, H[s], W[s], C] grid, off_s = sum of the earlier scales' H*W (B = 1: the paper's per-sample concatenation).
 * The multi-scale SSM scans, per sample, the concatenation of every scale's scan-order sequence (scale order).
 * RoPE uses each scale's own grid coordinates (Q20). */
#define PSCWIN_MAX_SCALES 4
typedef enum { PSCWIN_CS_NONE = 0, PSCWIN_CS_SINGLE_SCALE = 1, PSCWIN_CS_MULTI_SCALE = 2 } pscwin_cs_mode;
typedef struct {
  pscwin_layer_desc layer;     /* B, C, heads, window, shifts, pad_mode, rope, ssm_*, scan_order, bbar_mode,
                                  dtype (BF16 only here), ln_eps; layer.H / layer.W / layer.cycle_scan ignored */
  int32_t n_scales;            /* 1 .. PSCWIN_MAX_SCALES                                                      */
  int32_t H[PSCWIN_MAX_SCALES], W[PSCWIN_MAX_SCALES];  /* token grid of each scale, in packing order          */
  int32_t attention;           /* 1: run the multi-scale window-attention sub-layer; 0: cycle-scan module only */
  int32_t cycle_scan;          /* pscwin_cs_mode of the cycle-scan module run before attention                 */
} pscwin_ms_desc;
/* Windows of all scales (sum of pscwin_window_count over the scales; ERR_CONTRACT as for each scale). */
int pscwin_ms_window_count(const pscwin_ms_desc* desc, int32_t* n_windows /* host, out */);
/* Host-side multi-scale indexing operator (App. C): destination = scale 0's windows (row-major,
 * slots row-major) then scale 1's, ...; value = source position in ONE sample's packed sequence (scale s token
 * y*W[s]+x at off_s + y*W[s] + x) or 0xFFFFFFFF (PAD). host_map holds n_windows * window^2 entries. */
int pscwin_ms_index_map(const pscwin_ms_desc* desc, uint32_t* host_map);
size_t pscwin_ms_workspace_bytes(const pscwin_ms_desc* desc);
/* One HRSAM++ layer over a packed multi-scale sequence: [cycle-scan module (single- or multi-scale)] then
 * [x += multi-scale window attention]. x_in, x_out [B * sum_s H[s]*W[s], C] bf16 (x_out may alias x_in).
 * Errors: ERR_CONTRACT for a scale grid that violates the layer's window contract (plain windows: H, W divisible
 * by window) or a scan shorter than conv_k - 1 tokens; ERR_UNSUPPORTED for dtype F32.
 * Workspace: pscwin_ms_workspace_bytes(desc). */
int pscwin_ms_forward(const pscwin_ms_desc* desc, const pscwin_layer_weights* wts, const void* x_in, void* x_out,
                      void* workspace, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------ encoder ends */
/* Patch embedding (ViT; a 1024^2 image gives 64 x 64 tokens): img [B, 3, 16H, 16W] bf16 (NCHW),
 * w_patch [C, 768] bf16 = a Conv2d(3, C, 16, stride 16) weight [C, 3, 16, 16] flattened, b_patch [C] f32 ->
 * out [B, H, W, C] bf16. No absolute position embedding (RoPE carries positions; reading Q22).
 * Internally a patchify gather into the workspace and one tcgen05 GEMM with the bias in its epilogue. */
size_t pscwin_patch_embed_workspace_bytes(int32_t B, int32_t H, int32_t W);
int pscwin_patch_embed(const void* img, int32_t B, int32_t H, int32_t W, int32_t C, const void* w_patch,
                       const float* b_patch, void* out, void* workspace, size_t ws_bytes, void* stream);
/* Bilinear resize (align_corners = False: half-pixel centres, clamped), channels-last bf16
 * in [B, h, w, Cx] -> out [B, H, W, Cx]; accumulate != 0 adds into out (f32 sum, one rounding). Cx % 8 == 0. */
int pscwin_resize_bilinear(const void* in, int32_t B, int32_t h, int32_t w, int32_t Cx, int32_t H, int32_t W,
                           int32_t accumulate, void* out, void* stream);
/* Output fusion of the four stages ("fusing outputs from all four stages through summation, followed by a
 * convolutional block"; P:L625 stage output dimension 256; reading Q22):
 *   f = sum_s stage_s W_s^T  (1x1 projections C -> C_out, no bias) on the main grid (scale 0);
 *   HRSAM++ (n_scales > 1): every other scale's f is bilinearly resized to the main grid and added;
 *   out = LN2d(conv3x3(LN2d(f))) (SAM neck block; conv zero padding 1, no bias).
 * stage_outs[s]: device pointer to stage s's output, packed [B * sum_j H[j] W[j], C] bf16 (scale-outermost, the
 * pscwin_ms_forward layout; one scale = [B, H, W, C]); w_stage[s] [C_out, C] bf16; ln* [C_out] f32;
 * w_conv [C_out, 3, 3, C_out] bf16 (o, dy, dx, i); out [B, H[0], W[0], C_out] bf16. The pointer arrays are host
 * arrays of device pointers. Workspace: pscwin_neck_workspace_bytes. */
typedef struct {
  int32_t B, C, C_out, n_stages, n_scales;
  int32_t H[PSCWIN_MAX_SCALES], W[PSCWIN_MAX_SCALES];
  float ln_eps;
} pscwin_neck_desc;
size_t pscwin_neck_workspace_bytes(const pscwin_neck_desc* desc);
int pscwin_neck(const pscwin_neck_desc* desc, const void* const* stage_outs, const void* const* w_stage,
                const float* ln1_g, const float* ln1_b, const void* w_conv, const float* ln2_g, const float* ln2_b,
                void* out, void* workspace, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------- row bands (multi-GPU, §8(e)) */
/* Window-row sharding of ONE image (B = 1) over `world` ranks, one band of token rows per rank (SURVEY §8(e),
 * config 4; cycle-scan carries per SURVEY Appendix A). row_begin / row_end are multiples of the window (the
 * last band ends at H); rank 0 starts at row 0, rank world-1 ends at H. Token-local steps run on the band.
 * The caller moves three kinds of bytes between ranks between the phase calls (NCCL over NVLink; every offset
 * below is relative to the workspace, all buffers device memory):
 *   conv history (cycle-scan layers, ring): hist_send of rank g -> hist_recv of rank (g+1) mod world;
 *   scan records (cycle-scan layers): all-gather rec_send of every rank into rec_recv, rank order;
 *   QKV halo (shifted layers): send_prev of rank g -> recv_next of rank g-1, send_next of g -> recv_prev of g+1
 *     (pt = (w - shift_y) mod w rows from above, w - pt from below; sizes 0 at the image edges).
 * Phase order: [cycle-scan layer: scan_begin, ring(hist), scan_mid, allgather(rec), scan_end]
 *              attn_begin, halo exchange, attn_end.
 * x_band, x_out [rows, W, C] bf16 (x_out may not alias x_band). Results equal pscwin_forward on the whole
 * image up to fp32 summation order in the scan (bit-identical elsewhere). bf16 only; scan_order ROW_MAJOR, or
 * WINDOW_MAJOR when H, W and both band edges are multiples of the window (a band of whole window rows is then a
 * contiguous run of the window-major sequence, scanned in band-local window-major order; the exchanged conv
 * history is the last k-1 tokens in that order); COL_MAJOR gives no contiguous segments: ERR_CONTRACT.
 * Workspace: pscwin_band_workspace_bytes. */
typedef struct {
  int32_t row_begin, row_end;  /* this rank's token rows [row_begin, row_end) */
  int32_t rank, world;
} pscwin_band;
typedef struct {
  uint64_t hist_send, hist_recv, hist_bytes;      /* conv history (k-1 xin rows of D bf16)                 */
  uint64_t rec_send, rec_recv, rec_bytes;         /* scan record; rec_recv holds world x rec_bytes           */
  uint64_t send_prev, send_prev_bytes, send_next, send_next_bytes;  /* QKV halo rows to the neighbours     */
  uint64_t recv_prev, recv_prev_bytes, recv_next, recv_next_bytes;  /* QKV halo rows from the neighbours   */
} pscwin_band_io;
size_t pscwin_band_workspace_bytes(const pscwin_layer_desc* global_desc, const pscwin_band* band);
int pscwin_band_io_offsets(const pscwin_layer_desc* global_desc, const pscwin_band* band, pscwin_band_io* io);
int pscwin_band_scan_begin(const pscwin_layer_desc* global_desc, const pscwin_band* band,
                           const pscwin_layer_weights* wts, const void* x_band, void* workspace, size_t ws_bytes,
                           void* stream);
int pscwin_band_scan_mid(const pscwin_layer_desc* global_desc, const pscwin_band* band,
                         const pscwin_layer_weights* wts, void* workspace, size_t ws_bytes, void* stream);
int pscwin_band_scan_end(const pscwin_layer_desc* global_desc, const pscwin_band* band,
                         const pscwin_layer_weights* wts, const void* x_band, void* workspace, size_t ws_bytes,
                         void* stream);
int pscwin_band_attn_begin(const pscwin_layer_desc* global_desc, const pscwin_band* band,
                           const pscwin_layer_weights* wts, const void* x_band, void* workspace, size_t ws_bytes,
                           void* stream);
int pscwin_band_attn_end(const pscwin_layer_desc* global_desc, const pscwin_band* band,
                         const pscwin_layer_weights* wts, const void* x_band, void* x_out, void* workspace,
                         size_t ws_bytes, void* stream);
/* pscwin_band_attn_end split for overlapping the halo exchange with compute (pscwin_dist_forward does this on two
 * streams): the band's extended image has *nwy padded-grid window rows; rows [*top, *bot) read no halo row (they
 * can run before the halo arrives), rows [0, *top) and [*bot, *nwy) read halo rows. pscwin_band_attn_windows runs
 * the window attention of rows [wy_begin, wy_end) (wy_begin == wy_end: nothing); after every row has run once,
 * pscwin_band_out_proj runs the out-proj + residual (+ FFN). Together they equal pscwin_band_attn_end. */
int pscwin_band_window_split(const pscwin_layer_desc* global_desc, const pscwin_band* band, int32_t* top,
                             int32_t* bot, int32_t* nwy);
int pscwin_band_attn_windows(const pscwin_layer_desc* global_desc, const pscwin_band* band,
                             const pscwin_layer_weights* wts, void* workspace, size_t ws_bytes, int32_t wy_begin,
                             int32_t wy_end, void* stream);
int pscwin_band_out_proj(const pscwin_layer_desc* global_desc, const pscwin_band* band,
                         const pscwin_layer_weights* wts, const void* x_band, void* x_out, void* workspace,
                         size_t ws_bytes, void* stream);

/* One layer of a window-row-sharded image with the exchanges done inside the library over NCCL (SURVEY §8(b)
 * pscwin_dist_forward; §8(e)): the rank / world come from the communicator (an ncclComm_t passed as void*, from
 * the caller's own NCCL setup or pscwin_nccl_comm_init), the band is [row_begin, row_end) as for the band
 * phases. Kernels and the latency-sized scan exchanges (conv-history ring send/recv, ncclAllGather of the scan
 * records) run on `stream` (compute). The QKV halo send/recv with the neighbours runs on `comm_stream` when it is
 * non-NULL and differs from `stream`: it waits (event) for this band's QKV rows, the windows that need no halo row
 * are computed on `stream` meanwhile, then `stream` waits (event) for the halo and computes the band-edge windows
 * and the out-proj (SURVEY §8(e) overlap). comm_stream NULL: everything on `stream`. Both streams must be usable
 * by the caller's CUDA graph capture (the call is capturable: the fork / join are event edges). Every rank of the
 * communicator must call it for the same layer. x_band, x_band_out [rows, W, C] bf16 (no alias). Workspace:
 * pscwin_dist_workspace_bytes (= pscwin_band_workspace_bytes). Errors: as the band phases; PSCWIN_ERR_NCCL for an
 * NCCL call that fails, or when the communicator already carries an asynchronous error (checked on entry). */
int pscwin_nccl_get_unique_id(void* id_out /* host, 128 bytes */);
int pscwin_nccl_comm_init(const void* id /* host, 128 bytes */, int32_t world, int32_t rank, void** comm_out);
int pscwin_nccl_comm_destroy(void* comm);  /* after every CUDA graph holding its operations is destroyed */
/* Failure detection for the multi-GPU path: a rank that dies or stalls leaves its peers' NCCL kernels
 * spinning. pscwin_nccl_comm_check returns PSCWIN_ERR_NCCL if NCCL reports an asynchronous error on `comm`
 * (ncclCommGetAsyncError; e.g. a remote failure or a previous abort), else PSCWIN_OK; host only, never blocks.
 * pscwin_nccl_comm_abort aborts every outstanding operation on `comm` (ncclCommAbort; the communicator is freed and
 * must not be used again, its stream's pending work completes with the operations cancelled).
 * pscwin_nccl_wait polls `stream` (cudaStreamQuery) and `comm` (async error) every ~100 us until the stream has
 * drained (PSCWIN_OK), an async error appears (the comm is aborted, PSCWIN_ERR_NCCL) or timeout_ms passes (the comm
 * is aborted, PSCWIN_ERR_TIMEOUT); timeout_ms <= 0 waits without a deadline. A CUDA error on the stream gives
 * PSCWIN_ERR_CUDA. After an abort the caller re-creates the communicator (pscwin_nccl_comm_init) to go on. */
int pscwin_nccl_comm_check(void* comm);
int pscwin_nccl_comm_abort(void* comm);
int pscwin_nccl_wait(void* comm, void* stream, int64_t timeout_ms);
size_t pscwin_dist_workspace_bytes(const pscwin_layer_desc* global_desc, int32_t row_begin, int32_t row_end,
                                   int32_t rank, int32_t world);
int pscwin_dist_forward(const pscwin_layer_desc* global_desc, const pscwin_layer_weights* wts, const void* x_band,
                        void* x_band_out, int32_t row_begin, int32_t row_end, void* nccl_comm, void* workspace,
                        size_t ws_bytes, void* stream, void* comm_stream);

/* ------------------------------------------------------------------------------------ instrumentation */
/* Kernel launches issued by this library since it was loaded (every launcher counts itself). */
int64_t pscwin_launch_count(void);
/* on != 0: from now on every launch records a CUDA event pair on its own stream (bench.py per-kernel
 * timing); any call clears the records collected so far. Not thread-safe against concurrent reads. */
void pscwin_profile_enable(int on);
/* Synchronises on the recorded events and aggregates them by kernel label. Writes up to max_entries labels
 * ('\n'-separated, NUL-terminated, into names[names_len]), their summed milliseconds and launch counts
 * (host arrays). Returns the number of labels written. */
int pscwin_profile_read(char* names, size_t names_len, double* total_ms, int32_t* counts, int32_t max_entries);

#ifdef __cplusplus
}
#endif
#endif /* PSCWIN_H_ */
