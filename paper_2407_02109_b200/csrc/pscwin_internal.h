// Internal (non-ABI) declarations shared by the .cu translation units of libpscwin.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/pscwin.h"
#include "launch.h"
#include "prof.h"

namespace pscwin {

enum GemmEpilogue { EPI_STORE_BF16 = 0, EPI_STORE_F32 = 1, EPI_QKV_ROPE = 2, EPI_RESID_BF16 = 3 };

struct GemmArgs {
  int M, N, K;
  int lda, ldb;          // elements (row strides of A [M,K] and B [N,K])
  void* out;
  int ldo;               // elements
  int epi;               // GemmEpilogue
  int BN;                // 0 = auto
  const float* bias;     // [N] or null
  const void* residual;  // bf16 [M, ldr] or null
  int ldr;
  // QKV + RoPE epilogue
  int rope, HW, Wgrid, C, d_head;
  const char* prof_name;  // kernel label for pscwin_profile_read
  // split-K (f32 output only): splits > 1 needs partial [splits][M][N] f32 and sem [m_tiles * n_tiles] ints that
  // are zero before the first launch (the kernel leaves them zero again)
  int splits;
  float* partial;
  int* sem;
  // bf16 epilogues: columns >= silu_col leave as SiLU(value) (0 = off; must be a multiple of the tile width)
  int silu_col;
  int tf32;      // 1: A and B are f32 (row strides lda / ldb in f32 elements) multiplied as TF32 (kind::tf32,
                 //    K-blocks of 32); f32 output only
  int softplus;  // 1 (f32 output): softplus(value + bias) (the cycle scan's Delta = softplus(delta_low W_dt^T + b_dt))
  int gelu;    // 1: exact GELU 0.5 x (1 + erf(x / sqrt 2)) on every output (after bias; FFN fc1, reading Q21)
  int tok0;    // RoPE: global token index of GEMM row 0 (a row band of the image; 0 otherwise)
  // RoPE over a packed multi-scale sequence (HRSAM++): rows [seg_row[s], seg_row[s+1]) hold [B, H_s, W_s] grids
  // (seg_HW[s] = H_s*W_s, seg_W[s] = W_s); nseg <= 1 = one grid described by HW / Wgrid
  int nseg;
  int seg_row[4], seg_HW[4], seg_W[4];
  int stages;  // smem ring depth (set by the launcher)
  int f32_tma;  // f32 output staged in smem and TMA-stored (set by the launcher)
  int pair;    // 1 = 2-CTA cluster tiles (set by the launcher; PSCWIN_GEMM_PAIR=0 disables)
  int warp_epi;  // 1 = per-warp bf16 epilogue (32 x 32 boxes, no CTA-wide barrier per chunk; set by the launcher)
  int nbuf;       // per-warp epilogue: 2 KB staging boxes per warp, 1 or 2 (set by the launcher)
  int res_global;  // per-warp epilogue: residual read from global memory by the epilogue threads (launcher)
  int dbg_noepi;  // timing probe (PSCWIN_GEMM_DBG_NOEPI=1): bf16 epilogue warps release the accumulator untouched
  // LayerNorm folded into this projection (bf16 epilogues; rowops.cu ln_fold_kernel): A = x (not normalised),
  // B = W' = W diag(gamma), bias = c = W beta + b; the epilogue computes rstd_m (acc - mu_m s_n) + c_n
  const float2* ln_stats;  // [M] (mu, rstd) per A row, or null (no folding)
  const float* ln_colsum;  // [N] s_n = sum_k W'[n,k]
  int bias_l1;  // bf16 epilogue reads bias / column sums through L1 (no per-tile staging barrier; set by the launcher)
};

// host helpers (abi.cu)
int num_sms();
// A helper stream with a fork / join event pair, private to the calling host thread and to the current device
// (thread_local, indexed by device): concurrent callers on other threads never share its events, and one process
// can drive several GPUs. Slot 0: the side stream of the weight-only pad work; slot 1: the default-stream proxy of
// pscwin_dist_forward; slot 2: the halo-overlap events of pscwin_dist_forward. Created on first use, never
// destroyed (one set per thread and device). nullptr when creation fails.
struct AuxStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // extra join points (one per consumer)
  bool ok = false;
};
// A LayerNorm folded into the projection that follows it (rowops.cu): W' = W diag(gamma) [N, K] bf16, s [N],
// c = W beta + b [N] (weight-only, produced by launch_ln_fold, ready once `ready` has been waited on; null =
// stream-ordered), and a [T] float2 scratch for the row statistics of the projection's input.
struct LnFold {
  const void* wf;
  const float* colsum;
  const float* bias;
  float2* stats;
  cudaEvent_t ready;
};
AuxStream* aux_stream(int slot);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize, bytes) for `fn` on the current device, once per (device,
// function) and only when `bytes` exceeds what was set before (thread-safe; abi.cu).
void func_smem_once(const void* fn, int bytes);
// row-band attention phases (abi.cu), used by pscwin_dist_forward to overlap the QKV halo exchange
int band_attention(const pscwin_layer_desc* d, const pscwin_band* b, const pscwin_layer_weights* wt, void* ws,
                   size_t ws_bytes, int wy0, int wy1, int tables_ready, void* stream);
void band_window_rows(const pscwin_layer_desc* d, const pscwin_band* b, int* top, int* bot, int* nwy);
int band_out_proj(const pscwin_layer_desc* d, const pscwin_band* b, const pscwin_layer_weights* wt,
                  const void* x_band, void* x_out, void* ws, size_t ws_bytes, void* stream);
int make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, uint64_t inner, uint64_t outer,
                 uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz);
int make_tmap_5d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, const uint64_t dims[5],
                 const uint64_t strides_bytes[4], const uint32_t box[5], CUtensorMapSwizzle swz);

// launchers (return 0 or a cudaError_t / negative internal code)
int launch_partition(const void* x, const void* pad_row, int B, int H, int W, int Cx, int w, int sx, int sy,
                     int esize, void* out, cudaStream_t stream);
int launch_merge(const void* win, int B, int H, int W, int Cx, int w, int sx, int sy, const void* residual,
                 int is_f32, void* out, cudaStream_t stream);
int launch_gemm_bf16(const void* A, const void* B, const GemmArgs& args, cudaStream_t stream);
// bf16 row gather (scan order <- grid order, scatter = 0) or scatter (grid order <- scan order) of B [H, W] grids of
// D-channel rows in the given scan order (cyclescan.cu)
int launch_permute_rows(const __nv_bfloat16* src, long long ld_src, __nv_bfloat16* dst, long long ld_dst, int B, int H,
                        int W, int D, int order, int w, int scatter, cudaStream_t s);
int launch_row_stats(const void* x, long long rows, int C, float eps, float2* stats, cudaStream_t stream);
int launch_ln_fold(const void* W, int N, int K, const float* g, const float* beta, const float* bias, void* Wf,
                   float* s, float* c, cudaStream_t stream);
int launch_layer_norm(const void* x, long long rows, int C, const float* g, const float* b, float eps, int is_f32,
                      void* out, cudaStream_t stream);
int launch_pad_qkv(const void* pad, const void* w_qkv, const float* b_qkv, int C, int is_f32, float* out,
                   cudaStream_t stream);

struct AttnArgs {
  int B, H, W, C, heads, d, w, sx, sy, pad_mode, rope;
  int row0;              // global grid row of local row 0 (row bands: RoPE of pad keys at global coordinates)
  const void* qkv;       // [B,H,W,3C] bf16 (q,k rotated at their grid coordinates)
  const float* qkv_pad;  // [3C] f32 projection of p (unrotated) or null (plain / masked)
  void* out;             // [B,H,W,C] bf16
  void* pad_tab;         // workspace for rotated pad K halves + V (bf16)
  int tables_ready;      // 1: pad_tab was already filled by launch_pad_tables (e.g. on a side stream)
  int wy_begin, wy_end;  // padded-grid window rows to run, [wy_begin, wy_end); wy_end <= 0: all (row-band overlap)
};
size_t attn_pad_table_bytes(int H, int W, int C, int w);
// rotated pad-key / pad-value tables of a shifted LEARNABLE layer (depends only on qkv_pad and the geometry)
int launch_pad_tables(const AttnArgs& a, cudaStream_t stream);
int launch_window_attention(const AttnArgs& a, cudaStream_t stream);
int launch_window_attention_ws(const AttnArgs& a, const void* kx, const void* ky, const void* vp, int patch,
                               cudaStream_t stream);

}  // namespace pscwin


namespace pscwin {
// fp32 correctness path (f32path.cu)
struct LayerWsF32 {
  size_t u, qkv, qkv_pad, O, h, xz, g, scan, x1, total;
};
LayerWsF32 plan_layer_f32(const pscwin_layer_desc* d);
size_t layer_f32_ws_bytes(const pscwin_layer_desc* d);
size_t scan_f32_ws_bytes(int B, int L, int D, int N, int R, int k);
int forward_f32(const pscwin_layer_desc* d, const pscwin_layer_weights* wt, const void* x_in, void* x_out, void* ws,
                size_t ws_bytes, cudaStream_t s);
int qkv_project_f32(const pscwin_layer_desc* d, const pscwin_layer_weights* wt, const float* x, float* qkv,
                    float* qkv_pad, float* u, cudaStream_t s);
int launch_attention_f32(const pscwin_layer_desc* d, const float* qkv, const float* qkv_pad, float* out,
                         cudaStream_t s);
int run_cycle_scan_f32(int B, int H, int W, int order, int window, int D, int N, int R, int k, int bbar,
                       const float* xin, long long ld_x, const float* z, long long ld_z, bool z_gated,
                       const float* conv_w, const float* conv_b, const float* w_x, const float* w_dt,
                       const float* b_dt, const float* a_log, const float* d_skip, float* out, long long ld_out,
                       void* ws, size_t ws_bytes, cudaStream_t s);
// band mode of the cycle scan (cyclescan.cu)
size_t band_scan_ws_bytes(int L, int D, int N, int R, int k, int P);
size_t band_scan_record_bytes(int D, int N);
int band_scan_mid(int L, int D, int N, int R, int k, int P, int bbar, const __nv_bfloat16* xin, long long ld_x,
                  const __nv_bfloat16* hist, const float* conv_w, const float* conv_b, const void* w_x,
                  const float* w_dt, const float* b_dt, const float* a_log, const float* d_skip, float* rec, void* ws,
                  size_t ws_bytes, cudaStream_t s);
int band_scan_end(int L, int D, int N, int R, int k, int P, int bbar, const __nv_bfloat16* xin, long long ld_x,
                  const __nv_bfloat16* gz, long long ld_gz, const float* conv_w, const float* conv_b,
                  const float* w_dt, const float* b_dt, const float* a_log, const float* d_skip, const float* recs,
                  int rank, int world, __nv_bfloat16* out, long long ld_out, void* ws, size_t ws_bytes,
                  cudaStream_t s);
// packed multi-scale sequence (HRSAM++; reading Q20): scale s holds packed rows
// [B*off[s], B*off[s+1]) as a [B, H[s], W[s]] grid (off = per-sample token offsets)
struct MsGeo {
  int n;
  int off[5];
  int H[4], W[4];
};
size_t ms_scan_ws_bytes(int B, const MsGeo& g, int mode, int D, int N, int R, int k, int order);
// cycle-scan module over a packed multi-scale sequence: mode 1 = single-scale (each scale its own cycled
// sequence), 2 = multi-scale (one cycled sequence per sample over all scales)
int ms_cycle_scan_module(const void* desc, const void* wts, const MsGeo& g, int mode, const void* x_in, void* x_out,
                         void* ws, size_t off_u, size_t off_xz, size_t off_g, size_t off_scan, size_t scan_bytes,
                         cudaStream_t s);
// FFN sub-layer (NEXT-2): x += GELU(LN2(x) W_fc1^T + b_fc1) W_fc2^T + b_fc2 over T rows, in place; u [T, C] and
// h [T, hidden] bf16 scratch
int ffn_bf16(long long T, int C, int hidden, float eps, const void* wts, void* x, void* u, void* h, cudaStream_t s,
             const LnFold* lnf = nullptr);
// GEMM whose A operand is LayerNorm(x) (gamma g, beta be, eps): with lnf, the row statistics of x and the folded
// projection (A = x itself); without, the LayerNorm pass into u and the plain projection. a.bias is the
// projection's own bias (replaced by lnf->bias when folded); a.M / a.K are the rows / width of x.
int ln_gemm(const void* x, const float* g, const float* be, float eps, const void* W, GemmArgs a, void* u,
            const LnFold* lnf, cudaStream_t s);
// cycle-scan module of a layer (a1-a3): x_out = x_in + out_proj(cycle_scan(in_proj(LN_s(x_in))))
int cycle_scan_module(const void* desc, const void* wts, const LnFold* lnf, const void* x_in, void* x_out, void* ws,
                      size_t off_u,
                      size_t off_xz, size_t off_g, size_t off_scan, size_t scan_bytes, cudaStream_t s);
}  // namespace pscwin
