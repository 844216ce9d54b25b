// C-ABI entry points of libpscwin.so (declared and documented in include/pscwin.h): argument / contract
// validation, workspace planning, TMA descriptor encoding and the per-layer launch sequence.
#include <stdio.h>

#include <map>
#include <mutex>
#include <utility>
#include <stdlib.h>
#include <string.h>

#include "../../include/pscwin.h"
#include "common.cuh"
#include "pscwin_internal.h"

namespace pscwin {

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

int make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, uint64_t inner, uint64_t outer,
                 uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return -10;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -11;
}

int make_tmap_5d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, const uint64_t dims_in[5],
                 const uint64_t strides_in[4], const uint32_t box_in[5], CUtensorMapSwizzle swz) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return -10;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 5; ++i) {
    dims[i] = dims_in[i];
    box[i] = box_in[i];
  }
  for (int i = 0; i < 4; ++i) strides[i] = strides_in[i];
  CUresult r = fn(m, dt, 5, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -11;
}

int ln_gemm(const void* x, const float* g, const float* be, float eps, const void* W, GemmArgs a, void* u,
            const LnFold* lnf, cudaStream_t s) {
  if (!lnf) {
    int rc = launch_layer_norm(x, a.M, a.K, g, be, eps, 0, u, s);
    if (rc) return rc;
    return launch_gemm_bf16(u, W, a, s);
  }
  int rc = launch_row_stats(x, a.M, a.K, eps, lnf->stats, s);
  if (rc) return rc;
  if (lnf->ready && cudaStreamWaitEvent(s, lnf->ready, 0) != cudaSuccess) return (int)cudaErrorUnknown;
  a.bias = lnf->bias;
  a.ln_stats = lnf->stats;
  a.ln_colsum = lnf->colsum;
  return launch_gemm_bf16(x, lnf->wf, a, s);
}

int ffn_bf16(long long T, int C, int hidden, float eps, const void* wts_v, void* x, void* u, void* h,
             cudaStream_t s, const LnFold* lnf) {
  const pscwin_layer_weights* w = reinterpret_cast<const pscwin_layer_weights*>(wts_v);
  int rc;
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.prof_name = "gemm_fc1_gelu";
  a.M = (int)T;
  a.N = hidden;
  a.K = C;
  a.lda = C;
  a.ldb = C;
  a.out = h;
  a.ldo = hidden;
  a.epi = EPI_STORE_BF16;
  a.bias = (const float*)w->b_fc1;
  a.gelu = 1;
  rc = ln_gemm(x, (const float*)w->ln2_g, (const float*)w->ln2_b, eps, w->w_fc1, a, u, lnf, s);
  if (rc) return PSCWIN_ERR_CUDA;
  memset(&a, 0, sizeof(a));
  a.prof_name = "gemm_fc2";
  a.M = (int)T;
  a.N = C;
  a.K = hidden;
  a.lda = hidden;
  a.ldb = hidden;
  a.out = x;
  a.ldo = C;
  a.epi = EPI_RESID_BF16;
  a.bias = (const float*)w->b_fc2;
  a.residual = x;  // in place: every output tile reads its own residual tile before storing it
  a.ldr = C;
  return launch_gemm_bf16(h, w->w_fc2, a, s) ? PSCWIN_ERR_CUDA : PSCWIN_OK;
}

}  // namespace pscwin

using namespace pscwin;

namespace {

inline bool aligned16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline int status_from(int rc) {
  if (rc == 0) return PSCWIN_OK;
  if (rc == -2) return PSCWIN_ERR_UNSUPPORTED;
  if (rc == -3) return PSCWIN_ERR_CONTRACT;
  return PSCWIN_ERR_CUDA;
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Geo {
  int pt, pl, pb, pr, nw;
};

int geometry(int H, int W, int w, int sx, int sy, Geo* g) {
  if (H <= 0 || W <= 0 || w <= 0) return PSCWIN_ERR_SHAPE;
  if (sx < 0 || sy < 0 || sx >= w || sy >= w) return PSCWIN_ERR_CONTRACT;
  if (sx == 0 && sy == 0 && (H % w || W % w)) return PSCWIN_ERR_CONTRACT;
  g->pl = (w - sx) % w;
  g->pt = (w - sy) % w;
  g->pr = ((-(g->pl + W)) % w + w) % w;
  g->pb = ((-(g->pt + H)) % w + w) % w;
  g->nw = ((g->pt + H + g->pb) / w) * ((g->pl + W + g->pr) / w);
  return PSCWIN_OK;
}

int check_layer(const pscwin_layer_desc* d) {
  if (!d) return PSCWIN_ERR_SHAPE;
  if (d->B <= 0 || d->H <= 0 || d->W <= 0 || d->C <= 0 || d->heads <= 0) return PSCWIN_ERR_SHAPE;
  if (d->C % d->heads) return PSCWIN_ERR_CONTRACT;
  Geo g;
  int rc = geometry(d->H, d->W, d->window, d->shift_x, d->shift_y, &g);
  if (rc) return rc;
  const int dh = d->C / d->heads;
  if (d->rope && dh % 4) return PSCWIN_ERR_CONTRACT;
  if (d->dtype != PSCWIN_BF16 && d->dtype != PSCWIN_F32) return PSCWIN_ERR_UNSUPPORTED;
  if (!(dh == 32 || dh == 64)) return PSCWIN_ERR_UNSUPPORTED;
  if (d->dtype == PSCWIN_F32 && d->window > 16) return PSCWIN_ERR_UNSUPPORTED;  // f32 window lives in smem
  if (d->window < 4 || d->window > 128 || (d->window & (d->window - 1))) return PSCWIN_ERR_UNSUPPORTED;
  if (d->pad_mode != PSCWIN_PAD_LEARNABLE && d->pad_mode != PSCWIN_PAD_MASKED) return PSCWIN_ERR_CONTRACT;
  if (d->C % 64) return PSCWIN_ERR_UNSUPPORTED;  // GEMM K tiles
  if (d->mlp_hidden < 0 || d->mlp_hidden % 64) return PSCWIN_ERR_CONTRACT;
  return PSCWIN_OK;
}

bool ffn_weights_ok(const pscwin_layer_weights* w) {
  return w->ln2_g && w->ln2_b && w->w_fc1 && w->b_fc1 && w->w_fc2 && w->b_fc2;
}

// Workspace layout shared by qkv_project / window_attention / forward.
struct LayerWs {
  size_t u, qkv, qkv_pad, O, pad_tab, xz, g, h, scan, total;
  size_t stats, f_qkv, f_in, f_fc1;  // folded-LayerNorm scratch: row stats [T] float2; W' | s | c per projection
};

// LayerNorm folded into the projection after it (rowops.cu). Off by default (PSCWIN_LN_FOLD=1 enables it; A/B
// knob, read once): measured at 4096^2 (ncu, one eager step, profiles/r02/ln_fold_r02c.md) the row-stats pass
// saves 19 us per LayerNorm but the folded epilogue (two more FMAs per element, s_n from shared memory, register
// spills in the RoPE variant) makes the QKV GEMM 186 -> 213 us and in_proj 235 -> 272 us: the projections'
// epilogues, not their tensor pipes, bound them once the LayerNorm work moves in.
// PSCWIN_LN_FOLD = 2 (default): LN1 folded into the QKV projection on every path (whole image, row bands,
// multi-scale), LN_s -> in_proj and LN2 -> fc1 kept as LayerNorm passes; 1: all three folded (whole-image path);
// 0: no folding. Measured at 4096^2 (profiles/r02/ln_fold_r02x.log, bench --breakdown): the row-stats pass
// (33 us) replaces the LayerNorm (45 us) while the folded RoPE epilogue now costs the QKV GEMM < 1 us (the round-2
// per-warp epilogue; 27 us with the round-1 epilogue, r02c); in_proj's folded epilogue still costs +14 us, more
// than its LayerNorm saving, so LN_s stays a pass.
// Folding applies to images of at least PSCWIN_LN_FOLD_MIN_T tokens (B H W of the WHOLE image, so whole-image, band
// and multi-scale paths of one problem choose alike): at 1024^2 (4096 tokens) the weight fold on the side stream is
// not hidden behind the short row-stats pass and the stage measured 0.372 -> 0.391 ms with it.
int ln_fold_mode(long long tokens) {
  static const int mode = env_knob("PSCWIN_LN_FOLD", 2);
  static const int min_t = env_knob("PSCWIN_LN_FOLD_MIN_T", 16384);
  if (tokens < min_t) return 0;
  return (mode == 0 || mode == 1) ? mode : 2;
}
size_t fold_bytes(size_t N, size_t K) { return align256(N * K * 2) + align256(N * 4) * 2; }
LnFold fold_at(void* ws, size_t off, size_t N, size_t K, size_t stats_off) {
  LnFold f;
  uint8_t* b = reinterpret_cast<uint8_t*>(ws) + off;
  f.wf = b;
  f.colsum = reinterpret_cast<const float*>(b + align256(N * K * 2));
  f.bias = reinterpret_cast<const float*>(b + align256(N * K * 2) + align256(N * 4));
  f.stats = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(ws) + stats_off);
  f.ready = nullptr;
  return f;
}
int fold_launch(const LnFold& f, const void* W, int N, int K, const void* g, const void* be, const void* bias,
                cudaStream_t s) {
  return launch_ln_fold(W, N, K, (const float*)g, (const float*)be, (const float*)bias, const_cast<void*>(f.wf),
                        const_cast<float*>(f.colsum), const_cast<float*>(f.bias), s);
}

// LN1 -> QKV on the band and multi-scale paths: LayerNorm pass + GEMM, or (ln_fold_mode() != 0) the weight fold on
// the layer's stream, then the row statistics and the folded GEMM -- the same arithmetic as the whole-image forward,
// so the three paths stay bit-identical. fold_ws: fold_bytes(3C, C) bytes; stats: [M] float2.
int ln1_qkv(const pscwin_layer_weights* wt, float eps, const void* x, GemmArgs a, void* u, void* fold_ws,
            float2* stats, long long image_tokens, cudaStream_t s) {
  if (ln_fold_mode(image_tokens) == 0) return ln_gemm(x, (const float*)wt->ln1_g, (const float*)wt->ln1_b, eps, wt->w_qkv, a, u,
                                          nullptr, s);
  LnFold f;
  uint8_t* b = reinterpret_cast<uint8_t*>(fold_ws);
  const size_t N = a.N, K = a.K;
  f.wf = b;
  f.colsum = reinterpret_cast<const float*>(b + align256(N * K * 2));
  f.bias = reinterpret_cast<const float*>(b + align256(N * K * 2) + align256(N * 4));
  f.stats = stats;
  f.ready = nullptr;
  const int rc = fold_launch(f, wt->w_qkv, a.N, a.K, wt->ln1_g, wt->ln1_b, wt->b_qkv, s);
  if (rc) return rc;
  return ln_gemm(x, (const float*)wt->ln1_g, (const float*)wt->ln1_b, eps, wt->w_qkv, a, u, &f, s);
}

LayerWs plan_layer(const pscwin_layer_desc* d) {
  LayerWs w;
  const size_t T = (size_t)d->B * d->H * d->W;
  const size_t C = d->C;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return o;
  };
  w.u = take(T * C * 2);
  w.qkv = take(T * 3 * C * 2);
  w.qkv_pad = take(3 * C * 4);
  w.O = take(T * C * 2);
  w.pad_tab = take(attn_pad_table_bytes(d->H, d->W, d->C, d->window));
  w.h = d->mlp_hidden > 0 ? take(T * d->mlp_hidden * 2) : 0;
  w.xz = w.g = w.scan = 0;
  if (d->cycle_scan) {
    const size_t D = (size_t)d->ssm_expand * C;
    w.xz = take(T * 2 * D * 2);
    w.g = take(T * D * 2);
    pscwin_scan_desc sd;
    sd.B = d->B;
    sd.H = d->H;
    sd.W = d->W;
    sd.D = (int)D;
    sd.N = d->ssm_state;
    sd.R = d->ssm_dt_rank > 0 ? d->ssm_dt_rank : (d->C + 15) / 16;
    sd.conv_k = d->ssm_conv;
    sd.scan_order = d->scan_order;
    sd.bbar_mode = d->bbar_mode;
    sd.dtype = d->dtype;
    sd.window = d->window;
    w.scan = take(pscwin_scan_workspace_bytes(&sd));
  }
  w.stats = take(T * 8);
  w.f_qkv = take(fold_bytes(3 * C, C));
  w.f_in = d->cycle_scan ? take(fold_bytes(2 * (size_t)d->ssm_expand * C, C)) : 0;
  w.f_fc1 = d->mlp_hidden > 0 ? take(fold_bytes(d->mlp_hidden, C)) : 0;
  w.total = off;
  return w;
}

uint8_t* wsp(void* base, size_t off) { return reinterpret_cast<uint8_t*>(base) + off; }

int qkv_project_impl(const pscwin_layer_desc* d, const pscwin_layer_weights* wt, const void* x, void* qkv,
                     float* qkv_pad, void* ws, const LayerWs& L, cudaStream_t s, const LnFold* lnf = nullptr) {
  const long long T = (long long)d->B * d->H * d->W;
  const int C = d->C;
  void* u = wsp(ws, L.u);
  int rc;
  const int dh = C / d->heads;
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.M = (int)T;
  a.N = 3 * C;
  a.K = C;
  a.lda = C;
  a.ldb = C;
  a.out = qkv;
  a.ldo = 3 * C;
  a.epi = EPI_QKV_ROPE;
  a.prof_name = "gemm_qkv_rope";
  a.bias = (const float*)wt->b_qkv;
  a.rope = d->rope;
  a.HW = d->H * d->W;
  a.Wgrid = d->W;
  a.C = C;
  a.d_head = dh;
  rc = ln_gemm(x, (const float*)wt->ln1_g, (const float*)wt->ln1_b, d->ln_eps, wt->w_qkv, a, u, lnf, s);
  if (rc) return rc;
  if (qkv_pad && wt->pad) {
    rc = launch_pad_qkv(wt->pad, wt->w_qkv, (const float*)wt->b_qkv, C, 0, qkv_pad, s);
    if (rc) return rc;
  }
  return 0;
}

AttnArgs attn_args(const pscwin_layer_desc* d, const void* qkv, const float* qkv_pad, void* O, void* pad_tab) {
  AttnArgs a;
  memset(&a, 0, sizeof(a));
  a.B = d->B;
  a.H = d->H;
  a.W = d->W;
  a.C = d->C;
  a.heads = d->heads;
  a.d = d->C / d->heads;
  a.w = d->window;
  a.sx = d->shift_x;
  a.sy = d->shift_y;
  a.pad_mode = d->pad_mode;
  a.rope = d->rope;
  a.row0 = 0;
  a.qkv = qkv;
  a.qkv_pad = qkv_pad;
  a.out = O;
  a.pad_tab = pad_tab;
  return a;
}

int attention_impl(const pscwin_layer_desc* d, const void* qkv, const float* qkv_pad, void* O, void* ws,
                   const LayerWs& L, cudaStream_t s, int tables_ready = 0) {
  AttnArgs a = attn_args(d, qkv, qkv_pad, O, wsp(ws, L.pad_tab));
  a.tables_ready = tables_ready;
  return launch_window_attention(a, s);
}

// The side stream (aux_stream slot 0) for the weight-only pad work of a shifted LEARNABLE layer (qkv_pad =
// p W_qkv^T + b and its rotated pad-key / value tables): forked from the caller's stream at the start of the
// attention sub-layer and joined before the attention kernel, so it overlaps LN1 + the QKV GEMM instead of sitting
// on the critical path. Event fork / join is captured into CUDA graphs as graph edges. PSCWIN_NO_SIDE_STREAM=1 runs
// the pad work on the caller's stream (A/B knob, read once).
AuxStream* side() {
  static const bool off = getenv("PSCWIN_NO_SIDE_STREAM") != nullptr;
  return off ? nullptr : aux_stream(0);
}

}  // namespace

namespace pscwin {
void func_smem_once(const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[{dev, fn}];
  if (bytes > have && cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess)
    have = bytes;
}

AuxStream* aux_stream(int slot) {
  constexpr int kDev = 16, kSlots = 3;
  thread_local AuxStream tab[kDev][kSlots];
  int dev = 0;
  if (slot < 0 || slot >= kSlots || cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kDev) {
    cudaGetLastError();
    return nullptr;
  }
  AuxStream& a = tab[dev][slot];
  if (!a.ok) {
    // PSCWIN_AUX_PRIO=1 (A/B knob) gives the side stream (short weight-only kernels a main-stream kernel waits for:
    // LayerNorm weight fold, pad token projection / tables) the highest priority. Measured at 4096^2: the side kernels'
    // event times drop (weight fold 32 -> 11 us, pad tables 118 -> 24 us) but the step does not change beyond the
    // run-to-run spread (15.02 / 15.01 vs 14.87 / 15.07 ms, profiles/r02/aux_prio_r02aa.log): off by default.
    static const int prio_on = env_knob("PSCWIN_AUX_PRIO", 0);
    int lo = 0, hi = 0;
    if (prio_on && cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess) {
      if (!a.s && cudaStreamCreateWithPriority(&a.s, cudaStreamNonBlocking, hi) != cudaSuccess) a.s = nullptr;
    } else if (!a.s && cudaStreamCreateWithFlags(&a.s, cudaStreamNonBlocking) != cudaSuccess) {
      a.s = nullptr;
    }
    if (!a.fork && cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming) != cudaSuccess) a.fork = nullptr;
    if (!a.join && cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming) != cudaSuccess) a.join = nullptr;
    bool evs = true;
    for (cudaEvent_t& e : a.ev)
      if (!e && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) e = nullptr, evs = false;
    a.ok = a.s && a.fork && a.join && evs;
    if (!a.ok) {
      cudaGetLastError();
      return nullptr;
    }
  }
  return &a;
}
}  // namespace pscwin

extern "C" {

const char* pscwin_version(void) { return "pscwin-b200 0.1 (sm_100a)"; }

const char* pscwin_status_string(int st) {
  switch (st) {
    case PSCWIN_OK: return "ok";
    case PSCWIN_ERR_SHAPE: return "shape error";
    case PSCWIN_ERR_CONTRACT: return "contract violation";
    case PSCWIN_ERR_ALIGN: return "pointer not 16-byte aligned";
    case PSCWIN_ERR_WORKSPACE: return "workspace too small";
    case PSCWIN_ERR_CUDA: return "CUDA error";
    case PSCWIN_ERR_UNSUPPORTED: return "unsupported on this path";
    case PSCWIN_ERR_NCCL: return "NCCL error (failed call, asynchronous communicator error or aborted communicator)";
    case PSCWIN_ERR_TIMEOUT: return "timed out waiting for the stream (communicator aborted)";
    default: return "unknown status";
  }
}

int pscwin_last_async_error(void) { return cudaGetLastError() == cudaSuccess ? PSCWIN_OK : PSCWIN_ERR_CUDA; }

int pscwin_window_count(int32_t H, int32_t W, int32_t window, int32_t sx, int32_t sy, int32_t* n) {
  Geo g;
  int rc = geometry(H, W, window, sx, sy, &g);
  if (rc) return rc;
  if (n) *n = g.nw;
  return PSCWIN_OK;
}

int pscwin_index_map(int32_t H, int32_t W, int32_t w, int32_t sx, int32_t sy, uint32_t* map) {
  Geo g;
  int rc = geometry(H, W, w, sx, sy, &g);
  if (rc) return rc;
  if (!map) return PSCWIN_ERR_SHAPE;
  const int nwx = (g.pl + W + g.pr) / w;
  for (int win = 0; win < g.nw; ++win) {
    const int wy = win / nwx, wx = win % nwx;
    for (int iy = 0; iy < w; ++iy)
      for (int ix = 0; ix < w; ++ix) {
        const int y = wy * w + iy - g.pt, x = wx * w + ix - g.pl;
        map[((size_t)win * w + iy) * w + ix] =
            (y >= 0 && y < H && x >= 0 && x < W) ? (uint32_t)(y * W + x) : 0xFFFFFFFFu;
      }
  }
  return PSCWIN_OK;
}

int pscwin_window_partition(const void* x, int32_t B, int32_t H, int32_t W, int32_t Cx, int32_t window,
                            int32_t dtype, void* out, void* stream) {
  return pscwin_shifted_pad_partition(x, nullptr, B, H, W, Cx, window, 0, 0, dtype, out, stream);
}

int pscwin_shifted_pad_partition(const void* x, const void* pad_row, int32_t B, int32_t H, int32_t W, int32_t Cx,
                                 int32_t window, int32_t sx, int32_t sy, int32_t dtype, void* out, void* stream) {
  if (B <= 0 || Cx <= 0) return PSCWIN_ERR_SHAPE;
  if (dtype != PSCWIN_BF16 && dtype != PSCWIN_F32) return PSCWIN_ERR_CONTRACT;
  Geo g;
  int rc = geometry(H, W, window, sx, sy, &g);
  if (rc) return rc;
  const bool has_pad = (long long)g.nw * window * window != (long long)H * W;
  if (has_pad && !pad_row) return PSCWIN_ERR_CONTRACT;
  if (!x || !out) return PSCWIN_ERR_SHAPE;
  if (!aligned16(x) || !aligned16(out) || !aligned16(pad_row)) return PSCWIN_ERR_ALIGN;
  const int esize = dtype == PSCWIN_F32 ? 4 : 2;
  return status_from(launch_partition(x, has_pad ? pad_row : nullptr, B, H, W, Cx, window, sx, sy, esize, out,
                                      (cudaStream_t)stream));
}

int pscwin_window_merge(const void* win, int32_t B, int32_t H, int32_t W, int32_t Cx, int32_t window, int32_t sx,
                        int32_t sy, const void* residual, int32_t dtype, void* out, void* stream) {
  if (B <= 0 || Cx <= 0) return PSCWIN_ERR_SHAPE;
  if (dtype != PSCWIN_BF16 && dtype != PSCWIN_F32) return PSCWIN_ERR_CONTRACT;
  Geo g;
  int rc = geometry(H, W, window, sx, sy, &g);
  if (rc) return rc;
  if (!win || !out) return PSCWIN_ERR_SHAPE;
  if (!aligned16(win) || !aligned16(out) || !aligned16(residual)) return PSCWIN_ERR_ALIGN;
  return status_from(launch_merge(win, B, H, W, Cx, window, sx, sy, residual, dtype == PSCWIN_F32, out,
                                  (cudaStream_t)stream));
}

int pscwin_layer_norm(const void* x, int64_t rows, int32_t C, const float* g, const float* b, float eps,
                      int32_t dtype, void* out, void* stream) {
  if (rows < 0 || C <= 0 || !x || !out || !g || !b) return PSCWIN_ERR_SHAPE;
  if (!aligned16(x) || !aligned16(out)) return PSCWIN_ERR_ALIGN;
  int rc = launch_layer_norm(x, rows, C, g, b, eps, dtype == PSCWIN_F32, out, (cudaStream_t)stream);
  return rc == -1 ? PSCWIN_ERR_UNSUPPORTED : status_from(rc);
}

int pscwin_linear(const void* A, int64_t M, int32_t K, const void* Wt, int32_t N, const float* bias,
                  const void* residual, int32_t out_f32, void* out, void* stream) {
  if (M < 0 || K <= 0 || N <= 0 || !A || !Wt || !out) return PSCWIN_ERR_SHAPE;
  if (K % 8) return PSCWIN_ERR_UNSUPPORTED;
  if (!aligned16(A) || !aligned16(Wt) || !aligned16(out) || !aligned16(residual)) return PSCWIN_ERR_ALIGN;
  if (out_f32 && residual) return PSCWIN_ERR_CONTRACT;
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.M = (int)M;
  a.N = N;
  a.K = K;
  a.lda = K;
  a.ldb = K;
  a.out = out;
  a.ldo = N;
  a.epi = out_f32 ? EPI_STORE_F32 : (residual ? EPI_RESID_BF16 : EPI_STORE_BF16);
  a.bias = bias;
  a.residual = residual;
  a.ldr = N;
  return status_from(launch_gemm_bf16(A, Wt, a, (cudaStream_t)stream));
}

size_t pscwin_workspace_bytes(const pscwin_layer_desc* d) {
  if (check_layer(d) != PSCWIN_OK) return 0;
  if (d->dtype == PSCWIN_F32) return layer_f32_ws_bytes(d);
  return plan_layer(d).total;
}

int pscwin_qkv_project(const pscwin_layer_desc* d, const pscwin_layer_weights* wt, const void* x, void* qkv,
                       float* qkv_pad, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_layer(d);
  if (rc) return rc;
  if (!wt || !x || !qkv || !wt->w_qkv || !wt->ln1_g || !wt->ln1_b || !wt->b_qkv) return PSCWIN_ERR_SHAPE;
  if (d->dtype == PSCWIN_F32) {
    if (!ws || ws_bytes < layer_f32_ws_bytes(d)) return PSCWIN_ERR_WORKSPACE;
    if (!aligned16(x) || !aligned16(qkv) || !aligned16(ws)) return PSCWIN_ERR_ALIGN;
    float* u = reinterpret_cast<float*>(wsp(ws, plan_layer_f32(d).u));
    return qkv_project_f32(d, wt, (const float*)x, (float*)qkv, qkv_pad, u, (cudaStream_t)stream);
  }
  LayerWs L = plan_layer(d);
  if (!ws || ws_bytes < L.total) return PSCWIN_ERR_WORKSPACE;
  if (!aligned16(x) || !aligned16(qkv) || !aligned16(ws)) return PSCWIN_ERR_ALIGN;
  return status_from(qkv_project_impl(d, wt, x, qkv, qkv_pad, ws, L, (cudaStream_t)stream));
}

int pscwin_window_attention(const pscwin_layer_desc* d, const void* qkv, const float* qkv_pad, void* O, void* ws,
                            size_t ws_bytes, void* stream) {
  int rc = check_layer(d);
  if (rc) return rc;
  if (!qkv || !O) return PSCWIN_ERR_SHAPE;
  const bool shifted = d->shift_x || d->shift_y;
  if (shifted && d->pad_mode == PSCWIN_PAD_LEARNABLE && !qkv_pad) return PSCWIN_ERR_CONTRACT;
  if (d->dtype == PSCWIN_F32) {
    if (!aligned16(qkv) || !aligned16(O)) return PSCWIN_ERR_ALIGN;
    return launch_attention_f32(d, (const float*)qkv, qkv_pad, (float*)O, (cudaStream_t)stream);
  }
  LayerWs L = plan_layer(d);
  if (!ws || ws_bytes < L.total) return PSCWIN_ERR_WORKSPACE;
  if (!aligned16(qkv) || !aligned16(O) || !aligned16(ws)) return PSCWIN_ERR_ALIGN;
  return status_from(attention_impl(d, qkv, qkv_pad, O, ws, L, (cudaStream_t)stream));
}

int pscwin_forward(const pscwin_layer_desc* d, const pscwin_layer_weights* wt, const void* x_in, void* x_out,
                   void* ws, size_t ws_bytes, void* stream) {
  int rc = check_layer(d);
  if (rc) return rc;
  if (!wt || !x_in || !x_out) return PSCWIN_ERR_SHAPE;
  const bool shifted = d->shift_x || d->shift_y;
  if (shifted && d->pad_mode == PSCWIN_PAD_LEARNABLE && !wt->pad) return PSCWIN_ERR_CONTRACT;
  if (!wt->w_qkv || !wt->w_o || !wt->ln1_g || !wt->ln1_b || !wt->b_qkv || !wt->b_o) return PSCWIN_ERR_SHAPE;
  if (d->mlp_hidden > 0 && !ffn_weights_ok(wt)) return PSCWIN_ERR_SHAPE;
  if (d->dtype == PSCWIN_F32) {
    if (!aligned16(x_in) || !aligned16(x_out) || !aligned16(ws)) return PSCWIN_ERR_ALIGN;
    return forward_f32(d, wt, x_in, x_out, ws, ws_bytes, (cudaStream_t)stream);
  }
  LayerWs L = plan_layer(d);
  if (!ws || ws_bytes < L.total) return PSCWIN_ERR_WORKSPACE;
  if (!aligned16(x_in) || !aligned16(x_out) || !aligned16(ws)) return PSCWIN_ERR_ALIGN;
  cudaStream_t s = (cudaStream_t)stream;
  const long long T = (long long)d->B * d->H * d->W;
  const int C = d->C;
  void* qkv = wsp(ws, L.qkv);
  float* qkv_pad = reinterpret_cast<float*>(wsp(ws, L.qkv_pad));
  void* O = wsp(ws, L.O);
  const bool learn_pad = shifted && d->pad_mode == PSCWIN_PAD_LEARNABLE;
  const int fold_mode = ln_fold_mode(T);
  const bool fold = fold_mode != 0;                      // LN1 -> QKV
  const bool fold_fc1 = fold_mode == 1;                  // LN2 -> fc1
  const bool fold_in = fold_mode == 1 && d->cycle_scan;  // LN_s -> in_proj
  const int D2 = 2 * d->ssm_expand * C;
  // Weight-only work on the side stream, forked at the start of the layer: the LayerNorm folds of the projections
  // (cycle-scan in_proj, QKV, fc1) and the learnable pad token's projection + rotated tables. Each consumer waits
  // on its own event, so the fold of a projection overlaps everything before it.
  AuxStream* sd = (learn_pad || fold) ? side() : nullptr;
  const bool fork = sd != nullptr;
  cudaStream_t aux = fork ? sd->s : s;
  LnFold f_in = fold_at(ws, L.f_in, D2, C, L.stats), f_qkv = fold_at(ws, L.f_qkv, 3 * C, C, L.stats);
  LnFold f_fc1 = fold_at(ws, L.f_fc1, d->mlp_hidden, C, L.stats);
  if (fork && (cudaEventRecord(sd->fork, s) != cudaSuccess || cudaStreamWaitEvent(sd->s, sd->fork, 0) != cudaSuccess))
    return PSCWIN_ERR_CUDA;
  if (fold_in) {
    if ((rc = fold_launch(f_in, wt->w_in, D2, C, wt->lns_g, wt->lns_b, nullptr, aux))) return status_from(rc);
    if (fork && cudaEventRecord(f_in.ready = sd->ev[0], aux) != cudaSuccess) return PSCWIN_ERR_CUDA;
  }
  if (fold) {
    if ((rc = fold_launch(f_qkv, wt->w_qkv, 3 * C, C, wt->ln1_g, wt->ln1_b, wt->b_qkv, aux))) return status_from(rc);
    if (fork && cudaEventRecord(f_qkv.ready = sd->ev[1], aux) != cudaSuccess) return PSCWIN_ERR_CUDA;
  }
  if (learn_pad && fork) {  // the pad work overlaps everything up to the attention kernel
    rc = launch_pad_qkv(wt->pad, wt->w_qkv, (const float*)wt->b_qkv, C, 0, qkv_pad, aux);
    if (rc) return status_from(rc);
    AttnArgs pa = attn_args(d, qkv, qkv_pad, O, wsp(ws, L.pad_tab));
    if ((rc = launch_pad_tables(pa, aux))) return status_from(rc);
    if (cudaEventRecord(sd->join, aux) != cudaSuccess) return PSCWIN_ERR_CUDA;
  }
  if (fold_fc1 && d->mlp_hidden > 0) {
    if ((rc = fold_launch(f_fc1, wt->w_fc1, d->mlp_hidden, C, wt->ln2_g, wt->ln2_b, wt->b_fc1, aux)))
      return status_from(rc);
    if (fork && cudaEventRecord(f_fc1.ready = sd->ev[2], aux) != cudaSuccess) return PSCWIN_ERR_CUDA;
  }
  const void* x = x_in;
  if (d->cycle_scan) {
    rc = cycle_scan_module(d, wt, fold_in ? &f_in : nullptr, x_in, x_out, ws, L.u, L.xz, L.g, L.scan,
                           L.total - L.scan, s);
    if (rc) return rc;
    x = x_out;
  }
  rc = qkv_project_impl(d, wt, x, qkv, (learn_pad && !fork) ? qkv_pad : nullptr, ws, L, s, fold ? &f_qkv : nullptr);
  if (rc) return status_from(rc);
  if (learn_pad && fork && cudaStreamWaitEvent(s, sd->join, 0) != cudaSuccess) return PSCWIN_ERR_CUDA;
  rc = attention_impl(d, qkv, qkv_pad, O, ws, L, s, (learn_pad && fork) ? 1 : 0);
  if (rc) return status_from(rc);
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.M = (int)T;
  a.N = C;
  a.K = C;
  a.lda = C;
  a.ldb = C;
  a.out = x_out;
  a.ldo = C;
  a.epi = EPI_RESID_BF16;
  a.prof_name = "gemm_out_proj";
  a.bias = (const float*)wt->b_o;
  a.residual = x;
  a.ldr = C;
  rc = launch_gemm_bf16(O, wt->w_o, a, s);
  if (rc) return status_from(rc);
  if (d->mlp_hidden > 0)
    return ffn_bf16(T, C, d->mlp_hidden, d->ln_eps, wt, x_out, wsp(ws, L.u), wsp(ws, L.h), s, fold_fc1 ? &f_fc1 : nullptr);
  return PSCWIN_OK;
}

// ---------------------------------------------------------------------------- HRSAM++ multi-scale layer
namespace {
int ms_geo(const pscwin_ms_desc* m, MsGeo* g) {
  if (!m || m->n_scales < 1 || m->n_scales > PSCWIN_MAX_SCALES) return PSCWIN_ERR_SHAPE;
  g->n = m->n_scales;
  g->off[0] = 0;
  for (int i = 0; i < 4; ++i) {
    g->H[i] = i < m->n_scales ? m->H[i] : 1;
    g->W[i] = i < m->n_scales ? m->W[i] : 1;
  }
  for (int i = 0; i < m->n_scales; ++i) {
    if (m->H[i] <= 0 || m->W[i] <= 0) return PSCWIN_ERR_SHAPE;
    const long long nx = (long long)g->off[i] + (long long)m->H[i] * m->W[i];
    if (nx > (1ll << 30)) return PSCWIN_ERR_SHAPE;
    g->off[i + 1] = (int)nx;
  }
  for (int i = m->n_scales + 1; i < 5; ++i) g->off[i] = g->off[m->n_scales];
  return PSCWIN_OK;
}

pscwin_layer_desc scale_desc(const pscwin_ms_desc* m, int i) {
  pscwin_layer_desc d = m->layer;
  d.H = m->H[i];
  d.W = m->W[i];
  d.cycle_scan = 0;
  return d;
}

int check_ms(const pscwin_ms_desc* m, MsGeo* g) {
  int rc = ms_geo(m, g);
  if (rc) return rc;
  if (m->layer.dtype != PSCWIN_BF16) return PSCWIN_ERR_UNSUPPORTED;
  if (m->cycle_scan < PSCWIN_CS_NONE || m->cycle_scan > PSCWIN_CS_MULTI_SCALE) return PSCWIN_ERR_CONTRACT;
  if (!m->attention && !m->cycle_scan) return PSCWIN_ERR_CONTRACT;
  for (int i = 0; i < m->n_scales; ++i) {
    pscwin_layer_desc d = scale_desc(m, i);
    if (!m->attention) d.shift_x = d.shift_y = 0, d.H = d.W = d.window;  // only the shared fields matter
    rc = check_layer(&d);
    if (rc) return rc;
  }
  return PSCWIN_OK;
}

struct MsWs {
  size_t u, qkv, qkv_pad, O, pad_tab, h, xz, g, scan, total;
  size_t stats, fold;  // folded LN1 -> QKV: row statistics [T] float2, W' | s | c
};

MsWs plan_ms(const pscwin_ms_desc* m, const MsGeo& g) {
  MsWs w;
  const pscwin_layer_desc& d = m->layer;
  const size_t T = (size_t)d.B * g.off[g.n], C = d.C;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return o;
  };
  w.u = take(T * C * 2);
  w.qkv = w.qkv_pad = w.O = w.pad_tab = w.h = w.xz = w.g = w.scan = w.stats = w.fold = 0;
  if (m->attention) {
    w.stats = take(T * sizeof(float2));
    w.fold = take(fold_bytes(3 * C, C));
    w.qkv = take(T * 3 * C * 2);
    w.qkv_pad = take(3 * C * 4);
    w.O = take(T * C * 2);
    size_t pt = 0;
    for (int i = 0; i < g.n; ++i) {
      const size_t b = attn_pad_table_bytes(g.H[i], g.W[i], d.C, d.window);
      pt = b > pt ? b : pt;
    }
    w.pad_tab = take(pt);
    if (d.mlp_hidden > 0) w.h = take(T * d.mlp_hidden * 2);
  }
  if (m->cycle_scan) {
    const size_t D = (size_t)d.ssm_expand * C;
    w.xz = take(T * 2 * D * 2);
    w.g = take(T * D * 2);
    const int R = d.ssm_dt_rank > 0 ? d.ssm_dt_rank : (d.C + 15) / 16;
    w.scan = take(ms_scan_ws_bytes(d.B, g, m->cycle_scan, (int)D, d.ssm_state, R, d.ssm_conv, d.scan_order));
  }
  w.total = off;
  return w;
}
}  // namespace

int pscwin_ms_window_count(const pscwin_ms_desc* m, int32_t* n) {
  MsGeo g;
  int rc = ms_geo(m, &g);
  if (rc) return rc;
  int tot = 0;
  for (int i = 0; i < m->n_scales; ++i) {
    Geo q;
    rc = geometry(m->H[i], m->W[i], m->layer.window, m->layer.shift_x, m->layer.shift_y, &q);
    if (rc) return rc;
    tot += q.nw;
  }
  if (n) *n = tot;
  return PSCWIN_OK;
}

int pscwin_ms_index_map(const pscwin_ms_desc* m, uint32_t* map) {
  MsGeo g;
  int rc = ms_geo(m, &g);
  if (rc) return rc;
  if (!map) return PSCWIN_ERR_SHAPE;
  const int w = m->layer.window;
  for (int i = 0; i < m->n_scales; ++i) {
    Geo q;
    rc = pscwin_index_map(m->H[i], m->W[i], w, m->layer.shift_x, m->layer.shift_y, map);
    if (rc) return rc;
    geometry(m->H[i], m->W[i], w, m->layer.shift_x, m->layer.shift_y, &q);
    const size_t n = (size_t)q.nw * w * w;
    for (size_t j = 0; j < n; ++j)
      if (map[j] != 0xFFFFFFFFu) map[j] += (uint32_t)g.off[i];
    map += n;
  }
  return PSCWIN_OK;
}

size_t pscwin_ms_workspace_bytes(const pscwin_ms_desc* m) {
  MsGeo g;
  if (check_ms(m, &g) != PSCWIN_OK) return 0;
  return plan_ms(m, g).total;
}

int pscwin_ms_forward(const pscwin_ms_desc* m, const pscwin_layer_weights* wt, const void* x_in, void* x_out,
                      void* ws, size_t ws_bytes, void* stream) {
  MsGeo g;
  int rc = check_ms(m, &g);
  if (rc) return rc;
  if (!wt || !x_in || !x_out) return PSCWIN_ERR_SHAPE;
  const pscwin_layer_desc& d = m->layer;
  const bool shifted = d.shift_x || d.shift_y;
  const bool learn_pad = m->attention && shifted && d.pad_mode == PSCWIN_PAD_LEARNABLE;
  if (learn_pad && !wt->pad) return PSCWIN_ERR_CONTRACT;
  if (m->attention && (!wt->w_qkv || !wt->w_o || !wt->ln1_g || !wt->ln1_b || !wt->b_qkv || !wt->b_o))
    return PSCWIN_ERR_SHAPE;
  if (m->attention && d.mlp_hidden > 0 && !ffn_weights_ok(wt)) return PSCWIN_ERR_SHAPE;
  MsWs P = plan_ms(m, g);
  if (!ws || ws_bytes < P.total) return PSCWIN_ERR_WORKSPACE;
  if (!aligned16(x_in) || !aligned16(x_out) || !aligned16(ws)) return PSCWIN_ERR_ALIGN;
  cudaStream_t s = (cudaStream_t)stream;
  const long long T = (long long)d.B * g.off[g.n];
  const int C = d.C;
  const void* x = x_in;
  if (m->cycle_scan) {
    rc = ms_cycle_scan_module(&d, wt, g, m->cycle_scan, x_in, x_out, ws, P.u, P.xz, P.g, P.scan, P.total - P.scan, s);
    if (rc) return rc;
    x = x_out;
  }
  if (!m->attention) return PSCWIN_OK;
  // a4 over every packed row: LN1, QKV GEMM with RoPE at each scale's own grid coordinates (segment table)
  void* u = wsp(ws, P.u);
  __nv_bfloat16* qkv = reinterpret_cast<__nv_bfloat16*>(wsp(ws, P.qkv));
  float* qkv_pad = reinterpret_cast<float*>(wsp(ws, P.qkv_pad));
  __nv_bfloat16* O = reinterpret_cast<__nv_bfloat16*>(wsp(ws, P.O));
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.M = (int)T;
  a.N = 3 * C;
  a.K = C;
  a.lda = C;
  a.ldb = C;
  a.out = qkv;
  a.ldo = 3 * C;
  a.epi = EPI_QKV_ROPE;
  a.prof_name = "gemm_qkv_rope";
  a.bias = (const float*)wt->b_qkv;
  a.rope = d.rope;
  a.HW = g.H[0] * g.W[0];
  a.Wgrid = g.W[0];
  a.C = C;
  a.d_head = C / d.heads;
  a.nseg = g.n;
  for (int i = 0; i < g.n; ++i) {
    a.seg_row[i] = d.B * g.off[i];
    a.seg_HW[i] = g.H[i] * g.W[i];
    a.seg_W[i] = g.W[i];
  }
  rc = ln1_qkv(wt, d.ln_eps, x, a, u, wsp(ws, P.fold), reinterpret_cast<float2*>(wsp(ws, P.stats)), T, s);
  if (rc) return status_from(rc);
  if (learn_pad) {
    rc = launch_pad_qkv(wt->pad, wt->w_qkv, (const float*)wt->b_qkv, C, 0, qkv_pad, s);
    if (rc) return status_from(rc);
  }
  // a5 + a6 per scale (windows never span scales: the block-diagonal structure of P:L185)
  LayerWs L;
  memset(&L, 0, sizeof(L));
  L.pad_tab = P.pad_tab;
  for (int i = 0; i < g.n; ++i) {
    pscwin_layer_desc di = scale_desc(m, i);
    const long long r0 = (long long)d.B * g.off[i];
    rc = attention_impl(&di, qkv + r0 * 3 * C, learn_pad ? qkv_pad : nullptr, O + r0 * C, ws, L, s);
    if (rc) return status_from(rc);
  }
  // a7 over every packed row: x_out = x + O W_o^T + b_o
  memset(&a, 0, sizeof(a));
  a.M = (int)T;
  a.N = C;
  a.K = C;
  a.lda = C;
  a.ldb = C;
  a.out = x_out;
  a.ldo = C;
  a.epi = EPI_RESID_BF16;
  a.prof_name = "gemm_out_proj";
  a.bias = (const float*)wt->b_o;
  a.residual = x;
  a.ldr = C;
  rc = launch_gemm_bf16(O, wt->w_o, a, s);
  if (rc) return status_from(rc);
  if (d.mlp_hidden > 0) return ffn_bf16(T, C, d.mlp_hidden, d.ln_eps, wt, x_out, u, wsp(ws, P.h), s);
  return PSCWIN_OK;
}

}  // extern "C"

// =================================================================================================== row bands
// Window-row sharding of one image over `world` ranks. Rank g owns token rows
// [row_begin, row_end) (multiples of the window). Token-local steps run on the band; the shifted windows that
// straddle a band edge need the neighbours' QKV rows (halo: pt rows above, w - pt below, pt = (w - s_y) mod w);
// the cycle scan needs the previous rank's last k-1 xin rows (conv history, a ring) and one all-gather of the
// per-rank segment records. The caller moves those bytes (NCCL) between the
// phase calls; every byte offset is relative to the workspace and reported by pscwin_band_io_offsets.
namespace {
struct BandGeo {
  int r0, r1, rows, ht, hb, ht_eff, hb_eff, e0, ext_rows, sy_local, P;
  bool ok;
};

BandGeo band_geo(const pscwin_layer_desc* d, const pscwin_band* b) {
  BandGeo g;
  g.ok = false;
  const int w = d->window;
  if (!b || b->world < 1 || b->rank < 0 || b->rank >= b->world) return g;
  if (d->B != 1) return g;  // one image per band group
  g.r0 = b->row_begin;
  g.r1 = b->row_end;
  if (g.r0 < 0 || g.r1 > d->H || g.r1 <= g.r0 || g.r0 % w || (g.r1 % w && g.r1 != d->H)) return g;
  if ((b->rank == 0) != (g.r0 == 0) || (b->rank == b->world - 1) != (g.r1 == d->H)) return g;
  g.rows = g.r1 - g.r0;
  const int pt = (w - d->shift_y) % w;
  g.ht = pt;
  g.hb = pt ? w - pt : 0;
  g.ht_eff = b->rank > 0 ? g.ht : 0;
  g.hb_eff = b->rank < b->world - 1 ? g.hb : 0;
  // the band must hold the halo its neighbours read from it: its first hb rows go to rank - 1, its last ht rows
  // to rank + 1 (a shorter ragged band would send rows past its own into the workspace)
  if ((b->rank > 0 && g.rows < g.hb) || (b->rank < b->world - 1 && g.rows < g.ht)) return g;
  g.e0 = g.r0 - g.ht_eff;
  g.ext_rows = g.ht_eff + g.rows + g.hb_eff;
  // the extended buffer's window grid must coincide with the global one: local pad_top = (pt + e0) mod w
  const int pt_local = ((pt + g.e0) % w + w) % w;
  g.sy_local = (w - pt_local) % w;
  g.P = b->rank == 0 ? d->ssm_conv - 1 : 0;
  if (g.rows * d->W < d->ssm_conv - 1) return g;
  g.ok = true;
  return g;
}

pscwin_layer_desc sub_desc(const pscwin_layer_desc* d, int rows, int sy) {
  pscwin_layer_desc s = *d;
  s.H = rows;
  s.shift_y = sy;
  return s;
}

struct BandWs {
  size_t u, qkv, qkv_pad, O, pad_tab, h, xz, g, x1, hist_send, hist_recv, rec_send, rec_recv, scan, total;
  size_t xzp, gs;  // window-major scan order: xz rows gathered into scan order, gated output in scan order
  size_t stats, fold;  // folded LN1 -> QKV: row statistics [T] float2, W' | s | c
  size_t row_bytes_qkv;
  int D, N, R;
};

BandWs plan_band(const pscwin_layer_desc* d, const pscwin_band* b, const BandGeo& g) {
  BandWs w;
  memset(&w, 0, sizeof(w));
  const size_t Wd = d->W, C = d->C;
  const size_t T = (size_t)g.rows * Wd, Te = (size_t)g.ext_rows * Wd;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align256(bytes);
    return o;
  };
  w.row_bytes_qkv = Wd * 3 * C * 2;
  w.u = take(T * C * 2);
  w.stats = take(T * sizeof(float2));
  w.fold = take(fold_bytes(3 * C, C));
  w.qkv = take(Te * 3 * C * 2);
  w.qkv_pad = take(3 * C * 4);
  w.O = take(Te * C * 2);
  w.pad_tab = take(attn_pad_table_bytes(g.ext_rows, d->W, d->C, d->window));
  if (d->mlp_hidden > 0) w.h = take(T * d->mlp_hidden * 2);
  if (d->cycle_scan) {
    w.D = d->ssm_expand * d->C;
    w.N = d->ssm_state;
    w.R = d->ssm_dt_rank > 0 ? d->ssm_dt_rank : (d->C + 15) / 16;
    const int k = d->ssm_conv;
    w.xz = take(T * 2 * w.D * 2);
    if (d->scan_order == PSCWIN_SCAN_WINDOW_MAJOR) {
      w.xzp = take(T * 2 * w.D * 2);
      w.gs = take(T * w.D * 2);
    }
    w.g = take(T * w.D * 2);
    w.x1 = take(T * C * 2);
    w.hist_send = take((size_t)(k - 1) * w.D * 2);
    w.hist_recv = take((size_t)(k - 1) * w.D * 2);
    w.rec_send = take(band_scan_record_bytes(w.D, w.N));
    w.rec_recv = take((size_t)b->world * band_scan_record_bytes(w.D, w.N));
    w.scan = take(band_scan_ws_bytes((int)T, w.D, w.N, w.R, k, g.P));
  }
  w.total = off;
  return w;
}

int band_check(const pscwin_layer_desc* d, const pscwin_band* b, BandGeo* g) {
  int rc = check_layer(d);
  if (rc) return rc;
  if (d->dtype != PSCWIN_BF16) return PSCWIN_ERR_UNSUPPORTED;  // bands run the bf16 product path
  // a band's scan segment must be contiguous: row-major raster always; window-major when the band is whole window
  // rows of a window-divisible grid (its windows are then a contiguous run of the window-major sequence, scanned
  // in band-local window-major order); column-major never
  if (d->cycle_scan && d->scan_order == PSCWIN_SCAN_COL_MAJOR) return PSCWIN_ERR_CONTRACT;
  *g = band_geo(d, b);
  if (!g->ok) return PSCWIN_ERR_CONTRACT;
  if (d->cycle_scan && d->scan_order == PSCWIN_SCAN_WINDOW_MAJOR &&
      (d->H % d->window || d->W % d->window || g->r0 % d->window || g->r1 % d->window))
    return PSCWIN_ERR_CONTRACT;
  return PSCWIN_OK;
}
}  // namespace

extern "C" {

size_t pscwin_band_workspace_bytes(const pscwin_layer_desc* d, const pscwin_band* b) {
  BandGeo g;
  if (band_check(d, b, &g)) return 0;
  return plan_band(d, b, g).total;
}

int pscwin_band_io_offsets(const pscwin_layer_desc* d, const pscwin_band* b, pscwin_band_io* io) {
  BandGeo g;
  int rc = band_check(d, b, &g);
  if (rc) return rc;
  if (!io) return PSCWIN_ERR_SHAPE;
  const BandWs w = plan_band(d, b, g);
  memset(io, 0, sizeof(*io));
  if (d->cycle_scan) {
    io->hist_send = w.hist_send;
    io->hist_recv = w.hist_recv;
    io->hist_bytes = (uint64_t)(d->ssm_conv - 1) * w.D * 2;
    io->rec_send = w.rec_send;
    io->rec_recv = w.rec_recv;
    io->rec_bytes = band_scan_record_bytes(w.D, w.N);
  }
  const uint64_t rb = w.row_bytes_qkv;
  io->send_prev = w.qkv + (uint64_t)g.ht_eff * rb;                          // own first hb rows
  io->send_prev_bytes = b->rank > 0 ? (uint64_t)g.hb * rb : 0;
  io->send_next = w.qkv + (uint64_t)(g.ht_eff + g.rows - g.ht) * rb;        // own last ht rows
  io->send_next_bytes = b->rank < b->world - 1 ? (uint64_t)g.ht * rb : 0;
  io->recv_prev = w.qkv;                                                     // top halo
  io->recv_prev_bytes = (uint64_t)g.ht_eff * rb;
  io->recv_next = w.qkv + (uint64_t)(g.ht_eff + g.rows) * rb;               // bottom halo
  io->recv_next_bytes = (uint64_t)g.hb_eff * rb;
  return PSCWIN_OK;
}

int pscwin_band_scan_begin(const pscwin_layer_desc* d, const pscwin_band* b, const pscwin_layer_weights* wt,
                           const void* x_band, void* ws, size_t ws_bytes, void* stream) {
  BandGeo g;
  int rc = band_check(d, b, &g);
  if (rc) return rc;
  if (!d->cycle_scan || !wt || !x_band || !wt->lns_g || !wt->lns_b || !wt->w_in) return PSCWIN_ERR_SHAPE;
  const BandWs w = plan_band(d, b, g);
  if (!ws || ws_bytes < w.total) return PSCWIN_ERR_WORKSPACE;
  if (!aligned16(x_band) || !aligned16(ws)) return PSCWIN_ERR_ALIGN;
  cudaStream_t s = (cudaStream_t)stream;
  const long long T = (long long)g.rows * d->W;
  const int C = d->C, D = w.D, k = d->ssm_conv;
  void* u = wsp(ws, w.u);
  __nv_bfloat16* xz = reinterpret_cast<__nv_bfloat16*>(wsp(ws, w.xz));
  rc = launch_layer_norm(x_band, T, C, (const float*)wt->lns_g, (const float*)wt->lns_b, d->ln_eps, 0, u, s);
  if (rc) return PSCWIN_ERR_CUDA;
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.prof_name = "gemm_in_proj";
  a.M = (int)T;
  a.N = 2 * D;
  a.K = C;
  a.lda = C;
  a.ldb = C;
  a.out = xz;
  a.ldo = 2 * D;
  a.epi = EPI_STORE_BF16;
  a.silu_col = D;
  if (launch_gemm_bf16(u, wt->w_in, a, s)) return PSCWIN_ERR_CUDA;
  if (d->scan_order == PSCWIN_SCAN_WINDOW_MAJOR) {  // [xin | SiLU(z)] rows into band-local window-major order
    __nv_bfloat16* xzp = reinterpret_cast<__nv_bfloat16*>(wsp(ws, w.xzp));
    if (launch_permute_rows(xz, 2 * D, xzp, 2 * D, 1, g.rows, d->W, 2 * D, d->scan_order, d->window, 0, s))
      return PSCWIN_ERR_CUDA;
    xz = xzp;
  }
  // conv history for the next rank: this band's last k-1 xin rows (in scan order)
  if (k > 1 && cudaMemcpy2DAsync(wsp(ws, w.hist_send), (size_t)D * 2, xz + (T - (k - 1)) * 2 * D, (size_t)2 * D * 2,
                                 (size_t)D * 2, k - 1, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return PSCWIN_ERR_CUDA;
  return PSCWIN_OK;
}

int pscwin_band_scan_mid(const pscwin_layer_desc* d, const pscwin_band* b, const pscwin_layer_weights* wt, void* ws,
                         size_t ws_bytes, void* stream) {
  BandGeo g;
  int rc = band_check(d, b, &g);
  if (rc) return rc;
  if (!d->cycle_scan || !wt || !wt->conv_w || !wt->conv_b || !wt->w_x || !wt->w_dt || !wt->b_dt || !wt->a_log)
    return PSCWIN_ERR_SHAPE;
  const BandWs w = plan_band(d, b, g);
  if (!ws || ws_bytes < w.total) return PSCWIN_ERR_WORKSPACE;
  const long long T = (long long)g.rows * d->W;
  const __nv_bfloat16* xz =
      reinterpret_cast<const __nv_bfloat16*>(wsp(ws, d->scan_order == PSCWIN_SCAN_WINDOW_MAJOR ? w.xzp : w.xz));
  return band_scan_mid((int)T, w.D, w.N, w.R, d->ssm_conv, g.P, d->bbar_mode, xz, 2 * w.D,
                       reinterpret_cast<const __nv_bfloat16*>(wsp(ws, w.hist_recv)), (const float*)wt->conv_w,
                       (const float*)wt->conv_b, wt->w_x, (const float*)wt->w_dt, (const float*)wt->b_dt, wt->a_log,
                       wt->d_skip, reinterpret_cast<float*>(wsp(ws, w.rec_send)), wsp(ws, w.scan), w.total - w.scan,
                       (cudaStream_t)stream);
}

int pscwin_band_scan_end(const pscwin_layer_desc* d, const pscwin_band* b, const pscwin_layer_weights* wt,
                         const void* x_band, void* ws, size_t ws_bytes, void* stream) {
  BandGeo g;
  int rc = band_check(d, b, &g);
  if (rc) return rc;
  if (!d->cycle_scan || !wt || !x_band || !wt->d_skip || !wt->w_out) return PSCWIN_ERR_SHAPE;
  const BandWs w = plan_band(d, b, g);
  if (!ws || ws_bytes < w.total) return PSCWIN_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  const long long T = (long long)g.rows * d->W;
  const int C = d->C, D = w.D;
  const bool wm = d->scan_order == PSCWIN_SCAN_WINDOW_MAJOR;
  const __nv_bfloat16* xz = reinterpret_cast<const __nv_bfloat16*>(wsp(ws, wm ? w.xzp : w.xz));
  __nv_bfloat16* gb = reinterpret_cast<__nv_bfloat16*>(wsp(ws, wm ? w.gs : w.g));
  rc = band_scan_end((int)T, D, w.N, w.R, d->ssm_conv, g.P, d->bbar_mode, xz, 2 * D, xz + D, 2 * D,
                     (const float*)wt->conv_w, (const float*)wt->conv_b, (const float*)wt->w_dt,
                     (const float*)wt->b_dt, wt->a_log, wt->d_skip, reinterpret_cast<const float*>(wsp(ws, w.rec_recv)),
                     b->rank, b->world, gb, D, wsp(ws, w.scan), w.total - w.scan, s);
  if (rc) return rc;
  if (wm) {  // gated output rows back to grid order for the out-projection's residual
    __nv_bfloat16* g_grid = reinterpret_cast<__nv_bfloat16*>(wsp(ws, w.g));
    if (launch_permute_rows(gb, D, g_grid, D, 1, g.rows, d->W, D, d->scan_order, d->window, 1, s)) return PSCWIN_ERR_CUDA;
    gb = g_grid;
  }
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.prof_name = "gemm_out_proj_scan";
  a.M = (int)T;
  a.N = C;
  a.K = D;
  a.lda = D;
  a.ldb = D;
  a.out = wsp(ws, w.x1);
  a.ldo = C;
  a.epi = EPI_RESID_BF16;
  a.residual = x_band;
  a.ldr = C;
  return launch_gemm_bf16(gb, wt->w_out, a, s) ? PSCWIN_ERR_CUDA : PSCWIN_OK;
}

int pscwin_band_attn_begin(const pscwin_layer_desc* d, const pscwin_band* b, const pscwin_layer_weights* wt,
                           const void* x_band, void* ws, size_t ws_bytes, void* stream) {
  BandGeo g;
  int rc = band_check(d, b, &g);
  if (rc) return rc;
  if (!wt || !x_band || !wt->w_qkv || !wt->ln1_g || !wt->ln1_b || !wt->b_qkv) return PSCWIN_ERR_SHAPE;
  const bool shifted = d->shift_x || d->shift_y;
  if (shifted && d->pad_mode == PSCWIN_PAD_LEARNABLE && !wt->pad) return PSCWIN_ERR_CONTRACT;
  const BandWs w = plan_band(d, b, g);
  if (!ws || ws_bytes < w.total) return PSCWIN_ERR_WORKSPACE;
  if (!aligned16(x_band) || !aligned16(ws)) return PSCWIN_ERR_ALIGN;
  cudaStream_t s = (cudaStream_t)stream;
  const long long T = (long long)g.rows * d->W;
  const int C = d->C;
  const void* x = d->cycle_scan ? wsp(ws, w.x1) : x_band;
  void* u = wsp(ws, w.u);
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.M = (int)T;
  a.N = 3 * C;
  a.K = C;
  a.lda = C;
  a.ldb = C;
  a.out = wsp(ws, w.qkv + (size_t)g.ht_eff * w.row_bytes_qkv);  // own rows of the extended buffer
  a.ldo = 3 * C;
  a.epi = EPI_QKV_ROPE;
  a.prof_name = "gemm_qkv_rope";
  a.bias = (const float*)wt->b_qkv;
  a.rope = d->rope;
  a.HW = d->H * d->W;
  a.Wgrid = d->W;
  a.C = C;
  a.d_head = C / d->heads;
  a.tok0 = g.r0 * d->W;  // RoPE at global grid rows
  if (ln1_qkv(wt, d->ln_eps, x, a, u, wsp(ws, w.fold), reinterpret_cast<float2*>(wsp(ws, w.stats)),
              (long long)d->B * d->H * d->W, s))
    return PSCWIN_ERR_CUDA;
  if (shifted && d->pad_mode == PSCWIN_PAD_LEARNABLE) {
    rc = launch_pad_qkv(wt->pad, wt->w_qkv, (const float*)wt->b_qkv, C, 0, reinterpret_cast<float*>(wsp(ws, w.qkv_pad)),
                        s);
    if (rc) return PSCWIN_ERR_CUDA;
  }
  return PSCWIN_OK;
}

}  // extern "C"

namespace pscwin {

// Window attention of a band over the extended QKV buffer, padded-grid window rows [wy0, wy1) of the extended
// image (wy1 <= 0: all), and the band's out-proj + residual (+ FFN). pscwin_band_attn_end runs both; the NCCL path
// splits the attention into interior and halo window rows to overlap the halo exchange (distnccl.cu).
int band_attention(const pscwin_layer_desc* d, const pscwin_band* b, const pscwin_layer_weights* wt, void* ws,
                   size_t ws_bytes, int wy0, int wy1, int tables_ready, void* stream) {
  BandGeo g;
  int rc = band_check(d, b, &g);
  if (rc) return rc;
  if (!wt) return PSCWIN_ERR_SHAPE;
  const BandWs w = plan_band(d, b, g);
  if (!ws || ws_bytes < w.total) return PSCWIN_ERR_WORKSPACE;
  // the extended buffer is an image of ext_rows rows whose window grid matches the global one (band_geo)
  const pscwin_layer_desc e = sub_desc(d, g.ext_rows, g.sy_local);
  AttnArgs a;
  memset(&a, 0, sizeof(a));
  a.B = 1;
  a.H = g.ext_rows;
  a.W = d->W;
  a.C = d->C;
  a.heads = d->heads;
  a.d = d->C / d->heads;
  a.w = d->window;
  a.sx = e.shift_x;
  a.sy = e.shift_y;
  a.pad_mode = d->pad_mode;
  a.rope = d->rope;
  a.row0 = g.e0;
  a.qkv = wsp(ws, w.qkv);
  a.qkv_pad = reinterpret_cast<const float*>(wsp(ws, w.qkv_pad));
  a.out = wsp(ws, w.O);
  a.pad_tab = wsp(ws, w.pad_tab);
  a.tables_ready = tables_ready;
  a.wy_begin = wy0;
  a.wy_end = wy1;
  return status_from(launch_window_attention(a, (cudaStream_t)stream));
}

// Window-row ranges of the extended band image: [0, top) and [bot, nwy) hold the windows that read halo rows,
// [top, bot) the interior ones (computable before the halo arrives).
void band_window_rows(const pscwin_layer_desc* d, const pscwin_band* b, int* top, int* bot, int* nwy) {
  BandGeo g;
  *top = *bot = *nwy = 0;
  if (band_check(d, b, &g)) return;
  const int w = d->window;
  const int pt = (w - g.sy_local) % w;
  const int Hp = pt + g.ext_rows + ((-(pt + g.ext_rows)) % w + w) % w;
  *nwy = Hp / w;
  // window row j covers local token rows [j w - pt, (j + 1) w - pt); own rows are [ht_eff, ht_eff + rows)
  int t = 0, bo = *nwy;
  while (t < *nwy && g.ht_eff > 0 && t * w - pt < g.ht_eff) ++t;
  while (bo > t && g.hb_eff > 0 && bo * w - pt > g.ht_eff + g.rows) --bo;
  *top = t;
  *bot = bo;
}

int band_out_proj(const pscwin_layer_desc* d, const pscwin_band* b, const pscwin_layer_weights* wt,
                  const void* x_band, void* x_out, void* ws, size_t ws_bytes, void* stream) {
  BandGeo g;
  int rc = band_check(d, b, &g);
  if (rc) return rc;
  if (!wt || !x_band || !x_out || !wt->w_o || !wt->b_o) return PSCWIN_ERR_SHAPE;
  const BandWs w = plan_band(d, b, g);
  if (!ws || ws_bytes < w.total) return PSCWIN_ERR_WORKSPACE;
  if (!aligned16(x_out)) return PSCWIN_ERR_ALIGN;
  cudaStream_t s = (cudaStream_t)stream;
  const long long T = (long long)g.rows * d->W;
  const int C = d->C;
  const void* x = d->cycle_scan ? wsp(ws, w.x1) : x_band;
  GemmArgs o;
  memset(&o, 0, sizeof(o));
  o.M = (int)T;
  o.N = C;
  o.K = C;
  o.lda = C;
  o.ldb = C;
  o.out = x_out;
  o.ldo = C;
  o.epi = EPI_RESID_BF16;
  o.prof_name = "gemm_out_proj";
  o.bias = (const float*)wt->b_o;
  o.residual = x;
  o.ldr = C;
  const void* Ob = wsp(ws, w.O + (size_t)g.ht_eff * d->W * C * 2);
  rc = launch_gemm_bf16(Ob, wt->w_o, o, s);
  if (rc) return status_from(rc);
  if (d->mlp_hidden > 0) {  // the FFN is token-local: it runs on the band's own rows
    if (!ffn_weights_ok(wt)) return PSCWIN_ERR_SHAPE;
    return ffn_bf16(T, C, d->mlp_hidden, d->ln_eps, wt, x_out, wsp(ws, w.u), wsp(ws, w.h), s);
  }
  return PSCWIN_OK;
}

}  // namespace pscwin

extern "C" {

int pscwin_band_window_split(const pscwin_layer_desc* d, const pscwin_band* b, int32_t* top, int32_t* bot,
                             int32_t* nwy) {
  BandGeo g;
  int rc = band_check(d, b, &g);
  if (rc) return rc;
  if (!top || !bot || !nwy) return PSCWIN_ERR_SHAPE;
  int t, bo, n;
  pscwin::band_window_rows(d, b, &t, &bo, &n);
  *top = t;
  *bot = bo;
  *nwy = n;
  return PSCWIN_OK;
}

int pscwin_band_attn_windows(const pscwin_layer_desc* d, const pscwin_band* b, const pscwin_layer_weights* wt,
                             void* ws, size_t ws_bytes, int32_t wy_begin, int32_t wy_end, void* stream) {
  if (wy_begin < 0 || wy_end < wy_begin) return PSCWIN_ERR_SHAPE;
  if (wy_end == wy_begin) return PSCWIN_OK;
  return pscwin::band_attention(d, b, wt, ws, ws_bytes, wy_begin, wy_end, 0, stream);
}

int pscwin_band_out_proj(const pscwin_layer_desc* d, const pscwin_band* b, const pscwin_layer_weights* wt,
                         const void* x_band, void* x_out, void* ws, size_t ws_bytes, void* stream) {
  return pscwin::band_out_proj(d, b, wt, x_band, x_out, ws, ws_bytes, stream);
}

int pscwin_band_attn_end(const pscwin_layer_desc* d, const pscwin_band* b, const pscwin_layer_weights* wt,
                         const void* x_band, void* x_out, void* ws, size_t ws_bytes, void* stream) {
  if (!wt || !x_band || !x_out || !wt->w_o || !wt->b_o) return PSCWIN_ERR_SHAPE;
  int rc = band_attention(d, b, wt, ws, ws_bytes, 0, 0, 0, stream);
  if (rc) return rc;
  return band_out_proj(d, b, wt, x_band, x_out, ws, ws_bytes, stream);
}

}  // extern "C"
