// Encoder ends (PAPER.md P:L76 / L89 "fusing outputs from all four stages through summation,
// followed by a convolutional block", "the output dimension of each stage is 256"; reading Q22):
//   patch embedding  = patchify gather + tcgen05 GEMM (K = 3 * 16 * 16 = 768, bias in the epilogue)
//   neck             = per-stage 1x1 projections chained as GEMMs with an in-place residual (the sum over stages),
//                      [HRSAM++: the overview scale's sum bilinearly resized and added], LN2d, conv3x3 as
//                      im2col + GEMM (K = 9 * C_out), LN2d
// All data movement kernels move 16-byte vectors; the arithmetic runs in the GEMM / LayerNorm kernels.
#include <string.h>

#include "../../include/pscwin.h"
#include "common.cuh"
#include "pscwin_internal.h"

namespace pscwin {

// img [B, 3, 16H, 16W] bf16 (NCHW, as a PyTorch image) -> P [B*H*W, 768] bf16, column (c, ky, kx) = the flatten
// order of a Conv2d weight [C, 3, 16, 16]. One thread per (token, c, ky): 16 contiguous pixels = 2 x 16 bytes.
__global__ void __launch_bounds__(256) patchify_kernel(const __nv_bfloat16* __restrict__ img, int B, int H, int W,
                                                       __nv_bfloat16* __restrict__ P) {
  pdl_trigger();
  pdl_wait();
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long T = (long long)B * H * W;
  if (idx >= T * 48) return;
  const int cy = (int)(idx % 48);  // c * 16 + ky
  const long long t = idx / 48;
  const int x = (int)(t % W);
  const long long r = t / W;
  const int y = (int)(r % H), b = (int)(r / H);
  const int c = cy >> 4, ky = cy & 15;
  const size_t W16 = (size_t)W * 16;
  const uint4* src = reinterpret_cast<const uint4*>(img + (((size_t)b * 3 + c) * H * 16 + (size_t)y * 16 + ky) * W16 +
                                                    (size_t)x * 16);
  uint4* dst = reinterpret_cast<uint4*>(P + (size_t)t * 768 + cy * 16);
  dst[0] = src[0];
  dst[1] = src[1];
}

// u [B, H, W, C] bf16 -> A [B*H*W, 9*C]: column (tap, i), tap = dy * 3 + dx, zero outside the grid (padding 1).
__global__ void __launch_bounds__(256) im2col3x3_kernel(const __nv_bfloat16* __restrict__ u, int B, int H, int W,
                                                        int C, __nv_bfloat16* __restrict__ A) {
  pdl_trigger();
  pdl_wait();
  const int cv = C / 8;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long T = (long long)B * H * W;
  if (idx >= T * 9 * cv) return;
  const int v = (int)(idx % cv);
  const long long q = idx / cv;
  const int tap = (int)(q % 9);
  const long long t = q / 9;
  const int x = (int)(t % W);
  const long long r = t / W;
  const int y = (int)(r % H), b = (int)(r / H);
  const int sy = y + tap / 3 - 1, sx = x + tap % 3 - 1;
  uint4 val = make_uint4(0u, 0u, 0u, 0u);
  if (sy >= 0 && sy < H && sx >= 0 && sx < W)
    val = *reinterpret_cast<const uint4*>(u + (((size_t)b * H + sy) * W + sx) * C + v * 8);
  *reinterpret_cast<uint4*>(A + ((size_t)t * 9 + tap) * C + v * 8) = val;
}

// out[b, Y, X, :] (+)= bilinear(in)[b, Y, X, :], align_corners = False (half-pixel centres, clamped; reading Q22),
// f32 arithmetic, one bf16 rounding. One thread per (output token, 8 channels).
__global__ void __launch_bounds__(256) resize_bilinear_kernel(const __nv_bfloat16* __restrict__ in, int B, int h,
                                                              int w, int C, int H, int W, int accumulate,
                                                              __nv_bfloat16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int cv = C / 8;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)B * H * W * cv) return;
  const int v = (int)(idx % cv);
  const long long t = idx / cv;
  const int X = (int)(t % W);
  const long long r = t / W;
  const int Y = (int)(r % H), b = (int)(r / H);
  const float syf = fmaxf((Y + 0.5f) * ((float)h / H) - 0.5f, 0.f);
  const float sxf = fmaxf((X + 0.5f) * ((float)w / W) - 0.5f, 0.f);
  const int y0 = min((int)syf, h - 1), x0 = min((int)sxf, w - 1);
  const int y1 = min(y0 + 1, h - 1), x1 = min(x0 + 1, w - 1);
  const float fy = syf - y0, fx = sxf - x0;
  auto ld = [&](int yy, int xx) {
    return *reinterpret_cast<const uint4*>(in + (((size_t)b * h + yy) * w + xx) * C + v * 8);
  };
  const uint4 a = ld(y0, x0), bq = ld(y0, x1), c = ld(y1, x0), d = ld(y1, x1);
  const uint32_t* pa = &a.x;
  const uint32_t* pb = &bq.x;
  const uint32_t* pc = &c.x;
  const uint32_t* pd = &d.x;
  uint4* dst = reinterpret_cast<uint4*>(out + (size_t)t * C + v * 8);
  uint4 o = accumulate ? *dst : make_uint4(0u, 0u, 0u, 0u);
  uint32_t* po = &o.x;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float lo = (1.f - fy) * ((1.f - fx) * bf16_lo(pa[k]) + fx * bf16_lo(pb[k])) +
               fy * ((1.f - fx) * bf16_lo(pc[k]) + fx * bf16_lo(pd[k]));
    float hi = (1.f - fy) * ((1.f - fx) * bf16_hi(pa[k]) + fx * bf16_hi(pb[k])) +
               fy * ((1.f - fx) * bf16_hi(pc[k]) + fx * bf16_hi(pd[k]));
    if (accumulate) {
      lo += bf16_lo(po[k]);
      hi += bf16_hi(po[k]);
    }
    po[k] = pack_bf16(lo, hi);
  }
  *dst = o;
}

}  // namespace pscwin

using namespace pscwin;

namespace {
inline size_t al256e(size_t x) { return (x + 255) & ~size_t(255); }
inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int resize_launch(const void* in, int B, int h, int w, int C, int H, int W, int acc, void* out, cudaStream_t s) {
  const long long n = (long long)B * H * W * (C / 8);
  PSCWIN_PROF("resize_bilinear", s);
  launch_k(resize_bilinear_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s,
           reinterpret_cast<const __nv_bfloat16*>(in), B, h, w, C, H, W, acc, reinterpret_cast<__nv_bfloat16*>(out));
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

struct NeckWs {
  size_t f, fs, u, A, g, total;
};
NeckWs plan_neck(const pscwin_neck_desc* d) {
  NeckWs w;
  const size_t T0 = (size_t)d->B * d->H[0] * d->W[0];
  size_t Ts = 0;
  for (int i = 1; i < d->n_scales; ++i) {
    const size_t t = (size_t)d->B * d->H[i] * d->W[i];
    Ts = t > Ts ? t : Ts;
  }
  size_t off = 0;
  auto take = [&](size_t b) {
    size_t o = off;
    off += al256e(b);
    return o;
  };
  w.f = take(T0 * d->C_out * 2);
  w.fs = take((Ts ? Ts : 1) * d->C_out * 2);
  w.u = take(T0 * d->C_out * 2);
  w.A = take(T0 * 9 * d->C_out * 2);
  w.g = take(T0 * d->C_out * 2);
  w.total = off;
  return w;
}
int check_neck(const pscwin_neck_desc* d) {
  if (!d || d->B <= 0 || d->C <= 0 || d->C_out <= 0 || d->n_stages < 1 || d->n_stages > 8) return PSCWIN_ERR_SHAPE;
  if (d->n_scales < 1 || d->n_scales > PSCWIN_MAX_SCALES) return PSCWIN_ERR_SHAPE;
  for (int i = 0; i < d->n_scales; ++i)
    if (d->H[i] <= 0 || d->W[i] <= 0) return PSCWIN_ERR_SHAPE;
  if (d->C % 64 || d->C_out % 64 || d->C_out > 2048) return PSCWIN_ERR_UNSUPPORTED;  // GEMM K tiles, LN vectors
  return PSCWIN_OK;
}
// f[T, C_out] = sum_s x_s[T, C] W_s^T (GEMM chain: the first stores, the rest add in place)
int stage_sum(int n_stages, const void* const* xs, size_t row_off, long long T, int C, int C_out,
              const void* const* w_stage, void* f, cudaStream_t s) {
  for (int i = 0; i < n_stages; ++i) {
    GemmArgs a;
    memset(&a, 0, sizeof(a));
    a.prof_name = "gemm_stage_proj";
    a.M = (int)T;
    a.N = C_out;
    a.K = C;
    a.lda = C;
    a.ldb = C;
    a.out = f;
    a.ldo = C_out;
    a.epi = i == 0 ? EPI_STORE_BF16 : EPI_RESID_BF16;
    a.residual = i == 0 ? nullptr : f;
    a.ldr = C_out;
    const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(xs[i]) + row_off * C;
    if (launch_gemm_bf16(x, w_stage[i], a, s)) return -1;
  }
  return 0;
}
}  // namespace

extern "C" {

size_t pscwin_patch_embed_workspace_bytes(int32_t B, int32_t H, int32_t W) {
  if (B <= 0 || H <= 0 || W <= 0) return 0;
  return al256e((size_t)B * H * W * 768 * 2);
}

int pscwin_patch_embed(const void* img, int32_t B, int32_t H, int32_t W, int32_t C, const void* w_patch,
                       const float* b_patch, void* out, void* ws, size_t ws_bytes, void* stream) {
  if (!img || !w_patch || !out || B <= 0 || H <= 0 || W <= 0 || C <= 0) return PSCWIN_ERR_SHAPE;
  if (C % 8) return PSCWIN_ERR_UNSUPPORTED;
  if (!ws || ws_bytes < pscwin_patch_embed_workspace_bytes(B, H, W)) return PSCWIN_ERR_WORKSPACE;
  if (!al16(img) || !al16(w_patch) || !al16(out) || !al16(ws)) return PSCWIN_ERR_ALIGN;
  cudaStream_t s = (cudaStream_t)stream;
  const long long T = (long long)B * H * W;
  {
    PSCWIN_PROF("patchify", s);
    const long long n = T * 48;
    launch_k(patchify_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s,
             reinterpret_cast<const __nv_bfloat16*>(img), (int)B, (int)H, (int)W, reinterpret_cast<__nv_bfloat16*>(ws));
  }
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.prof_name = "gemm_patch_embed";
  a.M = (int)T;
  a.N = C;
  a.K = 768;
  a.lda = 768;
  a.ldb = 768;
  a.out = out;
  a.ldo = C;
  a.epi = EPI_STORE_BF16;
  a.bias = b_patch;
  return launch_gemm_bf16(ws, w_patch, a, s) ? PSCWIN_ERR_CUDA : PSCWIN_OK;
}

int pscwin_resize_bilinear(const void* in, int32_t B, int32_t h, int32_t w, int32_t Cx, int32_t H, int32_t W,
                           int32_t accumulate, void* out, void* stream) {
  if (!in || !out || B <= 0 || h <= 0 || w <= 0 || H <= 0 || W <= 0 || Cx <= 0) return PSCWIN_ERR_SHAPE;
  if (Cx % 8) return PSCWIN_ERR_UNSUPPORTED;
  if (!al16(in) || !al16(out)) return PSCWIN_ERR_ALIGN;
  return resize_launch(in, B, h, w, Cx, H, W, accumulate, out, (cudaStream_t)stream) ? PSCWIN_ERR_CUDA : PSCWIN_OK;
}

size_t pscwin_neck_workspace_bytes(const pscwin_neck_desc* d) {
  if (check_neck(d) != PSCWIN_OK) return 0;
  return plan_neck(d).total;
}

int pscwin_neck(const pscwin_neck_desc* d, const void* const* stage_outs, const void* const* w_stage,
                const float* ln1_g, const float* ln1_b, const void* w_conv, const float* ln2_g, const float* ln2_b,
                void* out, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_neck(d);
  if (rc) return rc;
  if (!stage_outs || !w_stage || !ln1_g || !ln1_b || !w_conv || !ln2_g || !ln2_b || !out) return PSCWIN_ERR_SHAPE;
  for (int i = 0; i < d->n_stages; ++i) {
    if (!stage_outs[i] || !w_stage[i]) return PSCWIN_ERR_SHAPE;
    if (!al16(stage_outs[i]) || !al16(w_stage[i])) return PSCWIN_ERR_ALIGN;
  }
  const NeckWs L = plan_neck(d);
  if (!ws || ws_bytes < L.total) return PSCWIN_ERR_WORKSPACE;
  if (!al16(ws) || !al16(out) || !al16(w_conv)) return PSCWIN_ERR_ALIGN;
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* base = reinterpret_cast<uint8_t*>(ws);
  const int Co = d->C_out;
  const long long T0 = (long long)d->B * d->H[0] * d->W[0];
  // fused stage sum on the main grid, then every other scale's sum resized onto it (HRSAM++, reading Q22)
  if (stage_sum(d->n_stages, stage_outs, 0, T0, d->C, Co, w_stage, base + L.f, s)) return PSCWIN_ERR_CUDA;
  size_t row_off = (size_t)T0;
  for (int j = 1; j < d->n_scales; ++j) {
    const long long Tj = (long long)d->B * d->H[j] * d->W[j];
    if (stage_sum(d->n_stages, stage_outs, row_off, Tj, d->C, Co, w_stage, base + L.fs, s)) return PSCWIN_ERR_CUDA;
    if (resize_launch(base + L.fs, d->B, d->H[j], d->W[j], Co, d->H[0], d->W[0], 1, base + L.f, s))
      return PSCWIN_ERR_CUDA;
    row_off += (size_t)Tj;
  }
  // conv block: LN2d -> conv3x3 (im2col + GEMM, K = 9 C_out) -> LN2d
  if (launch_layer_norm(base + L.f, T0, Co, ln1_g, ln1_b, d->ln_eps, 0, base + L.u, s)) return PSCWIN_ERR_CUDA;
  {
    PSCWIN_PROF("im2col3x3", s);
    const long long n = T0 * 9 * (Co / 8);
    launch_k(im2col3x3_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s,
             reinterpret_cast<const __nv_bfloat16*>(base + L.u), d->B, d->H[0], d->W[0], Co,
             reinterpret_cast<__nv_bfloat16*>(base + L.A));
  }
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.prof_name = "gemm_neck_conv";
  a.M = (int)T0;
  a.N = Co;
  a.K = 9 * Co;
  a.lda = 9 * Co;
  a.ldb = 9 * Co;
  a.out = base + L.g;
  a.ldo = Co;
  a.epi = EPI_STORE_BF16;
  if (launch_gemm_bf16(base + L.A, w_conv, a, s)) return PSCWIN_ERR_CUDA;
  if (launch_layer_norm(base + L.g, T0, Co, ln2_g, ln2_b, d->ln_eps, 0, out, s)) return PSCWIN_ERR_CUDA;
  return PSCWIN_OK;
}

}  // extern "C"
