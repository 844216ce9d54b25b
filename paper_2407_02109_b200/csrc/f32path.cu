// fp32 correctness path of the PSCWin layer (dtype PSCWIN_F32; north star "max relative error 1e-4 (fp32 path)").
// Every activation and weight is fp32 and every step runs in fp32 on CUDA cores; nothing is rounded to bf16:
//   a4 / a7 / a1 / a3 projections : sgemm_kernel (64x64 tiles, fused bias / 2-D RoPE / SiLU / residual epilogue)
//   a5 + a6 + crop                : attn_f32_kernel, one CTA per (image, window, head), the padded window built in
//                                   shared memory (learnable pad keys rotated at their geometric coordinates)
//   a2 cycle scan                 : conv / dt on CUDA cores, then the LITERAL 3L recurrence (scan_literal_kernel:
//                                   warp per channel, lane per state, sequential over the cycled sequence) — an
//                                   algorithm independent of the bf16 path's two-pass closed form.
// Performance is not the point of this path (it is the 1e-4 parity gate); the bf16 path is the product hot path.
#include <math.h>
#include <string.h>

#include "../../include/pscwin.h"
#include "common.cuh"
#include "pscwin_internal.h"

namespace pscwin {

// ------------------------------------------------------------------------------------------------- GEMM
// out[M, N] = epi(A[M, K] . B[N, K]^T); row-major, K contiguous in both operands.
struct SgemmArgs {
  int M, N, K;
  const float* A;
  int lda;
  const float* B;
  int ldb;
  float* out;
  int ldo;
  const float* bias;      // [N] or null
  const float* residual;  // [M, ldr] or null
  int ldr;
  int silu_col;           // columns >= silu_col get SiLU (0 = off)
  int gelu;               // 1: exact GELU on every output (FFN fc1)
  int rope, HW, Wgrid, C, d_head;  // 2-D RoPE on q = cols [0, C) and k = [C, 2C) (QKV projection)
};

__device__ __forceinline__ void rope_cs_f32(int pos, int fj, int d, float& c, float& s) {
  const float turns = (float)pos * kRopeTurns64[fj * (64 / d)];
  const float f = turns - rintf(turns);
  sincospif(2.f * f, &s, &c);
}

// RoPE of the pair (col, col+1) of a q or k head at grid position (px, py); pairs (2j, 2j+1) of the first half
// of a head rotate with x, of the second half with y (d = 64: frequency j within the half; d = 32: j & 7)
__device__ __forceinline__ void rope_apply(float& a, float& b, int hc, int d, int px, int py) {
  const int jj = hc >> 1;  // pair index within the head
  int axis, fj;
  if (d == 64) {
    axis = jj >= 16;
    fj = jj & 15;
  } else {
    axis = jj >= 8;
    fj = jj & 7;
  }
  float c, s;
  rope_cs_f32(axis ? py : px, fj, d, c, s);
  const float x0 = a * c - b * s, x1 = a * s + b * c;
  a = x0;
  b = x1;
}

constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16;
__global__ void __launch_bounds__(256) sgemm_kernel(SgemmArgs p) {
  pdl_trigger();
  pdl_wait();
  __shared__ float As[SG_BK][SG_BM + 4];
  __shared__ float Bs[SG_BK][SG_BN + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * SG_BM, n0 = blockIdx.x * SG_BN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < p.K; k0 += SG_BK) {
    // 64 x 16 of A and of B: thread loads 4 elements of each (row = tid / 4, k = (tid % 4) * 4 ..)
    {
      const int r = threadIdx.x >> 2, kq = (threadIdx.x & 3) * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int k = k0 + kq + e;
        const int ra = m0 + r, rb = n0 + r;
        As[kq + e][r] = (ra < p.M && k < p.K) ? p.A[(size_t)ra * p.lda + k] : 0.f;
        Bs[kq + e][r] = (rb < p.N && k < p.K) ? p.B[(size_t)rb * p.ldb + k] : 0.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SG_BK; ++k) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + ty * 4 + i;
    if (row >= p.M) continue;
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = n0 + tx * 4 + j;
      v[j] = acc[i][j] + ((p.bias && col < p.N) ? p.bias[col] : 0.f);
    }
    const int c0 = n0 + tx * 4;  // multiple of 4: the two pairs (c0, c0+1), (c0+2, c0+3)
    if (p.rope && c0 < 2 * p.C) {
      const int t = row % p.HW, py = t / p.Wgrid, px = t - py * p.Wgrid;
#pragma unroll
      for (int j = 0; j < 4; j += 2) rope_apply(v[j], v[j + 1], (c0 + j) % p.d_head, p.d_head, px, py);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = c0 + j;
      if (col >= p.N) continue;
      float y = v[j];
      if (p.gelu) y = 0.5f * y * (1.f + erff(y * 0.70710678118654752f));
      if (p.silu_col > 0 && col >= p.silu_col) y = y / (1.f + expf(-y));
      if (p.residual) y += p.residual[(size_t)row * p.ldr + col];
      p.out[(size_t)row * p.ldo + col] = y;
    }
  }
}

static int launch_sgemm(const SgemmArgs& a, cudaStream_t s) {
  if (a.M <= 0 || a.N <= 0) return 0;
  dim3 grid((a.N + SG_BN - 1) / SG_BN, (a.M + SG_BM - 1) / SG_BM);
  PSCWIN_PROF("sgemm_f32", s);
  launch_k(sgemm_kernel, grid, dim3(256), 0, s, a);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------- attention
// One CTA per (image, padded-grid window, head); thread = window slot. K / V of all w^2 slots in shared memory
// (real cells from qkv; LEARNABLE pad cells = the projected pad token, its k rotated at the cell's geometric
// coordinate; MASKED pad cells excluded); each real query runs an online softmax over the window's keys.
struct AttnF32Args {
  const float* qkv;      // [B, H, W, 3C], q / k already rotated
  const float* qkv_pad;  // [3C] unrotated (LEARNABLE shifted layers)
  float* out;            // [B, H, W, C]
  int B, H, W, C, heads, w, pl, pt, nwx, nw, pad_mode, rope;
};

template <int D>
__global__ void __launch_bounds__(256) attn_f32_kernel(AttnF32Args p) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float s_kv[];  // K [w^2][D] | V [w^2][D] | valid [w^2]
  const int ww = p.w * p.w;
  float* sK = s_kv;
  float* sV = s_kv + (size_t)ww * D;
  float* sValid = sV + (size_t)ww * D;
  const int h = blockIdx.x % p.heads;
  const int r = blockIdx.x / p.heads;
  const int win = r % p.nw, b = r / p.nw;
  const int wy = win / p.nwx, wx = win - wy * p.nwx;
  const int X0 = wx * p.w - p.pl, Y0 = wy * p.w - p.pt;
  const int C3 = 3 * p.C;
  for (int i = threadIdx.x; i < ww; i += blockDim.x) {
    const int X = X0 + i % p.w, Y = Y0 + i / p.w;
    const bool real = X >= 0 && X < p.W && Y >= 0 && Y < p.H;
    float* k = sK + (size_t)i * D;
    float* v = sV + (size_t)i * D;
    if (real) {
      const float* src = p.qkv + (((size_t)b * p.H + Y) * p.W + X) * C3 + h * D;
      for (int e = 0; e < D; ++e) {
        k[e] = src[p.C + e];
        v[e] = src[2 * p.C + e];
      }
      sValid[i] = 1.f;
    } else if (p.pad_mode == PSCWIN_PAD_LEARNABLE) {
      const float* src = p.qkv_pad + h * D;
      for (int e = 0; e < D; ++e) {
        k[e] = src[p.C + e];
        v[e] = src[2 * p.C + e];
      }
      if (p.rope)
        for (int e = 0; e < D; e += 2) rope_apply(k[e], k[e + 1], e, D, X, Y);
      sValid[i] = 1.f;
    } else {
      sValid[i] = 0.f;
    }
  }
  __syncthreads();
  const float scale = 1.f / sqrtf((float)D);
  for (int i = threadIdx.x; i < ww; i += blockDim.x) {
    const int X = X0 + i % p.w, Y = Y0 + i / p.w;
    if (X < 0 || X >= p.W || Y < 0 || Y >= p.H) continue;  // pad query rows are discarded
    const size_t tok = ((size_t)b * p.H + Y) * p.W + X;
    float q[D], o[D];
    const float* qs = p.qkv + tok * C3 + h * D;
#pragma unroll
    for (int e = 0; e < D; ++e) {
      q[e] = qs[e] * scale;
      o[e] = 0.f;
    }
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < ww; ++j) {
      if (sValid[j] == 0.f) continue;
      const float* k = sK + (size_t)j * D;
      float s = 0.f;
#pragma unroll
      for (int e = 0; e < D; ++e) s = fmaf(q[e], k[e], s);
      const float mn = fmaxf(m, s);
      const float corr = expf(m - mn), pj = expf(s - mn);
      l = l * corr + pj;
      const float* v = sV + (size_t)j * D;
#pragma unroll
      for (int e = 0; e < D; ++e) o[e] = fmaf(pj, v[e], o[e] * corr);
      m = mn;
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    float* dst = p.out + tok * p.C + h * D;
#pragma unroll
    for (int e = 0; e < D; ++e) dst[e] = o[e] * inv;
  }
}

int launch_attention_f32(const pscwin_layer_desc* d, const float* qkv, const float* qkv_pad, float* out,
                         cudaStream_t s) {
  const int w = d->window, D = d->C / d->heads;
  const int pl = (w - d->shift_x) % w, pt = (w - d->shift_y) % w;
  const int pr = ((-(pl + d->W)) % w + w) % w, pb = ((-(pt + d->H)) % w + w) % w;
  AttnF32Args a;
  a.qkv = qkv;
  a.qkv_pad = qkv_pad;
  a.out = out;
  a.B = d->B;
  a.H = d->H;
  a.W = d->W;
  a.C = d->C;
  a.heads = d->heads;
  a.w = w;
  a.pl = pl;
  a.pt = pt;
  a.nwx = (pl + d->W + pr) / w;
  a.nw = a.nwx * ((pt + d->H + pb) / w);
  a.pad_mode = d->pad_mode;
  a.rope = d->rope;
  const size_t smem = (size_t)w * w * (2 * D + 1) * 4;
  if (smem > 227 * 1024) return PSCWIN_ERR_UNSUPPORTED;
  const dim3 grid((unsigned)(d->B * a.nw * d->heads));
  PSCWIN_PROF("attention_f32", s);
  if (D == 64) {
    cudaFuncSetAttribute(attn_f32_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(attn_f32_kernel<64>, grid, dim3(256), smem, s, a);
  } else if (D == 32) {
    cudaFuncSetAttribute(attn_f32_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(attn_f32_kernel<32>, grid, dim3(256), smem, s, a);
  } else {
    return PSCWIN_ERR_UNSUPPORTED;
  }
  return cudaGetLastError() == cudaSuccess ? PSCWIN_OK : PSCWIN_ERR_CUDA;
}

// ------------------------------------------------------------------------------------------------- cycle scan
// Rows of the scan buffers: [0, L) the copy-2/3 stream in SCAN order, [L, L+P) copy 1's first P = k-1 tokens
// (whose causal conv sees zero history, reading Q10).
struct ScanF32Args {
  int B, H, W, order, window, D, N, R, k, P;
  const float* xin;  // [B, L, ld_x] grid order
  long long ld_x;
  const float* z;    // [B, L, ld_z] grid order or null
  long long ld_z;
  const float *conv_w, *conv_b, *w_dt, *b_dt, *a_log, *d_skip;
  float* v;          // [B, L+P, D]
  float* dbc;        // [B, L+P, R+2N]
  float* delta;      // [B, L+P, D]
  float* out;        // [B, L, ld_out] grid order
  long long ld_out;
  int bbar;
};

__device__ __forceinline__ int scan_pi_f32(int t, int H, int W, int order, int w) {
  if (order == PSCWIN_SCAN_COL_MAJOR) {
    const int c = t / H, r = t - c * H;
    return r * W + c;
  }
  if (order == PSCWIN_SCAN_WINDOW_MAJOR) {
    const int sx = t % w;
    int q = t / w;
    const int sy = q % w;
    q /= w;
    const int nwx = W / w;
    return ((q / nwx) * w + sy) * W + (q % nwx) * w + sx;
  }
  return t;
}

// v = SiLU(b + sum_i w[i] x[t - (k-1) + i]) along the scan order; thread per (row, channel)
__global__ void __launch_bounds__(256) conv_f32_kernel(ScanF32Args p) {
  pdl_trigger();
  pdl_wait();
  const int L = p.H * p.W, rows = L + p.P;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)p.B * rows * p.D) return;
  const int d = (int)(idx % p.D);
  const long long rr = idx / p.D;
  const int b = (int)(rr / rows), r = (int)(rr - (long long)b * rows);
  const bool copy1 = r >= L;
  const int t = copy1 ? r - L : r;
  float acc = p.conv_b[d];
  for (int i = 0; i < p.k; ++i) {
    int tt = t - (p.k - 1) + i;
    if (tt < 0) {
      if (copy1) continue;
      tt += L;
    }
    const int g = scan_pi_f32(tt, p.H, p.W, p.order, p.window);
    acc = fmaf(p.conv_w[d * p.k + i], p.xin[((long long)b * L + g) * p.ld_x + d], acc);
  }
  p.v[((long long)b * rows + r) * p.D + d] = acc / (1.f + expf(-acc));
}

// Delta = softplus(delta_low W_dt^T + b_dt), thread per (row, channel)
__global__ void __launch_bounds__(256) dt_f32_kernel(ScanF32Args p) {
  pdl_trigger();
  pdl_wait();
  const int rows = p.H * p.W + p.P, Wd = p.R + 2 * p.N;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)p.B * rows * p.D) return;
  const int d = (int)(idx % p.D);
  const long long row = idx / p.D;
  float x = p.b_dt[d];
  for (int r = 0; r < p.R; ++r) x = fmaf(p.dbc[row * Wd + r], p.w_dt[(size_t)d * p.R + r], x);
  p.delta[row * p.D + d] = x > 20.f ? x : log1pf(expf(x));
}

// The literal cycled recurrence (Eqs. 3-4): warp per (image, channel), lane per state
// (N <= 64: two per lane), j = 0 .. 3L-1 over copy c = j / L, token t = j mod L in scan order.
__global__ void __launch_bounds__(256) scan_literal_kernel(ScanF32Args p) {
  pdl_trigger();
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= p.B * p.D) return;
  const int b = warp / p.D, d = warp - b * p.D;
  const int L = p.H * p.W, rows = L + p.P, Wd = p.R + 2 * p.N;
  float A[2], h[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int n = lane + 32 * q;
    A[q] = n < p.N ? -expf(p.a_log[d * p.N + n]) : 0.f;
    h[q] = 0.f;
  }
  const float Ds = p.d_skip[d];
  for (int j = 0; j < 3 * L; ++j) {
    const int c = j / L, t = j - c * L;
    const long long row = (long long)b * rows + ((c == 0 && t < p.P) ? L + t : t);
    const float dt = p.delta[row * p.D + d], v = p.v[row * p.D + d];
    float y = 0.f;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int n = lane + 32 * q;
      if (n >= p.N) continue;
      const float Bn = p.dbc[row * Wd + p.R + n], Cn = p.dbc[row * Wd + p.R + p.N + n];
      const float x = dt * A[q];
      const float bbar = p.bbar == 0 ? expm1f(x) / A[q] * Bn : dt * Bn;
      h[q] = fmaf(expf(x), h[q], bbar * v);
      y = fmaf(Cn, h[q], y);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
    if (lane == 0) {
      y = fmaf(Ds, v, y);
      const long long tok = (long long)b * L + scan_pi_f32(t, p.H, p.W, p.order, p.window);
      float* dst = p.out + tok * p.ld_out + d;
      const float g = p.z ? p.z[tok * p.ld_z + d] : 1.f;  // gate: z already holds SiLU(z) (see callers)
      *dst = (c == 0 ? 0.f : *dst) + y * g;
    }
  }
}

// SiLU of the raw gate (standalone cycle_scan entry point), into a workspace buffer
__global__ void __launch_bounds__(256) silu_f32_kernel(const float* z, long long ld_z, long long rows, int D,
                                                       float* out) {
  pdl_trigger();
  pdl_wait();
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * D) return;
  const long long r = idx / D;
  const int d = (int)(idx - r * D);
  const float x = z[r * ld_z + d];
  out[idx] = x / (1.f + expf(-x));
}

static size_t al256f(size_t x) { return (x + 255) & ~size_t(255); }

size_t scan_f32_ws_bytes(int B, int L, int D, int N, int R, int k) {
  const size_t rows = (size_t)B * (L + k - 1);
  return al256f(rows * D * 4) * 2 + al256f(rows * (R + 2 * N) * 4) + al256f((size_t)B * L * D * 4);
}

// xin, z (gated if z_gated) grid order -> out grid order
int run_cycle_scan_f32(int B, int H, int W, int order, int window, int D, int N, int R, int k, int bbar,
                       const float* xin, long long ld_x, const float* z, long long ld_z, bool z_gated,
                       const float* conv_w, const float* conv_b, const float* w_x, const float* w_dt,
                       const float* b_dt, const float* a_log, const float* d_skip, float* out, long long ld_out,
                       void* ws, size_t ws_bytes, cudaStream_t s) {
  if (N > 64) return PSCWIN_ERR_UNSUPPORTED;
  const int L = H * W, P = k - 1;
  if (ws_bytes < scan_f32_ws_bytes(B, L, D, N, R, k)) return PSCWIN_ERR_WORKSPACE;
  const size_t rows = (size_t)B * (L + P);
  uint8_t* base = reinterpret_cast<uint8_t*>(ws);
  ScanF32Args p;
  p.B = B;
  p.H = H;
  p.W = W;
  p.order = order;
  p.window = window;
  p.D = D;
  p.N = N;
  p.R = R;
  p.k = k;
  p.P = P;
  p.xin = xin;
  p.ld_x = ld_x;
  p.z = z;
  p.ld_z = ld_z;
  p.conv_w = conv_w;
  p.conv_b = conv_b;
  p.w_dt = w_dt;
  p.b_dt = b_dt;
  p.a_log = a_log;
  p.d_skip = d_skip;
  p.v = reinterpret_cast<float*>(base);
  p.delta = reinterpret_cast<float*>(base + al256f(rows * D * 4));
  p.dbc = reinterpret_cast<float*>(base + 2 * al256f(rows * D * 4));
  float* gz = reinterpret_cast<float*>(base + 2 * al256f(rows * D * 4) + al256f(rows * (R + 2 * N) * 4));
  p.out = out;
  p.ld_out = ld_out;
  p.bbar = bbar;
  if (z && !z_gated) {
    const long long n = (long long)B * L * D;
    launch_k(silu_f32_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, z, ld_z, (long long)B * L, D, gz);
    p.z = gz;
    p.ld_z = D;
  }
  const long long n = (long long)rows * D;
  {
    PSCWIN_PROF("conv_f32", s);
    launch_k(conv_f32_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, p);
  }
  SgemmArgs g;
  memset(&g, 0, sizeof(g));
  g.M = (int)rows;
  g.N = R + 2 * N;
  g.K = D;
  g.A = p.v;
  g.lda = D;
  g.B = w_x;
  g.ldb = D;
  g.out = p.dbc;
  g.ldo = R + 2 * N;
  if (launch_sgemm(g, s)) return PSCWIN_ERR_CUDA;
  {
    PSCWIN_PROF("dt_f32", s);
    launch_k(dt_f32_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, p);
  }
  {
    PSCWIN_PROF("scan_literal_f32", s);
    const long long warps = (long long)B * D;
    launch_k(scan_literal_kernel, dim3((unsigned)((warps + 7) / 8)), dim3(256), 0, s, p);
  }
  return cudaGetLastError() == cudaSuccess ? PSCWIN_OK : PSCWIN_ERR_CUDA;
}

// ------------------------------------------------------------------------------------------------- layer
LayerWsF32 plan_layer_f32(const pscwin_layer_desc* d) {
  LayerWsF32 w;
  const size_t T = (size_t)d->B * d->H * d->W, C = d->C;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += al256f(bytes);
    return o;
  };
  w.u = take(T * C * 4);
  w.qkv = take(T * 3 * C * 4);
  w.qkv_pad = take(3 * C * 4);
  w.O = take(T * C * 4);
  w.h = d->mlp_hidden > 0 ? take(T * d->mlp_hidden * 4) : 0;
  w.xz = w.g = w.scan = w.x1 = 0;
  if (d->cycle_scan) {
    const size_t D = (size_t)d->ssm_expand * C;
    const int R = d->ssm_dt_rank > 0 ? d->ssm_dt_rank : (d->C + 15) / 16;
    w.xz = take(T * 2 * D * 4);
    w.g = take(T * D * 4);
    w.x1 = take(T * C * 4);
    w.scan = take(scan_f32_ws_bytes(d->B, d->H * d->W, (int)D, d->ssm_state, R, d->ssm_conv));
  }
  w.total = off;
  return w;
}

size_t layer_f32_ws_bytes(const pscwin_layer_desc* d) { return plan_layer_f32(d).total; }

int qkv_project_f32(const pscwin_layer_desc* d, const pscwin_layer_weights* wt, const float* x, float* qkv,
                    float* qkv_pad, float* u, cudaStream_t s) {
  const long long T = (long long)d->B * d->H * d->W;
  const int C = d->C;
  int rc = launch_layer_norm(x, T, C, (const float*)wt->ln1_g, (const float*)wt->ln1_b, d->ln_eps, 1, u, s);
  if (rc) return PSCWIN_ERR_CUDA;
  SgemmArgs g;
  memset(&g, 0, sizeof(g));
  g.M = (int)T;
  g.N = 3 * C;
  g.K = C;
  g.A = u;
  g.lda = C;
  g.B = (const float*)wt->w_qkv;
  g.ldb = C;
  g.out = qkv;
  g.ldo = 3 * C;
  g.bias = (const float*)wt->b_qkv;
  g.rope = d->rope;
  g.HW = d->H * d->W;
  g.Wgrid = d->W;
  g.C = C;
  g.d_head = C / d->heads;
  if (launch_sgemm(g, s)) return PSCWIN_ERR_CUDA;
  if (qkv_pad && wt->pad) {
    rc = launch_pad_qkv(wt->pad, wt->w_qkv, (const float*)wt->b_qkv, C, 1, qkv_pad, s);
    if (rc) return PSCWIN_ERR_CUDA;
  }
  return PSCWIN_OK;
}

int forward_f32(const pscwin_layer_desc* d, const pscwin_layer_weights* wt, const void* x_in_v, void* x_out_v,
                void* ws, size_t ws_bytes, cudaStream_t s) {
  const LayerWsF32 L = plan_layer_f32(d);
  if (ws_bytes < L.total) return PSCWIN_ERR_WORKSPACE;
  uint8_t* base = reinterpret_cast<uint8_t*>(ws);
  const float* x = reinterpret_cast<const float*>(x_in_v);
  float* x_out = reinterpret_cast<float*>(x_out_v);
  const long long T = (long long)d->B * d->H * d->W;
  const int C = d->C;
  int rc;
  if (d->cycle_scan) {
    if (!wt->lns_g || !wt->lns_b || !wt->w_in || !wt->conv_w || !wt->conv_b || !wt->w_x || !wt->w_dt ||
        !wt->b_dt || !wt->a_log || !wt->d_skip || !wt->w_out)
      return PSCWIN_ERR_SHAPE;
    const int D = d->ssm_expand * C, N = d->ssm_state;
    const int R = d->ssm_dt_rank > 0 ? d->ssm_dt_rank : (C + 15) / 16;
    float* u = reinterpret_cast<float*>(base + L.u);
    float* xz = reinterpret_cast<float*>(base + L.xz);
    float* g = reinterpret_cast<float*>(base + L.g);
    float* x1 = reinterpret_cast<float*>(base + L.x1);
    rc = launch_layer_norm(x, T, C, (const float*)wt->lns_g, (const float*)wt->lns_b, d->ln_eps, 1, u, s);
    if (rc) return PSCWIN_ERR_CUDA;
    SgemmArgs a;
    memset(&a, 0, sizeof(a));
    a.M = (int)T;
    a.N = 2 * D;
    a.K = C;
    a.A = u;
    a.lda = C;
    a.B = (const float*)wt->w_in;
    a.ldb = C;
    a.out = xz;
    a.ldo = 2 * D;
    a.silu_col = D;  // z half -> SiLU(z)
    if (launch_sgemm(a, s)) return PSCWIN_ERR_CUDA;
    rc = run_cycle_scan_f32(d->B, d->H, d->W, d->scan_order, d->window, D, N, R, d->ssm_conv, d->bbar_mode, xz, 2 * D,
                            xz + D, 2 * D, true, (const float*)wt->conv_w, (const float*)wt->conv_b,
                            (const float*)wt->w_x, (const float*)wt->w_dt, (const float*)wt->b_dt, wt->a_log,
                            wt->d_skip, g, D, base + L.scan, L.total - L.scan, s);
    if (rc) return rc;
    memset(&a, 0, sizeof(a));
    a.M = (int)T;
    a.N = C;
    a.K = D;
    a.A = g;
    a.lda = D;
    a.B = (const float*)wt->w_out;
    a.ldb = D;
    a.out = x1;
    a.ldo = C;
    a.residual = x;
    a.ldr = C;
    if (launch_sgemm(a, s)) return PSCWIN_ERR_CUDA;
    x = x1;
  }
  float* u = reinterpret_cast<float*>(base + L.u);
  float* qkv = reinterpret_cast<float*>(base + L.qkv);
  float* qkv_pad = reinterpret_cast<float*>(base + L.qkv_pad);
  float* O = reinterpret_cast<float*>(base + L.O);
  rc = qkv_project_f32(d, wt, x, qkv, qkv_pad, u, s);
  if (rc) return rc;
  rc = launch_attention_f32(d, qkv, qkv_pad, O, s);
  if (rc) return rc;
  SgemmArgs a;
  memset(&a, 0, sizeof(a));
  a.M = (int)T;
  a.N = C;
  a.K = C;
  a.A = O;
  a.lda = C;
  a.B = (const float*)wt->w_o;
  a.ldb = C;
  a.out = x_out;
  a.ldo = C;
  a.bias = (const float*)wt->b_o;
  a.residual = x;
  a.ldr = C;
  if (launch_sgemm(a, s)) return PSCWIN_ERR_CUDA;
  if (d->mlp_hidden > 0) {  // FFN sub-layer: x_out += GELU(LN2(x_out) W_fc1^T + b_fc1) W_fc2^T + b_fc2
    const int Hd = d->mlp_hidden;
    float* h = reinterpret_cast<float*>(base + L.h);
    rc = launch_layer_norm(x_out, T, C, (const float*)wt->ln2_g, (const float*)wt->ln2_b, d->ln_eps, 1, u, s);
    if (rc) return PSCWIN_ERR_CUDA;
    memset(&a, 0, sizeof(a));
    a.M = (int)T;
    a.N = Hd;
    a.K = C;
    a.A = u;
    a.lda = C;
    a.B = (const float*)wt->w_fc1;
    a.ldb = C;
    a.out = h;
    a.ldo = Hd;
    a.bias = (const float*)wt->b_fc1;
    a.gelu = 1;
    if (launch_sgemm(a, s)) return PSCWIN_ERR_CUDA;
    memset(&a, 0, sizeof(a));
    a.M = (int)T;
    a.N = C;
    a.K = Hd;
    a.A = h;
    a.lda = Hd;
    a.B = (const float*)wt->w_fc2;
    a.ldb = Hd;
    a.out = x_out;
    a.ldo = C;
    a.bias = (const float*)wt->b_fc2;
    a.residual = x_out;  // each element's residual is read by the thread that then writes it
    a.ldr = C;
    if (launch_sgemm(a, s)) return PSCWIN_ERR_CUDA;
  }
  return PSCWIN_OK;
}

}  // namespace pscwin
