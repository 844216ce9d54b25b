// Cycle-scan module (§3.3 Eqs. 2-4, Mamba selective SSM P:L161,
// cycle scan P:L165 "repeats the image token sequence three times ... scans ... split into the corresponding
// three sequences and ... merged through summation"; Mamba-1 block internals = DESIGN.md reading Q9).
//
// The literal method scans 3L tokens sequentially. The three copies see identical per-token parameters except
// for the first P = k-1 tokens of copy 1, whose causal conv sees zero history (reading Q10). With diagonal A the
// summed output obeys (pinned in fp64 by tests/test_oracle_pins.py):
//   prefix t < P : per copy, h^(c)_t from c_1 = 0, c_2 = end of copy 1, c_3 = end of copy 2
//   body  t >= P : H_t = A_bar_t H_{t-1} + 3 B_bar_t v_t ,  y_t = C_t . H_t + 3 D v_t ,  H_{P-1} = sum_c h^(c)_{P-1}
// so the GPU runs two chunk-parallel passes over L instead of one sequential pass over 3L:
//   conv      : v = SiLU(causal conv) for the copy-2/3 stream (history = sequence tail) + the P copy-1 rows
//   x_proj    : (delta_low, B, C) = v W_x^T on tcgen05 (f32 out)
//   dt        : Delta = softplus(delta_low W_dt^T + b_dt) for every stream row (fp32, stored)
//   pass 1    : per (chunk, channel): chunk sum of Delta and the chunk-end state from zero (b_c) — thread per
//               channel, N states in registers
//   carry     : per (image, channel) warp, lane = state: copy prefixes, fold of (exp(A sum Delta), b_c) over the
//               chunks, c_2, c_3, the prefix outputs, and every chunk's entry state H_in
//   pass 2    : per (chunk, channel): the summed recurrence from H_in, y, gate SiLU(z), bf16 store
// Transcendentals: ex2.approx on the MUFU pipe (A pre-scaled by log2 e); everything else FP32.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/pscwin.h"
#include "common.cuh"
#include "pscwin_internal.h"

namespace pscwin {

namespace {
constexpr float kLog2e = 1.4426950408889634f;
}

struct ScanParams {
  int B, L, D, N, R, k, P, Lc, n_chunks, bbar;
  const __nv_bfloat16* xin;
  long long ld_x;
  const __nv_bfloat16* gz;  // output gate SiLU(z) [B, L] rows of stride ld_gz, or null (no gate)
  long long ld_gz;
  const float *conv_w, *conv_b, *w_dt, *b_dt, *a_log, *d_skip;
  __nv_bfloat16* v;  // [B, L+P, D]
  float* dbc;        // [B, L+P, R+2N]
  float* delta;      // [B, L+P, D]
  float* sumdt;      // [B, n_chunks, D]
  float* hs;         // [B, n_chunks, D, N]
  __nv_bfloat16* out;
  long long ld_out;
  int vec_out;  // pass 2 may store 16-byte vectors of 8 channels (ld_out % 8 == 0, 16-byte aligned out)
  // band mode (window-row sharding): the k-1 xin rows preceding this segment in the cycled sequence
  // (the previous rank's tail; rank 0: the global sequence tail) replace the local wrap-around; null = one segment
  const __nv_bfloat16* hist;
  int conv_rev;  // conv_silu visits row groups last-first (A/B knob PSCWIN_CONV_REV)
};

// SiLU(x) = x / (1 + e^-x) with the fast division (MUFU rcp; -> 0 as e^-x overflows for very negative x)
__device__ __forceinline__ float silu_f(float x) { return __fdividef(x, 1.f + __expf(-x)); }
__device__ __forceinline__ float softplus_f(float x) { return x > 20.f ? x : log1pf(__expf(x)); }

// ------------------------------------------------------------------------------------------------- conv
// v rows [0, L): copy-2/3 stream (tap index wraps to the sequence tail); rows [L, L+P): copy-1 tokens 0..P-1
// (taps before the sequence start contribute 0). A thread owns 8 channels x CONV_T consecutive rows: it issues the
// CONV_T + k - 1 input loads of its window up front (independent 16-byte loads, coalesced across the warp's channel
// groups), keeps its 8 x k taps in registers, and slides the window in registers.
constexpr int KMAX = 4;  // conv width supported (Mamba default 4)
#ifndef PSCWIN_CONV_T
#define PSCWIN_CONV_T 8  // rows per thread (sweeps: PSCWIN_NVCC_FLAGS)
#endif
constexpr int CONV_T = PSCWIN_CONV_T;
__global__ void __launch_bounds__(256) conv_silu_kernel(ScanParams p) {
  pdl_trigger();
  pdl_wait();
  const int dv = p.D / 8;
  const int rows_img = p.L + p.P;
  const int groups_img = (rows_img + CONV_T - 1) / CONV_T;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)p.B * groups_img * dv) return;
  const int d0 = (int)(idx % dv) * 8;
  // row groups last-first (p.conv_rev): the in_proj GEMM has just written xin in row order, so its last rows are the
  // L2-resident ones; and the x_proj GEMM, which reads v first-to-last, then finds the rows written last first
  const long long ngrp = (long long)p.B * groups_img;
  const long long grp = p.conv_rev ? ngrp - 1 - idx / dv : idx / dv;
  const int b = (int)(grp / groups_img);
  const int r0 = (int)(grp - (long long)b * groups_img) * CONV_T;
  const __nv_bfloat16* xb = p.xin + (long long)b * p.L * p.ld_x + d0;
  __nv_bfloat16* vb = p.v + (long long)b * rows_img * p.D + d0;
  // token tt of the copy-2/3 stream; tt < 0 is the history before this segment (wrap-around or the band's hist)
  auto load_tok = [&](int tt) {
    if (tt < 0) {
      if (p.hist) return *reinterpret_cast<const uint4*>(p.hist + ((long long)b * (p.k - 1) + tt + p.k - 1) * p.D + d0);
      tt += p.L;
    }
    return *reinterpret_cast<const uint4*>(xb + (long long)tt * p.ld_x);
  };
  float wk[8][KMAX], bias[8];
  {
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(p.conv_b + d0));
    const float4 b1 = __ldg(reinterpret_cast<const float4*>(p.conv_b + d0 + 4));
    bias[0] = b0.x; bias[1] = b0.y; bias[2] = b0.z; bias[3] = b0.w;
    bias[4] = b1.x; bias[5] = b1.y; bias[6] = b1.z; bias[7] = b1.w;
  }
  auto emit = [&](int r, const uint4 (&xw)[KMAX]) {  // xw[i] = input of tap i (zeros where absent)
    uint4 o;
    uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float a0 = bias[2 * q], a1 = bias[2 * q + 1];
#pragma unroll
      for (int i = 0; i < KMAX; ++i) {
        const uint32_t u = reinterpret_cast<const uint32_t*>(&xw[i])[q];
        a0 = fmaf(wk[2 * q][i], bf16_lo(u), a0);
        a1 = fmaf(wk[2 * q + 1][i], bf16_hi(u), a1);
      }
      ow[q] = pack_bf16(silu_f(a0), silu_f(a1));
    }
    *reinterpret_cast<uint4*>(vb + (long long)r * p.D) = o;
  };
  if (r0 + CONV_T <= p.L) {
    // body rows: the window is tokens r0-(k-1) .. r0+CONV_T-1 (negative indices wrap to the sequence tail)
    uint4 xs[CONV_T + KMAX - 1];
#pragma unroll
    for (int m = 0; m < CONV_T + KMAX - 1; ++m) {
      const int tt = r0 - (p.k - 1) + m;
      xs[m] = (m < CONV_T + p.k - 1) ? load_tok(tt) : make_uint4(0u, 0u, 0u, 0u);
    }
    if (p.k == 4) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 w4 = __ldg(reinterpret_cast<const float4*>(p.conv_w + (d0 + c) * 4));
        wk[c][0] = w4.x; wk[c][1] = w4.y; wk[c][2] = w4.z; wk[c][3] = w4.w;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int i = 0; i < KMAX; ++i) wk[c][i] = i < p.k ? __ldg(p.conv_w + (d0 + c) * p.k + i) : 0.f;
    }
#pragma unroll
    for (int rr = 0; rr < CONV_T; ++rr) {
      uint4 xw[KMAX];
#pragma unroll
      for (int i = 0; i < KMAX; ++i) xw[i] = xs[rr + i];  // tap i of row r0+rr is token r0+rr-(k-1)+i
      emit(r0 + rr, xw);
    }
  } else {
    // rows at the end of the body and the copy-1 rows: generic per-row taps
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int i = 0; i < KMAX; ++i) wk[c][i] = i < p.k ? __ldg(p.conv_w + (d0 + c) * p.k + i) : 0.f;
    for (int rr = 0; rr < CONV_T; ++rr) {
      const int r = r0 + rr;
      if (r >= rows_img) break;
      const bool copy1 = r >= p.L;
      const int t = copy1 ? r - p.L : r;
      uint4 xw[KMAX];
#pragma unroll
      for (int i = 0; i < KMAX; ++i) {
        xw[i] = make_uint4(0u, 0u, 0u, 0u);
        if (i < p.k) {
          const int tt = t - (p.k - 1) + i;
          if (tt >= 0 || !copy1) xw[i] = load_tok(tt);
        }
      }
      emit(r, xw);
    }
  }
}

// Output gate SiLU(z) for the standalone pscwin_cycle_scan entry point (raw z). The module path gets SiLU(z)
// straight from the in_proj GEMM epilogue instead.
__global__ void __launch_bounds__(256) silu_gate_kernel(const __nv_bfloat16* z, long long ld_z, long long T, int D,
                                                        __nv_bfloat16* gz) {
  pdl_trigger();
  pdl_wait();
  const int dv = D / 8;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= T * dv) return;
  const long long tok = idx / dv;
  const int d0 = (int)(idx - tok * dv) * 8;
  const uint4 zv = *reinterpret_cast<const uint4*>(z + tok * ld_z + d0);
  const uint32_t* zw = reinterpret_cast<const uint32_t*>(&zv);
  uint4 g;
  uint32_t* gw = reinterpret_cast<uint32_t*>(&g);
#pragma unroll
  for (int q = 0; q < 4; ++q) gw[q] = pack_bf16(silu_f(bf16_lo(zw[q])), silu_f(bf16_hi(zw[q])));
  *reinterpret_cast<uint4*>(gz + tok * D + d0) = g;
}

// ------------------------------------------------------------------------------------------------- scan order
// pi: scan position t -> grid token index (oracle scan_permutation; reading Q13): row-major raster,
// column-major raster, or window-major (windows in raster order, raster inside each w x w window).
__device__ __forceinline__ int scan_pi(int t, int H, int W, int order, int w) {
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
    const int wx = q % nwx, wy = q / nwx;
    return (wy * w + sy) * W + wx * w + sx;
  }
  return t;
}
// Row gather (scan order <- grid order) or scatter (grid order <- scan order) of bf16 rows of D channels.
__global__ void __launch_bounds__(256) permute_rows_kernel(const __nv_bfloat16* src, long long ld_src,
                                                           __nv_bfloat16* dst, long long ld_dst, int B, int H, int W,
                                                           int D, int order, int w, int scatter) {
  pdl_trigger();
  pdl_wait();
  const int L = H * W, dv = D / 8;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)B * L * dv) return;
  const int c = (int)(idx % dv) * 8;
  const long long rr = idx / dv;
  const int b = (int)(rr / L), t = (int)(rr - (long long)b * L);
  const long long g = (long long)b * L + scan_pi(t, H, W, order, w), sq = (long long)b * L + t;
  const long long from = scatter ? sq : g, to = scatter ? g : sq;
  *reinterpret_cast<uint4*>(dst + to * ld_dst + c) = *reinterpret_cast<const uint4*>(src + from * ld_src + c);
}

int launch_permute_rows(const __nv_bfloat16* src, long long ld_src, __nv_bfloat16* dst, long long ld_dst, int B, int H,
                        int W, int D, int order, int w, int scatter, cudaStream_t s) {
  if (D % 8) return -1;
  const long long n = (long long)B * H * W * (D / 8);
  if (n == 0) return 0;
  PSCWIN_PROF(scatter ? "scan_order_scatter" : "scan_order_gather", s);
  launch_k(permute_rows_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, src, ld_src, dst, ld_dst, B, H, W, D,
           order, w, scatter);
  return (int)cudaGetLastError();
}

// Multi-scale row gather / scatter (HRSAM++ multi-scale cycle scan): sequence row (b, t) of the per-sample
// concatenation of every scale's scan-order sequence <-> packed row B*off[s] + b*L_s + pi_s(t - off[s]) of the
// scale-outermost packing (reading Q20). ncols % 8 == 0.
__global__ void __launch_bounds__(256) ms_permute_rows_kernel(const __nv_bfloat16* src, long long ld_src,
                                                              __nv_bfloat16* dst, long long ld_dst, int B, MsGeo g,
                                                              int ncols, int order, int w, int scatter) {
  pdl_trigger();
  pdl_wait();
  const int Lt = g.off[g.n], nv = ncols / 8;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)B * Lt * nv) return;
  const int c = (int)(idx % nv) * 8;
  const long long rr = idx / nv;
  const int b = (int)(rr / Lt), t = (int)(rr - (long long)b * Lt);
  int sg = 0;
#pragma unroll
  for (int q = 1; q < 4; ++q)
    if (q < g.n && t >= g.off[q]) sg = q;
  const int Hs = g.H[sg], Ws = g.W[sg];
  const long long packed =
      (long long)B * g.off[sg] + (long long)b * Hs * Ws + scan_pi(t - g.off[sg], Hs, Ws, order, w);
  const long long from = scatter ? rr : packed, to = scatter ? packed : rr;
  *reinterpret_cast<uint4*>(dst + to * ld_dst + c) = *reinterpret_cast<const uint4*>(src + from * ld_src + c);
}

// ------------------------------------------------------------------------------------------------- staging
// Per-chunk token loop with cp.async double buffering: every per-token operand (the shared (delta_low, B, C)
// row, and this CTA's slice of v, Delta, z) lands in shared memory one sub-chunk ahead of its use, so the
// sequential recurrence never waits on a global load. The state is kept scaled, h~ = A h (per (d, n) constant),
// which turns the ZOH update into h~ <- dA (h~ + w) - w with w = B_t[n] v_t (no 1/A per element), and pairs of
// states are updated with packed fp32x2 instructions (FFMA2 / FMUL2 on sm_100a).
#ifndef PSCWIN_TSUB
#define PSCWIN_TSUB 16  // tokens per staged sub-chunk of the passes (sweeps: PSCWIN_NVCC_FLAGS)
#endif
constexpr int TSUB = PSCWIN_TSUB;
// FDT (pass 1 with the dt projection fused): the whole x_proj row (delta_low | B | C) is staged at the padded stride
// W = fdt_stride(R + 2N) floats (an odd multiple of 4 mod 32: the tf32 mma's A-fragment loads hit 32 distinct banks)
// and Delta is not loaded (pass 1 computes it into the stage's Delta slot).
__host__ __device__ inline int fdt_stride(int w) {
  int s = (w + 3) & ~3;
  while ((s & 31) % 8 != 4) s += 4;
  return s;
}
template <int DPB, int NT, bool PASS2, bool FDT = false>  // DPB channels per CTA, NT threads
struct StageLayout {
  // byte offsets inside one stage buffer
  __host__ __device__ static size_t off_v(int W) { return (size_t)TSUB * W * 4; }
  __host__ __device__ static size_t off_dt(int W) { return off_v(W) + (size_t)TSUB * DPB * 2; }
  __host__ __device__ static size_t off_z(int W) { return off_dt(W) + (size_t)TSUB * DPB * 4; }
  __host__ __device__ static size_t bytes(int W) {
    size_t b = off_z(W) + (PASS2 ? (size_t)TSUB * DPB * 2 : 0);
    return (b + 127) & ~size_t(127);
  }
  // issue cp.async for tokens [t, t + nt) into stage buffer `buf`
  __device__ static void load(uint8_t* buf, const ScanParams& p, int W, long long rbase, long long tok0, int t, int nt,
                              int d0) {
    const int tid = threadIdx.x;
    // only the (B, C) columns of the x_proj rows are staged (W = 2N floats per token; delta_low is consumed by
    // the dt GEMM alone): row stride R + 2N in global memory, column offset R
    float* sd = reinterpret_cast<float*>(buf);
    __nv_bfloat16* sv = reinterpret_cast<__nv_bfloat16*>(buf + off_v(W));
    if (FDT) {  // whole rows (R + 2N floats) at stride W
      const int gw = p.R + 2 * p.N, W4 = gw / 4;
      const float* gd = p.dbc + (rbase + t) * gw;
      for (int i = tid; i < nt * W4; i += NT) {
        const int j = i / W4, q = i - j * W4;
        cp_async16(sd + j * W + 4 * q, gd + (long long)j * gw + 4 * q);
      }
    } else {
      const int gw = p.R + W, W4 = W / 4;
      const float* gd = p.dbc + (rbase + t) * gw + p.R;
      for (int i = tid; i < nt * W4; i += NT) {
        const int j = i / W4, q = i - j * W4;
        cp_async16(sd + 4 * i, gd + (long long)j * gw + 4 * q);
      }
    }
    constexpr int VPR = DPB / 8;  // 16-byte chunks per token row of bf16
    for (int i = tid; i < nt * VPR; i += NT) {
      const int j = i / VPR, cc = i - j * VPR;
      cp_async16(sv + j * DPB + cc * 8, p.v + (rbase + t + j) * p.D + d0 + cc * 8);
    }
    if (!FDT) {
      float* sdt = reinterpret_cast<float*>(buf + off_dt(W));
      constexpr int FPR = DPB / 4;
      for (int i = tid; i < nt * FPR; i += NT) {
        const int j = i / FPR, cc = i - j * FPR;
        cp_async16(sdt + j * DPB + cc * 4, p.delta + (rbase + t + j) * p.D + d0 + cc * 4);
      }
    }
    if (PASS2) {
      __nv_bfloat16* sz = reinterpret_cast<__nv_bfloat16*>(buf + off_z(W));
      if (p.gz)
        for (int i = tid; i < nt * VPR; i += NT) {
          const int j = i / VPR, cc = i - j * VPR;
          cp_async16(sz + j * DPB + cc * 8, p.gz + (tok0 + t + j) * p.ld_gz + d0 + cc * 8);
        }
    }
  }
};

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// ------------------------------------------------------------------------------------------------- dt
// Delta[row, d] = softplus(delta_low[row] . W_dt[d] + b_dt[d]) for every stream row (copy-2/3 rows and the P copy-1
// rows). Block = 64 threads x 2 channels x DT_ROWS rows: the rows' delta_low vectors are staged in shared memory
// (read back as broadcasts), each thread keeps its two channels' W_dt rows in registers as (d, d+1) pairs, so one
// packed fp32x2 FMA advances both channels, and four rows are accumulated at once (4 independent chains).
constexpr int DT_ROWS = 64;
constexpr int DT_THREADS = 64;
template <int RMAX>
__global__ void __launch_bounds__(DT_THREADS) scan_dt_kernel(ScanParams p) {
  pdl_trigger();
  pdl_wait();
  __shared__ float4 s_d4[DT_ROWS * (RMAX / 4)];
  const int W = p.R + 2 * p.N;
  const int d = blockIdx.x * (2 * DT_THREADS) + 2 * threadIdx.x;
  const long long rows = (long long)p.B * (p.L + p.P);
  const long long r0 = (long long)blockIdx.y * DT_ROWS;
  const int nr = (int)min((long long)DT_ROWS, rows - r0);
  const int R4 = p.R / 4;
  for (int i = threadIdx.x; i < nr * R4; i += DT_THREADS) {
    const int j = i / R4, q = i - j * R4;
    s_d4[j * (RMAX / 4) + q] = __ldg(reinterpret_cast<const float4*>(p.dbc + (r0 + j) * W) + q);
  }
  float2 wp[RMAX];  // (W_dt[d][k], W_dt[d+1][k])
  const bool dok = d < p.D;  // D % 64 == 0: the last block may be half used
  if (!dok) {
#pragma unroll
    for (int k = 0; k < RMAX; ++k) wp[k] = make_float2(0.f, 0.f);
  } else {
    const float4* w0 = reinterpret_cast<const float4*>(p.w_dt + (size_t)d * p.R);
    const float4* w1 = reinterpret_cast<const float4*>(p.w_dt + (size_t)(d + 1) * p.R);
#pragma unroll
    for (int q = 0; q < RMAX / 4; ++q) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), c = a;
      if (q < R4) {
        a = __ldg(w0 + q);
        c = __ldg(w1 + q);
      }
      wp[4 * q + 0] = make_float2(a.x, c.x);
      wp[4 * q + 1] = make_float2(a.y, c.y);
      wp[4 * q + 2] = make_float2(a.z, c.z);
      wp[4 * q + 3] = make_float2(a.w, c.w);
    }
  }
  const float2 bias = dok ? make_float2(p.b_dt[d], p.b_dt[d + 1]) : make_float2(0.f, 0.f);
  __syncthreads();
  if (!dok) return;
  auto softplus = [](float x) {
    // log(1 + e^x); for x < -5 the series u - u^2/2 (u = e^x < 7e-3) avoids the rounding of 1 + u
    const float u = __expf(x);
    const float sp = x < -5.f ? u * (1.f - 0.5f * u) : __logf(1.f + u);
    return x > 20.f ? x : sp;
  };
  auto store = [&](int j, float2 x) {
    *reinterpret_cast<float2*>(p.delta + (r0 + j) * p.D + d) = make_float2(softplus(x.x), softplus(x.y));
  };
  int j = 0;
  for (; j + 4 <= nr; j += 4) {
    float2 acc[4] = {bias, bias, bias, bias};
#pragma unroll
    for (int q = 0; q < RMAX / 4; ++q)
      if (q < R4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 x = s_d4[(j + i) * (RMAX / 4) + q];
          acc[i] = __ffma2_rn(f2(x.x), wp[4 * q + 0], acc[i]);
          acc[i] = __ffma2_rn(f2(x.y), wp[4 * q + 1], acc[i]);
          acc[i] = __ffma2_rn(f2(x.z), wp[4 * q + 2], acc[i]);
          acc[i] = __ffma2_rn(f2(x.w), wp[4 * q + 3], acc[i]);
        }
      }
#pragma unroll
    for (int i = 0; i < 4; ++i) store(j + i, acc[i]);
  }
  for (; j < nr; ++j) {
    float2 acc = bias;
#pragma unroll
    for (int q = 0; q < RMAX / 4; ++q)
      if (q < R4) {
        const float4 x = s_d4[j * (RMAX / 4) + q];
        acc = __ffma2_rn(f2(x.x), wp[4 * q + 0], acc);
        acc = __ffma2_rn(f2(x.y), wp[4 * q + 1], acc);
        acc = __ffma2_rn(f2(x.z), wp[4 * q + 2], acc);
        acc = __ffma2_rn(f2(x.w), wp[4 * q + 3], acc);
      }
    store(j, acc);
  }
}

// ------------------------------------------------------------------------------------------------- pass 1
// NS threads per channel, each owning NH = N / NS of its states (NS = 2 halves the registers per thread, which
// doubles the resident warps that hide the MUFU / FMA latencies).
// PK > 0: every PK-th state pair takes its decay factor from the degree-5 polynomial on the FMA pipe instead of MUFU
// ex2 (the MUFU pipe bounds the passes while the FMA pipe has slack; same accuracy, exp2_poly5x2)
template <int PK>
__device__ __forceinline__ float2 decay2(int k, float2 x) {
  if (PK > 0 && k % PK == PK - 1) return exp2_poly5x2(x);
  return make_float2(ex2_approx(x.x), ex2_approx(x.y));
}

// dt projection fused into pass 1 (FDT): Delta = softplus(delta_low W_dt^T + b_dt) (Q12) for the sub-chunk's 16
// tokens x this warp's 8 channels as TF32 tensor-core MMAs (mma.sync m16n8k8: A = the staged delta_low rows,
// B = the warp's W_dt rows held in registers as fragments), written into the stage's Delta slot for the recurrence
// and to global memory for the carry and pass 2, in place of the separate dt GEMM (whose 400 MB f32 write at 4096^2
// would happen inside a MUFU-bound kernel whose HBM is idle). Measured slower; off by default (launch_dt_pass1).
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return u;
}
__device__ __forceinline__ void mma_tf32_16x8x8(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                                uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// softplus with two MUFU: log1p(t), t = e^x, as t (1 - t/2 + t^2/3 - t^3/4 + t^4/5) below t = 1/32, else log(1 + t)
// (same formula as the dt GEMM's f32 epilogue)
__device__ __forceinline__ float softplus_dt(float x) {
  const float t = __expf(x);
  const float poly = t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, 0.2f, -0.25f), 0.33333334f), -0.5f), 1.f);
  const float lp = t < 0.03125f ? poly : __logf(1.f + t);
  return x > 20.f ? x : lp;
}
constexpr int FDT_KS = 8;  // k-steps of 8 (R <= 64)
// resident CTAs per SM the fused pass 1 is register-bounded for (4: <= 64 registers, the unfused pass 1's occupancy)
#ifndef PSCWIN_PASS1_FDT_MINB
#define PSCWIN_PASS1_FDT_MINB 4
#endif

template <int N, int DPB, int NS, bool ZOH, int PK, bool FDT = false>
__global__ void __launch_bounds__(DPB * NS, FDT ? PSCWIN_PASS1_FDT_MINB : 0) scan_pass1_kernel(ScanParams p) {
  pdl_trigger();
  pdl_wait();
  constexpr int NT = DPB * NS, NH = N / NS;
  static_assert(!FDT || (NS == 4 && DPB == 64), "fused dt: one warp = 8 channels x 4 state groups");
  using St = StageLayout<DPB, NT, false, FDT>;
  extern __shared__ __align__(128) uint8_t s_raw[];
  const int W = FDT ? fdt_stride(p.R + 2 * N) : 2 * N;  // staged row stride (floats)
  const int boff = FDT ? p.R : 0;                         // B columns inside the staged row
  const size_t SB = St::bytes(W);
  const int c = threadIdx.x / NS, sub = threadIdx.x % NS;
  const int d0 = blockIdx.x * DPB;
  const int d = d0 + c;
  const int n0 = sub * NH;
  const int chunk = blockIdx.y;
  const int b = blockIdx.z;
  const long long rbase = (long long)b * (p.L + p.P);
  float2 A2[NH / 2], h[NH / 2];
#pragma unroll
  for (int k = 0; k < NH / 2; ++k) {
    A2[k] = make_float2(-__expf(p.a_log[d * N + n0 + 2 * k]) * kLog2e, -__expf(p.a_log[d * N + n0 + 2 * k + 1]) * kLog2e);
    h[k] = make_float2(0.f, 0.f);
  }
  const int t0 = chunk * p.Lc;
  const int t1 = min(p.L, t0 + p.Lc);
  const int tb = max(t0, p.P);
  const int nsub = (t1 - tb + TSUB - 1) / TSUB;
  float sdt = 0.f;
  if (nsub > 0) {
    St::load(s_raw, p, W, rbase, 0, tb, min(TSUB, t1 - tb), d0);
    cp_async_commit();
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // FDT: the warp's B fragments (W_dt rows of its 8 channels, tf32) live in shared memory after the two stage
  // buffers, [warp][k-step][lane] pairs, reloaded per sub-chunk (kept in registers they cost the recurrence its ILP)
  uint2* s_wf = reinterpret_cast<uint2*>(s_raw + 2 * SB) + wid * (FDT_KS * 32);
  if constexpr (FDT) {
    const int g = lane >> 2, tq = lane & 3;
    const float* wr = p.w_dt + (size_t)(d0 + 8 * wid + g) * p.R;
#pragma unroll
    for (int ks = 0; ks < FDT_KS; ++ks) {
      const int r0 = 8 * ks + tq, r1 = r0 + 4;
      s_wf[ks * 32 + lane] = make_uint2(tf32_rna(r0 < p.R ? __ldg(wr + r0) : 0.f), tf32_rna(r1 < p.R ? __ldg(wr + r1) : 0.f));
    }
    __syncwarp();
    if (chunk == 0) {
      // the carry's prefix tokens, rows [0, P) (copies 2/3) and [L, L+P) (copy 1): plain dot products (delta_low
      // truncated to tf32 as the MMA reads it, W_dt rounded as its fragments), 16-byte loads all issued up front;
      // thread `sub` of each channel takes rows sub, sub + NS, ...
      const int gw = p.R + 2 * N;
      for (int i = sub; i < 2 * p.P; i += NS) {
        const long long row = rbase + (i < p.P ? i : p.L + i - p.P);
        const float4* dl = reinterpret_cast<const float4*>(p.dbc + row * gw);
        const float4* wd = reinterpret_cast<const float4*>(p.w_dt + (size_t)d * p.R);
        float acc = 0.f;
        auto tr = [](float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); };
        auto rn = [](float x) { return __uint_as_float(tf32_rna(x)); };
        for (int q0 = 0; 4 * q0 < p.R; q0 += 4) {  // four 16-byte loads of each operand in flight per round
          float4 xv[4], wv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (4 * (q0 + q) < p.R) {
              xv[q] = dl[q0 + q];
              wv[q] = __ldg(wd + q0 + q);
            }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (4 * (q0 + q) < p.R) {
              acc = fmaf(tr(xv[q].x), rn(wv[q].x), acc);
              acc = fmaf(tr(xv[q].y), rn(wv[q].y), acc);
              acc = fmaf(tr(xv[q].z), rn(wv[q].z), acc);
              acc = fmaf(tr(xv[q].w), rn(wv[q].w), acc);
            }
        }
        p.delta[row * p.D + d] = softplus_dt(acc + __ldg(p.b_dt + d));
      }
    }
  }
  const float2 m1 = f2(-1.f);
  for (int sc = 0; sc < nsub; ++sc) {
    const int ts = tb + sc * TSUB;
    const int nt = min(TSUB, t1 - ts);
    if (sc + 1 < nsub) {
      St::load(s_raw + ((sc + 1) & 1) * SB, p, W, rbase, 0, ts + TSUB, min(TSUB, t1 - ts - TSUB), d0);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    uint8_t* buf = s_raw + (sc & 1) * SB;
    const float* sdbc = reinterpret_cast<const float*>(buf);
    const __nv_bfloat16* sv = reinterpret_cast<const __nv_bfloat16*>(buf + St::off_v(W));
    float* sdelta = reinterpret_cast<float*>(buf + St::off_dt(W));
    float* sdw = sdelta + wid * (TSUB * 8);  // FDT: this warp's [TSUB][8] Delta block
    if constexpr (FDT) {
      const int g = lane >> 2, tq = lane & 3;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const int ks_n = (p.R + 7) / 8;
      const float2 bdt = make_float2(__ldg(p.b_dt + d0 + 8 * wid + 2 * tq), __ldg(p.b_dt + d0 + 8 * wid + 2 * tq + 1));
#pragma unroll
      for (int ks = 0; ks < FDT_KS; ++ks)
        if (ks < ks_n) {
          // A = the f32 bit patterns (the tensor core reads their tf32 part, as the kind::tf32 dt GEMM did): a
          // cvt.rna per element runs on the XU pipe that bounds this kernel (measured: +0.3 ms at 4096^2 with it)
          const uint32_t* a = reinterpret_cast<const uint32_t*>(sdbc) + 8 * ks + tq;
          const uint2 wf = s_wf[ks * 32 + lane];
          mma_tf32_16x8x8(acc, a[g * W], a[(g + 8) * W], a[g * W + 4], a[(g + 8) * W + 4], wf.x, wf.y);
        }
      *reinterpret_cast<float2*>(sdw + g * 8 + 2 * tq) =
          make_float2(softplus_dt(acc[0] + bdt.x), softplus_dt(acc[1] + bdt.y));
      *reinterpret_cast<float2*>(sdw + (g + 8) * 8 + 2 * tq) =
          make_float2(softplus_dt(acc[2] + bdt.x), softplus_dt(acc[3] + bdt.y));
      __syncwarp();
      const int j = lane >> 1, h4 = (lane & 1) * 4;  // Delta rows for the carry / pass 2: 32 bytes per token row
      if (j < nt)
        *reinterpret_cast<float4*>(p.delta + (rbase + ts + j) * p.D + d0 + 8 * wid + h4) =
            *reinterpret_cast<const float4*>(sdw + j * 8 + h4);
    }
    auto tstep = [&](int j) {
      const float v = __bfloat162float(sv[j * DPB + c]);
      const float dt = FDT ? sdw[j * 8 + (lane >> 2)] : sdelta[j * DPB + c];
      sdt += dt;
      const float4* b4 = reinterpret_cast<const float4*>(sdbc + j * W + boff + n0);  // two state pairs per load
      const float2 dt2 = f2(dt), nv2 = f2(-v);
#pragma unroll
      for (int k = 0; k < NH / 2; ++k) {
        const float4 bq = b4[k / 2];
        const float2 bk = (k & 1) ? make_float2(bq.z, bq.w) : make_float2(bq.x, bq.y);
        const float2 x = __fmul2_rn(dt2, A2[k]);
        const float2 dA = decay2<PK>(k, x);
        const float2 wn = __fmul2_rn(bk, nv2);                    // -w = -B v
        if (ZOH) {
          const float2 t = __ffma2_rn(wn, m1, h[k]);               // h~ + w
          h[k] = __ffma2_rn(dA, t, wn);                            // dA (h~ + w) - w
        } else {
          const float2 u = __fmul2_rn(__fmul2_rn(x, f2(0.69314718055994531f)), wn);  // -(Delta A) B v
          h[k] = __ffma2_rn(dA, h[k], __fmul2_rn(u, m1));
        }
      }
    };
    if (nt == TSUB) {  // full sub-chunk: unrolled (constant smem offsets, no per-step index math)
#pragma unroll
      for (int j = 0; j < TSUB; ++j) tstep(j);
    } else {
      for (int j = 0; j < nt; ++j) tstep(j);
    }
    __syncthreads();
  }
  if (sub == 0) p.sumdt[((long long)b * p.n_chunks + chunk) * p.D + d] = sdt;
  float4* dst = reinterpret_cast<float4*>(p.hs + (((long long)b * p.n_chunks + chunk) * p.D + d) * N + n0);
#pragma unroll
  for (int k = 0; k < NH / 2; k += 2) dst[k / 2] = make_float4(h[k].x, h[k].y, h[k + 1].x, h[k + 1].y);
}

// ------------------------------------------------------------------------------------------------- carry
// One warp per (image, channel); lane owns states n = lane + 32 j (scaled states h~ = A h throughout).
// Produces the prefix outputs and every chunk's entry state (overwriting the pass-1 chunk-end states).
// The warp's chunk summaries (sum of Delta, chunk-end states) are copied to shared memory asynchronously up front,
// so the two sequential folds over the chunks run from shared memory instead of one global round trip per batch.
template <int N>
__global__ void __launch_bounds__(256) scan_carry_kernel(ScanParams p) {
  pdl_trigger();
  pdl_wait();
  constexpr int NPL = (N + 31) / 32;
  extern __shared__ __align__(16) float s_carry[];
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp_global >= p.B * p.D) return;
  const int b = warp_global / p.D;
  const int d = warp_global - b * p.D;
  const int W = p.R + 2 * N;
  const int nch = p.n_chunks;
  float* s_sd = s_carry + (threadIdx.x >> 5) * nch * (N + 1);  // [nch] sum of Delta per chunk
  float* s_hs = s_sd + nch;                                    // [nch][N] chunk-end states from zero
  const float* sd = p.sumdt + (long long)b * nch * p.D + d;
  float* hs = p.hs + ((long long)b * nch * p.D + d) * N;
  for (int c = lane; c < nch; c += 32) cp_async4(s_sd + c, sd + (long long)c * p.D);
  for (int c = 0; c < nch; ++c)
#pragma unroll
    for (int j = 0; j < NPL; ++j)
      if (lane + 32 * j < N) cp_async4(s_hs + c * N + lane + 32 * j, hs + (long long)c * p.D * N + lane + 32 * j);
  cp_async_commit();
  const long long rbase = (long long)b * (p.L + p.P);
  const bool zoh = p.bbar == 0;
  float A2[NPL], invA[NPL];
  bool act[NPL];
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    const int n = lane + 32 * j;
    act[j] = n < N;
    const float A = act[j] ? -__expf(p.a_log[d * N + n]) : -1.f;
    A2[j] = A * kLog2e;
    invA[j] = 1.f / A;
  }
  // The P <= KMAX - 1 prefix rows of copy 1 (r1 = L + t) and of copies 2/3 (r2 = t) are read once, all up front
  // (independent loads in flight together, overlapping the summaries' cp.async), instead of one dependent global
  // round trip per recurrence step.
  constexpr int PM = KMAX - 1;
  float pdt1[PM], pdt2[PM], pv1[PM], pv2[PM], pb1[PM][NPL], pb2[PM][NPL], pc1[PM][NPL], pc2[PM][NPL], pg[PM];
#pragma unroll
  for (int t = 0; t < PM; ++t) {
    if (t >= p.P) break;
    const long long r1 = rbase + p.L + t, r2 = rbase + t;
    pdt1[t] = p.delta[r1 * p.D + d];
    pdt2[t] = p.delta[r2 * p.D + d];
    pv1[t] = __bfloat162float(p.v[r1 * p.D + d]);
    pv2[t] = __bfloat162float(p.v[r2 * p.D + d]);
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      const int n = act[j] ? lane + 32 * j : 0;
      pb1[t][j] = p.dbc[r1 * W + p.R + n];
      pb2[t][j] = p.dbc[r2 * W + p.R + n];
      pc1[t][j] = p.dbc[r1 * W + p.R + N + n];
      pc2[t][j] = p.dbc[r2 * W + p.R + N + n];
    }
    pg[t] = p.gz ? __bfloat162float(p.gz[((long long)b * p.L + t) * p.ld_gz + d]) : 1.f;
  }
  auto step = [&](float (&h)[NPL], float dt, float v, const float (&bv)[NPL]) {
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      if (!act[j]) continue;
      const float w = bv[j] * v;
      const float x = dt * A2[j];
      const float dA = ex2_approx(x);
      h[j] = zoh ? fmaf(dA, h[j] + w, -w) : fmaf(dA, h[j], x * 0.69314718055994531f * w);
    }
  };
  // copy prefixes (P tokens): beta1 = copy 1 from zero, beta2 = copies 2/3 from zero, alpha2 = their decay
  float beta1[NPL], beta2[NPL], alpha2[NPL];
#pragma unroll
  for (int j = 0; j < NPL; ++j) beta1[j] = beta2[j] = 0.f;
  float sdt2 = 0.f;
#pragma unroll
  for (int t = 0; t < PM; ++t) {
    if (t >= p.P) break;
    step(beta1, pdt1[t], pv1[t], pb1[t]);
    step(beta2, pdt2[t], pv2[t], pb2[t]);
    sdt2 += pdt2[t];
  }
#pragma unroll
  for (int j = 0; j < NPL; ++j) alpha2[j] = ex2_approx(sdt2 * A2[j]);
  cp_async_wait<0>();
  __syncwarp();
  // body from zero (input x1): Bb = fold of (exp(A sum Delta_c), b_c) over the chunks
  float Bb[NPL], sall = 0.f;
#pragma unroll
  for (int j = 0; j < NPL; ++j) Bb[j] = 0.f;
  for (int c = 0; c < nch; ++c) {
    const float sc = s_sd[c];
    sall += sc;
#pragma unroll
    for (int j = 0; j < NPL; ++j)
      if (act[j]) Bb[j] = fmaf(ex2_approx(sc * A2[j]), Bb[j], s_hs[c * N + lane + 32 * j]);
  }
  float c2[NPL], c3[NPL], H[NPL];
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    const float Ab = ex2_approx(sall * A2[j]);
    c2[j] = fmaf(Ab, beta1[j], Bb[j]);
    const float e2 = fmaf(alpha2[j], c2[j], beta2[j]);
    c3[j] = fmaf(Ab, e2, Bb[j]);
    const float e3 = fmaf(alpha2[j], c3[j], beta2[j]);
    H[j] = beta1[j] + e2 + e3;
  }
  {  // prefix outputs: out_t = (sum_copies C^(c)_t . h^(c)_t + D (v1_t + 2 v2_t)) * SiLU(z_t)
    float h1[NPL], h2[NPL], h3[NPL];
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      h1[j] = 0.f;
      h2[j] = c2[j];
      h3[j] = c3[j];
    }
    const float Ds = p.d_skip[d];
#pragma unroll
    for (int t = 0; t < PM; ++t) {
      if (t >= p.P) break;
      step(h1, pdt1[t], pv1[t], pb1[t]);
      step(h2, pdt2[t], pv2[t], pb2[t]);
      step(h3, pdt2[t], pv2[t], pb2[t]);
      float y = 0.f;
#pragma unroll
      for (int j = 0; j < NPL; ++j)
        if (act[j]) y += invA[j] * (pc1[t][j] * h1[j] + pc2[t][j] * (h2[j] + h3[j]));
#pragma unroll
      for (int o = 16; o; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
      if (lane == 0) {
        y += Ds * (pv1[t] + 2.f * pv2[t]);
        p.out[((long long)b * p.L + t) * p.ld_out + d] = __float2bfloat16_rn(y * pg[t]);
      }
    }
  }
  // chunk entry states of the summed recurrence (input x3): H_in(0) = H_{P-1}; H_in(c+1) = a_c H_in(c) + 3 b_c
  for (int c = 0; c < nch; ++c) {
    const float sc = s_sd[c];
#pragma unroll
    for (int j = 0; j < NPL; ++j)
      if (act[j]) {
        hs[(long long)c * p.D * N + lane + 32 * j] = H[j];
        H[j] = fmaf(ex2_approx(sc * A2[j]), H[j], 3.f * s_hs[c * N + lane + 32 * j]);
      }
  }
}

// ------------------------------------------------------------------------------------------------- band mode
// Window-row sharding of one image: rank g owns the contiguous scan segment of its
// token rows. After pass 1 each rank reduces its chunks to a segment record; the records of all ranks are
// all-gathered (NCCL); every rank then folds them locally to its segment's entry state.
// Record layout (floats): [D] sum of Delta over the segment body | [D][N] segment end state from zero (input x1)
//                         | [D] sum of Delta over the copy-2/3 prefix | [D][N] beta1 | [D][N] beta2
// (the last three from rank 0 only — it holds the P = k-1 prefix tokens; other ranks write zeros).
__host__ __device__ inline size_t band_record_floats(int D, int N) { return (size_t)D * (2 + 3 * (size_t)N); }

template <int N>
__global__ void __launch_bounds__(256) scan_segment_kernel(ScanParams p, float* rec) {
  pdl_trigger();
  pdl_wait();
  constexpr int NPL = (N + 31) / 32;
  const int d = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (d >= p.D) return;  // B = 1 in band mode
  const int W = p.R + 2 * N;
  const bool zoh = p.bbar == 0;
  float A2[NPL];
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    const int n = lane + 32 * j;
    A2[j] = n < N ? -__expf(p.a_log[d * N + n]) * kLog2e : 0.f;
  }
  float* r_sdt = rec;
  float* r_b = rec + p.D;
  float* r_sdt2 = r_b + (size_t)p.D * N;
  float* r_b1 = r_sdt2 + p.D;
  float* r_b2 = r_b1 + (size_t)p.D * N;
  // segment end state from zero and sum of Delta: fold of the chunk summaries
  float Bb[NPL], sall = 0.f;
#pragma unroll
  for (int j = 0; j < NPL; ++j) Bb[j] = 0.f;
  for (int c = 0; c < p.n_chunks; ++c) {
    const float sc = p.sumdt[(long long)c * p.D + d];
    sall += sc;
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      const int n = lane + 32 * j;
      if (n < N) Bb[j] = fmaf(ex2_approx(sc * A2[j]), Bb[j], p.hs[((long long)c * p.D + d) * N + n]);
    }
  }
  if (lane == 0) r_sdt[d] = sall;
#pragma unroll
  for (int j = 0; j < NPL; ++j)
    if (lane + 32 * j < N) r_b[(size_t)d * N + lane + 32 * j] = Bb[j];
  // copy prefixes (rank 0): beta1 = copy 1 from zero over rows [L, L+P), beta2 = copies 2/3 over rows [0, P)
  float b1[NPL], b2[NPL], sdt2 = 0.f;
#pragma unroll
  for (int j = 0; j < NPL; ++j) b1[j] = b2[j] = 0.f;
  auto step = [&](float (&h)[NPL], long long row) {
    const float dt = p.delta[row * p.D + d];
    const float v = __bfloat162float(p.v[row * p.D + d]);
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      const int n = lane + 32 * j;
      if (n >= N) continue;
      const float w = p.dbc[row * W + p.R + n] * v;
      const float x = dt * A2[j];
      const float dA = ex2_approx(x);
      h[j] = zoh ? fmaf(dA, h[j] + w, -w) : fmaf(dA, h[j], x * 0.69314718055994531f * w);
    }
  };
  for (int t = 0; t < p.P; ++t) {
    step(b1, p.L + t);
    step(b2, t);
    sdt2 += p.delta[(long long)t * p.D + d];
  }
  if (lane == 0) r_sdt2[d] = sdt2;
#pragma unroll
  for (int j = 0; j < NPL; ++j)
    if (lane + 32 * j < N) {
      r_b1[(size_t)d * N + lane + 32 * j] = b1[j];
      r_b2[(size_t)d * N + lane + 32 * j] = b2[j];
    }
}

// Entry states of this rank's chunks from the all-gathered records (recs [world][record]); rank 0 also writes the
// prefix outputs. Same algebra as scan_carry_kernel with the fold running over ranks first, then own chunks.
template <int N>
__global__ void __launch_bounds__(256) scan_dist_carry_kernel(ScanParams p, const float* recs, int rank, int world) {
  pdl_trigger();
  pdl_wait();
  constexpr int NPL = (N + 31) / 32;
  const int d = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (d >= p.D) return;
  const int W = p.R + 2 * N;
  const bool zoh = p.bbar == 0;
  const size_t RF = band_record_floats(p.D, N);
  float A2[NPL], invA[NPL];
  bool act[NPL];
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    const int n = lane + 32 * j;
    act[j] = n < N;
    const float A = act[j] ? -__expf(p.a_log[d * N + n]) : -1.f;
    A2[j] = A * kLog2e;
    invA[j] = 1.f / A;
  }
  auto rec_sdt = [&](int g) { return recs[g * RF + d]; };
  auto rec_b = [&](int g, int j) { return recs[g * RF + p.D + (size_t)d * N + lane + 32 * j]; };
  const float* r0 = recs;  // rank 0's prefix parts
  const float sdt2 = r0[p.D + (size_t)p.D * N + d];
  float beta1[NPL], beta2[NPL], alpha2[NPL];
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    beta1[j] = act[j] ? r0[2 * p.D + (size_t)p.D * N + (size_t)d * N + lane + 32 * j] : 0.f;
    beta2[j] = act[j] ? r0[2 * p.D + 2 * (size_t)p.D * N + (size_t)d * N + lane + 32 * j] : 0.f;
    alpha2[j] = ex2_approx(sdt2 * A2[j]);
  }
  // body from zero (input x1) over all segments in rank order
  float Bb[NPL], sall = 0.f;
#pragma unroll
  for (int j = 0; j < NPL; ++j) Bb[j] = 0.f;
  for (int g = 0; g < world; ++g) {
    const float sg = rec_sdt(g);
    sall += sg;
#pragma unroll
    for (int j = 0; j < NPL; ++j)
      if (act[j]) Bb[j] = fmaf(ex2_approx(sg * A2[j]), Bb[j], rec_b(g, j));
  }
  float c2[NPL], c3[NPL], H[NPL];
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    const float Ab = ex2_approx(sall * A2[j]);
    c2[j] = fmaf(Ab, beta1[j], Bb[j]);
    const float e2 = fmaf(alpha2[j], c2[j], beta2[j]);
    c3[j] = fmaf(Ab, e2, Bb[j]);
    const float e3 = fmaf(alpha2[j], c3[j], beta2[j]);
    H[j] = beta1[j] + e2 + e3;
  }
  auto step = [&](float (&h)[NPL], long long row) {
    const float dt = p.delta[row * p.D + d];
    const float v = __bfloat162float(p.v[row * p.D + d]);
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      if (!act[j]) continue;
      const float w = p.dbc[row * W + p.R + lane + 32 * j] * v;
      const float x = dt * A2[j];
      const float dA = ex2_approx(x);
      h[j] = zoh ? fmaf(dA, h[j] + w, -w) : fmaf(dA, h[j], x * 0.69314718055994531f * w);
    }
  };
  if (rank == 0) {  // prefix outputs: out_t = (sum_copies C^(c)_t . h^(c)_t + D (v1_t + 2 v2_t)) * SiLU(z_t)
    float h1[NPL], h2[NPL], h3[NPL];
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      h1[j] = 0.f;
      h2[j] = c2[j];
      h3[j] = c3[j];
    }
    const float Ds = p.d_skip[d];
    for (int t = 0; t < p.P; ++t) {
      const long long r1 = p.L + t, r2 = t;
      step(h1, r1);
      step(h2, r2);
      step(h3, r2);
      float y = 0.f;
#pragma unroll
      for (int j = 0; j < NPL; ++j)
        if (act[j]) {
          const int n = lane + 32 * j;
          y += invA[j] * (p.dbc[r1 * W + p.R + N + n] * h1[j] + p.dbc[r2 * W + p.R + N + n] * (h2[j] + h3[j]));
        }
#pragma unroll
      for (int o = 16; o; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
      if (lane == 0) {
        y += Ds * (__bfloat162float(p.v[r1 * p.D + d]) + 2.f * __bfloat162float(p.v[r2 * p.D + d]));
        const float g = p.gz ? __bfloat162float(p.gz[(long long)t * p.ld_gz + d]) : 1.f;
        p.out[(long long)t * p.ld_out + d] = __float2bfloat16_rn(y * g);
      }
    }
  }
  // entry state of this rank's segment: fold of the earlier segments (input x3)
  for (int g = 0; g < rank; ++g) {
    const float sg = rec_sdt(g);
#pragma unroll
    for (int j = 0; j < NPL; ++j)
      if (act[j]) H[j] = fmaf(ex2_approx(sg * A2[j]), H[j], 3.f * rec_b(g, j));
  }
  // and of every own chunk (overwriting the pass-1 chunk-end states with chunk entry states)
  for (int c = 0; c < p.n_chunks; ++c) {
    const float sc = p.sumdt[(long long)c * p.D + d];
#pragma unroll
    for (int j = 0; j < NPL; ++j)
      if (act[j]) {
        const long long idx = ((long long)c * p.D + d) * N + lane + 32 * j;
        const float hb = p.hs[idx];
        p.hs[idx] = H[j];
        H[j] = fmaf(ex2_approx(sc * A2[j]), H[j], 3.f * hb);
      }
  }
}

// ------------------------------------------------------------------------------------------------- pass 2
#ifndef PSCWIN_P2_UNROLL
#define PSCWIN_P2_UNROLL 8
#endif
constexpr int kP2Unroll = PSCWIN_P2_UNROLL;  // (#pragma unroll takes a constant expression, not a macro)
// resident CTAs per SM the register allocation of the NS = 2 pass 2 is sized for, and its token unroll. Swept on
// B200 (PSCWIN_NVCC_FLAGS rebuilds): 4 CTAs (<= 128 registers) with 8-token unroll beats 5 CTAs / 96 registers
// (1024^2 82.2 -> 78.4 us, 4096^2 1.047 -> 1.005 ms); 3 and 6 CTAs / SM and unroll 2 / 16 are slower or equal.
#ifndef PSCWIN_PASS2_MINB
#define PSCWIN_PASS2_MINB 4
#endif
template <int N, int DPB, int NS, bool ZOH, int PK>
__global__ void __launch_bounds__(DPB * NS, NS == 2 ? PSCWIN_PASS2_MINB : 1) scan_pass2_kernel(ScanParams p) {
  pdl_trigger();
  pdl_wait();
  constexpr int NT = DPB * NS, NH = N / NS;
  using St = StageLayout<DPB, NT, true>;
  extern __shared__ __align__(128) uint8_t s_raw[];
  const int W = 2 * N;  // staged (B, C) row
  const size_t SB = St::bytes(W);
  const int c = threadIdx.x / NS, sub = threadIdx.x % NS;
  const int d0 = blockIdx.x * DPB;
  const int d = d0 + c;
  const int n0 = sub * NH;
  const int chunk = blockIdx.y;
  const int b = blockIdx.z;
  const long long rbase = (long long)b * (p.L + p.P);
  const long long tok0 = (long long)b * p.L;
  float2 A2[NH / 2], invA[NH / 2], h[NH / 2];
  const float4* src = reinterpret_cast<const float4*>(p.hs + (((long long)b * p.n_chunks + chunk) * p.D + d) * N + n0);
#pragma unroll
  for (int k = 0; k < NH / 2; k += 2) {
    const float4 q = src[k / 2];
    h[k] = make_float2(q.x, q.y);
    h[k + 1] = make_float2(q.z, q.w);
  }
#pragma unroll
  for (int k = 0; k < NH / 2; ++k) {
    const float a0 = -__expf(p.a_log[d * N + n0 + 2 * k]), a1 = -__expf(p.a_log[d * N + n0 + 2 * k + 1]);
    A2[k] = make_float2(a0 * kLog2e, a1 * kLog2e);
    invA[k] = make_float2(__frcp_rn(a0), __frcp_rn(a1));
  }
  const float D3 = 3.f * p.d_skip[d];
  const int t0 = chunk * p.Lc;
  const int t1 = min(p.L, t0 + p.Lc);
  const int tb = max(t0, p.P);
  const int nsub = (t1 - tb + TSUB - 1) / TSUB;
  if (nsub > 0) {
    St::load(s_raw, p, W, rbase, tok0, tb, min(TSUB, t1 - tb), d0);
    cp_async_commit();
  }
  const float2 m1 = f2(-1.f);
  for (int sc = 0; sc < nsub; ++sc) {
    const int ts = tb + sc * TSUB;
    const int nt = min(TSUB, t1 - ts);
    if (sc + 1 < nsub) {
      St::load(s_raw + ((sc + 1) & 1) * SB, p, W, rbase, tok0, ts + TSUB, min(TSUB, t1 - ts - TSUB), d0);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint8_t* buf = s_raw + (sc & 1) * SB;
    const float* sdbc = reinterpret_cast<const float*>(buf);
    const __nv_bfloat16* sv = reinterpret_cast<const __nv_bfloat16*>(buf + St::off_v(W));
    const float* sdt = reinterpret_cast<const float*>(buf + St::off_dt(W));
    const __nv_bfloat16* sz = reinterpret_cast<const __nv_bfloat16*>(buf + St::off_z(W));
    // NS > 1: this thread's partial C . h per token goes to shared memory [TSUB][NS][DPB + 32 / NS] (the padding
    // puts the NS sub-rows of a warp's channels in disjoint banks)
    constexpr int RSTR = DPB + 32 / NS;
    float* red = reinterpret_cast<float*>(s_raw + 2 * SB);
    auto tstep = [&](int j) {
      const float4* b4 = reinterpret_cast<const float4*>(sdbc + j * W + n0);      // B pairs
      const float4* c4 = reinterpret_cast<const float4*>(sdbc + j * W + N + n0);  // C pairs
      const float v = __bfloat162float(sv[j * DPB + c]);
      const float dt = sdt[j * DPB + c];
      const float2 dt2 = f2(dt), nv3 = f2(-3.f * v);
      float2 y2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};  // two chains: shorter FFMA2 dependency
#pragma unroll
      for (int k = 0; k < NH / 2; ++k) {
        const float4 bq = b4[k / 2], cq = c4[k / 2];
        const float2 bk = (k & 1) ? make_float2(bq.z, bq.w) : make_float2(bq.x, bq.y);
        const float2 ck = (k & 1) ? make_float2(cq.z, cq.w) : make_float2(cq.x, cq.y);
        const float2 x = __fmul2_rn(dt2, A2[k]);
        const float2 dA = decay2<PK>(k, x);
        const float2 wn = __fmul2_rn(bk, nv3);                    // -3 B v
        if (ZOH) {
          const float2 t = __ffma2_rn(wn, m1, h[k]);
          h[k] = __ffma2_rn(dA, t, wn);
        } else {
          const float2 u = __fmul2_rn(__fmul2_rn(x, f2(0.69314718055994531f)), wn);
          h[k] = __ffma2_rn(dA, h[k], __fmul2_rn(u, m1));
        }
        y2[k & 1] = __ffma2_rn(__fmul2_rn(ck, invA[k]), h[k], y2[k & 1]);  // C . h = C . (h~ / A)
      }
      const float y = (y2[0].x + y2[1].x) + (y2[0].y + y2[1].y);
      if constexpr (NS > 1) {
        red[(j * NS + sub) * RSTR + c] = y;  // combined across the channel's NS threads once per sub-chunk
      } else {
        const float g = p.gz ? __bfloat162float(sz[j * DPB + c]) : 1.f;
        p.out[(tok0 + ts + j) * p.ld_out + d] = __float2bfloat16_rn(fmaf(D3, v, y) * g);
      }
    };
    if (nt == TSUB) {  // full sub-chunk: partially unrolled (PSCWIN_P2_UNROLL: A/B experiments via PSCWIN_NVCC_FLAGS)
#pragma unroll kP2Unroll
      for (int j = 0; j < TSUB; ++j) tstep(j);
    } else {
      for (int j = 0; j < nt; ++j) tstep(j);
    }
    if (NS == 2 && TSUB * DPB / 8 == NT && p.vec_out) {
      // deferred reduction, vectorised: thread (token j = tid / 8, channel group cg = tid % 8) finishes 8 channels of
      // one token from shared memory (partials of both state halves, v, gate: 16-byte reads) and writes them with
      // one 16-byte store (ld_out % 8 == 0 is checked on the host; the per-channel 2-byte stores were ~7 % of the
      // kernel's stall samples, ncu r02f)
      __syncthreads();
      const int j = threadIdx.x >> 3, cg = (threadIdx.x & 7) * 8;
      if (j < nt) {
        const float4* r0 = reinterpret_cast<const float4*>(red + (j * NS) * RSTR + cg);
        const float4* r1 = reinterpret_cast<const float4*>(red + (j * NS + 1) * RSTR + cg);
        const float4 a0 = r0[0], a1 = r0[1], b0 = r1[0], b1 = r1[1];
        const float y[8] = {a0.x + b0.x, a0.y + b0.y, a0.z + b0.z, a0.w + b0.w,
                            a1.x + b1.x, a1.y + b1.y, a1.z + b1.z, a1.w + b1.w};
        const uint4 vv = *reinterpret_cast<const uint4*>(sv + j * DPB + cg);
        const uint4 gg = p.gz ? *reinterpret_cast<const uint4*>(sz + j * DPB + cg)
                              : make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);  // bf16 1.0
        const float4 k0 = __ldg(reinterpret_cast<const float4*>(p.d_skip + d0 + cg));  // (L1-resident)
        const float4 k1 = __ldg(reinterpret_cast<const float4*>(p.d_skip + d0 + cg + 4));
        const float d3v[8] = {3.f * k0.x, 3.f * k0.y, 3.f * k0.z, 3.f * k0.w, 3.f * k1.x, 3.f * k1.y, 3.f * k1.z, 3.f * k1.w};
        const uint32_t* vw = reinterpret_cast<const uint32_t*>(&vv);
        const uint32_t* gw = reinterpret_cast<const uint32_t*>(&gg);
        uint4 o;
        uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          ow[q] = pack_bf16(fmaf(d3v[2 * q], bf16_lo(vw[q]), y[2 * q]) * bf16_lo(gw[q]),
                            fmaf(d3v[2 * q + 1], bf16_hi(vw[q]), y[2 * q + 1]) * bf16_hi(gw[q]));
        *reinterpret_cast<uint4*>(p.out + (tok0 + ts + j) * p.ld_out + d0 + cg) = o;
      }
    } else if constexpr (NS > 1) {
      // deferred reduction: partial sums to shared memory, then thread `sub` of each channel finishes the tokens
      // j = sub, sub + NS, ... (y = sum of the NS partials + 3 D v, gate, bf16 store)
      __syncthreads();
#pragma unroll
      for (int j0 = 0; j0 < TSUB; j0 += NS) {
        const int j = j0 + sub;
        if (j < nt) {
          float y = 0.f;
#pragma unroll
          for (int s2 = 0; s2 < NS; ++s2) y += red[(j * NS + s2) * RSTR + c];
          const float v = __bfloat162float(sv[j * DPB + c]);
          const float g = p.gz ? __bfloat162float(sz[j * DPB + c]) : 1.f;
          p.out[(tok0 + ts + j) * p.ld_out + d] = __float2bfloat16_rn(fmaf(D3, v, y) * g);
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------------- host
struct ScanPlan {
  int P, Lc, n_chunks, W, xsplits;
  size_t v, dbc, delta, sumdt, hs, gz, partial, sem, total;
};

static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// channels per CTA of the passes and threads per channel (the chunk plan depends on them)
constexpr int PASS_DPB = 64;
// threads per channel of the passes (each owns N / NS states). Measured at ViT-B 1024^2: pass 1 is fastest with
// NS = 4 (more warps, MUFU-bound), pass 2 with NS = 2 since its output reduction is deferred to one shared-memory
// combine per 16-token sub-chunk (82 vs 85 us at 1024^2, 1.04 vs 1.08 ms at 4096^2 with two waves). PSCWIN_SCAN_NS1 / PSCWIN_SCAN_NS2 = 1, 2 or 4 override (tuning knobs).
static int ns_env(const char* name, int dflt) {
  const char* e = getenv(name);
  const int v = e ? atoi(e) : dflt;
  return (v == 1 || v == 2 || v == 4) ? v : dflt;
}
static int pass1_ns() {
  static int ns = 0;
  if (!ns) ns = ns_env("PSCWIN_SCAN_NS1", 4);
  return ns;
}
static int pass_ns() {
  static int ns = 0;
  if (!ns) ns = ns_env("PSCWIN_SCAN_NS2", 2);
  return ns;
}

// Polynomial-exp2 period (state pairs) of the ZOH passes: every PK-th pair's decay factors come from the FMA pipe
// (decay2). PSCWIN_SCAN_POLY1 / PSCWIN_SCAN_POLY2 override (0 = all MUFU; pass 1: 2 or 4, pass 2: 4 or 8).
static int pk_env(const char* name, int dflt, int a, int b) {
  const char* e = getenv(name);
  const int v = e ? atoi(e) : dflt;
  return (v == 0 || v == a || v == b) ? v : dflt;
}
static int pass1_pk() {
  static int pk = -1;
  if (pk < 0) pk = pk_env("PSCWIN_SCAN_POLY1", 0, 2, 4);
  return pk;
}
static int pass2_pk() {
  static int pk = -1;
  if (pk < 0) pk = pk_env("PSCWIN_SCAN_POLY2", 0, 4, 8);
  return pk;
}

// pass-2 dynamic shared memory: two stage buffers (+ the [DPB][NS][TSUB] partial sums when NS > 1)
template <int NS>
static size_t pass2_smem(int W) {
  return 2 * StageLayout<PASS_DPB, PASS_DPB * NS, true>::bytes(W) +
         (NS > 1 ? (size_t)(PASS_DPB + 32 / NS) * NS * TSUB * 4 : 0);
}

template <int N, int NS>
static int pass2_slots_t(int W) {
  int n = 0;
  const size_t smem = pass2_smem<NS>(W);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, scan_pass2_kernel<N, PASS_DPB, NS, true, 0>,
                                                                PASS_DPB * NS, smem);
  if (e != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = 4;
  }
  return n;
}
template <int N>
static int pass2_slots_n(int W) {
  const int ns = pass_ns();
  return ns == 1 ? pass2_slots_t<N, 1>(W) : (ns == 4 ? pass2_slots_t<N, 4>(W) : pass2_slots_t<N, 2>(W));
}
// Pass-2 CTAs resident per SM (occupancy query; a fixed fallback without a device).
static int pass2_slots(int N, int W) {
  return N == 16 ? pass2_slots_n<16>(W) : (N == 32 ? pass2_slots_n<32>(W) : pass2_slots_n<64>(W));
}

// Chunk length: the (chunk, channel block) CTAs of a pass fill every SM's resident slots exactly `waves` times
// (one wave by default: all CTAs run concurrently and finish together). PSCWIN_SCAN_WAVES overrides the target
// (tuning knob; the result does not depend on the chunking beyond fp32 rounding order).
static int choose_chunk(int B, int L, int D, int N, int W) {
  static int waves = 0;
  if (!waves) {
    const char* e = getenv("PSCWIN_SCAN_WAVES");
    waves = e ? atoi(e) : 0;  // 0 = automatic: two waves for long sequences (chunks stay >= 256 tokens)
    if (waves < 0) waves = 0;
  }
  const int wv = waves ? waves : (L >= 32768 ? 2 : 1);
  int sms = 148;
  {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      sms = v;
    else
      cudaGetLastError();
  }
  const long long cblocks = (long long)B * (D / PASS_DPB);
  long long target_chunks = (long long)wv * sms * pass2_slots(N, W) / cblocks;
  if (target_chunks < 1) target_chunks = 1;
  const long long max_chunks = (48 * 1024) / ((long long)(N + 1) * 4);  // the carry stages one warp's summaries
  if (target_chunks > max_chunks) target_chunks = max_chunks;
  long long lc = (L + target_chunks - 1) / target_chunks;
  if (lc < TSUB) lc = TSUB;
  return (int)lc;
}

static ScanPlan plan_scan_p(int B, int L, int D, int N, int R, int k, int P) {
  ScanPlan s;
  s.P = P;
  s.Lc = choose_chunk(B, L, D, N, 2 * N);  // staged (B, C) row width
  s.n_chunks = (L + s.Lc - 1) / s.Lc;
  s.W = R + 2 * N;
  const size_t rows = (size_t)B * (L + s.P);
  size_t off = 0;
  s.v = off;
  off += al256(rows * D * 2);
  s.dbc = off;
  off += al256(rows * s.W * 4);
  s.delta = off;
  off += al256(rows * (size_t)D * 4);
  s.sumdt = off;
  off += al256((size_t)B * s.n_chunks * D * 4);
  s.hs = off;
  off += al256((size_t)B * s.n_chunks * D * N * 4);
  s.gz = off;
  off += al256((size_t)B * L * D * 2);
  // x_proj split-K (measured: the partial round trip costs more than the idle SMs it fills, so off by default)
  const int m_tiles = (int)((rows + 127) / 128);
  s.xsplits = 1;
  static const int xsplit_knob = env_knob("PSCWIN_XPROJ_SPLITS", 1);  // tuning knob (1..8)
  if (xsplit_knob >= 1 && xsplit_knob <= 8) {
    s.xsplits = xsplit_knob;
    if (s.xsplits > D / 64) s.xsplits = D / 64 > 0 ? D / 64 : 1;  // every split needs >= 1 K block (D / 64 of them)
  }
  s.partial = off;
  off += s.xsplits > 1 ? al256((size_t)s.xsplits * rows * s.W * 4) : 0;
  s.sem = off;
  off += al256((size_t)m_tiles * sizeof(int));
  s.total = off;
  return s;
}
static ScanPlan plan_scan(int B, int L, int D, int N, int R, int k) { return plan_scan_p(B, L, D, N, R, k, k - 1); }

static int check_scan(int B, int L, int D, int N, int R, int k) {
  if (B <= 0 || L <= 0 || D <= 0 || N <= 0 || R <= 0 || k <= 0) return PSCWIN_ERR_SHAPE;
  if (L < k - 1) return PSCWIN_ERR_CONTRACT;  // copies 2 and 3 must see a full history
  if (!(N == 16 || N == 32 || N == 64)) return PSCWIN_ERR_UNSUPPORTED;
  if (R > 64 || R % 4 || k > 4) return PSCWIN_ERR_UNSUPPORTED;  // float4 smem rows, register conv window
  if (D % 64) return PSCWIN_ERR_UNSUPPORTED;  // x_proj GEMM K tiles
  return PSCWIN_OK;
}

template <int N, int NS>
static void launch_pass1(ScanParams& p, cudaStream_t s, bool fdt = false) {
  const dim3 grid(p.D / PASS_DPB, p.n_chunks, p.B);
  if constexpr (NS == 4) {
    if (fdt) {
      const size_t smem = 2 * StageLayout<PASS_DPB, PASS_DPB * NS, false, true>::bytes(fdt_stride(p.R + 2 * N)) +
                          (size_t)(PASS_DPB * NS / 32) * FDT_KS * 32 * sizeof(uint2);  // + the W_dt fragments
      if (p.bbar != 0)
        launch_k_even(scan_pass1_kernel<N, PASS_DPB, NS, false, 0, true>, grid, dim3(PASS_DPB * NS), smem, s, p);
      else
        launch_k_even(scan_pass1_kernel<N, PASS_DPB, NS, true, 0, true>, grid, dim3(PASS_DPB * NS), smem, s, p);
      return;
    }
  }
  const size_t smem = 2 * StageLayout<PASS_DPB, PASS_DPB * NS, false>::bytes(2 * N);
  const int pk = pass1_pk();
  if (p.bbar != 0)
    launch_k_even(scan_pass1_kernel<N, PASS_DPB, NS, false, 0>, grid, dim3(PASS_DPB * NS), smem, s, p);
  else if (pk == 2)
    launch_k_even(scan_pass1_kernel<N, PASS_DPB, NS, true, 2>, grid, dim3(PASS_DPB * NS), smem, s, p);
  else if (pk == 4)
    launch_k_even(scan_pass1_kernel<N, PASS_DPB, NS, true, 4>, grid, dim3(PASS_DPB * NS), smem, s, p);
  else
    launch_k_even(scan_pass1_kernel<N, PASS_DPB, NS, true, 0>, grid, dim3(PASS_DPB * NS), smem, s, p);
}

template <int N, int NS>
static void launch_pass2(ScanParams& p, cudaStream_t s) {
  const dim3 grid(p.D / PASS_DPB, p.n_chunks, p.B);
  const size_t smem = pass2_smem<NS>(2 * N);
  const int pk = pass2_pk();
  if (p.bbar != 0)
    launch_k_even(scan_pass2_kernel<N, PASS_DPB, NS, false, 0>, grid, dim3(PASS_DPB * NS), smem, s, p);
  else if (pk == 4)
    launch_k_even(scan_pass2_kernel<N, PASS_DPB, NS, true, 4>, grid, dim3(PASS_DPB * NS), smem, s, p);
  else if (pk == 8)
    launch_k_even(scan_pass2_kernel<N, PASS_DPB, NS, true, 8>, grid, dim3(PASS_DPB * NS), smem, s, p);
  else
    launch_k_even(scan_pass2_kernel<N, PASS_DPB, NS, true, 0>, grid, dim3(PASS_DPB * NS), smem, s, p);
}

template <int N>
static void launch_dt_pass1(ScanParams& p, cudaStream_t s) {
  static const bool dt_ffma = getenv("PSCWIN_DT_FFMA") != nullptr;  // A/B knob: the CUDA-core dt kernel
  // A/B knob PSCWIN_DT_FUSE=1: the dt projection fused into pass 1 instead of the separate dt GEMM. Off: measured
  // at 4096^2 the fused pass 1 takes 1.06 ms against 0.796 + 0.117 ms for pass 1 + the dt GEMM (its per-sub-chunk
  // MMA / softplus phase stalls every warp of the CTA at once and adds MUFU work to the MUFU-bound loop)
  static const int dt_fuse = env_knob("PSCWIN_DT_FUSE", 0);
  const long long rows = (long long)p.B * (p.L + p.P);
  const bool fdt = dt_fuse != 0 && !dt_ffma && pass1_ns() == 4 && p.R % 4 == 0 && p.R <= 8 * FDT_KS;
  if (fdt) {
    PSCWIN_PROF("scan_pass1", s);
    launch_pass1<N, 4>(p, s, true);
    return;
  }
  if (!dt_ffma && p.R % 4 == 0) {
    // Delta = softplus(delta_low W_dt^T + b_dt) as a TF32 tensor-core GEMM (M = rows, N = D, K = R) reading
    // delta_low straight out of the x_proj output (row stride R + 2N) with the softplus in the f32 epilogue
    GemmArgs g;
    memset(&g, 0, sizeof(g));
    g.prof_name = "scan_dt";
    g.M = (int)rows;
    g.N = p.D;
    g.K = p.R;
    g.lda = p.R + 2 * N;
    g.ldb = p.R;
    g.out = p.delta;
    g.ldo = p.D;
    g.epi = EPI_STORE_F32;
    g.bias = p.b_dt;
    g.tf32 = 1;
    g.softplus = 1;
    launch_gemm_bf16(p.dbc, p.w_dt, g, s);
  } else {
    PSCWIN_PROF("scan_dt", s);
    dim3 gdt((p.D + 2 * DT_THREADS - 1) / (2 * DT_THREADS), (unsigned)((rows + DT_ROWS - 1) / DT_ROWS));
    if (p.R <= 16)
      launch_k(scan_dt_kernel<16>, gdt, dim3(DT_THREADS), 0, s, p);
    else if (p.R <= 48)
      launch_k(scan_dt_kernel<48>, gdt, dim3(DT_THREADS), 0, s, p);
    else
      launch_k(scan_dt_kernel<64>, gdt, dim3(DT_THREADS), 0, s, p);
  }
  {
    PSCWIN_PROF("scan_pass1", s);
    const int ns = pass1_ns();
    if (ns == 1) launch_pass1<N, 1>(p, s);
    else if (ns == 2) launch_pass1<N, 2>(p, s);
    else launch_pass1<N, 4>(p, s);
  }
}

template <int N>
static void launch_carry(ScanParams& p, cudaStream_t s) {
  PSCWIN_PROF("scan_carry", s);
  const int warps = p.B * p.D;
  const size_t per_warp = (size_t)p.n_chunks * (N + 1) * 4;
  int wpb = (int)((48 * 1024) / per_warp);  // warps per block within the default shared-memory window
  wpb = wpb > 8 ? 8 : (wpb < 1 ? 1 : wpb);
  launch_k(scan_carry_kernel<N>, dim3((warps + wpb - 1) / wpb), dim3(32 * wpb), wpb * per_warp, s, p);
}

template <int N>
static void launch_pass2_ns(ScanParams& p, cudaStream_t s) {
  PSCWIN_PROF("scan_pass2", s);
  const int ns = pass_ns();
  if (ns == 1) launch_pass2<N, 1>(p, s);
  else if (ns == 2) launch_pass2<N, 2>(p, s);
  else launch_pass2<N, 4>(p, s);
}

template <int N>
static int launch_passes(ScanParams& p, cudaStream_t s) {
  launch_dt_pass1<N>(p, s);
  launch_carry<N>(p, s);
  launch_pass2_ns<N>(p, s);
  return (int)cudaGetLastError();
}

// Full cycle scan given the in_proj output (xin, z with row strides) -> out (row stride ld_out). z_gated: z already
// holds SiLU(z) (module path: applied by the in_proj epilogue); otherwise the gate is computed into the workspace.
static ScanParams make_scan_params(const ScanPlan& pl, int B, int L, int D, int N, int R, int k, int bbar,
                                   const __nv_bfloat16* xin, long long ld_x, const __nv_bfloat16* gz, long long ld_gz,
                                   const float* conv_w, const float* conv_b, const float* w_dt, const float* b_dt,
                                   const float* a_log, const float* d_skip, __nv_bfloat16* out, long long ld_out,
                                   uint8_t* base) {
  ScanParams p;
  p.B = B;
  p.L = L;
  p.D = D;
  p.N = N;
  p.R = R;
  p.k = k;
  p.P = pl.P;
  p.Lc = pl.Lc;
  p.n_chunks = pl.n_chunks;
  p.bbar = bbar;
  p.xin = xin;
  p.ld_x = ld_x;
  p.gz = gz;
  p.ld_gz = ld_gz;
  p.conv_w = conv_w;
  p.conv_b = conv_b;
  p.w_dt = w_dt;
  p.b_dt = b_dt;
  p.a_log = a_log;
  p.d_skip = d_skip;
  p.v = reinterpret_cast<__nv_bfloat16*>(base + pl.v);
  p.dbc = reinterpret_cast<float*>(base + pl.dbc);
  p.delta = reinterpret_cast<float*>(base + pl.delta);
  p.sumdt = reinterpret_cast<float*>(base + pl.sumdt);
  p.hs = reinterpret_cast<float*>(base + pl.hs);
  p.out = out;
  p.ld_out = ld_out;
  p.vec_out = (ld_out % 8 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) ? 1 : 0;
  p.hist = nullptr;
  static const int conv_rev = env_knob("PSCWIN_CONV_REV", 1);
  p.conv_rev = conv_rev;
  return p;
}

// conv + x_proj (the front of the scan, before dt / pass 1)
static int scan_front(ScanParams& p, const ScanPlan& pl, const void* w_x, uint8_t* base, cudaStream_t s) {
  const long long rows = (long long)p.B * (p.L + pl.P);
  {
    PSCWIN_PROF("conv_silu", s);
    const long long nthreads = (long long)p.B * ((p.L + pl.P + CONV_T - 1) / CONV_T) * (p.D / 8);
    launch_k(conv_silu_kernel, dim3((unsigned)((nthreads + 255) / 256)), dim3(256), 0, s, p);
  }
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  g.prof_name = "gemm_x_proj";
  g.M = (int)rows;
  g.N = pl.W;
  g.K = p.D;
  g.lda = p.D;
  g.ldb = p.D;
  g.out = p.dbc;
  g.ldo = pl.W;
  g.epi = EPI_STORE_F32;
  g.BN = ((pl.W + 15) / 16) * 16;  // one N tile (R + 2N <= 256)
  g.splits = pl.xsplits;           // split-K when the M tiles alone cannot fill the SMs
  g.partial = reinterpret_cast<float*>(base + pl.partial);
  g.sem = reinterpret_cast<int*>(base + pl.sem);
  if (g.splits > 1) cudaMemsetAsync(g.sem, 0, (size_t)((g.M + 127) / 128) * sizeof(int), s);
  return launch_gemm_bf16(p.v, w_x, g, s) ? PSCWIN_ERR_CUDA : PSCWIN_OK;
}

static int run_cycle_scan(int B, int L, int D, int N, int R, int k, int bbar, const __nv_bfloat16* xin,
                          long long ld_x, const __nv_bfloat16* z, long long ld_z, bool z_gated, const float* conv_w,
                          const float* conv_b, const void* w_x, const float* w_dt, const float* b_dt,
                          const float* a_log, const float* d_skip, __nv_bfloat16* out, long long ld_out, void* ws,
                          size_t ws_bytes, cudaStream_t s) {
  ScanPlan pl = plan_scan(B, L, D, N, R, k);
  if (ws_bytes < pl.total) return PSCWIN_ERR_WORKSPACE;
  uint8_t* base = reinterpret_cast<uint8_t*>(ws);
  ScanParams p = make_scan_params(pl, B, L, D, N, R, k, bbar, xin, ld_x, z, ld_z, conv_w, conv_b, w_dt, b_dt, a_log,
                                  d_skip, out, ld_out, base);
  if (z && !z_gated) {
    PSCWIN_PROF("silu_gate", s);
    __nv_bfloat16* gz = reinterpret_cast<__nv_bfloat16*>(base + pl.gz);
    const long long n = (long long)B * L * (D / 8);
    launch_k(silu_gate_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, z, ld_z, (long long)B * L, D, gz);
    p.gz = gz;
    p.ld_gz = D;
  }
  int rc = scan_front(p, pl, w_x, base, s);
  if (rc) return rc;
  if (N == 16) rc = launch_passes<16>(p, s);
  else if (N == 32) rc = launch_passes<32>(p, s);
  else rc = launch_passes<64>(p, s);
  return rc ? PSCWIN_ERR_CUDA : PSCWIN_OK;
}

// ------------------------------------------------------------------------------------------------- band mode (host)
// One image (B = 1), this rank's contiguous scan segment of L tokens; P = k-1 on rank 0 (it holds the copy-1
// prefix), 0 elsewhere. The record buffer holds band_record_floats(D, N) floats.
size_t band_scan_ws_bytes(int L, int D, int N, int R, int k, int P) { return plan_scan_p(1, L, D, N, R, k, P).total; }
size_t band_scan_record_bytes(int D, int N) { return band_record_floats(D, N) * 4; }

// conv (with the preceding k-1 xin rows `hist`) -> x_proj -> dt -> pass 1 -> this segment's record
int band_scan_mid(int L, int D, int N, int R, int k, int P, int bbar, const __nv_bfloat16* xin, long long ld_x,
                  const __nv_bfloat16* hist, const float* conv_w, const float* conv_b, const void* w_x,
                  const float* w_dt, const float* b_dt, const float* a_log, const float* d_skip, float* rec, void* ws,
                  size_t ws_bytes, cudaStream_t s) {
  ScanPlan pl = plan_scan_p(1, L, D, N, R, k, P);
  if (ws_bytes < pl.total) return PSCWIN_ERR_WORKSPACE;
  uint8_t* base = reinterpret_cast<uint8_t*>(ws);
  ScanParams p = make_scan_params(pl, 1, L, D, N, R, k, bbar, xin, ld_x, nullptr, 0, conv_w, conv_b, w_dt, b_dt,
                                  a_log, d_skip, nullptr, 0, base);
  p.hist = hist;
  int rc = scan_front(p, pl, w_x, base, s);
  if (rc) return rc;
  if (N == 16) launch_dt_pass1<16>(p, s);
  else if (N == 32) launch_dt_pass1<32>(p, s);
  else launch_dt_pass1<64>(p, s);
  {
    PSCWIN_PROF("scan_segment", s);
    const dim3 grid((unsigned)((D + 7) / 8));
    if (N == 16) launch_k(scan_segment_kernel<16>, grid, dim3(256), 0, s, p, rec);
    else if (N == 32) launch_k(scan_segment_kernel<32>, grid, dim3(256), 0, s, p, rec);
    else launch_k(scan_segment_kernel<64>, grid, dim3(256), 0, s, p, rec);
  }
  return cudaGetLastError() == cudaSuccess ? PSCWIN_OK : PSCWIN_ERR_CUDA;
}

// all-gathered records (recs [world][record], rank order) -> chunk entry states (+ prefix outputs on rank 0)
// -> pass 2 -> out (gated by gz = SiLU(z))
int band_scan_end(int L, int D, int N, int R, int k, int P, int bbar, const __nv_bfloat16* xin, long long ld_x,
                  const __nv_bfloat16* gz, long long ld_gz, const float* conv_w, const float* conv_b,
                  const float* w_dt, const float* b_dt, const float* a_log, const float* d_skip, const float* recs,
                  int rank, int world, __nv_bfloat16* out, long long ld_out, void* ws, size_t ws_bytes,
                  cudaStream_t s) {
  ScanPlan pl = plan_scan_p(1, L, D, N, R, k, P);
  if (ws_bytes < pl.total) return PSCWIN_ERR_WORKSPACE;
  uint8_t* base = reinterpret_cast<uint8_t*>(ws);
  ScanParams p = make_scan_params(pl, 1, L, D, N, R, k, bbar, xin, ld_x, gz, ld_gz, conv_w, conv_b, w_dt, b_dt,
                                  a_log, d_skip, out, ld_out, base);
  {
    PSCWIN_PROF("scan_dist_carry", s);
    const dim3 grid((unsigned)((D + 7) / 8));
    if (N == 16) launch_k(scan_dist_carry_kernel<16>, grid, dim3(256), 0, s, p, recs, rank, world);
    else if (N == 32) launch_k(scan_dist_carry_kernel<32>, grid, dim3(256), 0, s, p, recs, rank, world);
    else launch_k(scan_dist_carry_kernel<64>, grid, dim3(256), 0, s, p, recs, rank, world);
  }
  if (N == 16) launch_pass2_ns<16>(p, s);
  else if (N == 32) launch_pass2_ns<32>(p, s);
  else launch_pass2_ns<64>(p, s);
  return cudaGetLastError() == cudaSuccess ? PSCWIN_OK : PSCWIN_ERR_CUDA;
}

// bytes of the scan-order copies (xin, z, out in scan order) a non-raster order needs in front of the scan plan
static size_t order_ws_bytes(int B, int L, int D, int order) {
  return order == PSCWIN_SCAN_ROW_MAJOR ? 0 : 3 * al256((size_t)B * L * D * 2);
}

size_t scan_ws_bytes(int B, int L, int D, int N, int R, int k, int order) {
  return order_ws_bytes(B, L, D, order) + plan_scan(B, L, D, N, R, k).total;
}

static int check_order(int H, int W, int order, int window) {
  if (order == PSCWIN_SCAN_ROW_MAJOR || order == PSCWIN_SCAN_COL_MAJOR) return PSCWIN_OK;
  if (order != PSCWIN_SCAN_WINDOW_MAJOR) return PSCWIN_ERR_SHAPE;
  if (window <= 0 || H % window || W % window) return PSCWIN_ERR_CONTRACT;
  return PSCWIN_OK;
}

// run_cycle_scan in any scan order: non-raster orders gather xin / z into scan order, scan, and scatter the output
// back to grid order (the recurrence itself is order-agnostic).
static int run_cycle_scan_ordered(int B, int H, int W, int order, int window, int D, int N, int R, int k, int bbar,
                                  const __nv_bfloat16* xin, long long ld_x, const __nv_bfloat16* z, long long ld_z,
                                  bool z_gated, const float* conv_w, const float* conv_b, const void* w_x,
                                  const float* w_dt, const float* b_dt, const float* a_log, const float* d_skip,
                                  __nv_bfloat16* out, long long ld_out, void* ws, size_t ws_bytes, cudaStream_t s) {
  const int L = H * W;
  if (order == PSCWIN_SCAN_ROW_MAJOR)
    return run_cycle_scan(B, L, D, N, R, k, bbar, xin, ld_x, z, ld_z, z_gated, conv_w, conv_b, w_x, w_dt, b_dt, a_log,
                          d_skip, out, ld_out, ws, ws_bytes, s);
  const size_t pre = order_ws_bytes(B, L, D, order), one = pre / 3;
  if (ws_bytes < pre) return PSCWIN_ERR_WORKSPACE;
  uint8_t* base = reinterpret_cast<uint8_t*>(ws);
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(base);
  __nv_bfloat16* zs = reinterpret_cast<__nv_bfloat16*>(base + one);
  __nv_bfloat16* os = reinterpret_cast<__nv_bfloat16*>(base + 2 * one);
  const long long n = (long long)B * L * (D / 8);
  const dim3 grid((unsigned)((n + 255) / 256));
  {
    PSCWIN_PROF("scan_order_gather", s);
    launch_k(permute_rows_kernel, grid, dim3(256), 0, s, xin, ld_x, xs, (long long)D, B, H, W, D, order, window, 0);
    if (z) launch_k(permute_rows_kernel, grid, dim3(256), 0, s, z, ld_z, zs, (long long)D, B, H, W, D, order, window, 0);
  }
  int rc = run_cycle_scan(B, L, D, N, R, k, bbar, xs, D, z ? zs : nullptr, D, z_gated, conv_w, conv_b, w_x, w_dt, b_dt,
                          a_log, d_skip, os, D, base + pre, ws_bytes - pre, s);
  if (rc) return rc;
  {
    PSCWIN_PROF("scan_order_scatter", s);
    launch_k(permute_rows_kernel, grid, dim3(256), 0, s, (const __nv_bfloat16*)os, (long long)D, out, ld_out, B, H, W,
             D, order, window, 1);
  }
  return cudaGetLastError() == cudaSuccess ? PSCWIN_OK : PSCWIN_ERR_CUDA;
}

int cycle_scan_module(const void* desc_v, const void* wts_v, const LnFold* lnf, const void* x_in, void* x_out, void* ws,
                      size_t off_u, size_t off_xz, size_t off_g, size_t off_scan, size_t scan_bytes, cudaStream_t s) {
  const pscwin_layer_desc* d = reinterpret_cast<const pscwin_layer_desc*>(desc_v);
  const pscwin_layer_weights* w = reinterpret_cast<const pscwin_layer_weights*>(wts_v);
  if (!w->lns_g || !w->lns_b || !w->w_in || !w->conv_w || !w->conv_b || !w->w_x || !w->w_dt || !w->b_dt ||
      !w->a_log || !w->d_skip || !w->w_out)
    return PSCWIN_ERR_SHAPE;
  const int C = d->C, D = d->ssm_expand * C, N = d->ssm_state;
  const int R = d->ssm_dt_rank > 0 ? d->ssm_dt_rank : (C + 15) / 16;
  const int L = d->H * d->W;
  int rc = check_scan(d->B, L, D, N, R, d->ssm_conv);
  if (rc) return rc;
  rc = check_order(d->H, d->W, d->scan_order, d->window);
  if (rc) return rc;
  const long long T = (long long)d->B * L;
  uint8_t* base = reinterpret_cast<uint8_t*>(ws);
  __nv_bfloat16* u = reinterpret_cast<__nv_bfloat16*>(base + off_u);
  __nv_bfloat16* xz = reinterpret_cast<__nv_bfloat16*>(base + off_xz);
  __nv_bfloat16* g = reinterpret_cast<__nv_bfloat16*>(base + off_g);
  // a1: u0 = LN_s(x); [xin, z] = u0 W_in^T (the LayerNorm folded into the projection when lnf is given)
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
  a.silu_col = D;  // the z half leaves the epilogue as the output gate SiLU(z)
  rc = ln_gemm(x_in, (const float*)w->lns_g, (const float*)w->lns_b, d->ln_eps, w->w_in, a, u, lnf, s);
  if (rc) return PSCWIN_ERR_CUDA;
  // a2: cycle scan -> g = sum over copies of y * SiLU(z)
  rc = run_cycle_scan_ordered(d->B, d->H, d->W, d->scan_order, d->window, D, N, R, d->ssm_conv, d->bbar_mode, xz,
                              2 * D, xz + D, 2 * D, true,
                      (const float*)w->conv_w, (const float*)w->conv_b, w->w_x, (const float*)w->w_dt,
                      (const float*)w->b_dt, w->a_log, w->d_skip, g, D, base + off_scan, scan_bytes, s);
  if (rc) return rc;
  // a3: x_out = x_in + g W_out^T (the sum over copies commutes with the bias-free out_proj)
  memset(&a, 0, sizeof(a));
  a.prof_name = "gemm_out_proj_scan";
  a.M = (int)T;
  a.N = C;
  a.K = D;
  a.lda = D;
  a.ldb = D;
  a.out = x_out;
  a.ldo = C;
  a.epi = EPI_RESID_BF16;
  a.residual = x_in;
  a.ldr = C;
  rc = launch_gemm_bf16(g, w->w_out, a, s);
  return rc ? PSCWIN_ERR_CUDA : PSCWIN_OK;
}

// ------------------------------------------------------------------------------------------------- multi-scale
static bool ms_needs_perm(int B, int order) { return B > 1 || order != PSCWIN_SCAN_ROW_MAJOR; }

size_t ms_scan_ws_bytes(int B, const MsGeo& g, int mode, int D, int N, int R, int k, int order) {
  if (mode == 1) {
    size_t m = 0;
    for (int i = 0; i < g.n; ++i) {
      const size_t b = scan_ws_bytes(B, g.H[i] * g.W[i], D, N, R, k, order);
      m = b > m ? b : m;
    }
    return m;
  }
  const int Lt = g.off[g.n];
  size_t pre = ms_needs_perm(B, order) ? al256((size_t)B * Lt * 2 * D * 2) + al256((size_t)B * Lt * D * 2) : 0;
  return pre + plan_scan(B, Lt, D, N, R, k).total;
}

int ms_cycle_scan_module(const void* desc_v, const void* wts_v, const MsGeo& g, int mode, const void* x_in,
                         void* x_out, void* ws, size_t off_u, size_t off_xz, size_t off_g, size_t off_scan,
                         size_t scan_bytes, cudaStream_t s) {
  const pscwin_layer_desc* d = reinterpret_cast<const pscwin_layer_desc*>(desc_v);
  const pscwin_layer_weights* w = reinterpret_cast<const pscwin_layer_weights*>(wts_v);
  if (!w->lns_g || !w->lns_b || !w->w_in || !w->conv_w || !w->conv_b || !w->w_x || !w->w_dt || !w->b_dt ||
      !w->a_log || !w->d_skip || !w->w_out)
    return PSCWIN_ERR_SHAPE;
  if (mode != 1 && mode != 2) return PSCWIN_ERR_CONTRACT;
  const int C = d->C, D = d->ssm_expand * C, N = d->ssm_state, B = d->B;
  const int R = d->ssm_dt_rank > 0 ? d->ssm_dt_rank : (C + 15) / 16;
  const int k = d->ssm_conv, order = d->scan_order;
  const int Lt = g.off[g.n];
  int rc;
  for (int i = 0; i < g.n; ++i) {
    rc = check_order(g.H[i], g.W[i], order, d->window);
    if (rc) return rc;
    if (mode == 1 && (rc = check_scan(B, g.H[i] * g.W[i], D, N, R, k))) return rc;
  }
  if (mode == 2 && (rc = check_scan(B, Lt, D, N, R, k))) return rc;
  const long long T = (long long)B * Lt;
  uint8_t* base = reinterpret_cast<uint8_t*>(ws);
  __nv_bfloat16* u = reinterpret_cast<__nv_bfloat16*>(base + off_u);
  __nv_bfloat16* xz = reinterpret_cast<__nv_bfloat16*>(base + off_xz);
  __nv_bfloat16* gout = reinterpret_cast<__nv_bfloat16*>(base + off_g);
  uint8_t* sws = base + off_scan;
  // a1 over every packed row at once (token-local): u0 = LN_s(x); [xin, SiLU(z)] = u0 W_in^T
  if (launch_layer_norm(x_in, T, C, (const float*)w->lns_g, (const float*)w->lns_b, d->ln_eps, 0, u, s))
    return PSCWIN_ERR_CUDA;
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
  if (launch_gemm_bf16(u, w->w_in, a, s)) return PSCWIN_ERR_CUDA;
  const float *cw = (const float*)w->conv_w, *cb = (const float*)w->conv_b, *wdt = (const float*)w->w_dt,
              *bdt = (const float*)w->b_dt;
  if (mode == 1) {
    // single-scale: every scale's [B, H_s, W_s] block is its own batch of cycled sequences
    for (int i = 0; i < g.n; ++i) {
      const long long r0 = (long long)B * g.off[i];
      rc = run_cycle_scan_ordered(B, g.H[i], g.W[i], order, d->window, D, N, R, k, d->bbar_mode, xz + r0 * 2 * D,
                                  2 * D, xz + r0 * 2 * D + D, 2 * D, true, cw, cb, w->w_x, wdt, bdt, w->a_log,
                                  w->d_skip, gout + r0 * D, D, sws, scan_bytes, s);
      if (rc) return rc;
    }
  } else if (!ms_needs_perm(B, order)) {
    // multi-scale, one sample, raster order: the packed rows ARE the concatenated sequence
    rc = run_cycle_scan(1, Lt, D, N, R, k, d->bbar_mode, xz, 2 * D, xz + D, 2 * D, true, cw, cb, w->w_x, wdt, bdt,
                        w->a_log, w->d_skip, gout, D, sws, scan_bytes, s);
    if (rc) return rc;
  } else {
    // multi-scale: gather [xin | SiLU(z)] rows into per-sample concatenated scan order, scan, scatter the output
    const size_t one = al256((size_t)T * 2 * D * 2), two = al256((size_t)T * D * 2);
    if (scan_bytes < one + two) return PSCWIN_ERR_WORKSPACE;
    __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(sws);
    __nv_bfloat16* os = reinterpret_cast<__nv_bfloat16*>(sws + one);
    {
      PSCWIN_PROF("scan_ms_gather", s);
      const long long n = T * (2 * D / 8);
      launch_k(ms_permute_rows_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s,
               (const __nv_bfloat16*)xz, (long long)2 * D, xs, (long long)2 * D, B, g, 2 * D, order, d->window, 0);
    }
    rc = run_cycle_scan(B, Lt, D, N, R, k, d->bbar_mode, xs, 2 * D, xs + D, 2 * D, true, cw, cb, w->w_x, wdt, bdt,
                        w->a_log, w->d_skip, os, D, sws + one + two, scan_bytes - one - two, s);
    if (rc) return rc;
    {
      PSCWIN_PROF("scan_ms_scatter", s);
      const long long n = T * (D / 8);
      launch_k(ms_permute_rows_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s,
               (const __nv_bfloat16*)os, (long long)D, gout, (long long)D, B, g, D, order, d->window, 1);
    }
  }
  // a3 over every packed row: x_out = x_in + g W_out^T
  memset(&a, 0, sizeof(a));
  a.prof_name = "gemm_out_proj_scan";
  a.M = (int)T;
  a.N = C;
  a.K = D;
  a.lda = D;
  a.ldb = D;
  a.out = x_out;
  a.ldo = C;
  a.epi = EPI_RESID_BF16;
  a.residual = x_in;
  a.ldr = C;
  return launch_gemm_bf16(gout, w->w_out, a, s) ? PSCWIN_ERR_CUDA : PSCWIN_OK;
}

}  // namespace pscwin

using namespace pscwin;

extern "C" size_t pscwin_scan_workspace_bytes(const pscwin_scan_desc* d) {
  if (!d) return 0;
  const int L = d->H * d->W;
  if (check_scan(d->B, L, d->D, d->N, d->R, d->conv_k) != PSCWIN_OK) return 0;
  if (check_order(d->H, d->W, d->scan_order, d->window) != PSCWIN_OK) return 0;
  if (d->dtype == PSCWIN_F32) return scan_f32_ws_bytes(d->B, L, d->D, d->N, d->R, d->conv_k);
  return scan_ws_bytes(d->B, L, d->D, d->N, d->R, d->conv_k, d->scan_order);
}

extern "C" int32_t pscwin_scan_chunk_length(const pscwin_scan_desc* d) {
  if (!d || d->dtype != PSCWIN_BF16) return 0;
  const int L = d->H * d->W;
  if (check_scan(d->B, L, d->D, d->N, d->R, d->conv_k) != PSCWIN_OK) return 0;
  return choose_chunk(d->B, L, d->D, d->N, 2 * d->N);
}

extern "C" int pscwin_cycle_scan(const pscwin_scan_desc* d, const void* xin, const void* z, const float* conv_w,
                                 const float* conv_b, const void* w_x, const float* w_dt, const float* b_dt,
                                 const float* a_log, const float* d_skip, void* out, void* ws, size_t ws_bytes,
                                 void* stream) {
  if (!d || !xin || !conv_w || !conv_b || !w_x || !w_dt || !b_dt || !a_log || !d_skip || !out)
    return PSCWIN_ERR_SHAPE;
  if (d->dtype != PSCWIN_BF16 && d->dtype != PSCWIN_F32) return PSCWIN_ERR_UNSUPPORTED;
  const int L = d->H * d->W;
  int rc = check_scan(d->B, L, d->D, d->N, d->R, d->conv_k);
  if (rc) return rc;
  rc = check_order(d->H, d->W, d->scan_order, d->window);
  if (rc) return rc;
  if (d->dtype == PSCWIN_F32) {
    if (((uintptr_t)xin | (uintptr_t)z | (uintptr_t)out | (uintptr_t)ws | (uintptr_t)w_x) & 15) return PSCWIN_ERR_ALIGN;
    return run_cycle_scan_f32(d->B, d->H, d->W, d->scan_order, d->window, d->D, d->N, d->R, d->conv_k, d->bbar_mode,
                              (const float*)xin, d->D, (const float*)z, d->D, false, conv_w, conv_b,
                              (const float*)w_x, w_dt, b_dt, a_log, d_skip, (float*)out, d->D, ws, ws_bytes,
                              (cudaStream_t)stream);
  }
  if (((uintptr_t)xin | (uintptr_t)z | (uintptr_t)out | (uintptr_t)ws | (uintptr_t)w_x) & 15) return PSCWIN_ERR_ALIGN;
  return run_cycle_scan_ordered(d->B, d->H, d->W, d->scan_order, d->window, d->D, d->N, d->R, d->conv_k,
                                d->bbar_mode, (const __nv_bfloat16*)xin, d->D, (const __nv_bfloat16*)z, d->D, false,
                                conv_w, conv_b, w_x, w_dt, b_dt, a_log, d_skip,
                        (__nv_bfloat16*)out, d->D, ws, ws_bytes, (cudaStream_t)stream);
}
