// Row-wise helper kernels: LayerNorm (pre-norm of a4 and a1; eps 1e-6, reading Q15) and the one-row
// projection of the learnable pad token p through the QKV linear ("F and the learnable padding
// embedding p are both projected through the attention's QKV-linear layer"; p is not normalised, reading Q14).
#include "common.cuh"
#include "pscwin_internal.h"

namespace pscwin {

// One warp per row; up to 8 x 32 vectors (C <= 2048 bf16 / 1024 f32) kept in registers (two-pass mean/var).
template <typename T>
__global__ void layer_norm_kernel(const T* __restrict__ x, long long rows, int C, const float* __restrict__ g,
                                  const float* __restrict__ b, float eps, T* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  constexpr int EPV = 16 / sizeof(T);  // elements per 16-byte vector
  long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const int nvec = C / EPV;
  const uint4* src = reinterpret_cast<const uint4*>(x + row * C);
  uint4 v[8];
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int i = lane + 32 * k;
    if (i < nvec) {
      v[k] = src[i];
      const T* e = reinterpret_cast<const T*>(&v[k]);
#pragma unroll
      for (int j = 0; j < EPV; ++j) {
        float f;
        if constexpr (sizeof(T) == 2) f = __bfloat162float(e[j]); else f = e[j];
        sum += f;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / C;
  float sq = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int i = lane + 32 * k;
    if (i < nvec) {
      const T* e = reinterpret_cast<const T*>(&v[k]);
#pragma unroll
      for (int j = 0; j < EPV; ++j) {
        float f;
        if constexpr (sizeof(T) == 2) f = __bfloat162float(e[j]); else f = e[j];
        sq += (f - mean) * (f - mean);
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  const float rstd = rsqrtf(sq / C + eps);
  uint4* dst = reinterpret_cast<uint4*>(out + row * C);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int i = lane + 32 * k;
    if (i < nvec) {
      uint4 w;
      const T* e = reinterpret_cast<const T*>(&v[k]);
      T* o = reinterpret_cast<T*>(&w);
      float gg[EPV], bb[EPV];  // gamma / beta for this vector, 16-byte loads
#pragma unroll
      for (int j = 0; j < EPV; j += 4) {
        const float4 g4 = __ldg(reinterpret_cast<const float4*>(g + i * EPV + j));
        const float4 b4 = __ldg(reinterpret_cast<const float4*>(b + i * EPV + j));
        gg[j] = g4.x; gg[j + 1] = g4.y; gg[j + 2] = g4.z; gg[j + 3] = g4.w;
        bb[j] = b4.x; bb[j + 1] = b4.y; bb[j + 2] = b4.z; bb[j + 3] = b4.w;
      }
#pragma unroll
      for (int j = 0; j < EPV; ++j) {
        float f;
        if constexpr (sizeof(T) == 2) f = __bfloat162float(e[j]); else f = e[j];
        float y = (f - mean) * rstd * gg[j] + bb[j];
        if constexpr (sizeof(T) == 2) o[j] = __float2bfloat16_rn(y); else o[j] = y;
      }
      dst[i] = w;
    }
  }
}

// bf16 LayerNorm with packed fp32x2 arithmetic: the kernel above spends ~10 instructions per element (ncu r02f: 75 %
// issue-bound at 39 % of DRAM bandwidth); here each 16-byte vector is four (lo, hi) pairs: FADD2 sums, the centred
// values d = x - mean kept for the variance and the output, FFMA2 d^2 sums, then y = d (rstd gamma) + beta as FMUL2 +
// FFMA2 and one F2FP pack per pair (~4.5 instructions per element).
// RPW rows per warp: the loads of all RPW rows are issued up front, then the rows are normalised in turn (ncu r02n
// shows long-scoreboard stalls of 11.7 warps per issue at one row per warp, but 2 / 4 rows per warp measured slower:
// the occupancy they cost outweighs the loads in flight they add; RPW = 1 is the default).
// rev: rows are visited last-first. The LayerNorm input is the residual stream the previous GEMM has just written in
// row order, so its LAST rows are the ones still resident in L2; reading them first turns part of the read into L2 hits.
template <int NV, int RPW>  // 16-byte vectors per lane: ceil(C / 256)
__global__ void layer_norm_bf16x2_kernel(const __nv_bfloat16* __restrict__ x, long long rows, int C,
                                         const float* __restrict__ g, const float* __restrict__ b, float eps,
                                         __nv_bfloat16* __restrict__ out, int rev) {
  pdl_trigger();
  pdl_wait();
  const long long wg = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long nwg = (rows + RPW - 1) / RPW;
  if (wg >= nwg) return;
  const long long row0 = (rev ? nwg - 1 - wg : wg) * RPW;
  const int lane = threadIdx.x & 31;
  const int nvec = C / 8;
  uint4 vr[RPW][NV];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const uint4* src = reinterpret_cast<const uint4*>(x + (row0 + r) * C);
#pragma unroll
    for (int k = 0; k < NV; ++k)
      if (row0 + r < rows && lane + 32 * k < nvec) vr[r][k] = src[lane + 32 * k];
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
  const long long row = row0 + r;
  if (row >= rows) break;
  const uint4 (&v)[NV] = vr[r];
  float2 d[NV][4];
  float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    if (lane + 32 * k < nvec) {
      const uint32_t* w = reinterpret_cast<const uint32_t*>(&v[k]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        d[k][q] = make_float2(bf16_lo(w[q]), bf16_hi(w[q]));
        s2 = __fadd2_rn(s2, d[k][q]);
      }
    }
  }
  float sum = s2.x + s2.y;
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / C;
  const float2 nm = make_float2(-mean, -mean);
  float2 q2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    if (lane + 32 * k < nvec) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        d[k][q] = __fadd2_rn(d[k][q], nm);
        q2 = __ffma2_rn(d[k][q], d[k][q], q2);
      }
    }
  }
  float sq = q2.x + q2.y;
#pragma unroll
  for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  const float rstd = rsqrtf(sq / C + eps);
  const float2 r2 = make_float2(rstd, rstd);
  uint4* dst = reinterpret_cast<uint4*>(out + row * C);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int i = lane + 32 * k;
    if (i < nvec) {
      const float4* g4 = reinterpret_cast<const float4*>(g + i * 8);
      const float4* b4 = reinterpret_cast<const float4*>(b + i * 8);
      const float4 ga = __ldg(g4), gb = __ldg(g4 + 1), ba = __ldg(b4), bb = __ldg(b4 + 1);
      const float2 gg[4] = {make_float2(ga.x, ga.y), make_float2(ga.z, ga.w), make_float2(gb.x, gb.y),
                            make_float2(gb.z, gb.w)};
      const float2 be[4] = {make_float2(ba.x, ba.y), make_float2(ba.z, ba.w), make_float2(bb.x, bb.y),
                            make_float2(bb.z, bb.w)};
      uint4 w;
      uint32_t* o = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 y = __ffma2_rn(__fmul2_rn(d[k][q], r2), gg[q], be[q]);
        o[q] = pack_bf16(y.x, y.y);
      }
      dst[i] = w;
    }
  }
  }  // rows of this warp
}

int launch_layer_norm(const void* x, long long rows, int C, const float* g, const float* b, float eps, int is_f32,
                      void* out, cudaStream_t stream) {
  if (rows == 0) return 0;
  unsigned grid = (unsigned)((rows + 7) / 8);
  PSCWIN_PROF("layer_norm", stream);
  // rows per warp of the packed bf16 kernel (A/B knob PSCWIN_LN_RPW = 1, 2 or 4, read once). One: measured at
  // 65536 x 768 (graph-timed, L2 flushed) 45.6 / 47.0 / 53.1 us for 1 / 2 / 4 rows per warp (profiles/r02/rowops_r02o.log)
  static const int rpw_knob = env_knob("PSCWIN_LN_RPW", 1);
  const int rpw = (rpw_knob == 2 || rpw_knob == 4) ? rpw_knob : 1;
  static const int rev = env_knob("PSCWIN_LN_REV", 1);  // A/B knob: 0 = rows first-to-last
  if (is_f32) {
    if (C % 4 || C > 1024) return -1;
    launch_k(layer_norm_kernel<float>, dim3(grid), dim3(256), 0, stream, (const float*)x, rows, C, g, b, eps, (float*)out);
  } else {
    if (C % 8 || C > 2048) return -1;
    static const int packed = env_knob("PSCWIN_LN_PACKED", 1);  // A/B knob: 0 = the scalar kernel
    if (packed) {
      const int nv = (C / 8 + 31) / 32;
      auto go = [&](auto kern, int r) {
        const unsigned gr = (unsigned)((rows + 8LL * r - 1) / (8LL * r));
        launch_k(kern, dim3(gr), dim3(256), 0, stream, (const __nv_bfloat16*)x, rows, C, g, b, eps, (__nv_bfloat16*)out,
                 rev);
      };
      if (nv <= 4 && rpw > 1) {  // (wide rows keep one row per warp: their loads already fill the warp)
        switch (nv * 8 + rpw) {
          case 10: go(layer_norm_bf16x2_kernel<1, 2>, 2); break;
          case 12: go(layer_norm_bf16x2_kernel<1, 4>, 4); break;
          case 18: go(layer_norm_bf16x2_kernel<2, 2>, 2); break;
          case 20: go(layer_norm_bf16x2_kernel<2, 4>, 4); break;
          case 26: go(layer_norm_bf16x2_kernel<3, 2>, 2); break;
          case 28: go(layer_norm_bf16x2_kernel<3, 4>, 4); break;
          case 34: go(layer_norm_bf16x2_kernel<4, 2>, 2); break;
          default: go(layer_norm_bf16x2_kernel<4, 4>, 4); break;
        }
        return (int)cudaGetLastError();
      }
      switch (nv) {
        case 1: go(layer_norm_bf16x2_kernel<1, 1>, 1); break;
        case 2: go(layer_norm_bf16x2_kernel<2, 1>, 1); break;
        case 3: go(layer_norm_bf16x2_kernel<3, 1>, 1); break;
        case 4: go(layer_norm_bf16x2_kernel<4, 1>, 1); break;
        case 5: case 6: go(layer_norm_bf16x2_kernel<6, 1>, 1); break;
        default: go(layer_norm_bf16x2_kernel<8, 1>, 1); break;
      }
      return (int)cudaGetLastError();
    }
    launch_k(layer_norm_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, stream, (const __nv_bfloat16*)x, rows, C, g, b, eps,
                                                               (__nv_bfloat16*)out);
  }
  return (int)cudaGetLastError();
}

// qkv_p[j] = sum_c p[c] W_qkv[j, c] + b_qkv[j]  (f32 accumulate, f32 result), one warp per output j
template <typename T>
__global__ void pad_qkv_kernel(const T* __restrict__ pad, const T* __restrict__ w, const float* __restrict__ bias,
                               int C, float* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= 3 * C) return;
  int lane = threadIdx.x & 31;
  float acc = 0.f;
  if constexpr (sizeof(T) == 2) {
    if (C % 8 == 0) {  // 16-byte vectors: the warp's row loads are independent (C = 768: 3 per lane)
      const uint4* w4 = reinterpret_cast<const uint4*>(w + (size_t)j * C);
      const uint4* p4 = reinterpret_cast<const uint4*>(pad);
      for (int i = lane; i < C / 8; i += 32) {
        const uint4 wv = __ldg(w4 + i), pv = __ldg(p4 + i);
        const uint32_t* ww = reinterpret_cast<const uint32_t*>(&wv);
        const uint32_t* pw = reinterpret_cast<const uint32_t*>(&pv);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc = fmaf(__uint_as_float(pw[q] << 16), __uint_as_float(ww[q] << 16), acc);
          acc = fmaf(__uint_as_float(pw[q] & 0xFFFF0000u), __uint_as_float(ww[q] & 0xFFFF0000u), acc);
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) out[j] = acc + (bias ? bias[j] : 0.f);
      return;
    }
  }
  for (int c = lane; c < C; c += 32) {
    float a, bw;
    if constexpr (sizeof(T) == 2) {
      a = __bfloat162float(pad[c]);
      bw = __bfloat162float(w[(size_t)j * C + c]);
    } else {
      a = pad[c];
      bw = w[(size_t)j * C + c];
    }
    acc = fmaf(a, bw, acc);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[j] = acc + (bias ? bias[j] : 0.f);
}

int launch_pad_qkv(const void* pad, const void* w_qkv, const float* b_qkv, int C, int is_f32, float* out,
                   cudaStream_t stream) {
  unsigned grid = (unsigned)((3 * C + 7) / 8);
  PSCWIN_PROF("pad_qkv", stream);
  if (is_f32)
    launch_k(pad_qkv_kernel<float>, dim3(grid), dim3(256), 0, stream, (const float*)pad, (const float*)w_qkv, b_qkv, C, out);
  else
    launch_k(pad_qkv_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, stream, (const __nv_bfloat16*)pad,
                                                            (const __nv_bfloat16*)w_qkv, b_qkv, C, out);
  return (int)cudaGetLastError();
}


// ---------------------------------------------------------------------------------------------------------------
// LayerNorm folded into the following projection (a1 LN_s -> in_proj, a4 LN1 -> QKV, FFN LN2 -> fc1):
//   LN(x) W^T + b = rstd (x W'^T - mu s) + c,   W' = W diag(gamma),  s_n = sum_k W'[n,k],  c = W beta + b
// (exact algebra of LN(x)_k = (x_k - mu) rstd gamma_k + beta_k). The GEMM reads x itself; its epilogue applies the
// row statistics (mu, rstd) and the folded column terms (s, c). Two small kernels feed it:
//   row_stats_kernel: (mu, rstd) per row of x, two-pass in registers (warp per row) -> 8 bytes per row instead of
//                     the C-element normalised row (the LayerNorm pass it replaces reads AND writes C elements);
//   ln_fold_kernel:   W' (bf16), s (from the rounded W' so x W'^T - mu s vanishes for a constant row) and c, from
//                     the weights alone (weight-only work: it runs on the side stream, off the critical path).
// ---------------------------------------------------------------------------------------------------------------
// Rows are visited last-first (rev): x was just written first-to-last by the previous GEMM, so its last rows are the
// L2-resident ones, and the projection that follows reads x first-to-last, i.e. the rows this kernel touched last.
template <int NV>  // 16-byte vectors per lane: ceil(C / 256)
__global__ void row_stats_kernel(const __nv_bfloat16* __restrict__ x, long long rows, int C, float eps,
                                 float2* __restrict__ stats, int rev) {
  pdl_trigger();
  pdl_wait();
  const long long wg = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wg >= rows) return;
  const long long row = rev ? rows - 1 - wg : wg;
  const int lane = threadIdx.x & 31;
  const int nvec = C / 8;
  const uint4* src = reinterpret_cast<const uint4*>(x + row * C);
  uint4 v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {  // all loads in flight before any arithmetic
    const int i = lane + 32 * k;
    if (i < nvec) v[k] = src[i];  // (normal caching: the projection re-reads x right after)
  }
  // packed fp32x2 arithmetic (ncu r02ac: the scalar form was issue-bound, 82 % issue): FADD2 sums, FADD2 centring,
  // FFMA2 squares
  float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    if (lane + 32 * k < nvec) {
      const uint32_t* w = reinterpret_cast<const uint32_t*>(&v[k]);
#pragma unroll
      for (int j = 0; j < 4; ++j) s2 = __fadd2_rn(s2, make_float2(bf16_lo(w[j]), bf16_hi(w[j])));
    }
  }
  float sum = s2.x + s2.y;
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / C;
  const float2 nm = make_float2(-mean, -mean);
  float2 q2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    if (lane + 32 * k < nvec) {
      const uint32_t* w = reinterpret_cast<const uint32_t*>(&v[k]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 dv = __fadd2_rn(make_float2(bf16_lo(w[j]), bf16_hi(w[j])), nm);
        q2 = __ffma2_rn(dv, dv, q2);
      }
    }
  }
  float sq = q2.x + q2.y;
#pragma unroll
  for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if (lane == 0) stats[row] = make_float2(mean, rsqrtf(sq / C + eps));
}

// one warp per output row n of W [N, K] (nn.Linear layout): W'[n,:] = bf16(W[n,:] * gamma), s[n] = sum W'[n,:],
// c[n] = sum_k beta_k W[n,k] + b[n]
__global__ void ln_fold_kernel(const __nv_bfloat16* __restrict__ Wt, int N, int K, const float* __restrict__ g,
                               const float* __restrict__ beta, const float* __restrict__ bias,
                               __nv_bfloat16* __restrict__ Wf, float* __restrict__ s, float* __restrict__ c) {
  pdl_trigger();
  pdl_wait();
  const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (n >= N) return;
  const int lane = threadIdx.x & 31;
  const uint4* src = reinterpret_cast<const uint4*>(Wt + (size_t)n * K);
  uint4* dst = reinterpret_cast<uint4*>(Wf + (size_t)n * K);
  float ss = 0.f, cc = 0.f;
  for (int i = lane; i < K / 8; i += 32) {
    const uint4 w = __ldg(src + i);
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(g + 8 * i));
    const float4 g1 = __ldg(reinterpret_cast<const float4*>(g + 8 * i + 4));
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(beta + 8 * i));
    const float4 b1 = __ldg(reinterpret_cast<const float4*>(beta + 8 * i + 4));
    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    const uint32_t* wi = reinterpret_cast<const uint32_t*>(&w);
    uint4 o;
    uint32_t* wo = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float w0 = bf16_lo(wi[j]), w1 = bf16_hi(wi[j]);
      wo[j] = pack_bf16(w0 * gg[2 * j], w1 * gg[2 * j + 1]);
      ss += bf16_lo(wo[j]) + bf16_hi(wo[j]);
      cc = fmaf(w0, bb[2 * j], fmaf(w1, bb[2 * j + 1], cc));
    }
    dst[i] = o;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    cc += __shfl_xor_sync(0xffffffffu, cc, o);
  }
  if (lane == 0) {
    s[n] = ss;
    c[n] = cc + (bias ? bias[n] : 0.f);
  }
}

int launch_row_stats(const void* x, long long rows, int C, float eps, float2* stats, cudaStream_t stream) {
  if (rows == 0) return 0;
  if (C % 8 || C > 2048) return -1;
  PSCWIN_PROF("row_stats", stream);
  static const int rev = env_knob("PSCWIN_LN_REV", 1);
  const int nv = (C / 8 + 31) / 32;
  auto go = [&](auto kern) {
    launch_k(kern, dim3((unsigned)((rows + 7) / 8)), dim3(256), 0, stream, (const __nv_bfloat16*)x, rows, C, eps, stats,
             rev);
  };
  if (nv <= 1) go(row_stats_kernel<1>);
  else if (nv == 2) go(row_stats_kernel<2>);
  else if (nv == 3) go(row_stats_kernel<3>);
  else if (nv == 4) go(row_stats_kernel<4>);
  else go(row_stats_kernel<8>);
  return (int)cudaGetLastError();
}

int launch_ln_fold(const void* W, int N, int K, const float* g, const float* beta, const float* bias, void* Wf,
                   float* s, float* c, cudaStream_t stream) {
  if (K % 8) return -1;
  PSCWIN_PROF("ln_fold", stream);
  launch_k(ln_fold_kernel, dim3((unsigned)((N + 7) / 8)), dim3(256), 0, stream, (const __nv_bfloat16*)W, N, K, g, beta,
           bias, (__nv_bfloat16*)Wf, s, c);
  return (int)cudaGetLastError();
}

}  // namespace pscwin
