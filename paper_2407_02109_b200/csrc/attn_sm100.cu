// Window attention core on tcgen05 tensor cores (SURVEY §8(a) a5 + a6 + crop of a7).
//
// Computes, for every window of the plain or padding-shifted layout and every head,
// O = softmax(q k^T / sqrt(d)) v over the window's w^2 slots (reading Q1: pre-softmax scale), with the flash
// recurrence of App. A.5 across 128-key tiles, and writes only real rows back to the [B,H,W,C]
// grid ("the paddings are discarded"). Pad slots: LEARNABLE (paper) = the projected pad token p's K/V,
// K rotated at the slot's geometric coordinate (reading Q6); MASKED (north star) = logits -inf (reading Q5).
//
// B200 design: the window partition IS the TMA box — a 5-D tensor map over QKV [B,H,W,3,heads,d] loads a
// (d x 1 x w x rows) box per operand straight into 128B-swizzled shared memory; boxes that hang off the grid
// (shifted windows) are zero-filled by TMA and the pad rows are patched in shared memory from tiny per-layer
// tables (rotated k_p halves per x / y coordinate, v_p). S = Q K^T accumulates in TMEM (fp32), softmax runs
// one row per thread in fp32 (exp2 with log2(e)/sqrt(d) folded), P is written bf16 to swizzled smem, O = P V
// accumulates in TMEM, and the merge/crop writes each real row straight to the [B,H,W,C] grid (pad rows dropped). No L^2 buffer exists anywhere (App. A.6).
#include <stdlib.h>

#include "common.cuh"
#include "pscwin_internal.h"

namespace pscwin {

namespace {
constexpr int ATT_THREADS = 128;
}

struct AttnKArgs {
  int B, H, W, C, heads, w, pt, pl, nwx, nw, pad_mode, patch;
  int rpt;        // window rows per 128-slot tile
  int n_tiles;    // tiles per window (= w / rpt)
  int tile_slots; // w * rpt
  float sl2;      // log2(e) / sqrt(d)
  const __nv_bfloat16* kx;  // [Wp][heads][d/2]  rotated first half of k_p at x = X (index X + pl)
  const __nv_bfloat16* ky;  // [Hp][heads][d/2]  rotated second half at y = Y (index Y + pt)
  const __nv_bfloat16* vp;  // [heads][d]
  int Wp, Hp;
  int win0, nw_run;         // windows [win0, win0 + nw_run) of every image (a window-row range; all by default)
  __nv_bfloat16* out;       // [B,H,W,C]
};

template <int D>
__global__ void __launch_bounds__(ATT_THREADS, 2)
    window_attn_kernel(const __grid_constant__ CUtensorMap tmQKV, AttnKArgs p) {
  pdl_trigger();
  pdl_wait();
  constexpr int ROWB = D * 2;                 // bytes per row of Q/K/V/O (64 or 128)
  constexpr int TILE_BYTES = 128 * ROWB;      // smem rows allocated per operand
  constexpr uint32_t LAYOUT = ROWB == 128 ? kLayoutSW128 : kLayoutSW64;
  constexpr uint32_t SBO = 8 * ROWB;

  const int qt = blockIdx.x;
  const int h = blockIdx.y;
  const int b = blockIdx.z / p.nw_run;
  const int win = p.win0 + (blockIdx.z - b * p.nw_run);
  const int wy = win / p.nwx, wx = win - (win / p.nwx) * p.nwx;
  const int X0 = wx * p.w - p.pl;
  const int Y0 = wy * p.w - p.pt;
  const int w = p.w;

  // q tile with no real row (fully padded window rows): nothing to compute or store
  {
    const int ylo = Y0 + qt * p.rpt, yhi = ylo + p.rpt;
    if (yhi <= 0 || ylo >= p.H) return;
  }

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + TILE_BYTES;
  uint8_t* sV = sK + TILE_BYTES;
  uint8_t* sP = sV + TILE_BYTES;             // 128 rows x 128 keys bf16, two 64-key SW128 blocks
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 128 * 256);
  uint64_t* bar_q = bars + 0;
  uint64_t* bar_kv = bars + 1;
  uint64_t* bar_s = bars + 2;
  uint64_t* bar_o = bars + 3;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int kv_n = p.tile_slots;
  const uint32_t tile_bytes_tx = (uint32_t)(p.tile_slots * ROWB);

  if (tid == 0) {
    tma_prefetch_desc(&tmQKV);
    mbar_init(bar_q, 1);
    mbar_init(bar_kv, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_o, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem;         // columns [0, kv_n)
  const uint32_t tO = tmem + 128;   // columns [128, 128 + D)
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;

  const uint64_t pol = policy_evict_first();
  if (tid == 0) {
    mbar_arrive_expect_tx(bar_q, tile_bytes_tx);
    tma_load_5d(sQ, &tmQKV, bar_q, 0, h, X0, Y0 + qt * p.rpt, b, pol);
    mbar_arrive_expect_tx(bar_kv, 2 * tile_bytes_tx);
    tma_load_5d(sK, &tmQKV, bar_kv, 0, p.heads + h, X0, Y0, b, pol);
    tma_load_5d(sV, &tmQKV, bar_kv, 0, 2 * p.heads + h, X0, Y0, b, pol);
  }

  const uint32_t idesc_s = make_idesc_bf16(128, kv_n, 0, 0);
  const uint32_t idesc_o = make_idesc_bf16(128, D, 0, 1);
  float o_acc[D];
#pragma unroll
  for (int j = 0; j < D; ++j) o_acc[j] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;

  for (int kt = 0; kt < p.n_tiles; ++kt) {
    const uint32_t ph = kt & 1;
    mbar_wait(bar_kv, ph);
    if (p.patch) {
      // LEARNABLE pad patch: slot rows outside the grid get the projected pad token's K (rotated) and V.
      if (tid < kv_n) {
        const int iy = kt * p.rpt + tid / w, ix = tid % w;
        const int Y = Y0 + iy, X = X0 + ix;
        if (Y < 0 || Y >= p.H || X < 0 || X >= p.W) {
          const uint4* kx = reinterpret_cast<const uint4*>(p.kx + ((size_t)(X + p.pl) * p.heads + h) * (D / 2));
          const uint4* ky = reinterpret_cast<const uint4*>(p.ky + ((size_t)(Y + p.pt) * p.heads + h) * (D / 2));
          const uint4* vp = reinterpret_cast<const uint4*>(p.vp + (size_t)h * D);
#pragma unroll
          for (int c = 0; c < D / 16; ++c) {
            *reinterpret_cast<uint4*>(sK + swz_offset(tid, c, ROWB)) = kx[c];
            *reinterpret_cast<uint4*>(sK + swz_offset(tid, c + D / 16, ROWB)) = ky[c];
          }
#pragma unroll
          for (int c = 0; c < D / 8; ++c) *reinterpret_cast<uint4*>(sV + swz_offset(tid, c, ROWB)) = vp[c];
        }
      }
      fence_proxy_async_smem();
      __syncthreads();
    }
    if (kt == 0) mbar_wait(bar_q, 0);
    // ---- S = Q K^T  (M=128, N=kv_n, K=D)
    if (tid == 0) {
      tc_fence_after();
      const uint32_t qa = smem_u32(sQ), ka = smem_u32(sK);
#pragma unroll
      for (int k = 0; k < D / 16; ++k)
        umma_ss(tS, make_sdesc(qa + k * 32, 16, SBO, LAYOUT), make_sdesc(ka + k * 32, 16, SBO, LAYOUT), idesc_s,
                k > 0);
      umma_commit(bar_s);
    }
    mbar_wait(bar_s, ph);
    tc_fence_after();

    // ---- online softmax for row `tid` over this tile's kv_n keys (App. A.5)
    const bool masked = p.pad_mode == 1;
    float mx = -INFINITY;
    for (int c0 = 0; c0 < kv_n; c0 += 16) {
      uint32_t r[16];
      tmem_ld16(tS + lane_base + c0, r);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        bool valid = true;
        if (masked) {
          const int col = c0 + j;
          const int Y = Y0 + kt * p.rpt + col / w, X = X0 + col % w;
          valid = (Y >= 0 && Y < p.H && X >= 0 && X < p.W);
        }
        if (valid) mx = fmaxf(mx, __uint_as_float(r[j]) * p.sl2);
      }
    }
    const float m_new = fmaxf(m_run, mx);
    const float base = (m_new == -INFINITY) ? 0.f : m_new;
    const float corr = (m_run == -INFINITY) ? 0.f : ex2_approx(m_run - base);
    float lsum = 0.f;
    for (int c0 = 0; c0 < kv_n; c0 += 16) {
      uint32_t r[16];
      tmem_ld16(tS + lane_base + c0, r);
      tmem_wait_ld();
      float pv[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        bool valid = true;
        if (masked) {
          const int col = c0 + j;
          const int Y = Y0 + kt * p.rpt + col / w, X = X0 + col % w;
          valid = (Y >= 0 && Y < p.H && X >= 0 && X < p.W);
        }
        pv[j] = valid ? ex2_approx(__uint_as_float(r[j]) * p.sl2 - base) : 0.f;
        lsum += pv[j];
      }
      // two 8-key chunks -> swizzled K-major P (64 keys per 128-byte row block)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int chunk = (c0 >> 3) + hh;
        uint4 v;
        v.x = pack_bf16(pv[hh * 8 + 0], pv[hh * 8 + 1]);
        v.y = pack_bf16(pv[hh * 8 + 2], pv[hh * 8 + 3]);
        v.z = pack_bf16(pv[hh * 8 + 4], pv[hh * 8 + 5]);
        v.w = pack_bf16(pv[hh * 8 + 6], pv[hh * 8 + 7]);
        *reinterpret_cast<uint4*>(sP + (chunk >> 3) * 16384 + swz_offset(tid, chunk & 7, 128)) = v;
      }
    }
    l_run = l_run * corr + lsum;
    m_run = m_new;
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();

    // ---- O_tile = P V  (M=128, N=D, K=kv_n); V is MN-major (rows = keys)
    if (tid == 0) {
      tc_fence_after();
      const uint32_t pa = smem_u32(sP), va = smem_u32(sV);
      for (int ks = 0; ks < kv_n / 16; ++ks) {
        uint64_t ad = make_sdesc(pa + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024, kLayoutSW128);
        uint64_t bd = make_sdesc(va + ks * 16 * ROWB, TILE_BYTES, SBO, LAYOUT);
        umma_ss(tO, ad, bd, idesc_o, ks > 0);
      }
      umma_commit(bar_o);
    }
    mbar_wait(bar_o, ph);
    tc_fence_after();
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 16) {
      uint32_t r[16];
      tmem_ld16(tO + lane_base + c0, r);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) o_acc[c0 + j] = o_acc[c0 + j] * corr + __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    // next K/V tile into the (now free) buffers
    if (tid == 0 && kt + 1 < p.n_tiles) {
      mbar_arrive_expect_tx(bar_kv, 2 * tile_bytes_tx);
      tma_load_5d(sK, &tmQKV, bar_kv, 0, p.heads + h, X0, Y0 + (kt + 1) * p.rpt, b, pol);
      tma_load_5d(sV, &tmQKV, bar_kv, 0, 2 * p.heads + h, X0, Y0 + (kt + 1) * p.rpt, b, pol);
    }
  }

  // ---- normalise and write this thread's row straight to the grid (merge/crop: pad query rows are dropped).
  // (A TMA tensor store would clip the box, but box origins left of / above the grid are illegal for stores.)
  {
    const int iy = qt * p.rpt + tid / w, ix = tid % w;
    const int Y = Y0 + iy, X = X0 + ix;
    if (tid < p.tile_slots && Y >= 0 && Y < p.H && X >= 0 && X < p.W) {
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      uint4* dst = reinterpret_cast<uint4*>(p.out + (((size_t)b * p.H + Y) * p.W + X) * p.C + (size_t)h * D);
#pragma unroll
      for (int c = 0; c < D / 8; ++c) {
        uint4 v;
        v.x = pack_bf16(o_acc[c * 8 + 0] * inv, o_acc[c * 8 + 1] * inv);
        v.y = pack_bf16(o_acc[c * 8 + 2] * inv, o_acc[c * 8 + 3] * inv);
        v.z = pack_bf16(o_acc[c * 8 + 4] * inv, o_acc[c * 8 + 5] * inv);
        v.w = pack_bf16(o_acc[c * 8 + 6] * inv, o_acc[c * 8 + 7] * inv);
        dst[c] = v;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

// Pad tables for the LEARNABLE patch: kx[X+pl][h][0:d/2] = rot_X(k_p[h][0:d/2]), ky[Y+pt][h][0:d/2] =
// rot_Y(k_p[h][d/2:d]), vp[h][:] = v_p[h][:]  (bf16; rotation in f32 from the f32 projection of p).
__global__ void pad_tables_kernel(const float* __restrict__ qkv_pad, int C, int heads, int d, int Wp, int Hp, int pl,
                                  int pt, int rope, int row0, __nv_bfloat16* kx, __nv_bfloat16* ky,
                                  __nv_bfloat16* vp) {
  pdl_trigger();
  pdl_wait();
  const int half = d / 2;
  const int nx = Wp * heads * half, ny = Hp * heads * half, nv = heads * d;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nx + ny) {
    const bool isy = i >= nx;
    int k = isy ? i - nx : i;
    const int pos_idx = k / (heads * half);
    const int hh = (k / half) % heads;
    const int e = k % half;  // element within the half
    const int pos = pos_idx - (isy ? pt - row0 : pl);
    const float* kp = qkv_pad + C + hh * d + (isy ? half : 0);
    float val;
    if (rope) {
      const int jpair = e >> 1;
      float c, sn;
      rope_cs(pos, jpair, d, c, sn);
      const float a = kp[jpair * 2], bb = kp[jpair * 2 + 1];
      val = (e & 1) ? (a * sn + bb * c) : (a * c - bb * sn);
    } else {
      val = kp[e];
    }
    (isy ? ky : kx)[k] = __float2bfloat16_rn(val);
  } else if (i < nx + ny + nv) {
    int k = i - nx - ny;
    vp[k] = __float2bfloat16_rn(qkv_pad[2 * C + k]);
  }
}

size_t attn_pad_table_bytes(int H, int W, int C, int w) {
  size_t Wp = (size_t)W + 2 * w, Hp = (size_t)H + 2 * w;
  size_t bytes = (Wp + Hp) * (size_t)C / 2 * 2 + (size_t)C * 2;
  return (bytes + 255) & ~size_t(255);
}

int launch_pad_tables(const AttnArgs& a, cudaStream_t stream) {
  const int d = a.d, w = a.w;
  const int pl = (w - a.sx) % w, pt = (w - a.sy) % w;
  const int Wp = pl + a.W + ((-(pl + a.W)) % w + w) % w;
  const int Hp = pt + a.H + ((-(pt + a.H)) % w + w) % w;
  if (!a.qkv_pad || !a.pad_tab) return -3;
  __nv_bfloat16* kx = reinterpret_cast<__nv_bfloat16*>(a.pad_tab);
  __nv_bfloat16* ky = kx + (size_t)Wp * a.C / 2;
  __nv_bfloat16* vp = ky + (size_t)Hp * a.C / 2;
  const int n = (Wp + Hp) * a.C / 2 + a.C;
  PSCWIN_PROF("pad_tables", stream);
  launch_k(pad_tables_kernel, dim3((n + 255) / 256), dim3(256), 0, stream, a.qkv_pad, a.C, a.heads, d, Wp, Hp, pl, pt,
           a.rope, a.row0, kx, ky, vp);
  return (int)cudaGetLastError();
}

int launch_window_attention(const AttnArgs& a, cudaStream_t stream) {
  const int d = a.d;
  if (!(d == 32 || d == 64)) return -2;
  const int w = a.w;
  if (w < 4 || w > 128 || (w & (w - 1))) return -2;
  AttnKArgs p;
  p.B = a.B;
  p.H = a.H;
  p.W = a.W;
  p.C = a.C;
  p.heads = a.heads;
  p.w = w;
  p.pl = (w - a.sx) % w;
  p.pt = (w - a.sy) % w;
  const int pr = ((-(p.pl + a.W)) % w + w) % w;
  const int pb = ((-(p.pt + a.H)) % w + w) % w;
  p.Wp = p.pl + a.W + pr;
  p.Hp = p.pt + a.H + pb;
  p.nwx = p.Wp / w;
  p.nw = (p.Hp / w) * p.nwx;
  p.pad_mode = a.pad_mode;
  const bool shifted = a.sx != 0 || a.sy != 0;
  p.patch = (shifted && a.pad_mode == 0) ? 1 : 0;
  p.rpt = w * w <= 128 ? w : 128 / w;
  p.n_tiles = w / p.rpt;
  p.tile_slots = w * p.rpt;
  p.sl2 = 1.4426950408889634f / sqrtf((float)d);
  p.kx = p.ky = p.vp = nullptr;
  if (p.patch) {
    if (!a.qkv_pad || !a.pad_tab) return -3;
    __nv_bfloat16* kx = reinterpret_cast<__nv_bfloat16*>(a.pad_tab);
    __nv_bfloat16* ky = kx + (size_t)p.Wp * a.C / 2;
    __nv_bfloat16* vp = ky + (size_t)p.Hp * a.C / 2;
    p.kx = kx;
    p.ky = ky;
    p.vp = vp;
    if (!a.tables_ready) {
      const int rc = launch_pad_tables(a, stream);
      if (rc) return rc;
    }
  }
  // windows of <= 256 slots: persistent warp-specialised kernel (attn_sm100_ws.cu); PSCWIN_ATTN_V1=1 forces this
  // file's one-CTA-per-(q tile, head, window) kernel, which also serves larger windows.
  static const bool force_v1 = env_knob("PSCWIN_ATTN_V1", 0) == 1;
  if (p.n_tiles <= 2 && !force_v1)
    return launch_window_attention_ws(a, p.kx, p.ky, p.vp, p.patch, stream);
  CUtensorMap tmQKV;
  const uint64_t dq[5] = {(uint64_t)d, (uint64_t)3 * a.heads, (uint64_t)a.W, (uint64_t)a.H, (uint64_t)a.B};
  const uint64_t sq[4] = {(uint64_t)d * 2, (uint64_t)3 * a.C * 2, (uint64_t)a.W * 3 * a.C * 2,
                          (uint64_t)a.H * a.W * 3 * a.C * 2};
  const uint32_t box[5] = {(uint32_t)d, 1, (uint32_t)w, (uint32_t)p.rpt, 1};
  const CUtensorMapSwizzle swz = d == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  int rc = make_tmap_5d(&tmQKV, a.qkv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, dq, sq, box, swz);
  if (rc) return rc;
  p.out = reinterpret_cast<__nv_bfloat16*>(a.out);
  const size_t smem = 1024 + 3 * 128 * d * 2 + 128 * 256 + 64;
  {
    const int nwy = p.nw / p.nwx;
    const int wy0 = a.wy_end > 0 ? a.wy_begin : 0, wy1 = a.wy_end > 0 ? (a.wy_end < nwy ? a.wy_end : nwy) : nwy;
    if (wy0 < 0 || wy0 >= wy1) return 0;
    p.win0 = wy0 * p.nwx;
    p.nw_run = (wy1 - wy0) * p.nwx;
  }
  dim3 grid(p.n_tiles, a.heads, a.B * p.nw_run);
  PSCWIN_PROF("window_attention", stream);
  if (d == 64) {
    func_smem_once((const void*)window_attn_kernel<64>, (int)smem);
    launch_k(window_attn_kernel<64>, dim3(grid), dim3(ATT_THREADS), smem, stream, tmQKV, p);
  } else {
    func_smem_once((const void*)window_attn_kernel<32>, (int)smem);
    launch_k(window_attn_kernel<32>, dim3(grid), dim3(ATT_THREADS), smem, stream, tmQKV, p);
  }
  return (int)cudaGetLastError();
}

}  // namespace pscwin
