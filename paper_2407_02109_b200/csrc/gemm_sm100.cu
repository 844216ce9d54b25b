// Projection GEMMs of the PSCWin layer on 5th-gen tensor cores:
//   out[M, N] = epilogue( A[M, K] . B[N, K]^T )      A, B bf16 K-major (activations x nn.Linear weight [out, in])
// Epilogues: plain bf16 / f32 store (in_proj, x_proj), bias + 2-D RoPE at the token's grid coordinate (QKV, a4,
// PAPER P:L89 "replaces SAM's relative encoding with RoPE", form = DESIGN.md reading Q6), bias + residual
// (out-proj a7 / cycle-scan out_proj a3).
//
// Structure (B200-native): persistent grid (one CTA per SM), warp-specialised —
//   warp 0: TMA producer (128B-swizzled A/B k-blocks of 64, 4-stage mbarrier ring)
//   warp 1: TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN<=256, K=16 per instruction)
//   warps 2-9: epilogue (tcgen05.ld 32x32b -> registers -> fused op -> per-warp swizzled smem box -> TMA store),
//   double-buffered TMEM accumulators (2 x 256 columns) so the epilogue of tile i overlaps the MMAs of tile i+1.
#include <stdlib.h>
#include <string.h>

#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "pscwin_internal.h"

namespace pscwin {

namespace {
constexpr int BM = 128;                          // accumulator rows per CTA (TMEM lanes)
constexpr int BK = 64;
constexpr int MAX_STAGES = 8;
constexpr int A_STAGE_BYTES = BM * BK * 2;       // 16 KB
constexpr int STAGE_OUT_BYTES = BM * 64 * 2;     // one 128x64 bf16 output / residual chunk (16 KB)
constexpr int GEMM_THREADS = 64 + 256;           // TMA warp, MMA warp, 8 epilogue warps
constexpr size_t GEMM_SMEM_MAX = 232448;         // 227 KB opt-in limit per CTA
// shared memory layout: [1 KB align slack][stages x (A 128x64 | B rows x 64)][output staging][residual tiles]
// [bias / LN sums][barriers]; B rows per CTA = BN (single CTA) or BN / 2 (CTA pair)
struct EpiSmem {
  size_t stg, res;  // output staging bytes, residual bytes
};
__host__ __device__ inline EpiSmem gemm_epi_smem(int BN, bool resid, bool f32, int warp_epi, int nbuf, int res_global) {
  const size_t nbx = (size_t)(BN + 31) / 32;
  // f32 outputs: four 16 KB staging boxes (a 64-column f32 chunk is two 128 x 32 boxes; two chunks in flight)
  if (f32) return {2 * (size_t)STAGE_OUT_BYTES, 2 * (size_t)STAGE_OUT_BYTES};
  // per-warp epilogue with the residual in shared memory: 32-column boxes of 128 rows, the output written over them
  if (resid && !res_global) return {0, (BN > 128 ? 1 : 2) * nbx * (size_t)(STAGE_OUT_BYTES / 2)};
  // per-warp epilogue, residual (if any) read from global memory: nbuf 2 KB staging boxes per epilogue warp
  return {(size_t)8 * nbuf * 2048, 0};
}
__host__ __device__ inline size_t gemm_fixed_bytes(const EpiSmem& e) {
  return 1024 + e.stg + e.res + 4 * 256 * 4 + 256;  // bias + LN column sums (double-buffered), barriers
}
__host__ __device__ inline size_t gemm_stage_bytes(int BN, bool pair) {
  return A_STAGE_BYTES + (size_t)(pair ? BN / 2 : BN) * BK * 2;
}
}  // namespace

// four per-column values (bias, LayerNorm column sums) at columns c..c+3 read through L1 (every lane of a warp reads
// the same addresses: broadcast), zero past N
__device__ __forceinline__ float4 bias_l1_4(const float* v, int c, int N) {
  if (c + 4 <= N) return __ldg(reinterpret_cast<const float4*>(v + c));
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
  float* rp = reinterpret_cast<float*>(&r);
  for (int e = 0; e < 4 && c + e < N; ++e) rp[e] = __ldg(v + c + e);
  return r;
}

__device__ __forceinline__ void rope_pair(float& a, float& b, float c, float s) {
  float x0 = a * c - b * s;
  float x1 = a * s + b * c;
  a = x0;
  b = x1;
}

// PAIR: a 2-CTA cluster shares each 256-row tile: tcgen05.mma.cta_group::2 (M = 256) issued by the leader CTA
// reads A rows [0,128) / [128,256) and B rows [0,BN/2) / [BN/2,BN) from the two CTAs' shared memory; each CTA's
// TMEM holds its 128 accumulator rows x BN columns and its own epilogue stores them. Per SM this halves the B
// bytes per MAC (the L2 -> SM traffic that bounds 1-CTA 128-row tiles).
// EK: epilogue kind, a compile-time specialisation so each variant's registers are allocated for its own work
// (EK_ROPE keeps 32 cos / sin values per row live across the tile; EK_GELU inlines 32 GELUs per chunk).
enum { EK_PLAIN = 0, EK_ROPE = 1, EK_GELU = 2, EK_F32 = 3 };
// MC = 2 (CTA pairs only): a 4-CTA cluster of two pairs takes two vertically adjacent 256-row tiles of the same
// column tile; every B k-block is loaded once per cluster (each CTA loads a quarter and multicasts it to the CTA of
// the same pair rank in both pairs), halving the B bytes moved from L2 (which would bound the big projections if
// their ~10 TB/s of A + B tile reads at 4096^2 were at the L2 limit). Measured bit-identical but 2-4 % slower (the
// 4-CTA clusters couple two pairs' rings and may leave SMs idle), so it is off by default (mc_enabled).
template <bool PAIR, int EK, int MC = 1>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmOut, const __grid_constant__ CUtensorMap tmRes,
                     GemmArgs p) {
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  const int BN = p.BN;
  const int STAGES = p.stages;
  const int B_STAGE_BYTES = (PAIR ? BN / 2 : BN) * BK * 2;
  const uint32_t crank = PAIR ? cluster_ctarank() : 0u;
  const uint32_t rank = crank & 1u;              // rank inside the pair
  const uint32_t pp = MC > 1 ? crank >> 1 : 0u;  // pair inside the cluster (MC = 2)
  const uint32_t lead = pp * 2u;                 // cluster rank of this pair's leader
  const bool resid = p.epi == EPI_RESID_BF16 && p.residual != nullptr;
  constexpr bool res_gmem_ek = EK == EK_PLAIN;                       // (only plain epilogues carry a residual)
  const bool res_gmem = res_gmem_ek && resid && p.res_global;  // the epilogue reads the residual from global
  const bool resid_tma = resid && !res_gmem;                   // residual tiles TMA-loaded into shared memory
  const int nch = (BN + 63) / 64;
  const EpiSmem es = gemm_epi_smem(BN, resid, EK == EK_F32, p.warp_epi, p.nbuf, p.res_global);
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
  uint8_t* s_stage = sB + STAGES * B_STAGE_BYTES;   // output staging (1024-aligned)
  uint8_t* s_res = s_stage + es.stg;                // residual tiles (TMA-loaded)
  // residual tiles: double-buffered (BN <= 128) or one set written over in place by the output (BN > 128)
  const bool res_inplace = resid_tma && BN > 128;
  float* s_bias = reinterpret_cast<float*>(s_res + es.res);  // [2][256] bias, then [2][256] LN s_n
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_bias + 4 * 256);
  uint64_t* full = bars;                 // [STAGES]
  uint64_t* empty = bars + STAGES;       // [STAGES]
  uint64_t* tfull = bars + 2 * STAGES;   // [2]
  uint64_t* tempty = bars + 2 * STAGES + 2;  // [2]
  uint64_t* rfull = bars + 2 * STAGES + 4;   // [2] residual tile landed
  uint64_t* rempty = bars + 2 * STAGES + 6;  // [2] residual tile consumed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 8);
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = warp_id();
  constexpr int TM = PAIR ? 2 * BM : BM;          // tile rows (the pair's 256 or one CTA's 128)
  const int n_tiles_n = (p.N + BN - 1) / BN;
  const int S = p.splits > 1 ? p.splits : 1;  // split-K factor (f32 outputs only; single-CTA tiles)
  const int n_tiles = ((p.M + MC * TM - 1) / (MC * TM)) * n_tiles_n * S;
  const int tile0 = PAIR ? (int)(blockIdx.x / (2 * MC)) : (int)blockIdx.x;   // this CTA's (cluster's) first tile
  const int tstride = PAIR ? (int)(gridDim.x / (2 * MC)) : (int)gridDim.x;
  const int BKe = p.tf32 ? BK / 2 : BK;  // K elements per 128-byte k-block row (bf16: 64, tf32: 32)
  const int nk = (p.K + BKe - 1) / BKe;
  // work tile -> output tile (m0, n0), k-block range [kb0, kb1) and split index
  auto coords = [&](int tile, int& m0, int& n0, int& kb0, int& kb1, int& s) {
    const int mn = tile / S;
    s = tile - mn * S;
    m0 = (mn / n_tiles_n) * (MC * TM) + (int)pp * TM;
    n0 = (mn % n_tiles_n) * BN;
    kb0 = (int)((long long)nk * s / S);
    kb1 = (int)((long long)nk * (s + 1) / S);
  };

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (p.epi != EPI_STORE_F32 || p.f32_tma) tma_prefetch_desc(&tmOut);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], MC);  // one multicast commit per pair that reads this CTA's stage
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], PAIR ? 16 : 8);  // one arrival per epilogue warp (of both CTAs of a pair)
      mbar_init(&rfull[i], 1);
      // each epilogue warp's lane 0, once that warp's in-place stores have read the residual set out
      mbar_init(&rempty[i], 8);
    }
    if (resid) tma_prefetch_desc(&tmRes);
    fence_barrier_init();
  }
  if (warp == 1) {
    if (PAIR)
      tmem_alloc_pair(tmem_slot, 512);
    else
      tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // the peer's barriers are initialised before any cross-CTA signal
  tc_fence_after();
  pdl_wait();  // barrier init / TMEM allocation / descriptor prefetch overlap the previous kernel
  const uint32_t tmem_base = *tmem_slot;
  // rows of the tile that this CTA loads / stores: [m0 + mrow, m0 + mrow + 128)
  const int mrow = PAIR ? (int)rank * BM : 0;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_a = policy_evict_normal();
      const uint64_t pol_b = policy_evict_last();
      // CTA pair: both CTAs' loads complete on the leader's full barrier (it issues the MMAs)
      const uint32_t full0 = PAIR ? smem_in_cta(&full[0], lead) : 0u;
      int stage = 0;
      uint32_t phase = 0;
      int rbuf = 0;
      uint32_t rphase = 0;
      auto load_res = [&](int m0, int n0, int buf) {  // this CTA's residual rows of the tile
        if (m0 + mrow >= p.M) {
          mbar_arrive(&rfull[buf]);  // no rows of this CTA in the tile: nothing to load
        } else {  // 32-column SW64 boxes of 128 rows (the per-warp epilogue's layout)
          const int nbx = (BN + 31) / 32;
          int nb = 0;
          for (int c = 0; c < nbx; ++c) nb += n0 + c * 32 < p.N;
          mbar_arrive_expect_tx(&rfull[buf], nb * (STAGE_OUT_BYTES / 2));
          for (int c = 0; c < nbx; ++c)
            if (n0 + c * 32 < p.N)
              tma_load_2d(s_res + (size_t)(buf * nbx + c) * (STAGE_OUT_BYTES / 2), &tmRes, &rfull[buf], n0 + c * 32,
                          m0 + mrow, pol_a);
        }
      };
      for (int tile = tile0; tile < n_tiles; tile += tstride) {
        int m0, n0, kb0, kb1, s;
        coords(tile, m0, n0, kb0, kb1, s);
        // in place: the single residual set is refilled once the previous tile's stores have read it out; probe
        // that between k-block loads so the mainloop never waits for it
        bool res_pending = res_inplace;
        auto try_res = [&](bool block) {
          if (!res_pending) return;
          if (block) mbar_wait(&rempty[0], rphase ^ 1);
          else if (!mbar_test(&rempty[0], rphase ^ 1)) return;
          load_res(m0, n0, 0);
          rphase ^= 1;
          res_pending = false;
        };
        if (res_gmem) {  // the epilogue reads this tile's residual from global memory: warm L2 with it now
          const int nbx = (BN + 31) / 32;
          if (m0 + mrow < p.M)
            for (int c = 0; c < nbx; ++c)
              if (n0 + c * 32 < p.N) tma_prefetch_l2_2d(&tmRes, n0 + c * 32, m0 + mrow);
        }
        if (resid_tma && !res_inplace) {
          // residual tile of this CTA's rows (double-buffered, consumed by the epilogue), issued ahead of the k-loop
          mbar_wait(&rempty[rbuf], rphase ^ 1);
          load_res(m0, n0, rbuf);
          if (++rbuf == 2) {
            rbuf = 0;
            rphase ^= 1;
          }
        }
        if (PAIR) {
          // boxes entirely outside A (rows >= M) or B (rows >= N) are not loaded; their bytes are not expected
          const bool a0_in = m0 < p.M, a1_in = m0 + BM < p.M;
          const bool b0_in = n0 < p.N, b1_in = n0 + BN / 2 < p.N;
          uint32_t bytes = ((int)a0_in + (int)a1_in) * A_STAGE_BYTES + ((int)b0_in + (int)b1_in) * B_STAGE_BYTES;
          const bool a_mine = rank ? a1_in : a0_in;
          bool b_mine = rank ? b1_in : b0_in;
          // MC = 2: B quarter (r, q) = rows n0 + r BN/2 + q BN/4 lands at offset q QB of the B stage of both pairs'
          // rank-r CTAs; this CTA loads quarter (rank, pp)
          const int QR = BN / 4;
          const uint32_t QB = (uint32_t)QR * BK * 2;
          const int qrow = n0 + (int)rank * (BN / 2) + (int)pp * QR;
          if (MC > 1) {
            bytes = ((int)a0_in + (int)a1_in) * A_STAGE_BYTES;
            for (int q = 0; q < 4; ++q) bytes += (n0 + q * QR < p.N) ? QB : 0u;
            b_mine = qrow < p.N;
          }
          const uint16_t qmask = (uint16_t)((1u << rank) | (1u << (2 + rank)));
          for (int kb = kb0; kb < kb1; ++kb) {
            try_res(false);
            mbar_wait(&empty[stage], phase ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], bytes);
            const uint32_t fb = full0 + stage * 8;
            if (a_mine) tma_load_2d_pair(sA + stage * A_STAGE_BYTES, &tmA, fb, kb * BKe, m0 + mrow, pol_a);
            if (MC > 1) {
              if (b_mine)
                tma_load_2d_pair_mc(sB + stage * B_STAGE_BYTES + pp * QB, &tmB, fb, kb * BKe, qrow, qmask, pol_b);
            } else if (b_mine) {
              tma_load_2d_pair(sB + stage * B_STAGE_BYTES, &tmB, fb, kb * BKe, n0 + (int)rank * (BN / 2), pol_b);
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        } else {
          for (int kb = kb0; kb < kb1; ++kb) {
            try_res(false);
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], A_STAGE_BYTES + B_STAGE_BYTES);
            tma_load_2d(sA + stage * A_STAGE_BYTES, &tmA, &full[stage], kb * BKe, m0, pol_a);
            tma_load_2d(sB + stage * B_STAGE_BYTES, &tmB, &full[stage], kb * BKe, n0, pol_b);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
        try_res(true);
      }
    }
  } else if (warp == 1) {
    if (!PAIR || rank == 0) {
      const uint32_t idesc = p.tf32 ? make_idesc_tf32(TM, BN) : make_idesc_bf16(TM, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = tile0; tile < n_tiles; tile += tstride) {
        int m0, n0, kb0, kb1, s;
        coords(tile, m0, n0, kb0, kb1, s);
        if (PAIR)
          mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
        else
          mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = kb0; kb < kb1; ++kb) {
          if (PAIR)
            mbar_wait_cluster(&full[stage], phase);
          else
            mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a0 = smem_u32(sA + stage * A_STAGE_BYTES);
            const uint32_t b0 = smem_u32(sB + stage * B_STAGE_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              uint64_t ad = make_sdesc(a0 + k * 32, 16, 1024, kLayoutSW128);
              uint64_t bd = make_sdesc(b0 + k * 32, 16, 1024, kLayoutSW128);
              const uint32_t accum = (kb != kb0 || k != 0) ? 1u : 0u;
              if (p.tf32) {
                if (PAIR)
                  umma_ss_pair_tf32(d_tmem, ad, bd, idesc, accum);
                else
                  umma_ss_tf32(d_tmem, ad, bd, idesc, accum);
              } else if (PAIR) {
                umma_ss_pair(d_tmem, ad, bd, idesc, accum);
              } else {
                umma_ss(d_tmem, ad, bd, idesc, accum);
              }
            }
            if (PAIR) {
              // frees the stage in both CTAs (MC = 2: in all four, whose B quarters this pair's MMAs read)
              umma_commit_pair_mc(&empty[stage], MC > 1 ? 0xF : 0x3);
              if (kb == kb1 - 1) umma_commit_pair_mc(&tfull[acc], (uint16_t)(0x3u << lead));
            } else {
              umma_commit(&empty[stage]);
              if (kb == kb1 - 1) umma_commit(&tfull[acc]);
            }
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue warps 2..9
    // Two warps per TMEM lane quarter (rows), each taking 32 of every 64 accumulator columns. bf16 outputs: each
    // warp stages its own 32 x 32 boxes (SW64) and TMA-stores them (no CTA-wide barrier per chunk); f32 outputs: per
    // -warp 32 x 32 f32 boxes (SW128) or direct stores (split-K).
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int lane = lane_id();
    const int etid = threadIdx.x - 64;                 // 0..255
    const bool issuer = etid == 0;
    const bool tma_out = EK != EK_F32;
    const bool f32_tma = EK == EK_F32 && S == 1 && p.f32_tma;  // f32 tiles staged in smem, TMA-stored
    const int row_local = quarter * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    int gseq = 0;
    int rbuf = 0;
    uint32_t rphase = 0;
    const uint32_t tempty0 = PAIR ? smem_in_cta(&tempty[0], lead) : 0u;  // the leader's accumulator-free barriers
    for (int tile = tile0; tile < n_tiles; tile += tstride) {
      int m0, n0, kb0, kb1, split;
      coords(tile, m0, n0, kb0, kb1, split);
      const int mb = m0 + mrow;                          // first row of this CTA's 128
      const int row = mb + row_local;
      const bool row_ok = row < p.M;
      // RoPE of this row (QKV epilogue): this thread's 32 columns of every 64-column chunk are one half of a head
      // (d = 64: axis = half, pair jj -> frequency jj) or one whole head (d = 32: pairs 0-7 x, 8-15 y).
      float rc[EK == EK_ROPE ? 16 : 1], rs[EK == EK_ROPE ? 16 : 1];
      if (EK == EK_ROPE && p.rope) {
        int r = row + p.tok0, HW = p.HW, Wg = p.Wgrid;
        if (p.nseg > 1) {  // packed multi-scale rows: each scale's grid has its own coordinates (reading Q20)
          int r0 = 0;
#pragma unroll
          for (int sg = 0; sg < 4; ++sg)
            if (sg < p.nseg && r >= p.seg_row[sg]) {
              r0 = p.seg_row[sg];
              HW = p.seg_HW[sg];
              Wg = p.seg_W[sg];
            }
          r -= r0;
        }
        const int t = r % HW;
        const int py = t / Wg, px = t - py * Wg;
        if constexpr (EK == EK_ROPE) {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const int axis = p.d_head == 64 ? half : (jj >= 8);
            const int fj = p.d_head == 64 ? jj : (jj & 7);
            rope_cs(axis ? py : px, fj, p.d_head, rc[jj], rs[jj]);
          }
        }
      }
      // bias of the tile's columns staged once in shared memory (read back as broadcasts), double-buffered by
      // accumulator so the next tile's staging never races this tile's readers
      float* sb = s_bias + acc * 256;
      float* sc = s_bias + 512 + acc * 256;              // LN column sums s_n (folded LayerNorm)
      const bool ln = EK != EK_F32 && p.ln_stats != nullptr;
      float ln_r = 1.f, ln_nmr = 0.f;                    // rstd and -mu * rstd of this row
      if (ln && row_ok) {
        const float2 st = __ldg(p.ln_stats + row);
        ln_r = st.y;
        ln_nmr = -st.x * st.y;
      }
      if (EK != EK_F32 && p.bias && !p.bias_l1) {  // (f32 tiles / bias_l1 read the bias straight from L1)
        if (etid < BN / 4) {
          const int c = n0 + 4 * etid;
          float4 b4 = make_float4(0.f, 0.f, 0.f, 0.f), s4 = make_float4(0.f, 0.f, 0.f, 0.f);
          if (c + 4 <= p.N) {
            b4 = __ldg(reinterpret_cast<const float4*>(p.bias + c));
            if (ln) s4 = __ldg(reinterpret_cast<const float4*>(p.ln_colsum + c));
          } else {
            float* bp = reinterpret_cast<float*>(&b4);
            float* sp = reinterpret_cast<float*>(&s4);
            for (int e = 0; e < 4 && c + e < p.N; ++e) {
              bp[e] = __ldg(p.bias + c + e);
              if (ln) sp[e] = __ldg(p.ln_colsum + c + e);
            }
          }
          reinterpret_cast<float4*>(sb)[etid] = b4;
          if (ln) reinterpret_cast<float4*>(sc)[etid] = s4;
        }
      }
      if constexpr (EK != EK_F32) {
        // ---------------------------------------------------------- per-warp bf16 epilogue
        // Warp (quarter, half) owns rows [32 quarter, +32) and the 32-column boxes i = half, half + 2, ... of the
        // tile. Each box goes TMEM -> registers (the next box's TMEM load is in flight meanwhile) -> fused op ->
        // a 2 KB SW64 staging box (this warp's own double buffer, or the residual box in place) -> one TMA store
        // by the warp's lane 0. The only CTA-wide barrier is the one per tile that publishes the staged bias.
        if (p.bias && !p.bias_l1) named_bar_sync(1, 256);
        const int nbx = p.dbg_noepi ? 0 : (BN + 31) / 32;  // (timing probe: no epilogue work at all)
        // residual from global memory (L2-warm: the producer prefetched the tile): this thread's 64 bytes of row
        // `row` per box, loaded one box ahead (the first box's before the accumulator wait). (Measured: loading all
        // of a warp's boxes up front with the box loop unrolled was slower for every GEMM of the step.)
        const __nv_bfloat16* rg =
            res_gmem ? reinterpret_cast<const __nv_bfloat16*>(p.residual) + (size_t)row * p.ldr + n0 : nullptr;
        uint4 rcur[res_gmem_ek ? 4 : 1], rnext[res_gmem_ek ? 4 : 1];
        auto load_res4 = [&](int bx, uint4* r) {
#pragma unroll
          for (int q = 0; q < 4; ++q) r[q] = make_uint4(0u, 0u, 0u, 0u);
          if (row_ok && n0 + bx * 32 < p.N) {
            const uint4* src = reinterpret_cast<const uint4*>(rg + bx * 32);
#pragma unroll
            for (int q = 0; q < 4; ++q) r[q] = __ldcs(src + q);
          }
        };
        if constexpr (res_gmem_ek)
          if (res_gmem && half < nbx) load_res4(half, rcur);
        if (PAIR)
          mbar_wait_cluster(&tfull[acc], acc_phase);
        else
          mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        if (resid_tma) mbar_wait(&rfull[rbuf], rphase);
        const uint32_t t_row = tmem_base + acc * 256 + ((uint32_t)(quarter * 32) << 16);
        const int ew = warp - 2;
        // the next box's TMEM load is issued before this box's math
        constexpr bool kPrefetch = true;
        uint32_t ra[32];
        if (kPrefetch && half < nbx) tmem_ld32(t_row + half * 32, ra);
        for (int bx = half; bx < nbx; bx += 2) {
          const int cl = bx * 32, col0 = n0 + cl;
          if (!kPrefetch) tmem_ld32(t_row + cl, ra);
          tmem_wait_ld_dep(ra);
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(ra[j]);
          if (kPrefetch && bx + 2 < nbx) {
            tmem_ld32(t_row + cl + 64, ra);
          } else if (bx + 2 >= nbx) {  // this warp's last TMEM read of the tile: the accumulator may be reused
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (PAIR)
                mbar_arrive_remote(tempty0 + acc * 8);
              else
                mbar_arrive(&tempty[acc]);
            }
          }
          if (p.bias) {
            if (ln) {
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                const float4 b4 = p.bias_l1 ? bias_l1_4(p.bias, col0 + j, p.N) : *reinterpret_cast<const float4*>(sb + cl + j);
                const float4 s4 = p.bias_l1 ? bias_l1_4(p.ln_colsum, col0 + j, p.N)
                                            : *reinterpret_cast<const float4*>(sc + cl + j);
                v[j] = fmaf(v[j], ln_r, fmaf(ln_nmr, s4.x, b4.x));
                v[j + 1] = fmaf(v[j + 1], ln_r, fmaf(ln_nmr, s4.y, b4.y));
                v[j + 2] = fmaf(v[j + 2], ln_r, fmaf(ln_nmr, s4.z, b4.z));
                v[j + 3] = fmaf(v[j + 3], ln_r, fmaf(ln_nmr, s4.w, b4.w));
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                const float4 b4 = p.bias_l1 ? bias_l1_4(p.bias, col0 + j, p.N) : *reinterpret_cast<const float4*>(sb + cl + j);
                v[j] += b4.x; v[j + 1] += b4.y; v[j + 2] += b4.z; v[j + 3] += b4.w;
              }
            }
          }
          if constexpr (EK == EK_ROPE) {
            if (p.rope && col0 < 2 * p.C) {
#pragma unroll
              for (int jj = 0; jj < 16; ++jj) rope_pair(v[2 * jj], v[2 * jj + 1], rc[jj], rs[jj]);
            }
          }
          if constexpr (EK == EK_GELU) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = gelu_erf(v[j]);
          }
          if (EK == EK_PLAIN && p.silu_col > 0 && col0 >= p.silu_col) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __fdividef(v[j], 1.f + __expf(-v[j]));
          }
          // staging box: the residual box itself (written over in place) or one of this warp's nbuf buffers
          const int nb = p.nbuf;
          uint8_t* box = resid_tma ? s_res + ((size_t)(rbuf * nbx + bx) * 128 + quarter * 32) * 64
                                   : s_stage + (size_t)(ew * nb + (nb == 2 ? (gseq & 1) : 0)) * 2048;
          if constexpr (res_gmem_ek) if (res_gmem) {
            if (bx + 2 < nbx) load_res4(bx + 2, rnext);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 rw = rcur[q];
              rcur[q] = rnext[q];
              v[8 * q + 0] += bf16_lo(rw.x); v[8 * q + 1] += bf16_hi(rw.x);
              v[8 * q + 2] += bf16_lo(rw.y); v[8 * q + 3] += bf16_hi(rw.y);
              v[8 * q + 4] += bf16_lo(rw.z); v[8 * q + 5] += bf16_hi(rw.z);
              v[8 * q + 6] += bf16_lo(rw.w); v[8 * q + 7] += bf16_hi(rw.w);
            }
          }
          if (resid_tma) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 rw = *reinterpret_cast<const uint4*>(box + swz_offset(lane, q, 64));
              v[8 * q + 0] += bf16_lo(rw.x); v[8 * q + 1] += bf16_hi(rw.x);
              v[8 * q + 2] += bf16_lo(rw.y); v[8 * q + 3] += bf16_hi(rw.y);
              v[8 * q + 4] += bf16_lo(rw.z); v[8 * q + 5] += bf16_hi(rw.z);
              v[8 * q + 6] += bf16_lo(rw.w); v[8 * q + 7] += bf16_hi(rw.w);
            }
          } else if (gseq >= nb) {  // the store from this buffer nb boxes ago has read it out
            if (lane == 0) {
              if (nb == 2)
                bulk_wait_read1();
              else
                bulk_wait_read0();
            }
            __syncwarp();
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 w;
            w.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
            w.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
            w.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
            w.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
            *reinterpret_cast<uint4*>(box + swz_offset(lane, q, 64)) = w;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (mb + quarter * 32 < p.M && col0 < p.N) tma_store_2d(&tmOut, box, col0, mb + quarter * 32);
            bulk_commit();
          }
          ++gseq;
        }
        if (half >= nbx) {  // (a tile of one 32-column box: the second half's warps only release the accumulator)
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (PAIR)
              mbar_arrive_remote(tempty0 + acc * 8);
            else
              mbar_arrive(&tempty[acc]);
          }
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        if (resid_tma) {  // the residual set may be refilled once this warp's in-place stores have read it out
          if (lane == 0) {
            bulk_wait_read0();
            mbar_arrive(&rempty[rbuf]);
          }
          if (res_inplace) {
            rphase ^= 1;
          } else if (++rbuf == 2) {
            rbuf = 0;
            rphase ^= 1;
          }
        }
        continue;
      }
      // ---------------------------------------------------------- f32 epilogue (x_proj, dt)
      if (PAIR)
        mbar_wait_cluster(&tfull[acc], acc_phase);
      else
        mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + acc * 256 + ((uint32_t)(quarter * 32) << 16);
      uint32_t r[32];  // TMEM load of the next chunk in flight while this one is processed
      if (half * 32 < BN) tmem_ld32(t_row + half * 32, r);
      for (int cc = 0; cc < nch; ++cc, ++gseq) {
        const int cl = cc * 64 + half * 32;            // tile-local first column of this thread's 32
        const int col0 = n0 + cl;
        if (f32_tma) {  // each warp stores its own 32 x 32 box (buffers of parity gseq & 1, two chunks in flight per
          if (lane == 0 && gseq >= 2) bulk_wait_read1();  // warp): its store from two chunks ago has been read out;
          __syncwarp();                                    // no barrier couples the epilogue warps
        }
        float v[32];
        if (cl < BN) {
          tmem_wait_ld_dep(r);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          if (cl + 64 < BN) tmem_ld32(t_row + cl + 64, r);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
        }
        if (p.bias && cl < BN) {  // L1-cached broadcast loads (zero past N)
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 b4 = col0 + j + 4 <= p.N ? __ldg(reinterpret_cast<const float4*>(p.bias + col0 + j))
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            v[j] += b4.x; v[j + 1] += b4.y; v[j + 2] += b4.z; v[j + 3] += b4.w;
          }
        }
        if (p.softplus) {  // Delta = softplus(delta_low W_dt^T + b_dt) = log1p(t), t = e^x (x for x > 20)
          // log1p(t): t (1 - t/2 + t^2/3 - t^3/4 + t^4/5) for t < 1/32 (truncation < t^6/6: 1e-9 relative), else
          // log(1 + t) on MUFU (the rounding of 1 + t costs <= 6e-8 / log1p(t) <= 2e-6 relative there): two MUFU
          // per element instead of three (no division)
          // Packed fp32x2 (round 2: the epilogue was issue-bound, ncu r02n 67 % issue with the softplus lines at 37 %
          // of the stall samples): per pair FMUL2 + 2 ex2, the polynomial as FFMA2s, FADD2 + 2 lg2 + FMUL2, selects
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float2 x = make_float2(v[j], v[j + 1]);
            const float2 xs = __fmul2_rn(x, make_float2(1.4426950408889634f, 1.4426950408889634f));
            const float2 t = make_float2(ex2_approx(xs.x), ex2_approx(xs.y));
            float2 q = __ffma2_rn(t, make_float2(0.2f, 0.2f), make_float2(-0.25f, -0.25f));
            q = __ffma2_rn(t, q, make_float2(0.33333334f, 0.33333334f));
            q = __ffma2_rn(t, q, make_float2(-0.5f, -0.5f));
            q = __ffma2_rn(t, q, make_float2(1.f, 1.f));
            q = __fmul2_rn(t, q);
            const float2 u = __fadd2_rn(t, make_float2(1.f, 1.f));
            const float2 l = __fmul2_rn(make_float2(lg2_approx(u.x), lg2_approx(u.y)),
                                        make_float2(0.69314718055994531f, 0.69314718055994531f));
            v[j] = x.x > 20.f ? x.x : (t.x < 0.03125f ? q.x : l.x);
            v[j + 1] = x.y > 20.f ? x.y : (t.y < 0.03125f ? q.y : l.y);
          }
        }
        if (f32_tma) {
          // this thread's 32 values are one 128-byte row of box `half` (128B-swizzled)
          uint8_t* sf = s_stage + (gseq & 1) * 2 * STAGE_OUT_BYTES;
          uint8_t* sh = sf + half * STAGE_OUT_BYTES;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<uint4*>(sh + swz_offset(row_local, q, 128)) =
                make_uint4(__float_as_uint(v[4 * q]), __float_as_uint(v[4 * q + 1]), __float_as_uint(v[4 * q + 2]),
                           __float_as_uint(v[4 * q + 3]));
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {  // this warp's 32 rows of box `half`
            const int r0 = mb + quarter * 32;
            if (r0 < p.M && col0 < p.N) tma_store_2d(&tmOut, sh + quarter * 32 * 128, col0, r0);
            bulk_commit();
          }
        } else if (row_ok && cl < BN) {
          // f32 output; with split-K each split first writes its partial tile ([S][M][N] workspace)
          const int ld = S > 1 ? p.N : p.ldo;
          float* o = (S > 1 ? p.partial + (size_t)split * p.M * p.N : reinterpret_cast<float*>(p.out)) +
                     (size_t)row * ld + col0;
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            if (col0 + j < p.N) {
              if (col0 + j + 4 <= p.N && (ld % 4) == 0) {
                *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
              } else {
                for (int e = 0; e < 4 && col0 + j + e < p.N; ++e) o[j + e] = v[j + e];
              }
            }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {  // one arrival per warp
        if (PAIR)
          mbar_arrive_remote(tempty0 + acc * 8);
        else
          mbar_arrive(&tempty[acc]);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      if (S > 1) {
        // deterministic split-K fix-up: the last split to finish this output tile sums the S partials in split
        // order (no floating-point atomics) and resets the tile's counter for the next launch.
        const int mn = tile / S;
        __threadfence();
        named_bar_sync(1, 256);
        if (issuer) *s_flag = atomicAdd(&p.sem[mn], 1);
        named_bar_sync(1, 256);
        if (*s_flag == S - 1) {
          __threadfence();
          for (int cc = 0; cc < nch; ++cc) {
            const int col0 = n0 + cc * 64 + half * 32;
            if (!row_ok || cc * 64 + half * 32 >= BN) continue;
            // 16-byte loads of all splits issued together, summed in split order (N % 4 == 0 checked on the host)
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              if (col0 + j >= p.N) break;
              float4 part[8];
#pragma unroll
              for (int s2 = 0; s2 < 8; ++s2)
                if (s2 < S)
                  part[s2] = __ldcg(reinterpret_cast<const float4*>(p.partial + ((size_t)s2 * p.M + row) * p.N + col0 + j));
              float4 sum = part[0];
#pragma unroll
              for (int s2 = 1; s2 < 8; ++s2)
                if (s2 < S) {
                  sum.x += part[s2].x; sum.y += part[s2].y; sum.z += part[s2].z; sum.w += part[s2].w;
                }
              *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + (size_t)row * p.ldo + col0 + j) = sum;
            }
          }
          if (issuer) p.sem[mn] = 0;
        }
        named_bar_sync(1, 256);
      }
    }
    if (tma_out && lane == 0) bulk_wait0();
    if (lane == 0 && f32_tma) bulk_wait0();
  }
  __syncthreads();
  if (PAIR) cluster_sync();  // the peer may still read this CTA's shared memory / signal its barriers until here
  if (warp == 1) {
    tc_fence_after();
    if (PAIR)
      tmem_dealloc_pair(tmem_base, 512);
    else
      tmem_dealloc(tmem_base, 512);
  }
}

static bool pair_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("PSCWIN_GEMM_PAIR");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// B multicast across two CTA pairs (4-CTA clusters): PSCWIN_GEMM_MC=2 turns it on (A/B knob, read once). Off by
// default: bit-identical but 2-4 % slower at every 4096^2 projection shape (profiles/r02/gemm_mc_r02m.log: QKV 183.9
// -> 188.3 us, out-proj 78.9 -> 82.4, in_proj 237 -> 247), so the B tile reads from L2 are not what bounds them
static bool mc_enabled() {
  static const int on = env_knob("PSCWIN_GEMM_MC", 1);
  return on == 2;
}

// co-resident clusters of `csize` CTAs (2: a pair, 4: two pairs) of the pair kernel (SMs left over in a GPC cannot
// host part of a cluster); cached per (device, smem, cluster size)
static int pair_clusters(size_t smem, int csize) {
  static std::mutex mu;
  static std::map<std::tuple<int, size_t, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(dev, smem, csize);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize * (num_sms() / csize));
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  const cudaError_t e = csize == 4
                            ? cudaOccupancyMaxActiveClusters(&n, gemm_bf16_kernel<true, EK_PLAIN, 2>, &cfg)
                            : cudaOccupancyMaxActiveClusters(&n, gemm_bf16_kernel<true, EK_PLAIN>, &cfg);
  if (e != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = num_sms() / csize;
  }
  cache[key] = n;
  return n;
}

int launch_gemm_bf16(const void* A, const void* Bw, const GemmArgs& args_in, cudaStream_t stream) {
  GemmArgs p = args_in;
  if (p.M <= 0 || p.N <= 0) return 0;
  if (p.K % (p.tf32 ? 4 : 8) != 0) return -1;
  if (p.epi == EPI_QKV_ROPE && p.rope && !(p.d_head == 32 || p.d_head == 64)) return -2;
  const bool resid = p.epi == EPI_RESID_BF16 && p.residual != nullptr;
  if (p.silu_col && (p.silu_col % 32 || p.epi == EPI_STORE_F32)) return -2;
  if (p.gelu && p.epi != EPI_STORE_BF16) return -2;
  if (p.ln_stats && (!p.ln_colsum || !p.bias || p.epi == EPI_STORE_F32 || p.splits > 1)) return -2;
  if ((p.tf32 || p.softplus) && (p.epi != EPI_STORE_F32 || p.splits > 1)) return -2;
  if (p.tf32 && (p.K % 4 || (p.lda * 4) % 16 || (p.ldb * 4) % 16)) return -1;
  if (p.splits > 1 && (p.epi != EPI_STORE_F32 || !p.partial || !p.sem || p.splits > 8 || p.N % 4 || p.ldo % 4))
    return -3;
  {  // every split needs at least one K block (a split without any would never commit its accumulator)
    const int nk = (p.K + (p.tf32 ? BK / 2 : BK) - 1) / (p.tf32 ? BK / 2 : BK);
    if (p.splits > nk) p.splits = nk;
  }
  // CTA pairs (256-row tiles, cta_group::2) whenever there are at least two row tiles and no split-K; not for the
  // TF32 dt GEMM (K = R = 48: nothing to share, and the cluster-scope barrier traffic slows its epilogue-bound
  // tiles: 4096^2 226 -> 208 us single-CTA)
  const bool pair = pair_enabled() && p.splits <= 1 && p.M > BM && !p.tf32;
  const int TMr = pair ? 2 * BM : BM;
  const int m_tiles = (p.M + TMr - 1) / TMr;
  const int slots = pair ? num_sms() / 2 : num_sms();
  // tile N: one tile when N <= 256 (<= 128 with a residual, whose tiles are staged in shared memory); else the
  // width (256 or 128) with the fewest scheduling rounds, weighting a round by its tile width
  if (p.BN <= 0) {
    if (p.N <= 256) {
      p.BN = ((p.N + 15) / 16) * 16;
    } else {
      auto cost = [&](int bn) {
        const long long tiles = (long long)m_tiles * ((p.N + bn - 1) / bn);
        return ((tiles + slots - 1) / slots) * (bn + 32);
      };
      p.BN = cost(256) <= cost(128) ? 256 : 128;
      // 192-column tiles when they quantise better. Unrestricted (PSCWIN_GEMM_BN192=1) they also replace 256 at
      // 4096^2 (N = 768: 13.8 of 14 rounds against 10.4 of 11), where the out-proj gains 2 us per launch but the step
      // measured 0.13 ms SLOWER in alternating runs (gemm_bn192_r02ab.log); PSCWIN_GEMM_BN192=0 never uses them.
      // The default rule below takes them only without extra rounds: 1024^2 stage 0.377 -> 0.370 ms (out-proj 20.0 ->
      // 18.1 us), 4096^2 unchanged (gemm_bn192_rule_r02ao.log).
      // Default (PSCWIN_GEMM_BN192 unset / 2): only when 192-column tiles need no more scheduling rounds than the
      // current width (e.g. the 1024^2 out-proj: 64 pair tiles in one round instead of 48 wider ones), never when they
      // add rounds (4096^2)
      static const int bn192 = env_knob("PSCWIN_GEMM_BN192", 2);
      auto rounds = [&](int bn) { return ((long long)m_tiles * ((p.N + bn - 1) / bn) + slots - 1) / slots; };
      if (p.N % 192 == 0 && cost(192) < cost(p.BN) && (bn192 == 1 || (bn192 == 2 && rounds(192) <= rounds(p.BN))))
        p.BN = 192;
      static const int bn_knob = env_knob("PSCWIN_GEMM_BN", 0);  // tuning knob for the multi-tile case: 128/192/256
      if (bn_knob == 128 || bn_knob == 192 || bn_knob == 256) p.BN = bn_knob;
    }
  }
  if (pair && (p.BN % 16)) return -2;
  // ring depth: as many stages as fit next to the staging / residual buffers
  const bool f32o = p.epi == EPI_STORE_F32;
  // bf16 outputs: per-warp epilogue (32 x 32 SW64 boxes). The residual is TMA-loaded into shared memory as 32-column
  // boxes that the output overwrites in place (one 64 KB set at BN = 256: two ring stages fewer), or read from
  // global memory by the epilogue threads one box ahead after an L2 prefetch of the tile (the ring keeps its depth,
  // the epilogue waits on L2). Measured at 4096^2 (s5): K = 768 out-proj 86 us smem / 103 us global, K = 1536
  // cycle-scan out-proj 133 / 126 us: a long mainloop hides the loads and profits from the deeper ring, so global
  // iff K >= 1024. PSCWIN_GEMM_RES = 1 forces global, 2 shared memory (A/B knobs, read once).
  static const int res_knob = env_knob("PSCWIN_GEMM_RES", 0);
  const int res_smem = res_knob == 2 || (res_knob == 0 && p.K < 1024);
  static const int nbuf_knob = env_knob("PSCWIN_GEMM_NBUF", 0);
  p.warp_epi = f32o ? 0 : 1;
  p.res_global = (p.warp_epi && !res_smem && p.N % 32 == 0 && p.ldr % 8 == 0) ? 1 : 0;
  static const int noepi = env_knob("PSCWIN_GEMM_DBG_NOEPI", 0);  // timing probe only: output left unwritten
  p.dbg_noepi = p.warp_epi && noepi ? 1 : 0;
  {
    // per-warp bf16 epilogue: two staging boxes per warp unless a single one buys another ring stage
    const size_t st = gemm_stage_bytes(p.BN, pair);
    auto ring = [&](int nbuf) {
      const size_t fixed = gemm_fixed_bytes(gemm_epi_smem(p.BN, resid, f32o, p.warp_epi, nbuf, p.res_global));
      const int n = (int)((GEMM_SMEM_MAX - fixed) / st);
      return n > MAX_STAGES ? MAX_STAGES : n;
    };
    p.nbuf = ring(1) > ring(2) ? 1 : 2;
    if (nbuf_knob == 1 || nbuf_knob == 2) p.nbuf = nbuf_knob;
    const int stages = ring(p.nbuf);
    if (stages < 2) return -2;
    p.stages = stages;
  }
  p.pair = pair ? 1 : 0;
  // PSCWIN_GEMM_BIAS_L1=1 (A/B knob): bf16 epilogues read the bias (and LayerNorm column sums) through L1 instead of
  // staging them in shared memory behind a CTA-wide barrier per tile (the out-proj's second stall reason in ncu
  // r02d). Measured much slower (QKV 200 -> 266 us, out-proj 86.7 -> 92.8 us at 4096^2, gemm_bias_l1_r02al.log):
  // the per-box global loads cost more than one barrier per tile; off
  static const int bias_l1 = env_knob("PSCWIN_GEMM_BIAS_L1", 0);
  p.bias_l1 = (bias_l1 && (reinterpret_cast<uintptr_t>(p.bias) & 15) == 0 &&
               (reinterpret_cast<uintptr_t>(p.ln_colsum) & 15) == 0) ? 1 : 0;
  CUtensorMap tmA, tmB, tmOut, tmRes;
  const CUtensorMapDataType in_t = p.tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const int esz = p.tf32 ? 4 : 2, bke = p.tf32 ? BK / 2 : BK;
  int rc = make_tmap_2d(&tmA, A, in_t, p.K, p.M, (uint64_t)p.lda * esz, bke, BM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  // B multicast across two pairs: bf16 epilogues, no split-K, whole 32-row quarters, at least two pair tiles
  const int mc = (pair && mc_enabled() && p.epi != EPI_STORE_F32 && p.BN % 32 == 0 && p.M > 2 * TMr) ? 2 : 1;
  rc = make_tmap_2d(&tmB, Bw, in_t, p.K, p.N, (uint64_t)p.ldb * esz, bke, pair ? p.BN / (2 * mc) : p.BN,
                    CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  memset(&tmOut, 0, sizeof(tmOut));
  // f32 outputs without split-K go through a TMA store when the row stride allows it (16-byte multiple)
  static const bool f32_direct = getenv("PSCWIN_GEMM_F32_DIRECT") != nullptr;  // A/B knob
  p.f32_tma = (p.epi == EPI_STORE_F32 && p.splits <= 1 && (p.ldo * 4) % 16 == 0 && !f32_direct) ? 1 : 0;
  if (p.f32_tma) {
    rc = make_tmap_2d(&tmOut, p.out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, p.N, p.M, (uint64_t)p.ldo * 4, 32, 32,
                      CU_TENSOR_MAP_SWIZZLE_128B);  // one 32 x 32 box per epilogue warp
    if (rc) return rc;
  }
  if (p.epi != EPI_STORE_F32) {
    if ((p.ldo * 2) % 16) return -1;
    rc = make_tmap_2d(&tmOut, p.out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, p.N, p.M, (uint64_t)p.ldo * 2, 32, 32,
                      CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  }
  memset(&tmRes, 0, sizeof(tmRes));
  if (resid) {  // (TMA-loaded residual boxes, or the L2 prefetch of the global-memory residual path)
    if ((p.ldr * 2) % 16) return -1;
    rc = make_tmap_2d(&tmRes, p.residual, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, p.N, p.M, (uint64_t)p.ldr * 2, 32, BM,
                      CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  }
  {
    const void* fns[11] = {(const void*)gemm_bf16_kernel<false, EK_PLAIN>, (const void*)gemm_bf16_kernel<false, EK_ROPE>,
                          (const void*)gemm_bf16_kernel<false, EK_GELU>, (const void*)gemm_bf16_kernel<false, EK_F32>,
                          (const void*)gemm_bf16_kernel<true, EK_PLAIN>, (const void*)gemm_bf16_kernel<true, EK_ROPE>,
                          (const void*)gemm_bf16_kernel<true, EK_GELU>, (const void*)gemm_bf16_kernel<true, EK_F32>,
                          (const void*)gemm_bf16_kernel<true, EK_PLAIN, 2>, (const void*)gemm_bf16_kernel<true, EK_ROPE, 2>,
                          (const void*)gemm_bf16_kernel<true, EK_GELU, 2>};
    for (const void* f : fns) func_smem_once(f, (int)GEMM_SMEM_MAX);
  }
  const int ek = p.epi == EPI_QKV_ROPE ? EK_ROPE : (p.gelu ? EK_GELU : (p.epi == EPI_STORE_F32 ? EK_F32 : EK_PLAIN));
  const size_t smem = gemm_fixed_bytes(gemm_epi_smem(p.BN, resid, f32o, p.warp_epi, p.nbuf, p.res_global)) +
                      (size_t)p.stages * gemm_stage_bytes(p.BN, pair);
  if (smem > GEMM_SMEM_MAX) return -2;
  const long long tiles = (long long)(mc > 1 ? (p.M + 2 * TMr - 1) / (2 * TMr) : m_tiles) *
                          ((p.N + p.BN - 1) / p.BN) * (p.splits > 1 ? p.splits : 1);
  PSCWIN_PROF(p.prof_name ? p.prof_name : "gemm", stream);
  if (!pair) {
    const int grid = tiles < num_sms() ? (int)tiles : num_sms();
    if (ek == EK_ROPE)
      launch_k(gemm_bf16_kernel<false, EK_ROPE>, dim3(grid), dim3(GEMM_THREADS), smem, stream, tmA, tmB, tmOut, tmRes, p);
    else if (ek == EK_GELU)
      launch_k(gemm_bf16_kernel<false, EK_GELU>, dim3(grid), dim3(GEMM_THREADS), smem, stream, tmA, tmB, tmOut, tmRes, p);
    else if (ek == EK_F32)
      launch_k(gemm_bf16_kernel<false, EK_F32>, dim3(grid), dim3(GEMM_THREADS), smem, stream, tmA, tmB, tmOut, tmRes, p);
    else
      launch_k(gemm_bf16_kernel<false, EK_PLAIN>, dim3(grid), dim3(GEMM_THREADS), smem, stream, tmA, tmB, tmOut, tmRes, p);
    return (int)cudaGetLastError();
  }
  const int csize = 2 * mc;
  const int clusters_max = pair_clusters(smem, csize);
  const int clusters = tiles < clusters_max ? (int)tiles : clusters_max;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize * clusters);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (mc > 1 && ek == EK_ROPE)
    cudaLaunchKernelEx(&cfg, gemm_bf16_kernel<true, EK_ROPE, 2>, tmA, tmB, tmOut, tmRes, p);
  else if (mc > 1 && ek == EK_GELU)
    cudaLaunchKernelEx(&cfg, gemm_bf16_kernel<true, EK_GELU, 2>, tmA, tmB, tmOut, tmRes, p);
  else if (mc > 1)
    cudaLaunchKernelEx(&cfg, gemm_bf16_kernel<true, EK_PLAIN, 2>, tmA, tmB, tmOut, tmRes, p);
  else if (ek == EK_ROPE)
    cudaLaunchKernelEx(&cfg, gemm_bf16_kernel<true, EK_ROPE>, tmA, tmB, tmOut, tmRes, p);
  else if (ek == EK_GELU)
    cudaLaunchKernelEx(&cfg, gemm_bf16_kernel<true, EK_GELU>, tmA, tmB, tmOut, tmRes, p);
  else if (ek == EK_F32)
    cudaLaunchKernelEx(&cfg, gemm_bf16_kernel<true, EK_F32>, tmA, tmB, tmOut, tmRes, p);
  else
    cudaLaunchKernelEx(&cfg, gemm_bf16_kernel<true, EK_PLAIN>, tmA, tmB, tmOut, tmRes, p);
  return (int)cudaGetLastError();
}

}  // namespace pscwin
