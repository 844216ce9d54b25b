// Window attention core, persistent warp-specialised tcgen05 kernel for windows of <= 256 slots (w <= 16).
// Same math as attn_sm100.cu (§3.2; App. A.5; readings Q1, Q5, Q6):
// O = softmax(q k^T / sqrt(d)) v per (window, head), pad slots LEARNABLE (projected p, K rotated at the slot's
// geometric coordinate) or MASKED (-inf), only real rows written back to the [B,H,W,C] grid.
//
// Roles (576 threads, one CTA per SM, loops over (image, window, head) work items):
//   warp 0     TMA: Q, K, V tiles of the item (5-D boxes straight from QKV [B,H,W,3,heads,d]; off-grid rows
//              zero-filled) into one of two shared-memory stages (prefetch of item i+1 overlaps item i)
//   warp 1     TMEM allocation + single-thread tcgen05.mma issue: S_a = Q_a K_t^T, O_a = P_a V_t (P from TMEM)
//   warps 2-17 four softmax warpgroups: q tile a = 0/1, each query row split over two threads by key halves
//              (row max / sum combined in shared memory). The whole window (w^2 <= 256 keys) is ONE key tile, so
//              softmax is a single exact pass (max, exp2, sum) in fp32; P is written back to TMEM as bf16 over
//              the consumed S columns
// TMEM per q tile a (256 columns): S at [256a, 256a+w^2); then P of keys < 128 at [256a, 256a+64), P of keys
// >= 128 at [256a+128, 256a+192) and O at [256a+192, 256a+192+d) (all alias S columns already consumed).
#include <stdio.h>
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"
#include "pscwin_internal.h"

namespace pscwin {

namespace {
constexpr int WS_THREADS = 64 + 512 + 32;  // TMA warp, MMA warp (slot 0), 4 softmax warpgroups (two threads per query
                                           // row), MMA warp (slot 1)
constexpr int WS1_THREADS = 64 + 256 + 32;  // TMA warp, MMA warp (slot 0), 2 softmax warpgroups (one thread per
                                            // query row), MMA warp (slot 1)
#ifndef PSCWIN_ATTN_POLY_MOD
// k > 0: every k-th exp2 pair on the FMA pipe (degree-3 polynomial, 7.5e-5 relative, far below the bf16 rounding of
// P). Round 1 (two threads per row, no ping-pong) swept 0 / 2 / 3 / 4: 125 / 133 / 128.5 / 127 us; round 2 (ROW1 with
// the exp ping-pong, MUFU-bound exp passes) 0 / 4 / 8: 119.8 / 115.5 / 117.2 us at 4096^2 (profiles/r02)
#define PSCWIN_ATTN_POLY_MOD 4
#endif
constexpr int kPolyMod = PSCWIN_ATTN_POLY_MOD;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
}
// debug timeline: role slot base (0 loader, 32 MMA, 64 WG0, 96 WG1), 32 events each per CTA
#define ATT_TS(base, cnt)                                                                   \
  do {                                                                                      \
    if (p.dbg && lane_id() == 0) p.dbg[blockIdx.x * 128 + (base) + ((cnt)++ & 31)] = gtimer(); \
  } while (0)
// item-indexed variant (ROW1 softmax slots): event e (0..5) of the CTA's k-th item at slot (k % 5) * 6 + e
#define ATT_TS6(base, k, e)                                                                          \
  do {                                                                                               \
    if (p.dbg && lane_id() == 0) p.dbg[blockIdx.x * 128 + (base) + ((k) % 5) * 6 + (e)] = gtimer(); \
  } while (0)

struct AttnWsArgs {
  int B, H, W, C, heads, w, lw, pt, pl, nwx, nw, pad_mode, patch;
  int rpt, n_tiles, tile_slots, n_items;
  int win0, nw_run;  // windows [win0, win0 + nw_run) of every image are run (a window-row range; all by default)
  int lockstep;  // -1: automatic (few items per CTA), 0 / 1 forced (PSCWIN_ATTN_LOCKSTEP knob)
  int tma_out;  // 1: O tiles staged in smem and TMA-stored; 0: 16-byte global stores of the real rows
  int pf;       // L2 prefetch distance of the TMA producer (items beyond the two staged ones; 0 = off)
  int pingpong;  // ROW1: the two q-tile slots take turns for their exp passes
  float sl2;
  const __nv_bfloat16 *kx, *ky, *vp;
  __nv_bfloat16* out;
  unsigned long long* dbg;  // debug timeline (PSCWIN_ATTN_TIMELINE), else null
};

// ROW1: one softmax thread per query row (8 softmax warps, 168 registers each: the whole 256-key row in one thread,
// no cross-thread max / sum exchange); else two threads per row (16 softmax warps at the 96-register cap).
template <int D, bool MASKED, bool ROW1>
__global__ void __launch_bounds__(ROW1 ? WS1_THREADS : WS_THREADS, 1)
    window_attn_ws_kernel(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmO,
                          AttnWsArgs p) {
  pdl_trigger();
  constexpr int ROWB = D * 2;
  constexpr int TILE = 128 * ROWB;           // smem bytes reserved per 128-slot tile
  constexpr int STAGE = 6 * TILE;            // Q0 Q1 K0 K1 V0 V1
  constexpr uint32_t LAYOUT = ROWB == 128 ? kLayoutSW128 : kLayoutSW64;
  constexpr uint32_t SBO = 8 * ROWB;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * STAGE);
  uint64_t* ld_full = bars + 0;      // [2]
  uint64_t* ld_empty = bars + 2;     // [2]
  uint64_t* patch_done = bars + 4;   // [2]
  uint64_t* s_full = bars + 6;       // [2] per warpgroup
  uint64_t* p_full = bars + 8;       // [2]
  uint64_t* o_full = bars + 10;      // [2]
  uint64_t* o_free = bars + 12;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);
  uint64_t* turn = bars + 16;  // [2] exp-pass turn of each q-tile slot (ping-pong)
  float* s_red = reinterpret_cast<float*>(bars + 18);  // ROW2: [2 q tiles][2 halves][128 rows] partial row max / sum

  const int warp = warp_id();
  constexpr int NTQ = ROW1 ? 128 : 256;  // softmax threads per q tile
  const int nt = p.n_tiles;
  const uint32_t tile_tx = (uint32_t)(p.tile_slots * ROWB);

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmQKV);
    tma_prefetch_desc(&tmO);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&ld_full[i], 1);
      // a stage is free once its MMAs completed (commit) AND both q-tile slots' O tiles, staged in the slot's Q
      // region of the stage, have been read out by their TMA stores (one arrival per slot)
      mbar_init(&ld_empty[i], 4);  // both issuers' commits + both slots' O stores
      mbar_init(&patch_done[i], NTQ);  // slot 0's threads patch (slot 1 runs half an item behind)
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], NTQ);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_free[i], NTQ);
      mbar_init(&turn[i], NTQ);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  pdl_wait();  // barrier init / TMEM allocation overlap the previous kernel; global accesses start here
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto decode = [&](int item, int& b, int& h, int& X0, int& Y0) {
    h = item % p.heads;
    const int r = item / p.heads;
    const int win = p.win0 + r % p.nw_run;
    b = r / p.nw_run;
    const int wy = win / p.nwx, wx = win - wy * p.nwx;
    X0 = wx * p.w - p.pl;
    Y0 = wy * p.w - p.pt;
  };
  // q tile a of an item has at least one real query row
  auto q_active = [&](int a, int Y0) {
    if (a >= nt) return false;
    const int ylo = Y0 + a * p.rpt;
    return ylo + p.rpt > 0 && ylo < p.H;
  };

  if (warp == 0) {
    // ------------------------------------------------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();
      int stage = 0, ev = 0;
      uint32_t phase = 0;
      // L2 prefetch p.pf items ahead of the loads: a stage is refilled only when its previous item is done, and a
      // cold item's strided 128-byte rows took ~4 us to land from HBM (timeline r02e) — longer than an item
      auto prefetch = [&](int item) {
        if (item >= p.n_items) return;
        int b, h, X0, Y0;
        decode(item, b, h, X0, Y0);
        for (int t = 0; t < nt; ++t) {
          const int y = Y0 + t * p.rpt;
          for (int q = 0; q < 3; ++q) tma_prefetch_l2_5d(&tmQKV, 0, q * p.heads + h, X0, y, b);
        }
      };
      for (int k = 2; k < 2 + p.pf; ++k) prefetch(blockIdx.x + k * gridDim.x);
      for (int item = blockIdx.x; item < p.n_items; item += gridDim.x) {
        int b, h, X0, Y0;
        decode(item, b, h, X0, Y0);
        if (p.pf) prefetch(item + (2 + p.pf) * gridDim.x);
        mbar_wait(&ld_empty[stage], phase ^ 1);
        ATT_TS(0, ev);
        mbar_arrive_expect_tx(&ld_full[stage], 3 * nt * tile_tx);
        uint8_t* st = smem + stage * STAGE;
        for (int t = 0; t < nt; ++t) {
          const int y = Y0 + t * p.rpt;
          tma_load_5d(st + t * TILE, &tmQKV, &ld_full[stage], 0, h, X0, y, b, pol);
          tma_load_5d(st + (2 + t) * TILE, &tmQKV, &ld_full[stage], 0, p.heads + h, X0, y, b, pol);
          tma_load_5d(st + (4 + t) * TILE, &tmQKV, &ld_full[stage], 0, 2 * p.heads + h, X0, y, b, pol);
        }
        if (++stage == 2) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 || warp == (ROW1 ? 10 : 18)) {
    // ------------------------------------------------------------------------------------------ MMA issuers (ROW1)
    // One issuing warp per q-tile slot (warp 1: slot 0, warp 10: slot 1), so neither slot's S / PV MMAs wait behind
    // the other slot's barriers: per item S_a = Q_a K^T (after the previous item's O_a, which aliases S columns, has
    // been read out), then O_a = P_a V once P_a is in TMEM, then a commit that releases the stage (4 arrivals: both
    // issuers' commits and both slots' O stores)
    const int a = warp == 1 ? 0 : 1;  // (the issuer of slot 1 is the last warp)
    const int NK = nt * p.tile_slots;
    const uint32_t idesc_s = make_idesc_bf16(128, NK, 0, 0);
    const uint32_t idesc_o = make_idesc_bf16(128, D, 0, 1);
    int stage = 0;
    uint32_t phase = 0, ph_p = 0, ph_of = 0;
    int ev = 0;
    for (int item = blockIdx.x; item < p.n_items; item += gridDim.x) {
      int b, h, X0, Y0;
      decode(item, b, h, X0, Y0);
      const bool act = q_active(a, Y0);
      mbar_wait(&ld_full[stage], phase);
      if (p.patch) mbar_wait(&patch_done[stage], phase);
      if (a == 0) ATT_TS(32, ev);
      const uint32_t sb = smem_u32(smem + stage * STAGE);
      if (act) {
        mbar_wait(&o_free[a], ph_of ^ 1);
        ph_of ^= 1;
        tc_fence_after();
        if (elect_one()) {
          const uint32_t qa = sb + a * TILE, ka = sb + 2 * TILE;
#pragma unroll
          for (int k = 0; k < D / 16; ++k)
            umma_ss(tmem + 256 * a, make_sdesc(qa + k * 32, 16, SBO, LAYOUT),
                    make_sdesc(ka + k * 32, 16, SBO, LAYOUT), idesc_s, k > 0);
          umma_commit(&s_full[a]);
        }
        __syncwarp();
        mbar_wait(&p_full[a], ph_p);
        ph_p ^= 1;
        tc_fence_after();
        if (elect_one()) {
          const uint32_t va = sb + 4 * TILE;
          for (int ks = 0; ks < NK / 16; ++ks)  // P of keys 16ks.. at column 8ks (+64 for keys >= 128 in ROW2)
            umma_ts(tmem + 256 * a + 192, tmem + 256 * a + ks * 8 + (!ROW1 && ks >= 8 ? 64 : 0),
                    make_sdesc(va + ks * 16 * ROWB, TILE, SBO, LAYOUT), idesc_o, ks > 0);
          umma_commit(&o_full[a]);
        }
        __syncwarp();
      }
      if (elect_one()) umma_commit(&ld_empty[stage]);  // once this slot's MMAs have read the stage
      __syncwarp();
      if (++stage == 2) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if constexpr (ROW1) {
    // ------------------------------------------------------------------------------------------ softmax WGs (ROW1)
    // 8 warps: q tile a = (warp - 2) >> 2; the thread of TMEM lane `row` owns query row `row` of its q tile and all
    // of the window's keys: max pass, then exp pass (P bf16 pairs written over consumed S columns: keys 16ks..
    // at column 8ks), then O read-out, normalisation and the merge / crop store.
    const int sw = warp - 2;
    const int a = sw >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane_id();        // query slot within the q tile (= TMEM lane)
    const int gtid = (sw & 3) * 32 + lane_id();      // 0..127 within the q tile's warpgroup
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tmem + 256 * a + lane_base;
    const uint32_t tO = tmem + 256 * a + 192 + lane_base;
    int stage = 0;
    uint32_t phase = 0;
    uint32_t ph_s = 0, ph_o = 0;
    int ev = 0;
    const int NK = nt * p.tile_slots;                // keys of the window (one S tile): 16, 64 or 256
    const uint32_t tail_mask = NK >= 32 ? 0xFFFFFFFFu : ((1u << NK) - 1u);  // 16-key windows (w = 4)
    const float2 sl2 = make_float2(p.sl2, p.sl2);
    const bool pingpong = p.pingpong && nt == 2;  // (one q tile per window: nothing to alternate with)
    uint32_t ph_t = 0;
    // LEARNABLE pad patch of the K/V rows outside the grid by slot 0's 128 threads (slot 1 only reads the stage
    // through its MMAs, after patch_done): entry e = key tile e>>7, slot e&127. It runs one item ahead — the next
    // item's stage is patched while this item's PV MMA runs — so the next S MMA does not wait for it.
    // returns false (nothing done) when block is false and the stage has not landed yet
    auto patch = [&](int pitem, int pstage, uint32_t pphase, bool block) -> bool {
      int b, h, X0, Y0;
      decode(pitem, b, h, X0, Y0);
      if (X0 >= 0 && Y0 >= 0 && X0 + p.w <= p.W && Y0 + nt * p.rpt <= p.H) {  // no pad slot in this window
        mbar_arrive(&patch_done[pstage]);
        __syncwarp();
        return true;
      }
      if (!block && !__all_sync(0xffffffffu, mbar_test(&ld_full[pstage], pphase))) return false;  // (warp-uniform)
      mbar_wait(&ld_full[pstage], pphase);  // (TMA zero-fills the pad rows: patch only after it landed)
      for (int e = gtid; e < nt * 128; e += 128) {
        const int kt = e >> 7, r = e & 127;
        if (r >= p.tile_slots) continue;
        const int Y = Y0 + kt * p.rpt + (r >> p.lw), X = X0 + (r & (p.w - 1));
        if (Y < 0 || Y >= p.H || X < 0 || X >= p.W) {
          uint8_t* sK = smem + pstage * STAGE + (2 + kt) * TILE;
          uint8_t* sV = smem + pstage * STAGE + (4 + kt) * TILE;
          const uint4* kx = reinterpret_cast<const uint4*>(p.kx + ((size_t)(X + p.pl) * p.heads + h) * (D / 2));
          const uint4* ky = reinterpret_cast<const uint4*>(p.ky + ((size_t)(Y + p.pt) * p.heads + h) * (D / 2));
          const uint4* vp = reinterpret_cast<const uint4*>(p.vp + (size_t)h * D);
#pragma unroll
          for (int c = 0; c < D / 16; ++c) {
            *reinterpret_cast<uint4*>(sK + swz_offset(r, c, ROWB)) = kx[c];
            *reinterpret_cast<uint4*>(sK + swz_offset(r, c + D / 16, ROWB)) = ky[c];
          }
#pragma unroll
          for (int c = 0; c < D / 8; ++c) *reinterpret_cast<uint4*>(sV + swz_offset(r, c, ROWB)) = vp[c];
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&patch_done[pstage]);
      __syncwarp();
      return true;
    };
    // the stage after `stage` holds item + gridDim.x; if its data has not landed yet, the patch is deferred to the end
    // of this item (block = true there) instead of stalling this slot's O read-out behind the next item's load
    bool patch_deferred = false;
    auto patch_next = [&](int item, bool block) {
      if (p.patch && a == 0 && item + (int)gridDim.x < p.n_items) {
        // (the defer decision is warp-uniform; warps may differ, each thread still arrives exactly once)
        patch_deferred = !patch(item + gridDim.x, stage ^ 1, stage == 1 ? phase ^ 1 : phase, block);
      }
    };
    if (p.patch && a == 0 && (int)blockIdx.x < p.n_items) patch(blockIdx.x, 0, 0, true);
    int kk = 0;  // this CTA's item count (debug timeline)
    for (int item = blockIdx.x; item < p.n_items; item += gridDim.x, ++kk) {
      int b, h, X0, Y0;
      decode(item, b, h, X0, Y0);
      const bool active = q_active(a, Y0);
      if (active) {
        // MASKED: valid-key bitmask per 32-column chunk (real slots only); columns past the window are never read
        uint32_t xmask = 0xFFFFFFFFu;
        int iy_lo = 0, iy_hi = 1 << 30;
        if (MASKED) {
          const int xl = max(0, -X0), xh = min(p.w, p.W - X0);
          xmask = (xh > xl) ? (((1u << (xh - xl)) - 1u) << xl) : 0u;
          iy_lo = -Y0;
          iy_hi = p.H - Y0;
        }
        auto chunk_mask = [&](int c0) -> uint32_t {
          uint32_t m = 0;
          const int rows = 32 >> p.lw;
#pragma unroll 8
          for (int rr = 0; rr < rows; ++rr) {
            const int iy = (c0 >> p.lw) + rr;
            if (iy >= iy_lo && iy < iy_hi) m |= (xmask & ((1u << p.w) - 1u)) << (rr * p.w);
          }
          return m;
        };
        mbar_wait(&s_full[a], ph_s);
        ph_s ^= 1;
        if (row == 0) ATT_TS6(64 + 32 * a, kk, 0);
        tc_fence_after();
        // pass 1: row max over the window's keys (two 32-column TMEM loads per wait, four independent max chains)
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        for (int c0 = 0; c0 < NK; c0 += 64) {
          uint32_t r0[32], r1[32];
          const bool two = c0 + 32 < NK;
          tmem_ld32(tS + c0, r0);
          if (two) tmem_ld32(tS + c0 + 32, r1);
          tmem_wait_ld();
          if (MASKED || tail_mask != 0xFFFFFFFFu) {
            const uint32_t m0 = (MASKED ? chunk_mask(c0) : 0xFFFFFFFFu) & tail_mask;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if ((m0 >> j) & 1u) mx4[j & 3] = fmaxf(mx4[j & 3], __uint_as_float(r0[j]));
            if (two) {
              const uint32_t m1 = MASKED ? chunk_mask(c0 + 32) : 0xFFFFFFFFu;
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if ((m1 >> j) & 1u) mx4[j & 3] = fmaxf(mx4[j & 3], __uint_as_float(r1[j]));
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              mx4[(j >> 1) & 3] = fmaxf(mx4[(j >> 1) & 3], fmaxf(__uint_as_float(r0[j]), __uint_as_float(r0[j + 1])));
            }
            if (two) {
#pragma unroll
              for (int j = 0; j < 32; j += 2)
                mx4[(j >> 1) & 3] =
                    fmaxf(mx4[(j >> 1) & 3], fmaxf(__uint_as_float(r1[j]), __uint_as_float(r1[j + 1])));
            }
          }
        }
        const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
        if (row == 0) ATT_TS6(64 + 32 * a, kk, 1);  // max pass done (debug timeline)
        const float base = (mx == -INFINITY) ? 0.f : mx * p.sl2;
        const float2 nb = make_float2(-base, -base);
        // pass 2: p = 2^(s log2(e)/sqrt(d) - base) (packed fp32x2 scale, MUFU ex2), row sum, P (bf16 pairs) written
        // over the consumed S columns; 32-column TMEM loads double-buffered (the next chunk's load is in flight
        // while this one is exponentiated)
        float2 ls[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        // ping-pong: the two slots' exp passes alternate (slot 0 of item i, slot 1 of item i, slot 0 of item i+1,
        // ...), so one slot's MUFU-bound exponentials overlap the other slot's max pass, MMAs and O read-out instead
        // of the two contending for the MUFU pipe and then idling together
        uint32_t ra[32], rb[32], pk[16];
        tmem_ld32(tS, ra);  // (the first chunk's TMEM load is issued before waiting for the exp turn)
        if (pingpong) {
          mbar_wait(&turn[a], a == 0 ? ph_t ^ 1 : ph_t);
          ph_t ^= 1;
        }
        if (row == 0) ATT_TS6(64 + 32 * a, kk, 2);
        long long clk_e0 = 0;
        if (p.dbg && row == 0) clk_e0 = clock64();
        auto exp32 = [&](const uint32_t (&r)[32], uint32_t m, uint32_t (&pk)[16]) {
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float2 x = __ffma2_rn(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), sl2, nb);
            float e0, e1;
            if (kPolyMod > 0 && (j / 2) % kPolyMod == kPolyMod - 1) {
              const float2 e = exp2_poly2(x);
              e0 = e.x;
              e1 = e.y;
            } else {
              e0 = ex2_approx(x.x);
              e1 = ex2_approx(x.y);
            }
            if (MASKED || m != 0xFFFFFFFFu) {  // invalid keys, or stale columns past a 16-key window
              e0 = ((m >> j) & 1u) ? e0 : 0.f;
              e1 = ((m >> (j + 1)) & 1u) ? e1 : 0.f;
            }
            ls[(j >> 1) & 1] = __fadd2_rn(ls[(j >> 1) & 1], make_float2(e0, e1));
            pk[j / 2] = pack_bf16(e0, e1);
          }
        };
        {
          for (int c0 = 0; c0 < NK; c0 += 64) {
            tmem_wait_ld_dep(ra);
            const bool two = c0 + 32 < NK;
            if (two) tmem_ld32(tS + c0 + 32, rb);  // (a 16-key window reads 16 stale columns: masked by tail_mask)
            exp32(ra, (MASKED ? chunk_mask(c0) : 0xFFFFFFFFu) & tail_mask, pk);
            tmem_st16(tS + c0 / 2, pk);
            if (two) {
              tmem_wait_ld_dep(rb);
              if (c0 + 64 < NK) tmem_ld32(tS + c0 + 64, ra);
              exp32(rb, MASKED ? chunk_mask(c0 + 32) : 0xFFFFFFFFu, pk);
              tmem_st16(tS + c0 / 2 + 16, pk);
            }
          }
        }
        if (pingpong) mbar_arrive(&turn[a ^ 1]);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&p_full[a]);
        patch_next(item, false);
        const float lsum = (ls[0].x + ls[1].x) + (ls[0].y + ls[1].y);
        if (row == 0) ATT_TS6(64 + 32 * a, kk, 3);
        if (p.dbg && row == 0) {  // SM clocks of this exp pass + globaltimer ns (debug: effective clock)
          p.dbg[blockIdx.x * 128 + 64 + 32 * a + 30] = (unsigned long long)(clock64() - clk_e0);
          p.dbg[blockIdx.x * 128 + 64 + 32 * a + 31] = p.dbg[blockIdx.x * 128 + 64 + 32 * a + (kk % 5) * 6 + 3] -
                                                      p.dbg[blockIdx.x * 128 + 64 + 32 * a + (kk % 5) * 6 + 2];
        }
        // O = P V lands in columns [192, 192 + d): copied to registers, the TMEM columns released (the next item's
        // S may overwrite them), then normalised and written to the grid (merge / crop)
        mbar_wait(&o_full[a], ph_o);
        ph_o ^= 1;
        if (row == 0) ATT_TS6(64 + 32 * a, kk, 4);
        tc_fence_after();
        uint32_t o0[32], o1[32];
        tmem_ld32(tO, o0);
        if constexpr (D == 64) tmem_ld32(tO + 32, o1);
        tmem_wait_ld();
        auto oval = [&](int j) { return __uint_as_float(j < 32 ? o0[j] : o1[j - 32]); };  // (j compile-time)
        tc_fence_before();
        mbar_arrive(&o_free[a]);
        const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
        // the normalised O tile is staged in this slot's Q region of the stage (Q_a is dead once S_a has been
        // computed) and ONE 5-D tensor store writes the window's rows back to the [B,H,W,C] grid; pad rows fall
        // outside the tensor and are clipped (a box starting at a negative coordinate traps: windows of the first
        // padded row / column store their real rows directly)
        if (p.tma_out && X0 >= 0 && Y0 + a * p.rpt >= 0) {
          uint8_t* so = smem + stage * STAGE + a * TILE;
#pragma unroll
          for (int c = 0; c < D / 8; ++c) {
            uint4 v;
            v.x = pack_bf16(oval(c * 8 + 0) * inv, oval(c * 8 + 1) * inv);
            v.y = pack_bf16(oval(c * 8 + 2) * inv, oval(c * 8 + 3) * inv);
            v.z = pack_bf16(oval(c * 8 + 4) * inv, oval(c * 8 + 5) * inv);
            v.w = pack_bf16(oval(c * 8 + 6) * inv, oval(c * 8 + 7) * inv);
            *reinterpret_cast<uint4*>(so + swz_offset(row, c, ROWB)) = v;
          }
          fence_proxy_async_smem();
          named_bar_sync(1 + a, 128);
          if (gtid == 0) {
            tma_store_5d(&tmO, so, 0, h, X0, Y0 + a * p.rpt, b);
            bulk_commit();
            bulk_wait_read0();  // the stage's Q region may be refilled once the store has read it
            mbar_arrive(&ld_empty[stage]);
          }
        } else {
          const int iy = a * p.rpt + (row >> p.lw), ix = row & (p.w - 1);
          const int Y = Y0 + iy, X = X0 + ix;
          if (row < p.tile_slots && Y >= 0 && Y < p.H && X >= 0 && X < p.W) {
            uint4* dst = reinterpret_cast<uint4*>(p.out + (((size_t)b * p.H + Y) * p.W + X) * p.C + (size_t)h * D);
#pragma unroll
            for (int c = 0; c < D / 8; ++c) {
              uint4 v;
              v.x = pack_bf16(oval(c * 8 + 0) * inv, oval(c * 8 + 1) * inv);
              v.y = pack_bf16(oval(c * 8 + 2) * inv, oval(c * 8 + 3) * inv);
              v.z = pack_bf16(oval(c * 8 + 4) * inv, oval(c * 8 + 5) * inv);
              v.w = pack_bf16(oval(c * 8 + 6) * inv, oval(c * 8 + 7) * inv);
              dst[c] = v;
            }
          }
          if (gtid == 0) mbar_arrive(&ld_empty[stage]);
        }
        if (row == 0) ATT_TS6(64 + 32 * a, kk, 5);
      } else {
        if (pingpong) {  // an inactive q tile passes its exp turn on
          mbar_wait(&turn[a], a == 0 ? ph_t ^ 1 : ph_t);
          ph_t ^= 1;
          mbar_arrive(&turn[a ^ 1]);
        }
        if (gtid == 0) mbar_arrive(&ld_empty[stage]);  // nothing staged for an inactive q tile
        patch_next(item, false);
      }
      __syncwarp();  // lane 0's store / arrival branch rejoins before the next item's .sync.aligned tcgen05 ops
      if (patch_deferred) patch_next(item, true);
      if (++stage == 2) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------------------------------------ softmax WGs
    // 16 warps: q tile a = sw >> 3, column half hc = (sw >> 2) & 1. The two warps of a q tile that share a TMEM
    // lane quarter split each query row's keys in halves; row max / sum are combined through shared memory.
    const int sw = warp - 2;
    const int a = sw >> 3;
    const int hc = (sw >> 2) & 1;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane_id();        // query slot within the q tile (= TMEM lane)
    const int wtid = sw * 32 + lane_id();            // 0..511
    const int gtid = (sw & 7) * 32 + lane_id();      // 0..255 within the q tile's two warpgroups
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tmem + 256 * a + lane_base;
    const uint32_t tO = tmem + 256 * a + 192 + lane_base;
    float* red_max = s_red + (a * 2) * 128;          // [2][128]
    float* red_sum = s_red + 512 + (a * 2) * 128;
    int stage = 0;
    uint32_t phase = 0;
    uint32_t ph_s = 0, ph_o = 0;
    int ev = 0;
    const int NK = nt * p.tile_slots;                // keys of the window (one S tile)
    // keys are split between the two threads of a row only for 256-key windows (w = 16); smaller windows use one
    const bool split = NK == 256;
    const int half_cols = split ? 128 : NK;
    const bool col_active = split || hc == 0;
    const uint32_t tail_mask = NK >= 32 ? 0xFFFFFFFFu : ((1u << NK) - 1u);  // 16-key windows (w = 4)
    const int c_lo = hc * half_cols;
    const bool pingpong = p.pingpong && nt == 2;
    uint32_t ph_t = 0;
    const float2 sl2 = make_float2(p.sl2, p.sl2);
    for (int item = blockIdx.x; item < p.n_items; item += gridDim.x) {
      int b, h, X0, Y0;
      decode(item, b, h, X0, Y0);
      const bool active = q_active(a, Y0);
      if (p.patch && a == 0) {
        // LEARNABLE pad patch of K/V rows outside the grid, by slot 0's 256 threads (slot 1 runs half an item
        // behind and never touches the stage's shared memory): entry e = key tile e>>7, slot e&127
        mbar_wait(&ld_full[stage], phase);
        for (int e = gtid; e < nt * 128; e += 256) {
          const int kt = e >> 7, r = e & 127;
          if (r >= p.tile_slots) continue;
          const int Y = Y0 + kt * p.rpt + (r >> p.lw), X = X0 + (r & (p.w - 1));
          if (Y < 0 || Y >= p.H || X < 0 || X >= p.W) {
            uint8_t* sK = smem + stage * STAGE + (2 + kt) * TILE;
            uint8_t* sV = smem + stage * STAGE + (4 + kt) * TILE;
            const uint4* kx = reinterpret_cast<const uint4*>(p.kx + ((size_t)(X + p.pl) * p.heads + h) * (D / 2));
            const uint4* ky = reinterpret_cast<const uint4*>(p.ky + ((size_t)(Y + p.pt) * p.heads + h) * (D / 2));
            const uint4* vp = reinterpret_cast<const uint4*>(p.vp + (size_t)h * D);
#pragma unroll
            for (int c = 0; c < D / 16; ++c) {
              *reinterpret_cast<uint4*>(sK + swz_offset(r, c, ROWB)) = kx[c];
              *reinterpret_cast<uint4*>(sK + swz_offset(r, c + D / 16, ROWB)) = ky[c];
            }
#pragma unroll
            for (int c = 0; c < D / 8; ++c) *reinterpret_cast<uint4*>(sV + swz_offset(r, c, ROWB)) = vp[c];
          }
        }
        fence_proxy_async_smem();
        mbar_arrive(&patch_done[stage]);
        __syncwarp();
      }
      if (active) {
        // MASKED: valid-key bitmask per 32-column chunk (real slots only); columns past the window are never read
        uint32_t xmask = 0xFFFFFFFFu;
        int iy_lo = 0, iy_hi = 1 << 30;
        if (MASKED) {
          const int xl = max(0, -X0), xh = min(p.w, p.W - X0);
          xmask = (xh > xl) ? (((1u << (xh - xl)) - 1u) << xl) : 0u;
          iy_lo = -Y0;
          iy_hi = p.H - Y0;
        }
        auto chunk_mask = [&](int c0) -> uint32_t {
          uint32_t m = 0;
          const int rows = 32 >> p.lw;
#pragma unroll 8
          for (int rr = 0; rr < rows; ++rr) {
            const int iy = (c0 >> p.lw) + rr;
            if (iy >= iy_lo && iy < iy_hi) m |= (xmask & ((1u << p.w) - 1u)) << (rr * p.w);
          }
          return m;
        };
        const int nc = col_active ? half_cols : 0;   // this thread's columns [c_lo, c_lo + nc)
        mbar_wait(&s_full[a], ph_s);
        ph_s ^= 1;
        if (row == 0 && hc == 0) ATT_TS(64 + 32 * a, ev);
        tc_fence_after();
        // pass 1: partial row max (two TMEM loads per wait::ld)
        float mx = -INFINITY;
        for (int c0 = c_lo; c0 < c_lo + nc; c0 += 64) {
          uint32_t r0[32], r1[32];
          const bool two = c0 + 32 < c_lo + nc;
          tmem_ld32(tS + c0, r0);
          if (two) tmem_ld32(tS + c0 + 32, r1);
          tmem_wait_ld();
          if (MASKED || tail_mask != 0xFFFFFFFFu) {
            const uint32_t m0 = (MASKED ? chunk_mask(c0) : 0xFFFFFFFFu) & tail_mask;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if ((m0 >> j) & 1u) mx = fmaxf(mx, __uint_as_float(r0[j]));
            if (two) {
              const uint32_t m1 = MASKED ? chunk_mask(c0 + 32) : 0xFFFFFFFFu;
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if ((m1 >> j) & 1u) mx = fmaxf(mx, __uint_as_float(r1[j]));
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(r0[j]));
            if (two) {
#pragma unroll
              for (int j = 0; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(r1[j]));
            }
          }
        }
        red_max[hc * 128 + row] = mx;
        named_bar_sync(1 + a, 256);
        mx = fmaxf(mx, red_max[(hc ^ 1) * 128 + row]);
        if (row == 0 && hc == 0) ATT_TS(64 + 32 * a, ev);  // max pass done (debug timeline)
        const float base = (mx == -INFINITY) ? 0.f : mx * p.sl2;
        const float2 nb = make_float2(-base, -base);
        // pass 2: p = 2^(s log2(e)/sqrt(d) - base) (packed fp32x2 scale, MUFU ex2), partial sums, P (bf16 pairs)
        // written over the consumed S columns
        float2 ls = make_float2(0.f, 0.f);
        // 16 columns per call; with kPolyMod = k > 0 the pairs of global index (OFF + j) / 2 = k - 1 (mod k) take the
        // FMA-pipe polynomial instead of MUFU ex2 (off: the softmax is latency-, not MUFU-bound, see the sweep)
        auto exp16 = [&](auto off_c, const uint32_t (&r)[16], uint32_t m, uint32_t (&pk)[8]) {
          constexpr int OFF = decltype(off_c)::value;
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            const float2 x = __ffma2_rn(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), sl2, nb);
            float e0, e1;
            if (kPolyMod > 0 && ((OFF + j) / 2) % kPolyMod == kPolyMod - 1) {
              const float2 e = exp2_poly2(x);
              e0 = e.x;
              e1 = e.y;
            } else {
              e0 = ex2_approx(x.x);
              e1 = ex2_approx(x.y);
            }
            if (MASKED || m != 0xFFFFFFFFu) {  // invalid keys, or stale columns past a 16-key window
              e0 = ((m >> (OFF + j)) & 1u) ? e0 : 0.f;
              e1 = ((m >> (OFF + j + 1)) & 1u) ? e1 : 0.f;
            }
            ls = __fadd2_rn(ls, make_float2(e0, e1));
            pk[j / 2] = pack_bf16(e0, e1);
          }
        };
        // P for key k goes to TMEM column k/2 (keys < 128) or 64 + k/2 (keys >= 128): each thread overwrites only S
        // columns it has already consumed (the PV MMA reads A from columns [0,64) and [128,192)).
        const int p_off = (split && hc) ? 64 : 0;
        {  // two 16-column register sets: the TMEM load of the next 16 columns is in flight while these are
           // exponentiated (the 96-register budget of 18 warps rules out 32-column double buffering)
          uint32_t ra[16], rb[16], pk[8];
          if (nc > 0) tmem_ld16(tS + c_lo, ra);
          if (pingpong) {  // the two slots' exp passes alternate (as in ROW1)
            mbar_wait(&turn[a], a == 0 ? ph_t ^ 1 : ph_t);
            ph_t ^= 1;
          }
          for (int c0 = c_lo; c0 < c_lo + nc; c0 += 32) {
            const uint32_t m = (MASKED ? chunk_mask(c0) : 0xFFFFFFFFu) & tail_mask;
            tmem_wait_ld_dep16(ra);
            tmem_ld16(tS + c0 + 16, rb);  // (a 16-key window reads 16 stale columns here, masked by tail_mask)
            exp16(std::integral_constant<int, 0>(), ra, m, pk);
            tmem_st8(tS + p_off + c0 / 2, pk);
            tmem_wait_ld_dep16(rb);
            if (c0 + 32 < c_lo + nc) tmem_ld16(tS + c0 + 32, ra);
            exp16(std::integral_constant<int, 16>(), rb, m, pk);
            tmem_st8(tS + p_off + c0 / 2 + 8, pk);
          }
        }
        if (pingpong) mbar_arrive(&turn[a ^ 1]);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&p_full[a]);
        red_sum[hc * 128 + row] = ls.x + ls.y;
        if (row == 0 && hc == 0) ATT_TS(64 + 32 * a, ev);
        // O = P V lands in columns [192, 192 + d): this thread takes d/2 of them (its column half), copies them to
        // registers, releases the TMEM columns (the next item's S may overwrite them), then normalises and writes
        // its half of the real query row to the grid (merge / crop)
        mbar_wait(&o_full[a], ph_o);
        ph_o ^= 1;
        if (row == 0 && hc == 0) ATT_TS(64 + 32 * a, ev);
        tc_fence_after();
        constexpr int DH = D / 2;
        uint32_t o[32];
        if (DH == 32) {
          tmem_ld32(tO + hc * 32, o);
        } else {
          uint32_t o16[16];
          tmem_ld16(tO + hc * 16, o16);
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] = o16[j];
        }
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&o_free[a]);
        named_bar_sync(1 + a, 256);  // partial sums of both halves are in shared memory
        const float lsum = red_sum[row] + (split ? red_sum[128 + row] : 0.f);
        // merge / crop: the normalised O tile is staged in this slot's Q region of the stage (Q_a is dead
        // once S_a has been computed) in the TMA box layout, and ONE 5-D tensor store writes the window's rows back
        // to the [B,H,W,C] grid; rows outside the grid (the pads) fall outside the tensor and are clipped by TMA
        // (a TMA tensor store whose box starts at a negative coordinate traps: windows of the first padded row /
        // column store their real rows directly instead; boxes running past the far edges are clipped)
        if (p.tma_out && X0 >= 0 && Y0 + a * p.rpt >= 0) {
          const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
          uint8_t* so = smem + stage * STAGE + a * TILE;
#pragma unroll
          for (int c = 0; c < DH / 8; ++c) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(o[c * 8 + 0]) * inv, __uint_as_float(o[c * 8 + 1]) * inv);
            v.y = pack_bf16(__uint_as_float(o[c * 8 + 2]) * inv, __uint_as_float(o[c * 8 + 3]) * inv);
            v.z = pack_bf16(__uint_as_float(o[c * 8 + 4]) * inv, __uint_as_float(o[c * 8 + 5]) * inv);
            v.w = pack_bf16(__uint_as_float(o[c * 8 + 6]) * inv, __uint_as_float(o[c * 8 + 7]) * inv);
            *reinterpret_cast<uint4*>(so + swz_offset(row, hc * (DH / 8) + c, ROWB)) = v;
          }
          fence_proxy_async_smem();
          named_bar_sync(1 + a, 256);
          if (gtid == 0) {
            tma_store_5d(&tmO, so, 0, h, X0, Y0 + a * p.rpt, b);
            bulk_commit();
            bulk_wait_read0();  // the stage's Q region may be refilled once the store has read it
            mbar_arrive(&ld_empty[stage]);
          }
        } else {
          const int iy = a * p.rpt + (row >> p.lw), ix = row & (p.w - 1);
          const int Y = Y0 + iy, X = X0 + ix;
          if (row < p.tile_slots && Y >= 0 && Y < p.H && X >= 0 && X < p.W) {
            const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
            uint4* dst =
                reinterpret_cast<uint4*>(p.out + (((size_t)b * p.H + Y) * p.W + X) * p.C + (size_t)h * D + hc * DH);
#pragma unroll
            for (int c = 0; c < DH / 8; ++c) {
              uint4 v;
              v.x = pack_bf16(__uint_as_float(o[c * 8 + 0]) * inv, __uint_as_float(o[c * 8 + 1]) * inv);
              v.y = pack_bf16(__uint_as_float(o[c * 8 + 2]) * inv, __uint_as_float(o[c * 8 + 3]) * inv);
              v.z = pack_bf16(__uint_as_float(o[c * 8 + 4]) * inv, __uint_as_float(o[c * 8 + 5]) * inv);
              v.w = pack_bf16(__uint_as_float(o[c * 8 + 6]) * inv, __uint_as_float(o[c * 8 + 7]) * inv);
              dst[c] = v;
            }
          }
          if (gtid == 0) mbar_arrive(&ld_empty[stage]);
        }
        if (row == 0 && hc == 0) ATT_TS(64 + 32 * a, ev);
      } else {
        if (pingpong) {  // an inactive q tile passes its exp turn on
          mbar_wait(&turn[a], a == 0 ? ph_t ^ 1 : ph_t);
          ph_t ^= 1;
          mbar_arrive(&turn[a ^ 1]);
        }
        if (gtid == 0) mbar_arrive(&ld_empty[stage]);  // nothing staged for an inactive q tile
      }
      __syncwarp();  // lane 0's store / arrival branch rejoins before the next item's .sync.aligned tcgen05 ops
      if (++stage == 2) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int launch_window_attention_ws(const AttnArgs& a, const void* kx, const void* ky, const void* vp, int patch,
                               cudaStream_t stream) {
  const int d = a.d, w = a.w;
  AttnWsArgs p;
  p.B = a.B;
  p.H = a.H;
  p.W = a.W;
  p.C = a.C;
  p.heads = a.heads;
  p.w = w;
  p.lw = 0;
  while ((1 << p.lw) < w) ++p.lw;
  p.pl = (w - a.sx) % w;
  p.pt = (w - a.sy) % w;
  const int pr = ((-(p.pl + a.W)) % w + w) % w;
  const int pb = ((-(p.pt + a.H)) % w + w) % w;
  p.nwx = (p.pl + a.W + pr) / w;
  p.nw = ((p.pt + a.H + pb) / w) * p.nwx;
  p.pad_mode = a.pad_mode;
  p.patch = patch;
  p.rpt = w * w <= 128 ? w : 128 / w;
  p.n_tiles = w / p.rpt;
  p.tile_slots = w * p.rpt;
  {
    const int nwy = p.nw / p.nwx;
    const int wy0 = a.wy_end > 0 ? a.wy_begin : 0, wy1 = a.wy_end > 0 ? (a.wy_end < nwy ? a.wy_end : nwy) : nwy;
    if (wy0 < 0 || wy0 >= wy1) return 0;  // empty range: nothing to run
    p.win0 = wy0 * p.nwx;
    p.nw_run = (wy1 - wy0) * p.nwx;
  }
  p.n_items = a.B * p.nw_run * a.heads;
  p.sl2 = 1.4426950408889634f / sqrtf((float)d);
  p.kx = reinterpret_cast<const __nv_bfloat16*>(kx);
  p.ky = reinterpret_cast<const __nv_bfloat16*>(ky);
  p.vp = reinterpret_cast<const __nv_bfloat16*>(vp);
  p.out = reinterpret_cast<__nv_bfloat16*>(a.out);
  p.dbg = nullptr;
  static const int direct_store = getenv("PSCWIN_ATTN_DIRECT_STORE") ? 1 : 0;  // A/B knob
  p.tma_out = !direct_store;
  static const int lockstep_knob = getenv("PSCWIN_ATTN_LOCKSTEP") ? atoi(getenv("PSCWIN_ATTN_LOCKSTEP")) : -1;
  p.lockstep = lockstep_knob;
  static const int pf_knob = env_knob("PSCWIN_ATTN_PF", 0);  // A/B knob: L2 prefetch distance (0 = off)
  p.pf = pf_knob < 0 ? 0 : pf_knob;
  static const int pp_knob = env_knob("PSCWIN_ATTN_PINGPONG", 1);  // A/B knob
  p.pingpong = pp_knob;
  static unsigned long long* dbg_buf = nullptr;
  static const char* tl = getenv("PSCWIN_ATTN_TIMELINE");  // debug knob, read once
  if (tl) {
    if (!dbg_buf) cudaMalloc(&dbg_buf, 148 * 128 * sizeof(unsigned long long));
    cudaMemsetAsync(dbg_buf, 0, 148 * 128 * sizeof(unsigned long long), stream);
    p.dbg = dbg_buf;
  }
  if (p.n_tiles > 2 || p.tile_slots < 16) return -2;
  CUtensorMap tmQKV, tmO;
  const uint64_t dq[5] = {(uint64_t)d, (uint64_t)3 * a.heads, (uint64_t)a.W, (uint64_t)a.H, (uint64_t)a.B};
  const uint64_t sq[4] = {(uint64_t)d * 2, (uint64_t)3 * a.C * 2, (uint64_t)a.W * 3 * a.C * 2,
                          (uint64_t)a.H * a.W * 3 * a.C * 2};
  const uint32_t box[5] = {(uint32_t)d, 1, (uint32_t)w, (uint32_t)p.rpt, 1};
  int rc = make_tmap_5d(&tmQKV, a.qkv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, dq, sq, box,
                        d == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
  if (rc) return rc;
  {  // O [B,H,W,heads,d]: the same window box, stored
    const uint64_t dout[5] = {(uint64_t)d, (uint64_t)a.heads, (uint64_t)a.W, (uint64_t)a.H, (uint64_t)a.B};
    const uint64_t sout[4] = {(uint64_t)d * 2, (uint64_t)a.C * 2, (uint64_t)a.W * a.C * 2, (uint64_t)a.H * a.W * a.C * 2};
    rc = make_tmap_5d(&tmO, a.out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, dout, sout, box,
                      d == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  }
  const size_t smem = 1024 + 2 * 6 * 128 * d * 2 + 18 * 8 + 1024 * 4;
  const int grid = p.n_items < num_sms() ? p.n_items : num_sms();
  PSCWIN_PROF("window_attention", stream);
  // one softmax thread per query row (default) or two (PSCWIN_ATTN_ROW2=1, the round-1 layout; A/B knob)
  static const bool row2 = env_knob("PSCWIN_ATTN_ROW2", 0) == 1;
  auto launch = [&](auto kern, int threads) {
    func_smem_once((const void*)kern, (int)smem);
    launch_k(kern, dim3(grid), dim3(threads), smem, stream, tmQKV, tmO, p);
  };
  const bool masked = p.pad_mode == 1;
  if (!row2) {
    if (d == 64)
      masked ? launch(window_attn_ws_kernel<64, true, true>, WS1_THREADS)
             : launch(window_attn_ws_kernel<64, false, true>, WS1_THREADS);
    else
      masked ? launch(window_attn_ws_kernel<32, true, true>, WS1_THREADS)
             : launch(window_attn_ws_kernel<32, false, true>, WS1_THREADS);
  } else if (d == 64) {
    masked ? launch(window_attn_ws_kernel<64, true, false>, WS_THREADS)
           : launch(window_attn_ws_kernel<64, false, false>, WS_THREADS);
  } else {
    masked ? launch(window_attn_ws_kernel<32, true, false>, WS_THREADS)
           : launch(window_attn_ws_kernel<32, false, false>, WS_THREADS);
  }
  if (tl) {  // debug: dump the per-CTA phase timeline (globaltimer ns)
    static unsigned long long host[148 * 128];
    cudaMemcpyAsync(host, dbg_buf, sizeof(host), cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    FILE* f = fopen(tl, "ab");
    if (f) {
      fwrite(host, sizeof(host), 1, f);
      fclose(f);
    }
  }
  return (int)cudaGetLastError();
}

}  // namespace pscwin
