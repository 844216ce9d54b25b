// Projection GEMMs of the PSCWin layer on 5th-gen tensor cores:
//   out[M, N] = epilogue( A[M, K] . B[N, K]^T )      A, B bf16 K-major (activations x nn.Linear weight [out, in])
// Epilogues: plain bf16 / f32 store (in_proj, x_proj), bias + 2-D RoPE at the token's grid coordinate (QKV, a4,
// PAPER P:L89 "replaces SAM's relative encoding with RoPE", form = DESIGN.md reading Q6), bias + residual
// (out-proj a7 / cycle-scan out_proj a3).
//
// Structure (B200-native): persistent grid (one CTA per SM), warp-specialised —
//   warp 0: TMA producer (128B-swizzled A/B k-blocks of 64, 4-stage mbarrier ring)
//   warp 1: TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN<=256, K=16 per instruction)
//   warps 2-9: epilogue (tcgen05.ld 32x32b -> registers -> fused op -> swizzled smem -> TMA tensor store),
//   double-buffered TMEM accumulators (2 x 256 columns) so the epilogue of tile i overlaps the MMAs of tile i+1.
#include <string.h>

#include "common.cuh"
#include "pscwin_internal.h"

namespace pscwin {

namespace {
constexpr int BM = 128;
constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int A_STAGE_BYTES = BM * BK * 2;       // 16 KB
constexpr int STAGE_OUT_BYTES = BM * 64 * 2;     // one 128x64 bf16 output / residual chunk (16 KB)
constexpr int GEMM_THREADS = 64 + 256;           // TMA warp, MMA warp, 8 epilogue warps
constexpr size_t GEMM_SMEM_MAX = 230656;         // 1024 + 4 x 48 KB + 32 KB + 256 (also = BN 128 + residual)
// shared memory layout for a tile width BN (B stage = BN x 64 bf16; residual tiles double-buffered)
__host__ __device__ inline size_t gemm_smem_bytes(int BN, bool resid) {
  const size_t nch = (size_t)(BN + 63) / 64;
  return 1024 + (size_t)STAGES * (A_STAGE_BYTES + (size_t)BN * BK * 2) + 2 * STAGE_OUT_BYTES +
         (resid ? 2 * nch * STAGE_OUT_BYTES : 0) + 256;
}
}  // namespace

__device__ __forceinline__ void rope_pair(float& a, float& b, float c, float s) {
  float x0 = a * c - b * s;
  float x1 = a * s + b * c;
  a = x0;
  b = x1;
}

__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmOut, const __grid_constant__ CUtensorMap tmRes,
                     GemmArgs p) {
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  const int BN = p.BN;
  const int B_STAGE_BYTES = BN * BK * 2;
  const bool resid_tma = p.epi == EPI_RESID_BF16 && p.residual != nullptr;
  const int nch = (BN + 63) / 64;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
  uint8_t* s_stage = sB + STAGES * B_STAGE_BYTES;   // 2 x 16 KB output staging (1024-aligned)
  uint8_t* s_res = s_stage + 2 * STAGE_OUT_BYTES;   // 2 x nch x 16 KB residual tiles (TMA-loaded)
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_res + (resid_tma ? 2 * nch * STAGE_OUT_BYTES : 0));
  uint64_t* full = bars;                 // [STAGES]
  uint64_t* empty = bars + STAGES;       // [STAGES]
  uint64_t* tfull = bars + 2 * STAGES;   // [2]
  uint64_t* tempty = bars + 2 * STAGES + 2;  // [2]
  uint64_t* rfull = bars + 2 * STAGES + 4;   // [2] residual tile landed
  uint64_t* rempty = bars + 2 * STAGES + 6;  // [2] residual tile consumed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 8);
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = warp_id();
  const int n_tiles_n = (p.N + BN - 1) / BN;
  const int S = p.splits > 1 ? p.splits : 1;  // split-K factor (f32 outputs only)
  const int n_tiles = ((p.M + BM - 1) / BM) * n_tiles_n * S;
  const int nk = (p.K + BK - 1) / BK;
  // work tile -> output tile (m0, n0), k-block range [kb0, kb1) and split index
  auto coords = [&](int tile, int& m0, int& n0, int& kb0, int& kb1, int& s) {
    const int mn = tile / S;
    s = tile - mn * S;
    m0 = (mn / n_tiles_n) * BM;
    n0 = (mn % n_tiles_n) * BN;
    kb0 = (int)((long long)nk * s / S);
    kb1 = (int)((long long)nk * (s + 1) / S);
  };

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (p.epi != EPI_STORE_F32) tma_prefetch_desc(&tmOut);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 256);
      mbar_init(&rfull[i], 1);
      mbar_init(&rempty[i], 256);
    }
    if (resid_tma) tma_prefetch_desc(&tmRes);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();  // barrier init / TMEM allocation / descriptor prefetch overlap the previous kernel
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_a = policy_evict_normal();
      const uint64_t pol_b = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      int rbuf = 0;
      uint32_t rphase = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        int m0, n0, kb0, kb1, s;
        coords(tile, m0, n0, kb0, kb1, s);
        if (resid_tma) {
          // residual tile of this output tile (double-buffered, consumed by the epilogue), issued ahead of the k-loop
          mbar_wait(&rempty[rbuf], rphase ^ 1);
          mbar_arrive_expect_tx(&rfull[rbuf], nch * STAGE_OUT_BYTES);
          for (int c = 0; c < nch; ++c)
            tma_load_2d(s_res + (rbuf * nch + c) * STAGE_OUT_BYTES, &tmRes, &rfull[rbuf], n0 + c * 64, m0, pol_a);
          if (++rbuf == 2) {
            rbuf = 0;
            rphase ^= 1;
          }
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], A_STAGE_BYTES + BN * BK * 2);
          tma_load_2d(sA + stage * A_STAGE_BYTES, &tmA, &full[stage], kb * BK, m0, pol_a);
          tma_load_2d(sB + stage * B_STAGE_BYTES, &tmB, &full[stage], kb * BK, n0, pol_b);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc_bf16(BM, BN, 0, 0);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      int m0, n0, kb0, kb1, s;
      coords(tile, m0, n0, kb0, kb1, s);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * 256;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a0 = smem_u32(sA + stage * A_STAGE_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * B_STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t ad = make_sdesc(a0 + k * 32, 16, 1024, kLayoutSW128);
            uint64_t bd = make_sdesc(b0 + k * 32, 16, 1024, kLayoutSW128);
            umma_ss(d_tmem, ad, bd, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (kb == kb1 - 1) umma_commit(&tfull[acc]);
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
  } else {
    // ------------------------------------------------------------------ epilogue warps 2..9
    // Two warps per TMEM lane quarter (rows), each taking 32 of every 64 accumulator columns. bf16 outputs are
    // staged in 128B-swizzled smem (two 128x64 buffers) and written by TMA tensor stores (coalesced, async);
    // f32 outputs are stored directly.
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int lane = lane_id();
    const int etid = threadIdx.x - 64;                 // 0..255
    const bool issuer = etid == 0;
    const bool tma_out = p.epi != EPI_STORE_F32;
    const int row_local = quarter * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    int gseq = 0;
    int rbuf = 0;
    uint32_t rphase = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      int m0, n0, kb0, kb1, split;
      coords(tile, m0, n0, kb0, kb1, split);
      const int row = m0 + row_local;
      const bool row_ok = row < p.M;
      // RoPE of this row (QKV epilogue): this thread's 32 columns of every 64-column chunk are one half of a head
      // (d = 64: axis = half, pair jj -> frequency jj) or one whole head (d = 32: pairs 0-7 x, 8-15 y).
      float rc[16], rs[16];
      if (p.epi == EPI_QKV_ROPE && p.rope) {
        const int t = row % p.HW;
        const int py = t / p.Wgrid, px = t - py * p.Wgrid;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int axis = p.d_head == 64 ? half : (jj >= 8);
          const int fj = p.d_head == 64 ? jj : (jj & 7);
          rope_cs(axis ? py : px, fj, p.d_head, rc[jj], rs[jj]);
        }
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (resid_tma) mbar_wait(&rfull[rbuf], rphase);
      const uint32_t t_row = tmem_base + acc * 256 + ((uint32_t)(quarter * 32) << 16);
      for (int cc = 0; cc < nch; ++cc, ++gseq) {
        const int cl = cc * 64 + half * 32;            // tile-local first column of this thread's 32
        const int col0 = n0 + cl;
        // residual: this thread's 4 x 16B of the TMA-loaded tile (swizzled like the output staging)
        uint4 res[4];
        if (resid_tma) {
          const uint8_t* rt = s_res + (rbuf * nch + cc) * STAGE_OUT_BYTES;
#pragma unroll
          for (int q = 0; q < 4; ++q) res[q] = *reinterpret_cast<const uint4*>(rt + swz_offset(row_local, half * 4 + q, 128));
        }
        uint8_t* stg = s_stage + (gseq & 1) * STAGE_OUT_BYTES;
        if (tma_out) {
          if (issuer && gseq >= 2) bulk_wait_read1();
          named_bar_sync(1, 256);
        }
        uint32_t r[32];
        if (cl < BN) {
          tmem_ld32(t_row + cl, r);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = 0u;
        }
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (p.bias) {  // 16-byte broadcast loads (every lane of the warp reads the same columns)
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            if (col0 + j + 4 <= p.N) {
              const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + col0 + j));
              v[j] += b4.x; v[j + 1] += b4.y; v[j + 2] += b4.z; v[j + 3] += b4.w;
            } else {
              for (int e = 0; e < 4 && col0 + j + e < p.N; ++e) v[j + e] += __ldg(p.bias + col0 + j + e);
            }
        }
        if (p.epi == EPI_QKV_ROPE && p.rope && col0 < 2 * p.C) {  // q = cols [0,C), k = [C,2C)
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) rope_pair(v[2 * jj], v[2 * jj + 1], rc[jj], rs[jj]);
        }
        if (p.silu_col > 0 && col0 >= p.silu_col) {  // gate columns: SiLU(x) = x / (1 + e^-x)
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __fdividef(v[j], 1.f + __expf(-v[j]));
        }
        if (resid_tma) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t* rw = reinterpret_cast<const uint32_t*>(&res[q]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              v[8 * q + 2 * e] += bf16_lo(rw[e]);
              v[8 * q + 2 * e + 1] += bf16_hi(rw[e]);
            }
          }
        }
        if (tma_out) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 w;
            w.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
            w.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
            w.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
            w.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
            *reinterpret_cast<uint4*>(stg + swz_offset(row_local, half * 4 + q, 128)) = w;
          }
          fence_proxy_async_smem();
          named_bar_sync(1, 256);
          if (issuer) {
            tma_store_2d(&tmOut, stg, n0 + cc * 64, m0);
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
      mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      if (resid_tma) {
        mbar_arrive(&rempty[rbuf]);
        if (++rbuf == 2) {
          rbuf = 0;
          rphase ^= 1;
        }
      }
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
    if (issuer && tma_out) bulk_wait0();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

int launch_gemm_bf16(const void* A, const void* Bw, const GemmArgs& args_in, cudaStream_t stream) {
  GemmArgs p = args_in;
  if (p.M <= 0 || p.N <= 0) return 0;
  if (p.K % 8 != 0) return -1;
  if (p.epi == EPI_QKV_ROPE && p.rope && !(p.d_head == 32 || p.d_head == 64)) return -2;
  const bool resid = p.epi == EPI_RESID_BF16 && p.residual != nullptr;
  // tile N: a single tile when N <= 256; else 256, or 128 when 256-wide tiles would leave SMs idle. Residual
  // epilogues stage the residual tile in shared memory, which fits next to the 4-stage ring only for BN <= 128.
  if (p.BN <= 0) {
    if (p.N <= (resid ? 128 : 256)) {
      p.BN = ((p.N + 15) / 16) * 16;
    } else {
      const long long t256 = (long long)((p.M + BM - 1) / BM) * ((p.N + 255) / 256);
      p.BN = (!resid && t256 >= 2LL * num_sms()) ? 256 : 128;
    }
  }
  if (resid && p.BN > 128) return -2;
  if (p.silu_col && (p.silu_col % 32 || p.epi == EPI_STORE_F32)) return -2;
  if (p.splits > 1 && (p.epi != EPI_STORE_F32 || !p.partial || !p.sem || p.splits > 8 || p.N % 4 || p.ldo % 4))
    return -3;
  CUtensorMap tmA, tmB, tmOut, tmRes;
  int rc = make_tmap_2d(&tmA, A, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, p.K, p.M, (uint64_t)p.lda * 2, BK, BM,
                        CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_2d(&tmB, Bw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, p.K, p.N, (uint64_t)p.ldb * 2, BK, p.BN,
                    CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  memset(&tmOut, 0, sizeof(tmOut));
  if (p.epi != EPI_STORE_F32) {
    if ((p.ldo * 2) % 16) return -1;
    rc = make_tmap_2d(&tmOut, p.out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, p.N, p.M, (uint64_t)p.ldo * 2, 64, BM,
                      CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  memset(&tmRes, 0, sizeof(tmRes));
  if (resid) {
    if ((p.ldr * 2) % 16) return -1;
    rc = make_tmap_2d(&tmRes, p.residual, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, p.N, p.M, (uint64_t)p.ldr * 2, 64, BM,
                      CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM_MAX);
    attr_set = true;
  }
  const size_t smem = gemm_smem_bytes(p.BN, resid);
  if (smem > GEMM_SMEM_MAX) return -2;
  const long long tiles = (long long)((p.M + BM - 1) / BM) * ((p.N + p.BN - 1) / p.BN) * (p.splits > 1 ? p.splits : 1);
  const int grid = tiles < num_sms() ? (int)tiles : num_sms();
  PSCWIN_PROF(p.prof_name ? p.prof_name : "gemm", stream);
  launch_k(gemm_bf16_kernel, dim3(grid), dim3(GEMM_THREADS), smem, stream, tmA, tmB, tmOut, tmRes, p);
  return (int)cudaGetLastError();
}

}  // namespace pscwin
