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
constexpr int B_STAGE_BYTES = 256 * BK * 2;      // 32 KB (max BN)
constexpr int STAGE_OUT_BYTES = BM * 64 * 2;   // one 128x64 bf16 output chunk
constexpr int GEMM_THREADS = 64 + 256;      // TMA warp, MMA warp, 8 epilogue warps
constexpr size_t GEMM_SMEM = 1024 /*align slack*/ + STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + 2 * STAGE_OUT_BYTES + 256;
}  // namespace

__device__ __forceinline__ void rope_pair(float& a, float& b, float c, float s) {
  float x0 = a * c - b * s;
  float x1 = a * s + b * c;
  a = x0;
  b = x1;
}

__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmOut, GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
  uint8_t* s_stage = sB + STAGES * B_STAGE_BYTES;   // 2 x 16 KB output staging (1024-aligned)
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_stage + 2 * STAGE_OUT_BYTES);
  uint64_t* full = bars;                 // [STAGES]
  uint64_t* empty = bars + STAGES;       // [STAGES]
  uint64_t* tfull = bars + 2 * STAGES;   // [2]
  uint64_t* tempty = bars + 2 * STAGES + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = warp_id();
  const int BN = p.BN;
  const int n_tiles_n = (p.N + BN - 1) / BN;
  const int n_tiles = ((p.M + BM - 1) / BM) * n_tiles_n;
  const int nk = (p.K + BK - 1) / BK;

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
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_a = policy_evict_normal();
      const uint64_t pol_b = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int m0 = (tile / n_tiles_n) * BM;
        const int n0 = (tile % n_tiles_n) * BN;
        for (int kb = 0; kb < nk; ++kb) {
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
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * 256;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a0 = smem_u32(sA + stage * A_STAGE_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * B_STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t ad = make_sdesc(a0 + k * 32, 16, 1024, kLayoutSW128);
            uint64_t bd = make_sdesc(b0 + k * 32, 16, 1024, kLayoutSW128);
            umma_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (kb == nk - 1) umma_commit(&tfull[acc]);
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
    const int nch = (BN + 63) / 64;
    int acc = 0;
    uint32_t acc_phase = 0;
    int gseq = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const int m0 = (tile / n_tiles_n) * BM;
      const int n0 = (tile % n_tiles_n) * BN;
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
      const uint32_t t_row = tmem_base + acc * 256 + ((uint32_t)(quarter * 32) << 16);
      for (int cc = 0; cc < nch; ++cc, ++gseq) {
        const int cl = cc * 64 + half * 32;            // tile-local first column of this thread's 32
        const int col0 = n0 + cl;
        // residual prefetch (bf16, 4 x 16B) before the TMEM load
        uint4 res[4];
        const bool use_res = p.epi == EPI_RESID_BF16 && p.residual != nullptr;
        if (use_res) {
          const uint4* rp = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p.residual) +
                                                           (size_t)row * p.ldr + col0);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            res[q] = (row_ok && cl < BN && col0 + 8 * q < p.N) ? rp[q] : make_uint4(0, 0, 0, 0);
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
        if (p.bias) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col0 + j < p.N) v[j] += __ldg(p.bias + col0 + j);
        }
        if (p.epi == EPI_QKV_ROPE && p.rope && col0 < 2 * p.C) {  // q = cols [0,C), k = [C,2C)
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) rope_pair(v[2 * jj], v[2 * jj + 1], rc[jj], rs[jj]);
        }
        if (use_res) {
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
          float* o = reinterpret_cast<float*>(p.out) + (size_t)row * p.ldo + col0;
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            if (col0 + j < p.N) {
              if (col0 + j + 4 <= p.N && (p.ldo % 4) == 0) {
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
  // tile N: a single tile when N <= 256; else 256, or 128 when 256-wide tiles would leave SMs idle
  if (p.BN <= 0) {
    if (p.N <= 256) {
      p.BN = ((p.N + 15) / 16) * 16;
    } else {
      const long long t256 = (long long)((p.M + BM - 1) / BM) * ((p.N + 255) / 256);
      p.BN = t256 >= 2LL * num_sms() ? 256 : 128;
    }
  }
  CUtensorMap tmA, tmB, tmOut;
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
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM);
    attr_set = true;
  }
  int tiles = ((p.M + BM - 1) / BM) * ((p.N + p.BN - 1) / p.BN);
  int grid = tiles < num_sms() ? tiles : num_sms();
  PSCWIN_PROF(p.prof_name ? p.prof_name : "gemm", stream);
  gemm_bf16_kernel<<<grid, GEMM_THREADS, GEMM_SMEM, stream>>>(tmA, tmB, tmOut, p);
  return (int)cudaGetLastError();
}

}  // namespace pscwin
