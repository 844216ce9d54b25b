// Projection GEMMs of the PSCWin layer on 5th-gen tensor cores:
//   out[M, N] = epilogue( A[M, K] . B[N, K]^T )      A, B bf16 K-major (activations x nn.Linear weight [out, in])
// Epilogues: plain bf16 / f32 store (in_proj, x_proj), bias + 2-D RoPE at the token's grid coordinate (QKV, a4,
// PAPER P:L89 "replaces SAM's relative encoding with RoPE", form = DESIGN.md reading Q6), bias + residual
// (out-proj a7 / cycle-scan out_proj a3).
//
// Structure (B200-native): persistent grid (one CTA per SM), warp-specialised —
//   warp 0: TMA producer (128B-swizzled A/B k-blocks of 64, 4-stage mbarrier ring)
//   warp 1: TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN<=256, K=16 per instruction)
//   warps 2-5: epilogue (tcgen05.ld 32x32b -> registers -> fused op -> global), double-buffered TMEM
//   accumulators (2 x 256 columns) so the epilogue of tile i overlaps the MMAs of tile i+1.
#include "common.cuh"
#include "pscwin_internal.h"

namespace pscwin {

namespace {
constexpr int BM = 128;
constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int A_STAGE_BYTES = BM * BK * 2;       // 16 KB
constexpr int B_STAGE_BYTES = 256 * BK * 2;      // 32 KB (max BN)
constexpr int GEMM_THREADS = 192;
constexpr size_t GEMM_SMEM = 1024 /*align slack*/ + STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + 256;
}  // namespace

__device__ __forceinline__ void rope_pair(float& a, float& b, float c, float s) {
  float x0 = a * c - b * s;
  float x1 = a * s + b * c;
  a = x0;
  b = x1;
}

__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE_BYTES);
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
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
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
    // ------------------------------------------------------------------ epilogue warps 2..5
    const int quarter = warp & 3;            // TMEM lane quarter this warp may access
    const int lane = lane_id();
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const int m0 = (tile / n_tiles_n) * BM;
      const int n0 = (tile % n_tiles_n) * BN;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + quarter * 32 + lane;
      const bool row_ok = row < p.M;
      // RoPE coordinates of this token (QKV epilogue): row = b*H*W + y*W + x
      int px = 0, py = 0;
      if (p.epi == EPI_QKV_ROPE && p.rope) {
        int t = row % p.HW;
        py = t / p.Wgrid;
        px = t - py * p.Wgrid;
      }
      const uint32_t t_row = tmem_base + acc * 256 + ((uint32_t)(quarter * 32) << 16);
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(t_row + c0, r);
        tmem_wait_ld();
        const int col0 = n0 + c0;
        if (!row_ok || col0 >= p.N) continue;
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
        const int ncols = min(16, p.N - col0);
        if (p.bias) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < ncols) v[j] += p.bias[col0 + j];
        }
        if (p.epi == EPI_QKV_ROPE && p.rope && col0 < 2 * p.C) {
          // columns [0,C) = q, [C,2C) = k; head-local index i = col % d; half = i / (d/2); pair j = (i % (d/2))/2
          const int d = p.d_head;
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            const int i = (col0 + j) % d;
            const int half = i / (d >> 1);
            const int fj = (i - half * (d >> 1)) >> 1;
            const int pos = half ? py : px;
            const float2 cs = p.rope_tab[(pos + p.rope_off) * (d >> 2) + fj];
            rope_pair(v[j], v[j + 1], cs.x, cs.y);
          }
        }
        if (p.epi == EPI_RESID_BF16 && p.residual) {
          const __nv_bfloat16* res = reinterpret_cast<const __nv_bfloat16*>(p.residual) + (size_t)row * p.ldr + col0;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < ncols) v[j] += __bfloat162float(res[j]);
        }
        if (p.epi == EPI_STORE_F32) {
          float* o = reinterpret_cast<float*>(p.out) + (size_t)row * p.ldo + col0;
          if (ncols == 16 && (p.ldo % 4) == 0) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
            for (int j = 0; j < ncols; ++j) o[j] = v[j];
          }
        } else {
          __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + (size_t)row * p.ldo + col0;
          if (ncols == 16 && (p.ldo % 8) == 0) {
            uint4 w0, w1;
            w0.x = pack_bf16(v[0], v[1]);
            w0.y = pack_bf16(v[2], v[3]);
            w0.z = pack_bf16(v[4], v[5]);
            w0.w = pack_bf16(v[6], v[7]);
            w1.x = pack_bf16(v[8], v[9]);
            w1.y = pack_bf16(v[10], v[11]);
            w1.z = pack_bf16(v[12], v[13]);
            w1.w = pack_bf16(v[14], v[15]);
            reinterpret_cast<uint4*>(o)[0] = w0;
            reinterpret_cast<uint4*>(o)[1] = w1;
          } else {
            for (int j = 0; j < ncols; ++j) o[j] = __float2bfloat16_rn(v[j]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// RoPE table: tab[(pos + off) * (d/4) + j] = (cos, sin)(pos * 10000^(-4j/d)), pos in [-off, n - off).
__global__ void rope_table_kernel(float2* tab, int n_pos, int off, int d) {
  int q = d / 4;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pos * q) return;
  int pos = i / q - off;
  int j = i % q;
  double theta = pow(10000.0, -4.0 * j / d);
  double s, c;
  sincos((double)pos * theta, &s, &c);
  tab[i] = make_float2((float)c, (float)s);
}

int launch_rope_table(float2* tab, int n_pos, int off, int d, cudaStream_t stream) {
  int n = n_pos * (d / 4);
  PSCWIN_PROF("rope_table", stream);
  rope_table_kernel<<<(n + 255) / 256, 256, 0, stream>>>(tab, n_pos, off, d);
  return (int)cudaGetLastError();
}

int launch_gemm_bf16(const void* A, const void* Bw, const GemmArgs& args_in, cudaStream_t stream) {
  GemmArgs p = args_in;
  if (p.M <= 0 || p.N <= 0) return 0;
  if (p.K % 8 != 0) return -1;
  // tile N: 256 when N is large, else N rounded up to 16
  if (p.BN <= 0) p.BN = p.N >= 256 ? 256 : ((p.N + 15) / 16) * 16;
  CUtensorMap tmA, tmB;
  int rc = make_tmap_2d(&tmA, A, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, p.K, p.M, (uint64_t)p.lda * 2, BK, BM,
                        CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_2d(&tmB, Bw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, p.K, p.N, (uint64_t)p.ldb * 2, BK, p.BN,
                    CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM);
    attr_set = true;
  }
  int tiles = ((p.M + BM - 1) / BM) * ((p.N + p.BN - 1) / p.BN);
  int grid = tiles < num_sms() ? tiles : num_sms();
  PSCWIN_PROF(p.prof_name ? p.prof_name : "gemm", stream);
  gemm_bf16_kernel<<<grid, GEMM_THREADS, GEMM_SMEM, stream>>>(tmA, tmB, p);
  return (int)cudaGetLastError();
}

}  // namespace pscwin
