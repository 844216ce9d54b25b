// The attention softmax's exp pass in isolation (sm_100a): one CTA per SM, 4 warps (one per SM sub-partition, one
// thread per TMEM lane = query row), each pass reads a row's 256 f32 logits from TMEM in 32-column chunks (next
// chunk's tcgen05.ld in flight), computes p = 2^(s c - m) (FFMA2 + MUFU.EX2), the row sum (FADD2) and bf16 pairs
// (F2FP) written back to TMEM (tcgen05.st.x16). MODE 0: as in the kernel; 1: no TMEM store; 2: no TMEM load (logits
// from registers); 3: mode 0 plus 4 more warps streaming TMEM loads (the other q-tile slot's max pass).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o softmax_pass softmax_pass.cu && ./softmax_pass
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../paper_2407_02109_b200/csrc/common.cuh"

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pack(float a, float b) {
  uint32_t r; asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b)); return r;
}
#define LD32(addr, r)                                                                                           \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                        \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),       \
                 "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),     \
                 "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),     \
                 "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                           \
               : "r"(addr))
#define WAITLD(r)                                                                                                \
  asm volatile("tcgen05.wait::ld.sync.aligned;"                                                                  \
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]), \
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),       \
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),     \
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),     \
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])::"memory")
#define ST16(addr, r)                                                                                             \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
               ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),   \
               "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory")

template <int MODE>
__global__ void __launch_bounds__(320, 1) kern(int iters, long long* clk, float* out) {
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tS = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >= 4 ? 256u : 0u);
  float2 ls[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  const float2 sc = make_float2(0.18f, 0.18f), nb = make_float2(-1.f, -1.f);
  uint32_t acc = 0;
  long long t0 = clock64();
  if (warp < 4) {
    for (int it = 0; it < iters; ++it) {
      uint32_t ra[32], rb[32], pk[16];
      if (MODE != 2) LD32(tS, ra); else for (int j = 0; j < 32; ++j) ra[j] = __float_as_uint(0.001f * j + it);
      auto exp32 = [&](const uint32_t (&r)[32]) {
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), sc, nb);
          const float e0 = ex2(x.x), e1 = ex2(x.y);
          ls[(j >> 1) & 1] = __fadd2_rn(ls[(j >> 1) & 1], make_float2(e0, e1));
          pk[j / 2] = pack(e0, e1);
        }
      };
      for (int c0 = 0; c0 < 256; c0 += 64) {
        if (MODE != 2) WAITLD(ra);
        if (MODE != 2) LD32(tS + c0 + 32, rb); else for (int j = 0; j < 32; ++j) rb[j] = ra[j] ^ 1u;
        exp32(ra);
        if (MODE != 1) ST16(tS + c0 / 2, pk); else acc ^= pk[3] ^ pk[11];
        if (MODE != 2) WAITLD(rb);
        if (MODE != 2 && c0 + 64 < 256) LD32(tS + c0 + 64, ra);
        exp32(rb);
        if (MODE != 1) ST16(tS + c0 / 2 + 16, pk); else acc ^= pk[5] ^ pk[9];
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  } else if (MODE == 5) {  // warp 4: back-to-back tcgen05.mma (M 128, N 256, K 64 per group) into TMEM columns
    // [256, 512) (the other q-tile slot's S), operands from shared memory, one commit + wait per group
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    const uint32_t idesc = pscwin::make_idesc_bf16(128, 256, 0, 0);
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sm), b0 = a0 + 16384;
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      if (pscwin::elect_one()) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          pscwin::umma_ss(slot + 256, pscwin::make_sdesc(a0 + k * 32, 16, 1024, pscwin::kLayoutSW128),
                          pscwin::make_sdesc(b0 + k * 32, 16, 1024, pscwin::kLayoutSW128), idesc, k > 0);
        pscwin::umma_commit(&bar);
      }
      __syncwarp();
      pscwin::mbar_wait(&bar, ph);
      ph ^= 1;
    }
  } else if (MODE == 4) {  // idle warps spinning on an mbarrier (try_wait loop, as the kernel's waiting roles do)
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"((uint32_t)__cvta_generic_to_shared(&bar))
        : "memory");
  } else if (MODE == 3) {  // the other slot: max passes (TMEM loads + max) over its own 256 columns
    float mx = -1e30f;
    for (int it = 0; it < iters; ++it) {
      for (int c0 = 0; c0 < 256; c0 += 64) {
        uint32_t r0[32], r1[32];
        LD32(tS + c0, r0);
        LD32(tS + c0 + 32, r1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) mx = fmaxf(mx, fmaxf(__uint_as_float(r0[j]), __uint_as_float(r1[j])));
      }
    }
    acc = __float_as_uint(mx);
  }
  long long t1 = clock64();
  if (MODE == 4 && warp < 4) {  // release the spinners once every exp warp is done
    __syncwarp();
    if (threadIdx.x == 0) {
      // (other exp warps may still run: the spinners only need to finish eventually)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = ls[0].x + ls[1].y + (float)acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int MODE>
void run(const char* name, int threads) {
  long long* clk; float* out;
  cudaMalloc(&clk, 8); cudaMalloc(&out, 148 * 320 * 4);
  const int iters = 2000;
  const int smem = MODE == 5 ? 50 * 1024 : 0;
  if (smem) cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<MODE><<<148, threads, smem>>>(10, clk, out);
  cudaDeviceSynchronize();
  kern<MODE><<<148, threads, smem>>>(iters, clk, out);
  cudaError_t e = cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  // MUFU floor per pass: 128 rows x 256 ex2 / 16 per clk = 2048 clk
  printf("%-28s %7.0f clk per 256-key pass (MUFU floor 2048) %s\n", name, (double)c / iters, cudaGetErrorString(e));
  cudaFree(clk); cudaFree(out);
}

int main() {
  run<0>("exp pass (kernel loop)", 128);
  run<1>("  no TMEM store", 128);
  run<2>("  no TMEM load", 128);
  run<3>("  + 4 warps of max passes", 256);
  run<4>("  + 4 warps spinning", 256);
  run<4>("  + 6 warps spinning", 320);
  run<5>("  + MMAs into the other TMEM half", 160);
  return 0;
}
