// Pipe-throughput microbenchmark (sm_100a): MUFU.EX2, FFMA, FFMA2 and the scan's mix, per SM per clock.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu && ./pipes
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
// packed half-precision exp2: two results per lane per instruction (MODE 4: f16x2, MODE 5: bf16x2)
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2b2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }

template <int MODE>
__global__ void kern(float* out, int iters, long long* clk) {
  float a[16];
  float2 b[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { a[i] = threadIdx.x * 1e-6f + i * 1e-3f; b[i] = make_float2(a[i], -a[i]); }
  const float2 m = make_float2(0.999f, 0.999f), c = make_float2(1e-4f, 1e-4f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) * -0.5f;                       // MUFU + FMUL
      if (MODE == 1) a[i] = fmaf(a[i], 0.999f, 1e-4f);                // FFMA
      if (MODE == 2) b[i] = __ffma2_rn(b[i], m, c);                    // FFMA2
      if (MODE == 4) {  // packed f16x2 exp2 (the chain keeps values in (0, 1): y = 2^x * -0.5 via the sign bit)
        uint32_t h = __float_as_uint(a[i]);
        h = ex2h2(h) ^ 0x80008000u;
        a[i] = __uint_as_float(h);
      }
      if (MODE == 5) {
        uint32_t h = __float_as_uint(a[i]);
        h = ex2b2(h) ^ 0x80008000u;
        a[i] = __uint_as_float(h);
      }
      if (MODE == 6) {  // F2FP: cvt.rn.bf16x2.f32 (the softmax's P pack), chained through a LOP3
        uint32_t h;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(a[i]), "f"(b[i].x));
        a[i] = __uint_as_float(h & 0x3f7f3f7fu);
      }
      if (MODE == 7) {  // softmax mix per pair: FFMA2 scale, 2 MUFU ex2, FADD2 sum, F2FP pack
        const float2 x = __ffma2_rn(b[i], m, c);
        const float2 e = make_float2(ex2(x.x), ex2(x.y));
        uint32_t h;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(e.x), "f"(e.y));
        b[i] = __fadd2_rn(e, make_float2(__uint_as_float(h & 0x3f7f3f7fu), 0.f));
      }
      if (MODE == 3) {                                                 // scan pass-2 mix per pair: 2 MUFU, 3 FMUL2, 3 FFMA2
        float2 x = __fmul2_rn(b[i], m);
        float2 e = make_float2(ex2(x.x), ex2(x.y));
        float2 w = __fmul2_rn(e, c);
        float2 t = __ffma2_rn(w, m, b[i]);
        b[i] = __ffma2_rn(e, t, w);
        float2 q = __fmul2_rn(t, c);
        b[i] = __ffma2_rn(q, b[i], c);
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i] + b[i].x + b[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int MODE>
void run(const char* name, double ops_per_inner, int threads, int per_sm = 2048) {
  float* out; long long* clk;
  cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaMalloc(&clk, 8);
  const int iters = 4096;
  const int blocks = 148 * (per_sm / threads);
  kern<MODE><<<blocks, threads>>>(out, 16, clk);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<MODE><<<blocks, threads>>>(out, iters, clk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  double total = (double)blocks * threads * iters * 16 * ops_per_inner;
  // per-SM per-clock from the cycle count of block 0 (blocks resident at once: 2048 threads / SM)
  double per_sm_clk = (double)(per_sm) * iters * 16 * ops_per_inner / (double)c;
  printf("%-10s %8.3f ms  %8.1f G/s  %6.2f per SM-clk (clk %lld)\n", name, ms, total / ms / 1e6, per_sm_clk, c);
  cudaFree(out); cudaFree(clk);
}

int main() {
  run<0>("ex2", 1, 256);
  run<1>("ffma", 1, 256);
  run<2>("ffma2(x2)", 2, 256);
  run<3>("scanmix/el", 2, 256);
  run<4>("ex2.f16x2(el)", 2, 256);
  run<5>("ex2.bf16x2(el)", 2, 256);
  run<6>("f2fp.bf16x2", 1, 256);
  run<7>("smaxmix/el", 2, 256);
  // few warps per SM sub-partition (the attention softmax runs one or two warps per SMSP per q tile)
  run<0>("ex2 1w/SMSP", 1, 128, 128);
  run<0>("ex2 2w/SMSP", 1, 256, 256);
  run<0>("ex2 4w/SMSP", 1, 512, 512);
  run<7>("smax 1w/SMSP", 2, 128, 128);
  run<7>("smax 2w/SMSP", 2, 256, 256);
  run<7>("smax 4w/SMSP", 2, 512, 512);
  return 0;
}
