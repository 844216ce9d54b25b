// Packed fp32x2 pipe rates on sm_100a: FFMA2 (3 register sources), FMUL2 / FADD2 (2 sources), FFMA2 with a
// negated addend, scalar FFMA; per SM per clock, 2048 threads / SM, 16 independent chains per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma2_rates fma2_rates.cu && ./fma2_rates
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void kern(float* out, int iters) {
  float2 b[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) b[i] = make_float2(threadIdx.x * 1e-6f + i * 1e-3f, -(float)i * 1e-3f);
  // per-thread operands (registers, as in the scan), not immediates or constant-bank operands
  const float2 m = make_float2(0.999f + threadIdx.x * 1e-9f, 0.9991f - threadIdx.x * 1e-9f);
  const float2 c = make_float2(1e-4f * (1 + (threadIdx.x & 3)), 2e-4f * (1 + (threadIdx.x & 7)));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) b[i] = __ffma2_rn(b[i], m, c);
      if (MODE == 1) b[i] = __fmul2_rn(b[i], m);
      if (MODE == 2) b[i] = __fadd2_rn(b[i], c);
      if (MODE == 3) b[i] = __ffma2_rn(b[i], m, make_float2(-c.x, -c.y));
      if (MODE == 4) b[i].x = fmaf(b[i].x, m.x, c.x);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += b[i].x + b[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, double elems) {
  float* out;
  cudaMalloc(&out, 148 * 2048 * 4);
  const int iters = 8192, blocks = 148 * 8;
  kern<MODE><<<blocks, 256>>>(out, 16);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<MODE><<<blocks, 256>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double instr = (double)blocks * 256 * iters * 16 / 32;  // warp instructions
  const double sm_clk = ms * 1e-3 * clk_khz * 1e3 * 148;
  printf("%-18s %8.3f ms  %6.3f warp-instr / SMSP-clk  %7.1f elements / SM-clk (at %d MHz nominal)\n", name, ms,
         instr / sm_clk / 4, instr * 32 * elems / sm_clk, clk_khz / 1000);
  cudaFree(out);
}

int main() {
  run<0>("FFMA2", 2);
  run<1>("FMUL2", 2);
  run<2>("FADD2", 2);
  run<3>("FFMA2 neg addend", 2);
  run<4>("FFMA", 1);
  return 0;
}
