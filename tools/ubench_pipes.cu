// Pipe-throughput microbenchmark for the softmin inner loop on sm_100a:
// FFMA (scalar), FFMA2 (fma.rn.f32x2), MUFU.EX2 (ex2.approx.ftz.f32), and a
// mixed loop shaped like the K=4 softmin body. Prints ops/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(*(uint64_t*)&d)
               : "l"(*(uint64_t*)&a), "l"(*(uint64_t*)&b), "l"(*(uint64_t*)&c));
  return d;
}
__device__ __forceinline__ float ex2(float x) {
  float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y;
}

template <int MODE>
__global__ void k(float* out, int iters, float seed) {
  float a[8]; float2 b[8];
  for (int i = 0; i < 8; ++i) { a[i] = seed + threadIdx.x * 1e-3f + i; b[i] = make_float2(a[i], a[i] + 1); }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) { a[i] = fmaf(a[i], 0.999f, 0.001f); }
      if (MODE == 1) { b[i] = ffma2(b[i], make_float2(0.999f, 0.999f), make_float2(0.001f, 0.002f)); }
      if (MODE == 2) { a[i] = ex2(a[i]) * -0.5f; }
      if (MODE == 3) { a[i] = ex2(a[i]); }
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + b[i].x + b[i].y;
  if (s == 1234.5f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
}

int main() {
  float* d; cudaMalloc(&d, 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000, threads = 512, blocks = sms * 4;
  const char* names[] = {"FFMA", "FFMA2(f32x2, counted as 2 FMA)", "EX2+FMUL", "EX2"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(d, iters, 0.1f);
      if (mode == 1) k<1><<<blocks, threads>>>(d, iters, 0.1f);
      if (mode == 2) k<2><<<blocks, threads>>>(d, iters, 0.1f);
      if (mode == 3) k<3><<<blocks, threads>>>(d, iters, 0.1f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      float cyc; cudaMemcpy(&cyc, d + 1, 4, cudaMemcpyDeviceToHost);
      double ops = (double)blocks * threads * iters * 8 * (mode == 1 ? 2 : 1);
      double per_s = ops / (ms * 1e-3);
      // ops/clk/SM from the in-kernel clock of block 0 (4 blocks per SM co-resident)
      double per_clk_sm = (double)threads * 4 * iters * 8 * (mode == 1 ? 2 : 1) / cyc;
      if (rep) printf("%-32s %.3e ops/s  %.1f ops/clk/SM (clock-based)  eff_clk=%.0f MHz\n", names[mode], per_s,
                      per_clk_sm, per_s / per_clk_sm / sms / 1e6);
    }
  }
  printf("SMs=%d clockRate=%d kHz\n", sms, clk);
  return 0;
}
