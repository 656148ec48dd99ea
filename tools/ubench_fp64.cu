// FP64 pipe throughput on sm_100a: DFMA, DADD, F2F.F32.F64 (cvt.rn.f32.f64),
// and a mixed loop shaped like the fp64-exponent softmin body.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y;
}

template <int MODE>
__global__ void k(float* out, int iters, double seed) {
  double a[8]; float f[8];
  for (int i = 0; i < 8; ++i) { a[i] = seed + threadIdx.x * 1e-3 + i; f[i] = 0.f; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = fma(a[i], 0.999, 0.001);
      if (MODE == 1) { f[i] += __double2float_rn(a[i]); a[i] = a[i] * 0.5 + 1e-3; }
      if (MODE == 2) {  // K=3 body: 3 DFMA + DADD + DFMA + DADD + F2F + EX2 + FADD
        double q = fma(a[i], 1.0001, -3.0);
        q = fma(a[i], 0.9999, q);
        q = fma(a[i], 1.00001, q);
        double u = a[i] - 2.0;
        q = fma(u, u, q);
        double v = 1.0 - q;
        f[i] += ex2(__double2float_rn(v));
        a[i] = a[i] + 1e-9;
      }
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += (float)a[i] + f[i];
  if (s == 1234.5f) out[0] = s;
}

int main() {
  float* d; cudaMalloc(&d, 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000, threads = 512, blocks = sms * 4;
  const char* names[] = {"DFMA", "F2F.F32.F64 (+DFMA+FADD)", "K3 fp64 body (per pair)"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(d, iters, 0.1);
      if (mode == 1) k<1><<<blocks, threads>>>(d, iters, 0.1);
      if (mode == 2) k<2><<<blocks, threads>>>(d, iters, 0.1);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 8;
      if (rep) printf("%-28s %.3e ops/s = %.1f /clk/SM @1.965GHz\n", names[mode], ops / (ms * 1e-3),
                      ops / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  return 0;
}
