// Achievable rate of the fp64 softmin per-pair instruction mix on sm_100a:
// 4 DFMA (K=3 dot + sq term) + 1 DADD (reference) + the 3-op ALU f64->f32
// conversion + MUFU.EX2 + FADD, with many independent pairs per thread, and
// subsets of it, to find which pipe (or dispatch) bounds the mix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_f64mix tools/ubench_f64mix.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float conv(double w) {
  const uint32_t lo = (uint32_t)__double2loint(w);
  const uint32_t hi = (uint32_t)__double2hiint(w);
  const uint32_t f = __funnelshift_l(lo, hi - 0x38000000u, 3);
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xE2;" : "=r"(r) : "r"(f), "n"(0x7fffffff), "r"(hi));
  return __uint_as_float(r);
}

// MODE 0: full pair; 1: no MUFU (sum the converted value); 2: DP only (5 DP);
// 3: no DP (ALU conv + MUFU + FADD on a fixed double); 4: full pair with F2F
template <int MODE, int PAIRS>
__global__ void __launch_bounds__(128) k(float* out, int iters, const double* __restrict__ cin) {
  __shared__ double c[64 * 5];
  for (int i = threadIdx.x; i < 64 * 5; i += blockDim.x) c[i] = cin[i];
  __syncthreads();
  const double x0 = 0.1 + threadIdx.x * 1e-6, x1 = 0.2, x2 = 0.3, s = 0.4;
  double mq = 3.0;
  float acc[PAIRS];
  double xa[PAIRS];  // distinct rows
#pragma unroll
  for (int p = 0; p < PAIRS; ++p) acc[p] = 0.f, xa[p] = x0 + p;
  for (int it = 0; it < iters; ++it) {
    const double* cc = c + (it & 63) * 5;
#pragma unroll
    for (int p = 0; p < PAIRS; ++p) {
      double q = cc[4];
      if (MODE != 3) {
        q = fma(xa[p], cc[0], q);
        q = fma(x1, cc[1], q);
        q = fma(x2, cc[2], q);
        q = fma(s, cc[3], q);
      }
      const double d = mq - q;
      float v = MODE == 4 ? __double2float_rn(d) : (MODE == 2 ? (float)0 : conv(d));
      if (MODE == 2) {
        acc[p] += (float)__double2hiint(d);  // keep d live with one ALU op
      } else {
        acc[p] += (MODE == 1) ? v : ex2(v);
      }
    }
    mq += 1e-12;
  }
  float t = 0.f;
#pragma unroll
  for (int p = 0; p < PAIRS; ++p) t += acc[p];
  if (t == 1234.5f) out[0] = t;
}

// pure DFMA chains, 16 per thread: MODE 5 = three register operands (distinct
// b per chain), MODE 6 = (reg, immediate, reg)
template <int MODE, int PAIRS>
__global__ void __launch_bounds__(128) kf(float* out, int iters, const double* __restrict__ cin) {
  double a[PAIRS], b[PAIRS], acc[PAIRS];
#pragma unroll
  for (int p = 0; p < PAIRS; ++p) {
    a[p] = cin[p] + threadIdx.x * 1e-9;
    b[p] = cin[p + 16];
    acc[p] = 0.0;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int p = 0; p < PAIRS; ++p) acc[p] = fma(a[p], MODE == 5 ? b[p] : 0.999, acc[p]);
  }
  double t = 0.0;
#pragma unroll
  for (int p = 0; p < PAIRS; ++p) t += acc[p];
  if (t == 1234.5) out[0] = (float)t;
}

template <int MODE>
void runf(const char* name, float* d, const double* c, int sms) {
  constexpr int P = 16;
  const int iters = 4000, threads = 128, blocks = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    kf<MODE, P><<<blocks, threads>>>(d, iters, c);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * P;
    if (rep)
      printf("%-34s %.3e DFMA/s = %5.2f /clk/SM @1.965GHz\n", name, ops / (ms * 1e-3),
             ops / (ms * 1e-3) / sms / 1.965e9);
  }
}

// DMMA m8n8k4 (mma.sync f64) throughput: 8 independent accumulators per warp
__global__ void __launch_bounds__(128) kd(float* out, int iters, const double* __restrict__ cin) {
  double a = cin[threadIdx.x & 15], b = cin[(threadIdx.x + 3) & 15];
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1])
                   : "d"(a), "d"(b));
  }
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += c[i][0] + c[i][1];
  if (t == 1234.5) out[0] = (float)t;
}

void rund(float* d, const double* c, int sms) {
  const int iters = 2000, threads = 128, blocks = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    kd<<<blocks, threads>>>(d, iters, c);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // per warp-MMA: 8*8*4 = 256 FMA
    const double fmas = (double)blocks * (threads / 32) * iters * 8 * 256;
    if (rep)
      printf("%-34s %.3e FMA/s = %5.2f /clk/SM @1.965GHz\n", "DMMA m8n8k4", fmas / (ms * 1e-3),
             fmas / (ms * 1e-3) / sms / 1.965e9);
  }
}

// DMMA-based C4 mix: per 8x8 tile one DMMA (C init = column constants), then
// per lane 2 pairs: DADD (row reference), 3-op conversion, EX2, FADD.
// MODE 0 full; 1 no DADD (convert D directly); 2 no conversion (cvt of hi
// word only, 1 ALU); 3 no MUFU; 4 DMMA only (+1 FADD to keep it live)
template <int MODE, int NT>
__global__ void __launch_bounds__(128) km(float* out, int iters, const double* __restrict__ cin) {
  const int lane = threadIdx.x & 31;
  const double a0 = cin[lane & 15] * 1e-3, a1 = cin[(lane + 5) & 15] * 1e-3;
  double b[NT], c0[NT], c1[NT];
#pragma unroll
  for (int u = 0; u < NT; ++u) b[u] = cin[(lane + u) & 15], c0[u] = u, c1[u] = u + 0.5;
  double mq0 = 40.0, mq1 = 41.0;
  float acc0 = 0.f, acc1 = 0.f;
  for (int it = 0; it < iters; ++it) {
    double q[2][NT][2];
#pragma unroll
    for (int u = 0; u < NT; ++u) {
      q[0][u][0] = c0[u]; q[0][u][1] = c1[u];
      q[1][u][0] = c0[u]; q[1][u][1] = c1[u];
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(q[0][u][0]), "+d"(q[0][u][1]) : "d"(a0), "d"(b[u]));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(q[1][u][0]), "+d"(q[1][u][1]) : "d"(a1), "d"(b[u]));
    }
    if (MODE == 5) {  // the row reference as a second k-step: A = [-mq,0,0,0], B = [1,0,0,0]
      const double am0 = (lane & 3) == 0 ? -mq0 : 0.0, am1 = (lane & 3) == 0 ? -mq1 : 0.0;
      const double one = (lane & 3) == 0 ? 1.0 : 0.0;
#pragma unroll
      for (int u = 0; u < NT; ++u) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(q[0][u][0]), "+d"(q[0][u][1]) : "d"(am0), "d"(one));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(q[1][u][0]), "+d"(q[1][u][1]) : "d"(am1), "d"(one));
      }
    }
#pragma unroll
    for (int u = 0; u < NT; ++u) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double d0 = (MODE == 1 || MODE == 5) ? q[0][u][h] : mq0 - q[0][u][h];
        const double d1 = (MODE == 1 || MODE == 5) ? q[1][u][h] : mq1 - q[1][u][h];
        float v0, v1;
        if (MODE == 2) {
          v0 = __int_as_float(__double2hiint(d0));
          v1 = __int_as_float(__double2hiint(d1));
        } else {
          v0 = conv(d0);
          v1 = conv(d1);
        }
        if (MODE == 4) {
          acc0 += (float)__double2hiint(q[0][u][h]);  // keep live (I2F on XU, 1/pair)
        } else if (MODE == 3) {
          acc0 += v0;
          acc1 += v1;
        } else {
          acc0 += ex2(v0);
          acc1 += ex2(v1);
        }
      }
    }
    mq0 += 1e-12;
  }
  if (acc0 + acc1 == 1234.5f) out[0] = acc0;
}

template <int MODE>
void runm(const char* name, float* d, const double* c, int sms) {
  constexpr int NT = 4;
  const int iters = 2000, threads = 128, blocks = sms * 5;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    km<MODE, NT><<<blocks, threads>>>(d, iters, c);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // per warp per iteration: 2 x NT MMAs of 64 pairs
    const double pairs = (double)blocks * (threads / 32) * iters * 2 * NT * 64;
    if (rep)
      printf("%-34s %.3e pairs/s = %5.2f pairs/clk/SM @1.965GHz\n", name, pairs / (ms * 1e-3),
             pairs / (ms * 1e-3) / sms / 1.965e9);
  }
}

// m16n8k8 f64: one MMA per 16x8 tile with K = 8 = [4 features | -mq | 0 0 0],
// C init = column constants; epilogue 4 pairs per lane, no DADD.
template <int NT>
__global__ void __launch_bounds__(128) k168(float* out, int iters, const double* __restrict__ cin) {
  const int lane = threadIdx.x & 31, tig = lane & 3;
  double a[4];
  a[0] = cin[lane & 15] * 1e-3;
  a[1] = cin[(lane + 3) & 15] * 1e-3;
  a[2] = tig == 0 ? -40.0 : 0.0;
  a[3] = tig == 0 ? -41.0 : 0.0;
  double b0[NT], b1 = tig == 0 ? 1.0 : 0.0, c0[NT], c1[NT];
#pragma unroll
  for (int u = 0; u < NT; ++u) b0[u] = cin[(lane + u) & 15], c0[u] = u, c1[u] = u + 0.5;
  float acc0 = 0.f, acc1 = 0.f;
  for (int it = 0; it < iters; ++it) {
    double q[NT][4];
#pragma unroll
    for (int u = 0; u < NT; ++u) {
      q[u][0] = c0[u]; q[u][1] = c1[u]; q[u][2] = c0[u]; q[u][3] = c1[u];
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+d"(q[u][0]), "+d"(q[u][1]), "+d"(q[u][2]), "+d"(q[u][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b0[u]), "d"(b1));
    }
#pragma unroll
    for (int u = 0; u < NT; ++u) {
      acc0 += ex2(-conv(q[u][0])) + ex2(-conv(q[u][1]));
      acc1 += ex2(-conv(q[u][2])) + ex2(-conv(q[u][3]));
    }
    a[2] -= 1e-12;
  }
  if (acc0 + acc1 == 1234.5f) out[0] = acc0;
}

void run168(float* d, const double* c, int sms) {
  constexpr int NT = 4;
  const int iters = 2000, threads = 128, blocks = sms * 5;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k168<NT><<<blocks, threads>>>(d, iters, c);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double pairs = (double)blocks * (threads / 32) * iters * NT * 128;
    if (rep)
      printf("%-34s %.3e pairs/s = %5.2f pairs/clk/SM @1.965GHz\n", "m16n8k8 C4 mix (K=8, no DADD)",
             pairs / (ms * 1e-3), pairs / (ms * 1e-3) / sms / 1.965e9);
  }
}

template <int MODE>
void run(const char* name, float* d, const double* c, int sms) {
  constexpr int P = 16;
  const int iters = 2000, threads = 128, blocks = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k<MODE, P><<<blocks, threads>>>(d, iters, c);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double pairs = (double)blocks * threads * iters * P;
    if (rep)
      printf("%-34s %.3e pairs/s = %5.2f pairs/clk/SM @1.965GHz\n", name, pairs / (ms * 1e-3),
             pairs / (ms * 1e-3) / sms / 1.965e9);
  }
}

int main() {
  float* d;
  double* c;
  cudaMalloc(&d, 16);
  cudaMalloc(&c, 64 * 5 * sizeof(double));
  double h[64 * 5];
  for (int i = 0; i < 64 * 5; ++i) h[i] = 0.01 * (i % 7) - 0.02;
  cudaMemcpy(c, h, sizeof(h), cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("full pair (4 DFMA+DADD+3 ALU+EX2)", d, c, sms);
  run<1>("no MUFU", d, c, sms);
  run<2>("DP only (4 DFMA + DADD)", d, c, sms);
  run<3>("no dot (DADD+ALU+EX2)", d, c, sms);
  run<4>("full pair, F2F conversion", d, c, sms);
  runf<5>("DFMA r,r,r", d, c, sms);
  runf<6>("DFMA r,imm,r", d, c, sms);
  rund(d, c, sms);
  runm<0>("DMMA C4 mix: full", d, c, sms);
  runm<1>("DMMA C4 mix: no DADD", d, c, sms);
  runm<2>("DMMA C4 mix: 1-op conversion", d, c, sms);
  runm<3>("DMMA C4 mix: no MUFU", d, c, sms);
  runm<4>("DMMA C4 mix: DMMA only", d, c, sms);
  runm<5>("DMMA C4 mix: ref as 2nd MMA, no DADD", d, c, sms);
  run168(d, c, sms);
  return 0;
}
