// Shared device helpers for the cntgw_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "cntgw_b200.h"

namespace cntgw {

constexpr double kLog2eD = 1.4426950408889634;
constexpr double kLn2D = 0.6931471805599453;

// Columns per shared-memory stage of the streaming kernels; column buffers
// are padded to a multiple of this so every tile is full.
constexpr int kColTile = 256;

// Finite sentinels of the fp64 path (the ALU double->float conversion below
// is valid for |v| < 2^127): padding columns carry -beta = +kPadQ, and a
// row's reference starts at kStartQ > kPadQ so the first group rebases.
constexpr double kPadQ = 1.0e30;
constexpr double kStartQ = 3.0e30;

// Lazy-rebase trigger: a group of G terms summing above 2^16 (or inf/NaN).
constexpr float kRebase = 65536.0f;

// MUFU.EX2 without range fix-up (flush-to-zero); argument in log2 units.
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// double -> float on the integer ALU pipe (truncating the mantissa), so the
// fp64 path does not spend a second XU-pipe op (F2F shares the pipe with
// MUFU.EX2, measured 16/clk/SM). |v| is clamped below at 2^-126.
__device__ __forceinline__ float f64_to_f32_alu(double v) {
  const uint32_t lo = (uint32_t)__double2loint(v);
  const uint32_t hi = (uint32_t)__double2hiint(v);
  const uint32_t mag = max(hi & 0x7fffffffu, 0x38100000u);
  const uint32_t f = __funnelshift_l(lo, mag - 0x38000000u, 3);
  return __uint_as_float((f & 0x7fffffffu) | (hi & 0x80000000u));
}

// Cheaper conversion for the streaming fp64 softmin (3 ALU ops: IADD, SHF,
// LOP3): the kernel keeps every exponent argument away from zero by carrying
// its row reference kRefOffset log2 units above the row minimum, so the only
// "tiny" argument possible is an exact 0, which this maps to +-2.0 instead of
// 1.0 — an error of < 4 * 2^-kRefOffset relative to the row's largest term.
constexpr double kRefOffset = 32.0;
constexpr float kRebaseF64 = 281474976710656.0f;  // 2^(16 + kRefOffset)
__device__ __forceinline__ float f64_to_f32_fast(double w) {
  const uint32_t lo = (uint32_t)__double2loint(w);
  const uint32_t hi = (uint32_t)__double2hiint(w);
  const uint32_t f = __funnelshift_l(lo, hi - 0x38000000u, 3);
  // (f & 0x7fffffff) | (hi & 0x80000000) as ONE bit-select LOP3 (LUT 0xE2:
  // a&b | c&~b); the compiler otherwise emits two
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xE2;" : "=r"(r) : "r"(f), "n"(0x7fffffff), "r"(hi));
  return __uint_as_float(r);
}

// float -> double with integer ops (exact for normal v >= 0; 0 and subnormals
// -> 0): F2F.F64.F32 would queue on the XU pipe behind the MUFU.EX2 stream
// of the streaming kernels and stall the warp at every tile end.
__device__ __forceinline__ double f32_to_f64_alu(float v) {
  const uint32_t u = __float_as_uint(v);
  const uint32_t hi = u >= 0x00800000u ? (u >> 3) + (896u << 20) : 0u;
  return __hiloint2double((int)hi, (int)(hi ? u << 29 : 0u));
}

// Float-float running sum (hi + lo, ~44-bit significand) on the FMA pipe: the
// epilogue of the tcgen05 kernel folds one fp32 tile sum per row per tile, and
// a DADD there stalls on math-pipe throttle behind the MUFU.EX2 stream.
struct FFSum {
  float hi = 0.f, lo = 0.f;
  __device__ __forceinline__ void add(float t) {  // Knuth TwoSum
    const float s = hi + t;
    const float bp = s - hi;
    lo += (hi - (s - bp)) + (t - bp);
    hi = s;
  }
  __device__ __forceinline__ void scale(float c) {
    hi *= c;
    lo *= c;
  }
  __device__ __forceinline__ double value() const { return (double)hi + (double)lo; }
};

// Packed fp32x2 arithmetic (sm_100a FFMA2/FADD2): two rows per instruction.
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(*reinterpret_cast<uint64_t*>(&d))
      : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)),
        "l"(*reinterpret_cast<const uint64_t*>(&c)));
  return d;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  float2 d;
  asm("add.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<uint64_t*>(&d))
      : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)));
  return d;
}
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// ---- mbarrier + 1-D bulk copy (TMA engine, UBLKCP) ------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// global -> shared bulk copy completing on `bar` (bytes % 16 == 0, 16B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Double-buffered streaming of fixed-size column tiles through shared memory:
// thread 0 issues the bulk copies, every thread waits on the stage barrier.
struct TilePipe {
  uint64_t* bars;
  __device__ void init() {
    if (threadIdx.x == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      fence_mbar_init();
    }
    __syncthreads();
  }
};

// skip modes: 1 = the loop is done; 2 = the loop ended on a symmetrized
// threshold break (its tentatives are already the final ones)
__device__ __forceinline__ bool skip_now(const cntgw_sweep_state* st, int skip) {
  if (!skip || st == nullptr) return false;
  if (skip == 2) return st->converged && st->threshold > 0.0 && st->mode == 1;
  return st->done;
}

__device__ __forceinline__ double block_sum_f64(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  __syncthreads();
  return t;  // valid on thread 0
}

}  // namespace cntgw
