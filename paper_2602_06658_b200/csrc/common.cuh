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

// 2^y to fp64 accuracy (< 2 ulp) on the FP64 pipe, for the plan passes (K4)
// whose outputs are reported in fp64: 0 below 2^-1022, y capped at 64
// (anything above 2^16 only triggers a rebase),
// y = n + r with n = rint(y) by the 1.5 * 2^52 trick (n lands in the low
// mantissa word), |r| <= 1/2, e^(r ln2) by its degree-12 Taylor polynomial
// (truncation < 2e-16), and 2^n written into the exponent field on the ALU.
__device__ __forceinline__ double exp2_f64(double y) {
  const bool under = !(y >= -1022.0);  // (also -inf and NaN: a zero-weight term)
  y = fmin(fmax(y, -1022.0), 64.0);
  const double t = y + 6755399441055744.0;  // 1.5 * 2^52
  const double n = t - 6755399441055744.0;
  const double r = (y - n) * 0.69314718055994530942;
  double p = 2.0876756987868099e-09;  // 1/12!
  p = fma(p, r, 2.5052108385441720e-08);
  p = fma(p, r, 2.7557319223985893e-07);
  p = fma(p, r, 2.7557319223985888e-06);
  p = fma(p, r, 2.4801587301587302e-05);
  p = fma(p, r, 1.9841269841269841e-04);
  p = fma(p, r, 1.3888888888888889e-03);
  p = fma(p, r, 8.3333333333333332e-03);
  p = fma(p, r, 4.1666666666666664e-02);
  p = fma(p, r, 1.6666666666666666e-01);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int e = __double2loint(t) + 1023;  // biased exponent of 2^n, in [1, 1087]
  return under ? 0.0 : p * __hiloint2double(e << 20, 0);
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

// double -> float rounded to nearest on the ALU (|v| < 2^127): add half an
// fp32 ulp to the 29 mantissa bits the truncation drops, then truncate.
__device__ __forceinline__ float f64_to_f32_rn_alu(double v) {
  const long long w = __double_as_longlong(v) + (1LL << 28);
  return f64_to_f32_alu(__longlong_as_double(w));
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

// Signed variant of f32_to_f64_alu (normal v of either sign exact; 0 and
// subnormals -> +-0).
__device__ __forceinline__ double f32_to_f64_alu_s(float v) {
  const uint32_t u = __float_as_uint(v), mag = u & 0x7fffffffu;
  const uint32_t hi = mag >= 0x00800000u ? (mag >> 3) + (896u << 20) : 0u;
  return __hiloint2double((int)(hi | (u & 0x80000000u)), (int)(hi ? mag << 29 : 0u));
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
// three-input minimum (FMNMX3)
__device__ __forceinline__ float fmin3f(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

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

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 2^x for two values on the FMA pipe (FA4-style MUFU offload): x clamped to
// [-125, 64], split x = j + r with |r| <= 1/2 by the 1.5*2^23 rounding trick,
// 2^r by a degree-5 minimax polynomial (max rel. error 2.3e-7 in fp32 Horner,
// on par with MUFU.EX2), and j added to the exponent field with an integer op.
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x.x = fminf(fmaxf(x.x, -125.f), 64.f);
  x.y = fminf(fmaxf(x.y, -125.f), 64.f);
  const float2 t = add2(x, f2(12582912.f, 12582912.f));
  const float2 j = add2(t, f2(-12582912.f, -12582912.f));
  const float2 r = fma2(j, f2(-1.f, -1.f), x);
  float2 p = f2(1.3276470126584172e-3f, 1.3276470126584172e-3f);
  p = fma2(p, r, f2(9.675541892647743e-3f, 9.675541892647743e-3f));
  p = fma2(p, r, f2(5.550713464617729e-2f, 5.550713464617729e-2f));
  p = fma2(p, r, f2(0.24022120237350464f, 0.24022120237350464f));
  p = fma2(p, r, f2(0.6931469440460205f, 0.6931469440460205f));
  p = fma2(p, r, f2(1.0000001192092896f, 1.0000001192092896f));
  return f2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
            __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}

// NS-stage ring of fixed-size column tiles with per-stage full (TMA bytes) and
// empty (one arrival per warp) mbarriers: no block-wide barrier per tile.
// Thread 0 is the producer; it refills the stage of tile t - LAG (with tile
// t - LAG + NS) once every warp has released it, LAG = NS / 2 tiles behind its
// own position, so it rarely waits.
template <int NS>
struct StageRing {
  static constexpr int kLag = NS / 2 > 0 ? NS / 2 : 1;
  uint64_t* full;
  uint64_t* empty;
  __device__ void init(int nwarps) {
    if (threadIdx.x == 0) {
      for (int s = 0; s < NS; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], nwarps);
      }
      fence_mbar_init();
    }
    __syncthreads();
  }
  // thread 0 only: tile t into stage t % NS
  __device__ void load(void* stage, const void* src, uint32_t bytes, int t) {
    mbar_expect_tx(&full[t % NS], bytes);
    bulk_g2s(stage, src, bytes, &full[t % NS]);
  }
  // thread 0 only, before consuming tile t: the tile to refill now, or -1
  __device__ int refill_slot(int t, int ntiles) {
    const int done = t - kLag;  // tile whose stage is recycled
    if (done < 0 || done + NS >= ntiles) return -1;
    mbar_wait(&empty[done % NS], (done / NS) & 1);
    return done + NS;
  }
  __device__ void wait_full(int t) { mbar_wait(&full[t % NS], (t / NS) & 1); }
  __device__ void release(int t) {  // every thread of the warp has finished tile t
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[t % NS]);
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
