// K1/K2 on the 5th-generation tensor cores: the half-update for well-scaled
// problems with K >= 8 dot features (the C2 micro-benchmark shape).
//
// t_ij = beta_j + sum_k x_ik (2 lam z_jk) is a GEMM-shaped score, evaluated as
// a split-precision tcgen05 MMA so that it keeps ~fp32 accuracy: with hi =
// tf32 rounding and lo = tf32(x - hi),
//     A'_i . B'_j = hi.hi + hi.lo + lo.hi  (+ the bias, split exactly).
// Two operand formats (CNTGW_TC_KIND):
//   * fp16 (default, TcLayoutH below): the 11-bit parts scaled into fp16's
//     range, kind::f16 at K = 16 per instruction: 4 MMAs and 32 KB of B' per
//     256 columns at KD = 16;
//   * tf32 (TcLayout): A'_i = [hi(x_i), 1 | hi(x_i), 1 | lo(x_i), 0],
//     B'_j = [hi(zt_j), hi(b_j) | lo(zt_j), lo(b_j) | hi(zt_j), 0], K' = 3 KD + 2
//     padded to 8, kind::tf32 at K = 8: 7 MMAs and 56 KB.
// The accumulator lives in TMEM (128 lanes = rows x 256 fp32 columns,
// double-buffered = all 512 TMEM columns), so the FMA pipe does only the
// online log-sum-exp epilogue: tcgen05.ld -> subtract the lazily rebased row
// reference (one FADD2, or one FFMA2 that also undoes the fp16 scaling) ->
// MUFU.EX2 (a few per chunk as an FMA-pipe polynomial) -> sum.
//
// Warp roles (one CTA per SM, 128 rows x one column chunk):
//   warp 0      TMA producer: 1-D bulk copies of prepacked B' tiles into a
//               kTcStages-deep shared-memory ring (mbarrier full/empty); three
//               stages keep two tiles of L2/DRAM latency in flight ahead of
//               the MMA (column chunks of 48 MB keep a chunk's tiles in L2)
//   warp 1      TMEM allocator + MMA issuer: one elected lane issues
//               tcgen05.mma (M=128, N=256) and tcgen05.commit to release the
//               smem stage and publish the tile
//   warps 2..   EPI epilogue warps: warp w reads TMEM lane quadrant w%4 (32
//               rows) and column part (w-2)/4 of each tile (32x32b.x32 loads,
//               the next chunk's load in flight while the current is consumed)
// Operands use the canonical K-major no-swizzle layout: 8-row x 16-byte core
// matrices, SBO = 128 B between 8-row groups, LBO = rows*16 B between the two
// 16-byte K chunks of one MMA step.
#pragma once

#include <cuda_fp16.h>

#include <type_traits>

#include "common.cuh"
#include "softmin.cuh"

namespace cntgw {

constexpr int kTcRows = 128;   // rows per CTA (= TMEM lanes)
constexpr int kTcCols = 256;   // columns per tile (= MMA N)
constexpr int kTcStages = 3;   // B' shared-memory ring depth
// producer + MMA warps + EPI epilogue warps (EPI/4 per TMEM lane quadrant)
constexpr int tc_threads(int epi) { return 64 + 32 * epi; }

template <int KD>
struct TcLayout {
  static constexpr int kKp = (3 * KD + 2 + 7) / 8 * 8;  // K' padded to the MMA K step
  static constexpr int kChunks = kKp / 4;                // 16-byte K chunks
  static constexpr int kBTileFloats = kChunks * kTcCols * 4;
  static constexpr int kATileFloats = kChunks * kTcRows * 4;
  // K' positions of the three blocks
  static constexpr int kHi = 0, kLo = KD + 1, kHi2 = 2 * KD + 2;
  static constexpr int kATileBytes = kATileFloats * 4, kBTileBytes = kBTileFloats * 4;
  static constexpr int kMmas = kKp / 8;                  // K = 8 per tf32 instruction
  static constexpr int kRecBytes = kKp * 4;              // per column
};

// The same split on fp16 operands (kind::f16, K = 16 per instruction at twice
// the tf32 rate and half the operand bytes). The tf32 parts hi = tf32(x) and
// lo = tf32(x - hi) carry 11 significant bits, exactly what fp16 holds, so
// once both sides are scaled into fp16's exponent range the products are the
// ones the tf32 MMA forms. Scaling: with 2^eb > max_jk |zt_jk| (an absmax
// pass over the column features, tc_absmax_kernel) the column side is stored
// as zt * 2^(14 - eb) (|.| < 2^14) and the row side as x * 2^(eb + 1)
// (|.| < 4 max|x| max|zt| < 2^14 on this path, whose exponent scale is < 4096);
// the accumulator then holds t * 2^15 and the epilogue's reference
// subtraction becomes one FFMA2, x = v * 2^-15 - mref. A value too small for
// fp16's normal range is off by at most 2^-25 before the 2^14 * 2^-15 of its
// partner and the rescale, i.e. 2^-26 per product in t. The bias is split in
// three fp16 parts against 2^15 on the row side.
//     A'_i = [hi(x_i) | lo(x_i) | hi(x_i)] * 2^(eb+1) | 2^15 2^15 2^15
//     B'_j = [hi(zt_j) | hi(zt_j) | lo(zt_j)] * 2^(14-eb) | b_hi b_mid b_lo
template <int KD>
struct TcLayoutH {
  static constexpr int kKp = (3 * KD + 3 + 15) / 16 * 16;  // halfs, padded to the MMA K step
  static constexpr int kChunks = kKp / 8;                   // 16-byte K chunks
  static constexpr int kATileBytes = kChunks * kTcRows * 16, kBTileBytes = kChunks * kTcCols * 16;
  static constexpr int kMmas = kKp / 16;
  static constexpr int kRecBytes = kKp * 2;
  static constexpr int kHH = 0, kLH = KD, kHL = 2 * KD, kBias = 3 * KD;
};
constexpr float kTcHScale = 0x1p-15f;  // accumulator -> log2 units
constexpr float kTcHPadBias = -60000.f;

// 2^eb > max |2 lam z| from the absmax word (float bits of max |z|)
__device__ __forceinline__ int tch_col_exp(uint32_t maxbits, float two_lam) {
  const float mz = fabsf(two_lam) * __uint_as_float(maxbits);
  if (!(mz > 0.f) || !(mz < CUDART_INF_F)) return 0;
  return ilogbf(mz) + 1;
}
__device__ __forceinline__ float pow2i(int k) {
  k = k < -126 ? -126 : (k > 127 ? 127 : k);
  return __int_as_float((127 + k) << 23);
}
// ... for a scale that must be exact: NaN (loud) when 2^k is not a normal fp32
__device__ __forceinline__ float pow2i_exact(int k) {
  return (k < -126 || k > 127) ? __int_as_float(0x7fc00000) : __int_as_float((127 + k) << 23);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// -- tcgen05 wrappers ----------------------------------------------------------
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  // base_offset 0, lbo_mode 0, layout_type 0 = SWIZZLE_NONE (K-major interleave)
  return d;
}

// kind::tf32, fp32 accumulate, A/B K-major, M=128, N=256
constexpr uint32_t kTcIdesc = (1u << 4)            // c_format F32
                              | (2u << 7)          // a_format TF32
                              | (2u << 10)         // b_format TF32
                              | ((uint32_t)(kTcCols >> 3) << 17)
                              | ((uint32_t)(kTcRows >> 4) << 24);

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kTcIdesc), "r"(acc));
}
// kind::f16 (fp16 A/B = format 0), fp32 accumulate, K-major, M=128, N=256
constexpr uint32_t kTcIdescH = (1u << 4) | ((uint32_t)(kTcCols >> 3) << 17) | ((uint32_t)(kTcRows >> 4) << 24);
__device__ __forceinline__ void tc_mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kTcIdescH), "r"(acc));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t* u = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
        "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
        "=r"(u[14]), "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]),
        "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]),
        "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Pack the column side in the B' tile layout [tile][chunk][256 cols][4 floats].
template <int KD>
__global__ void prep_cols_tc_kernel(const cntgw_sweep_state* st, const float* feat, int64_t ld,
                                    const double* pot, const double* log2w, int64_t m,
                                    int64_t mpad, float* rec) {
  using L = TcLayout<KD>;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= mpad) return;
  const int64_t tile = j / kTcCols;
  const int col = (int)(j % kTcCols);
  float* base = rec + tile * L::kBTileFloats + col * 4;
  auto put = [&](int p, float v) { base[(p >> 2) * (kTcCols * 4) + (p & 3)] = v; };
  for (int p = 0; p < L::kKp; ++p) put(p, 0.f);
  if (j < m) {
    const double lam = (double)st->lam;
    const float two_lam = (float)(2.0 * lam);
    for (int k = 0; k < KD; ++k) {
      const float z = two_lam * feat[j * ld + k];
      const float zh = tf32_rna(z);
      const float zl = tf32_rna(z - zh);
      put(L::kHi + k, zh);
      put(L::kLo + k, zl);
      put(L::kHi2 + k, zh);
    }
    const float beta = (float)(lam * (pot ? pot[j] : 0.0) + log2w[j]);
    const float bh = tf32_rna(beta);
    put(L::kHi + KD, bh);
    put(L::kLo + KD, tf32_rna(beta - bh));
  } else {
    put(L::kHi + KD, -1.0e30f);  // padding column: 2^(t - max) == 0
  }
}

// fp16 operands: absmax of the column features (float bits, >= 0, so the
// unsigned order is the float order), then the pack. The absmax word sits
// right after the records (byte mpad * kRecBytes), outside the MMA's reads.
__global__ void tc_absmax_kernel(const float* feat, int64_t ld, int kd, int64_t m, uint32_t* out) {
  float mx = 0.f;
  const int64_t total = m * kd;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x)
    mx = fmaxf(mx, fabsf(feat[(idx / kd) * ld + idx % kd]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx > 0.f) atomicMax(out, __float_as_uint(mx));
}

template <int KD>
__global__ void prep_cols_tch_kernel(const cntgw_sweep_state* st, const float* feat, int64_t ld,
                                     const double* pot, const double* log2w, int64_t m, int64_t mpad,
                                     __half* rec, const uint32_t* absmax) {
  using L = TcLayoutH<KD>;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= mpad) return;
  const int64_t tile = j / kTcCols;
  const int col = (int)(j % kTcCols);
  __half* base = rec + tile * (L::kBTileBytes / 2) + col * 8;
  auto put = [&](int p, float v) { base[(p >> 3) * (kTcCols * 8) + (p & 7)] = __float2half_rn(v); };
  for (int p = 0; p < L::kKp; ++p) put(p, 0.f);
  if (j < m) {
    const double lam = (double)st->lam;
    const float two_lam = (float)(2.0 * lam);
    const float sb = pow2i_exact(14 - tch_col_exp(*absmax, two_lam));
    for (int k = 0; k < KD; ++k) {
      const float z = two_lam * feat[j * ld + k];
      const float zh = tf32_rna(z);
      const float zl = tf32_rna(z - zh);
      put(L::kHH + k, zh * sb);
      put(L::kLH + k, zh * sb);
      put(L::kHL + k, zl * sb);
    }
    // (zero-weight columns: log2 w = -inf, kept finite so the parts stay exact)
    float beta = (float)(lam * (pot ? pot[j] : 0.0) + log2w[j]);
    if (beta < kTcHPadBias) beta = kTcHPadBias;  // (a NaN stays a NaN)
    const float b1 = __half2float(__float2half_rn(beta));
    const float b2 = __half2float(__float2half_rn(beta - b1));
    put(L::kBias, b1);
    put(L::kBias + 1, b2);
    put(L::kBias + 2, beta - b1 - b2);
  } else {
    put(L::kBias, kTcHPadBias);  // padding column: 2^(t - max) == 0
  }
}

// One 32-column chunk of the epilogue: terms 2^(v - mref) summed with FADD2
// pairs into four independent accumulators, NPOLY of the 16 pairs exponentiated
// on the FMA pipe and the rest on MUFU.EX2; a chunk whose sum leaves [0, 2^20]
// (or is inf/NaN) rebases the row reference at the chunk maximum.
template <int NPOLY, bool SCALED = false>
__device__ __forceinline__ void tc_chunk(const float (&v)[32], float& mref, float& tsum, FFSum& S) {
  // SCALED: the accumulator holds t * 2^15 (fp16 operands); the rescale rides
  // on the reference subtraction as one FFMA2
  const float2 sc2 = f2(kTcHScale, kTcHScale);
  auto arg = [&](int u, float2 nm) {
    const float2 t = f2(v[2 * u], v[2 * u + 1]);
    return SCALED ? fma2(t, sc2, nm) : add2(t, nm);
  };
  float2 nm = f2(-mref, -mref);
  float2 acc[4];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const float2 x = arg(u, nm);
    // offloaded pairs spread over the four accumulators
    constexpr uint32_t kMask = NPOLY == 2   ? 0x0201u
                               : NPOLY == 3 ? 0x0421u
                               : NPOLY == 4 ? 0x8421u
                               : NPOLY == 6 ? 0x9249u
                               : NPOLY == 8 ? 0x5555u
                                            : 0u;
    const bool poly = (kMask >> u) & 1u;
    const float2 e = poly ? exp2_poly2(x) : f2(ex2(x.x), ex2(x.y));
    acc[u & 3] = u < 4 ? e : add2(acc[u & 3], e);
  }
  float2 t2 = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
  float csum = t2.x + t2.y;
  if (!(csum <= 1048576.0f)) {
    float cm = v[0];
#pragma unroll
    for (int u = 1; u < 32; ++u) cm = fmaxf(cm, v[u]);
    if (SCALED) cm *= kTcHScale;
    if (cm > mref) {
      const float sc = ex2(mref - cm);
      S.scale(sc);
      tsum *= sc;
      mref = cm;
    }
    nm = f2(-mref, -mref);
    float2 r = f2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const float2 x = arg(u, nm);
      r = add2(r, f2(ex2(x.x), ex2(x.y)));
    }
    csum = r.x + r.y;
  }
  tsum += csum;
}

template <int KD, int NPOLY, int EPI, bool H = false>
__global__ void __launch_bounds__(tc_threads(EPI), 1) softmin_tc_kernel(const SoftminArgs a) {
  using L = std::conditional_t<H, TcLayoutH<KD>, TcLayout<KD>>;
  extern __shared__ __align__(1024) char smem_tc[];
  __shared__ uint64_t full_bar[kTcStages], empty_bar[kTcStages], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  constexpr int kParts = EPI / 4;                  // column parts per TMEM quadrant
  constexpr int kChunksPerPart = kTcCols / kParts / 32;
  __shared__ float red_m[kParts][kTcRows];
  __shared__ double red_s[kParts][kTcRows];
  if (skip_now(a.st, a.skip)) return;

  char* sA = smem_tc;                      // A' : kChunks x 128 rows x 16 B
  char* sB = smem_tc + L::kATileBytes;     // B' : kTcStages stages
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunk = blockIdx.y;
  const int64_t row0 = (int64_t)blockIdx.x * kTcRows;
  const int64_t c0 = (int64_t)chunk * a.chunk_cols;
  const int64_t mpad = (a.m + kColTile - 1) / kColTile * kColTile;
  const int ntiles = (int)((min(c0 + a.chunk_cols, mpad) - c0) / kTcCols);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], EPI);
    }
    fence_mbar_init();
  }
  if (warp == 1) {  // TMEM: two 128 x 256 fp32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // A' rows (epilogue warps): hi/lo split of this CTA's row features
  if (warp >= 2) {
    const int t = threadIdx.x - 64;
    const int r = t & (kTcRows - 1), h = t >> 7;
    const int64_t i = row0 + r;
    const float* xf = static_cast<const float*>(a.row_feat);
    if constexpr (H) {
      __half* hA = reinterpret_cast<__half*>(sA);
      auto put = [&](int p, float v) { hA[(p >> 3) * (kTcRows * 8) + r * 8 + (p & 7)] = __float2half_rn(v); };
      const uint32_t absmax = *reinterpret_cast<const uint32_t*>(static_cast<const char*>(a.col_rec) +
                                                                 mpad * L::kRecBytes);
      const float sa = pow2i_exact(tch_col_exp(absmax, (float)(2.0 * (double)a.st->lam)) + 1);
      for (int k = h * (KD / kParts); k < (h + 1) * (KD / kParts); ++k) {
        const float x = i < a.n ? xf[i * a.ld_row + k] : 0.f;
        const float xh = tf32_rna(x);
        put(L::kHH + k, xh * sa);
        put(L::kLH + k, tf32_rna(x - xh) * sa);
        put(L::kHL + k, xh * sa);
      }
      if (h == 0) {
        for (int p = 0; p < 3; ++p) put(L::kBias + p, 32768.f);
        for (int p = L::kBias + 3; p < L::kKp; ++p) put(p, 0.f);
      }
    } else {
      float* fA = reinterpret_cast<float*>(sA);
      auto put = [&](int p, float v) { fA[(p >> 2) * (kTcRows * 4) + r * 4 + (p & 3)] = v; };
      for (int k = h * (KD / kParts); k < (h + 1) * (KD / kParts); ++k) {
        const float x = i < a.n ? xf[i * a.ld_row + k] : 0.f;
        const float xh = tf32_rna(x);
        put(L::kHi + k, xh);
        put(L::kLo + k, xh);
        put(L::kHi2 + k, tf32_rna(x - xh));
      }
      if (h == 0) {
        put(L::kHi + KD, 1.f);
        put(L::kLo + KD, 1.f);
        for (int p = L::kHi2 + KD; p < L::kKp; ++p) put(p, 0.f);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic -> tensor-core proxy
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {  // producer
      const uint32_t bytes = L::kBTileBytes;
      const char* src = static_cast<const char*>(a.col_rec) + (c0 / kTcCols) * L::kBTileBytes;
      for (int t = 0, s = 0, ph = 0; t < ntiles; ++t) {
        mbar_wait(&empty_bar[s], ph ^ 1);
        mbar_expect_tx(&full_bar[s], bytes);
        bulk_g2s(sB + s * L::kBTileBytes, src + (int64_t)t * L::kBTileBytes, bytes, &full_bar[s]);
        if (++s == kTcStages) s = 0, ph ^= 1;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      const uint32_t a0 = smem_u32(sA);
      for (int t = 0, s = 0, ph = 0; t < ntiles; ++t) {
        const int ab = t & 1;  // TMEM accumulator buffer
        mbar_wait(&full_bar[s], ph);
        mbar_wait(&tempty_bar[ab], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t b0 = smem_u32(sB + s * L::kBTileBytes);
        const uint32_t d = tmem + (uint32_t)(ab * kTcCols);
#pragma unroll
        for (int ks = 0; ks < L::kMmas; ++ks) {  // two 16-byte K chunks per instruction
          const uint64_t ad = umma_desc(a0 + ks * 2 * (kTcRows * 16), kTcRows * 16, 128);
          const uint64_t bd = umma_desc(b0 + ks * 2 * (kTcCols * 16), kTcCols * 16, 128);
          if constexpr (H) tc_mma_f16(d, ad, bd, ks > 0 ? 1u : 0u);
          else tc_mma(d, ad, bd, ks > 0 ? 1u : 0u);
        }
        tc_commit(&empty_bar[s]);   // smem stage reusable once these MMAs completed
        tc_commit(&tfull_bar[ab]);  // accumulator ab ready for the epilogue
        if (++s == kTcStages) s = 0, ph ^= 1;
      }
    }
  } else {  // epilogue warps
    const int q = warp & 3;             // TMEM lane quadrant (rows 32q..32q+31)
    const int part = (warp - 2) >> 2;   // column part of each tile
    float mref = -CUDART_INF_F;         // lazily rebased row reference (log2 units)
    FFSum S;                                    // sum over finished tiles of 2^(t - mref)
    float va[32], vb[32];
    for (int t = 0; t < ntiles; ++t) {
      const int s = t & 1;
      mbar_wait(&tfull_bar[s], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) +
                             (uint32_t)(s * kTcCols + part * (kTcCols / kParts));
      float tsum = 0.f;  // this tile's sum against mref (fp32; folded into S per tile)
      tmem_ld32(taddr, va);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < kChunksPerPart; ++c) {
        float(&cur)[32] = (c & 1) ? vb : va;
        float(&nxt)[32] = (c & 1) ? va : vb;
        if (c + 1 < kChunksPerPart) {
          tmem_ld32(taddr + 32 * (c + 1), nxt);  // overlaps this chunk's math
        } else {
          tc_fence_before();  // every TMEM load of this tile has completed
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[s]);  // accumulator s may be overwritten
        }
        tc_chunk<NPOLY, H>(cur, mref, tsum, S);
        if (c + 1 < kChunksPerPart) tmem_wait_ld();
      }
      S.add(tsum);
    }
    // merge the column parts of each row, then store
    const int r = 32 * q + lane;
    red_m[part][r] = mref;
    red_s[part][r] = S.value();
    asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI) : "memory");  // epilogue warps only
    if (part == 0) {
      float mm = red_m[0][r];
#pragma unroll
      for (int p = 1; p < kParts; ++p) mm = fmaxf(mm, red_m[p][r]);
      double tot = 0.0;
#pragma unroll
      for (int p = 0; p < kParts; ++p)
        if (red_s[p][r] > 0.0) tot += red_s[p][r] * exp2((double)(red_m[p][r] - mm));
      const int64_t i = row0 + r;
      if (i < a.n) softmin_store(a, chunk, i, (double)mm, tot, 1.0 / (double)a.st->lam);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace cntgw
