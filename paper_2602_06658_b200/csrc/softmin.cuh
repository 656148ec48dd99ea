// K1/K2: streaming online-log-sum-exp half-update (the Sinkhorn softmin).
//
// Replaces the reference `_softmin` (sinkhorn.py:166-176) evaluated over a
// `SquaredEuclideanCost` (sinkhorn.py:59-109): the N x M cost is rebuilt on
// the fly from per-point features and never materialised.
//
// Work decomposition (both precisions): a CTA of 128 threads owns 128*R rows
// (R rows per thread, kept in registers) and one chunk of columns. Column
// records stream through shared memory in kColTile-column stages filled by the
// TMA bulk-copy engine (cp.async.bulk + mbarrier, double-buffered); every warp
// reads the same record (broadcast LDS.128), so one record load feeds R pairs.
//
// Per pair the kernel evaluates, sign-flipped so every step is a plain FMA,
//     q_ij = -beta_j + sum_k x_ik (-2 lam z_jk) + (sqrt(lam) s_i - sqrt(lam) s_j)^2 = -t_ij
// and accumulates sum_j 2^(mq_i - q_ij) against a lazily updated per-row
// reference mq_i: a group of G terms is summed against the current reference
// and only if that sum leaves [0, 2^16] (or is inf/NaN) is the row rebased at
// the group minimum. Steady state: no per-pair max, one MUFU.EX2 per pair.
//
//  * fp32 path: rows packed in pairs, q assembled with FFMA2/FADD2
//    (KD/2 + 1.5 FP32 instructions per pair).
//  * fp64 path: q assembled with DFMA (KD + 2 fp64 ops per pair: in fp64 the
//    squared coordinate is expanded, (s_i - s_j)^2 -> -2 s_i s_j + s_j^2 with the
//    s_i^2 row constant re-added at the end; B200 runs fp64 at half the fp32
//    rate), the small difference mq - q converted to
//    fp32 on the integer ALU (f64_to_f32_alu) and exponentiated on MUFU. This
//    is the path for cold problems where |t_ij| ~ 1e6-1e7 log2 units (C4/C5):
//    fp32 rounding there is 0.06-1 log2 units per plan entry.
#pragma once

#include "common.cuh"

namespace cntgw {

struct SoftminArgs {
  const cntgw_sweep_state* st;
  int skip;
  const void* row_feat;
  int64_t ld_row;
  const void* row_sq;
  const double* row_add;
  const void* col_rec;
  int64_t n, m;
  int64_t chunk_cols;  // multiple of kColTile
  int nchunks;
  double* out;       // final value (nchunks == 1, no partial output requested)
  double* out_max;   // per-row partial LSE pair (nchunks == 1)
  double* out_sum;
  double* part_max;  // [nchunks][n] split-column partials (nchunks > 1)
  double* part_sum;
  double ctr_limit;  // CNTGW_F32C: per-(group, tile) bound on the fp32 pair term
  const uint32_t* ctr_need;  // CNTGW_F32C: [CTA][tile] needed-tile votes (ctr_plan_kernel) or null
};

template <typename T, int KD, int SQ>
struct ColLayout {
  static constexpr int kRaw = KD + SQ + 1;
  static constexpr int kPerVec = 16 / sizeof(T);                        // elements per 16 B
  // elements; fp64 records also cover the DMMA k4 steps of [features | sq]
  static constexpr int kVec = (kRaw + kPerVec - 1) / kPerVec * kPerVec;
  static constexpr int kK4 = (KD + SQ + 3) / 4 * 4;
  static constexpr int kStride = (sizeof(T) == 8 && kK4 > kVec) ? kK4 : kVec;
  static constexpr int kBeta = KD + SQ;                                    // index of -beta
};

// Shared epilogue: write the partial (max, sum) or the final potential.
__device__ __forceinline__ void softmin_store(const SoftminArgs& a, int chunk, int64_t i, double pmax,
                                              double sum, double inv_lam) {
  if (a.nchunks > 1) {
    a.part_max[(int64_t)chunk * a.n + i] = pmax;
    a.part_sum[(int64_t)chunk * a.n + i] = sum;
  } else if (a.out_max) {
    a.out_max[i] = pmax;
    a.out_sum[i] = sum;
  } else {
    const double add = a.row_add ? a.row_add[i] : 0.0;
    a.out[i] = add - (pmax + log2(sum)) * inv_lam;
  }
}

// ------------------------------------------------------------------------------
// fp32 path
// ------------------------------------------------------------------------------
template <int KD, int SQ, int R, int G, int TILE>
__device__ __forceinline__ void softmin_tile_f32(const float* __restrict__ rec,
                                                 const float2 (&x2)[R / 2][KD],
                                                 const float2 (&s2)[R / 2], float (&mq)[R],
                                                 double (&S)[R]) {
  using L = ColLayout<float, KD, SQ>;
  constexpr int P = R / 2;
  // per-tile fp32 sums (row pairs), folded into the fp64 S once per tile so no
  // F2F.F64 conversion (an XU-pipe op, shared with MUFU.EX2) runs per group
  float2 T[P];
#pragma unroll
  for (int p = 0; p < P; ++p) T[p] = f2(0.f, 0.f);
#pragma unroll 1
  for (int j = 0; j < TILE; j += G) {
    float2 q[P][G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float c[L::kStride];
      const float4* r4 = reinterpret_cast<const float4*>(rec + (j + g) * L::kStride);
#pragma unroll
      for (int v = 0; v < L::kStride / 4; ++v) {
        const float4 t = r4[v];
        c[4 * v + 0] = t.x;
        c[4 * v + 1] = t.y;
        c[4 * v + 2] = t.z;
        c[4 * v + 3] = t.w;
      }
#pragma unroll
      for (int p = 0; p < P; ++p) {
        float2 acc = f2(c[L::kBeta], c[L::kBeta]);
#pragma unroll
        for (int k = 0; k < KD; ++k) acc = fma2(x2[p][k], f2(c[k], c[k]), acc);
        if (SQ) {
          const float2 u = add2(s2[p], f2(c[KD], c[KD]));
          acc = fma2(u, u, acc);
        }
        q[p][g] = acc;
      }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const float2 m2 = f2(mq[2 * p], mq[2 * p + 1]);
      float2 gs = f2(0.f, 0.f);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float2 v = fma2(q[p][g], f2(-1.f, -1.f), m2);
        gs = add2(gs, f2(ex2(v.x), ex2(v.y)));
      }
      if (!(gs.x <= kRebase) || !(gs.y <= kRebase)) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // rare: rebase the row reference at the group minimum
          const int r = 2 * p + h;
          float gsum = h ? gs.y : gs.x;
          if (!(gsum <= kRebase)) {
            float qmin = h ? q[p][0].y : q[p][0].x;
#pragma unroll
            for (int g = 1; g < G; ++g) qmin = fminf(qmin, h ? q[p][g].y : q[p][g].x);
            if (qmin < mq[r]) {
              const float sc = ex2(qmin - mq[r]);
              S[r] *= (double)sc;
              if (h) T[p].y *= sc; else T[p].x *= sc;
              mq[r] = qmin;
            }
            gsum = 0.f;
#pragma unroll
            for (int g = 0; g < G; ++g) gsum += ex2(mq[r] - (h ? q[p][g].y : q[p][g].x));
            if (h) gs.y = gsum; else gs.x = gsum;
          }
        }
      }
      T[p] = add2(T[p], gs);
    }
  }
#pragma unroll
  for (int p = 0; p < P; ++p) {
    S[2 * p] += f32_to_f64_alu(T[p].x);
    if (2 * p + 1 < R) S[2 * p + 1] += f32_to_f64_alu(T[p].y);
  }
}

template <int KD, int SQ, int R, int G, int MINB, int TILE>
__global__ void __launch_bounds__(128, MINB) softmin_f32_kernel(const SoftminArgs a) {
  using L = ColLayout<float, KD, SQ>;
  constexpr int P = R / 2;
  constexpr int kStage = TILE * L::kStride;
  extern __shared__ __align__(128) float smem_f[];
  __shared__ uint64_t bars[2];
  if (skip_now(a.st, a.skip)) return;

  const int chunk = blockIdx.y;
  const int64_t row0 = (int64_t)blockIdx.x * (128 * R) + threadIdx.x;
  const float sl = a.st->sqrt_lam;
  const float* rf = static_cast<const float*>(a.row_feat);
  const float* rs = static_cast<const float*>(a.row_sq);

  float2 x2[P][KD];
  float2 s2[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    float xv[2][KD], sv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t i = row0 + (int64_t)(2 * p + h) * 128;
      const bool ok = i < a.n;
#pragma unroll
      for (int k = 0; k < KD; ++k) xv[h][k] = ok ? rf[i * a.ld_row + k] : 0.f;
      sv[h] = (SQ && ok) ? sl * rs[i] : 0.f;
    }
#pragma unroll
    for (int k = 0; k < KD; ++k) x2[p][k] = f2(xv[0][k], xv[1][k]);
    s2[p] = f2(sv[0], sv[1]);
  }
  float mq[R];
  double S[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    mq[r] = CUDART_INF_F;
    S[r] = 0.0;
  }

  const int64_t c0 = (int64_t)chunk * a.chunk_cols;
  const int64_t mpad = (a.m + kColTile - 1) / kColTile * kColTile;
  const int ntiles = (int)((min(c0 + a.chunk_cols, mpad) - c0) / TILE);
  const uint32_t bytes = kStage * sizeof(float);
  const float* src = static_cast<const float*>(a.col_rec) + c0 * L::kStride;
  TilePipe pipe{bars};
  pipe.init();
  if (threadIdx.x == 0)
    for (int s = 0; s < 2 && s < ntiles; ++s) {
      mbar_expect_tx(&bars[s], bytes);
      bulk_g2s(smem_f + s * kStage, src + (int64_t)s * kStage, bytes, &bars[s]);
    }
  for (int t = 0; t < ntiles; ++t) {
    const int s = t & 1;
    mbar_wait(&bars[s], (t >> 1) & 1);
    softmin_tile_f32<KD, SQ, R, G, TILE>(smem_f + s * kStage, x2, s2, mq, S);
    __syncthreads();  // every warp is done with stage s
    if (threadIdx.x == 0 && t + 2 < ntiles) {
      mbar_expect_tx(&bars[s], bytes);
      bulk_g2s(smem_f + s * kStage, src + (int64_t)(t + 2) * kStage, bytes, &bars[s]);
    }
  }
  const double inv_lam = 1.0 / (double)a.st->lam;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = row0 + (int64_t)r * 128;
    if (i < a.n) softmin_store(a, chunk, i, -(double)mq[r], S[r], inv_lam);
  }
}

// ------------------------------------------------------------------------------
// fp64 path
// ------------------------------------------------------------------------------
template <int KD, int SQ, int R, int G>
__device__ __forceinline__ void f64_scores(const double* __restrict__ rec, const double (&x)[R][KD],
                                           const double (&s)[R], double (&q)[R][G]) {
  using L = ColLayout<double, KD, SQ>;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    double c[L::kStride];
    const double2* r2 = reinterpret_cast<const double2*>(rec + g * L::kStride);
#pragma unroll
    for (int v = 0; v < L::kStride / 2; ++v) {
      const double2 t = r2[v];
      c[2 * v + 0] = t.x;
      c[2 * v + 1] = t.y;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc = c[L::kBeta];
#pragma unroll
      for (int k = 0; k < KD; ++k) acc = fma(x[r][k], c[k], acc);
      if (SQ) acc = fma(s[r], c[KD], acc);  // -2 lam s_i t_j; lam s_i^2 added per row
      q[r][g] = acc;
    }
  }
}

// Group sums 2^(mq - q) for row pairs (FADD2); an odd last row uses .x only.
template <int R, int G>
__device__ __forceinline__ void f64_group_sums(const double (&q)[R][G], const double (&mq)[R],
                                               float2 (&gs)[(R + 1) / 2]) {
#pragma unroll
  for (int p = 0; p < (R + 1) / 2; ++p) {
    const int r1 = 2 * p + 1 < R ? 2 * p + 1 : R - 1;
    gs[p] = f2(0.f, 0.f);
#pragma unroll
    for (int g = 0; g < G; ++g)
      gs[p] = add2(gs[p], f2(ex2(f64_to_f32_fast(mq[2 * p] - q[2 * p][g])),
                             2 * p + 1 < R ? ex2(f64_to_f32_fast(mq[r1] - q[r1][g])) : 0.f));
  }
}

// Rare path: a group sum left [0, kRebaseF64] (or is inf/NaN) -> rebase the
// row reference kRefOffset above the group minimum and redo that row's sum.
template <int R, int G>
__device__ __forceinline__ void f64_fold(const double (&q)[R][G], double (&mq)[R], double (&S)[R],
                                         float2 (&gs)[(R + 1) / 2], float2 (&T)[(R + 1) / 2]) {
#pragma unroll
  for (int p = 0; p < (R + 1) / 2; ++p) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = 2 * p + h;
      if (r >= R) break;
      float& gsum = h ? gs[p].y : gs[p].x;
      float& tr = h ? T[p].y : T[p].x;
      if (!(gsum <= kRebaseF64)) {
        double qmin = q[r][0];
#pragma unroll
        for (int g = 1; g < G; ++g) qmin = fmin(qmin, q[r][g]);
        const double ref = qmin + kRefOffset;
        if (ref < mq[r]) {
          const double sc = exp2(ref - mq[r]);
          S[r] *= sc;
          tr *= (float)sc;
          mq[r] = ref;
        }
        gsum = 0.f;
#pragma unroll
        for (int g = 0; g < G; ++g) gsum += ex2(f64_to_f32_fast(mq[r] - q[r][g]));
      }
    }
    T[p] = add2(T[p], gs[p]);
  }
}

// One shared-memory tile of the fp64 path: per group of G columns, R x G
// DFMA score chains, then the ALU conversion + MUFU.EX2 + FADD2 sums and the
// (rare) rebase. Software-pipelining the next group's DFMA chains into the
// current group's exponentials measured no faster: the per-pair mix (4 DFMA +
// DADD + 3 ALU + EX2 + FADD) runs at the ceiling tools/ubench_f64mix measures
// for it in isolation (~6.2 pairs/clk/SM).
template <int KD, int SQ, int R, int G, int TILE>
__device__ __forceinline__ void softmin_tile_f64(const double* __restrict__ rec,
                                                 const double (&x)[R][KD], const double (&s)[R],
                                                 double (&mq)[R], double (&S)[R]) {
  using L = ColLayout<double, KD, SQ>;
  constexpr int P = (R + 1) / 2;
  float2 T[P];  // per-tile fp32 sums of row pairs, folded into S once per tile
#pragma unroll
  for (int p = 0; p < P; ++p) T[p] = f2(0.f, 0.f);
#pragma unroll 1
  for (int j = 0; j < TILE; j += G) {
    double q[R][G];
    float2 gs[P];
    f64_scores<KD, SQ, R, G>(rec + j * L::kStride, x, s, q);
    f64_group_sums<R, G>(q, mq, gs);
    f64_fold<R, G>(q, mq, S, gs, T);
  }
#pragma unroll
  for (int p = 0; p < P; ++p) {
    S[2 * p] += f32_to_f64_alu(T[p].x);
    if (2 * p + 1 < R) S[2 * p + 1] += f32_to_f64_alu(T[p].y);
  }
}

template <int KD, int SQ, int R, int G, int MINB, int TILE>
__global__ void __launch_bounds__(128, MINB) softmin_f64_kernel(const SoftminArgs a) {
  using L = ColLayout<double, KD, SQ>;
  constexpr int kStage = TILE * L::kStride;
  extern __shared__ __align__(128) double smem_d[];
  __shared__ uint64_t bars[2];
  if (skip_now(a.st, a.skip)) return;

  const int chunk = blockIdx.y;
  const int64_t row0 = (int64_t)blockIdx.x * (128 * R) + threadIdx.x;
  const double* rf = static_cast<const double*>(a.row_feat);
  const double* rs = static_cast<const double*>(a.row_sq);
  double x[R][KD], s[R], mq[R], S[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = row0 + (int64_t)r * 128;
    const bool ok = i < a.n;
#pragma unroll
    for (int k = 0; k < KD; ++k) x[r][k] = ok ? rf[i * a.ld_row + k] : 0.0;
    s[r] = (SQ && ok) ? rs[i] : 0.0;
    mq[r] = kStartQ;
    S[r] = 0.0;
  }

  const int64_t c0 = (int64_t)chunk * a.chunk_cols;
  const int64_t mpad = (a.m + kColTile - 1) / kColTile * kColTile;
  const int ntiles = (int)((min(c0 + a.chunk_cols, mpad) - c0) / TILE);
  const uint32_t bytes = kStage * sizeof(double);
  const double* src = static_cast<const double*>(a.col_rec) + c0 * L::kStride;
  TilePipe pipe{bars};
  pipe.init();
  if (threadIdx.x == 0)
    for (int st = 0; st < 2 && st < ntiles; ++st) {
      mbar_expect_tx(&bars[st], bytes);
      bulk_g2s(smem_d + st * kStage, src + (int64_t)st * kStage, bytes, &bars[st]);
    }
  for (int t = 0; t < ntiles; ++t) {
    const int sb = t & 1;
    mbar_wait(&bars[sb], (t >> 1) & 1);
    softmin_tile_f64<KD, SQ, R, G, TILE>(smem_d + sb * kStage, x, s, mq, S);
    __syncthreads();
    if (threadIdx.x == 0 && t + 2 < ntiles) {
      mbar_expect_tx(&bars[sb], bytes);
      bulk_g2s(smem_d + sb * kStage, src + (int64_t)(t + 2) * kStage, bytes, &bars[sb]);
    }
  }
  const double lam = a.st->lam_d, inv_lam = 1.0 / lam;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = row0 + (int64_t)r * 128;
    // q accumulated without the row constant lam s_i^2 (expanded square)
    if (i < a.n) softmin_store(a, chunk, i, -mq[r] - (SQ ? lam * s[r] * s[r] : 0.0), S[r], inv_lam);
  }
}

// Fixed-order merge of the split-column partials of each row (also the
// finaliser of a cross-GPU partial LSE when nchunks == 1).
static __global__ void lse_combine_kernel(const cntgw_sweep_state* st, int skip, int prec,
                                          const double* pm, const double* ps, int nchunks,
                                          int64_t n, const double* row_add, double* out,
                                          double* out_max, double* out_sum) {
  if (skip_now(st, skip)) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double mx = -CUDART_INF;
  for (int c = 0; c < nchunks; ++c) mx = fmax(mx, pm[(int64_t)c * n + i]);
  double sm = 0.0;
  for (int c = 0; c < nchunks; ++c) {
    const double v = ps[(int64_t)c * n + i];
    if (v > 0.0) sm += v * exp2(pm[(int64_t)c * n + i] - mx);
  }
  if (out_max) {
    out_max[i] = mx;
    out_sum[i] = sm;
  } else {
    const double inv_lam =
        (prec == CNTGW_F64 || prec == CNTGW_F32C || prec == CNTGW_F64S) ? 1.0 / st->lam_d
                                                                         : 1.0 / (double)st->lam;
    out[i] = (row_add ? row_add[i] : 0.0) - (mx + log2(sm)) * inv_lam;
  }
}

}  // namespace cntgw
