// K1/K2: streaming online-log-sum-exp half-update on the FP32/FMA + MUFU pipes.
//
// Replaces the reference `_softmin` (sinkhorn.py:166-176) evaluated over a
// `SquaredEuclideanCost` (sinkhorn.py:59-109): the N x M cost is rebuilt on
// the fly from per-point features and never materialised.
//
// Work decomposition: a CTA of 128 threads owns 128*R rows (R rows per
// thread, packed in pairs for fma.rn.f32x2) and one chunk of columns. Column
// records stream through shared memory in kColTile-column stages filled by the
// TMA engine (cp.async.bulk + mbarrier, double-buffered). Every warp reads the
// same record (broadcast LDS.128), so one record load feeds R pairs.
//
// Per pair the kernel evaluates, in log2 units and with the sign flipped so
// that every step is a plain FMA,
//     q_ij = -beta_j + sum_k x_ik (-2 lam z_jk) + (sqrt(lam) s_i - sqrt(lam) s_j)^2
//          = -t_ij
// and accumulates sum_j 2^(mq_i - q_ij) against a lazily updated reference
// mq_i (rebased only when a group of G terms sums above 2^16, or on inf/NaN),
// so the steady state costs KD/2 FFMA2 + FADD2 + FFMA2 + FFMA2 + MUFU.EX2 +
// FADD2 per two pairs: 1 MUFU per pair and no per-pair max.
#pragma once

#include "common.cuh"

namespace cntgw {

struct SoftminArgs {
  const cntgw_sweep_state* st;
  int skip;
  const float* row_feat;
  int64_t ld_row;
  const float* row_sq;
  const float* row_add;
  const float* col_rec;
  int64_t n, m;
  int64_t chunk_cols;  // multiple of kColTile
  int nchunks;
  float* out;       // final (nchunks == 1 and no partial output requested)
  float* out_max;   // per-row partial LSE pair (nchunks == 1)
  float* out_sum;
  float* part_max;  // [nchunks][n] split-column partials (nchunks > 1)
  float* part_sum;
};

template <int KD, int SQ>
struct ColLayout {
  static constexpr int kRaw = KD + SQ + 1;
  static constexpr int kStride = (kRaw + 3) / 4 * 4;  // floats, 16-byte multiple
  static constexpr int kBeta = KD + SQ;                // index of -beta
};

constexpr float kRebase = 65536.0f;  // 2^16: lazy-rebase trigger per group sum

template <int KD, int SQ, int R, int G>
__device__ __forceinline__ void softmin_tile(const float* __restrict__ rec, const float2 (&x2)[R / 2][KD],
                                             const float2 (&s2)[R / 2], float (&mq)[R], float (&S)[R]) {
  using L = ColLayout<KD, SQ>;
  constexpr int P = R / 2;
#pragma unroll 1
  for (int j = 0; j < kColTile; j += G) {
    float2 q[P][G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float c[L::kStride];
      const float4* r4 = reinterpret_cast<const float4*>(rec + (j + g) * L::kStride);
#pragma unroll
      for (int v = 0; v < L::kStride / 4; ++v) {
        float4 t = r4[v];
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
          float2 u = add2(s2[p], f2(c[KD], c[KD]));
          acc = fma2(u, u, acc);
        }
        q[p][g] = acc;
      }
    }
    // group sums against the current references
#pragma unroll
    for (int p = 0; p < P; ++p) {
      float2 m2 = f2(mq[2 * p], mq[2 * p + 1]);
      float2 gs = f2(0.f, 0.f);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float2 v = fma2(q[p][g], f2(-1.f, -1.f), m2);
        gs = add2(gs, f2(ex2(v.x), ex2(v.y)));
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 2 * p + h;
        float gsum = h ? gs.y : gs.x;
        if (!(gsum <= kRebase)) {
          // rare path: rebase the row reference at the group minimum
          float qmin = h ? q[p][0].y : q[p][0].x;
#pragma unroll
          for (int g = 1; g < G; ++g) qmin = fminf(qmin, h ? q[p][g].y : q[p][g].x);
          if (qmin < mq[r]) {
            S[r] *= ex2(qmin - mq[r]);
            mq[r] = qmin;
          }
          gsum = 0.f;
#pragma unroll
          for (int g = 0; g < G; ++g) gsum += ex2(mq[r] - (h ? q[p][g].y : q[p][g].x));
        }
        S[r] += gsum;
      }
    }
  }
}

template <int KD, int SQ, int R, int G, int MINB>
static __global__ void __launch_bounds__(128, MINB) softmin_fma_kernel(const SoftminArgs a) {
  using L = ColLayout<KD, SQ>;
  constexpr int P = R / 2;
  constexpr int kStageFloats = kColTile * L::kStride;
  extern __shared__ __align__(128) float smem[];
  __shared__ uint64_t bars[2];
  if (skip_now(a.st, a.skip)) return;

  const int chunk = blockIdx.y;
  const int64_t row0 = (int64_t)blockIdx.x * (128 * R) + threadIdx.x;
  const float lam = a.st->lam;
  const float sl = a.st->sqrt_lam;

  // this thread's rows, unscaled dot features + sqrt(lam) * s_i
  float2 x2[P][KD];
  float2 s2[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    float xv[2][KD];
    float sv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t i = row0 + (int64_t)(2 * p + h) * 128;
      const bool ok = i < a.n;
#pragma unroll
      for (int k = 0; k < KD; ++k) xv[h][k] = ok ? a.row_feat[i * a.ld_row + k] : 0.f;
      sv[h] = (SQ && ok) ? sl * a.row_sq[i] : 0.f;
    }
#pragma unroll
    for (int k = 0; k < KD; ++k) x2[p][k] = f2(xv[0][k], xv[1][k]);
    s2[p] = f2(sv[0], sv[1]);
  }
  float mq[R], S[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    mq[r] = CUDART_INF_F;
    S[r] = 0.f;
  }

  const int64_t c0 = (int64_t)chunk * a.chunk_cols;
  const int64_t mpad = (a.m + kColTile - 1) / kColTile * kColTile;
  const int64_t c1 = min(c0 + a.chunk_cols, mpad);
  const int ntiles = (int)((c1 - c0) / kColTile);
  const uint32_t tile_bytes = kStageFloats * sizeof(float);
  const float* src = a.col_rec + c0 * L::kStride;

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2 && s < ntiles; ++s) {
      mbar_expect_tx(&bars[s], tile_bytes);
      bulk_g2s(smem + s * kStageFloats, src + (int64_t)s * kStageFloats, tile_bytes, &bars[s]);
    }
  }
  for (int t = 0; t < ntiles; ++t) {
    const int s = t & 1;
    mbar_wait(&bars[s], (t >> 1) & 1);
    softmin_tile<KD, SQ, R, G>(smem + s * kStageFloats, x2, s2, mq, S);
    __syncthreads();  // every warp is done with stage s
    if (threadIdx.x == 0 && t + 2 < ntiles) {
      mbar_expect_tx(&bars[s], tile_bytes);
      bulk_g2s(smem + s * kStageFloats, src + (int64_t)(t + 2) * kStageFloats, tile_bytes, &bars[s]);
    }
  }

  const float inv_lam = a.st->inv_lam;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = row0 + (int64_t)r * 128;
    if (i >= a.n) continue;
    const float pmax = -mq[r];  // max_j t_ij up to the lazy slack
    if (a.nchunks > 1) {
      a.part_max[(int64_t)chunk * a.n + i] = pmax;
      a.part_sum[(int64_t)chunk * a.n + i] = S[r];
    } else if (a.out_max) {
      a.out_max[i] = pmax;
      a.out_sum[i] = S[r];
    } else {
      const float add = a.row_add ? a.row_add[i] : 0.f;
      a.out[i] = add - (pmax + log2f(S[r])) * inv_lam;
    }
  }
  (void)lam;
}

// Fixed-order merge of the split-column partials of each row.
static __global__ void lse_combine_kernel(const cntgw_sweep_state* st, int skip, const float* pm,
                                   const float* ps, int nchunks, int64_t n, const float* row_add,
                                   float* out, float* out_max, float* out_sum) {
  if (skip_now(st, skip)) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float mx = -CUDART_INF_F;
  for (int c = 0; c < nchunks; ++c) mx = fmaxf(mx, pm[(int64_t)c * n + i]);
  float sm = 0.f;
  for (int c = 0; c < nchunks; ++c) {
    const float v = ps[(int64_t)c * n + i];
    if (v > 0.f) sm += v * ex2(pm[(int64_t)c * n + i] - mx);
  }
  if (out_max) {
    out_max[i] = mx;
    out_sum[i] = sm;
  } else {
    const float add = row_add ? row_add[i] : 0.f;
    out[i] = add - (mx + log2f(sm)) * st->inv_lam;
  }
}

}  // namespace cntgw
