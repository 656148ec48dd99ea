// K1/K2 fp64 half-update on the FP64 tensor pipe: the score
// q_ij = -beta_j + <[x_i | s_i], c_j> is a K' = roundup4(KD + SQ) dot product
// evaluated with DMMA (mma.sync.m8n8k4.f64: 256 fp64 FMAs per warp
// instruction, IEEE fp64 multiply-adds) whose accumulator is initialised with
// the column constant -beta_j, so C4's K=3 + squared coordinate is ONE MMA
// per 8x8 tile. Measured on B200 (tools/ubench_f64mix): DMMA and DFMA share
// one ~63 FMA/clk/SM pipe, but the DFMA form of this dot needs one issue slot
// per FMA and its dependent chains leave the pipe half idle; DMMA issues 1/8
// as many instructions, so the pipe stays busy and the epilogue (DADD, 3-op ALU
// f64->f32, MUFU.EX2, FADD) runs in the gaps.
//
// Warp tile: 8 rows x 8 columns per MMA; each warp owns RG row groups of 8
// rows (A fragments for all K' steps held in registers) and walks the column
// tiles staged in shared memory by 1-D TMA bulk copies (StageRing: per-stage
// full/empty mbarriers, each warp releases a stage when done with it). Fragment layouts (m8n8k4, f64): A[row = lane/4][k = lane%4],
// B[k = lane%4][col = lane/4], D[row = lane/4][col = 2(lane%4) + {0,1}].
// Each lane keeps its own lazily rebased (reference, sum) per row group over
// its columns (2 per 8-column tile, NT tiles per check group); the four lanes
// of a row merge at the end.
#pragma once

#include "common.cuh"
#include "softmin.cuh"

namespace cntgw {

__device__ __forceinline__ void dmma_m8n8k4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Scores of RG row groups x NT 8-column tiles starting at column ct of the
// staged tile: all MMAs independent, accumulators initialised with -beta.
template <int KD, int SQ, int RG, int NT, int KS>
__device__ __forceinline__ void dmma_scores(const double* __restrict__ tile, int ct, int lr, int lk,
                                            const double (&afr)[RG][KS], double (&q)[RG][NT][2]) {
  using L = ColLayout<double, KD, SQ>;
#pragma unroll
  for (int u = 0; u < NT; ++u) {
    double bfr[KS];
    const double* bc = tile + (ct + 8 * u + lr) * L::kStride + lk;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) bfr[ks] = bc[4 * ks];
    const double* cc = tile + (ct + 8 * u + 2 * lk) * L::kStride + L::kBeta;
    const double beta0 = cc[0], beta1 = cc[L::kStride];
#pragma unroll
    for (int rg = 0; rg < RG; ++rg) {
      q[rg][u][0] = beta0;
      q[rg][u][1] = beta1;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) dmma_m8n8k4(q[rg][u], afr[rg][ks], bfr[ks]);
    }
  }
}

// Exponentials and sums of one step, then the (rare) rebase checks last. The
// first NPOLY of the NT column tiles are exponentiated on the FMA pipe
// (degree-5 polynomial) to unload MUFU.
template <int RG, int NT, int NPOLY = 0>
__device__ __forceinline__ void dmma_consume(const double (&q)[RG][NT][2], double (&mq)[RG],
                                             double (&S)[RG], float (&T)[RG]) {
  float gsum[RG];
#pragma unroll
  for (int rg = 0; rg < RG; ++rg) {
    float2 acc = f2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < NT; ++u) {
      const float2 x = f2(f64_to_f32_fast(mq[rg] - q[rg][u][0]), f64_to_f32_fast(mq[rg] - q[rg][u][1]));
      acc = add2(acc, u < NPOLY ? exp2_poly2(x) : f2(ex2(x.x), ex2(x.y)));
    }
    gsum[rg] = acc.x + acc.y;
  }
#pragma unroll
  for (int rg = 0; rg < RG; ++rg) {
    if (!(gsum[rg] <= kRebaseF64)) {  // rare: rebase kRefOffset above the group minimum
      double qmin = q[rg][0][0];
#pragma unroll
      for (int u = 0; u < NT; ++u) qmin = fmin(qmin, fmin(q[rg][u][0], q[rg][u][1]));
      const double ref = qmin + kRefOffset;
      if (ref < mq[rg]) {
        const double sc = exp2(ref - mq[rg]);
        S[rg] *= sc;
        T[rg] *= (float)sc;
        mq[rg] = ref;
      }
      float r = 0.f;
#pragma unroll
      for (int u = 0; u < NT; ++u)
        r += ex2(f64_to_f32_fast(mq[rg] - q[rg][u][0])) + ex2(f64_to_f32_fast(mq[rg] - q[rg][u][1]));
      gsum[rg] = r;
    }
    T[rg] += gsum[rg];
  }
}

template <int KD, int SQ, int RG, int NT, int TILE, int MINB, int NS = 2, int NPOLY = 0>
__global__ void __launch_bounds__(128, MINB) softmin_dmma_kernel(const SoftminArgs a) {
  using L = ColLayout<double, KD, SQ>;
  constexpr int KS = (KD + SQ + 3) / 4;  // m8n8k4 steps per score
  static_assert(4 * KS <= L::kStride, "column record must cover the padded k4 steps");
  constexpr int kStage = TILE * L::kStride;
  extern __shared__ __align__(128) double smem_d[];
  __shared__ uint64_t full_bar[NS], empty_bar[NS];
  if (skip_now(a.st, a.skip)) return;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lr = lane >> 2, lk = lane & 3;
  const int chunk = blockIdx.y;
  const int64_t wrow = (int64_t)blockIdx.x * (32 * RG) + warp * (8 * RG);  // warp's first row
  const double* rf = static_cast<const double*>(a.row_feat);
  const double* rs = static_cast<const double*>(a.row_sq);

  // A fragments: feature k = 4 ks + lk of row wrow + 8 rg + lr, features [x | s | 0...]
  // (record entries past KD + SQ, including -beta, meet a zero feature)
  double afr[RG][KS];
  double mq[RG], S[RG];
#pragma unroll
  for (int rg = 0; rg < RG; ++rg) {
    const int64_t i = wrow + 8 * rg + lr;
    const bool ok = i < a.n;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = 4 * ks + lk;
      double v = 0.0;
      if (k < KD) v = ok ? rf[i * a.ld_row + k] : 0.0;
      else if (SQ && k == KD) v = ok ? rs[i] : 0.0;
      afr[rg][ks] = v;
    }
    mq[rg] = kStartQ;
    S[rg] = 0.0;
  }

  const int64_t c0 = (int64_t)chunk * a.chunk_cols;
  const int64_t mpad = (a.m + kColTile - 1) / kColTile * kColTile;
  const int ntiles = (int)((min(c0 + a.chunk_cols, mpad) - c0) / TILE);
  const uint32_t bytes = kStage * sizeof(double);
  const double* src = static_cast<const double*>(a.col_rec) + c0 * L::kStride;
  StageRing<NS> ring{full_bar, empty_bar};
  ring.init(4);
  if (threadIdx.x == 0)
    for (int st = 0; st < NS && st < ntiles; ++st)
      ring.load(smem_d + st * kStage, src + (int64_t)st * kStage, bytes, st);
  for (int t = 0; t < ntiles; ++t) {
    if (threadIdx.x == 0) {
      const int r = ring.refill_slot(t, ntiles);
      if (r >= 0) ring.load(smem_d + (r % NS) * kStage, src + (int64_t)r * kStage, bytes, r);
    }
    ring.wait_full(t);
    const double* tile = smem_d + (t % NS) * kStage;
    float T[RG];  // this tile's fp32 sums against mq, folded into S per tile
#pragma unroll
    for (int rg = 0; rg < RG; ++rg) T[rg] = 0.f;
#pragma unroll 1
    for (int ct = 0; ct < TILE; ct += 8 * NT) {
      // all RG x NT MMAs of this step first (independent), then the
      // exponentials, then the rare-rebase checks: branches come last so
      // the scheduler can overlap the MMA latency with the epilogue
      double q[RG][NT][2];
      dmma_scores<KD, SQ, RG, NT, KS>(tile, ct, lr, lk, afr, q);
      dmma_consume<RG, NT, NPOLY>(q, mq, S, T);
    }
#pragma unroll
    for (int rg = 0; rg < RG; ++rg) S[rg] += f32_to_f64_alu(T[rg]);
    ring.release(t);
  }

  // merge the four lanes of each row (their column subsets), then store
  const double lam = a.st->lam_d, inv_lam = 1.0 / lam;
#pragma unroll
  for (int rg = 0; rg < RG; ++rg) {
    double m = -mq[rg], s = S[rg];  // partial: 2^m * s, in log2 units
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const double m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const double s2 = __shfl_xor_sync(0xffffffffu, s, o);
      const double mm = fmax(m, m2);
      s = (s > 0.0 ? s * exp2(m - mm) : 0.0) + (s2 > 0.0 ? s2 * exp2(m2 - mm) : 0.0);
      m = mm;
    }
    const int64_t i = wrow + 8 * rg + lr;
    if (lk == 0 && i < a.n) {
      const double si = SQ ? rs[i] : 0.0;
      // q accumulated without the row constant lam s_i^2 (expanded square)
      softmin_store(a, chunk, i, m - (SQ ? lam * si * si : 0.0), s, inv_lam);
    }
  }
}

}  // namespace cntgw
