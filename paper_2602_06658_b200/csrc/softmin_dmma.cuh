// K1/K2 fp64 half-update for wide features (KD >= 16, the C5 shape) on the
// FP64 tensor pipe: the score q_ij = -beta_j + <[x_i | s_i | 1], c_j> is a
// K' = roundup4(KD + SQ + 1) dot product, evaluated with DMMA
// (mma.sync.m8n8k4.f64: 256 fp64 FMAs per warp instruction, IEEE fp64
// multiply-adds). Measured on B200 (tools/ubench_f64mix): DMMA and DFMA share
// one ~63 FMA/clk/SM pipe, but the DFMA form of this dot needs one issue slot
// per FMA and its dependent chains leave the pipe half idle; DMMA issues 1/8
// as many instructions, so the pipe stays busy and the epilogue (DADD, 3-op ALU
// f64->f32, MUFU.EX2, FADD) runs in the gaps.
//
// Warp tile: 8 rows x 8 columns per MMA; each warp owns RG row groups of 8
// rows (A fragments for all K' steps held in registers) and walks the column
// tiles staged in shared memory by the TMA bulk-copy ring (same as the DFMA
// kernel). Fragment layouts (m8n8k4, f64): A[row = lane/4][k = lane%4],
// B[k = lane%4][col = lane/4], D[row = lane/4][col = 2(lane%4) + {0,1}].
// Each lane keeps its own lazily rebased (reference, sum) per row group over
// its two columns per tile; the four lanes of a row merge at the end.
#pragma once

#include "common.cuh"
#include "softmin.cuh"

namespace cntgw {

__device__ __forceinline__ void dmma_m8n8k4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int KD, int SQ, int RG, int TILE, int MINB>
__global__ void __launch_bounds__(128, MINB) softmin_dmma_kernel(const SoftminArgs a) {
  using L = ColLayout<double, KD, SQ>;
  static_assert(L::kStride % 4 == 0, "DMMA path needs K' padded to the k4 step");
  constexpr int KS = L::kStride / 4;  // m8n8k4 steps per score
  constexpr int kStage = TILE * L::kStride;
  extern __shared__ __align__(128) double smem_d[];
  __shared__ uint64_t bars[2];
  if (skip_now(a.st, a.skip)) return;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lr = lane >> 2, lk = lane & 3;
  const int chunk = blockIdx.y;
  const int64_t wrow = (int64_t)blockIdx.x * (32 * RG) + warp * (8 * RG);  // warp's first row
  const double* rf = static_cast<const double*>(a.row_feat);
  const double* rs = static_cast<const double*>(a.row_sq);

  // A fragments: feature k = 4 ks + lk of row wrow + 8 rg + lr, features [x | s | 1 | 0...]
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
      else if (k == KD + SQ) v = 1.0;
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
    const double* tile = smem_d + sb * kStage;
    float T[RG];  // this tile's fp32 sums against mq, folded into S per tile
#pragma unroll
    for (int rg = 0; rg < RG; ++rg) T[rg] = 0.f;
#pragma unroll 1
    for (int ct = 0; ct < TILE; ct += 8) {
      double bfr[KS];
      const double* bc = tile + (ct + lr) * L::kStride + lk;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) bfr[ks] = bc[4 * ks];
#pragma unroll
      for (int rg = 0; rg < RG; ++rg) {
        double q[2] = {0.0, 0.0};
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) dmma_m8n8k4(q, afr[rg][ks], bfr[ks]);
        float gsum = ex2(f64_to_f32_fast(mq[rg] - q[0])) + ex2(f64_to_f32_fast(mq[rg] - q[1]));
        if (!(gsum <= kRebaseF64)) {  // rare: rebase kRefOffset above the pair minimum
          const double ref = fmin(q[0], q[1]) + kRefOffset;
          if (ref < mq[rg]) {
            const double sc = exp2(ref - mq[rg]);
            S[rg] *= sc;
            T[rg] *= (float)sc;
            mq[rg] = ref;
          }
          gsum = ex2(f64_to_f32_fast(mq[rg] - q[0])) + ex2(f64_to_f32_fast(mq[rg] - q[1]));
        }
        T[rg] += gsum;
      }
    }
#pragma unroll
    for (int rg = 0; rg < RG; ++rg) S[rg] += f32_to_f64_alu(T[rg]);
    __syncthreads();
    if (threadIdx.x == 0 && t + 2 < ntiles) {
      mbar_expect_tx(&bars[sb], bytes);
      bulk_g2s(smem_d + sb * kStage, src + (int64_t)(t + 2) * kStage, bytes, &bars[sb]);
    }
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
