// K4 on the centred path's block-sparse plan (CNTGW_F32C problems).
//
// Same reductions as plan_reduce_kernel (reduce.cuh; reference
// `_cnt_reductions`, solvers.py:227-256, plus argmax): per row i the mass
// r_i = sum_j pi_ij, pi Y, pi s and argmax_j pi_ij of
//     pi_ij = a_i 2^(lam f~_i - lam s_i^2 - q_ij),  q_ij = c_j + <X_i, Zr_j>
// in fp64, but visiting rows and columns in the locality order of the
// centred half-update and skipping the (row group, column tile) pairs its
// plan (ctr_plan_kernel, softmin_ctr.cuh) marks as unable to hold a term
// within 2^-T (T >= 64) of the row's maximum. A skipped tile holds neither
// the argmax nor more than m 2^-64 of the row's mass, so every output equals
// the dense pass to rounding. The exponent uses the ORIGINAL fp64 row
// features (gathered through the row order) and the fp64 column records
// [Zr | c] of the centred column block, i.e. the expanded-square q of the
// fp64 path; argmax ties break at the lowest original column index.
#pragma once

#include "common.cuh"
#include "reduce.cuh"
#include "softmin_ctr.cuh"

namespace cntgw {

struct PlanReduceCtrArgs {
  const cntgw_sweep_state* st;
  const int64_t* row_order;  // locality position -> caller row (ctr row block)
  const int64_t* col_order;  // locality position -> caller column
  const double* row_feat;    // caller order, n x kd fp64 (stride ld_row)
  int64_t ld_row;
  int kd, sq;
  const double* row_sq;
  const double* f_tilde;
  const double* log2a;
  const double* rec64;  // [mpad][stride] fp64 [Zr (KX) | c | pad], locality order
  const double* acc;    // [mpad][AccLayout<E>::kStride] [Y | s], locality order
  const uint32_t* need; // CNTGW_F32C: [CTA of R groups][256-col tile] votes, or null (dense)
  int ctr_r;
  const uint8_t* need8; // CNTGW_F64S: [row group of grows rows][stage] bytes, or null
  const int* replan;    // CNTGW_F64S: the plan is stale for these records (walk every stage)
  int grows;
  int64_t n, m;
  double* row_mass;
  double* pi_y;
  int e_real;
  double* pi_s;
  int64_t* argmax;
};

// [Y | s] records in the column locality order (stride AccLayout<E>::kStride).
__global__ void pack_acc_ordered_kernel(const double* y, int64_t ld, int e_real, int e_pad, int stride,
                                        const double* s, const int64_t* order, int64_t m, int64_t mpad,
                                        double* out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= mpad) return;
  double* r = out + j * stride;
  for (int k = 0; k < stride; ++k) r[k] = 0.0;
  if (j < m) {
    const int64_t src = order ? order[j] : j;
    for (int k = 0; k < e_real; ++k) r[k] = y[src * ld + k];
    r[e_pad] = s[src];
  }
}

template <int STRIDE, int E, int TILE = kColTile>
struct CtrReduceSmem {
  static constexpr int kRec = TILE * STRIDE;                  // doubles per stage
  static constexpr int kAcc = TILE * AccLayout<E>::kStride;
  static constexpr size_t kBytes = 2 * sizeof(double) * (kRec + kAcc);
};

// CTA = 128 rows (locality order), one thread per row, all needed column
// stages of those rows through a 2-stage bulk-copy ring. KX features [x | s]
// per row against records [Zr (KX) | c | pad] of STRIDE doubles, stages of
// TILE columns. The plan is the centred path's (need: words per 256-column
// tile and CTA of ctr_r groups) or CNTGW_F64S's (need8: bytes per stage and
// row group of `grows` rows, ignored while *replan).
template <int KX, int E, int G, int STRIDE = KX + 1, int TILE = kColTile>
__global__ void __launch_bounds__(128) plan_reduce_ctr_kernel(const PlanReduceCtrArgs a) {
  using SM = CtrReduceSmem<STRIDE, E, TILE>;
  using A = AccLayout<E>;
  extern __shared__ __align__(128) double smem_k4[];
  __shared__ uint64_t bars[2];
  const int64_t grp = blockIdx.x;
  const int64_t i = grp * kCtrRowGroup + threadIdx.x;
  const bool live = i < a.n;
  const int64_t src = live ? a.row_order[i] : 0;
  double x[KX];
#pragma unroll
  for (int k = 0; k < KX; ++k)
    x[k] = !live ? 0.0 : (k < a.kd ? a.row_feat[src * a.ld_row + k] : (a.sq && k == a.kd ? a.row_sq[src] : 0.0));
  const double s = live && a.sq ? a.row_sq[src] : 0.0;

  double mq = kStartQ, S = 0.0, acc_s = 0.0, qbest = CUDART_INF;
  double acc_y[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc_y[e] = 0.0;
  int64_t jbest = INT64_MAX;

  const int64_t mpad = (a.m + kColTile - 1) / kColTile * kColTile;
  const int ntiles = (int)(mpad / TILE);
  const uint32_t* need = a.need ? a.need + (grp / a.ctr_r) * ntiles : nullptr;
  const uint32_t vote = 0x01010101u << (grp % a.ctr_r);
  // F64S: this CTA's 128 rows span 128 / grows plan row groups
  const bool use8 = a.need8 != nullptr && !(a.replan && *a.replan);
  const int64_t g8 = grp * kCtrRowGroup / (a.grows > 0 ? a.grows : 1);
  const int n8 = a.grows > 0 && a.grows < kCtrRowGroup ? kCtrRowGroup / a.grows : 1;
  const int64_t ng8 = a.grows > 0 ? (a.n + a.grows - 1) / a.grows : 0;
  auto needed8 = [&](int t) {
    for (int h = 0; h < n8; ++h)
      if (g8 + h < ng8 && a.need8[(g8 + h) * ntiles + t]) return true;
    return false;
  };
  // ... and a stage the CTA walks is needed by some of them only: this row's own
  // group decides whether it takes part (warp-uniform: the groups are multiples
  // of 32 rows; at 32-row groups a CTA's union is ~4x what each warp needs)
  const uint8_t* mine8 = use8 && live && a.grows > 0 ? a.need8 + (i / a.grows) * ntiles : nullptr;
  auto next_needed = [&](int t) {
    if (need)
      while (t < ntiles && !(need[t] & vote)) ++t;
    else if (use8)
      while (t < ntiles && !needed8(t)) ++t;
    return t;
  };
  const uint32_t rec_bytes = SM::kRec * sizeof(double), acc_bytes = SM::kAcc * sizeof(double);
  TilePipe pipe{bars};
  pipe.init();
  auto issue = [&](int t, int sb) {
    double* base = smem_k4 + sb * (SM::kRec + SM::kAcc);
    mbar_expect_tx(&bars[sb], rec_bytes + acc_bytes);
    bulk_g2s(base, a.rec64 + (int64_t)t * SM::kRec, rec_bytes, &bars[sb]);
    bulk_g2s(base + SM::kRec, a.acc + (int64_t)t * SM::kAcc, acc_bytes, &bars[sb]);
  };
  int tq[2];
  tq[0] = next_needed(0);
  tq[1] = next_needed(tq[0] + 1);
  if (threadIdx.x == 0)
    for (int sb = 0; sb < 2; ++sb)
      if (tq[sb] < ntiles) issue(tq[sb], sb);

  for (int it = 0; tq[it & 1] < ntiles; ++it) {
    const int sb = it & 1;
    const int t = tq[sb];
    mbar_wait(&bars[sb], (it >> 1) & 1);
    const double* rec = smem_k4 + sb * (SM::kRec + SM::kAcc);
    const double* acr = rec + SM::kRec;
    const int jend = (use8 && (!mine8 || !mine8[t])) ? 0 : TILE;  // (dead rows of an F64S plan skip too)
#pragma unroll 1
    for (int j = 0; j < jend; j += G) {
      double q[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double* c = rec + (j + g) * STRIDE;
        double acc = c[KX];
#pragma unroll
        for (int k = 0; k < KX; ++k) acc = fma(x[k], c[k], acc);
        q[g] = acc;
        const int64_t jj = (int64_t)t * TILE + j + g;
        if (acc <= qbest && acc < kPadQ && jj < a.m) {  // ties: lowest ORIGINAL column (numpy.argmax)
          const int64_t oj = a.col_order ? a.col_order[jj] : jj;
          if (acc < qbest || oj < jbest) {
            qbest = acc;
            jbest = oj;
          }
        }
      }
      double ev[G], gs = 0.0;  // fp64 exponentials: the pass reports fp64 sums
#pragma unroll
      for (int g = 0; g < G; ++g) {
        ev[g] = exp2_f64(mq - q[g]);
        gs += ev[g];
      }
      if (!(gs <= (double)kRebase)) {
        double qmin = q[0];
#pragma unroll
        for (int g = 1; g < G; ++g) qmin = fmin(qmin, q[g]);
        if (qmin < mq) {
          const double sc = exp2(qmin - mq);
          S *= sc;
          acc_s *= sc;
#pragma unroll
          for (int e = 0; e < E; ++e) acc_y[e] *= sc;
          mq = qmin;
        }
#pragma unroll
        for (int g = 0; g < G; ++g) ev[g] = exp2_f64(mq - q[g]);
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double* y = acr + (j + g) * A::kStride;
        const double w = ev[g];
        S += w;
        acc_s = fma(w, y[E], acc_s);
#pragma unroll
        for (int e = 0; e < E; ++e) acc_y[e] = fma(w, y[e], acc_y[e]);
      }
    }
    __syncthreads();  // every thread is done with stage sb
    tq[sb] = next_needed(tq[sb ^ 1] + 1);  // the needed tile after the one in the other stage
    if (threadIdx.x == 0 && tq[sb] < ntiles) issue(tq[sb], sb);
  }
  if (!live) return;
  const double scale = exp2(a.st->lam_d * (a.f_tilde[src] - s * s) + a.log2a[src] - mq);
  a.row_mass[src] = S * scale;
  a.pi_s[src] = acc_s * scale;
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (e < a.e_real) a.pi_y[src * a.e_real + e] = acc_y[e] * scale;
  a.argmax[src] = jbest == INT64_MAX ? 0 : jbest;
}

}  // namespace cntgw
