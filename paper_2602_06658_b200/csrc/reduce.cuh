// K4-K7: fused plan reductions, operator application, outer-step reductions
// and the closed-form loss constant.
//
// K4 replaces the reference's `_cnt_reductions` (solvers.py:227-256), the
// plan marginals behind `marginal_error` (measures.py:197-235) and adds the
// argmax plan indices: one streaming pass over
//     pi_ij = a_i 2^(lam f~_i + t_ij)          (t_ij as in the half-update)
// accumulating per row the mass r_i, pi Y (e-wide), pi s and the argmax, with
// the same lazily rebased online exponent as softmin_fma.cuh. The remaining
// O(N D E) / O(M) reductions run in fp64 with fixed-order block trees so that
// reruns are bit-identical (no float atomics).
#pragma once

#include "common.cuh"
#include "softmin.cuh"

namespace cntgw {

struct PlanReduceArgs {
  const cntgw_sweep_state* st;
  const double* row_feat;
  int64_t ld_row;
  const double* row_sq;
  const double* f_tilde;
  const double* log2a;
  const double* col_rec;  // packed fp64 q-records (cntgw_prep_cols, CNTGW_F64, sq=1)
  const double* col_acc;  // packed [Y (E) | s | pad] fp64 records, stride AccLayout<E>
  int64_t n, m;
  double* row_mass;
  double* pi_y;  // n x e_real
  int e_real;
  double* pi_s;
  int64_t* argmax;
};

template <int E>
struct AccLayout {
  static constexpr int kStride = (E + 1 + 1) / 2 * 2;  // doubles, 16-byte multiple
};

// One fp64 pass per row: mass, pi Y, pi s and argmax against a lazily
// rebased reference (same scheme as the fp64 softmin).
template <int KD, int E, int G, int TILE>
__global__ void __launch_bounds__(128) plan_reduce_kernel(const PlanReduceArgs a) {
  using L = ColLayout<double, KD, 1>;
  using A = AccLayout<E>;
  constexpr int kRecN = TILE * L::kStride;
  constexpr int kAccN = TILE * A::kStride;
  extern __shared__ __align__(128) double smem_r[];
  __shared__ uint64_t bars[2];

  const int64_t i = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const bool live = i < a.n;
  double x[KD];
#pragma unroll
  for (int k = 0; k < KD; ++k) x[k] = live ? a.row_feat[i * a.ld_row + k] : 0.0;
  const double s = live ? a.row_sq[i] : 0.0;

  double mq = kStartQ, S = 0.0, acc_s = 0.0, qbest = CUDART_INF;
  double acc_y[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc_y[e] = 0.0;
  int64_t jbest = 0;

  const int64_t mpad = (a.m + kColTile - 1) / kColTile * kColTile;
  const int ntiles = (int)(mpad / TILE);
  const uint32_t rec_bytes = kRecN * sizeof(double), acc_bytes = kAccN * sizeof(double);
  TilePipe pipe{bars};
  pipe.init();
  auto issue = [&](int t, int sb) {
    double* base = smem_r + sb * (kRecN + kAccN);
    mbar_expect_tx(&bars[sb], rec_bytes + acc_bytes);
    bulk_g2s(base, a.col_rec + (int64_t)t * kRecN, rec_bytes, &bars[sb]);
    bulk_g2s(base + kRecN, a.col_acc + (int64_t)t * kAccN, acc_bytes, &bars[sb]);
  };
  if (threadIdx.x == 0)
    for (int sb = 0; sb < 2 && sb < ntiles; ++sb) issue(sb, sb);

  for (int t = 0; t < ntiles; ++t) {
    const int sb = t & 1;
    mbar_wait(&bars[sb], (t >> 1) & 1);
    const double* rec = smem_r + sb * (kRecN + kAccN);
    const double* acr = rec + kRecN;
#pragma unroll 1
    for (int j = 0; j < TILE; j += G) {
      double q[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double* c = rec + (j + g) * L::kStride;
        double acc = c[L::kBeta];
#pragma unroll
        for (int k = 0; k < KD; ++k) acc = fma(x[k], c[k], acc);
        acc = fma(s, c[KD], acc);  // expanded square; lam s_i^2 is a row constant
        q[g] = acc;
        if (acc < qbest) {  // strict: the first (lowest) j wins ties, numpy.argmax rule
          qbest = acc;
          jbest = (int64_t)t * TILE + j + g;
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
    __syncthreads();
    if (threadIdx.x == 0 && t + 2 < ntiles) issue(t + 2, sb);
  }
  if (!live) return;
  // pi_ij = a_i 2^(lam f~_i) 2^(t_ij) and sum_j 2^(t_ij) = 2^(-mq) S
  const double scale = exp2(a.st->lam_d * (a.f_tilde[i] - s * s) + a.log2a[i] - mq);
  a.row_mass[i] = S * scale;
  a.pi_s[i] = acc_s * scale;
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (e < a.e_real) a.pi_y[i * a.e_real + e] = acc_y[e] * scale;
  a.argmax[i] = jbest;
}

// ---- fp64 fixed-order reductions --------------------------------------------
constexpr int kRedThreads = 256;

// Stage 1 of the outer-step row reduction: block b sums rows [b*rpb, (b+1)*rpb).
static __global__ void outer_rows_kernel(const double* x, int64_t ldx, int d, const double* pi_y,
                                         int e, int ld_piy, const double* r, const double* pi_s,
                                         const double* ft, const double* s_half, const double* a,
                                         int64_t n, int64_t rpb, double* part, int stride) {
  __shared__ double red[32];
  const int64_t i0 = (int64_t)blockIdx.x * rpb, i1 = min(n, i0 + rpb);
  double v0 = 0, v1 = 0, v2 = 0, v3 = 0, v4 = 0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const double ri = r[i], si = s_half[i];
    v0 += ft[i] * ri;
    v1 += si * si * ri;
    v2 += fabs(ri - a[i]);
    v3 += si * pi_s[i];
    v4 += ri;
  }
  double* out = part + (int64_t)blockIdx.x * stride;
  double t;
  t = block_sum_f64(v0, red);
  if (threadIdx.x == 0) out[0] = t;
  t = block_sum_f64(v1, red);
  if (threadIdx.x == 0) out[1] = t;
  t = block_sum_f64(v2, red);
  if (threadIdx.x == 0) out[2] = t;
  t = block_sum_f64(v3, red);
  if (threadIdx.x == 0) out[3] = t;
  t = block_sum_f64(v4, red);
  if (threadIdx.x == 0) out[4] = t;
  // Gamma_next partial: thread-owned (p, q) entries, fixed row order
  for (int idx = threadIdx.x; idx < d * e; idx += blockDim.x) {
    const int p = idx / e, q = idx % e;
    double acc = 0.0;
    for (int64_t i = i0; i < i1; ++i) acc += x[i * ldx + p] * pi_y[i * ld_piy + q];
    out[16 + idx] = acc;
  }
}

// Stage 2: sum `nb` partial vectors of length `len` in block order.
static __global__ void sum_partials_kernel(const double* part, int nb, int stride, int len, double* out) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < len; k += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int b = 0; b < nb; ++b) acc += part[(int64_t)b * stride + k];
    out[k] = acc;
  }
}

// Column side: c_j = b_j 2^(lam (g~_j - gt_j)) from the g-tentative of the final pair.
static __global__ void outer_cols_kernel(const cntgw_sweep_state* st, int prec, const double* g,
                                         const double* gt, const double* t_half, const double* b,
                                         int64_t m, double* part) {
  __shared__ double red[32];
  const double lam = prec == CNTGW_F64 ? st->lam_d : (double)st->lam;
  double v0 = 0, v1 = 0, v2 = 0, v3 = 0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double c = b[j] * exp2(lam * (g[j] - gt[j]));
    const double tj = t_half[j];
    v0 += g[j] * c;
    v1 += tj * tj * c;
    v2 += fabs(c - b[j]);
    v3 += c;
  }
  double t;
  double* out = part + (int64_t)blockIdx.x * 8;
  t = block_sum_f64(v0, red);
  if (threadIdx.x == 0) out[0] = t;
  t = block_sum_f64(v1, red);
  if (threadIdx.x == 0) out[1] = t;
  t = block_sum_f64(v2, red);
  if (threadIdx.x == 0) out[2] = t;
  t = block_sum_f64(v3, red);
  if (threadIdx.x == 0) {
    out[3] = t;
    out[4] = out[5] = out[6] = out[7] = 0.0;
  }
}

// out_i = op . feat_i  (op: dout x din fp64, staged in shared memory)
static __global__ void apply_operator_kernel(const double* op, int dout, int din, const double* feat,
                                             int64_t ld, int64_t n, double* out64, float* out32,
                                             int64_t ld_out) {
  extern __shared__ double sop[];
  for (int k = threadIdx.x; k < dout * din; k += blockDim.x) sop[k] = op[k];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* fi = feat + i * ld;
  for (int o = 0; o < dout; ++o) {
    double acc = 0.0;
    for (int k = 0; k < din; ++k) acc = fma(sop[o * din + k], fi[k], acc);
    out64[i * ld_out + o] = acc;
    if (out32) out32[i * ld_out + o] = (float)acc;
  }
}

// moments: pass 1 (weighted mean + raw T), pass 2 (centered 2nd/4th moments, covariance)
static __global__ void moments_pass1_kernel(const double* x, int64_t ldx, int d, const double* w, int64_t n,
                                     int64_t rpb, double* part, int stride) {
  __shared__ double red[32];
  const int64_t i0 = (int64_t)blockIdx.x * rpb, i1 = min(n, i0 + rpb);
  double tr = 0.0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    double nn = 0.0;
    for (int k = 0; k < d; ++k) nn += x[i * ldx + k] * x[i * ldx + k];
    tr += w[i] * nn;
  }
  double* out = part + (int64_t)blockIdx.x * stride;
  double t = block_sum_f64(tr, red);
  if (threadIdx.x == 0) out[0] = t;
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    double acc = 0.0;
    for (int64_t i = i0; i < i1; ++i) acc += w[i] * x[i * ldx + k];
    out[1 + k] = acc;
  }
}

static __global__ void moments_pass2_kernel(const double* x, int64_t ldx, int d, const double* w, int64_t n,
                                     int64_t rpb, const double* mean, double* part, int stride) {
  __shared__ double red[32];
  __shared__ double mu[64];
  for (int k = threadIdx.x; k < d; k += blockDim.x) mu[k] = mean[1 + k];
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * rpb, i1 = min(n, i0 + rpb);
  double q4 = 0.0, q2 = 0.0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    double nn = 0.0;
    for (int k = 0; k < d; ++k) {
      const double c = x[i * ldx + k] - mu[k];
      nn += c * c;
    }
    q4 += w[i] * nn * nn;
    q2 += w[i] * nn;
  }
  double* out = part + (int64_t)blockIdx.x * stride;
  double t = block_sum_f64(q4, red);
  if (threadIdx.x == 0) out[0] = t;
  t = block_sum_f64(q2, red);
  if (threadIdx.x == 0) out[1] = t;
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) {
    const int p = idx / d, q = idx % d;
    double acc = 0.0;
    for (int64_t i = i0; i < i1; ++i)
      acc += w[i] * (x[i * ldx + p] - mu[p]) * (x[i * ldx + q] - mu[q]);
    out[2 + idx] = acc;
  }
}

}  // namespace cntgw
