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
#include "softmin_fma.cuh"

namespace cntgw {

struct PlanReduceArgs {
  const cntgw_sweep_state* st;
  const float* row_feat;
  int64_t ld_row;
  const float* row_sq;
  const float* f_tilde;
  const float* log2a;
  const float* col_rec;  // packed q-records (cntgw_prep_cols)
  const float* col_acc;  // packed [Y (E) | s | pad] records, stride EA
  int64_t n, m;
  float* row_mass;
  float* pi_y;  // n x e_real
  int e_real;
  float* pi_s;
  int64_t* argmax;
};

template <int E>
struct AccLayout {
  static constexpr int kStride = (E + 1 + 3) / 4 * 4;
};

template <int KD, int SQ, int E, int G>
static __global__ void __launch_bounds__(128) plan_reduce_kernel(const PlanReduceArgs a) {
  using L = ColLayout<KD, SQ>;
  using A = AccLayout<E>;
  constexpr int kRecF = kColTile * L::kStride;
  constexpr int kAccF = kColTile * A::kStride;
  extern __shared__ __align__(128) float smem[];
  __shared__ uint64_t bars[2];

  const int64_t i = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const bool live = i < a.n;
  const float sl = a.st->sqrt_lam;
  float x[KD];
#pragma unroll
  for (int k = 0; k < KD; ++k) x[k] = live ? a.row_feat[i * a.ld_row + k] : 0.f;
  const float s = (SQ && live) ? sl * a.row_sq[i] : 0.f;

  float mq = CUDART_INF_F, S = 0.f, acc_s = 0.f, qbest = CUDART_INF_F;
  float acc_y[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc_y[e] = 0.f;
  int64_t jbest = 0;

  const int64_t mpad = (a.m + kColTile - 1) / kColTile * kColTile;
  const int ntiles = (int)(mpad / kColTile);
  const uint32_t rec_bytes = kRecF * sizeof(float), acc_bytes = kAccF * sizeof(float);
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int t, int s_) {
    float* base = smem + s_ * (kRecF + kAccF);
    mbar_expect_tx(&bars[s_], rec_bytes + acc_bytes);
    bulk_g2s(base, a.col_rec + (int64_t)t * kRecF, rec_bytes, &bars[s_]);
    bulk_g2s(base + kRecF, a.col_acc + (int64_t)t * kAccF, acc_bytes, &bars[s_]);
  };
  if (threadIdx.x == 0)
    for (int s_ = 0; s_ < 2 && s_ < ntiles; ++s_) issue(s_, s_);

  for (int t = 0; t < ntiles; ++t) {
    const int sb = t & 1;
    mbar_wait(&bars[sb], (t >> 1) & 1);
    const float* rec = smem + sb * (kRecF + kAccF);
    const float* acr = rec + kRecF;
#pragma unroll 1
    for (int j = 0; j < kColTile; j += G) {
      float q[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float* c = rec + (j + g) * L::kStride;
        float acc = c[L::kBeta];
#pragma unroll
        for (int k = 0; k < KD; ++k) acc = fmaf(x[k], c[k], acc);
        if (SQ) {
          const float u = s + c[KD];
          acc = fmaf(u, u, acc);
        }
        q[g] = acc;
        if (acc < qbest) {  // strict: first (lowest) j wins ties, numpy.argmax convention
          qbest = acc;
          jbest = (int64_t)t * kColTile + j + g;
        }
      }
      float ev[G], gs = 0.f;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        ev[g] = ex2(mq - q[g]);
        gs += ev[g];
      }
      if (!(gs <= kRebase)) {
        float qmin = q[0];
#pragma unroll
        for (int g = 1; g < G; ++g) qmin = fminf(qmin, q[g]);
        if (qmin < mq) {
          const float sc = ex2(qmin - mq);
          S *= sc;
          acc_s *= sc;
#pragma unroll
          for (int e = 0; e < E; ++e) acc_y[e] *= sc;
          mq = qmin;
        }
#pragma unroll
        for (int g = 0; g < G; ++g) ev[g] = ex2(mq - q[g]);
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float* y = acr + (j + g) * A::kStride;
        S += ev[g];
        acc_s = fmaf(ev[g], y[E], acc_s);
#pragma unroll
        for (int e = 0; e < E; ++e) acc_y[e] = fmaf(ev[g], y[e], acc_y[e]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && t + 2 < ntiles) issue(t + 2, sb);
  }
  if (!live) return;
  // pi_ij = a_i 2^(lam f~_i) 2^(t_ij); sum_j 2^(t_ij) = 2^(-mq) S
  const float scale = ex2(a.st->lam * a.f_tilde[i] + a.log2a[i] - mq);
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
static __global__ void outer_rows_kernel(const float* x, int64_t ldx, int d, const float* pi_y, int e,
                                  int ld_piy, const float* r, const float* pi_s, const float* ft,
                                  const float* s_half, const double* a, int64_t n, int64_t rpb,
                                  double* part, int stride) {
  __shared__ double red[32];
  const int64_t i0 = (int64_t)blockIdx.x * rpb, i1 = min(n, i0 + rpb);
  double v0 = 0, v1 = 0, v2 = 0, v3 = 0, v4 = 0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const double ri = r[i], si = s_half[i];
    v0 += (double)ft[i] * ri;
    v1 += si * si * ri;
    v2 += fabs(ri - a[i]);
    v3 += si * (double)pi_s[i];
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
    for (int64_t i = i0; i < i1; ++i) acc += (double)x[i * ldx + p] * (double)pi_y[i * ld_piy + q];
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
static __global__ void outer_cols_kernel(const cntgw_sweep_state* st, const float* g, const float* gt,
                                  const float* t_half, const double* b, int64_t m, double* part) {
  __shared__ double red[32];
  const double lam = (double)st->lam;
  double v0 = 0, v1 = 0, v2 = 0, v3 = 0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double c = b[j] * exp2(lam * ((double)g[j] - (double)gt[j]));
    const double tj = t_half[j];
    v0 += (double)g[j] * c;
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
static __global__ void apply_operator_kernel(const double* op, int dout, int din, const float* feat,
                                      int64_t ld, int64_t n, float* out) {
  extern __shared__ double sop[];
  for (int k = threadIdx.x; k < dout * din; k += blockDim.x) sop[k] = op[k];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* fi = feat + i * ld;
  for (int o = 0; o < dout; ++o) {
    double acc = 0.0;
    for (int k = 0; k < din; ++k) acc += sop[o * din + k] * (double)fi[k];
    out[i * dout + o] = (float)acc;
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
