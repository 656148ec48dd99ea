// CNTGW_F64S: the fp32 probe that replaces the dense fp64 measuring sweep.
//
// The first sweep of every Sinkhorn loop (new operator Gamma, new lam) must
// measure the plan from scratch: each row's minimum q over each column stage
// (tmin, softmin_f64s.cuh). The fp64 kernel did that by walking every pair
// with its exponentials (MUFU-bound, ~0.5-0.66 s per half-update at C4).
// A plan only needs LOWER BOUNDS of the stage minima, accurate to a few log2
// units against the plan's 64-unit margin, and no exponentials: this kernel
// evaluates q_ij = beta_j + sum_k a_ik b_jk in fp32 with FFMA2 (two rows per
// instruction) and takes the minimum with FMNMX3, then subtracts a rigorous
// bound of the fp32 evaluation error. The exact fp64 sweep that follows walks
// only the stages the probe's plan keeps.
//
// Error bound (per row i and stage t). The inputs are rounded to fp32
// (relative u = 2^-24 each) and the K-term FMA chain rounds K times, so
//   |fl(q_ij) - q_ij| <= (K + 4) u (|beta_j| + sum_k |a_ik| |b_jk|)
//                    <= E_it = (K + 4) u (Bb_t + sum_k |a_ik| B_tk) (1 + 2^-10)
// with B_tk, Bb_t the stage's largest |b_jk|, |beta_j| (finite betas: +inf is
// a zero-weight column, exactly +inf in fp32 too). The probe stores
// tmin = round_down(min_j fl(q_ij) - E_it), a lower bound of the stage
// minimum, and publishes slack = max 2 E_it: the true row minimum is at most
// the smallest tmin plus the slack (the plan's reduce lowers gmin by it).
// Non-finite features or NaN constants make the probe stand down (*nan), and
// the dense fp64 measurement runs instead (NaN propagates as before).
#pragma once

#include "common.cuh"
#include "softmin.cuh"

namespace cntgw {

// fp32 probe record: [b_0 .. b_{K-1}, beta] padded to a multiple of 4 floats
template <int K>
struct ProbeLayout {
  static constexpr int kP = (K + 1 + 3) / 4 * 4;
};

// (1 thread) the probe runs iff this sweep must measure over every stage and
// no record is non-finite; resets the published slack
__global__ void f64s_probe_gate_kernel(const int* full, const int* nan, int* probe_ok, float* slack) {
  *probe_ok = (*full && !*nan) ? 1 : 0;  // (*full is 0 when the loop is done, f64s_begin_kernel)
  *slack = 0.f;
}

// one block per stage (gated on *full): fp32 copies of the ordered fp64
// records and the stage's magnitude bounds [B_t0 .. B_t(K-1), Bb_t]; columns
// past m get b = 0, beta = +inf (no term)
template <int K>
__global__ void __launch_bounds__(128) f64s_probe_prep_kernel(const int* full, const double* rec, int stride,
                                                              int64_t m, int tile, float* rec32, float* sbound,
                                                              int* nan) {
  if (!*full) return;
  constexpr int P = ProbeLayout<K>::kP;
  __shared__ float red[4][K + 1];
  float bmax[K + 1];
#pragma unroll
  for (int k = 0; k <= K; ++k) bmax[k] = 0.f;
  bool bad = false;
  const int64_t j0 = (int64_t)blockIdx.x * tile;
  for (int u = threadIdx.x; u < tile; u += blockDim.x) {
    const int64_t j = j0 + u;
    float* o = rec32 + j * P;
    if (j >= m) {
#pragma unroll
      for (int k = 0; k < P; ++k) o[k] = 0.f;
      o[K] = CUDART_INF_F;
      continue;
    }
    const double* r = rec + j * stride;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double v = r[k];
      bad |= !(fabs(v) < 1e30);
      const float f = (float)v;
      o[k] = f;
      bmax[k] = fmaxf(bmax[k], fabsf(f));
    }
    const double beta = r[K];
    bad |= (beta != beta) || beta == -CUDART_INF;
    const float fb = beta == CUDART_INF ? CUDART_INF_F : (float)beta;
    bad |= !(fabsf(fb) < 1e30f) && beta != CUDART_INF;
    o[K] = fb;
    if (beta != CUDART_INF) bmax[K] = fmaxf(bmax[K], fabsf(fb));
#pragma unroll
    for (int k = K + 1; k < P; ++k) o[k] = 0.f;
  }
  if (bad) atomicOr(nan, 1);
#pragma unroll
  for (int k = 0; k <= K; ++k) {
    float v = bmax[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][k] = v;
  }
  __syncthreads();
  if (threadIdx.x <= K) {
    float v = red[0][threadIdx.x];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = fmaxf(v, red[w][threadIdx.x]);
    sbound[(int64_t)blockIdx.x * P + threadIdx.x] = v;
  }
}

// grid-stride over the rows block (gated on *full): non-finite row features
__global__ void f64s_probe_rows_check_kernel(const int* full, const void* rows_block, int64_t n, int kd, int sq,
                                             int* nan) {
  if (!*full) return;
  const char* rb = static_cast<const char*>(rows_block);
  const double* rf = reinterpret_cast<const double*>(rb + align256(sizeof(int64_t) * n));
  const double* rs = reinterpret_cast<const double*>(rb + align256(sizeof(int64_t) * n) +
                                                     align256(sizeof(double) * n * kd));
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int k = 0; k < kd; ++k) bad |= !(fabs(rf[i * kd + k]) < 1e30);
    if (sq) bad |= !(fabs(rs[i]) < 1e30);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nan, 1);
}

// The probe. CTA = 128 threads x R rows (row r*128 + tid of the CTA's block
// of ordered rows) over one chunk of stages (blockIdx.y); stages arrive by
// 1-D bulk copies into a 2-slot ring. Per two columns and row pair: K FFMA2
// per column, one FMNMX3 per row.
template <int KD, int SQ, int R, int TD, int NS = 2>
__global__ void __launch_bounds__(128) f64s_probe_kernel(const cntgw_sweep_state* st, int skip, const int* probe_ok,
                                                         const void* rows_block, int64_t n, const float* rec32,
                                                         const float* sbound, int stages, int chunk_stages,
                                                         float* tmin, float* slack) {
  constexpr int K = KD + SQ;
  constexpr int P = ProbeLayout<K>::kP;
  static_assert(R % 2 == 0, "rows go in pairs");
  extern __shared__ __align__(128) float psm[];
  __shared__ uint64_t full_bar[NS], empty_bar[NS];
  if (!*probe_ok) return;

  const char* rb = static_cast<const char*>(rows_block);
  const double* rf = reinterpret_cast<const double*>(rb + align256(sizeof(int64_t) * n));
  const double* rs = reinterpret_cast<const double*>(rb + align256(sizeof(int64_t) * n) +
                                                     align256(sizeof(double) * n * KD));
  const int64_t i0 = (int64_t)blockIdx.x * (128 * R) + threadIdx.x;
  float2 a2[R / 2][K];  // row pairs (2p, 2p + 1)
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = i0 + 128 * r;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      float v = 0.f;
      if (i < n) v = (float)(k < KD ? rf[i * KD + k] : rs[i]);
      if (r & 1) a2[r / 2][k].y = v;
      else a2[r / 2][k].x = v;
    }
  }

  const int t0 = blockIdx.y * chunk_stages;
  const int nt = min(stages - t0, chunk_stages);
  const uint32_t bytes = TD * P * sizeof(float);
  StageRing<NS> ring{full_bar, empty_bar};
  ring.init(4);
  if (threadIdx.x == 0)
    for (int s = 0; s < NS && s < nt; ++s) ring.load(psm + s * TD * P, rec32 + (int64_t)(t0 + s) * TD * P, bytes, s);
  constexpr float kE = (float)(K + 4) * 0x1p-24f * (1.f + 0x1p-10f);
  float smax = 0.f;
  for (int k = 0; k < nt; ++k) {
    if (threadIdx.x == 0) {
      const int rr = ring.refill_slot(k, nt);
      if (rr >= 0) ring.load(psm + (rr % NS) * TD * P, rec32 + (int64_t)(t0 + rr) * TD * P, bytes, rr);
    }
    ring.wait_full(k);
    const float* tile = psm + (k % NS) * TD * P;
    float mn[R];
#pragma unroll
    for (int r = 0; r < R; ++r) mn[r] = CUDART_INF_F;
#pragma unroll 2
    for (int j = 0; j < TD; j += 2) {
      float b0[P], b1[P];
#pragma unroll
      for (int v = 0; v < P; v += 4) {
        const float4 x = *reinterpret_cast<const float4*>(tile + j * P + v);
        const float4 y = *reinterpret_cast<const float4*>(tile + (j + 1) * P + v);
        b0[v] = x.x, b0[v + 1] = x.y, b0[v + 2] = x.z, b0[v + 3] = x.w;
        b1[v] = y.x, b1[v + 1] = y.y, b1[v + 2] = y.z, b1[v + 3] = y.w;
      }
#pragma unroll
      for (int p = 0; p < R / 2; ++p) {
        float2 q0 = f2(b0[K], b0[K]), q1 = f2(b1[K], b1[K]);
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
          q0 = fma2(a2[p][kk], f2(b0[kk], b0[kk]), q0);
          q1 = fma2(a2[p][kk], f2(b1[kk], b1[kk]), q1);
        }
        mn[2 * p] = fmin3f(mn[2 * p], q0.x, q1.x);
        mn[2 * p + 1] = fmin3f(mn[2 * p + 1], q0.y, q1.y);
      }
    }
    ring.release(k);
    const int t = t0 + k;
    const float* sb = sbound + (int64_t)t * P;
    float bk[K + 1];
#pragma unroll
    for (int kk = 0; kk <= K; ++kk) bk[kk] = __ldg(sb + kk);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t i = i0 + 128 * r;
      float e = bk[K];
#pragma unroll
      for (int kk = 0; kk < K; ++kk) e = __fmaf_ru(fabsf((r & 1) ? a2[r / 2][kk].y : a2[r / 2][kk].x), bk[kk], e);
      e = __fmul_ru(e, kE);
      smax = fmaxf(smax, e);
      if (i < n) tmin[i * stages + t] = __fsub_rd(mn[r], e);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) smax = fmaxf(smax, __shfl_xor_sync(0xffffffffu, smax, o));
  if ((threadIdx.x & 31) == 0 && smax > 0.f)  // (non-negative floats order as their bits)
    atomicMax(reinterpret_cast<int*>(slack), __float_as_int(__fmul_ru(2.f, smax)));
}

// (1 thread) after a successful probe (and its reduce and commit): this sweep
// is no longer a measuring one; the re-vote runs again on the fresh plan
__global__ void f64s_probed_kernel(const int* probe_ok, int* flag, int* full, int* counter) {
  if (!*probe_ok) return;
  *flag = 0;
  *full = 0;
  *counter = 0;
}

}  // namespace cntgw
