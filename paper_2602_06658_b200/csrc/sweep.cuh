// K3: device-side Sinkhorn sweep control (sinkhorn.py:191-258).
//
// The loop state lives in device memory so that a whole sweep (and a chunk
// of sweeps) can be enqueued or CUDA-graph-captured without a host round
// trip; every sweep kernel returns immediately once `done` is set, which is
// how a captured chunk early-exits after a threshold break.
#pragma once

#include "common.cuh"

namespace cntgw {

constexpr int kGapThreads = 256;
constexpr int kGapMaxBlocks = 296;

static __global__ void sweep_init_kernel(cntgw_sweep_state* st, double eps, double anneal_from,
                                  double threshold, int max_sweeps, int mode) {
  st->eps = eps;
  st->anneal_from = anneal_from;
  st->threshold = threshold;
  st->eps_n = eps;
  st->gap_r = 0.0;
  st->gap_c = 0.0;
  st->lam_d = kLog2eD / eps;
  st->sqrt_lam_d = sqrt(st->lam_d);
  st->lam = (float)st->lam_d;
  st->sqrt_lam = (float)st->sqrt_lam_d;
  st->max_sweeps = max_sweeps;
  st->mode = mode;
  st->sweep = 0;
  st->applied = 0;
  st->done = 0;
  st->converged = threshold > 0.0 ? 0 : 1;  // fixed budgets report converged (sinkhorn.py:221)
  st->check = 0;
}

// eps_n = max(anneal_from / sqrt(n), eps) (sinkhorn.py:223-226), in fp64 like the reference
static __global__ void sweep_begin_kernel(cntgw_sweep_state* st) {
  if (st->done) return;
  const int k = st->sweep + 1;
  if (k > st->max_sweeps) {
    st->done = 1;
    return;
  }
  double e = st->eps;
  if (st->anneal_from > 0.0) e = fmax(st->anneal_from / sqrt((double)k), st->eps);
  st->eps_n = e;
  st->lam_d = kLog2eD / e;
  st->sqrt_lam_d = sqrt(st->lam_d);
  st->lam = (float)st->lam_d;
  st->sqrt_lam = (float)st->sqrt_lam_d;
  st->check = (st->threshold > 0.0) && (e == st->eps);  // sinkhorn.py:228
  st->sweep = k;
}

// sum_i w_i^2 |exp(min((pot_i - tent_i)/eps_n, 700)) - 1|  (sinkhorn.py:179-188)
static __global__ void sweep_gap_kernel(const cntgw_sweep_state* st, const double* w,
                                        const double* pot, const double* tent, int64_t n,
                                        double* partials) {
  __shared__ double red[32];
  if (st->done || !st->check) return;
  const double eps = st->eps_n;
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double r = fmin((pot[i] - tent[i]) / eps, 700.0);
    acc += w[i] * w[i] * fabs(exp(r) - 1.0);
  }
  const double t = block_sum_f64(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

__host__ __device__ inline int gap_blocks(int64_t n) {
  int64_t b = (n + kGapThreads - 1) / kGapThreads;
  return (int)(b < kGapMaxBlocks ? (b < 1 ? 1 : b) : kGapMaxBlocks);
}

// break decision (sinkhorn.py:232-237, 242-248) and the applied counter (:251)
static __global__ void sweep_finish_kernel(cntgw_sweep_state* st, const double* pr, int nbr,
                                    const double* pc, int nbc) {
  if (st->done) return;
  if (st->check) {
    double gr = 0.0, gc = 0.0;
    for (int i = 0; i < nbr; ++i) gr += pr[i];
    if (pc)
      for (int i = 0; i < nbc; ++i) gc += pc[i];
    st->gap_r = gr;
    st->gap_c = gc;
    const bool brk = st->mode == 1 ? (gr < st->threshold && gc < st->threshold) : (gr < st->threshold);
    if (brk) {
      st->converged = 1;
      st->done = 1;
      return;
    }
  }
  st->applied = st->sweep;
}

// symmetrized: pot <- (pot + tent)/2 (sinkhorn.py:238-239); standard: pot <- tent (:249)
static __global__ void sweep_apply_kernel(const cntgw_sweep_state* st, double* pot,
                                          const double* tent, int64_t n, int average) {
  if (st->done) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    pot[i] = average ? 0.5 * (pot[i] + tent[i]) : tent[i];
}

}  // namespace cntgw
