// K1/K2, CNTGW_F64S: the fp64 (DMMA) half-update on locality-ordered rows
// and columns with a MEASURED block-sparse plan — the path of cold problems
// whose points have no low-dimensional locality to centre on (C5: 64/32-dim
// features, |exponent| ~ 1e6 log2 units), where the geometric tile bounds of
// the centred path (softmin_ctr.cuh) are ~1e6 log2 units wide and skip
// nothing.
//
// Same arithmetic as softmin_dmma_kernel (fp64 q_ij = -beta_j + <[x|s]_i,
// c_j> on mma.sync.m8n8k4.f64, lazily rebased MUFU.EX2 sums). Rows are
// gathered into a block in the caller-supplied order (cntgw_prep_rows_f64s)
// and the results scattered back; column records are packed in the column
// order (cntgw_prep_cols_f64s). A plan is a per-(CTA row group, column
// stage) mask derived from MEASURED stage minima, not from geometric bounds:
//   * a measuring sweep (the first of a loop, see below) walks every stage —
//     its outputs are exact — and also writes each row's minimum q over each
//     stage (tmin, fp32 rounded down). The dense measurement of a loop's
//     first sweep is the fp32 probe instead (softmin_f64s_probe.cuh) when the
//     width allows, and this kernel then walks only the probe's kept stages;
//   * every later sweep re-votes the mask from tmin and the per-stage range
//     of the column-constant shifts since the measurement (f64s_shift /
//     f64s_vote kernels, below) and walks only the needed stages (their
//     compacted list is built in shared memory, so the bulk-copy ring stays
//     dense).
// Skipped terms are below 2^-48 of their row's maximum in the sweeps (2^-64
// for the plan consumers; exact bounds, no assumption on how the potentials
// move), so the skipped mass is < m 2^-48
// of every row's sum. On the C5 law 8% of the (row group, stage) pairs are
// needed right after a measurement (tools/c5_sparsity.py).
#pragma once

#include "common.cuh"
#include "softmin.cuh"
#include "softmin_ctr.cuh"
#include "softmin_dmma.cuh"

namespace cntgw {

// Columns per stage of the measured plan, shared by the sweeps, the probes and
// the plan consumers (K4): the unit of columns the plan keeps or skips.
constexpr int f64s_stage_cols(int kd) { return kd >= 16 ? 64 : 256; }

struct F64sArgs {
  const int64_t* row_order;  // ordered position -> caller row (rows block)
  const int* replan;         // this sweep measures (writes tmin for the stages it walks)
  const int* full;           // ... and walks every stage (else only the re-vote's kept ones)
  const uint8_t* need;       // [row groups][stages] (row group = one CTA's rows)
  float* tmin;               // [n][stages] min q per row and stage (replan sweeps)
  int stages;                // mpad / TD
  const int* dotzero;        // [0] any nonzero row dot feature, [1] any nonzero column dot feature
};

// Rows block: order [n] int64 | features [n][kd] fp64 | sq [n] fp64.
__host__ __device__ inline size_t f64s_rows_bytes(int64_t n, int kd) {
  return align256(sizeof(int64_t) * n) + align256(sizeof(double) * n * kd) + align256(sizeof(double) * n);
}

__global__ void f64s_prep_rows_kernel(int kd, int sq_flag, const double* feat, int64_t ld, const double* sq,
                                      const int64_t* order, int64_t n, void* block) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  char* b = static_cast<char*>(block);
  int64_t* ord = reinterpret_cast<int64_t*>(b);
  double* f = reinterpret_cast<double*>(b + align256(sizeof(int64_t) * n));
  double* s = reinterpret_cast<double*>(b + align256(sizeof(int64_t) * n) + align256(sizeof(double) * n * kd));
  const int64_t src = order ? order[i] : i;
  ord[i] = src;
  for (int k = 0; k < kd; ++k) f[i * kd + k] = feat[src * ld + k];
  s[i] = sq_flag ? sq[src] : 0.0;
}

// Order of the points for the next loop, chosen on the device from Gamma:
// at Gamma = 0 (the product init) the cost depends on the points only through
// (s_i - t_j)^2, so the squared-coordinate order makes the plan a band; any
// other operator takes the geometric order (Morton / k-means).
__global__ void select_order_kernel(const double* gamma, int de, const int64_t* if_zero, const int64_t* otherwise,
                                    int64_t n, int64_t* out) {
  __shared__ int nonzero;
  if (threadIdx.x == 0) nonzero = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < de; k += blockDim.x)
    if (gamma[k] != 0.0) nonzero = 1;
  __syncthreads();
  const int64_t* src = nonzero ? otherwise : if_zero;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src[i];
}

// ---- the measured plan, re-voted every sweep ---------------------------------
// State (workspace, f64s_layout): from the last MEASURED sweep, each row's
// minimum q over each stage (tmin[n][stages], reduced right away to gmin =
// per (row group, stage) the smallest tmin[i][t] - Mq_i, and t*_i = the stage
// holding row i's minimum Mq_i), and c_plan, the column constants -beta_j at
// that sweep. Every later sweep sees column shifts d_j = c_j - c_plan_j; with
// [dmin_t, dmax_t] their range over stage t, for every row i of group g
//   stage-t minimum >= Mq_i + gmin[g][t] + dmin_t,
//   row minimum     <= Mq_i + dmax_{t*_i},
// so a stage with gmin[g][t] + dmin_t > max_i dmax_{t*_i} + T holds only
// terms below 2^-T of each of the group's rows' maxima and is skipped. Uniform
// drifts cancel exactly, and per-stage ranges stay narrow while the global
// spread of the shifts is large (a stage is 64-256 columns of one cluster).
// A sweep measures anew (dense, tmin rewritten) on the first sweep of a
// loop, for a new operator or lam, on a NaN record, or when the re-vote
// keeps more than CNTGW_F64S_REMEASURE of the (group, stage) pairs.

// (1 block) replan = first sweep / new key; the counter of needed pairs = 0
__global__ void f64s_begin_kernel(const cntgw_sweep_state* st, int skip, CtrPlanKey* key, const void* rows,
                                  const void* cols, int64_t n, int64_t m, int* flag, int* counter, int* full,
                                  int* sched) {
  if (skip_now(st, skip)) {  // (the loop is done: no sweep, no measurement)
    *flag = 0;
    *full = 0;
    *counter = 0;
    return;
  }
  const double lam = st ? st->lam_d : 0.0;
  const bool first = st == nullptr || st->sweep <= 1 || key->lam != lam || key->rows != rows ||
                     key->cols != cols || key->n != n || key->m != m;
  *flag = first ? 1 : 0;
  *full = first ? 1 : 0;  // a measurement over every stage (else: over the kept ones)
  *counter = 0;
  if (first) {  // a new plan: the re-measurement schedule starts over, the dot-term flags are re-detected
    sched[0] = 1;
    sched[2] = 0;
    sched[4] = sched[5] = 0;  // (= F64sPlan::dotzero)
  }
}

// one block per stage: the range of the column shifts over the stage's real
// columns (+inf / -inf when it has none: never needed, never bounds a row);
// a NaN record or planned constant forces a measurement
__global__ void __launch_bounds__(128) f64s_shift_kernel(const double* rec, int stride, int off, int64_t m,
                                                         int tile, const double* c_plan, double2* range,
                                                         int* flag, int* full, const int* gate) {
  __shared__ double smn[4], smx[4];
  if (gate && !*gate) return;
  const int64_t j0 = (int64_t)blockIdx.x * tile;
  double mn = CUDART_INF, mx = -CUDART_INF;
  bool bad = false;
  for (int u = threadIdx.x; u < tile; u += blockDim.x) {
    const int64_t j = j0 + u;
    if (j >= m) break;
    const double c = rec[j * stride + off], cp = c_plan[j];
    bad |= (c != c) || (cp != cp);
    if (c == cp && !(c < CUDART_INF && c > -CUDART_INF)) continue;  // zero weight: no term at all
    const double d = c == cp ? 0.0 : c - cp;
    mn = fmin(mn, d);
    mx = fmax(mx, d);
  }
  if (bad) {
    atomicOr(flag, 1);
    atomicOr(full, 1);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    smn[threadIdx.x >> 5] = mn;
    smx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mn = fmin(mn, smn[w]);
      mx = fmax(mx, smx[w]);
    }
    range[blockIdx.x] = make_double2(mn, mx);
  }
}

// After a measuring sweep (one block per row group of `grows` rows): each
// row's minimum Mq_i and argmin stage t*_i over the stage minima, and per
// (group, stage) the smallest relative minimum gmin = min_i (tmin[i][t] -
// Mq_i) (rounded down). The per-sweep re-vote reads only gmin and t*, not the
// [n][stages] tmin (16 GB at N = M = 2^20). A PARTIAL measurement (re-measure
// within a loop) walked only the stages the re-vote kept; a stage it skipped
// keeps the re-vote's lower bound of its minimum, Mq_i(old) + gmin(old) +
// dmin_t (valid in the current frame, and > the row minimum + T), so the new
// plan stays a plan of lower bounds.
constexpr int kF64sListMax = 16384;  // walked-stage list held in shared memory (32 KB)
__global__ void __launch_bounds__(256) f64s_reduce_kernel(const int* flag, const int* full, const float* tmin,
                                                          const uint8_t* need, const double2* range, int64_t n,
                                                          int stages, int grows, float* gmin, int* tstar,
                                                          double* rowmin, float slack_c, const float* slack_p) {
  if (!*flag) return;
  const bool all = *full != 0;
  // dynamic: [grows] new row minima | [grows] previous ones | [stages] uint16 walked-stage list
  extern __shared__ double rsh[];
  __shared__ int wsum[8];
  __shared__ int nwalk_s;
  __shared__ double dmin_s;
  double* rnew = rsh;
  double* rold = rsh + grows;
  uint16_t* walk = reinterpret_cast<uint16_t*>(rsh + 2 * grows);
  const int64_t r0 = (int64_t)blockIdx.x * grows;
  const uint8_t* nd = need + (int64_t)blockIdx.x * stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // a partial measurement walked only the kept stages (a few per group): their
  // compacted list, so that the per-row scans below do not visit every stage
  const bool listed = !all && stages <= kF64sListMax;
  if (listed) {
    const int per = (stages + (int)blockDim.x - 1) / (int)blockDim.x;
    const int first = (int)threadIdx.x * per;
    int cnt = 0;
    for (int u = 0; u < per; ++u)
      if (first + u < stages && nd[first + u]) ++cnt;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int pos = incl - cnt;
    for (int w = 0; w < warp; ++w) pos += wsum[w];
    for (int u = 0; u < per; ++u)
      if (first + u < stages && nd[first + u]) walk[pos++] = (uint16_t)(first + u);
    if (threadIdx.x == blockDim.x - 1) nwalk_s = pos;
    __syncthreads();
  }
  const int nwalk = listed ? nwalk_s : stages;
  for (int r = warp; r < grows; r += nw) {
    float mn = CUDART_INF_F;
    int at = 0;
    if (r0 + r < n)
      for (int k = lane; k < nwalk; k += 32) {
        const int t = listed ? (int)walk[k] : k;
        if (!all && !listed && !nd[t]) continue;
        const float v = tmin[(r0 + r) * stages + t];
        if (v < mn) {
          mn = v;
          at = t;
        }
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, mn, o);
      const int a2 = __shfl_xor_sync(0xffffffffu, at, o);
      if (m2 < mn || (m2 == mn && a2 < at)) {
        mn = m2;
        at = a2;
      }
    }
    if (lane == 0) {
      rnew[r] = mn;
      rold[r] = r0 + r < n ? rowmin[r0 + r] : 0.0;
      if (r0 + r < n) tstar[r0 + r] = at;
    }
  }
  __syncthreads();
  // the stage minima were rounded down to fp32: the rows' true minima can sit
  // up to an ulp of |Mq| above rnew, so gmin is lowered by two ulps of the
  // group's largest |Mq| (keeps every bound of the vote conservative)
  double amax = 0.0;
  for (int r = 0; r < grows && r0 + r < n; ++r)
    if (fabs(rnew[r]) < CUDART_INF) amax = fmax(amax, fabs(rnew[r]));
  const double allow = amax * 0x1p-22 + (slack_p ? (double)*slack_p : (double)slack_c);
  // a stage the measurement skipped keeps the re-vote's bound: over the rows,
  // min (rold + gold - rnew) = gold + min (rold - rnew), the same for every such stage
  if (warp == 0) {
    double dm = CUDART_INF;
    for (int r = lane; r < grows && r0 + r < n; r += 32) dm = fmin(dm, rold[r] - rnew[r]);  // (NaN dropped)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dm = fmin(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    if (lane == 0) dmin_s = dm;
  }
  __syncthreads();
  const double dmin = dmin_s;
  for (int t = threadIdx.x; t < stages; t += blockDim.x) {
    double g = CUDART_INF;
    if (all || nd[t]) {
      for (int r = 0; r < grows && r0 + r < n; ++r)
        g = fmin(g, (double)tmin[(r0 + r) * stages + t] - rnew[r]);  // (inf - inf: an empty row, NaN dropped)
    } else {
      g = dmin + ((double)gmin[(int64_t)blockIdx.x * stages + t] + range[t].x);
    }
    gmin[(int64_t)blockIdx.x * stages + t] = __double2float_rd(g - allow);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < grows; r += blockDim.x)
    if (r0 + r < n) rowmin[r0 + r] = rnew[r];
}

// One block per row group (skipped on a measuring sweep). For a row i of the
// group, its current stage-t minimum is >= Mq_i + gmin[g][t] + dmin_t and
// its current row minimum <= Mq_i + dmax_{t*_i} (the stage that held its
// minimum at the measurement), so stage t can hold a term within T of the
// row's maximum only if gmin[g][t] + dmin_t <= D_g + T, D_g = max over the
// group's rows of dmax_{t*_i}. Counts the needed pairs.
__global__ void __launch_bounds__(256) f64s_vote_kernel(const int* flag, const float* gmin, const int* tstar,
                                                        const double2* range, int64_t n, int stages, int grows,
                                                        double T, uint8_t* need, int* counter, const int* gate) {
  if (*flag || (gate && !*gate)) return;
  __shared__ double dg_s[8];
  const int64_t r0 = (int64_t)blockIdx.x * grows;
  double dg = -CUDART_INF;
  for (int r = threadIdx.x; r < grows; r += blockDim.x)
    if (r0 + r < n) dg = fmax(dg, range[tstar[r0 + r]].y);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dg = fmax(dg, __shfl_xor_sync(0xffffffffu, dg, o));
  if ((threadIdx.x & 31) == 0) dg_s[threadIdx.x >> 5] = dg;
  __syncthreads();
  dg = dg_s[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) dg = fmax(dg, dg_s[w]);
  const double lim = dg + T;  // (gmin already carries the fp32 rounding allowance)
  int cnt = 0;
  for (int t = threadIdx.x; t < stages; t += blockDim.x) {
    const uint8_t v = !((double)gmin[(int64_t)blockIdx.x * stages + t] + range[t].x > lim) ? 1 : 0;
    need[(int64_t)blockIdx.x * stages + t] = v;
    cnt += v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(counter, cnt);
}

// (1 thread) measure anew when the re-vote kept too much, and on an adaptive
// schedule while it keeps more than 0.2%: a plan measured early in a loop
// reflects transient potentials, and the re-vote only ever loosens it. Within
// a loop a measurement walks only the kept stages (~1.3-2 sparse sweeps); the
// first one of a loop is dense (or the fp32 probe). The first vote after a
// measurement tells whether it paid: if it cut the kept pairs by more than 5%
// the interval to the next measurement halves (down to the very next sweep),
// otherwise it doubles (sched: interval, kept pairs before the last
// measurement, pending flag, sweep of the last measurement).
__global__ void f64s_decide_kernel(const cntgw_sweep_state* st, int* flag, const int* counter,
                                   int* next_measure, int64_t pairs, double max_frac, int schedule,
                                   const int* gate, int skip, int* sched, int* full, int reprobe) {
  if (*flag || (gate && !*gate) || skip_now(st, skip)) return;
  const double kept = (double)*counter / (double)pairs;
  const int sweep = st ? st->sweep : 0;
  if (schedule && sched[2]) {
    sched[2] = 0;
    const int before = sched[1];
    const bool paid = before <= 0 || (double)(before - *counter) > 0.05 * (double)before;
    const int prev = sched[0] > 1 ? sched[0] : 1;
    sched[0] = paid ? (prev > 2 ? prev / 2 : 1) : (prev < 32768 ? 2 * prev : prev);
    *next_measure = sched[3] + sched[0];
  }
  if (kept > max_frac || (schedule && sweep >= *next_measure && kept > 0.002)) *flag = 1;
  // the re-vote lost the plan (potentials moved far, e.g. the second sweep from
  // zero potentials keeps 99%): where the fp32 probe exists, a fresh probe
  // (0.3 dense sweeps) beats walking that much in fp64
  if (reprobe && schedule && !gate && kept > max_frac) *full = 1;
}

// diagnostics: needed (group, stage) pairs of the current mask and the flag
__global__ void f64s_density_kernel(const uint8_t* need, int64_t pairs, const int* flag, const int* probed,
                                    int64_t* out) {
  int64_t c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pairs; i += (int64_t)gridDim.x * blockDim.x)
    c += need[i] ? 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(reinterpret_cast<unsigned long long*>(out), (unsigned long long)c);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[1] = pairs;
    out[2] = *flag + (probed ? 2 * *probed : 0);
  }
}

// after a measuring sweep: the plan's reference constants and key
__global__ void __launch_bounds__(1024) f64s_commit_kernel(const int* flag, const cntgw_sweep_state* st,
                                                           const double* rec, int stride, int off, int64_t mpad,
                                                           double* c_plan, CtrPlanKey* key, const void* rows,
                                                           const void* cols, int64_t n, int64_t m,
                                                           int* next_measure, const int* counter, int* sched) {
  if (!*flag) return;
  for (int64_t j = threadIdx.x; j < mpad; j += blockDim.x) c_plan[j] = rec[j * stride + off];
  if (threadIdx.x == 0) {
    const int sweep = st ? st->sweep : 0;
    // the next vote decides when to measure again (f64s_decide_kernel)
    *next_measure = sweep + 1;
    sched[1] = *counter;  // kept pairs of the vote this measurement followed (0: a first, dense one)
    sched[2] = 1;
    sched[3] = sweep;
    key->lam = st ? st->lam_d : 0.0;
    key->rows = rows;
    key->cols = cols;
    key->n = n;
    key->m = m;
  }
}

// The dot term <x_i, c_j> vanishes when one side's dot features are all zero:
// at Gamma = 0 (the product coupling every solve starts from) the operator's
// features X Gamma are, so the whole first outer step runs on q_ij = -beta_j
// + s_i c_sj alone. This kernel records, per call, whether any row or any
// column dot feature is nonzero (blocks leave early once a side is known to
// be nonzero); the sweep then takes one DFMA per pair instead of the DMMA
// k-steps (C5: 9 k-steps -> 1 FMA, first outer step 1.42 -> 1.0 s). Runs on
// the sweeps that measure over every stage (*gate: the first of a loop, where
// f64s_begin_kernel cleared the flags; the operator is fixed within a loop).
__global__ void f64s_dotzero_kernel(const int* gate, const void* rows_block, int64_t n, int kd, const double* rec,
                                    int stride, int64_t m, int* flags) {
  if (!*gate) return;
  const char* rb = static_cast<const char*>(rows_block);
  const double* rf = reinterpret_cast<const double*>(rb + align256(sizeof(int64_t) * n));
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  if (!flags[0]) {
    bool nz = false;
    for (int64_t e = tid; e < n * kd && !nz; e += nth) nz = rf[e] != 0.0;
    if (nz) flags[0] = 1;
  }
  if (!flags[1]) {
    bool nz = false;
    for (int64_t j = tid; j < m && !nz; j += nth)
      for (int k = 0; k < kd; ++k) nz |= rec[j * stride + k] != 0.0;
    if (nz) flags[1] = 1;
  }
}

// q of RG row groups x NT 8-column tiles in the DMMA accumulator layout (lane
// (lr, lk): row lr of each group, columns 2 lk and 2 lk + 1 of each tile) when
// the dot term vanishes: -beta_j + s_i c_sj
template <int KD, int SQ, int RG, int NT>
__device__ __forceinline__ void sq_scores(const double* __restrict__ tile, int ct, int lk, const double (&as)[RG],
                                          double (&q)[RG][NT][2]) {
  using L = ColLayout<double, KD, SQ>;
#pragma unroll
  for (int u = 0; u < NT; ++u) {
    const double* cc = tile + (ct + 8 * u + 2 * lk) * L::kStride;
    const double b0 = cc[KD], b1 = cc[L::kStride + KD];
    const double beta0 = cc[L::kBeta], beta1 = cc[L::kStride + L::kBeta];
#pragma unroll
    for (int rg = 0; rg < RG; ++rg) {
      q[rg][u][0] = fma(as[rg], b0, beta0);
      q[rg][u][1] = fma(as[rg], b1, beta1);
    }
  }
}

// dmma_consume plus the step's minimum q per row group, tracked on the fp32
// exponent arguments x = mq - q (FMNMX on the ALU, not a DMNMX per term on
// the FP64 pipe): tm = min(tm, mq - max x), one fp64 op per row group and
// step. The fp32 argument (truncated, ~2^-18 relative at 32-48 log2 units)
// is exact enough for a plan whose margins are 64 log2 units.
template <int RG, int NT>
__device__ __forceinline__ void dmma_consume_min(const double (&q)[RG][NT][2], double (&mq)[RG], double (&S)[RG],
                                                 float (&T)[RG], double (&tm)[RG]) {
  float gsum[RG], xmax[RG];
#pragma unroll
  for (int rg = 0; rg < RG; ++rg) {
    float2 acc = f2(0.f, 0.f);
    float xm = -CUDART_INF_F;
#pragma unroll
    for (int u = 0; u < NT; ++u) {
      const float2 x = f2(f64_to_f32_fast(mq[rg] - q[rg][u][0]), f64_to_f32_fast(mq[rg] - q[rg][u][1]));
      xm = fmaxf(xm, fmaxf(x.x, x.y));
      acc = add2(acc, f2(ex2(x.x), ex2(x.y)));
    }
    gsum[rg] = acc.x + acc.y;
    xmax[rg] = xm;
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
      tm[rg] = fmin(tm[rg], qmin);
    } else {
      tm[rg] = fmin(tm[rg], mq[rg] - (double)xmax[rg]);
    }
    T[rg] += gsum[rg];
  }
}

template <int KD, int SQ, int RG, int NT, int TILE, int MINB, int NS = 2>
__global__ void __launch_bounds__(128, MINB) softmin_f64s_kernel(const SoftminArgs a, const F64sArgs p) {
  using L = ColLayout<double, KD, SQ>;
  constexpr int KS = (KD + SQ + 3) / 4;
  static_assert(4 * KS <= L::kStride, "column record must cover the padded k4 steps");
  constexpr int kStage = TILE * L::kStride;
  constexpr int kMaxList = 4096;  // stages per chunk held in the compacted list
  extern __shared__ __align__(128) double smem_d[];
  __shared__ uint64_t full_bar[NS], empty_bar[NS];
  __shared__ int16_t list[kMaxList];
  __shared__ int nlist;
  if (skip_now(a.st, a.skip)) return;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lr = lane >> 2, lk = lane & 3;
  const int chunk = blockIdx.y;
  const int64_t wrow = (int64_t)blockIdx.x * (32 * RG) + warp * (8 * RG);
  const char* rb = static_cast<const char*>(a.row_feat);
  const double* rf = reinterpret_cast<const double*>(rb + align256(sizeof(int64_t) * a.n));
  const double* rs = reinterpret_cast<const double*>(rb + align256(sizeof(int64_t) * a.n) +
                                                     align256(sizeof(double) * a.n * KD));
  const bool replan = *p.replan != 0, full = *p.full != 0;
  const bool dotzero = SQ && (p.dotzero[0] == 0 || p.dotzero[1] == 0);

  double afr[RG][KS];
  double as_row[RG];
  double mq[RG], S[RG];
#pragma unroll
  for (int rg = 0; rg < RG; ++rg) {
    const int64_t i = wrow + 8 * rg + lr;
    const bool ok = i < a.n;
    as_row[rg] = SQ && ok ? rs[i] : 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = 4 * ks + lk;
      double v = 0.0;
      if (k < KD) v = ok ? rf[i * KD + k] : 0.0;
      else if (SQ && k == KD) v = ok ? rs[i] : 0.0;
      afr[rg][ks] = v;
    }
    mq[rg] = kStartQ;
    S[rg] = 0.0;
  }

  const int64_t c0 = (int64_t)chunk * a.chunk_cols;
  const int64_t mpad = (a.m + kColTile - 1) / kColTile * kColTile;
  const int ntiles = (int)((min(c0 + a.chunk_cols, mpad) - c0) / TILE);
  const int t0 = (int)(c0 / TILE);  // global stage index of the chunk's first stage
  // compacted list of the stages this CTA walks (all of them on a full
  // measuring sweep), in increasing order: every thread takes a contiguous run
  // of <= 32 stages (its mask bytes are independent loads, one L2 round trip
  // for the CTA), and a block prefix sum of the counts places the runs
  {
    __shared__ int wsum[4];
    const uint8_t* nd = p.need + (int64_t)blockIdx.x * p.stages + t0;
    const int per = (ntiles + (int)blockDim.x - 1) / (int)blockDim.x;  // <= kMaxList / 128
    const int first = (int)threadIdx.x * per;
    uint32_t mask = 0;
#pragma unroll 8
    for (int u = 0; u < per; ++u) {
      const int t = first + u;
      if (t < ntiles && (full || nd[t])) mask |= 1u << u;
    }
    const int cnt = __popc(mask);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int pos = incl - cnt;
    for (int w = 0; w < warp; ++w) pos += wsum[w];
    for (uint32_t b = mask; b; b &= b - 1) list[pos++] = (int16_t)(first + __ffs(b) - 1);
    if (threadIdx.x == blockDim.x - 1) nlist = pos;
    __syncthreads();
  }
  const int nt = nlist;
  const uint32_t bytes = kStage * sizeof(double);
  const double* src = static_cast<const double*>(a.col_rec) + c0 * L::kStride;
  StageRing<NS> ring{full_bar, empty_bar};
  ring.init(4);
  if (threadIdx.x == 0)
    for (int st = 0; st < NS && st < nt; ++st)
      ring.load(smem_d + st * kStage, src + (int64_t)list[st] * kStage, bytes, st);
  for (int k = 0; k < nt; ++k) {
    if (threadIdx.x == 0) {
      const int r = ring.refill_slot(k, nt);
      if (r >= 0) ring.load(smem_d + (r % NS) * kStage, src + (int64_t)list[r] * kStage, bytes, r);
    }
    ring.wait_full(k);
    const double* tile = smem_d + (k % NS) * kStage;
    float T[RG];
    double tm[RG];
#pragma unroll
    for (int rg = 0; rg < RG; ++rg) {
      T[rg] = 0.f;
      tm[rg] = CUDART_INF;
    }
#pragma unroll 1
    for (int ct = 0; ct < TILE; ct += 8 * NT) {
      double q[RG][NT][2];
      if (dotzero) sq_scores<KD, SQ, RG, NT>(tile, ct, lk, as_row, q);
      else dmma_scores<KD, SQ, RG, NT, KS>(tile, ct, lr, lk, afr, q);
      if (replan)  // (the measuring sweep: stage minima ride on the exponent arguments)
        dmma_consume_min<RG, NT>(q, mq, S, T, tm);
      else
        dmma_consume<RG, NT>(q, mq, S, T);
    }
#pragma unroll
    for (int rg = 0; rg < RG; ++rg) S[rg] += f32_to_f64_alu(T[rg]);
    if (replan) {  // the rows' minimum q over this stage (quad = the row's 4 lanes)
#pragma unroll
      for (int rg = 0; rg < RG; ++rg) {
        double v = tm[rg];
        v = fmin(v, __shfl_xor_sync(0xffffffffu, v, 1));
        v = fmin(v, __shfl_xor_sync(0xffffffffu, v, 2));
        const int64_t i = wrow + 8 * rg + lr;
        if (lk == 0 && i < a.n)  // (- 2^-10: the fp32 exponent arguments were truncated)
          p.tmin[i * p.stages + t0 + list[k]] = __double2float_rd(v - 0x1p-10);
      }
    }
    ring.release(k);
  }

  const double lam = a.st->lam_d, inv_lam = 1.0 / lam;
#pragma unroll
  for (int rg = 0; rg < RG; ++rg) {
    double m = -mq[rg], s = S[rg];
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
      softmin_store(a, chunk, p.row_order[i], m - (SQ ? lam * si * si : 0.0), s, inv_lam);
    }
  }
}

}  // namespace cntgw
