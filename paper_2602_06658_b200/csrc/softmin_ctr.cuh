// K1/K2, CNTGW_F32C: the half-update of cold problems with fp32 pair
// arithmetic on locality-ordered tiles.
//
// Same reference arithmetic as softmin.cuh (`_softmin`, sinkhorn.py:166-176,
// over SquaredEuclideanCost, :59-109). In the expanded-square parametrisation
// of the fp64 path, with row coordinates X_i = [x_i | s_i] and column records
// Zr_j = [-2 lam z_j | -2 lam s_j], c_j = -(lam (pot_j - s_j^2) + log2 w_j),
//     q_ij = c_j + <X_i, Zr_j>        (t_ij = -q_ij - lam s_i^2).
// On the cold C4/C5 laws |q| reaches 1e6-1e7 log2 units, so the fp32 paths
// lose 0.06-1 log2 units per term and the default is fp64 (DMMA, ~half the
// MUFU roof). Here rows and columns are visited in a locality order (Morton
// codes of the point coordinates, computed once per solve) and each 128-row
// group I and 256-column tile J is centred: X_i = Xc_I + dX_i, Zr_j = Zc_J +
// dZ_j, so that exactly
//     q_ij = A_j^I + B_i^J + <dX_i, dZ_j>,
//     A_j^I = c_j + <Xc_I, Zr_j>,   B_i^J = <dX_i, Zc_J>.
// A and B carry the large magnitudes and are formed in fp64 once per (group,
// column) and (row, tile) — 1/128 and 1/256 of the pair count; the pair term
// <dX, dZ> is bounded by 2 lam |dx| |dz| over a tile (a few 1e3 log2 units at
// N = 2^20 on the C4 law) and runs on the fp32 FFMA2 path of softmin.cuh. Per
// tile the group biases a_j = fp32(A_j^I - min_j A_j^I) are written to shared
// memory, and the row's fp64 reference M_i enters the tile as the fp32 offset
// fp32(M_i - min A - B_i). Rows are processed in locality order and their
// results scattered back to the caller's order. A (group, tile) pair whose
// pair-term bound exceeds ctr_limit runs in fp64 in the same kernel, and a
// planning pass (ctr_plan_kernel, below) lets the sweep skip the tiles that
// cannot hold a term within 2^-64 of any of the CTA's rows' maxima.
#pragma once

#include "common.cuh"
#include "softmin.cuh"

namespace cntgw {

constexpr int kCtrRowGroup = 128;  // rows per centring group (one per row of a thread)

// Column block (prep_cols_ctr): rec64 [mpad][KX+1] fp64 [Zr | c] | rec32
// [mpad][KX] fp32 dZ | tctr [mpad/256][KX+1] fp64 tile centres + radius
// max_j |dZ_j|. Row block (prep_rows_ctr): order [n] int64 | ctr
// [groups][KX+1] fp64 group centres + radius max_i |dX_i| |
// dx64 [npad][KX] fp64 | dx32 [npad][KX] fp32, npad = groups * 128.
struct CtrCols {
  const double* rec64;
  const float* rec32;
  const double* tctr;
};
struct CtrRows {
  const int64_t* order;
  const double* ctr;
  const double* dx64;
  const float* dx32;
};

__host__ __device__ inline int64_t ctr_groups(int64_t n) { return (n + kCtrRowGroup - 1) / kCtrRowGroup; }
__host__ __device__ inline size_t align256(size_t b) { return (b + 255) / 256 * 256; }

__host__ __device__ inline size_t ctr_cols_bytes(int64_t mpad, int kx) {
  return align256(sizeof(double) * mpad * (kx + 1)) + align256(sizeof(float) * mpad * kx) +
         align256(sizeof(double) * (mpad / kColTile) * (kx + 1));
}
// + the tcgen05 B' tiles of the kx = 4 block (softmin_ctr_tc.cuh): 16 floats per column
__host__ __device__ inline size_t ctr_cols_bytes_all(int64_t mpad, int kx) {
  return ctr_cols_bytes(mpad, kx) + (kx == 4 ? sizeof(float) * 16 * (size_t)mpad : 0);
}
__host__ __device__ inline size_t ctr_rows_bytes(int64_t n, int kx) {
  const int64_t np = ctr_groups(n) * kCtrRowGroup;
  return align256(sizeof(int64_t) * n) + align256(sizeof(double) * ctr_groups(n) * (kx + 1)) +
         align256(sizeof(double) * np * kx) + align256(sizeof(float) * np * kx);
}
template <typename P>
__host__ __device__ inline CtrCols ctr_cols_view(P base, int64_t mpad, int kx) {
  const char* b = (const char*)base;
  CtrCols c;
  c.rec64 = (const double*)b;
  b += align256(sizeof(double) * mpad * (kx + 1));
  c.rec32 = (const float*)b;
  b += align256(sizeof(float) * mpad * kx);
  c.tctr = (const double*)b;
  return c;
}
template <typename P>
__host__ __device__ inline CtrRows ctr_rows_view(P base, int64_t n, int kx) {
  const int64_t g = ctr_groups(n), np = g * kCtrRowGroup;
  const char* b = (const char*)base;
  CtrRows r;
  r.order = (const int64_t*)b;
  b += align256(sizeof(int64_t) * n);
  r.ctr = (const double*)b;
  b += align256(sizeof(double) * g * (kx + 1));
  r.dx64 = (const double*)b;
  b += align256(sizeof(double) * np * kx);
  r.dx32 = (const float*)b;
  return r;
}

// ---- packing ------------------------------------------------------------------
// One block per 256-column tile: gather the tile's columns in locality order,
// build [Zr | c] in fp64, the tile centre (mean of the real columns), dZ in fp32.
template <int KX>
__global__ void __launch_bounds__(kColTile) prep_cols_ctr_kernel(
    const cntgw_sweep_state* st, int kd, int sq_flag, const double* feat, int64_t ld,
    const double* sq, const double* pot, const double* log2w, const int64_t* order, int64_t m,
    int64_t mpad, void* block) {
  __shared__ double red[KX][kColTile / 32];
  __shared__ double cnt_s[kColTile / 32];
  const int64_t j = (int64_t)blockIdx.x * kColTile + threadIdx.x;
  const double lam = st->lam_d;
  double zr[KX], c = kPadQ;
  const bool ok = j < m;
#pragma unroll
  for (int k = 0; k < KX; ++k) zr[k] = 0.0;
  if (ok) {
    const int64_t src = order ? order[j] : j;
    const double sj = sq_flag ? sq[src] : 0.0;
#pragma unroll
    for (int k = 0; k < KX; ++k)
      zr[k] = k < kd ? -2.0 * lam * feat[src * ld + k] : (sq_flag && k == kd ? -2.0 * lam * sj : 0.0);
    c = -(lam * (pot ? pot[src] : 0.0) + log2w[src] - lam * sj * sj);
  }
  // tile centre = mean of the real columns (fixed-order block reduction)
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  double cnt = ok ? 1.0 : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
  if (l == 0) cnt_s[w] = cnt;
#pragma unroll
  for (int k = 0; k < KX; ++k) {
    double v = zr[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (l == 0) red[k][w] = v;
  }
  __syncthreads();
  double tc[KX];
  double tot = 0.0;
  for (int q = 0; q < kColTile / 32; ++q) tot += cnt_s[q];
#pragma unroll
  for (int k = 0; k < KX; ++k) {
    double s = 0.0;
    for (int q = 0; q < kColTile / 32; ++q) s += red[k][q];
    tc[k] = s / tot;  // every tile holds >= 1 real column (m padded to 256)
  }
  const CtrCols cv = ctr_cols_view(block, mpad, KX);
  double* rec64 = const_cast<double*>(cv.rec64) + j * (KX + 1);
  float* rec32 = const_cast<float*>(cv.rec32) + j * KX;
  double r2 = 0.0;
#pragma unroll
  for (int k = 0; k < KX; ++k) {
    const double d = ok ? zr[k] - tc[k] : 0.0;
    rec64[k] = zr[k];
    rec32[k] = (float)d;
    r2 = fma(d, d, r2);
  }
  rec64[KX] = c;
  double* tcj = const_cast<double*>(cv.tctr) + (int64_t)blockIdx.x * (KX + 1);
  if (threadIdx.x < KX) tcj[threadIdx.x] = tc[threadIdx.x];
  // tile radius max_j |dZ_j| (the per-tile fp32 error bound, with the group radius)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r2 = fmax(r2, __shfl_xor_sync(0xffffffffu, r2, o));
  __syncthreads();  // red[] reads above are done
  if (l == 0) red[0][w] = r2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m2 = 0.0;
    for (int q = 0; q < kColTile / 32; ++q) m2 = fmax(m2, red[0][q]);
    tcj[KX] = sqrt(m2);
  }
}

// One block per 128-row group: X_i = [x | s] in locality order, the group
// centre (mean of the real rows), dX in fp64 and fp32.
template <int KX>
__global__ void __launch_bounds__(kCtrRowGroup) prep_rows_ctr_kernel(
    int kd, int sq_flag, const double* feat, int64_t ld, const double* sq, const int64_t* order,
    int64_t n, void* block) {
  __shared__ double red[KX][kCtrRowGroup / 32];
  __shared__ double cnt_s[kCtrRowGroup / 32];
  const int64_t i = (int64_t)blockIdx.x * kCtrRowGroup + threadIdx.x;
  const bool ok = i < n;
  double x[KX];
#pragma unroll
  for (int k = 0; k < KX; ++k) x[k] = 0.0;
  int64_t src = i;
  if (ok) {
    src = order ? order[i] : i;
#pragma unroll
    for (int k = 0; k < KX; ++k)
      x[k] = k < kd ? feat[src * ld + k] : (sq_flag && k == kd ? sq[src] : 0.0);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  double cnt = ok ? 1.0 : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
  if (l == 0) cnt_s[w] = cnt;
#pragma unroll
  for (int k = 0; k < KX; ++k) {
    double v = x[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (l == 0) red[k][w] = v;
  }
  __syncthreads();
  double tot = 0.0;
  for (int q = 0; q < kCtrRowGroup / 32; ++q) tot += cnt_s[q];
  const CtrRows rv = ctr_rows_view(block, n, KX);
  double gc[KX];
#pragma unroll
  for (int k = 0; k < KX; ++k) {
    double s = 0.0;
    for (int q = 0; q < kCtrRowGroup / 32; ++q) s += red[k][q];
    gc[k] = s / tot;
  }
  double* gcj = const_cast<double*>(rv.ctr) + (int64_t)blockIdx.x * (KX + 1);
  if (threadIdx.x < KX) gcj[threadIdx.x] = gc[threadIdx.x];
  if (ok) const_cast<int64_t*>(rv.order)[i] = src;
  double* d64 = const_cast<double*>(rv.dx64) + i * KX;
  float* d32 = const_cast<float*>(rv.dx32) + i * KX;
  double r2 = 0.0;
#pragma unroll
  for (int k = 0; k < KX; ++k) {
    const double d = ok ? x[k] - gc[k] : 0.0;
    d64[k] = d;
    d32[k] = (float)d;
    r2 = fma(d, d, r2);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r2 = fmax(r2, __shfl_xor_sync(0xffffffffu, r2, o));
  __syncthreads();
  if (l == 0) red[0][w] = r2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m2 = 0.0;
    for (int q = 0; q < kCtrRowGroup / 32; ++q) m2 = fmax(m2, red[0][q]);
    gcj[KX] = sqrt(m2);
  }
}

// ---- streaming kernel -----------------------------------------------------------
// One shared-memory tile: per group of G columns, the fp32 pair terms
// <dX_i, dZ_j> start from the per-(row group, column) bias and feed the same
// lazily rebased MUFU.EX2 sums as softmin_tile_f32.
// POLY: row pairs (of the first column of each group) whose exp2 runs on the
// FMA pipe (exp2_poly2) instead of MUFU, balancing the two pipes.
template <int KX, int R, int G, int POLY, int PM = (1 << (R / 2)) - 1>
__device__ __forceinline__ void softmin_tile_ctr(const float* __restrict__ rec,
                                                 const float* __restrict__ bias,
                                                 const float2 (&x2)[R / 2][KX], float (&mq)[R],
                                                 double (&S)[R]) {
  constexpr int P = R / 2;
  float2 T[P];
#pragma unroll
  for (int p = 0; p < P; ++p) T[p] = f2(0.f, 0.f);
#pragma unroll 1
  for (int j = 0; j < kColTile; j += G) {
    float2 q[P][G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float c[KX];
      const float4* r4 = reinterpret_cast<const float4*>(rec + (j + g) * KX);
#pragma unroll
      for (int v = 0; v < KX / 4; ++v) {
        const float4 t = r4[v];
        c[4 * v + 0] = t.x;
        c[4 * v + 1] = t.y;
        c[4 * v + 2] = t.z;
        c[4 * v + 3] = t.w;
      }
      float bv[R];
      const float4* b4 = reinterpret_cast<const float4*>(bias + (j + g) * R);
#pragma unroll
      for (int v = 0; v < R / 4; ++v) {
        const float4 t = b4[v];
        bv[4 * v + 0] = t.x;
        bv[4 * v + 1] = t.y;
        bv[4 * v + 2] = t.z;
        bv[4 * v + 3] = t.w;
      }
      if constexpr (R % 4 == 2) {  // (R = 2: one float2)
        const float2 t = reinterpret_cast<const float2*>(bias + (j + g) * R)[R / 2 - 1];
        bv[R - 2] = t.x;
        bv[R - 1] = t.y;
      }
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (!((PM >> p) & 1)) continue;  // row pair without a needed group (block-sparse plan)
        float2 acc = f2(bv[2 * p], bv[2 * p + 1]);
#pragma unroll
        for (int k = 0; k < KX; ++k) acc = fma2(x2[p][k], f2(c[k], c[k]), acc);
        q[p][g] = acc;
      }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (!((PM >> p) & 1)) continue;
      const float2 m2 = f2(mq[2 * p], mq[2 * p + 1]);
      float2 gs = f2(0.f, 0.f);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float2 v = fma2(q[p][g], f2(-1.f, -1.f), m2);
        gs = add2(gs, (g == 0 && p < POLY) ? exp2_poly2(v) : f2(ex2(v.x), ex2(v.y)));
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
              S[r] *= sc;
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
    if (!((PM >> p) & 1)) continue;
    S[2 * p] += f32_to_f64_alu(T[p].x);
    S[2 * p + 1] += f32_to_f64_alu(T[p].y);
  }
}

template <int KX, int R>
struct CtrSmem {
  static constexpr int kStage64 = kColTile * (KX + 1);  // doubles
  static constexpr int kStage32 = kColTile * KX;        // floats
  static constexpr size_t kBytes =
      2 * sizeof(double) * kStage64 + 2 * sizeof(float) * kStage32 + sizeof(float) * kColTile * R +
      2 * sizeof(double) * R * 128;  // + row reference M and tile offset per (row, thread)
};

// CTA: 128 threads x R rows (R consecutive 128-row groups in locality order) x
// one column chunk; 256-column tiles of [Zr | c] (fp64) and dZ (fp32) arrive
// by two bulk copies on one mbarrier, double-buffered.
template <int KX, int R, int G, int MINB, int POLY>
__global__ void __launch_bounds__(128, MINB) softmin_ctr_kernel(const SoftminArgs a) {
  using SM = CtrSmem<KX, R>;
  constexpr int P = R / 2;
  extern __shared__ __align__(128) unsigned char smem_c[];
  double* s64 = reinterpret_cast<double*>(smem_c);
  float* s32 = reinterpret_cast<float*>(s64 + 2 * SM::kStage64);
  float* sbias = s32 + 2 * SM::kStage32;                          // [256][R]
  double* sM = reinterpret_cast<double*>(sbias + kColTile * R);   // [R][128]
  double* sOff = sM + R * 128;                                    // [R][128]
  __shared__ double gctr[R][KX];
  __shared__ double grad[R];
  __shared__ double red[4][R];
  __shared__ uint64_t bars[2];
  if (skip_now(a.st, a.skip)) return;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int chunk = blockIdx.y;
  const int64_t mpad = (a.m + kColTile - 1) / kColTile * kColTile;
  const CtrRows rows = ctr_rows_view(a.row_feat, a.n, KX);
  const CtrCols cols = ctr_cols_view(a.col_rec, mpad, KX);
  const int64_t g0 = (int64_t)blockIdx.x * R;  // first row group of the CTA
  const int64_t ngroups = ctr_groups(a.n);

  float2 x2[P][KX];
#pragma unroll
  for (int p = 0; p < P; ++p) {
#pragma unroll
    for (int k = 0; k < KX; ++k) {
      float v[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t g = g0 + 2 * p + h;
        v[h] = g < ngroups ? rows.dx32[(g * kCtrRowGroup + tid) * KX + k] : 0.f;
      }
      x2[p][k] = f2(v[0], v[1]);
    }
  }
  if (tid < R * KX) {
    const int r = tid / KX, k = tid % KX;
    gctr[r][k] = g0 + r < ngroups ? rows.ctr[(g0 + r) * (KX + 1) + k] : 0.0;
  }
  if (tid < R) grad[tid] = g0 + tid < ngroups ? rows.ctr[(g0 + tid) * (KX + 1) + KX] : 0.0;
  float mq[R];
  double S[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    sM[r * 128 + tid] = CUDART_INF;
    S[r] = 0.0;
  }

  const int64_t c0 = (int64_t)chunk * a.chunk_cols;
  const int ntiles = (int)((min(c0 + a.chunk_cols, mpad) - c0) / kColTile);
  const uint32_t b64 = SM::kStage64 * sizeof(double), b32 = SM::kStage32 * sizeof(float);
  const double* src64 = cols.rec64 + c0 * (KX + 1);
  const float* src32 = cols.rec32 + c0 * KX;
  // Block-sparse plan (ctr_plan_kernel): tiles that cannot hold a term within
  // 2^-T of any of this CTA's rows' maxima are skipped; every thread walks the
  // same sequence of needed tiles (a uniform scan of a byte mask in L1/L2).
  const uint32_t* need = a.ctr_need ? a.ctr_need + (int64_t)blockIdx.x * (mpad / kColTile) + c0 / kColTile
                                    : nullptr;
  auto next_needed = [&](int t) {
    if (need)
      while (t < ntiles && !need[t]) ++t;
    return t;
  };
  auto load_tile = [&](int s, int t) {
    mbar_expect_tx(&bars[s], b64 + b32);
    bulk_g2s(s64 + s * SM::kStage64, src64 + (int64_t)t * SM::kStage64, b64, &bars[s]);
    bulk_g2s(s32 + s * SM::kStage32, src32 + (int64_t)t * SM::kStage32, b32, &bars[s]);
  };
  int tq[2];  // needed tiles in the two stages
  tq[0] = next_needed(0);
  tq[1] = next_needed(tq[0] + 1);
  TilePipe pipe{bars};
  pipe.init();  // (also publishes gctr and sM)
  if (tid == 0)
    for (int s = 0; s < 2; ++s)
      if (tq[s] < ntiles) load_tile(s, tq[s]);
  for (int k = 0; tq[k & 1] < ntiles; ++k) {
    const int s = k & 1;
    const int64_t J = c0 / kColTile + tq[s];
    mbar_wait(&bars[s], (k >> 1) & 1);
    // (1) group biases A_j^I = c_j + <Xc_I, Zr_j> for this thread's 2 columns, fp64
    const double* rec = s64 + s * SM::kStage64;
    double A[R][2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double* rj = rec + (tid + 128 * h) * (KX + 1);
      double z[KX];
#pragma unroll
      for (int k = 0; k < KX; ++k) z[k] = rj[k];
      const double c = rj[KX];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double acc = c;
#pragma unroll
        for (int k = 0; k < KX; ++k) acc = fma(gctr[r][k], z[k], acc);
        A[r][h] = acc;
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double v = fmin(A[r][0], A[r][1]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (lane == 0) red[warp][r] = v;
    }
    __syncthreads();
    // (2) rho_r = min_j A_j^I; biases to shared memory; row offsets rho + B_i^J.
    // A group whose pair-term bound |dX| |dZ| exceeds ctr_limit on this tile
    // (a locality jump, a sparse outer region) takes the tile in fp64 below:
    // its fp32 biases are +inf so the fp32 sweep adds nothing for it.
    const double radJ = cols.tctr[J * (KX + 1) + KX];
    unsigned bad = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) bad |= (grad[r] * radJ > a.ctr_limit ? 1u : 0u) << r;
    double rho[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      rho[r] = fmin(fmin(red[0][r], red[1][r]), fmin(red[2][r], red[3][r]));
      if (!(rho[r] < CUDART_INF)) rho[r] = 0.0;  // a tile of zero-weight columns: all biases +inf
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float bb[R];
#pragma unroll
      // (finite cap: a zero-weight column, A = +inf, must not meet an infinite
      // row reference as inf - inf)
      for (int r = 0; r < R; ++r)
        bb[r] = (bad >> r) & 1u ? CUDART_INF_F : (float)fmin(A[r][h] - rho[r], kPadQ);
      float4* b4 = reinterpret_cast<float4*>(sbias + (tid + 128 * h) * R);
#pragma unroll
      for (int v = 0; v < R / 4; ++v) b4[v] = make_float4(bb[4 * v], bb[4 * v + 1], bb[4 * v + 2], bb[4 * v + 3]);
      if constexpr (R % 4 == 2)
        reinterpret_cast<float2*>(sbias + (tid + 128 * h) * R)[R / 2 - 1] = make_float2(bb[R - 2], bb[R - 1]);
    }
    double tc[KX];
#pragma unroll
    for (int k = 0; k < KX; ++k) tc[k] = cols.tctr[J * (KX + 1) + k];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t g = g0 + r;
      double b = rho[r];
      if (g < ngroups) {
        const double* d = rows.dx64 + (g * kCtrRowGroup + tid) * KX;
#pragma unroll
        for (int k = 0; k < KX; ++k) b = fma(d[k], tc[k], b);
      }
      sOff[r * 128 + tid] = b;
      // (a finite reference keeps the +inf biases of a deferred group at 0 terms)
      mq[r] = (bad >> r) & 1u ? 0.f : (float)(sM[r * 128 + tid] - b);
    }
    __syncthreads();  // biases visible
    float mq0[R];
#pragma unroll
    for (int r = 0; r < R; ++r) mq0[r] = mq[r];
    if constexpr (R == 4) {  // skip a row pair none of whose groups needs the tile
      uint32_t v = need ? need[tq[s]] : 0xFFu;
      v = (v | (v >> 8) | (v >> 16) | (v >> 24)) & 0xFu;
      const int pm = ((v & 3u) ? 1 : 0) | ((v & 12u) ? 2 : 0);
      if (pm == 1)
        softmin_tile_ctr<KX, R, G, POLY, 1>(s32 + s * SM::kStage32, sbias, x2, mq, S);
      else if (pm == 2)
        softmin_tile_ctr<KX, R, G, POLY, 2>(s32 + s * SM::kStage32, sbias, x2, mq, S);
      else
        softmin_tile_ctr<KX, R, G, POLY>(s32 + s * SM::kStage32, sbias, x2, mq, S);
    } else {
      softmin_tile_ctr<KX, R, G, POLY>(s32 + s * SM::kStage32, sbias, x2, mq, S);
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (mq[r] != mq0[r]) sM[r * 128 + tid] = sOff[r * 128 + tid] + (double)mq[r];
    if (bad) {  // CTA-uniform: the deferred groups of this tile in fp64
#pragma unroll 1
      for (int r = 0; r < R; ++r) {
        if (!((bad >> r) & 1u)) continue;
        double xi[KX];
        const double* d = rows.dx64 + ((g0 + r) * kCtrRowGroup + tid) * KX;
#pragma unroll
        for (int k = 0; k < KX; ++k) xi[k] = gctr[r][k] + d[k];
        double M = sM[r * 128 + tid], Sd = 0.0;
        // S[r] is a register array: move it through a uniform switch
#pragma unroll
        for (int q = 0; q < R; ++q)
          if (q == r) Sd = S[q];
        // 8 independent columns per step: fp64 scores, a (rare) rebase of the
        // reference at their minimum, then 8 exponentials summed in fp32
#pragma unroll 1
        for (int j = 0; j < kColTile; j += 8) {
          double qv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const double* rj = rec + (j + u) * (KX + 1);
            double acc = rj[KX];
#pragma unroll
            for (int k = 0; k < KX; ++k) acc = fma(xi[k], rj[k], acc);
            qv[u] = fmin(acc, kPadQ);  // zero-weight columns: finite, zero-weight terms
          }
          double qmin = qv[0];
#pragma unroll
          for (int u = 1; u < 8; ++u) qmin = fmin(qmin, qv[u]);
          if (qmin < M) {
            Sd *= exp2(qmin - M);
            M = qmin;
          }
          float t = 0.f;
#pragma unroll
          for (int u = 0; u < 8; ++u) t += ex2(-f64_to_f32_alu(qv[u] - M));  // (no F2F on the XU pipe)
          Sd += (double)t;
        }
        sM[r * 128 + tid] = M;
#pragma unroll
        for (int q = 0; q < R; ++q)
          if (q == r) S[q] = Sd;
      }
    }
    __syncthreads();  // every warp is done with stage s and the biases
    tq[s] = next_needed(tq[s ^ 1] + 1);  // the needed tile after the one in the other stage
    if (tid == 0 && tq[s] < ntiles) load_tile(s, tq[s]);
  }
  const double lam = a.st->lam_d, inv_lam = 1.0 / lam;
  const double* rs = static_cast<const double*>(a.row_sq);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t ip = (g0 + r) * kCtrRowGroup + tid;  // locality position
    if (ip < a.n) {
      const int64_t i = rows.order[ip];
      const double si = rs ? rs[i] : 0.0;
      softmin_store(a, chunk, i, -sM[r * 128 + tid] - lam * si * si, S[r], inv_lam);
    }
  }
}

// ---- block-sparse plan ---------------------------------------------------------
// For the CTA of R row groups the streaming kernel will use, over ALL column
// tiles: rho_IJ = min_j A_j^I (fp64, as the streaming prologue), per row
// B_i^J, and the bounds on the row's terms in tile J (log2 units, t = -q)
//     t_ij <= -(rho_IJ + B_i^J) + C_IJ,   max_j t_ij >= -(rho_IJ + B_i^J) - C_IJ,
// C_IJ = R_I R_J the pair-term bound. (1) each warp takes every 4th tile and
// reduces rho over its 256 columns (no block barrier per tile), stored in fp32
// rounded down; (2) every row keeps L_i = max_J of the lower bound (with rho
// rounded back up, so it stays a lower bound); (3) a warp votes tile J needed
// when one of its 32 rows has an upper bound (rho rounded down) reaching
// L_i - T. A skipped tile holds only terms below 2^-T of its row's maximum,
// so with T = 64 the skipped mass is < m 2^-64 of every row's sum. need:
// [CTA][tile] 32-bit words, one byte per warp whose bit r votes for group r.
// Plan reuse across sweeps. Column potentials move every sweep, but every
// term t_ij of a half-update shifts by exactly the change d_j of its column's
// c_j (log2 units; rows' own potentials do not enter) and a row's maximum by
// the d of some other column, so a plan made with threshold T + 2 budget
// stays valid while max_j d_j - min_j d_j <= 2 budget and the rest of the
// records (lam-scaled features) is unchanged. One block
// compares the current column records with the copy taken at the last plan
// and sets key->replan. It replans unconditionally on the first sweep of a
// loop (features change only between loops), whenever lam differs from the
// plan's (annealed sweeps rescale Zr = -2 lam z, not only c), whenever the
// operator differs (row/column block pointers and sizes: a workspace shared
// by two operators never reuses the other's plan), and whenever a column
// record or its planned copy is NaN.
struct CtrPlanKey {
  int32_t replan;
  int32_t pad_;
  double lam;
  const void* rows;
  const void* cols;
  int64_t n, m;
};

template <int KX>
__global__ void __launch_bounds__(1024) ctr_plan_check_kernel(const cntgw_sweep_state* st, const double* rec64,
                                                              int64_t mpad, double* c_plan, CtrPlanKey* key,
                                                              const void* rows, const void* cols, int64_t n,
                                                              int64_t m, double budget) {
  __shared__ double red[32], red2[32];
  __shared__ int go, nan_seen;
  const double lam = st ? st->lam_d : 0.0;
  const bool first = st == nullptr || st->sweep <= 1 || key->lam != lam || key->rows != rows ||
                     key->cols != cols || key->n != n || key->m != m;
  if (threadIdx.x == 0) nan_seen = 0;
  __syncthreads();
  // validity of the plan: a term skipped with margin T + 2 budget moved by
  // its column's shift d_j = c_j - c_j(plan), its row's maximum by the shift
  // of another column, so the plan holds while max_j d_j - min_j d_j <=
  // 2 budget (a uniform shift of every column changes nothing)
  double dmx = 0.0, dmn = 0.0;
  bool bad = false;
  if (!first)
    for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
      const double c = rec64[j * (KX + 1) + KX], cp = c_plan[j];
      bad |= (c != c) || (cp != cp);
      const double d = c == cp ? 0.0 : c - cp;  // equal infinities (zero weight): no change
      dmx = fmax(dmx, d);
      dmn = fmin(dmn, d);
    }
  if (bad) nan_seen = 1;  // fmax/fmin drop NaN, so it is flagged separately
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dmx = fmax(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
    dmn = fmin(dmn, __shfl_xor_sync(0xffffffffu, dmn, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = dmx;
    red2[threadIdx.x >> 5] = dmn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mx = 0.0, mn = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      mx = fmax(mx, red[q]);
      mn = fmin(mn, red2[q]);
    }
    go = (first || nan_seen || !(mx - mn <= 2.0 * budget)) ? 1 : 0;
    key->replan = go;
    if (go) {
      key->lam = lam;
      key->rows = rows;
      key->cols = cols;
      key->n = n;
      key->m = m;
    }
  }
  __syncthreads();
  if (go)
    for (int64_t j = threadIdx.x; j < mpad; j += blockDim.x) c_plan[j] = rec64[j * (KX + 1) + KX];
}

template <int KX, int R, int S>
__global__ void __launch_bounds__(128) ctr_plan_kernel(const SoftminArgs a, float* rho_tab, uint32_t* need,
                                                       double T, const int* replan) {
  if (replan && !*replan) return;  // the previous plan still holds (ctr_plan_check_kernel)
  // one block plans S consecutive streaming CTAs (S * R row groups): each
  // column record is read once per S * R groups
  constexpr int GB = S * R;
  __shared__ double gctr[GB][KX];
  __shared__ double grad[GB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t mpad = (a.m + kColTile - 1) / kColTile * kColTile;
  const int64_t TL = mpad / kColTile;
  const CtrRows rows = ctr_rows_view(a.row_feat, a.n, KX);
  const CtrCols cols = ctr_cols_view(a.col_rec, mpad, KX);
  const int64_t ngroups = ctr_groups(a.n);
  const int64_t nctas = (ngroups + R - 1) / R;
  const int64_t cta0 = (int64_t)blockIdx.x * S, g0 = cta0 * R;
  for (int e = tid; e < GB * KX; e += blockDim.x) {
    const int r = e / KX, k = e % KX;
    gctr[r][k] = g0 + r < ngroups ? rows.ctr[(g0 + r) * (KX + 1) + k] : 0.0;
  }
  if (tid < GB) grad[tid] = g0 + tid < ngroups ? rows.ctr[(g0 + tid) * (KX + 1) + KX] : 0.0;
  __syncthreads();
  float* rho_blk = rho_tab + g0 * TL;  // [group][tile], groups of consecutive CTAs are contiguous
  for (int64_t J = warp; J < TL; J += 4) {  // (1) rho, one tile per warp
    double mn[GB];
#pragma unroll
    for (int r = 0; r < GB; ++r) mn[r] = CUDART_INF;
#pragma unroll 4
    for (int u = 0; u < kColTile / 32; ++u) {
      const double* rj = cols.rec64 + (J * kColTile + lane + 32 * u) * (KX + 1);
      double z[KX];
#pragma unroll
      for (int k = 0; k < KX; ++k) z[k] = rj[k];
      const double c = rj[KX];
#pragma unroll
      for (int r = 0; r < GB; ++r) {
        double acc = c;
#pragma unroll
        for (int k = 0; k < KX; ++k) acc = fma(gctr[r][k], z[k], acc);
        mn[r] = fmin(mn[r], acc);
      }
    }
#pragma unroll
    for (int r = 0; r < GB; ++r) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mn[r] = fmin(mn[r], __shfl_xor_sync(0xffffffffu, mn[r], o));
      if (lane == r % 32 && g0 + r < ngroups) rho_blk[r * TL + J] = __double2float_rd(mn[r]);
    }
  }
  __syncthreads();  // rho_blk visible to the block
  // (2)/(3) in fp32 with an explicit rounding allowance: every quantity is a
  // bound, so it is enough that the lower bound is rounded down and the upper
  // one up; err = (|rho| + |B| + C) 2^-20 covers the fp32 roundings of rho
  // (stored rounded down), of B = <dx, Zc> and of the sums.
  for (int sc = 0; sc < S && cta0 + sc < nctas; ++sc) {
    const int r0 = sc * R;
    float dx[R][KX], L[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int k = 0; k < KX; ++k)
        dx[r][k] = g0 + r0 + r < ngroups ? (float)rows.dx64[((g0 + r0 + r) * kCtrRowGroup + tid) * KX + k] : 0.f;
      L[r] = -CUDART_INF_F;
    }
    for (int64_t J = 0; J < TL; ++J) {  // (2) L_i
      const double* tc = cols.tctr + J * (KX + 1);
      float zc[KX];
#pragma unroll
      for (int k = 0; k < KX; ++k) zc[k] = (float)tc[k];
      const float radJ = (float)tc[KX];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (g0 + r0 + r >= ngroups) break;
        const float rd = rho_blk[(r0 + r) * TL + J];
        float bb = 0.f;
#pragma unroll
        for (int k = 0; k < KX; ++k) bb = fmaf(dx[r][k], zc[k], bb);
        const float cc = (float)grad[r0 + r] * radJ;
        const float err = (fabsf(rd) + fabsf(bb) + cc) * 0x1p-20f;
        L[r] = fmaxf(L[r], -(rd + bb) - cc - err);  // (+inf rho: zero-weight tile, no bound)
      }
    }
    uint8_t* vote = reinterpret_cast<uint8_t*>(need + (cta0 + sc) * TL);
    for (int64_t J = 0; J < TL; ++J) {  // (3) verdicts
      const double* tc = cols.tctr + J * (KX + 1);
      float zc[KX];
#pragma unroll
      for (int k = 0; k < KX; ++k) zc[k] = (float)tc[k];
      const float radJ = (float)tc[KX];
      uint32_t keep = 0;  // bit r: group r needs the tile
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (g0 + r0 + r >= ngroups) break;
        const float rd = rho_blk[(r0 + r) * TL + J];
        float bb = 0.f;
#pragma unroll
        for (int k = 0; k < KX; ++k) bb = fmaf(dx[r][k], zc[k], bb);
        const float cc = (float)grad[r0 + r] * radJ;
        const float err = (fabsf(rd) + fabsf(bb) + cc) * 0x1p-20f;
        keep |= (__any_sync(0xffffffffu, -(rd + bb) + cc + err >= L[r] - (float)T) ? 1u : 0u) << r;
      }
      if (lane == 0) vote[J * 4 + warp] = (uint8_t)keep;
    }
  }
}

}  // namespace cntgw
