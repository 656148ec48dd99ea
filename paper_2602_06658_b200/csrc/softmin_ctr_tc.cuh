// K1/K2, CNTGW_F32C on the tensor cores (kd + sq <= 4: the C3/C4 shapes).
//
// Same decomposition as softmin_ctr.cuh (centred 128-row groups and
// 256-column tiles in locality order, q_ij = A_j^I + B_i^J + <dX_i, dZ_j>),
// with the pair term and the per-group bias on tcgen05 in the split-precision
// (3xTF32) form of softmin_tc.cuh. One CTA = one 128-row group, so the bias
// -fp32(A_j^I - min_j A_j^I) of a tile is one extra K column of B', written by
// the CTA into its shared-memory copy of the tile:
//     A'_i = [hi(dX_i), 1 | hi(dX_i), 1 | lo(dX_i), 0]          (K' = 16)
//     B'_j = [hi(-dZ_j), hi(-a_j) | lo(-dZ_j), lo(-a_j) | hi(-dZ_j), 0]
// so the accumulator is the tile-local score t_ij - off_i (t = -q) and the
// epilogue is the lazily rebased MUFU.EX2 sum of softmin_tc.cuh, entered per
// tile with the fp32 reference fp32(M_i - off_i), off_i = -(min A + B_i^J).
//
// Warp roles (1 CTA per SM):
//   warp 0   TMA producer: B' tile (prepacked -dZ splits, 16 KB) and the
//            tile's fp64 records [Zr | c] (10 KB) into a 3-stage ring
//   warp 1   TMEM allocator + MMA issuer (2 x tcgen05.mma kind::tf32 K=8)
//   warp 2   bias warp: A_j^I = c_j + <Xc_I, Zr_j> in fp64 for the tile's 256
//            columns, min, the bias column of B' (generic stores + proxy
//            fence), the tile's (min A, centre, fallback flag) for the
//            epilogue; for a tile whose pair-term bound exceeds the limit it
//            copies the fp64 records for the epilogue's fp64 fallback
//   warps 3.. EPI epilogue warps (TMEM lane quadrant x column part)
#pragma once

#include "common.cuh"
#include "softmin.cuh"
#include "softmin_ctr.cuh"
#include "softmin_tc.cuh"

namespace cntgw {

constexpr int kCtcKx = 4;                             // kd + sq padded
using CtcL = TcLayout<kCtcKx>;                         // K' = 16: two K=8 MMA steps
constexpr int kCtcRecD = kColTile * (kCtcKx + 1);      // doubles of one fp64 record tile
constexpr int ctc_threads(int epi) { return 96 + 32 * epi; }

struct CtcTileInfo {
  double rho;            // min_j A_j^I of the tile (q-space)
  double zc[kCtcKx];     // tile centre Zc_J
  int bad;               // fp64 fallback for this (group, tile)
  int pad_;
};

// B' tiles of -dZ (tf32 hi/lo splits, bias slots zero) in the tcgen05
// K-major layout [tile][K' / 4 chunks][256 cols][4 floats], from the dZ
// records of the centred column block.
__global__ void prep_cols_ctc_kernel(const float* rec32, int64_t mpad, float* bt) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= mpad) return;
  const int64_t tile = j / kTcCols;
  const int col = (int)(j % kTcCols);
  float* base = bt + tile * CtcL::kBTileFloats + col * 4;
  auto put = [&](int p, float v) { base[(p >> 2) * (kTcCols * 4) + (p & 3)] = v; };
  for (int p = 0; p < CtcL::kKp; ++p) put(p, 0.f);
#pragma unroll
  for (int k = 0; k < kCtcKx; ++k) {
    const float z = -rec32[j * kCtcKx + k];
    const float zh = tf32_rna(z);
    put(CtcL::kHi + k, zh);
    put(CtcL::kLo + k, tf32_rna(z - zh));
    put(CtcL::kHi2 + k, zh);
  }
}

template <int EPI>
struct CtcSmem {
  static constexpr size_t kA = (size_t)CtcL::kATileFloats * 4;
  static constexpr size_t kB = (size_t)kTcStages * CtcL::kBTileFloats * 4;
  static constexpr size_t kR = (size_t)kTcStages * kCtcRecD * 8;
  static constexpr size_t kF = (size_t)2 * kCtcRecD * 8;  // fallback copies, per accumulator
  static constexpr size_t kBytes = kA + kB + kR + kF;
};

template <int EPI, int NPOLY>
__global__ void __launch_bounds__(ctc_threads(EPI), 1) softmin_ctc_kernel(const SoftminArgs a) {
  using SM = CtcSmem<EPI>;
  extern __shared__ __align__(1024) unsigned char smem_ctc[];
  float* sA = reinterpret_cast<float*>(smem_ctc);
  float* sB = reinterpret_cast<float*>(smem_ctc + SM::kA);
  double* sR = reinterpret_cast<double*>(smem_ctc + SM::kA + SM::kB);
  double* sF = reinterpret_cast<double*>(smem_ctc + SM::kA + SM::kB + SM::kR);
  __shared__ uint64_t full_bar[kTcStages], empty_bar[kTcStages], bias_bar[kTcStages];
  __shared__ uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ CtcTileInfo info[2];
  __shared__ uint32_t tmem_base_sh;
  constexpr int kParts = EPI / 4;
  constexpr int kChunksPerPart = kTcCols / kParts / 32;
  __shared__ double red_m[kParts][kTcRows];
  __shared__ double red_s[kParts][kTcRows];
  if (skip_now(a.st, a.skip)) return;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunk = blockIdx.y;
  const int64_t g = blockIdx.x;  // row group
  const int64_t mpad = (a.m + kColTile - 1) / kColTile * kColTile;
  const int64_t c0 = (int64_t)chunk * a.chunk_cols;
  const int ntiles = (int)((min(c0 + a.chunk_cols, mpad) - c0) / kTcCols);
  const CtrRows rows = ctr_rows_view(a.row_feat, a.n, kCtcKx);
  const CtrCols cols = ctr_cols_view(a.col_rec, mpad, kCtcKx);
  const float* btiles = reinterpret_cast<const float*>(
      reinterpret_cast<const char*>(a.col_rec) + ctr_cols_bytes(mpad, kCtcKx));

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
      mbar_init(&bias_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], EPI);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp >= 3 && threadIdx.x - 96 < kTcRows) {  // A' rows: splits of dX, bias ones
    const int r = threadIdx.x - 96;
    auto put = [&](int p, float v) { sA[(p >> 2) * (kTcRows * 4) + r * 4 + (p & 3)] = v; };
#pragma unroll
    for (int k = 0; k < kCtcKx; ++k) {
      const float x = rows.dx32[(g * kCtrRowGroup + r) * kCtcKx + k];
      const float xh = tf32_rna(x);
      put(CtcL::kHi + k, xh);
      put(CtcL::kLo + k, xh);
      put(CtcL::kHi2 + k, tf32_rna(x - xh));
    }
    put(CtcL::kHi + kCtcKx, 1.f);
    put(CtcL::kLo + kCtcKx, 1.f);
    for (int p = CtcL::kHi2 + kCtcKx; p < CtcL::kKp; ++p) put(p, 0.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {  // producer
      const uint32_t bb = CtcL::kBTileFloats * sizeof(float), rb = kCtcRecD * sizeof(double);
      const float* srcB = btiles + (c0 / kTcCols) * CtcL::kBTileFloats;
      const double* srcR = cols.rec64 + c0 * (kCtcKx + 1);
      for (int t = 0, s = 0, ph = 0; t < ntiles; ++t) {
        mbar_wait(&empty_bar[s], ph ^ 1);
        mbar_expect_tx(&full_bar[s], bb + rb);
        bulk_g2s(sB + s * CtcL::kBTileFloats, srcB + (int64_t)t * CtcL::kBTileFloats, bb, &full_bar[s]);
        bulk_g2s(sR + s * kCtcRecD, srcR + (int64_t)t * kCtcRecD, rb, &full_bar[s]);
        if (++s == kTcStages) s = 0, ph ^= 1;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      const uint32_t a0 = smem_u32(sA);
      for (int t = 0, s = 0, ph = 0; t < ntiles; ++t) {
        const int ab = t & 1;
        mbar_wait(&bias_bar[s], ph);
        mbar_wait(&tempty_bar[ab], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t b0 = smem_u32(sB + s * CtcL::kBTileFloats);
        const uint32_t d = tmem + (uint32_t)(ab * kTcCols);
#pragma unroll
        for (int ks = 0; ks < CtcL::kKp / 8; ++ks) {
          const uint64_t ad = umma_desc(a0 + ks * 2 * (kTcRows * 16), kTcRows * 16, 128);
          const uint64_t bd = umma_desc(b0 + ks * 2 * (kTcCols * 16), kTcCols * 16, 128);
          tc_mma(d, ad, bd, ks > 0 ? 1u : 0u);
        }
        tc_commit(&empty_bar[s]);
        tc_commit(&tfull_bar[ab]);
        if (++s == kTcStages) s = 0, ph ^= 1;
      }
    }
  } else if (warp == 2) {  // bias warp
    double xc[kCtcKx];
#pragma unroll
    for (int k = 0; k < kCtcKx; ++k) xc[k] = rows.ctr[g * (kCtcKx + 1) + k];
    const double grad = rows.ctr[g * (kCtcKx + 1) + kCtcKx];
    for (int t = 0, s = 0, ph = 0; t < ntiles; ++t) {
      const int ab = t & 1;
      const int64_t J = c0 / kColTile + t;
      mbar_wait(&full_bar[s], ph);
      mbar_wait(&tempty_bar[ab], ((t >> 1) & 1) ^ 1);  // info[ab] / sF[ab] are free
      const double* rec = sR + s * kCtcRecD;
      double A[8];
      double mn = CUDART_INF;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double* rj = rec + (lane + 32 * u) * (kCtcKx + 1);
        double acc = rj[kCtcKx];
#pragma unroll
        for (int k = 0; k < kCtcKx; ++k) acc = fma(xc[k], rj[k], acc);
        A[u] = acc;
        mn = fmin(mn, acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      if (!(mn < CUDART_INF)) mn = 0.0;  // a tile of zero-weight columns: all biases +inf
      const double radJ = cols.tctr[J * (kCtcKx + 1) + kCtcKx];
      const bool bad = grad * radJ > a.ctr_limit;
      float* bt = sB + s * CtcL::kBTileFloats;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int col = lane + 32 * u;
        // -bias as two tf32 terms of its fp32 rounding; the double -> float
        // conversion on the ALU (F2F would queue on the XU pipe behind the
        // epilogue's MUFU stream and stall this warp, the MMA's critical path);
        // padding columns -> -1e30 (zero weight)
        const float v = f64_to_f32_rn_alu(fmax(mn - A[u], -kPadQ));  // (zero weights: A = +inf)
        const float vh = tf32_rna(v);
        bt[(CtcL::kHi + kCtcKx) / 4 * (kTcCols * 4) + col * 4 + (CtcL::kHi + kCtcKx) % 4] = vh;
        bt[(CtcL::kLo + kCtcKx) / 4 * (kTcCols * 4) + col * 4 + (CtcL::kLo + kCtcKx) % 4] =
            tf32_rna(v - vh);
      }
      if (bad) {  // fp64 records for the epilogue's fallback
        double* f = sF + ab * kCtcRecD;
        for (int e = lane; e < kCtcRecD; e += 32) f[e] = rec[e];
      }
      if (lane < kCtcKx) info[ab].zc[lane] = cols.tctr[J * (kCtcKx + 1) + lane];
      if (lane == 0) {
        info[ab].rho = mn;
        info[ab].bad = bad ? 1 : 0;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // bias column -> tensor proxy
      __syncwarp();
      if (lane == 0) mbar_arrive(&bias_bar[s]);
      if (++s == kTcStages) s = 0, ph ^= 1;
    }
  } else {  // epilogue warps
    const int q = warp & 3;
    const int part = (warp - 3) >> 2;
    const int r = 32 * q + lane;
    const int64_t ip = g * kCtrRowGroup + r;  // locality position of this row
    double dx[kCtcKx];
#pragma unroll
    for (int k = 0; k < kCtcKx; ++k) dx[k] = rows.dx64[ip * kCtcKx + k];
    double M = -CUDART_INF;  // row reference in t-space (fp64), S relative to it
    FFSum S;
    float va[32], vb[32];
    for (int t = 0; t < ntiles; ++t) {
      const int ab = t & 1;
      const int s = t % kTcStages;
      mbar_wait(&tfull_bar[ab], (t >> 1) & 1);
      mbar_wait(&bias_bar[s], (t / kTcStages) & 1);  // orders info[ab] (already complete)
      tc_fence_after();
      double b = info[ab].rho;
#pragma unroll
      for (int k = 0; k < kCtcKx; ++k) b = fma(dx[k], info[ab].zc[k], b);
      const double off = -b;  // t_abs = off + accumulator
      if (info[ab].bad) {
        // fp64 fallback: t = -(c_j + <X_i, Zr_j>) over this part's columns
        const double* f = sF + ab * kCtcRecD;
        double xi[kCtcKx];
        // X_i = Xc + dX (the bias warp's group centre, reloaded)
#pragma unroll
        for (int k = 0; k < kCtcKx; ++k) xi[k] = rows.ctr[g * (kCtcKx + 1) + k] + dx[k];
        double Sd = S.value();
        const int j0 = part * (kTcCols / kParts);
        for (int j = j0; j < j0 + kTcCols / kParts; j += 8) {
          double tv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const double* rj = f + (j + u) * (kCtcKx + 1);
            double acc = rj[kCtcKx];
#pragma unroll
            for (int k = 0; k < kCtcKx; ++k) acc = fma(xi[k], rj[k], acc);
            tv[u] = fmax(-acc, -kPadQ);
          }
          double tmax = tv[0];
#pragma unroll
          for (int u = 1; u < 8; ++u) tmax = fmax(tmax, tv[u]);
          if (tmax > M) {
            Sd *= exp2(M - tmax);
            M = tmax;
          }
          float ts = 0.f;
#pragma unroll
          for (int u = 0; u < 8; ++u) ts += ex2(-f64_to_f32_alu(M - tv[u]));
          Sd += (double)ts;
        }
        S.hi = (float)Sd;
        S.lo = (float)(Sd - (double)S.hi);
        // release the accumulator (and info / sF of this buffer) only now
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[ab]);
        continue;
      }
      float mref = f64_to_f32_rn_alu(M - off);  // (no F2F on the XU pipe)
      if (!(M - off > -1e30)) mref = -CUDART_INF_F;
      const float mref0 = mref;
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) +
                             (uint32_t)(ab * kTcCols + part * (kTcCols / kParts));
      float tsum = 0.f;
      tmem_ld32(taddr, va);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < kChunksPerPart; ++c) {
        float(&cur)[32] = (c & 1) ? vb : va;
        float(&nxt)[32] = (c & 1) ? va : vb;
        if (c + 1 < kChunksPerPart) {
          tmem_ld32(taddr + 32 * (c + 1), nxt);
        } else {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[ab]);
        }
        tc_chunk<NPOLY>(cur, mref, tsum, S);
        if (c + 1 < kChunksPerPart) tmem_wait_ld();
      }
      S.add(tsum);
      if (mref != mref0) M = off + f32_to_f64_alu_s(mref);
    }
    red_m[part][r] = M;
    red_s[part][r] = S.value();
    asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI) : "memory");
    if (part == 0 && ip < a.n) {
      double mm = red_m[0][r];
#pragma unroll
      for (int p = 1; p < kParts; ++p) mm = fmax(mm, red_m[p][r]);
      double tot = 0.0;
#pragma unroll
      for (int p = 0; p < kParts; ++p)
        if (red_s[p][r] > 0.0) tot += red_s[p][r] * exp2(red_m[p][r] - mm);
      const int64_t i = rows.order[ip];
      const double lam = a.st->lam_d;
      const double* rs = static_cast<const double*>(a.row_sq);
      const double si = rs ? rs[i] : 0.0;
      softmin_store(a, chunk, i, mm - lam * si * si, tot, 1.0 / lam);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace cntgw
