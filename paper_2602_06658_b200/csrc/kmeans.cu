// Weighted k-means for the multiscale front end (reference solvers.py:668-726,
// `_weighted_kmeans` / `coarsen`), on the device and
// bit-compatible with the reference's numpy arithmetic:
//   * squared distances sum (x_d - c_d)^2 over d in numpy's pairwise order
//     (8 accumulators for 8 <= D <= 128), products/sums unfused (_rn
//     intrinsics, never contracted into FMAs);
//   * argmin keeps the first minimum;
//   * k-means++ draws reproduce Generator.choice(n, p): p = mass / total with
//     total the numpy pairwise sum over n, cdf = sequential cumsum,
//     cdf /= cdf[-1], first index with cdf > u (u drawn on the host from the
//     same Generator). The cdf is scanned in parallel; a draw whose u falls
//     within the rounding band of a boundary is redone by the exact
//     sequential pass for n <= kExactMaxN (a single-thread pass costs ~50 ns
//     per element). Above that — sizes the reference's dense N x k x D
//     k-means cannot run — the parallel answer stands: it can differ from
//     numpy's sequential cumsum only inside that band, i.e. pick a neighbour
//     of numpy's index with probability ~n * 1e-15 per draw;
//   * centres: sequential sum over members in index order of fl(w_i x_i)
//     (numpy's axis-0 reduction) divided by the pairwise sum of the member
//     weights; centre masses: sequential np.add.at order.
// Declarations: include/cntgw_b200.h.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

using namespace cntgw;

namespace cntgw {
int set_error(int code, const char* msg);
}

namespace {

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return cntgw::set_error(code, buf);
}

int check_launch(const char* what) {
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(CNTGW_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  }
  return CNTGW_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// numpy pairwise_sum for n <= 128 values (loops_utils.h: n < 8 sequential
// from 0; otherwise 8 strided accumulators, a fixed combine, then the rest)
template <typename F>
__device__ __forceinline__ double np_pw_leaf(int64_t n, F at) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, at(i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = at(j);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], at(i + j));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, at(i));
  return res;
}

// full numpy pairwise sum (recursive halving on multiples of 8 above 128),
// evaluated with an explicit frame stack: device recursion would run past the
// default per-thread stack on large clusters
template <typename F>
__device__ double np_pw(int64_t off, int64_t n, F at) {
  struct Frame {
    int64_t off, len;
    int state;
    double left;
  };
  Frame st[48];  // depth <= log2(n / 64) + 1
  int sp = 0;
  st[0] = {off, n, 0, 0.0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.len <= 128) {
      const int64_t o = f.off;
      ret = np_pw_leaf(f.len, [&](int64_t i) { return at(o + i); });
      --sp;
      continue;
    }
    int64_t n2 = f.len / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {  // left half first
      f.state = 1;
      st[sp + 1] = {f.off, n2, 0, 0.0};
      ++sp;
    } else if (f.state == 1) {  // then the right half
      f.left = ret;
      f.state = 2;
      st[sp + 1] = {f.off + n2, f.len - n2, 0, 0.0};
      ++sp;
    } else {  // combine
      ret = __dadd_rn(f.left, ret);
      --sp;
    }
  }
  return ret;
}

template <int D>
__device__ __forceinline__ double sq_dist(const double* __restrict__ x, const double* __restrict__ c) {
  double t[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double v = __dsub_rn(x[d], c[d]);
    t[d] = __dmul_rn(v, v);
  }
  return np_pw_leaf(D, [&](int64_t i) { return t[i]; });
}

// ---- Lloyd assignment: first argmin over all centres -----------------------
template <int D>
constexpr int tile_k() { return D <= 8 ? 256 : 4096 / D; }  // <= 32 KB of centres

template <int D>
__global__ void km_assign_kernel(const double* __restrict__ x, int64_t n,
                                 const double* __restrict__ centers, int64_t k, int64_t* assign,
                                 double* own) {
  constexpr int kTileK = tile_k<D>();
  __shared__ double sc[kTileK * D];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double xi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) xi[d] = i < n ? x[i * D + d] : 0.0;
  double best = CUDART_INF;
  int64_t bj = 0;
  for (int64_t t0 = 0; t0 < k; t0 += kTileK) {
    const int cnt = (int)min((int64_t)kTileK, k - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * D; e += blockDim.x) sc[e] = centers[t0 * D + e];
    __syncthreads();
    for (int c = 0; c < cnt; ++c) {
      const double dist = sq_dist<D>(xi, sc + c * D);
      if (dist < best) {
        best = dist;
        bj = t0 + c;
      }
    }
  }
  if (i < n) {
    assign[i] = bj;
    own[i] = best;
  }
}

// ---- k-means++ draw ---------------------------------------------------------
// workspace: [leaf sums (nleaves)] [total, flag, last] [cdf (n)] [block sums (nb)]
constexpr int kScanThreads = 256, kScanChunk = 8;
constexpr int64_t kExactMaxN = 1 << 17;  // exact sequential fallback up to here
constexpr int64_t kScanBlock = (int64_t)kScanThreads * kScanChunk;

struct DrawWs {
  double* leaf;
  double* scal;  // [0] total, [1] ambiguity flag, [2] cdf_last
  double* cdf;   // per element, inclusive within its scan block
  double* bsum;
};

__device__ __forceinline__ double mass_at(const double* w, const double* d2, int64_t i) {
  return d2 ? __dmul_rn(w[i], d2[i]) : w[i];
}

// one warp per leaf: lane j < 8 runs numpy's accumulator r[j] (elements j,
// j+8, ... of the unrolled part — coalesced 64-byte rows), lane 0 combines
// them in numpy's fixed order and adds the tail; leaves shorter than 8 are
// summed sequentially from 0 by lane 0
__global__ void km_leaf_kernel(const double* w, const double* d2, const int64_t* leaf_off,
                               int nleaves, double* leaf) {
  const int l = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (l >= nleaves) return;
  const int64_t o = leaf_off[l], len = leaf_off[l + 1] - o;
  if (len < 8) {
    if (lane == 0) {
      double r = 0.0;
      for (int64_t i = 0; i < len; ++i) r = __dadd_rn(r, mass_at(w, d2, o + i));
      leaf[l] = r;
    }
    return;
  }
  const int64_t body = len - (len % 8);
  double r = 0.0;
  if (lane < 8) {
    r = mass_at(w, d2, o + lane);
    for (int64_t i = 8 + lane; i < body; i += 8) r = __dadd_rn(r, mass_at(w, d2, o + i));
  }
  double rr[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) rr[j] = __shfl_sync(0xffffffffu, r, j);
  if (lane == 0) {
    double res = __dadd_rn(__dadd_rn(__dadd_rn(rr[0], rr[1]), __dadd_rn(rr[2], rr[3])),
                           __dadd_rn(__dadd_rn(rr[4], rr[5]), __dadd_rn(rr[6], rr[7])));
    for (int64_t i = body; i < len; ++i) res = __dadd_rn(res, mass_at(w, d2, o + i));
    leaf[l] = res;
  }
}

// combine the leaves along numpy's recursion: the host lists the internal
// nodes of the pairwise tree by height (children before parents); one block
// evaluates a height level per step. node ids: leaves 0..L-1, internal L.. .
__global__ void km_total_kernel(const int* tree, const int* hoff, int nh, int nleaves, DrawWs ws) {
  double* val = ws.leaf;  // leaf sums followed by the internal nodes
  for (int h = 0; h < nh; ++h) {
    for (int e = hoff[h] + threadIdx.x; e < hoff[h + 1]; e += blockDim.x) {
      const int node = tree[3 * e], l = tree[3 * e + 1], r = tree[3 * e + 2];
      val[node] = __dadd_rn(val[l], val[r]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int root = hoff[nh] > 0 ? tree[3 * (hoff[nh] - 1)] : 0;
    ws.scal[0] = val[root];
    ws.scal[1] = 0.0;
  }
}

__device__ __forceinline__ double prob_at(const double* w, const double* d2, double total, int64_t i) {
  // numpy: probs = mass / total if total > 0 else weights (first draw: p = weights)
  if (!d2) return w[i];
  return total > 0.0 ? __ddiv_rn(__dmul_rn(w[i], d2[i]), total) : w[i];
}

__global__ void km_scan_kernel(const double* w, const double* d2, int64_t n, DrawWs ws) {
  __shared__ double tsum[kScanThreads];
  const double total = ws.scal[0];
  const int64_t base = (int64_t)blockIdx.x * kScanBlock + (int64_t)threadIdx.x * kScanChunk;
  double loc[kScanChunk];
  double run = 0.0;
#pragma unroll
  for (int c = 0; c < kScanChunk; ++c) {
    const int64_t i = base + c;
    if (i < n) run = c == 0 ? prob_at(w, d2, total, i) : __dadd_rn(run, prob_at(w, d2, total, i));
    loc[c] = run;
  }
  tsum[threadIdx.x] = base < n ? run : 0.0;
  __syncthreads();
  if (threadIdx.x == 0) {  // fixed-order exclusive scan of the thread sums
    double acc = 0.0;
    for (int t = 0; t < kScanThreads; ++t) {
      const double v = tsum[t];
      tsum[t] = acc;
      acc = __dadd_rn(acc, v);
    }
    ws.bsum[blockIdx.x] = acc;
  }
  __syncthreads();
  const double off = tsum[threadIdx.x];
#pragma unroll
  for (int c = 0; c < kScanChunk; ++c) {
    const int64_t i = base + c;
    if (i < n) ws.cdf[i] = __dadd_rn(off, loc[c]);
  }
}

// block prefixes, cdf_last, the crossing index and its ambiguity (one block):
// binary search over the block boundaries, then the block's elements
__global__ void km_find_kernel(int64_t n, int nb, const double* u_all, const int* jp, DrawWs ws,
                               int64_t* out_idx) {
  __shared__ double s_last;
  __shared__ int s_blk;
  __shared__ unsigned long long found;
  const double u = u_all[*jp];
  extern __shared__ double sb[];  // block sums staged in parallel
  for (int b = threadIdx.x; b < nb; b += blockDim.x) sb[b] = ws.bsum[b];
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int b = 0; b < nb; ++b) {
      const double v = sb[b];
      sb[b] = acc;  // exclusive block prefixes
      acc = __dadd_rn(acc, v);
    }
    ws.scal[2] = acc;
    s_last = acc;
    const double target = u * acc;
    int lo = 0, hi = nb - 1;  // first block whose end prefix exceeds target
    while (lo < hi) {
      const int mid = (lo + hi) / 2;
      const double end = mid + 1 < nb ? sb[mid + 1] : acc;
      if (end > target) hi = mid;
      else lo = mid + 1;
    }
    s_blk = lo;
    found = (unsigned long long)n;
  }
  __syncthreads();
  const double last = s_last, target = u * last;
  const int64_t b0 = (int64_t)s_blk * kScanBlock, b1 = min(n, b0 + kScanBlock);
  const double pre = sb[s_blk];
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x)
    if (__dadd_rn(pre, ws.cdf[i]) > target) {
      atomicMin(&found, (unsigned long long)i);
      break;
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t idx = (int64_t)found;
    const double band = 8.0 * (double)n * 1.1102230246251565e-16 * last;
    bool amb = idx >= n;
    if (!amb) {
      const double v = __dadd_rn(sb[idx / kScanBlock], ws.cdf[idx]);
      amb = fabs(v - target) <= band;
      if (idx > 0) {
        const double p = __dadd_rn(sb[(idx - 1) / kScanBlock], ws.cdf[idx - 1]);
        amb = amb || fabs(p - target) <= band;
      }
    }
    ws.scal[1] = amb ? 1.0 : 0.0;
    *out_idx = idx < n ? idx : n - 1;
  }
}

// exact numpy semantics when the parallel scan could not decide (one thread)
__global__ void km_exact_kernel(const double* w, const double* d2, int64_t n, const double* u_all,
                                const int* jp, DrawWs ws, int64_t* out_idx) {
  if (ws.scal[1] == 0.0) return;
  const double total = ws.scal[0], u = u_all[*jp];
  double last = 0.0;
  for (int64_t i = 0; i < n; ++i) last = i == 0 ? prob_at(w, d2, total, 0) : __dadd_rn(last, prob_at(w, d2, total, i));
  double c = 0.0;
  int64_t idx = n;
  for (int64_t i = 0; i < n; ++i) {
    c = i == 0 ? prob_at(w, d2, total, 0) : __dadd_rn(c, prob_at(w, d2, total, i));
    if (__ddiv_rn(c, last) > u) {
      idx = i;
      break;
    }
  }
  *out_idx = idx < n ? idx : n - 1;
}

template <int D>
__global__ void km_d2_kernel(const double* __restrict__ x, int64_t n, const int64_t* idx_dev,
                             double* centers, const int* jp, double* d2, int first) {
  double* center_out = centers + (int64_t)(*jp) * D;
  const int64_t c = *idx_dev;
  double cc[D];
#pragma unroll
  for (int d = 0; d < D; ++d) cc[d] = x[c * D + d];
  if (blockIdx.x == 0 && threadIdx.x < D) center_out[threadIdx.x] = cc[threadIdx.x];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = sq_dist<D>(x + i * D, cc);
  d2[i] = first ? v : fmin(d2[i], v);
}

__global__ void km_advance_kernel(int* jp) { *jp += 1; }

// ---- centres from member lists (CSR in index order) ------------------------
template <int D>
__global__ void km_centers_kernel(const double* __restrict__ x, const double* __restrict__ w,
                                  const int64_t* members, const int64_t* offsets, int64_t ncl,
                                  const int64_t* ids, double* centers, double* masses) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  const int64_t beg = offsets[c], end = offsets[c + 1];
  const int64_t j = ids ? ids[c] : c;
  if (masses) {  // np.add.at: sequential from 0 in index order
    double s = 0.0;
    for (int64_t t = beg; t < end; ++t) s = __dadd_rn(s, w[members[t]]);
    masses[j] = s;
    return;
  }
  if (beg == end) return;
  double num[D];
#pragma unroll
  for (int d = 0; d < D; ++d) num[d] = __dmul_rn(w[members[beg]], x[members[beg] * D + d]);
  for (int64_t t = beg + 1; t < end; ++t) {
    const int64_t m = members[t];
#pragma unroll
    for (int d = 0; d < D; ++d) num[d] = __dadd_rn(num[d], __dmul_rn(w[m], x[m * D + d]));
  }
  const double ws = np_pw(beg, end - beg, [&](int64_t t) { return w[members[t]]; });
#pragma unroll
  for (int d = 0; d < D; ++d) centers[j * D + d] = __ddiv_rn(num[d], ws);
}

#define KM_DIMS(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(16) X(32) X(64)

bool dim_ok(int d) {
  switch (d) {
#define DCASE(V) case V:
    KM_DIMS(DCASE)
#undef DCASE
    return true;
    default:
      return false;
  }
}

}  // namespace

extern "C" {

size_t cntgw_km_draw_workspace(int64_t n, int nleaves) {
  const int64_t nb = (n + kScanBlock - 1) / kScanBlock;
  // leaves + internal nodes (nleaves - 1) + scalars + cdf + block sums
  return sizeof(double) * (size_t)(2 * nleaves + 4 + n + nb);
}

int cntgw_km_draw(const double* w, const double* d2, int64_t n, const int64_t* leaf_off,
                  int nleaves, const int* tree, const int* hoff, int nh, const double* u, const int* jp,
                  int64_t* out_idx, void* workspace, size_t workspace_bytes, void* stream) {
  if (!w || !leaf_off || !tree || !hoff || !u || !out_idx || !jp || n < 1 || nleaves < 1 || nh < 0)
    return fail(CNTGW_EINVAL, "km_draw: bad arguments");
  if (!workspace || workspace_bytes < cntgw_km_draw_workspace(n, nleaves))
    return fail(CNTGW_ENOSPACE, "km_draw: workspace too small");
  const int nb = (int)((n + kScanBlock - 1) / kScanBlock);
  double* p = static_cast<double*>(workspace);
  double* after = p + 2 * nleaves;
  DrawWs ws{p, after, after + 4, after + 4 + n};
  cudaStream_t s = as_stream(stream);
  km_leaf_kernel<<<(nleaves + 7) / 8, 256, 0, s>>>(w, d2, leaf_off, nleaves, ws.leaf);
  km_total_kernel<<<1, 1024, 0, s>>>(tree, hoff, nh, nleaves, ws);
  km_scan_kernel<<<nb, kScanThreads, 0, s>>>(w, d2, n, ws);
  if ((size_t)nb * sizeof(double) > 200 * 1024)
    return fail(CNTGW_EINVAL, "km_draw: n = %lld too large for the block-sum stage", (long long)n);
  if (nb * sizeof(double) > 48 * 1024)
    cudaFuncSetAttribute(km_find_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  km_find_kernel<<<1, 1024, (size_t)nb * sizeof(double), s>>>(n, nb, u, jp, ws, out_idx);
  if (n <= kExactMaxN) km_exact_kernel<<<1, 1, 0, s>>>(w, d2, n, u, jp, ws, out_idx);
  return check_launch("km_draw");
}

int cntgw_km_update_d2(const double* x, int64_t n, int d, const int64_t* idx, double* centers, int* jp,
                       double* d2, int first, void* stream) {
  if (!x || !idx || !centers || !jp || !d2 || n < 1) return fail(CNTGW_EINVAL, "km_update_d2: bad arguments");
  if (!dim_ok(d)) return fail(CNTGW_EINVAL, "km_update_d2: unsupported dimension %d", d);
  const unsigned blocks = (unsigned)((n + 255) / 256);
  cudaStream_t s = as_stream(stream);
  switch (d) {
#define DCASE(V) \
  case V: km_d2_kernel<V><<<blocks, 256, 0, s>>>(x, n, idx, centers, jp, d2, first); break;
    KM_DIMS(DCASE)
#undef DCASE
  }
  km_advance_kernel<<<1, 1, 0, s>>>(jp);  // next draw index (graph-replayable sequence)
  return check_launch("km_update_d2");
}

int cntgw_km_assign(const double* x, int64_t n, int d, const double* centers, int64_t k,
                    int64_t* assign, double* own, void* stream) {
  if (!x || !centers || !assign || !own || n < 1 || k < 1) return fail(CNTGW_EINVAL, "km_assign: bad arguments");
  if (!dim_ok(d)) return fail(CNTGW_EINVAL, "km_assign: unsupported dimension %d", d);
  const unsigned blocks = (unsigned)((n + 127) / 128);
  cudaStream_t s = as_stream(stream);
  switch (d) {
#define DCASE(V) \
  case V: km_assign_kernel<V><<<blocks, 128, 0, s>>>(x, n, centers, k, assign, own); break;
    KM_DIMS(DCASE)
#undef DCASE
  }
  return check_launch("km_assign");
}

int cntgw_km_centers(const double* x, int d, const double* w, const int64_t* members,
                     const int64_t* offsets, int64_t ncl, const int64_t* ids, double* centers,
                     double* masses, void* stream) {
  if (!x || !w || !members || !offsets || ncl < 1 || (!centers && !masses))
    return fail(CNTGW_EINVAL, "km_centers: bad arguments");
  if (!dim_ok(d)) return fail(CNTGW_EINVAL, "km_centers: unsupported dimension %d", d);
  const unsigned blocks = (unsigned)((ncl + 127) / 128);
  cudaStream_t s = as_stream(stream);
  switch (d) {
#define DCASE(V)                                                                           \
  case V:                                                                                  \
    km_centers_kernel<V><<<blocks, 128, 0, s>>>(x, w, members, offsets, ncl, ids, centers, \
                                                masses);                                   \
    break;
    KM_DIMS(DCASE)
#undef DCASE
  }
  return check_launch("km_centers");
}

}  // extern "C"
