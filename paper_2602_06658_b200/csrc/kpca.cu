// Matrix-free products with a point-cloud cost matrix for kernel PCA
// (reference kernels.py:233-345). The reference builds
// the dense N x N cost and centred kernel (and runs dense eigh or subspace
// iteration on it); here P = C V is streamed: each CTA owns 32 rows, walks
// 64-point column tiles staged in shared memory (coordinates and the V rows),
// evaluates c(x_i, x_j) on the fly in fp64 with the reference's formulas
//   sq = |x_i|^2 + |x_j|^2 - 2 x_i.x_j, clipped at 0 (kernels.py:149-154),
//   sq_euclidean / precomputed: sq;  euclidean: sqrt(sq);  p_norm: sq^(p/2);
//   exp_kernel: 2 (1 - exp(-sq / (2 sigma^2)));  c_ii = 0,
// and accumulates the B columns of V. Nothing of size N x N is stored, so the
// centred-kernel products K Q = -1/2 H C H^T Q of the subspace iteration run
// at any N. Declarations: include/cntgw_b200.h.
#include <cstdarg>
#include <cstdio>
#include <type_traits>

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

constexpr int kRows = 32, kCols = 64;  // rows per CTA (one per lane), column tile

template <int KIND>
__device__ __forceinline__ double cost_of(double sq, double par) {
  sq = fmax(sq, 0.0);
  if (KIND == CNTGW_COST_EUCLIDEAN) return sqrt(sq);
  if (KIND == CNTGW_COST_PNORM) return pow(sq, 0.5 * par);
  if (KIND == CNTGW_COST_EXP) return 2.0 * (1.0 - exp(-sq / (2.0 * par * par)));
  return sq;  // squared Euclidean (also precomputed embeddings)
}

// P[i, :] = sum_j c(x_i, x_j) V[j, :], V: n x B (ld B), x: n x d. Lane = row,
// warp = column quarter; the quarters are summed in a fixed order.
template <int KIND, int B>
__global__ void __launch_bounds__(128) cost_product_kernel(const double* __restrict__ x, int64_t n,
                                                           int d, const double* __restrict__ sqn,
                                                           const double* __restrict__ v, double par,
                                                           double* __restrict__ out) {
  extern __shared__ double sm[];
  double* sx = sm;                  // kCols x d
  double* sv = sm + kCols * d;      // kCols x B
  double* ssq = sv + kCols * B;     // kCols
  const int t = threadIdx.x;
  const int r0 = t & 31, quarter = t >> 5;
  const int64_t i = (int64_t)blockIdx.x * kRows + r0;
  const bool ok = i < n;
  double acc[B];
#pragma unroll
  for (int b = 0; b < B; ++b) acc[b] = 0.0;
  const double sqi = ok ? sqn[i] : 0.0;
  const double* xi = x + (ok ? i : 0) * d;
  for (int64_t j0 = 0; j0 < n; j0 += kCols) {
    const int cnt = (int)min((int64_t)kCols, n - j0);
    __syncthreads();
    for (int e = t; e < cnt * d; e += blockDim.x) sx[e] = x[j0 * d + e];
    for (int e = t; e < cnt * B; e += blockDim.x) sv[e] = v[j0 * B + e];
    for (int e = t; e < cnt; e += blockDim.x) ssq[e] = sqn[j0 + e];
    __syncthreads();
    for (int c = quarter; c < cnt; c += 4) {
      double dot = 0.0;
      for (int k = 0; k < d; ++k) dot = fma(xi[k], sx[c * d + k], dot);
      const double cij = (ok && j0 + c != i) ? cost_of<KIND>(sqi + ssq[c] - 2.0 * dot, par) : 0.0;
#pragma unroll
      for (int b = 0; b < B; ++b) acc[b] = fma(cij, sv[c * B + b], acc[b]);
    }
  }
  __syncthreads();
  double* red = sm;  // 4 x kRows x B
#pragma unroll
  for (int b = 0; b < B; ++b) red[(quarter * kRows + r0) * B + b] = acc[b];
  __syncthreads();
  for (int e = t; e < kRows * B; e += blockDim.x) {
    const int r = e / B, b = e - r * B;
    const int64_t row = (int64_t)blockIdx.x * kRows + r;
    if (row >= n) continue;
    double s = red[(0 * kRows + r) * B + b];
    s += red[(1 * kRows + r) * B + b];
    s += red[(2 * kRows + r) * B + b];
    s += red[(3 * kRows + r) * B + b];
    out[row * B + b] = s;
  }
}

template <int KIND>
int launch_kind(const double* x, int64_t n, int d, const double* sqn, const double* v, int bcols,
                double par, double* out, cudaStream_t s) {
  const unsigned blocks = (unsigned)((n + kRows - 1) / kRows);
  auto go = [&](auto bconst) {
    constexpr int B = decltype(bconst)::value;
    const size_t tile = sizeof(double) * ((size_t)kCols * d + (size_t)kCols * B + kCols);
    const size_t red = sizeof(double) * 4 * kRows * B;
    const size_t smem = tile > red ? tile : red;
    auto fn = cost_product_kernel<KIND, B>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fn<<<blocks, 128, smem, s>>>(x, n, d, sqn, v, par, out);
  };
  switch (bcols) {
    case 8: go(std::integral_constant<int, 8>{}); break;
    case 16: go(std::integral_constant<int, 16>{}); break;
    case 32: go(std::integral_constant<int, 32>{}); break;
    case 64: go(std::integral_constant<int, 64>{}); break;
    default: return fail(CNTGW_EINVAL, "cost_product: column count %d not in {8,16,32,64}", bcols);
  }
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(CNTGW_ECUDA, "cost_product: %s", cudaGetErrorString(e));
  }
  return CNTGW_OK;
}

}  // namespace

extern "C" {

int cntgw_cost_product(int kind, double par, const double* x, int64_t n, int d, const double* sqn,
                       const double* v, int bcols, double* out, void* stream) {
  if (!x || !sqn || !v || !out || n < 1 || d < 1 || d > 1024)
    return fail(CNTGW_EINVAL, "cost_product: bad arguments");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  switch (kind) {
    case CNTGW_COST_SQEUCLID: return launch_kind<CNTGW_COST_SQEUCLID>(x, n, d, sqn, v, bcols, par, out, s);
    case CNTGW_COST_EUCLIDEAN: return launch_kind<CNTGW_COST_EUCLIDEAN>(x, n, d, sqn, v, bcols, par, out, s);
    case CNTGW_COST_PNORM: return launch_kind<CNTGW_COST_PNORM>(x, n, d, sqn, v, bcols, par, out, s);
    case CNTGW_COST_EXP: return launch_kind<CNTGW_COST_EXP>(x, n, d, sqn, v, bcols, par, out, s);
    default: return fail(CNTGW_EINVAL, "cost_product: unknown cost kind %d", kind);
  }
}

}  // extern "C"
