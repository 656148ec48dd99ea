// C ABI of the B200-native CNT-GW hot path: kernel dispatch, argument checks,
// workspace sizing and error reporting. Declarations: include/cntgw_b200.h.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "softmin_fma.cuh"
#include "sweep.cuh"

using namespace cntgw;

namespace {

thread_local std::string g_last_error;

}  // namespace

namespace cntgw {
int set_error(int code, const char* msg) {
  g_last_error = msg;
  return code;
}
}  // namespace cntgw

namespace {

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(CNTGW_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return CNTGW_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
      sms = 148;
  }
  return sms;
}

bool kd_supported(int kd) {
  return kd == 1 || kd == 2 || kd == 3 || kd == 4 || kd == 8 || kd == 16 || kd == 32 || kd == 64;
}

// ---- softmin dispatch table --------------------------------------------------
struct SoftminCfg {
  int R;        // rows per thread
  int minb;     // min CTAs per SM (launch bounds)
  int stride;   // column record stride (floats)
  size_t smem;  // dynamic shared memory bytes
};

template <int KD, int SQ>
constexpr int rows_per_thread() {
  return KD <= 8 ? 8 : (KD <= 16 ? 4 : 2);
}
template <int KD, int SQ>
constexpr int min_blocks() {
  return KD <= 4 ? 4 : (KD <= 16 ? 3 : (KD <= 32 ? 2 : 1));
}

template <int KD, int SQ>
SoftminCfg softmin_cfg() {
  SoftminCfg c;
  c.R = rows_per_thread<KD, SQ>();
  c.minb = min_blocks<KD, SQ>();
  c.stride = ColLayout<KD, SQ>::kStride;
  c.smem = 2 * (size_t)kColTile * c.stride * sizeof(float);
  return c;
}

#define KD_SQ_SWITCH(kd, sq, FN)                     \
  switch ((kd) * 2 + ((sq) ? 1 : 0)) {              \
    case 2: FN(1, 0); break;                        \
    case 3: FN(1, 1); break;                        \
    case 4: FN(2, 0); break;                        \
    case 5: FN(2, 1); break;                        \
    case 6: FN(3, 0); break;                        \
    case 7: FN(3, 1); break;                        \
    case 8: FN(4, 0); break;                        \
    case 9: FN(4, 1); break;                        \
    case 16: FN(8, 0); break;                       \
    case 17: FN(8, 1); break;                       \
    case 32: FN(16, 0); break;                      \
    case 33: FN(16, 1); break;                      \
    case 64: FN(32, 0); break;                      \
    case 65: FN(32, 1); break;                      \
    case 128: FN(64, 0); break;                     \
    case 129: FN(64, 1); break;                     \
    default: return fail(CNTGW_EINVAL, "unsupported feature width kd=%d", kd); \
  }

template <int KD, int SQ>
void* softmin_kernel_ptr() {
  constexpr int R = rows_per_thread<KD, SQ>();
  constexpr int G = KD <= 32 ? 4 : 2;
  return (void*)softmin_fma_kernel<KD, SQ, R, G, min_blocks<KD, SQ>()>;
}

struct Plan {
  int row_tiles;
  int nchunks;
  int64_t chunk_cols;
};

// Split the padded columns into chunks so that row_tiles * nchunks CTAs fill
// whole waves of the resident-CTA capacity (tail < 3% when possible).
Plan plan_softmin(int64_t n, int64_t m, int R, void* kernel, size_t smem) {
  Plan p;
  const int64_t rows_per_cta = 128LL * R;
  p.row_tiles = (int)((n + rows_per_cta - 1) / rows_per_cta);
  const int64_t tiles = (m + kColTile - 1) / kColTile;
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 128, smem);
  if (occ < 1) occ = 1;
  const int64_t resident = (int64_t)num_sms() * occ;
  int best_c = 1;
  double best_eff = -1.0;
  const int64_t max_c = tiles < 64 ? tiles : 64;
  for (int64_t c = 1; c <= max_c; ++c) {
    const int64_t cpc = (tiles + c - 1) / c;  // tiles per chunk
    const int64_t cc = (tiles + cpc - 1) / cpc;
    if (cc != c) continue;
    const int64_t ctas = (int64_t)p.row_tiles * c;
    const int64_t waves = (ctas + resident - 1) / resident;
    double eff = (double)ctas / (double)(waves * resident);
    if (ctas < 2 * resident) eff *= 0.5 + 0.5 * (double)ctas / (2.0 * resident);
    if (eff > best_eff + 0.03) {
      best_eff = eff;
      best_c = (int)c;
    }
  }
  const int64_t cpc = (tiles + best_c - 1) / best_c;
  p.chunk_cols = cpc * kColTile;
  p.nchunks = (int)((tiles + cpc - 1) / cpc);
  return p;
}

template <int KD, int SQ>
int launch_softmin(const SoftminArgs& a0, void* ws, size_t ws_bytes, cudaStream_t s) {
  constexpr int R = rows_per_thread<KD, SQ>();
  constexpr int G = KD <= 32 ? 4 : 2;
  auto kern = softmin_fma_kernel<KD, SQ, R, G, min_blocks<KD, SQ>()>;
  SoftminCfg c = softmin_cfg<KD, SQ>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
    attr = true;
  }
  Plan p = plan_softmin(a0.n, a0.m, R, (void*)kern, c.smem);
  SoftminArgs a = a0;
  a.chunk_cols = p.chunk_cols;
  a.nchunks = p.nchunks;
  if (p.nchunks > 1) {
    const size_t need = 2 * sizeof(float) * (size_t)p.nchunks * (size_t)a.n;
    if (ws == nullptr || ws_bytes < need)
      return fail(CNTGW_ENOSPACE, "softmin workspace %zu < %zu bytes", ws_bytes, need);
    a.part_max = static_cast<float*>(ws);
    a.part_sum = a.part_max + (size_t)p.nchunks * a.n;
  }
  dim3 grid(p.row_tiles, p.nchunks);
  kern<<<grid, 128, c.smem, s>>>(a);
  int rc = check_launch("softmin_fma_kernel");
  if (rc) return rc;
  if (p.nchunks > 1) {
    const int th = 256;
    lse_combine_kernel<<<(unsigned)((a.n + th - 1) / th), th, 0, s>>>(
        a.st, a.skip, a.part_max, a.part_sum, p.nchunks, a.n, a.row_add, a.out, a.out_max,
        a.out_sum);
    rc = check_launch("lse_combine_kernel");
  }
  return rc;
}

template <int KD, int SQ>
size_t softmin_ws(int64_t n, int64_t m) {
  constexpr int R = rows_per_thread<KD, SQ>();
  constexpr int G = KD <= 32 ? 4 : 2;
  auto kern = softmin_fma_kernel<KD, SQ, R, G, min_blocks<KD, SQ>()>;
  SoftminCfg c = softmin_cfg<KD, SQ>();
  Plan p = plan_softmin(n, m, R, (void*)kern, c.smem);
  return p.nchunks > 1 ? 2 * sizeof(float) * (size_t)p.nchunks * (size_t)n : 0;
}

// ---- column record packing ------------------------------------------------------
__global__ void prep_cols_kernel(const cntgw_sweep_state* st, int kd, int sq_flag, int stride,
                                 const float* feat, int64_t ld, const float* sq, const float* pot,
                                 const float* log2w, int64_t m, int64_t mpad, float* rec) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= mpad) return;
  float* r = rec + j * stride;
  const float lam = st->lam;
  if (j < m) {
    const float two_lam = 2.0f * lam;
    for (int k = 0; k < kd; ++k) r[k] = -two_lam * feat[j * ld + k];
    if (sq_flag) r[kd] = -st->sqrt_lam * sq[j];
    const double beta = (double)lam * (pot ? (double)pot[j] : 0.0) + (double)log2w[j];
    r[kd + sq_flag] = (float)(-beta);
  } else {
    for (int k = 0; k < kd + sq_flag; ++k) r[k] = 0.f;
    r[kd + sq_flag] = CUDART_INF_F;  // -beta = +inf: exactly zero weight
  }
  for (int k = kd + sq_flag + 1; k < stride; ++k) r[k] = 0.f;
}

// ---- dense cost half-update -----------------------------------------------------
__global__ void softmin_dense_kernel(const cntgw_sweep_state* st, int skip, const float* cost,
                                     int64_t ld, const float* pot, const float* log2w,
                                     const float* row_add, int64_t n, int64_t m, float* out) {
  if (skip_now(st, skip)) return;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const float lam = st->lam;
  float mx = -CUDART_INF_F, sm = 0.f;
  const float* ci = cost + i * ld;
  for (int64_t j = lane; j < m; j += 32) {
    const float t = (float)((double)lam * (double)pot[j] + (double)log2w[j]) - lam * ci[j];
    if (t > mx) {
      sm = sm * ex2(mx - t) + 1.0f;
      mx = t;
    } else {
      sm += ex2(t - mx);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, mx, o);
    const float os = __shfl_xor_sync(0xffffffffu, sm, o);
    const float nm = fmaxf(mx, om);
    sm = (sm > 0.f ? sm * ex2(mx - nm) : 0.f) + (os > 0.f ? os * ex2(om - nm) : 0.f);
    mx = nm;
  }
  if (lane == 0) out[i] = (row_add ? row_add[i] : 0.f) - (mx + log2f(sm)) * st->inv_lam;
}

}  // namespace

// ================================================================================
extern "C" {

int cntgw_abi_version(void) { return CNTGW_ABI_VERSION; }
const char* cntgw_last_error(void) { return g_last_error.c_str(); }
int cntgw_sweep_state_size(void) { return (int)sizeof(cntgw_sweep_state); }

int cntgw_col_stride(int kd, int sq) {
  if (!kd_supported(kd)) return fail(CNTGW_EINVAL, "unsupported feature width kd=%d", kd);
  return (kd + (sq ? 1 : 0) + 1 + 3) / 4 * 4;
}
int64_t cntgw_cols_padded(int64_t m) { return (m + kColTile - 1) / kColTile * kColTile; }

int cntgw_sweep_init(cntgw_sweep_state* st, double eps, double anneal_from, double threshold,
                     int max_sweeps, int mode, void* stream) {
  if (!st) return fail(CNTGW_EINVAL, "null sweep state");
  if (!(eps > 0.0)) return fail(CNTGW_EINVAL, "eps must be positive");
  sweep_init_kernel<<<1, 1, 0, as_stream(stream)>>>(st, eps, anneal_from, threshold, max_sweeps, mode);
  return check_launch("sweep_init");
}

int cntgw_sweep_begin(cntgw_sweep_state* st, void* stream) {
  sweep_begin_kernel<<<1, 1, 0, as_stream(stream)>>>(st);
  return check_launch("sweep_begin");
}

int cntgw_gap_blocks(int64_t n) { return gap_blocks(n); }

int cntgw_sweep_gap(cntgw_sweep_state* st, int side, const double* w, const float* pot,
                    const float* tent, int64_t n, double* partials, void* stream) {
  (void)side;
  if (n < 1) return fail(CNTGW_EINVAL, "empty marginal");
  sweep_gap_kernel<<<gap_blocks(n), kGapThreads, 0, as_stream(stream)>>>(st, w, pot, tent, n, partials);
  return check_launch("sweep_gap");
}

int cntgw_sweep_finish(cntgw_sweep_state* st, const double* partials_r, int64_t n,
                       const double* partials_c, int64_t m, void* stream) {
  sweep_finish_kernel<<<1, 1, 0, as_stream(stream)>>>(st, partials_r, gap_blocks(n), partials_c,
                                                       partials_c ? gap_blocks(m) : 0);
  return check_launch("sweep_finish");
}

int cntgw_sweep_apply(const cntgw_sweep_state* st, float* pot, const float* tent, int64_t n,
                      int average, void* stream) {
  const int th = 256;
  int64_t b = (n + th - 1) / th;
  if (b > 4 * num_sms()) b = 4 * num_sms();
  sweep_apply_kernel<<<(unsigned)b, th, 0, as_stream(stream)>>>(st, pot, tent, n, average);
  return check_launch("sweep_apply");
}

int cntgw_prep_cols(const cntgw_sweep_state* st, int kd, int sq_flag, const float* feat, int64_t ld,
                    const float* sq, const float* pot, const float* log2w, int64_t m, float* rec,
                    void* stream) {
  if (!kd_supported(kd)) return fail(CNTGW_EINVAL, "unsupported feature width kd=%d", kd);
  if (sq_flag && !sq) return fail(CNTGW_EINVAL, "sq_flag set without sq values");
  if (!st || !feat || !log2w || !rec || m < 1) return fail(CNTGW_EINVAL, "prep_cols: bad arguments");
  const int stride = cntgw_col_stride(kd, sq_flag);
  const int64_t mpad = cntgw_cols_padded(m);
  const int th = 256;
  prep_cols_kernel<<<(unsigned)((mpad + th - 1) / th), th, 0, as_stream(stream)>>>(
      st, kd, sq_flag ? 1 : 0, stride, feat, ld, sq, pot, log2w, m, mpad, rec);
  return check_launch("prep_cols");
}

size_t cntgw_softmin_workspace(int64_t n, int64_t m, int kd, int sq_flag) {
#define WS_CASE(KD_, SQ_) return softmin_ws<KD_, SQ_>(n, m)
  switch (kd * 2 + (sq_flag ? 1 : 0)) {
    case 2: WS_CASE(1, 0);
    case 3: WS_CASE(1, 1);
    case 4: WS_CASE(2, 0);
    case 5: WS_CASE(2, 1);
    case 6: WS_CASE(3, 0);
    case 7: WS_CASE(3, 1);
    case 8: WS_CASE(4, 0);
    case 9: WS_CASE(4, 1);
    case 16: WS_CASE(8, 0);
    case 17: WS_CASE(8, 1);
    case 32: WS_CASE(16, 0);
    case 33: WS_CASE(16, 1);
    case 64: WS_CASE(32, 0);
    case 65: WS_CASE(32, 1);
    case 128: WS_CASE(64, 0);
    case 129: WS_CASE(64, 1);
    default: return 0;
  }
#undef WS_CASE
}

int cntgw_softmin(const cntgw_sweep_state* st, int skip_if_done, int kd, int sq_flag,
                  const float* row_feat, int64_t ld_row, const float* row_sq, const float* row_add,
                  const float* col_rec, int64_t n, int64_t m, float* out, float* out_max,
                  float* out_sum, void* workspace, size_t workspace_bytes, void* stream) {
  if (!st || !row_feat || !col_rec || n < 1 || m < 1)
    return fail(CNTGW_EINVAL, "softmin: bad arguments (n=%lld m=%lld)", (long long)n, (long long)m);
  if (sq_flag && !row_sq) return fail(CNTGW_EINVAL, "softmin: sq_flag without row_sq");
  if (!out && !(out_max && out_sum)) return fail(CNTGW_EINVAL, "softmin: no output");
  SoftminArgs a{};
  a.st = st;
  a.skip = skip_if_done;
  a.row_feat = row_feat;
  a.ld_row = ld_row;
  a.row_sq = row_sq;
  a.row_add = row_add;
  a.col_rec = col_rec;
  a.n = n;
  a.m = m;
  a.out = out;
  a.out_max = out_max;
  a.out_sum = out_sum;
  cudaStream_t s = as_stream(stream);
#define SM_CASE(KD_, SQ_) return launch_softmin<KD_, SQ_>(a, workspace, workspace_bytes, s)
  KD_SQ_SWITCH(kd, sq_flag, SM_CASE)
#undef SM_CASE
  return CNTGW_OK;
}

int cntgw_lse_finalize(const cntgw_sweep_state* st, int skip_if_done, const float* mx,
                       const float* sm, const float* row_add, int64_t n, float* out, void* stream) {
  const int th = 256;
  lse_combine_kernel<<<(unsigned)((n + th - 1) / th), th, 0, as_stream(stream)>>>(
      st, skip_if_done, mx, sm, 1, n, row_add, out, nullptr, nullptr);
  return check_launch("lse_finalize");
}

int cntgw_softmin_dense(const cntgw_sweep_state* st, int skip_if_done, const float* cost,
                        int64_t ld, const float* pot, const float* log2w, const float* row_add,
                        int64_t n, int64_t m, float* out, void* stream) {
  if (!st || !cost || !pot || !log2w || !out || n < 1 || m < 1)
    return fail(CNTGW_EINVAL, "softmin_dense: bad arguments");
  const int warps = 8;
  softmin_dense_kernel<<<(unsigned)((n + warps - 1) / warps), warps * 32, 0, as_stream(stream)>>>(
      st, skip_if_done, cost, ld, pot, log2w, row_add, n, m, out);
  return check_launch("softmin_dense");
}

}  // extern "C"
