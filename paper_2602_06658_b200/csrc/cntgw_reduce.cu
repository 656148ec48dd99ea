// C ABI for K4-K7: fused plan reductions, operator application, outer-step
// reductions and the loss-constant moments. Declarations: include/cntgw_b200.h.
#include <cstdarg>
#include <cstdio>
#include <string>

#include "common.cuh"
#include "reduce.cuh"

using namespace cntgw;

namespace cntgw {
int set_error(int code, const char* msg);
}

namespace {

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

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
  if (e != cudaSuccess) cudaGetLastError();
  if (e != cudaSuccess) return fail(CNTGW_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return CNTGW_OK;
}

int e_padded(int e) { return e <= 2 ? 2 : e <= 4 ? 4 : e <= 8 ? 8 : e <= 16 ? 16 : e <= 32 ? 32 : e <= 64 ? 64 : -1; }

// [Y (e_real, zero-padded to e_pad) | s | pad] fp64 accumulation records
__global__ void pack_acc_kernel(const double* y, int64_t ld, int e_real, int e_pad, int stride,
                                const double* s, int64_t m, int64_t mpad, double* out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= mpad) return;
  double* r = out + j * stride;
  for (int k = 0; k < stride; ++k) r[k] = 0.0;
  if (j < m) {
    for (int k = 0; k < e_real; ++k) r[k] = y[j * ld + k];
    r[e_pad] = s[j];
  }
}

// columns per shared-memory stage: the largest of 256/128/64 whose two stages fit in 200 KB
template <int KD, int E>
constexpr int plan_tile() {
  constexpr int per_col = (ColLayout<double, KD, 1>::kStride + AccLayout<E>::kStride) * 8 * 2;
  return per_col * 256 <= 200 * 1024 ? 256 : (per_col * 128 <= 200 * 1024 ? 128 : 64);
}

template <int KD, int E>
int launch_plan_reduce(const PlanReduceArgs& a, cudaStream_t s) {
  constexpr int G = 4;
  constexpr int TILE = plan_tile<KD, E>();
  auto kern = plan_reduce_kernel<KD, E, G, TILE>;
  const size_t smem =
      2 * (size_t)TILE * (ColLayout<double, KD, 1>::kStride + AccLayout<E>::kStride) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const unsigned blocks = (unsigned)((a.n + 127) / 128);
  kern<<<blocks, 128, smem, s>>>(a);
  return check_launch("plan_reduce_kernel");
}

int64_t reduce_blocks(int64_t n) {
  int64_t b = (n + 1023) / 1024;
  if (b > 1024) b = 1024;
  return b < 1 ? 1 : b;
}

}  // namespace

extern "C" {

size_t cntgw_plan_reduce_workspace(int64_t n, int64_t m, int kd, int e) {
  (void)n;
  (void)kd;
  const int ep = e_padded(e);
  if (ep < 0) return 0;
  return (size_t)cntgw_cols_padded(m) * (size_t)((ep + 1 + 1) / 2 * 2) * sizeof(double);
}

int cntgw_plan_reduce(const cntgw_sweep_state* st, int kd, int e, const double* row_feat,
                      int64_t ld_row, const double* row_sq, const double* f_tilde,
                      const double* log2a, const double* col_rec, const double* col_acc,
                      int64_t ld_acc, const double* col_s, int64_t n, int64_t m, double* row_mass,
                      double* pi_y, double* pi_s, int64_t* argmax, void* workspace,
                      size_t workspace_bytes, void* stream) {
  const int ep = e_padded(e);
  if (ep < 0 || e < 1) return fail(CNTGW_EINVAL, "plan_reduce: unsupported e=%d", e);
  if (!st || !row_feat || !row_sq || !f_tilde || !log2a || !col_rec || !col_acc || !col_s ||
      !row_mass || !pi_y || !pi_s || !argmax || n < 1 || m < 1)
    return fail(CNTGW_EINVAL, "plan_reduce: bad arguments");
  const size_t need = cntgw_plan_reduce_workspace(n, m, kd, e);
  if (!workspace || workspace_bytes < need)
    return fail(CNTGW_ENOSPACE, "plan_reduce workspace %zu < %zu", workspace_bytes, need);
  cudaStream_t s = as_stream(stream);
  const int stride = (ep + 1 + 1) / 2 * 2;
  const int64_t mpad = cntgw_cols_padded(m);
  double* acc = static_cast<double*>(workspace);
  const int th = 256;
  pack_acc_kernel<<<(unsigned)((mpad + th - 1) / th), th, 0, s>>>(col_acc, ld_acc, e, ep, stride,
                                                                  col_s, m, mpad, acc);
  int rc = check_launch("pack_acc");
  if (rc) return rc;
  PlanReduceArgs a{};
  a.st = st;
  a.row_feat = row_feat;
  a.ld_row = ld_row;
  a.row_sq = row_sq;
  a.f_tilde = f_tilde;
  a.log2a = log2a;
  a.col_rec = col_rec;
  a.col_acc = acc;
  a.n = n;
  a.m = m;
  a.row_mass = row_mass;
  a.pi_y = pi_y;
  a.e_real = e;
  a.pi_s = pi_s;
  a.argmax = argmax;
  // the kernel's E must be the padded accumulation width (record layout)
#define PR(KD_, E_) \
  if (kd == KD_ && ep == E_) return launch_plan_reduce<KD_, E_>(a, s);
  PR(1, 2) PR(2, 2)
  PR(1, 4) PR(2, 4) PR(3, 4) PR(4, 4)
  PR(1, 8) PR(2, 8) PR(3, 8) PR(4, 8) PR(8, 8)
  PR(1, 16) PR(2, 16) PR(3, 16) PR(4, 16) PR(8, 16) PR(16, 16)
  PR(1, 32) PR(2, 32) PR(3, 32) PR(4, 32) PR(8, 32) PR(16, 32) PR(32, 32)
  PR(1, 64) PR(2, 64) PR(3, 64) PR(4, 64) PR(8, 64) PR(16, 64) PR(32, 64) PR(64, 64)
#undef PR
  return fail(CNTGW_EINVAL, "plan_reduce: unsupported kd=%d e=%d", kd, e);
}

int cntgw_apply_operator(const double* op, int dout, int din, const double* feat, int64_t ld,
                         int64_t n, double* out64, float* out32, int64_t ld_out, void* stream) {
  if (!op || !feat || !out64 || dout < 1 || din < 1 || dout * din > 64 * 64 || n < 1 || ld_out < dout)
    return fail(CNTGW_EINVAL, "apply_operator: bad arguments");
  const int th = 128;
  apply_operator_kernel<<<(unsigned)((n + th - 1) / th), th, sizeof(double) * dout * din,
                          as_stream(stream)>>>(op, dout, din, feat, ld, n, out64, out32, ld_out);
  return check_launch("apply_operator");
}

size_t cntgw_outer_reduce_workspace(int64_t n, int d, int e) {
  const int64_t nb = reduce_blocks(n);
  const int stride = 16 + d * e;
  const int64_t colb = 296;
  const int64_t a = nb * stride, b = colb * 8;
  return sizeof(double) * (size_t)(a > b ? a : b);
}

int cntgw_outer_reduce_rows(const double* x, int64_t ldx, int d, const double* pi_y, int e,
                            const double* row_mass, const double* pi_s, const double* f_tilde,
                            const double* s_half, const double* a, int64_t n, double* acc,
                            void* workspace, size_t workspace_bytes, void* stream) {
  if (!x || !pi_y || !row_mass || !pi_s || !f_tilde || !s_half || !a || !acc || n < 1 || d < 1 ||
      e < 1)
    return fail(CNTGW_EINVAL, "outer_reduce_rows: bad arguments");
  const size_t need = cntgw_outer_reduce_workspace(n, d, e);
  if (!workspace || workspace_bytes < need)
    return fail(CNTGW_ENOSPACE, "outer_reduce workspace %zu < %zu", workspace_bytes, need);
  cudaStream_t s = as_stream(stream);
  const int64_t nb = reduce_blocks(n);
  const int64_t rpb = (n + nb - 1) / nb;
  const int stride = 16 + d * e;
  double* part = static_cast<double*>(workspace);
  cudaMemsetAsync(part, 0, sizeof(double) * nb * stride, s);
  outer_rows_kernel<<<(unsigned)nb, kRedThreads, 0, s>>>(x, ldx, d, pi_y, e, e, row_mass, pi_s,
                                                         f_tilde, s_half, a, n, rpb, part, stride);
  sum_partials_kernel<<<(stride + 255) / 256, 256, 0, s>>>(part, (int)nb, stride, stride, acc);
  return check_launch("outer_reduce_rows");
}

int cntgw_outer_reduce_cols(const cntgw_sweep_state* st, const double* g_tilde,
                            const double* g_tent, const double* t_half, const double* b, int64_t m,
                            double* acc, void* workspace, size_t workspace_bytes, void* stream) {
  if (!st || !g_tilde || !g_tent || !t_half || !b || !acc || m < 1)
    return fail(CNTGW_EINVAL, "outer_reduce_cols: bad arguments");
  const int nb = 296;
  if (!workspace || workspace_bytes < sizeof(double) * nb * 8)
    return fail(CNTGW_ENOSPACE, "outer_reduce_cols workspace too small");
  cudaStream_t s = as_stream(stream);
  double* part = static_cast<double*>(workspace);
  outer_cols_kernel<<<nb, kRedThreads, 0, s>>>(st, CNTGW_F64, g_tilde, g_tent, t_half, b, m, part);
  sum_partials_kernel<<<1, 32, 0, s>>>(part, nb, 8, 8, acc);
  return check_launch("outer_reduce_cols");
}

size_t cntgw_moments_workspace(int64_t n, int d) {
  const int64_t nb = reduce_blocks(n);
  return sizeof(double) * (size_t)(nb * (2 + d * d + 1 + d) + (2 + d * d + 1 + d));
}

int cntgw_moments(const double* x, int64_t ldx, int d, const double* w, int64_t n, double* out,
                  void* workspace, size_t workspace_bytes, void* stream) {
  if (!x || !w || !out || n < 1 || d < 1 || d > 64) return fail(CNTGW_EINVAL, "moments: bad arguments");
  const size_t need = cntgw_moments_workspace(n, d);
  if (!workspace || workspace_bytes < need)
    return fail(CNTGW_ENOSPACE, "moments workspace %zu < %zu", workspace_bytes, need);
  cudaStream_t s = as_stream(stream);
  const int64_t nb = reduce_blocks(n);
  const int64_t rpb = (n + nb - 1) / nb;
  const int stride = 2 + d * d + 1 + d;
  double* part = static_cast<double*>(workspace);
  double* mean = part + nb * stride;  // [T, mean (d)]
  moments_pass1_kernel<<<(unsigned)nb, kRedThreads, 0, s>>>(x, ldx, d, w, n, rpb, part, stride);
  sum_partials_kernel<<<1, 128, 0, s>>>(part, (int)nb, stride, 1 + d, mean);
  moments_pass2_kernel<<<(unsigned)nb, kRedThreads, 0, s>>>(x, ldx, d, w, n, rpb, mean, part, stride);
  // out = [T, sum w|xc|^4, sum w|xc|^2, cov (d x d)]
  sum_partials_kernel<<<(2 + d * d + 255) / 256, 256, 0, s>>>(part, (int)nb, stride, 2 + d * d, out + 1);
  cudaMemcpyAsync(out, mean, sizeof(double), cudaMemcpyDeviceToDevice, s);
  return check_launch("moments");
}

}  // extern "C"
