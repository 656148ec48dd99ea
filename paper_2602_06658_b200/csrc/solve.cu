// Solve-level C ABI: the CNT-GW feature-space solve (reference solve_cnt_gw,
// solvers.py:628-632; state and step :285-350; outer control :556-625) as a
// native driver over the library's own kernels — what a non-Python caller
// links against. One handle per device and problem: cntgw_solver_create
// allocates every buffer once (fixed addresses), cntgw_solver_run captures
// the whole solve as ONE CUDA graph (outer conditional WHILE node; inside it
// K5, the Sinkhorn loop — a fixed number of captured sweeps or a nested WHILE
// that exits on the device-side threshold decision — the final g-tentative,
// K4, K7 and cntgw_outer_finish) and launches it once; the host reads back
// only the trace and the stop flags. With a communicator the rows are this
// rank's shard and every exchange is an NCCL collective inside the graph.
//
// It issues exactly the calls of the Python package's device solve
// (paper_2602_06658_b200/solvers.py _GwDevice + _DeviceSolve), so the two
// give the same trajectories (tests/test_gpu_native_solve.py).
#include <cstdarg>
#include <cstdio>
#include <cstring>

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

int cuda_ok(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return CNTGW_OK;
  cudaGetLastError();
  return fail(CNTGW_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define TRY(expr)              \
  do {                         \
    const int rc_ = (expr);    \
    if (rc_) return rc_;       \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int padded_kd(int k) {
  const int kds[] = {1, 2, 3, 4, 8, 16, 32, 64};
  for (int v : kds)
    if (k <= v) return v;
  return -1;
}

__global__ void half_sq_kernel(const double* x, int64_t n, int d, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int k = 0; k < d; ++k) s += x[i * d + k] * x[i * d + k];
  out[i] = 0.5 * s;
}

__global__ void pad_copy_kernel(const double* x, int64_t n, int d, int kd, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int k = 0; k < kd; ++k) out[i * kd + k] = k < d ? x[i * d + k] : 0.0;
}

__global__ void log2_kernel(const double* w, int64_t n, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = log2(w[i]);
}

__global__ void square_kernel(const double* s, int64_t n, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = s[i] * s[i];
}

__global__ void to_f32_kernel(const double* in, int64_t n, float* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (float)in[i];
}

__global__ void transpose_kernel(const double* g, int d, int e, double* gt) {  // gt (e x d) = g^T
  for (int k = threadIdx.x; k < d * e; k += blockDim.x) gt[(k % e) * d + k / e] = g[k];
}

unsigned blocks_for(int64_t n, int th = 256) { return (unsigned)((n + th - 1) / th); }

template <typename T>
int alloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return CNTGW_OK;
  return cuda_ok(cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * count), "cudaMalloc");
}

struct Side {
  int64_t n = 0;
  double* feat64 = nullptr;  // n x kd
  float* feat32 = nullptr;
  double* sq = nullptr;       // half squared norms
  float* sq32 = nullptr;
  const double* w = nullptr;
  double* log2w = nullptr;
  const int64_t* order = nullptr;
};

struct Half {
  Side* rows = nullptr;
  Side* cols = nullptr;
  double* rec = nullptr;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  void* f64s_rows = nullptr;
};

}  // namespace

extern "C" {
// prototypes of the library's own entry points (include/cntgw_b200.h)
int cntgw_col_stride(int prec, int kd, int sq);
int64_t cntgw_cols_padded(int64_t m);
int cntgw_gap_blocks(int64_t n);
size_t cntgw_softmin_workspace(int prec, int64_t n, int64_t m, int kd, int sq_flag);
size_t cntgw_f64s_rows_bytes(int64_t n, int kd);
size_t cntgw_plan_reduce_workspace(int64_t n, int64_t m, int kd, int e);
size_t cntgw_plan_reduce_ctr_workspace(int64_t m, int e);
size_t cntgw_outer_reduce_workspace(int64_t n, int d, int e);
size_t cntgw_moments_workspace(int64_t n, int d);
}

struct cntgw_solver {
  cntgw_solve_config cfg;
  int64_t n, m, n_gap;
  int d, e, k, kd;
  bool proj_rows;
  const double *x, *y, *a, *b;
  Side src, tgt;
  Half fwd, bwd;
  cntgw_comm* comm;
  // loop
  cntgw_sweep_state* st = nullptr;
  double *ft = nullptr, *gt = nullptr, *pr = nullptr, *pc = nullptr, *pr_glob = nullptr;
  double *mx = nullptr, *sm = nullptr, *mglob = nullptr;  // sharded g-update partials
  // K4 / K7 / outer
  double *r = nullptr, *pi_y = nullptr, *pi_s = nullptr;
  int64_t* argmax = nullptr;
  void* ws_plan = nullptr;
  size_t ws_plan_bytes = 0;
  double* acc = nullptr;
  void* ws_outer = nullptr;
  size_t ws_outer_bytes = 0;
  double* gamma_t = nullptr;  // e x d (rows side projection)
  cntgw_outer_state* os = nullptr;
  double* trace = nullptr;
};

namespace {

int half_alloc(Half& h, Side* rows, Side* cols, int kd, int prec) {
  h.rows = rows;
  h.cols = cols;
  const int s64 = cntgw_col_stride(CNTGW_F64, kd, 1), s32 = cntgw_col_stride(CNTGW_F32, kd, 1);
  if (s64 < 0 || s32 < 0) return s64 < 0 ? s64 : s32;
  const size_t per_col = (size_t)s64 * 8 > (size_t)s32 * 4 ? (size_t)s64 * 8 : (size_t)s32 * 4;
  TRY(alloc(reinterpret_cast<char**>(&h.rec), per_col * (size_t)cntgw_cols_padded(cols->n)));
  h.ws_bytes = cntgw_softmin_workspace(prec, rows->n, cols->n, kd, 1);
  if (h.ws_bytes < 16) h.ws_bytes = 16;
  TRY(alloc(reinterpret_cast<char**>(&h.ws), h.ws_bytes));
  if (prec == CNTGW_F64S) TRY(alloc(reinterpret_cast<char**>(&h.f64s_rows), cntgw_f64s_rows_bytes(rows->n, kd)));
  return CNTGW_OK;
}

void half_free(Half& h) {
  cudaFree(h.rec);
  cudaFree(h.ws);
  cudaFree(h.f64s_rows);
}

// out_rows = S(pot_cols) (engine.HalfUpdate pack + stream); partials when mx/sm are set
int half_apply(cntgw_solver* s, Half& h, const double* pot, double* out, int skip, double* mx, double* sm,
               cudaStream_t st) {
  const int prec = s->cfg.precision, kd = s->kd;
  Side& c = *h.cols;
  Side& r = *h.rows;
  if (prec == CNTGW_F64S) {
    // (the rows blocks are gathered once per loop in set_gamma; within a loop only the bias
    // column of the records moves)
    TRY(cntgw_update_cols_f64s(s->st, kd, 1, c.feat64, kd, c.sq, pot, c.log2w, c.order, c.n, h.rec, st));
    return cntgw_softmin(s->st, skip, prec, kd, 1, h.f64s_rows, kd, r.sq, nullptr, h.rec, r.n, c.n, out, mx, sm,
                         h.ws, h.ws_bytes, st);
  }
  const bool f32 = prec == CNTGW_F32;
  TRY(cntgw_prep_cols(s->st, prec, kd, 1, f32 ? (const void*)c.feat32 : (const void*)c.feat64, kd,
                      f32 ? (const void*)c.sq32 : (const void*)c.sq, pot, c.log2w, c.n, h.rec, st));
  return cntgw_softmin(s->st, skip, prec, kd, 1, f32 ? (const void*)r.feat32 : (const void*)r.feat64, kd,
                       f32 ? (const void*)r.sq32 : (const void*)r.sq, nullptr, h.rec, r.n, c.n, out, mx, sm, h.ws,
                       h.ws_bytes, st);
}

// g-tentative over every rank's rows (dist.RowShardComm.g_update)
int g_update(cntgw_solver* s, const double* f, double* out, int skip, cudaStream_t st) {
  if (!s->comm) return half_apply(s, s->bwd, f, out, skip, nullptr, nullptr, st);
  TRY(half_apply(s, s->bwd, f, nullptr, skip, s->mx, s->sm, st));
  TRY(cntgw_comm_combine_lse(s->comm, s->mx, s->mglob, s->sm, s->m, st));
  return cntgw_lse_finalize(s->st, skip, s->cfg.precision, s->mglob, s->sm, nullptr, s->m, out, st);
}

int sweep(cntgw_solver* s, double* f, double* g, cudaStream_t st) {
  TRY(cntgw_sweep_begin(s->st, st));
  const bool sym = s->cfg.mode == 1;
  TRY(half_apply(s, s->fwd, g, s->ft, 1, nullptr, nullptr, st));
  if (sym) TRY(g_update(s, f, s->gt, 1, st));
  TRY(cntgw_sweep_gap(s->st, s->a, f, s->ft, s->n, s->pr, st));
  if (sym) TRY(cntgw_sweep_gap(s->st, s->b, g, s->gt, s->m, s->pc, st));
  const double* pr = s->pr;
  if (s->comm) {  // row-gap partials over every rank (out of place: no feedback)
    TRY(cntgw_comm_allreduce(s->comm, s->pr, s->pr_glob, cntgw_gap_blocks(s->n_gap), 0, st));
    pr = s->pr_glob;
  }
  TRY(cntgw_sweep_finish(s->st, pr, s->n_gap, sym ? s->pc : nullptr, sym ? s->m : 0, st));
  TRY(cntgw_sweep_apply(s->st, f, s->ft, s->n, sym ? 1 : 0, st));
  if (sym) return cntgw_sweep_apply(s->st, g, s->gt, s->m, 1, st);
  return g_update(s, f, g, 1, st);
}

// K5: the Gamma-dependent features from the device Gamma (d x e)
int set_gamma(cntgw_solver* s, const double* gamma, cudaStream_t st) {
  const double* op;
  Side* side;
  const double* feat;
  int64_t count;
  int din, dout;
  if (s->proj_rows) {  // rows: Gamma^T X_i
    transpose_kernel<<<1, 256, 0, st>>>(gamma, s->d, s->e, s->gamma_t);
    TRY(cuda_ok(cudaPeekAtLastError(), "transpose"));
    op = s->gamma_t, side = &s->src, feat = s->x, count = s->n, din = s->d, dout = s->e;
  } else {  // cols: Gamma Y_j
    op = gamma, side = &s->tgt, feat = s->y, count = s->m, din = s->e, dout = s->d;
  }
  TRY(cntgw_apply_operator(op, dout, din, feat, din, count, side->feat64,
                           s->cfg.precision == CNTGW_F32 ? side->feat32 : nullptr, s->kd, st));
  if (s->cfg.precision == CNTGW_F64S)  // new features: the F64S rows blocks of both half-updates
    for (Half* h : {&s->fwd, &s->bwd})
      TRY(cntgw_prep_rows_f64s(s->kd, 1, h->rows->feat64, s->kd, h->rows->sq, h->rows->order, h->rows->n,
                               h->f64s_rows, st));
  return CNTGW_OK;
}

// K2 tentative (skipped after a symmetrized threshold break), K4, K7
int reductions(cntgw_solver* s, double* f, double* g, cudaStream_t st) {
  TRY(g_update(s, f, s->gt, 2, st));
  Half& h = s->fwd;
  const int kd = s->kd;
  if (s->cfg.precision == CNTGW_F64S) {
    TRY(cntgw_prep_rows_f64s(kd, 1, s->src.feat64, kd, s->src.sq, s->src.order, s->n, h.f64s_rows, st));
    TRY(cntgw_prep_cols_f64s(s->st, kd, 1, s->tgt.feat64, kd, s->tgt.sq, g, s->tgt.log2w, s->tgt.order, s->m,
                             h.rec, st));
    TRY(cntgw_plan_reduce_f64s(s->st, kd, 1, s->e, h.f64s_rows, h.rec, s->tgt.order, s->src.feat64, kd,
                               s->src.sq, f, s->src.log2w, s->y, s->e, s->tgt.sq, s->n, s->m, s->r, s->pi_y,
                               s->pi_s, s->argmax, h.ws, h.ws_bytes, s->ws_plan, s->ws_plan_bytes, st));
  } else {
    TRY(cntgw_prep_cols(s->st, CNTGW_F64, kd, 1, s->tgt.feat64, kd, s->tgt.sq, g, s->tgt.log2w, s->m, h.rec, st));
    TRY(cntgw_plan_reduce(s->st, kd, s->e, s->src.feat64, kd, s->src.sq, f, s->src.log2w, h.rec, s->y, s->e,
                          s->tgt.sq, s->n, s->m, s->r, s->pi_y, s->pi_s, s->argmax, s->ws_plan, s->ws_plan_bytes,
                          st));
  }
  const int nrow = 16 + s->d * s->e;
  TRY(cntgw_outer_reduce_rows(s->x, s->d, s->d, s->pi_y, s->e, s->r, s->pi_s, f, s->src.sq, s->a, s->n, s->acc,
                              s->ws_outer, s->ws_outer_bytes, st));
  if (s->comm) TRY(cntgw_comm_allreduce(s->comm, s->acc, s->acc, nrow, 0, st));
  return cntgw_outer_reduce_cols(s->st, g, s->gt, s->tgt.sq, s->b, s->m, s->acc + nrow, s->ws_outer,
                                 s->ws_outer_bytes, st);
}

}  // namespace

extern "C" {

int cntgw_solver_create(cntgw_solver** out, const double* x, int64_t n, int d, const double* y, int64_t m, int e,
                        const double* a, const double* b, const int64_t* order_x, const int64_t* order_y,
                        const cntgw_solve_config* cfg, cntgw_comm* comm, int64_t n_rows_max, void* stream) {
  if (!out || !x || !y || !a || !b || !cfg || n < 1 || m < 1 || d < 1 || e < 1 || d > 64 || e > 64)
    return fail(CNTGW_EINVAL, "solver_create: bad arguments");
  const int prec = cfg->precision;
  if (prec != CNTGW_F32 && prec != CNTGW_F64 && prec != CNTGW_F64S)
    return fail(CNTGW_EINVAL, "solver_create: precision %d (supported: CNTGW_F32, CNTGW_F64, CNTGW_F64S)", prec);
  if (cfg->max_outer < 1 || !(cfg->eps > 0.0) || (cfg->threshold <= 0.0 && cfg->n_inner < 1) ||
      (cfg->threshold > 0.0 && cfg->max_inner < 1))
    return fail(CNTGW_EINVAL, "solver_create: bad configuration");
  auto* s = new cntgw_solver{};
  s->cfg = *cfg;
  s->n = n, s->m = m, s->d = d, s->e = e;
  s->x = x, s->y = y, s->a = a, s->b = b;
  s->comm = comm;
  s->proj_rows = d > e;
  s->k = d < e ? d : e;
  s->kd = padded_kd(s->k);
  s->n_gap = comm && n_rows_max > n ? n_rows_max : n;
  cudaStream_t st = as_stream(stream);
  int rc = CNTGW_OK;
  auto side_init = [&](Side& sd, const double* pts, int64_t cnt, int dim, const double* w, const int64_t* order,
                       bool gamma_side) -> int {
    sd.n = cnt, sd.w = w, sd.order = order;
    TRY(alloc(&sd.feat64, (size_t)cnt * s->kd));
    TRY(alloc(&sd.sq, (size_t)cnt));
    TRY(alloc(&sd.log2w, (size_t)cnt));
    half_sq_kernel<<<blocks_for(cnt), 256, 0, st>>>(pts, cnt, dim, sd.sq);
    log2_kernel<<<blocks_for(cnt), 256, 0, st>>>(w, cnt, sd.log2w);
    if (gamma_side)
      TRY(cuda_ok(cudaMemsetAsync(sd.feat64, 0, sizeof(double) * cnt * s->kd, st), "memset"));
    else
      pad_copy_kernel<<<blocks_for(cnt), 256, 0, st>>>(pts, cnt, dim, s->kd, sd.feat64);
    if (prec == CNTGW_F32) {
      TRY(alloc(&sd.feat32, (size_t)cnt * s->kd));
      TRY(alloc(&sd.sq32, (size_t)cnt));
      to_f32_kernel<<<blocks_for(cnt * s->kd), 256, 0, st>>>(sd.feat64, cnt * s->kd, sd.feat32);
      to_f32_kernel<<<blocks_for(cnt), 256, 0, st>>>(sd.sq, cnt, sd.sq32);
    }
    return cuda_ok(cudaPeekAtLastError(), "solver side init");
  };
  if ((rc = side_init(s->src, x, n, d, a, order_x, s->proj_rows)) ||
      (rc = side_init(s->tgt, y, m, e, b, order_y, !s->proj_rows)) ||
      (rc = half_alloc(s->fwd, &s->src, &s->tgt, s->kd, prec)) ||
      (rc = half_alloc(s->bwd, &s->tgt, &s->src, s->kd, prec))) {
    cntgw_solver_destroy(s);
    return rc;
  }
  const size_t plan_ws = cntgw_plan_reduce_workspace(n, m, s->kd, e), plan_ws2 = cntgw_plan_reduce_ctr_workspace(m, e);
  s->ws_plan_bytes = plan_ws > plan_ws2 ? plan_ws : plan_ws2;
  const size_t o1 = cntgw_outer_reduce_workspace(n, d, e), o2 = cntgw_outer_reduce_workspace(m, 1, 1);
  s->ws_outer_bytes = o1 > o2 ? o1 : o2;
  if ((rc = alloc(reinterpret_cast<char**>(&s->st), sizeof(cntgw_sweep_state))) ||
      (rc = alloc(&s->ft, n)) || (rc = alloc(&s->gt, m)) ||
      (rc = alloc(&s->pr, (size_t)cntgw_gap_blocks(s->n_gap))) || (rc = alloc(&s->pc, (size_t)cntgw_gap_blocks(m))) ||
      (rc = alloc(&s->r, n)) || (rc = alloc(&s->pi_y, (size_t)n * e)) || (rc = alloc(&s->pi_s, n)) ||
      (rc = alloc(&s->argmax, n)) || (rc = alloc(reinterpret_cast<char**>(&s->ws_plan), s->ws_plan_bytes)) ||
      (rc = alloc(&s->acc, (size_t)(16 + d * e + 8))) ||
      (rc = alloc(reinterpret_cast<char**>(&s->ws_outer), s->ws_outer_bytes)) ||
      (rc = alloc(&s->gamma_t, (size_t)d * e)) ||
      (rc = alloc(reinterpret_cast<char**>(&s->os), sizeof(cntgw_outer_state))) ||
      (rc = alloc(&s->trace, (size_t)5 * cfg->max_outer))) {
    cntgw_solver_destroy(s);
    return rc;
  }
  if (comm && ((rc = alloc(&s->mx, m)) || (rc = alloc(&s->sm, m)) || (rc = alloc(&s->mglob, m)) ||
               (rc = alloc(&s->pr_glob, (size_t)cntgw_gap_blocks(s->n_gap))))) {
    cntgw_solver_destroy(s);
    return rc;
  }
  cudaMemsetAsync(s->pr, 0, sizeof(double) * cntgw_gap_blocks(s->n_gap), st);
  cudaMemsetAsync(s->pc, 0, sizeof(double) * cntgw_gap_blocks(m), st);
  cudaMemsetAsync(s->acc, 0, sizeof(double) * (16 + d * e + 8), st);
  if ((rc = cuda_ok(cudaStreamSynchronize(st), "solver_create"))) {
    cntgw_solver_destroy(s);
    return rc;
  }
  *out = s;
  return CNTGW_OK;
}

int cntgw_solver_destroy(cntgw_solver* s) {
  if (!s) return CNTGW_OK;
  for (Side* sd : {&s->src, &s->tgt}) {
    cudaFree(sd->feat64);
    cudaFree(sd->feat32);
    cudaFree(sd->sq);
    cudaFree(sd->sq32);
    cudaFree(sd->log2w);
  }
  half_free(s->fwd);
  half_free(s->bwd);
  void* bufs[] = {s->st, s->ft, s->gt, s->pr, s->pc, s->pr_glob, s->mx, s->sm, s->mglob, s->r, s->pi_y,
                  s->pi_s, s->argmax, s->ws_plan, s->acc, s->ws_outer, s->gamma_t, s->os, s->trace};
  for (void* p : bufs) cudaFree(p);
  delete s;
  return CNTGW_OK;
}

int cntgw_solver_init_potentials(cntgw_solver* s, double* f, double* g, void* stream) {
  if (!s || !f || !g) return fail(CNTGW_EINVAL, "solver_init_potentials: bad arguments");
  cudaStream_t st = as_stream(stream);
  square_kernel<<<blocks_for(s->n), 256, 0, st>>>(s->src.sq, s->n, f);
  square_kernel<<<blocks_for(s->m), 256, 0, st>>>(s->tgt.sq, s->m, g);
  return cuda_ok(cudaPeekAtLastError(), "solver_init_potentials");
}

int cntgw_solver_run(cntgw_solver* s, double constant, double* gamma, double* gamma_prev, double* f, double* g,
                     double* trace_host, int* status_host, void* stream) {
  if (!s || !gamma || !gamma_prev || !f || !g || !trace_host || !status_host)
    return fail(CNTGW_EINVAL, "solver_run: bad arguments");
  // capture on streams of our own (the caller's may be the legacy default
  // stream, which cannot be captured), ordered after the caller's work
  cudaStream_t caller = as_stream(stream), s0 = nullptr, s1 = nullptr, s2 = nullptr;
  cudaEvent_t ev = nullptr;
  TRY(cuda_ok(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking), "cudaStreamCreate"));
  TRY(cuda_ok(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking), "cudaStreamCreate"));
  TRY(cuda_ok(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking), "cudaStreamCreate"));
  TRY(cuda_ok(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate"));
  TRY(cuda_ok(cudaEventRecord(ev, caller), "cudaEventRecord"));
  TRY(cuda_ok(cudaStreamWaitEvent(s0, ev, 0), "cudaStreamWaitEvent"));
  const cntgw_solve_config& c = s->cfg;
  const double eps = c.eps / 8.0;
  const bool thr = c.threshold > 0.0;
  const int max_sweeps = thr ? c.max_inner : c.n_inner;
  void* exec = nullptr;
  int rc = CNTGW_OK;
  auto capture = [&]() -> int {
    TRY(cntgw_graph_begin(s0));
    TRY(cntgw_outer_init(s->os, constant, c.eps, c.delta_outer, c.max_outer, s0));
    uint64_t h1 = 0, h2 = 0;
    TRY(cntgw_graph_while_begin(s0, s1, &h1));
    TRY(set_gamma(s, gamma, s1));
    TRY(cntgw_sweep_init(s->st, eps, c.anneal_from, thr ? c.threshold : 0.0, max_sweeps, c.mode, s1));
    if (!thr) {
      for (int k = 0; k < max_sweeps; ++k) TRY(sweep(s, f, g, s1));
    } else {
      TRY(cntgw_graph_while_begin(s1, s2, &h2));
      TRY(sweep(s, f, g, s2));
      TRY(cntgw_graph_set_condition(h2, &s->st->done, s2));
      TRY(cntgw_graph_while_end(s2));
    }
    TRY(cntgw_sweep_begin(s->st, s1));  // a fully used budget is marked done
    TRY(reductions(s, f, g, s1));
    TRY(cntgw_outer_finish(s->os, s->st, s->acc, s->acc + 16 + s->d * s->e, gamma, gamma_prev, s->d * s->e,
                           s->trace, s1));
    TRY(cntgw_graph_set_condition(h1, &s->os->done, s1));
    TRY(cntgw_graph_while_end(s1));
    return cntgw_graph_end(s0, &exec);
  };
  rc = capture();
  if (rc) {  // leave no capture open on the caller's stream
    cudaGraph_t g_;
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(s2, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) cudaStreamEndCapture(s2, &g_);
    if (cudaStreamIsCapturing(s1, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) cudaStreamEndCapture(s1, &g_);
    if (cudaStreamIsCapturing(s0, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) cudaStreamEndCapture(s0, &g_);
    cudaGetLastError();
  }
  if (!rc) rc = cntgw_graph_launch(exec, s0);
  if (!rc) rc = cuda_ok(cudaStreamSynchronize(s0), "solve");
  if (exec) cntgw_graph_destroy(exec);
  cudaEventDestroy(ev);
  cudaStreamDestroy(s0);
  cudaStreamDestroy(s1);
  cudaStreamDestroy(s2);
  if (rc) return rc;
  cntgw_outer_state os;
  TRY(cuda_ok(cudaMemcpy(&os, s->os, sizeof(os), cudaMemcpyDeviceToHost), "outer state"));
  TRY(cuda_ok(cudaMemcpy(trace_host, s->trace, sizeof(double) * 5 * os.step, cudaMemcpyDeviceToHost), "trace"));
  cntgw_sweep_state sw;
  TRY(cuda_ok(cudaMemcpy(&sw, s->st, sizeof(sw), cudaMemcpyDeviceToHost), "sweep state"));
  status_host[0] = os.step;
  status_host[1] = os.converged;
  status_host[2] = os.error;
  status_host[3] = sw.applied;
  return CNTGW_OK;
}

int cntgw_solver_results(const cntgw_solver* s, double* row_mass, int64_t* argmax, double* eps_eff, void* stream) {
  if (!s) return fail(CNTGW_EINVAL, "solver_results: null solver");
  cudaStream_t st = as_stream(stream);
  if (row_mass)
    TRY(cuda_ok(cudaMemcpyAsync(row_mass, s->r, sizeof(double) * s->n, cudaMemcpyDeviceToDevice, st), "row_mass"));
  if (argmax)
    TRY(cuda_ok(cudaMemcpyAsync(argmax, s->argmax, sizeof(int64_t) * s->n, cudaMemcpyDeviceToDevice, st), "argmax"));
  if (eps_eff) {
    cntgw_sweep_state sw;
    TRY(cuda_ok(cudaMemcpyAsync(&sw, s->st, sizeof(sw), cudaMemcpyDeviceToHost, as_stream(stream)), "sweep state"));
    TRY(cuda_ok(cudaStreamSynchronize(as_stream(stream)), "solver_results"));
    *eps_eff = sw.eps_n;
  }
  return CNTGW_OK;
}

int cntgw_gw_constant(const double* x, int64_t n, int d, const double* a, const double* y, int64_t m, int e,
                      const double* b, double* out_host, void* stream) {
  if (!x || !y || !a || !b || !out_host || n < 1 || m < 1 || d < 1 || e < 1 || d > 64 || e > 64)
    return fail(CNTGW_EINVAL, "gw_constant: bad arguments");
  cudaStream_t st = as_stream(stream);
  double q[2], t[2];
  const double* pts[2] = {x, y};
  const double* ws_[2] = {a, b};
  const int64_t cnt[2] = {n, m};
  const int dim[2] = {d, e};
  for (int side = 0; side < 2; ++side) {
    const int dd = dim[side];
    double* mom = nullptr;
    void* ws = nullptr;
    const size_t wsb = cntgw_moments_workspace(cnt[side], dd);
    TRY(alloc(&mom, (size_t)(3 + dd * dd)));
    int rc = alloc(reinterpret_cast<char**>(&ws), wsb);
    if (!rc) rc = cntgw_moments(pts[side], dd, dd, ws_[side], cnt[side], mom, ws, wsb, st);
    double h[3 + 64 * 64];
    if (!rc) rc = cuda_ok(cudaMemcpyAsync(h, mom, sizeof(double) * (3 + dd * dd), cudaMemcpyDeviceToHost, st), "moments");
    if (!rc) rc = cuda_ok(cudaStreamSynchronize(st), "moments");
    cudaFree(mom);
    cudaFree(ws);
    if (rc) return rc;
    double cov2 = 0.0;
    for (int k = 0; k < dd * dd; ++k) cov2 += h[3 + k] * h[3 + k];
    q[side] = 2.0 * h[1] + 2.0 * h[2] * h[2] + 4.0 * cov2;
    t[side] = h[0];
  }
  *out_host = q[0] + q[1] - 4.0 * t[0] * t[1];
  return CNTGW_OK;
}

}  // extern "C"
