/*
 * cntgw_b200 — C ABI of the B200-native CNT-GW hot path (sm_100a).
 *
 * Drop-in boundary for the reference package `cntgw` (arXiv 2602.06658,
 * /root/reference/pkg/src/cntgw). The reference is pure Python with no FFI,
 * so each entry point below replaces one arithmetic site of its hot path
 * (cited per function); the Python host package `paper_2602_06658_b200`
 * binds them with ctypes and keeps the reference's Python API on top.
 *
 * Conventions
 *  - Every pointer is a caller-owned DEVICE buffer (fp32 unless stated;
 *    weights/gaps/objective accumulators are fp64). No allocation happens
 *    inside the library; scratch is passed in, sized by the *_workspace calls.
 *  - All work is enqueued on `stream` (a cudaStream_t); nothing synchronises
 *    the host. Every launch is CUDA-graph capturable.
 *  - Functions return 0 on success or a negative cntgw_status; the message
 *    of the last failure on the calling thread is cntgw_last_error().
 *  - Potentials on device are INTERACTION potentials:
 *    f~ = f - |x_i|^2 and g~ = g - |z_j|^2 over the dot coordinates, the
 *    separable parts being re-added in fp64 by the host at the boundary.
 *
 * Half-update (the kernel every Sinkhorn sweep runs twice):
 *   t_ij   = beta_j + sum_k x_ik * zt_jk - (sqrt(lam) s_i - st_j)^2      (log2 units)
 *   out_i  = row_add_i - (max_j t_ij + log2 sum_j 2^(t_ij - max)) / lam
 * with lam = log2(e)/eps_n read from the sweep state, zt = 2 lam z,
 * st_j = sqrt(lam) s_j and beta_j = lam * pot_j + log2 w_j packed per column
 * by cntgw_prep_cols. This equals the reference half-update
 *   out_i = -eps * logsumexp_j(log w_j + (pot_j - C_ij)/eps)
 * (sinkhorn.py:166-176) for C_ij = |x_i-z_j|^2 over the dot coordinates plus
 * (s_i - s_j)^2 over the optional squared-difference coordinate.
 */
#ifndef CNTGW_B200_H
#define CNTGW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CNTGW_ABI_VERSION 1

typedef enum cntgw_status {
  CNTGW_OK = 0,
  CNTGW_EINVAL = -1,   /* bad argument (shape, null pointer, unsupported k) */
  CNTGW_ECUDA = -2,    /* a CUDA launch or query failed */
  CNTGW_ENOSPACE = -3  /* workspace smaller than the *_workspace query */
} cntgw_status;

/* Device-resident state of one Sinkhorn loop (sinkhorn.py:191-258 control).
 * Lives in device memory; the host initialises it with cntgw_sweep_init and
 * reads it back (plain memcpy of sizeof(cntgw_sweep_state) bytes). */
typedef struct cntgw_sweep_state {
  double eps;          /* target temperature (SinkhornConfig.eps)            */
  double anneal_from;  /* 0 => no annealing (SinkhornConfig.anneal_from)      */
  double threshold;    /* 0 => fixed budget (SinkhornConfig.threshold)        */
  double eps_n;        /* temperature of the current sweep                   */
  double gap_r;        /* weighted row gap of the current sweep              */
  double gap_c;        /* weighted column gap of the current sweep           */
  float lam;           /* log2(e) / eps_n                                     */
  float inv_lam;       /* eps_n * ln 2                                        */
  float sqrt_lam;      /* sqrt(lam)                                           */
  int32_t max_sweeps;  /* n_inner, or max_inner in threshold mode             */
  int32_t mode;        /* 0 standard, 1 symmetrized                           */
  int32_t sweep;       /* index of the sweep in flight (1-based)             */
  int32_t applied;     /* sweeps applied (SinkhornResult.iterations)          */
  int32_t done;        /* 1 once the loop has finished                        */
  int32_t converged;   /* SinkhornResult.converged                            */
  int32_t check;       /* threshold checked this sweep (eps_n == eps)         */
  int32_t pad_[2];
} cntgw_sweep_state;

/* ---- library ------------------------------------------------------------ */
int cntgw_abi_version(void);
const char* cntgw_last_error(void);
/* sizeof(cntgw_sweep_state), for host-side mirrors */
int cntgw_sweep_state_size(void);
/* float stride of one packed column record for (kd, sq) */
int cntgw_col_stride(int kd, int sq);
/* columns the packed column buffer must hold (m rounded up to the tile) */
int64_t cntgw_cols_padded(int64_t m);

/* ---- K3: sweep control (sinkhorn.py:222-251, gaps :179-188) ------------- */
/* Initialise `st`: config fields, sweep=applied=done=0, converged = (threshold==0). */
int cntgw_sweep_init(cntgw_sweep_state* st, double eps, double anneal_from, double threshold,
                     int max_sweeps, int mode, void* stream);
/* Start the next sweep: eps_n = max(anneal_from/sqrt(n), eps), lam, check flag;
 * marks the loop done when the budget is exhausted. */
int cntgw_sweep_begin(cntgw_sweep_state* st, void* stream);
/* Weighted marginal gap partials sum_i w_i^2 |exp(min((pot-tent)/eps_n,700)) - 1|
 * (fp64) for the row side (side=0) or column side (side=1); runs only when the
 * current sweep checks the threshold. `partials` holds cntgw_gap_blocks(n) doubles. */
int cntgw_gap_blocks(int64_t n);
int cntgw_sweep_gap(cntgw_sweep_state* st, int side, const double* w, const float* pot,
                    const float* tent, int64_t n, double* partials, void* stream);
/* Reduce the gap partials in a fixed order, decide the threshold break
 * (sinkhorn.py:232-237 / :242-248) and count the sweep as applied otherwise. */
int cntgw_sweep_finish(cntgw_sweep_state* st, const double* partials_r, int64_t n,
                       const double* partials_c, int64_t m, void* stream);
/* Apply the sweep unless it broke: symmetrized pot = (pot + tent)/2, standard pot = tent. */
int cntgw_sweep_apply(const cntgw_sweep_state* st, float* pot, const float* tent, int64_t n,
                      int average, void* stream);

/* ---- K1/K2: half-update (sinkhorn.py:166-176) ---------------------------- */
/* Pack column records for the current lam of `st`, in the sign-flipped form
 * the kernels accumulate with plain FMAs: [-2 lam z (kd), -sqrt(lam) s (if
 * sq_flag), -(lam pot + log2 w), zero pad to a multiple of 4 floats]. Columns
 * m..cntgw_cols_padded(m)-1 get -beta = +inf (exactly zero weight).
 * feat: m x kd row-major (stride ld); sq, pot: m (sq needed iff sq_flag);
 * log2w: m fp32; pot may be null (treated as 0). */
int cntgw_prep_cols(const cntgw_sweep_state* st, int kd, int sq_flag, const float* feat, int64_t ld,
                    const float* sq, const float* pot, const float* log2w, int64_t m, float* rec,
                    void* stream);
/* Scratch bytes the half-update needs for split-column partials. */
size_t cntgw_softmin_workspace(int64_t n, int64_t m, int kd, int sq_flag);
/* out_i = row_add_i - LSE2_j(t_ij)/lam  (row_add nullable => 0).
 * If out_max/out_sum are non-null the per-row (max, sum 2^(t-max)) pair is
 * written instead of `out` (partial LSE for the multi-GPU column combine).
 * skip_if_done: return immediately when st->done (graph early exit). */
int cntgw_softmin(const cntgw_sweep_state* st, int skip_if_done, int kd, int sq_flag,
                  const float* row_feat, int64_t ld_row, const float* row_sq, const float* row_add,
                  const float* col_rec, int64_t n, int64_t m, float* out, float* out_max,
                  float* out_sum, void* workspace, size_t workspace_bytes, void* stream);
/* Finalise partial LSE pairs: out_i = row_add_i - (mx_i + log2 sm_i)/lam. */
int cntgw_lse_finalize(const cntgw_sweep_state* st, int skip_if_done, const float* mx,
                       const float* sm, const float* row_add, int64_t n, float* out, void* stream);

/* Dense-cost half-update (DenseCost provider, sinkhorn.py:30-56):
 * out_i = row_add_i - LSE2_j(lam pot_j + log2w_j - lam C_ij)/lam, C row-major n x m. */
int cntgw_softmin_dense(const cntgw_sweep_state* st, int skip_if_done, const float* cost,
                        int64_t ld, const float* pot, const float* log2w, const float* row_add,
                        int64_t n, int64_t m, float* out, void* stream);

/* ---- K4: fused plan reductions (solvers.py:227-256, measures.py:185-235) -- */
/* One streaming pass over pi_ij = a_i 2^(lam f~_i + t_ij) for the final pair.
 * Per row i: r_i = sum_j pi_ij, piY_i = sum_j pi_ij Y_j (e floats), pit_i =
 * sum_j pi_ij s_j, and argmax_j pi_ij (lowest j on ties).
 * col_acc: m x e accumulation features Y (row-major, stride ld_acc), col_s: m. */
size_t cntgw_plan_reduce_workspace(int64_t n, int64_t m, int kd, int sq_flag, int e);
int cntgw_plan_reduce(const cntgw_sweep_state* st, int kd, int sq_flag, int e,
                      const float* row_feat, int64_t ld_row, const float* row_sq,
                      const float* f_tilde, const float* log2a, const float* col_rec,
                      const float* col_acc, int64_t ld_acc, const float* col_s, int64_t n,
                      int64_t m, float* row_mass, float* pi_y, float* pi_s, int64_t* argmax,
                      void* workspace, size_t workspace_bytes, void* stream);

/* ---- K5/K7: operator, features and objective (solvers.py:219-220, 330-334) */
/* out (n x dout) = feat (n x din) @ op^T where op is dout x din fp64 (i.e.
 * out_i = op . feat_i), in fp32 with fp64 accumulation. */
int cntgw_apply_operator(const double* op, int dout, int din, const float* feat, int64_t ld,
                         int64_t n, float* out, void* stream);
/* Deterministic fp64 row reduction for the outer step. Writes 16 + d*e doubles
 * to `acc`: [0] sum f~_i r_i, [1] sum s_i^2 r_i, [2] sum |r_i - a_i|,
 * [3] sigma_ss = sum s_i pit_i, [4] sum r_i, [5..15] reserved,
 * [16..] Gamma_next = sum_i X_i piY_i^T (d x e row-major).
 * scratch: cntgw_outer_reduce_workspace(n, d, e) bytes. */
size_t cntgw_outer_reduce_workspace(int64_t n, int d, int e);
int cntgw_outer_reduce_rows(const float* x, int64_t ldx, int d, const float* pi_y, int e,
                            const float* row_mass, const float* pi_s, const float* f_tilde,
                            const float* s_half, const double* a, int64_t n, double* acc,
                            void* workspace, size_t workspace_bytes, void* stream);
/* Column side: c_j = b_j 2^(lam (g~_j - gt_j)); writes 8 doubles:
 * [0] sum g~_j c_j, [1] sum t_j^2 c_j, [2] sum |c_j - b_j|, [3] sum c_j. */
int cntgw_outer_reduce_cols(const cntgw_sweep_state* st, const float* g_tilde, const float* g_tent,
                            const float* t_half, const double* b, int64_t m, double* acc,
                            void* workspace, size_t workspace_bytes, void* stream);
/* Weighted moments for the closed-form loss constant (divergence.py:28-47):
 * writes [sum w|x|^2 (raw T), sum w|xc|^4, sum w|xc|^2, then sum w xc xc^T (d x d)]
 * with xc = x - sum w x, x fp64 (n x d, stride ldx). Needs (3 + d*d) doubles in `out`. */
size_t cntgw_moments_workspace(int64_t n, int d);
int cntgw_moments(const double* x, int64_t ldx, int d, const double* w, int64_t n, double* out,
                  void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CNTGW_B200_H */
