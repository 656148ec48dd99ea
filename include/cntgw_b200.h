/*
 * cntgw_b200 — C ABI of the B200-native CNT-GW hot path (sm_100a).
 *
 * Drop-in boundary for the reference package `cntgw` (arXiv 2602.06658,
 * /root/reference/pkg/src/cntgw). The reference is pure Python with no FFI;
 * its only plugin seam is the duck-typed cost-provider protocol consumed by
 * `_softmin` (sinkhorn.py:166-176). Each entry point below replaces one
 * arithmetic site of the hot path (cited per function); the Python host
 * package `paper_2602_06658_b200` binds them with ctypes and
 * keeps the reference's Python API on top.
 *
 * Conventions
 *  - Every pointer is a caller-owned DEVICE buffer. Potentials, weights and
 *    reductions are fp64; feature/record buffers are fp32 or fp64 according to
 *    the `prec` argument (CNTGW_F32 / CNTGW_F64). No allocation happens inside
 *    the library; scratch is passed in, sized by the *_workspace queries.
 *  - All work is enqueued on `stream` (a cudaStream_t); nothing synchronises
 *    the host; every launch is CUDA-graph capturable.
 *  - Functions return 0 on success or a negative cntgw_status; the message of
 *    the last failure on the calling thread is cntgw_last_error().
 *  - Potentials on device are INTERACTION potentials: f~ = f - row_sep and
 *    g~ = g - col_sep for the cost
 *        C_ij = row_sep_i + col_sep_j - 2 <x_i, z_j> + (s_i - s_j)^2
 *    (the last term only with sq_flag); the host re-adds the separable parts.
 *
 * Half-update (run twice per Sinkhorn sweep), in log2 units with
 * lam = log2(e)/eps_n from the sweep state:
 *   t_ij  = lam (pot_j + 2 <x_i, z_j> - (s_i - s_j)^2) + log2 w_j
 *   out_i = row_add_i - (max_j t_ij + log2 sum_j 2^(t_ij - max)) / lam
 * which is the reference half-update
 *   out_i = -eps * logsumexp_j(log w_j + (pot_j - C_ij)/eps)   (sinkhorn.py:166-176)
 * on interaction potentials. CNTGW_F32 assembles t_ij with fp32 FFMA2;
 * CNTGW_F64 assembles it with fp64 DFMA (needed when |t| ~ 1e6: the cold C4/C5
 * laws) and both evaluate 2^(t - max) on MUFU.EX2.
 */
#ifndef CNTGW_B200_H
#define CNTGW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CNTGW_ABI_VERSION 4

typedef enum cntgw_status {
  CNTGW_OK = 0,
  CNTGW_EINVAL = -1,   /* bad argument (shape, null pointer, unsupported k) */
  CNTGW_ECUDA = -2,    /* a CUDA launch or query failed */
  CNTGW_ENOSPACE = -3  /* workspace smaller than the *_workspace query */
} cntgw_status;

/* Exponent assembly: fp32 FFMA2, fp64 DFMA, the tcgen05 tensor cores with a
 * 3xTF32 split (kd in {8, 16}, no sq coordinate; well-scaled problems), or
 * CNTGW_F32C: fp32 pair terms on locality-ordered, centred tiles with fp64
 * per-tile offsets (kd + sq <= 8; the cold low-dimensional laws, see
 * cntgw_prep_cols_ctr). */
typedef enum cntgw_precision {
  CNTGW_F32 = 0,
  CNTGW_F64 = 1,
  CNTGW_TF32X3 = 2,
  CNTGW_F32C = 3,
  CNTGW_F64S = 4
} cntgw_precision;

/* Device-resident state of one Sinkhorn loop (sinkhorn.py:191-258 control).
 * Lives in device memory; the host initialises it with cntgw_sweep_init and
 * reads it back as a plain copy of sizeof(cntgw_sweep_state) bytes. */
typedef struct cntgw_sweep_state {
  double eps;          /* target temperature (SinkhornConfig.eps)            */
  double anneal_from;  /* 0 => no annealing (SinkhornConfig.anneal_from)      */
  double threshold;    /* 0 => fixed budget (SinkhornConfig.threshold)        */
  double eps_n;        /* temperature of the current sweep                   */
  double gap_r;        /* weighted row gap of the current sweep              */
  double gap_c;        /* weighted column gap of the current sweep           */
  double lam_d;        /* log2(e) / eps_n                                     */
  double sqrt_lam_d;   /* sqrt(lam_d)                                         */
  float lam;           /* (float) lam_d, used by the fp32 records             */
  float sqrt_lam;      /* (float) sqrt_lam_d                                  */
  int32_t max_sweeps;  /* n_inner, or max_inner in threshold mode             */
  int32_t mode;        /* 0 standard, 1 symmetrized                           */
  int32_t sweep;       /* index of the sweep in flight (1-based)             */
  int32_t applied;     /* sweeps applied (SinkhornResult.iterations)          */
  int32_t done;        /* 1 once the loop has finished                        */
  int32_t converged;   /* SinkhornResult.converged                            */
  int32_t check;       /* threshold checked this sweep (eps_n == eps)         */
  int32_t pad_;
} cntgw_sweep_state;

/* Device-resident state of the CNT-GW outer loop (solvers.py:556-625 control)
 * for the graph-captured solve (cntgw_outer_finish). */
typedef struct cntgw_outer_state {
  double constant;       /* loss constant C (divergence.py:41-47)              */
  double eps_outer;      /* EgwConfig.eps                                       */
  double delta_outer;    /* EgwConfig.delta_outer                               */
  double prev_objective; /* objective of the previous outer step               */
  double t0_ns;          /* %globaltimer at cntgw_outer_init                    */
  int32_t max_outer;     /* EgwConfig.max_outer                                 */
  int32_t step;          /* outer steps completed                               */
  int32_t ups;           /* consecutive objective increases                     */
  int32_t done;          /* 1: stop (converged, guard tripped or budget used)   */
  int32_t converged;     /* |dobj| < delta_outer reached                        */
  int32_t error;         /* 1: divergence guard (SolverError, solvers.py:604)   */
  int32_t has_prev;
  int32_t pad_;
} cntgw_outer_state;

/* ---- library ------------------------------------------------------------ */
int cntgw_abi_version(void);
const char* cntgw_last_error(void);
/* sizeof(cntgw_sweep_state), for host-side mirrors */
int cntgw_sweep_state_size(void);
/* elements (fp32 or fp64 per prec) of one packed column record for (kd, sq) */
int cntgw_col_stride(int prec, int kd, int sq);
/* columns a packed column buffer must hold (m rounded up to the 256-column tile) */
int64_t cntgw_cols_padded(int64_t m);

/* ---- K3: sweep control (sinkhorn.py:222-251, gaps :179-188) ------------- */
/* Initialise `st`: config fields, sweep=applied=done=0, converged=(threshold==0),
 * lam for eps. */
int cntgw_sweep_init(cntgw_sweep_state* st, double eps, double anneal_from, double threshold,
                     int max_sweeps, int mode, void* stream);
/* Start the next sweep: eps_n = max(anneal_from/sqrt(n), eps) (sinkhorn.py:223-226),
 * lam, check flag (:228); marks the loop done once the budget is exhausted. */
int cntgw_sweep_begin(cntgw_sweep_state* st, void* stream);
/* Weighted marginal gap sum_i w_i^2 |exp(min((pot-tent)/eps_n, 700)) - 1|
 * (sinkhorn.py:179-188) as cntgw_gap_blocks(n) fp64 partials; runs only when
 * the current sweep checks the threshold. */
int cntgw_gap_blocks(int64_t n);
int cntgw_sweep_gap(cntgw_sweep_state* st, const double* w, const double* pot, const double* tent,
                    int64_t n, double* partials, void* stream);
/* Reduce the gap partials in a fixed order, decide the threshold break
 * (sinkhorn.py:232-237 symmetrized, :242-248 standard; partials_c may be null
 * for standard mode) and count the sweep as applied otherwise (:251). */
int cntgw_sweep_finish(cntgw_sweep_state* st, const double* partials_r, int64_t n,
                       const double* partials_c, int64_t m, void* stream);
/* Apply the sweep unless it broke: average ? pot=(pot+tent)/2 (:238-239) : pot=tent (:249). */
int cntgw_sweep_apply(const cntgw_sweep_state* st, double* pot, const double* tent, int64_t n,
                      int average, void* stream);

/* ---- K1/K2: half-update (sinkhorn.py:166-176) ---------------------------- */
/* Pack the column side for the current lam of `st`, sign-flipped so the
 * kernels accumulate with plain FMAs: fp32 [-2 lam z (kd) | -sqrt(lam) s (if
 * sq) | -(lam pot + log2 w) | zero pad] (squared coordinate kept as a
 * difference); fp64 [-2 lam z | -2 lam s | -(lam (pot - s^2) + log2 w)]
 * (square expanded, exact enough in fp64); tensor-core (CNTGW_TF32X3): the
 * 3-way split tiles of softmin_tc.cuh, on fp16 operands scaled from the
 * absmax of the column features (default) or on tf32 operands
 * (CNTGW_TC_KIND=tf32, read by this call and by cntgw_softmin alike); that
 * path is for well-scaled problems, 2 lam max|x| max|z| < 2^13 (larger
 * scores overflow fp16 and come back as inf/NaN, never silently wrong). Padding columns m..cols_padded(m)-1 get an exactly-zero
 * weight. feat: m x kd row-major (stride ld), fp32 or fp64 per
 * prec, as is sq; pot (nullable => 0) and log2w are fp64. */
int cntgw_prep_cols(const cntgw_sweep_state* st, int prec, int kd, int sq_flag, const void* feat,
                    int64_t ld, const void* sq, const double* pot, const double* log2w, int64_t m,
                    void* rec, void* stream);
/* ---- K1/K2, CNTGW_F32C: centred fp32 on locality-ordered tiles ----------
 * Same half-update (sinkhorn.py:166-176) for problems whose exponent terms are
 * too large for fp32 (|t| ~ 1e6 on the C4 law) but whose points are
 * low-dimensional. Rows and columns are visited in a locality order `order`
 * (a permutation; NULL = identity), 128-row groups I and 256-column tiles J
 * are centred, and with X_i = [x_i | s_i], Zr_j = [-2 lam z_j | -2 lam s_j]
 * (expanded square, as the fp64 records) the exponent splits exactly into
 *   q_ij = A_j^I (fp64, per group and column) + B_i^J (fp64, per row and tile)
 *        + <dX_i, dZ_j> (fp32 FFMA2 per pair, small after centring).
 * cntgw_locality_codes: 63-bit Morton codes of the first min(d, 3)
 * coordinates (x: n x d fp64, stride ld; bbox: 6 doubles of scratch); the
 * caller sorts them (stable) to obtain `order`.
 * cntgw_prep_rows_ctr / cntgw_prep_cols_ctr fill the row block / column block
 * (sizes from the *_bytes queries) from fp64 features in the caller's order;
 * the column block is per half-update (it holds lam and pot). cntgw_softmin
 * with prec = CNTGW_F32C then takes row_feat = the row block, row_sq = the
 * rows' fp64 squared coordinate in the caller's order (or NULL without sq),
 * col_rec = the column block; outputs are in the caller's order. Its
 * workspace (cntgw_softmin_workspace) also holds a block-sparse plan: a first
 * kernel bounds every (row group, column tile) pair and the sweep skips the
 * tiles that cannot hold a term within 2^-64 of any of its rows' maxima
 * (CNTGW_CTR_SKIP=0 disables it); the plan is reused across the sweeps of a
 * loop (st->sweep > 1) while no column record moved by more than its margin
 * (CNTGW_CTR_REUSE=0 replans every call). The plan is keyed on the operator
 * (row block and column block pointers, n, m) and on st->lam_d: a call with a
 * different key, an annealed lam, or a NaN column record replans. */
int cntgw_locality_codes(const double* x, int64_t n, int d, int64_t ld, double* bbox, int64_t* codes,
                         void* stream);
size_t cntgw_ctr_rows_bytes(int64_t n, int kd, int sq_flag);
size_t cntgw_ctr_cols_bytes(int64_t m, int kd, int sq_flag);
int cntgw_prep_rows_ctr(int kd, int sq_flag, const double* feat, int64_t ld, const double* sq,
                        const int64_t* order, int64_t n, void* rows, void* stream);
int cntgw_prep_cols_ctr(const cntgw_sweep_state* st, int kd, int sq_flag, const double* feat, int64_t ld,
                        const double* sq, const double* pot, const double* log2w, const int64_t* order,
                        int64_t m, void* cols, void* stream);
/* ---- K1/K2, CNTGW_F64S: fp64 (DMMA) on ordered rows/columns with a measured
 * block-sparse plan (softmin_f64s.cuh) — cold problems without low-dimensional
 * locality (C5). Rows are gathered once per operator into a block in a caller
 * order (a clustering of the points), columns are packed in their order. The
 * first sweep of a loop (or any sweep whose re-vote keeps more than 12% of
 * the pairs) probes every row's minimum exponent over every column stage on
 * the tensor cores (lower bounds, softmin_f64s_tcprobe.cuh; CNTGW_F64S_PROBE=0:
 * a dense fp64 measuring sweep instead), the exact sweeps record exact
 * minima for the stages they walk, and every sweep walks only the (row
 * group, stage) pairs that can hold a term within 2^-48 of a row's maximum
 * (CNTGW_CTR_SKIP_T overrides). Outputs are in the caller's order; the
 * workspace (cntgw_softmin_workspace) holds the plan and must stay with one
 * (rows, cols) operator for the length of a loop. */
size_t cntgw_f64s_rows_bytes(int64_t n, int kd);
int cntgw_prep_rows_f64s(int kd, int sq_flag, const double* feat, int64_t ld, const double* sq,
                         const int64_t* order, int64_t n, void* rows, void* stream);
/* Diagnostics of the plan in an F64S workspace: out (3 int64, device) =
 * [needed (row group, stage) pairs, all pairs, flags of the last sweep: bit 0
 * measured with the fp64 kernel, bit 1 planned by a probe]. */
int cntgw_f64s_plan_density(int kd, int sq_flag, int64_t n, int64_t m, const void* workspace, int64_t* out,
                            void* stream);
/* Host-side query: out (3 int64, host) = [byte offset in the workspace of the
 * plan's stage minima tmin, fp32 [n][stages] indexed by ordered row; stages;
 * columns per stage]. After a probe sweep tmin holds the probe's lower
 * bounds (tests/test_gpu_softmin.py checks them against exact fp64 minima). */
int cntgw_f64s_plan_layout(int kd, int sq_flag, int64_t n, int64_t m, int64_t* out);
/* out = (Gamma == 0 ? order_if_zero : order_otherwise), decided on the device
 * (graph-capturable): at Gamma = 0 the GW cost depends on the points only
 * through (s_i - t_j)^2 and the squared-coordinate order makes the plan a band. */
int cntgw_select_order(const double* gamma, int de, const int64_t* order_if_zero, const int64_t* order_otherwise,
                       int64_t n, int64_t* out, void* stream);
/* cntgw_prep_cols (CNTGW_F64 records) with the columns gathered in `order`. */
int cntgw_prep_cols_f64s(const cntgw_sweep_state* st, int kd, int sq_flag, const double* feat, int64_t ld,
                         const double* sq, const double* pot, const double* log2w, const int64_t* order,
                         int64_t m, void* rec, void* stream);
/* The same pack for a caller that owns a whole loop over fixed column features
 * (sinkhorn.py:222-251: only the potentials change between sweeps): the first
 * sweep of the loop (st->sweep <= 1) and every sweep of an annealed loop
 * (st->anneal_from > 0: lam changes) pack everything, the others rewrite the
 * bias column -(lam (pot - s^2) + log2 w) alone. Same arguments. */
int cntgw_update_cols_f64s(const cntgw_sweep_state* st, int kd, int sq_flag, const double* feat, int64_t ld,
                           const double* sq, const double* pot, const double* log2w, const int64_t* order,
                           int64_t m, void* rec, void* stream);
/* Workspace bytes of one half-update: split-column partials and, for
 * CNTGW_F32C, the block-sparse plan. The F32C part carries state from call to
 * call (the plan and its key, see above); a caller may share one workspace
 * between operators (the key forces a replan on every switch) but then pays a
 * planning pass per call — keep one workspace per (rows, cols) operator. */
size_t cntgw_softmin_workspace(int prec, int64_t n, int64_t m, int kd, int sq_flag);
/* out_i = row_add_i - LSE2_j(t_ij)/lam (row_add nullable => 0). If out_max and
 * out_sum are non-null the per-row (max, sum 2^(t-max)) pair is written instead
 * of `out` (partial LSE, finalised after a cross-GPU combine).
 * skip_if_done: 1 = return immediately when st->done (graph early exit);
 * 2 = return when the loop ended on a symmetrized threshold break (the
 * tentatives of that sweep are already the final ones). */
int cntgw_softmin(const cntgw_sweep_state* st, int skip_if_done, int prec, int kd, int sq_flag,
                  const void* row_feat, int64_t ld_row, const void* row_sq, const double* row_add,
                  const void* col_rec, int64_t n, int64_t m, double* out, double* out_max,
                  double* out_sum, void* workspace, size_t workspace_bytes, void* stream);
/* Finalise partial LSE pairs: out_i = row_add_i - (mx_i + log2 sm_i)/lam. */
int cntgw_lse_finalize(const cntgw_sweep_state* st, int skip_if_done, int prec, const double* mx,
                       const double* sm, const double* row_add, int64_t n, double* out,
                       void* stream);
/* Dense-cost half-update (DenseCost provider, sinkhorn.py:30-56), fp64 cost
 * n x m row-major (stride ld), fp64 throughout like the reference:
 * out_i = row_add_i - LSE2_j(lam pot_j + log2w_j - lam C_ij)/lam. */
int cntgw_softmin_dense(const cntgw_sweep_state* st, int skip_if_done, const double* cost,
                        int64_t ld, const double* pot, const double* log2w, const double* row_add,
                        int64_t n, int64_t m, double* out, void* stream);

/* ---- K4: fused plan pass (solvers.py:227-256, measures.py:185-235) ------- */
/* One fp64 streaming pass over pi_ij = a_i 2^(lam f~_i + t_ij) for the final
 * pair, with fp64 column records (prep_cols prec=CNTGW_F64, sq_flag=1). Per
 * row i: r_i = sum_j pi_ij, piY_i = sum_j pi_ij Y_j (e doubles), pis_i =
 * sum_j pi_ij s_j, and argmax_j pi_ij (lowest j on ties, numpy convention).
 * col_acc: m x e fp64 accumulation features Y (stride ld_acc); col_s: m fp64. */
size_t cntgw_plan_reduce_workspace(int64_t n, int64_t m, int kd, int e);
int cntgw_plan_reduce(const cntgw_sweep_state* st, int kd, int e, const double* row_feat,
                      int64_t ld_row, const double* row_sq, const double* f_tilde,
                      const double* log2a, const double* col_rec, const double* col_acc,
                      int64_t ld_acc, const double* col_s, int64_t n, int64_t m, double* row_mass,
                      double* pi_y, double* pi_s, int64_t* argmax, void* workspace,
                      size_t workspace_bytes, void* stream);

/* K4 for CNTGW_F32C problems: the same per-row outputs (caller order), from
 * the centred blocks of the f-half-update (ctr_rows from cntgw_prep_rows_ctr,
 * ctr_cols from cntgw_prep_cols_ctr with the final g) and that half-update's
 * workspace (plan_ws: its block-sparse plan is checked / rebuilt for the
 * current records and the pass skips the (row group, column tile) pairs that
 * cannot hold a term within 2^-64 of the row's maximum — neither the argmax
 * nor more than m 2^-64 of the row's mass). Exponents are fp64 from the
 * original row features (row_feat n x kd, row_sq); col_order = the column
 * locality order (argmax ties break at the lowest original column);
 * acc_ws: cntgw_plan_reduce_ctr_workspace(m, e) bytes. */
size_t cntgw_plan_reduce_ctr_workspace(int64_t m, int e);
int cntgw_plan_reduce_ctr(const cntgw_sweep_state* st, int kd, int sq_flag, int e, const void* ctr_rows,
                          const void* ctr_cols, const int64_t* col_order, const double* row_feat,
                          int64_t ld_row, const double* row_sq, const double* f_tilde, const double* log2a,
                          const double* col_acc, int64_t ld_acc, const double* col_s, int64_t n, int64_t m,
                          double* row_mass, double* pi_y, double* pi_s, int64_t* argmax, void* plan_ws,
                          size_t plan_ws_bytes, void* acc_ws, size_t acc_ws_bytes, void* stream);

/* K4 for CNTGW_F64S problems: the same per-row outputs (caller order) from
 * the f-half-update's rows block (cntgw_prep_rows_f64s) and ordered fp64
 * records of the final g (cntgw_prep_cols_f64s), skipping the (row group,
 * stage) pairs of that half-update's measured plan (plan_ws = its workspace)
 * while the plan still holds for these records, every stage otherwise;
 * col_order = the column order (argmax ties at the lowest original column).
 * sq_flag must be 1 (the GW cost). acc_ws: cntgw_plan_reduce_ctr_workspace. */
int cntgw_plan_reduce_f64s(const cntgw_sweep_state* st, int kd, int sq_flag, int e, const void* f64s_rows,
                           const double* col_rec, const int64_t* col_order, const double* row_feat,
                           int64_t ld_row, const double* row_sq, const double* f_tilde, const double* log2a,
                           const double* col_acc, int64_t ld_acc, const double* col_s, int64_t n, int64_t m,
                           double* row_mass, double* pi_y, double* pi_s, int64_t* argmax, void* plan_ws,
                           size_t plan_ws_bytes, void* acc_ws, size_t acc_ws_bytes, void* stream);

/* ---- K5/K7: operator, features and objective (solvers.py:219-220, 330-334) */
/* out_i = op . feat_i for op dout x din (fp64, dout*din <= 4096): fp64 result
 * in out64 (n x ld_out) and, if out32 is non-null, its fp32 rounding. */
int cntgw_apply_operator(const double* op, int dout, int din, const double* feat, int64_t ld,
                         int64_t n, double* out64, float* out32, int64_t ld_out, void* stream);
/* Deterministic fp64 row reduction of an outer step. Writes 16 + d*e doubles:
 * [0] sum f~_i r_i, [1] sum s_i^2 r_i, [2] sum |r_i - a_i|, [3] sigma_ss =
 * sum s_i pis_i, [4] sum r_i, [5..15] 0, [16..] Gamma_next = sum_i X_i piY_i^T. */
size_t cntgw_outer_reduce_workspace(int64_t n, int d, int e);
int cntgw_outer_reduce_rows(const double* x, int64_t ldx, int d, const double* pi_y, int e,
                            const double* row_mass, const double* pi_s, const double* f_tilde,
                            const double* s_half, const double* a, int64_t n, double* acc,
                            void* workspace, size_t workspace_bytes, void* stream);
/* Column side from the g-tentative gt of the final pair: c_j = b_j 2^(lam (g~_j
 * - gt_j)); writes 8 doubles: [0] sum g~_j c_j, [1] sum t_j^2 c_j,
 * [2] sum |c_j - b_j|, [3] sum c_j, [4..7] 0. */
int cntgw_outer_reduce_cols(const cntgw_sweep_state* st, const double* g_tilde,
                            const double* g_tent, const double* t_half, const double* b, int64_t m,
                            double* acc, void* workspace, size_t workspace_bytes, void* stream);
/* Weighted moments for the closed-form loss constant (divergence.py:28-47):
 * out = [sum w|x|^2 (raw T), sum w|xc|^4, sum w|xc|^2, sum w xc xc^T (d x d)]
 * with xc = x - sum w x; x fp64 n x d (stride ldx), d <= 64. */
size_t cntgw_moments_workspace(int64_t n, int d);
int cntgw_moments(const double* x, int64_t ldx, int d, const double* w, int64_t n, double* out,
                  void* workspace, size_t workspace_bytes, void* stream);

/* ---- row-sharded multi-GPU exchange (dist.py) ---------------
 * One process per GPU, rows partitioned over ranks. The library talks to NCCL
 * directly (resolved at run time from libnccl.so.2, the instance torch maps)
 * so that every collective is enqueued on the caller's stream and a sharded
 * solve is still one graph-captured launch. cntgw_comm_init is collective:
 * every rank passes the same unique id (rank 0 creates it with
 * cntgw_comm_unique_id and broadcasts cntgw_comm_id_bytes() bytes). */
typedef struct cntgw_comm cntgw_comm;
int cntgw_comm_available(void);  /* 1 if libnccl.so.2 could be resolved */
int cntgw_comm_nccl_version(void);
int cntgw_comm_id_bytes(void);
int cntgw_comm_unique_id(void* id_out);
int cntgw_comm_init(cntgw_comm** out, int world, int rank, const void* id);
int cntgw_comm_destroy(cntgw_comm* comm);
/* fp64 all-reduce, op 0 = sum, 1 = max; send == recv for in place. */
int cntgw_comm_allreduce(cntgw_comm* comm, const double* send, double* recv, int64_t count, int op,
                         void* stream);
/* s_j <- s_j 2^(m_local_j - m_glob_j), 0 for an empty partial (s_j = 0 or
 * m_local_j = -inf): the local step of the partial-LSE combine. */
int cntgw_lse_rescale(const double* m_local, const double* m_glob, double* s, int64_t n, void* stream);
/* The g-update's exchange step: m_glob = allreduce_max(m_local) (out of
 * place), rescale, s = allreduce_sum(s); then cntgw_lse_finalize(m_glob, s)
 * gives every rank the identical full g (no broadcast). */
int cntgw_comm_combine_lse(cntgw_comm* comm, const double* m_local, double* m_glob, double* s, int64_t n,
                           void* stream);

/* ---- device-resident outer loop under CUDA graphs ------------------------- */
int cntgw_outer_state_size(void);
int cntgw_outer_init(cntgw_outer_state* os, double constant, double eps_outer, double delta_outer,
                     int max_outer, void* stream);
/* Objective, gamma_delta, Err and the stop rule / divergence guard for one
 * outer step from the K7 reductions (acc_rows = cntgw_outer_reduce_rows output,
 * acc_cols = cntgw_outer_reduce_cols output); appends one 5-double trace row
 * [objective, gamma_delta, marginal_err, inner_iters, elapsed_s] at
 * trace + 5*step; moves gamma -> gamma_prev and Gamma_{t+1} -> gamma (d*e). */
int cntgw_outer_finish(cntgw_outer_state* os, const cntgw_sweep_state* st, const double* acc_rows,
                       const double* acc_cols, double* gamma, double* gamma_prev, int de,
                       double* trace, void* stream);
/* Stream-capture helpers: begin a capture on `stream` (relaxed mode); open a
 * conditional WHILE node whose body is captured on `body_stream` until
 * cntgw_graph_while_end; the body sets its continuation with
 * cntgw_graph_set_condition (continue while *done_flag == 0). */
int cntgw_graph_begin(void* stream);
int cntgw_graph_while_begin(void* stream, void* body_stream, uint64_t* handle_out);
int cntgw_graph_while_end(void* body_stream);
int cntgw_graph_set_condition(uint64_t handle, const int32_t* done_flag, void* stream);
int cntgw_graph_end(void* stream, void** exec_out);
int cntgw_graph_launch(void* exec, void* stream);
int cntgw_graph_destroy(void* exec);

/* ---- solve-level API: the CNT-GW feature-space solve (solvers.py:628-632) ---
 * A native driver over the entry points above, for callers without the Python
 * package. One handle per device and problem; every buffer is allocated by
 * cntgw_solver_create (the only allocating call of the library) and freed by
 * cntgw_solver_destroy. cntgw_solver_run captures the whole solve — outer loop
 * (stop rule, 5-increase divergence guard), Sinkhorn loops at eps/8 (fixed
 * budget or threshold), plan passes — as ONE CUDA graph and launches it. */
typedef struct cntgw_solve_config {
  double eps;          /* EgwConfig.eps (the Sinkhorn loops run at eps/8)           */
  int mode;            /* 1 symmetrized (default), 0 standard                        */
  int n_inner;         /* fixed sweep budget (threshold == 0)                         */
  double threshold;    /* weighted-gap tolerance, 0 for a fixed budget              */
  int max_inner;       /* sweep cap in threshold mode                                 */
  double anneal_from;  /* SinkhornConfig.anneal_from in eps/8 units, 0 = none         */
  int max_outer;       /* EgwConfig.max_outer                                         */
  double delta_outer;  /* EgwConfig.delta_outer                                       */
  int precision;       /* half-update path: CNTGW_F32, CNTGW_F64 or CNTGW_F64S        */
} cntgw_solve_config;
typedef struct cntgw_solver cntgw_solver;
/* x: n x d and y: m x e centred features, a, b weights (device fp64, caller-
 * owned, alive until destroy). order_x / order_y: locality orders for
 * CNTGW_F64S (NULL = identity). comm: NULL, or a communicator whose ranks each
 * pass their row shard (n rows of n_total; n_rows_max = the largest shard). */
int cntgw_solver_create(cntgw_solver** out, const double* x, int64_t n, int d, const double* y, int64_t m, int e,
                        const double* a, const double* b, const int64_t* order_x, const int64_t* order_y,
                        const cntgw_solve_config* cfg, cntgw_comm* comm, int64_t n_rows_max, void* stream);
int cntgw_solver_destroy(cntgw_solver* solver);
/* f~ = s^2, g~ = t^2: the interaction potentials of the default init (solvers.py:297-301). */
int cntgw_solver_init_potentials(cntgw_solver* solver, double* f, double* g, void* stream);
/* One solve. constant: the loss constant (cntgw_gw_constant). gamma: d*e device
 * fp64, in Gamma_0, out Gamma_{t+1} = EgwResult.gamma; gamma_prev: out Gamma_t
 * (the returned coupling's operator); f, g: device interaction potentials, in
 * the warm start, out the coupling's. trace_host: 5*max_outer doubles, rows
 * [objective, gamma_delta, marginal_err, inner_iters, elapsed_s];
 * status_host[4] = {outer steps, converged, error (SolverError), sweeps applied}. */
int cntgw_solver_run(cntgw_solver* solver, double constant, double* gamma, double* gamma_prev, double* f, double* g,
                     double* trace_host, int* status_host, void* stream);
/* Outputs of the last plan pass copied into caller device buffers (each
 * nullable): row masses (n fp64), argmax plan indices (n int64); eps_eff (host). */
int cntgw_solver_results(const cntgw_solver* solver, double* row_mass, int64_t* argmax, double* eps_eff,
                         void* stream);
/* The loss constant C = Q(X) + Q(Y) - 4 T_X T_Y (divergence.py:28-47) in closed form. */
int cntgw_gw_constant(const double* x, int64_t n, int d, const double* a, const double* y, int64_t m, int e,
                      const double* b, double* out_host, void* stream);

/* ---- kernel PCA: matrix-free cost products (kernels.py:149-345) --------
 * out (n x bcols) = C V with C_ij = c(x_i, x_j) evaluated on the fly in fp64
 * from sq = |x_i|^2 + |x_j|^2 - 2 x_i.x_j clipped at 0 (sqn = |x|^2), c_ii = 0;
 * V: n x bcols row-major, bcols in {8, 16, 32, 64}; par = p (p_norm) or sigma. */
enum cntgw_cost_kind {
  CNTGW_COST_SQEUCLID = 0,
  CNTGW_COST_EUCLIDEAN = 1,
  CNTGW_COST_PNORM = 2,
  CNTGW_COST_EXP = 3
};
int cntgw_cost_product(int kind, double par, const double* x, int64_t n, int d, const double* sqn,
                       const double* v, int bcols, double* out, void* stream);

/* ---- multiscale front end: weighted k-means (solvers.py:668-726) -------
 * Bit-compatible with the reference's numpy _weighted_kmeans (pairwise
 * distance sums, first argmin, Generator.choice draws, index-order centre
 * sums). Points x: n x d fp64 contiguous, d in {1..8, 16, 32, 64}.
 * k-means++ draw j: p = w (d2 == NULL) or w*d2 / pairwise_sum(w*d2) (w if the
 * sum is 0); idx = first i with cumsum(p)_i / cumsum(p)_{n-1} > u[j] (device
 * u[*jp]). leaf_off: nleaves+1 offsets of numpy's pairwise-sum leaves of n;
 * tree/hoff/nh: the internal nodes of numpy's pairwise recursion, level by
 * level (nh levels, hoff[nh+1] offsets into tree, each entry a
 * (node, left, right) id triple; leaves are 0..nleaves-1), combined in the
 * reference's order. The draw index lives on the device (*jp) so a captured
 * sequence of draws can be replayed. */
size_t cntgw_km_draw_workspace(int64_t n, int nleaves);
int cntgw_km_draw(const double* w, const double* d2, int64_t n, const int64_t* leaf_off,
                  int nleaves, const int* tree, const int* hoff, int nh, const double* u,
                  const int* jp, int64_t* out_idx, void* workspace, size_t workspace_bytes,
                  void* stream);
/* centers[*jp] = x[*idx]; d2 = |x - c|^2 (first) or min(d2, |x - c|^2); then ++*jp */
int cntgw_km_update_d2(const double* x, int64_t n, int d, const int64_t* idx, double* centers,
                       int* jp, double* d2, int first, void* stream);
/* assign_i = first argmin_j |x_i - c_j|^2, own_i = that distance */
int cntgw_km_assign(const double* x, int64_t n, int d, const double* centers, int64_t k,
                    int64_t* assign, double* own, void* stream);
/* per listed cluster c (id ids[c], or c): members[offsets[c]:offsets[c+1]] in
 * index order -> centers[id] = sum fl(w x) / pairwise_sum(w) (skipped when
 * empty), or, if masses != NULL, masses[id] = sequential sum of w. */
int cntgw_km_centers(const double* x, int d, const double* w, const int64_t* members,
                     const int64_t* offsets, int64_t ncl, const int64_t* ids, double* centers,
                     double* masses, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CNTGW_B200_H */
