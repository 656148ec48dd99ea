// C ABI of the B200-native CNT-GW hot path: sweep control, column packing,
// half-update dispatch (fp32 / fp64 paths), workspace sizing and error
// reporting. Declarations and contracts: include/cntgw_b200.h.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <string>

#include "common.cuh"
#include "softmin.cuh"
#include "softmin_ctr.cuh"
#include "softmin_ctr_tc.cuh"
#include "softmin_dmma.cuh"
#include "softmin_f64s.cuh"
#include "softmin_f64s_probe.cuh"
#include "softmin_f64s_tcprobe.cuh"
#include "reduce_ctr.cuh"
#include "softmin_tc.cuh"
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
  return set_error(code, buf);
}

int check_launch(const char* what) {
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) cudaGetLastError();
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

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// ---- per-(precision, kd, sq) kernel configuration --------------------------
template <int KD>
constexpr int rows_f32() { return KD <= 8 ? 8 : (KD <= 16 ? 4 : 2); }
template <int KD>
constexpr int minb_f32() { return KD <= 4 ? 4 : (KD <= 16 ? 3 : (KD <= 32 ? 2 : 1)); }
template <int KD>
constexpr int rows_f64() { return KD <= 8 ? 4 : (KD <= 32 ? 2 : 1); }
template <int KD>
constexpr int minb_f64() { return KD <= 4 ? 3 : (KD <= 16 ? 2 : 1); }
template <int KD>
constexpr int group_g() { return KD <= 32 ? 4 : 2; }
template <int KD>
// small-K fp64: 8-term groups halve the per-row check/fold overhead (measured +4%)
constexpr int group_f64() { return KD <= 4 ? 8 : group_g<KD>(); }
// columns per shared-memory stage: 256 unless two stages would exceed 200 KB
template <typename T, int KD, int SQ>
constexpr int stage_cols() {
  return 2 * 256 * ColLayout<T, KD, SQ>::kStride * (int)sizeof(T) <= 200 * 1024 ? 256 : 128;
}

struct KernelPick {
  void* fn;
  int rows;  // rows per thread (CTA rows = 128 * rows)
  size_t smem;
  int threads = 128;
  size_t rec_bytes = 0;  // bytes of column records per column (L2 chunking)
  int l2_chunk_mb = 32;  // default L2 budget of one column chunk (CNTGW_L2_CHUNK_MB overrides)
  int cta_rows = 0;      // rows per CTA when not 128 * rows
  int ctr_kx = 0;        // CNTGW_F32C FFMA2 kernel: feature width and groups per CTA
  int ctr_r = 0;         //   (block-sparse plan, ctr_plan_kernel)
  int f64s_tile = 0;     // CNTGW_F64S: column stage of the measured plan (kernel takes F64sArgs)
  void* probe_fn = nullptr;  // CNTGW_F64S, kd + sq <= 8: the fp32 probe of a dense measurement
  void* probe_prep_fn = nullptr;
  int probe_rows = 0;        //   rows per probe CTA (128 threads x R)
  int probe_p = 0;           //   floats per probe record (fp32 record / fp16 stage tile column)
  void* tcp_fn = nullptr;        // CNTGW_F64S: the tcgen05 probe (softmin_f64s_tcprobe.cuh), any width
  void* tcp_stats_fn = nullptr;
  void* tcp_pack_fn = nullptr;
  int tcp_threads = 0;
  int tcp_tile = 0;              //   columns per probe tile (a whole number of plan stages)
  size_t tcp_smem = 0;
  size_t tcp_stage_bytes = 0;
};

// CNTGW_F64S: the DMMA kernel's tiling on ordered rows and columns with a
// measured block-sparse plan (softmin_f64s.cuh). RG groups of 8 rows per warp
// (32 RG rows per CTA = the plan's row group), NT 8-column tiles per step, TD
// columns per stage, MB CTAs per SM.
template <int KD, int SQ, int RG, int NT, int TD, int MB>
KernelPick f64s_variant() {
  KernelPick k;
  k.fn = (void*)softmin_f64s_kernel<KD, SQ, RG, NT, TD, MB>;
  k.rows = 1;
  k.cta_rows = 32 * RG;
  k.smem = (size_t)2 * TD * ColLayout<double, KD, SQ>::kStride * sizeof(double);
  k.rec_bytes = ColLayout<double, KD, SQ>::kStride * sizeof(double);
  k.f64s_tile = TD;
  // the sweeps are sparse (the probe re-plans above 12% kept), so their records fit the L2
  // without column chunks: half the CTAs and no partials to combine at C4 2^20
  k.l2_chunk_mb = 1024;
  if constexpr (KD + SQ <= 8) {
    constexpr int R = KD + SQ <= 4 ? 16 : 8;
    k.probe_fn = (void*)f64s_probe_kernel<KD, SQ, R, TD>;
    k.probe_prep_fn = (void*)f64s_probe_prep_kernel<KD + SQ>;
    k.probe_rows = 128 * R;
    k.probe_p = ProbeLayout<KD + SQ>::kP;
  }
  {
    using TL = TcpLayout<KD + SQ>;
    constexpr int PT = TD < 128 ? 128 : TD;  // probe tile: two 64-column stages per MMA tile
    constexpr int NB = 512 / PT < 4 ? 512 / PT : 4;
    k.tcp_fn = (void*)f64s_tcp_kernel<KD + SQ, PT, TD>;
    k.tcp_stats_fn = (void*)f64s_tcp_stats_kernel<KD + SQ>;
    k.tcp_pack_fn = (void*)f64s_tcp_pack_kernel<KD + SQ>;
    k.tcp_threads = 64 + 128 * NB;
    k.tcp_tile = PT;
    k.tcp_stage_bytes = (size_t)TL::kChunks * PT * 16;
    k.tcp_smem = (size_t)TL::kATileBytes + tcp_ring<KD + SQ, PT>() * k.tcp_stage_bytes;
    if (TL::kP > k.probe_p) k.probe_p = TL::kP;
  }
  return k;
}

// Plan granularity, measured on the 10-step solves (tools/gpu/r2_s3_20.sh .. r2_s3_25.sh): the
// (row group, column stage) block is the unit the plan keeps or skips, so smaller blocks walk
// fewer pairs at a lower DMMA reuse of each B fragment and a longer probe (more stages).
// kd < 16 (C4 2^20): 32-row groups 16.1 s, 64-row 17.2 s; 128-column stages 18.0 s (probe 67 ->
// 109 ms). 16 <= kd < 64 (C5 2^18): 128 rows x 128 columns 17.1 s, 64 x 128 13.3 s, 64 x 64
// 11.2 s, 32 x 64 10.0 s. (The stage width is f64s_stage_cols, shared with the plan consumers.)
template <int KD, int SQ>
KernelPick pick_f64s() {
  constexpr int RG = KD >= 64 ? 2 : 1, NT = KD >= 16 ? 1 : 4;
  constexpr int TD = f64s_stage_cols(KD), MB = KD >= 64 ? 3 : 5;
  return f64s_variant<KD, SQ, RG, NT, TD, MB>();
}

template <int PREC, int KD, int SQ>
KernelPick pick() {
  KernelPick k;
  if (PREC == CNTGW_F32) {
    constexpr int T = stage_cols<float, KD, SQ>();
    k.fn = (void*)softmin_f32_kernel<KD, SQ, rows_f32<KD>(), group_g<KD>(), minb_f32<KD>(), T>;
    k.rows = rows_f32<KD>();
    k.smem = 2 * (size_t)T * ColLayout<float, KD, SQ>::kStride * sizeof(float);
    k.rec_bytes = ColLayout<float, KD, SQ>::kStride * sizeof(float);
  } else {
    constexpr int T = stage_cols<double, KD, SQ>();
    k.fn = (void*)softmin_f64_kernel<KD, SQ, rows_f64<KD>(), group_f64<KD>(), minb_f64<KD>(), T>;
    k.rows = rows_f64<KD>();
    k.smem = 2 * (size_t)T * ColLayout<double, KD, SQ>::kStride * sizeof(double);
    k.rec_bytes = ColLayout<double, KD, SQ>::kStride * sizeof(double);
    // the dot on the FP64 tensor pipe (DMMA); CNTGW_F64_DMMA=0 keeps the DFMA kernel
    if (env_int("CNTGW_F64_DMMA", 1)) {
      // wide K: 4 row groups x 1 column tile per step (the A fragments dominate
      // the registers); small K: 2 row groups x 4 column tiles per step (all 8
      // MMAs of a step in flight before the epilogue). 2-stage column ring
      // with per-warp release (StageRing; measured equal to a block barrier
      // per tile, and to 4/6 stages).
      constexpr int RG = KD >= 64 ? 2 : (KD >= 16 ? 4 : 2), NT = KD >= 16 ? 1 : 4;
      constexpr int TD = KD >= 64 ? 64 : (KD >= 16 ? 128 : 256), MB = KD >= 16 ? 3 : 4;
      k.fn = (void*)softmin_dmma_kernel<KD, SQ, RG, NT, TD, MB>;
      k.cta_rows = 32 * RG;
      k.smem = (size_t)2 * TD * ColLayout<double, KD, SQ>::kStride * sizeof(double);
      if constexpr (KD < 16) {  // tuning alternatives (tools/sweep_paths.py)
        const int v = env_int("CNTGW_DMMA_NT", 0);
        if (v == 2) k.fn = (void*)softmin_dmma_kernel<KD, SQ, 4, 2, TD, MB>, k.cta_rows = 128;
        if (v == 11) k.fn = (void*)softmin_dmma_kernel<KD, SQ, RG, NT, TD, MB, 2, 1>;
      }
    }
  }
  return k;
}

#define KD_SQ_CASES(PREC, X) \
  X(PREC, 1, 0) X(PREC, 1, 1) X(PREC, 2, 0) X(PREC, 2, 1) X(PREC, 3, 0) X(PREC, 3, 1) \
  X(PREC, 4, 0) X(PREC, 4, 1) X(PREC, 8, 0) X(PREC, 8, 1) X(PREC, 16, 0) X(PREC, 16, 1) \
  X(PREC, 32, 0) X(PREC, 32, 1) X(PREC, 64, 0) X(PREC, 64, 1)

// Tensor-core variant knobs (read per call so tools can sweep them):
// CNTGW_TC_KIND = f16 (default: the 3-way split on fp16 operands, kind::f16)
// or tf32 (kind::tf32); CNTGW_TC_POLY in {0,2,3,4,6} (default 3 with fp16
// operands, 2 with tf32: fastest in tools/sweep_paths.py): pairs (of 16 per
// 32-column chunk) whose exp2 runs on the FMA pipe instead of MUFU;
// CNTGW_TC_EPI in {8,16}: epilogue warps (default 16). Measured slower and
// removed: one reference check per 64 columns (both chunks loaded up front,
// 253 vs 245 ms per C2 half-update: the next chunk's TMEM load no longer
// overlaps the math).
bool tc_f16() {
  const char* e = getenv("CNTGW_TC_KIND");
  return !(e && (e[0] == 't' || e[0] == 'T'));
}

template <int KD, int EPI, bool H>
void* tc_fn(int poly) {
  switch (poly) {
    case 2: return (void*)softmin_tc_kernel<KD, 2, EPI, H>;
    case 3: return (void*)softmin_tc_kernel<KD, 3, EPI, H>;
    case 4: return (void*)softmin_tc_kernel<KD, 4, EPI, H>;
    case 6: return (void*)softmin_tc_kernel<KD, 6, EPI, H>;
    default: return (void*)softmin_tc_kernel<KD, 0, EPI, H>;
  }
}

template <int KD>
KernelPick pick_tc() {
  KernelPick k;
  const bool h = tc_f16();
  const int poly = env_int("CNTGW_TC_POLY", h ? 3 : 2);
  const int epi = env_int("CNTGW_TC_EPI", 16) == 8 ? 8 : 16;
  if (h) k.fn = epi == 16 ? tc_fn<KD, 16, true>(poly) : tc_fn<KD, 8, true>(poly);
  else k.fn = epi == 16 ? tc_fn<KD, 16, false>(poly) : tc_fn<KD, 8, false>(poly);
  k.rows = 1;  // 128 rows per CTA = 128 threads x 1 in the planner's units
  const size_t a_bytes = h ? TcLayoutH<KD>::kATileBytes : TcLayout<KD>::kATileBytes;
  const size_t b_bytes = h ? TcLayoutH<KD>::kBTileBytes : TcLayout<KD>::kBTileBytes;
  k.smem = a_bytes + kTcStages * b_bytes;
  k.rec_bytes = h ? TcLayoutH<KD>::kRecBytes : TcLayout<KD>::kRecBytes;
  // C2 2^20 per half-update: 48 MB chunks 245.1 ms / 0.45 GB of DRAM traffic, 32 MB 245.5 ms /
  // 0.48 GB, 64 MB 243.2 ms / 3.5 GB (past the L2's effective capacity), unchunked 243.9 ms
  k.l2_chunk_mb = 48;
  k.threads = tc_threads(epi);
  return k;
}

// CNTGW_F32C: centred fp32 pairs over locality-ordered tiles (softmin_ctr.cuh);
// KX = kd + sq padded to 4 (8 rows per thread) or 8 (4 rows per thread).
template <int KX, int R = (KX <= 4 ? 8 : 4)>
KernelPick pick_ctr() {
  constexpr int MINB = KX <= 4 ? (R <= 4 ? 6 : 4) : 3;
  KernelPick k;
  // tuning alternatives (tools/ctr_check.py): CNTGW_CTR_POLY=1 puts one row
  // pair of each column group on the FMA-pipe exp2; CNTGW_CTR_G=8 checks the
  // lazy rebase once per 8 columns instead of 4
  const int poly = env_int("CNTGW_CTR_POLY", 0), g8 = env_int("CNTGW_CTR_G", 4) == 8;
  k.fn = g8 ? (void*)softmin_ctr_kernel<KX, R, 8, MINB, 0>
       : poly == 1 ? (void*)softmin_ctr_kernel<KX, R, 4, MINB, 1>
                   : (void*)softmin_ctr_kernel<KX, R, 4, MINB, 0>;
  k.rows = R;
  k.smem = CtrSmem<KX, R>::kBytes;
  k.rec_bytes = (KX + 1) * sizeof(double) + KX * sizeof(float);
  k.ctr_kx = KX;
  k.ctr_r = R;
  return k;
}

// Block-sparse plan of the centred FFMA2 kernel: fp32 rho table [CTA][R][tile]
// and the needed-tile mask [CTA][tile]; CNTGW_CTR_SKIP=0 disables it.
bool ctr_skip_enabled(const KernelPick& k) { return k.ctr_kx > 0 && env_int("CNTGW_CTR_SKIP", 1) != 0; }
size_t ctr_plan_bytes(const KernelPick& k, int64_t n, int64_t m) {
  if (!ctr_skip_enabled(k)) return 0;
  const int64_t ctas = (ctr_groups(n) + k.ctr_r - 1) / k.ctr_r;
  const int64_t tl = (m + kColTile - 1) / kColTile;
  return align256(sizeof(float) * ctas * k.ctr_r * tl) + align256(sizeof(uint32_t) * ctas * tl) +
         align256(sizeof(double) * tl * kColTile) + 256;  // + c at the last plan, CtrPlanKey
}

// Measured plan of the CNTGW_F64S kernel: tmin [n][stages] fp32, need
// [row tiles][stages] bytes, c at the last plan [mpad] fp64, CtrPlanKey.
struct F64sPlanLayout {
  size_t tmin, need, cplan, range, gmin, tstar, rowmin, rec32, sbound, total;
  int stages;
  int64_t row_tiles;
};
F64sPlanLayout f64s_layout(const KernelPick& k, int64_t n, int64_t m) {
  F64sPlanLayout l{};
  if (k.f64s_tile == 0) return l;
  const int64_t mpad = (m + kColTile - 1) / kColTile * kColTile;
  l.stages = (int)(mpad / k.f64s_tile);
  l.row_tiles = (n + k.cta_rows - 1) / k.cta_rows;
  l.tmin = align256(sizeof(float) * (size_t)n * l.stages);
  l.need = align256((size_t)l.row_tiles * l.stages);
  l.cplan = align256(sizeof(double) * (size_t)mpad);
  l.range = align256(sizeof(double2) * (size_t)l.stages);
  l.gmin = align256(sizeof(float) * (size_t)l.row_tiles * l.stages);
  l.tstar = align256(sizeof(int) * (size_t)n);
  l.rowmin = align256(sizeof(double) * (size_t)n);
  l.rec32 = k.probe_p ? align256(sizeof(float) * (size_t)mpad * k.probe_p) : 0;
  l.sbound = k.probe_p ? std::max(align256(sizeof(float) * (size_t)l.stages * k.probe_p), tcp_bounds_bytes(l.stages)) : 0;
  l.total = l.tmin + l.need + l.cplan + l.range + l.gmin + l.tstar + l.rowmin + 256 + l.rec32 + l.sbound;
  // (the 256 bytes after rowmin: CtrPlanKey, flags)
  return l;
}

// Pointers into the F64S plan workspace (after the split-column partials).
struct F64sPlan {
  float* tmin;
  uint8_t* need;
  double* c_plan;
  double2* range;
  float* gmin;
  int* tstar;
  double* rowmin;
  CtrPlanKey* key;
  int* flag;
  int* counter;
  int* next_measure;
  int* full;
  int* nan;        // the probe stands down (non-finite records)
  int* probe_ok;   // this sweep's plan came from the probe
  float* slack;    // the probe's 2 max E (log2 units)
  int* sched;      // re-measurement schedule: interval, kept pairs before the last one, pending, its sweep
  int* dotzero;    // [0] any nonzero row dot feature, [1] any nonzero column dot feature (per call)
  float* rec32;    // fp32 probe records [mpad][P]
  float* sbound;   // per stage magnitude bounds [stages][P]
};
F64sPlan f64s_plan(void* base_v, const F64sPlanLayout& l) {
  char* base = static_cast<char*>(base_v);
  F64sPlan p;
  p.tmin = reinterpret_cast<float*>(base);
  p.need = reinterpret_cast<uint8_t*>(base + l.tmin);
  p.c_plan = reinterpret_cast<double*>(base + l.tmin + l.need);
  p.range = reinterpret_cast<double2*>(base + l.tmin + l.need + l.cplan);
  p.gmin = reinterpret_cast<float*>(base + l.tmin + l.need + l.cplan + l.range);
  p.tstar = reinterpret_cast<int*>(base + l.tmin + l.need + l.cplan + l.range + l.gmin);
  p.rowmin = reinterpret_cast<double*>(base + l.tmin + l.need + l.cplan + l.range + l.gmin + l.tstar);
  p.key = reinterpret_cast<CtrPlanKey*>(base + l.tmin + l.need + l.cplan + l.range + l.gmin + l.tstar + l.rowmin);
  p.flag = &p.key->replan;
  p.counter = reinterpret_cast<int*>(reinterpret_cast<char*>(p.key) + 128);
  p.next_measure = p.counter + 1;
  p.full = p.counter + 2;
  p.nan = p.counter + 3;
  p.probe_ok = p.counter + 4;
  p.slack = reinterpret_cast<float*>(p.counter + 5);
  p.sched = p.counter + 6;
  p.dotzero = p.counter + 10;
  char* tail = base + l.tmin + l.need + l.cplan + l.range + l.gmin + l.tstar + l.rowmin + 256;
  p.rec32 = l.rec32 ? reinterpret_cast<float*>(tail) : nullptr;
  p.sbound = l.sbound ? reinterpret_cast<float*>(tail + l.rec32) : nullptr;
  return p;
}

// CNTGW_F64S_PROBE=0: dense fp64 measurements; CNTGW_F64S_PROBE_TC=0: the FFMA2 probe (kd + sq <= 8)
bool f64s_tcp_enabled(const KernelPick& k) {
  return k.tcp_fn != nullptr && env_int("CNTGW_F64S_PROBE", 1) != 0 && env_int("CNTGW_F64S_PROBE_TC", 1) != 0;
}
bool f64s_probe_enabled(const KernelPick& k) {
  return (k.probe_fn != nullptr || f64s_tcp_enabled(k)) && env_int("CNTGW_F64S_PROBE", 1) != 0;
}

// f64s_reduce_kernel: two row-minimum arrays + the walked-stage list (uint16)
size_t f64s_reduce_smem(const KernelPick& k, int stages) {
  return 2 * sizeof(double) * k.cta_rows + (stages <= kF64sListMax ? sizeof(uint16_t) * (size_t)stages : 0);
}

// Re-vote the measured plan for the current records (f64s_* kernels,
// softmin_f64s.cuh); leaves *flag = 1 when the sweep must measure anew (or,
// for a consumer such as K4, walk every stage).
// (gate: run only when *gate, e.g. the re-vote after a probe)
int f64s_vote(const KernelPick& k, const F64sPlanLayout& l, const F64sPlan& pl, const cntgw_sweep_state* st,
              const double* rec, int kd, int sq, int64_t n, int64_t m, cudaStream_t s, int schedule,
              const int* gate, int skip) {
  const int stride = (kd + sq + 1 + 1) / 2 * 2 > (kd + sq + 3) / 4 * 4 ? (kd + sq + 1 + 1) / 2 * 2
                                                                       : (kd + sq + 3) / 4 * 4;
  f64s_shift_kernel<<<(unsigned)l.stages, 128, 0, s>>>(rec, stride, kd + sq, m, k.f64s_tile, pl.c_plan, pl.range,
                                                        pl.flag, pl.full, gate);
  // Sweeps skip terms below 2^-48 of their row's maximum: the skipped mass, < m 2^-48 of the row
  // sum, stays 16x under the fp32 rounding (2^-24) of the kernel's per-stage partial sums at
  // m = 2^20. The plan consumers (K4: fp64 exponentials and sums, schedule == 0) keep 2^-64.
  const char* te = getenv("CNTGW_CTR_SKIP_T");
  const double T = te ? atof(te) : (schedule ? 48.0 : 64.0);
  f64s_vote_kernel<<<(unsigned)l.row_tiles, 256, 0, s>>>(pl.flag, pl.gmin, pl.tstar, pl.range, n, l.stages,
                                                         k.cta_rows, T, pl.need, pl.counter, gate);
  // kept fraction above which the sweep measures anew: with the tcgen05 probe a fresh plan costs
  // ~0.1 dense sweeps (probe + exact sweep on its plan), so walking more than 12% does not pay
  const char* fe = getenv("CNTGW_F64S_REMEASURE");
  const double frac = fe ? atof(fe) : (f64s_tcp_enabled(k) ? 0.12 : 0.25);
  f64s_decide_kernel<<<1, 1, 0, s>>>(st, pl.flag, pl.counter, pl.next_measure, l.row_tiles * (int64_t)l.stages,
                                     frac, schedule, gate, skip, pl.sched, pl.full,
                                     f64s_probe_enabled(k) ? 1 : 0);
  return check_launch("f64s_vote");
}
int f64s_revote(const KernelPick& k, const F64sPlanLayout& l, const F64sPlan& pl, const cntgw_sweep_state* st,
                const double* rec, int kd, int sq, const void* rows, const void* cols, int64_t n, int64_t m,
                cudaStream_t s, int schedule, int skip) {
  f64s_begin_kernel<<<1, 1, 0, s>>>(st, skip, pl.key, rows, cols, n, m, pl.flag, pl.counter, pl.full, pl.sched);
  return f64s_vote(k, l, pl, st, rec, kd, sq, n, m, s, schedule, nullptr, skip);
}

// The probe of a dense measurement, all gated on the device flags: statistics
// / prep + row check (iff *full), gate, probe, reduce and commit of its plan,
// then the re-vote on it. Leaves the sweep non-measuring (or a partial
// measurement when the probe's plan keeps too much).
// -- the tensor-core probe (softmin_f64s_tcprobe.cuh), any width
int f64s_probe_tc(const KernelPick& k, const F64sPlanLayout& l, const F64sPlan& pl, const double* rec, int stride,
                  int kd, int sq, const void* rows, int64_t n, int64_t m, int64_t mpad, cudaStream_t s) {
  int stages = l.stages;
  __half* tiles = reinterpret_cast<__half*>(pl.rec32);
  f64s_tcp_begin_kernel<<<1, 1, 0, s>>>(pl.sbound, stages);
  {
    void* args[] = {(void*)&pl.full,     (void*)&rec,       (void*)&stride, (void*)&m,
                    (void*)&k.f64s_tile, (void*)&pl.sbound, (void*)&stages, (void*)&pl.nan};
    const cudaError_t e = cudaLaunchKernel(k.tcp_stats_fn, dim3(l.stages), dim3(128), args, 0, s);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(CNTGW_ECUDA, "f64s tc probe stats: %s", cudaGetErrorString(e));
    }
  }
  f64s_tcp_rows_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 8 * num_sms()), 256, 0, s>>>(
      pl.full, rows, n, kd, sq, pl.sbound, stages, pl.nan);
  f64s_probe_gate_kernel<<<1, 1, 0, s>>>(pl.full, pl.nan, pl.probe_ok, pl.slack);
  f64s_tcp_scales_kernel<<<1, 1, 0, s>>>(pl.probe_ok, pl.sbound, stages);
  const int ptiles = (int)(mpad / k.tcp_tile);
  {
    void* args[] = {(void*)&pl.probe_ok, (void*)&rec,   (void*)&stride,    (void*)&m,
                    (void*)&k.tcp_tile,  (void*)&tiles, (void*)&pl.sbound, (void*)&stages};
    const cudaError_t e = cudaLaunchKernel(k.tcp_pack_fn, dim3(ptiles), dim3(128), args, 0, s);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(CNTGW_ECUDA, "f64s tc probe pack: %s", cudaGetErrorString(e));
    }
  }
  // probe tiles in chunks of <= 48 MB (L2), at least ~2 waves of CTAs
  const int64_t rt = (n + kTcRows - 1) / kTcRows;
  const int64_t fit = std::max<int64_t>(1, ((int64_t)48 << 20) / (int64_t)k.tcp_stage_bytes);
  int chunks = (int)((ptiles + fit - 1) / fit);
  chunks = (int)std::max<int64_t>(chunks, std::min<int64_t>(ptiles, (2 * num_sms() + rt - 1) / rt));
  const int cs = (ptiles + chunks - 1) / chunks;
  chunks = (ptiles + cs - 1) / cs;
  cudaFuncSetAttribute(k.tcp_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.tcp_smem);
  void* args[] = {(void*)&pl.probe_ok, (void*)&rows,   (void*)&n,  (void*)&kd,      (void*)&tiles,
                  (void*)&pl.sbound,   (void*)&stages, (void*)&cs, (void*)&pl.tmin, (void*)&pl.slack};
  const cudaError_t e =
      cudaLaunchKernel(k.tcp_fn, dim3((unsigned)rt, (unsigned)chunks), dim3(k.tcp_threads), args, k.tcp_smem, s);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(CNTGW_ECUDA, "f64s tc probe: %s", cudaGetErrorString(e));
  }
  return CNTGW_OK;
}

// -- the fp32 FFMA2 probe (softmin_f64s_probe.cuh), kd + sq <= 8
int f64s_probe_ffma(const KernelPick& k, const F64sPlanLayout& l, const F64sPlan& pl, const cntgw_sweep_state* st,
                    int skip, const double* rec, int stride, int kd, int sq, const void* rows, int64_t n, int64_t m,
                    cudaStream_t s) {
  {
    void* args[] = {(void*)&pl.full, (void*)&rec, (void*)&stride, (void*)&m, (void*)&k.f64s_tile,
                    (void*)&pl.rec32, (void*)&pl.sbound, (void*)&pl.nan};
    const cudaError_t e = cudaLaunchKernel(k.probe_prep_fn, dim3(l.stages), dim3(128), args, 0, s);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(CNTGW_ECUDA, "f64s probe prep: %s", cudaGetErrorString(e));
    }
  }
  f64s_probe_rows_check_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 8 * num_sms()), 256, 0, s>>>(
      pl.full, rows, n, kd, sq, pl.nan);
  f64s_probe_gate_kernel<<<1, 1, 0, s>>>(pl.full, pl.nan, pl.probe_ok, pl.slack);
  const int64_t rt = (n + k.probe_rows - 1) / k.probe_rows;
  // enough CTAs for ~4 waves of 2 per SM: split the stages into chunks
  int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(l.stages, (8 * num_sms() + rt - 1) / rt));
  const int cs = (l.stages + chunks - 1) / chunks;
  chunks = (l.stages + cs - 1) / cs;
  const size_t smem = (size_t)2 * k.f64s_tile * k.probe_p * sizeof(float);
  int stages = l.stages;
  void* args[] = {(void*)&st, (void*)&skip, (void*)&pl.probe_ok, (void*)&rows, (void*)&n, (void*)&pl.rec32,
                  (void*)&pl.sbound, (void*)&stages, (void*)&cs, (void*)&pl.tmin, (void*)&pl.slack};
  const cudaError_t e = cudaLaunchKernel(k.probe_fn, dim3((unsigned)rt, (unsigned)chunks), dim3(128), args, smem, s);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(CNTGW_ECUDA, "f64s probe: %s", cudaGetErrorString(e));
  }
  return CNTGW_OK;
}

int f64s_probe(const KernelPick& k, const F64sPlanLayout& l, const F64sPlan& pl, const cntgw_sweep_state* st,
               int skip, const double* rec, int kd, int sq, const void* rows, const void* cols, int64_t n, int64_t m,
               cudaStream_t s) {
  const int stride = cntgw_col_stride(CNTGW_F64S, kd, sq);
  const int64_t mpad = (m + kColTile - 1) / kColTile * kColTile;
  cudaMemsetAsync(pl.nan, 0, sizeof(int), s);
  const int rc = f64s_tcp_enabled(k) ? f64s_probe_tc(k, l, pl, rec, stride, kd, sq, rows, n, m, mpad, s)
                                     : f64s_probe_ffma(k, l, pl, st, skip, rec, stride, kd, sq, rows, n, m, s);
  if (rc != CNTGW_OK) return rc;
  f64s_reduce_kernel<<<(unsigned)l.row_tiles, 256, f64s_reduce_smem(k, l.stages), s>>>(
      pl.probe_ok, pl.probe_ok, pl.tmin, pl.need, pl.range, n, l.stages, k.cta_rows, pl.gmin, pl.tstar, pl.rowmin,
      0.f, pl.slack);
  f64s_commit_kernel<<<1, 1024, 0, s>>>(pl.probe_ok, st, rec, stride, kd + sq, mpad, pl.c_plan, pl.key, rows, cols,
                                        n, m, pl.next_measure, pl.counter, pl.sched);
  f64s_probed_kernel<<<1, 1, 0, s>>>(pl.probe_ok, pl.flag, pl.full, pl.counter);
  return f64s_vote(k, l, pl, st, rec, kd, sq, n, m, s, 1, pl.probe_ok, skip);
}
size_t f64s_plan_bytes(const KernelPick& k, int64_t n, int64_t m) { return f64s_layout(k, n, m).total; }

// CNTGW_F32C, kx <= 4, on tcgen05 (softmin_ctr_tc.cuh), opt-in with CNTGW_CTR_TC=1:
// 11% faster than the FFMA2 kernel at the C4 law but its split-tf32 products
// and tensor-core accumulation move the 10-step C4 trajectory by up to 5.5e-4
// (objective) against 2.3e-5 for the FFMA2 kernel (profiles/r1_ctr_c4_solve.txt)
KernelPick pick_ctc() {
  KernelPick k;
  // CNTGW_CTR_TC_POLY: pairs (of 16 per 32-column chunk) exponentiated on the FMA pipe
  switch (env_int("CNTGW_CTR_TC_POLY", 4)) {
    case 0: k.fn = (void*)softmin_ctc_kernel<16, 0>; break;
    case 2: k.fn = (void*)softmin_ctc_kernel<16, 2>; break;
    case 6: k.fn = (void*)softmin_ctc_kernel<16, 6>; break;
    case 8: k.fn = (void*)softmin_ctc_kernel<16, 8>; break;
    default: k.fn = (void*)softmin_ctc_kernel<16, 4>; break;
  }
  k.rows = 1;  // one 128-row group per CTA
  k.smem = CtcSmem<16>::kBytes;
  k.threads = ctc_threads(16);
  k.rec_bytes = 16 * sizeof(float) + (kCtcKx + 1) * sizeof(double);
  return k;
}

bool lookup(int prec, int kd, int sq, KernelPick* out) {
  if (prec == CNTGW_F32C) {
    if (!kd_supported(kd)) return false;
    const int kx = kd + (sq ? 1 : 0);
    if (kx <= 4 && env_int("CNTGW_CTR_TC", 0)) { *out = pick_ctc(); return true; }
    // 4 row groups per CTA (finer block-sparse granularity, and faster dense:
    // 3.3e12 vs 3.14e12 at the C4 law); CNTGW_CTR_R=8 / 2 for 8 / 2 groups
    // (2 groups: 12.8e12 vs 14.8e12 N*M pairs/s 100 sweeps into C4)
    if (kx <= 4) {
      const int r = env_int("CNTGW_CTR_R", 4);
      *out = r == 8 ? pick_ctr<4, 8>() : (r == 2 ? pick_ctr<4, 2>() : pick_ctr<4, 4>());
      return true;
    }
    if (kx <= 8) { *out = pick_ctr<8>(); return true; }
    return false;
  }
  if (prec == CNTGW_F64S) {
#define PICK_S(K, Q) \
  if (kd == K && (sq ? 1 : 0) == Q) { *out = pick_f64s<K, Q>(); return true; }
    PICK_S(1, 0) PICK_S(1, 1) PICK_S(2, 0) PICK_S(2, 1) PICK_S(3, 0) PICK_S(3, 1) PICK_S(4, 0) PICK_S(4, 1)
    PICK_S(8, 0) PICK_S(8, 1) PICK_S(16, 0) PICK_S(16, 1) PICK_S(32, 0) PICK_S(32, 1) PICK_S(64, 0) PICK_S(64, 1)
#undef PICK_S
    return false;
  }
  if (prec == CNTGW_TF32X3) {
    if (sq) return false;
    if (kd == 8) { *out = pick_tc<8>(); return true; }
    if (kd == 16) { *out = pick_tc<16>(); return true; }
    return false;
  }
#define PICK_CASE(P, K, Q) \
  if (prec == P && kd == K && (sq ? 1 : 0) == Q) { *out = pick<P, K, Q>(); return true; }
  KD_SQ_CASES(CNTGW_F32, PICK_CASE)
  KD_SQ_CASES(CNTGW_F64, PICK_CASE)
#undef PICK_CASE
  return false;
}

struct Plan {
  int row_tiles;
  int nchunks;
  int64_t chunk_cols;
};

// Split the padded columns into chunks so that row_tiles * nchunks CTAs fill
// whole waves of the resident-CTA capacity (tail < 3% when possible).
Plan plan_softmin(int64_t n, int64_t m, const KernelPick& k) {
  Plan p;
  const int64_t rows_per_cta = k.cta_rows > 0 ? k.cta_rows : 128LL * k.rows;
  p.row_tiles = (int)((n + rows_per_cta - 1) / rows_per_cta);
  const int64_t tiles = (m + kColTile - 1) / kColTile;
  int occ = 1;
  // the dynamic shared-memory opt-in must precede the occupancy query, or a
  // workspace query made before the first launch plans with a different
  // occupancy (and chunk count) than the launch itself
  cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k.fn, k.threads, k.smem) != cudaSuccess) {
    cudaGetLastError();
    occ = 1;
  }
  if (occ < 1) occ = 1;
  const int64_t resident = (int64_t)num_sms() * occ;
  // L2 chunking: every CTA streams the column records of its chunk, and CTAs
  // are launched row-tile-fastest, so all resident CTAs walk the same chunk.
  // Keeping a chunk's records within an L2 budget turns the re-reads of
  // 8000+ row tiles into L2 hits instead of DRAM misses (B' for N = 2^20,
  // K = 16 is 235 MB against a 126 MB L2).
  const int64_t budget = (int64_t)env_int("CNTGW_L2_CHUNK_MB", k.l2_chunk_mb) << 20;
  int64_t min_c = 1;
  if (budget > 0 && k.rec_bytes > 0) {
    const int64_t tile_bytes = (int64_t)k.rec_bytes * kColTile;
    const int64_t tiles_fit = budget / tile_bytes > 0 ? budget / tile_bytes : 1;
    min_c = (tiles + tiles_fit - 1) / tiles_fit;
  }
  if (k.f64s_tile > 0) {  // the F64S kernel lists at most 4096 stages per chunk
    const int64_t cap = (tiles * kColTile + 4096LL * k.f64s_tile - 1) / (4096LL * k.f64s_tile);
    if (cap > min_c) min_c = cap;
  }
  int best_c = (int)min_c;
  double best_eff = -1.0;
  const int64_t max_c = tiles < 64 + min_c ? tiles : 64 + min_c;
  for (int64_t c = min_c; c <= max_c; ++c) {
    const int64_t cpc = (tiles + c - 1) / c;  // tiles per chunk
    if ((tiles + cpc - 1) / cpc != c) continue;
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

size_t plan_workspace(const Plan& p, int64_t n) {
  return p.nchunks > 1 ? 2 * sizeof(double) * (size_t)p.nchunks * (size_t)n : 0;
}

// ---- column record packing --------------------------------------------------
template <typename T>
__global__ void prep_cols_kernel(const cntgw_sweep_state* st, int kd, int sq_flag, int stride,
                                 const T* feat, int64_t ld, const T* sq, const double* pot,
                                 const double* log2w, int64_t m, int64_t mpad, T* rec,
                                 const int64_t* order = nullptr, int within_loop = 0) {
  const int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (jj >= mpad) return;
  T* r = rec + jj * stride;
  const int64_t j = jj < m && order ? order[jj] : jj;  // source column (CNTGW_F64S: gathered)
  const bool f64 = sizeof(T) == 8;
  const double lam = f64 ? st->lam_d : (double)st->lam;
  const double sl = f64 ? st->sqrt_lam_d : (double)st->sqrt_lam;
  // within a loop (same features, same lam: no annealing) only the potential moves:
  // rewrite the bias column alone (cntgw_update_cols_f64s)
  if (within_loop && st->sweep > 1 && !(st->anneal_from > 0.0)) {
    if (jj < m) {
      double beta = lam * (pot ? pot[j] : 0.0) + log2w[j];
      if (sq_flag && f64) beta -= lam * (double)sq[j] * (double)sq[j];
      r[kd + sq_flag] = (T)(-beta);
    }
    return;
  }
  if (jj < m) {
    const T two_lam = (T)(2.0 * lam);
    for (int k = 0; k < kd; ++k) r[k] = -two_lam * feat[j * ld + k];
    double beta = lam * (pot ? pot[j] : 0.0) + log2w[j];
    if (sq_flag) {
      if (f64) {  // expanded square: -2 lam s_j multiplies the raw row s_i
        const double sj = (double)sq[j];
        r[kd] = (T)(-2.0 * lam * sj);
        beta -= lam * sj * sj;
      } else {  // difference form: sqrt(lam) s_j, squared against sqrt(lam) s_i
        r[kd] = (T)(-sl) * sq[j];
      }
    }
    r[kd + sq_flag] = (T)(-beta);
  } else {
    for (int k = 0; k < kd + sq_flag; ++k) r[k] = (T)0;
    r[kd + sq_flag] = f64 ? (T)kPadQ : (T)CUDART_INF_F;  // exactly zero weight
  }
  for (int k = kd + sq_flag + 1; k < stride; ++k) r[k] = (T)0;
}

// ---- dense cost half-update ---------------------------------------------------
__global__ void softmin_dense_kernel(const cntgw_sweep_state* st, int skip, const double* cost,
                                     int64_t ld, const double* pot, const double* log2w,
                                     const double* row_add, int64_t n, int64_t m, double* out) {
  if (skip_now(st, skip)) return;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const double lam = st->lam_d;
  double mx = -CUDART_INF;
  double sm = 0.0;
  const double* ci = cost + i * ld;
  for (int64_t j = lane; j < m; j += 32) {
    const double t = lam * (pot[j] - ci[j]) + log2w[j];
    if (t > mx) {
      sm = sm * exp2(mx - t) + 1.0;
      mx = t;
    } else {
      sm += exp2(t - mx);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double om = __shfl_xor_sync(0xffffffffu, mx, o);
    const double os = __shfl_xor_sync(0xffffffffu, sm, o);
    const double nm = fmax(mx, om);
    sm = (sm > 0.0 ? sm * exp2(mx - nm) : 0.0) + (os > 0.0 ? os * exp2(om - nm) : 0.0);
    mx = nm;
  }
  if (lane == 0) out[i] = (row_add ? row_add[i] : 0.0) - (mx + log2(sm)) / lam;
}

// ---- locality order (CNTGW_F32C) ---------------------------------------------
// Bounding box of the first d3 <= 3 coordinates (one block; O(n d3) loads).
__global__ void __launch_bounds__(1024) bbox_kernel(const double* x, int64_t n, int d3, int64_t ld,
                                                    double* bb) {
  __shared__ double lo_s[3][32], hi_s[3][32];
  double lo[3] = {CUDART_INF, CUDART_INF, CUDART_INF}, hi[3] = {-CUDART_INF, -CUDART_INF, -CUDART_INF};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    for (int k = 0; k < d3; ++k) {
      const double v = x[i * ld + k];
      lo[k] = fmin(lo[k], v);
      hi[k] = fmax(hi[k], v);
    }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int k = 0; k < 3; ++k) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[k] = fmin(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmax(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
    if (l == 0) {
      lo_s[k][w] = lo[k];
      hi_s[k][w] = hi[k];
    }
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    const int k = threadIdx.x;
    double a = CUDART_INF, b = -CUDART_INF;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      a = fmin(a, lo_s[k][q]);
      b = fmax(b, hi_s[k][q]);
    }
    bb[k] = a;
    bb[3 + k] = b;
  }
}

// 63-bit Morton (Z-order) code: 63/d3 bits per coordinate, bits interleaved.
__global__ void morton_kernel(const double* x, int64_t n, int d3, int64_t ld, const double* bb,
                              int64_t* codes) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int bits = 63 / d3;
  const double top = (double)((1ULL << bits) - 1);
  uint64_t q[3] = {0, 0, 0};
  for (int k = 0; k < d3; ++k) {
    const double span = bb[3 + k] - bb[k];
    const double u = span > 0.0 ? (x[i * ld + k] - bb[k]) / span : 0.0;
    q[k] = (uint64_t)fmin(fmax(u * top, 0.0), top);
  }
  uint64_t c = 0;
  for (int b = bits - 1; b >= 0; --b)
    for (int k = 0; k < d3; ++k) c = (c << 1) | ((q[k] >> b) & 1ULL);
  codes[i] = (int64_t)c;
}

}  // namespace

// ================================================================================
// Block-sparse plan of the centred kernel (ctr_plan_kernel) in `plan_ws`
// (ctr_plan_bytes): the reuse check (ctr_plan_check_kernel, keyed on the
// operator and lam), then the planning pass unless the previous plan holds.
// Returns the needed-tile votes.
static const uint32_t* ctr_build_plan(const KernelPick& k, const SoftminArgs& a, void* plan_ws, cudaStream_t s) {
  const int64_t n = a.n, m = a.m;
  const int64_t ctas = (ctr_groups(n) + k.ctr_r - 1) / k.ctr_r, tl = (m + kColTile - 1) / kColTile;
  float* rho = static_cast<float*>(plan_ws);
  uint32_t* need = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(rho) +
                                               align256(sizeof(float) * ctas * k.ctr_r * tl));
  double* c_plan = reinterpret_cast<double*>(reinterpret_cast<char*>(need) +
                                             align256(sizeof(uint32_t) * ctas * tl));
  CtrPlanKey* key =
      reinterpret_cast<CtrPlanKey*>(reinterpret_cast<char*>(c_plan) + align256(sizeof(double) * tl * kColTile));
  const char* e = getenv("CNTGW_CTR_SKIP_T");
  const double T = e ? atof(e) : 64.0;
  // plans are reused across sweeps while the column records moved by at
  // most `budget` log2 units (CNTGW_CTR_REUSE=0: replan every half-update)
  const double budget = 8.0;
  const bool reuse = env_int("CNTGW_CTR_REUSE", 1) != 0;
  const int64_t mp = tl * kColTile;
  const CtrCols cv = ctr_cols_view(a.col_rec, mp, k.ctr_kx);
  const int* rp = nullptr;
  if (reuse) {
    if (k.ctr_kx == 4)
      ctr_plan_check_kernel<4><<<1, 1024, 0, s>>>(a.st, cv.rec64, mp, c_plan, key, a.row_feat, a.col_rec, n, m,
                                                  budget);
    else
      ctr_plan_check_kernel<8><<<1, 1024, 0, s>>>(a.st, cv.rec64, mp, c_plan, key, a.row_feat, a.col_rec, n, m,
                                                  budget);
    rp = &key->replan;
  }
  const double Tp = reuse ? T + 2.0 * budget : T;
  // one planning block per streaming CTA (S = 1: planning 4 CTAs per block
  // to share the column reads measured 2.6x slower, 43 vs 17 ms at 2^20)
  if (k.ctr_kx == 4 && k.ctr_r == 8)
    ctr_plan_kernel<4, 8, 1><<<(unsigned)ctas, 128, 0, s>>>(a, rho, need, Tp, rp);
  else if (k.ctr_kx == 4 && k.ctr_r == 2)
    ctr_plan_kernel<4, 2, 1><<<(unsigned)ctas, 128, 0, s>>>(a, rho, need, Tp, rp);
  else if (k.ctr_kx == 4)
    ctr_plan_kernel<4, 4, 1><<<(unsigned)ctas, 128, 0, s>>>(a, rho, need, Tp, rp);
  else
    ctr_plan_kernel<8, 4, 1><<<(unsigned)ctas, 128, 0, s>>>(a, rho, need, Tp, rp);
  return need;
}

extern "C" {

int cntgw_abi_version(void) { return CNTGW_ABI_VERSION; }
const char* cntgw_last_error(void) { return g_last_error.c_str(); }
int cntgw_sweep_state_size(void) { return (int)sizeof(cntgw_sweep_state); }

int cntgw_col_stride(int prec, int kd, int sq) {
  if (!kd_supported(kd)) return fail(CNTGW_EINVAL, "unsupported feature width kd=%d", kd);
  const int raw = kd + (sq ? 1 : 0) + 1;
  if (prec == CNTGW_F32) return (raw + 3) / 4 * 4;
  if (prec == CNTGW_F64 || prec == CNTGW_F64S) {
    const int vec = (raw + 1) / 2 * 2, k4 = (kd + (sq ? 1 : 0) + 3) / 4 * 4;
    return k4 > vec ? k4 : vec;
  }
  if (prec == CNTGW_F32C) {
    const int kx = kd + (sq ? 1 : 0);
    if (kx > 8) return fail(CNTGW_EINVAL, "centred fp32 path supports kd + sq <= 8 (kd=%d sq=%d)", kd, sq);
    return kx <= 4 ? 4 : 8;  // fp32 dZ floats per column (see cntgw_ctr_cols_bytes for the block)
  }
  if (prec == CNTGW_TF32X3) {
    if (sq || (kd != 8 && kd != 16))
      return fail(CNTGW_EINVAL, "tensor-core path supports kd in {8,16} without sq (kd=%d sq=%d)", kd, sq);
    return (3 * kd + 2 + 7) / 8 * 8;  // K' floats per column, in 256-column tiles
  }
  return fail(CNTGW_EINVAL, "unknown precision %d", prec);
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
  if (!st) return fail(CNTGW_EINVAL, "null sweep state");
  sweep_begin_kernel<<<1, 1, 0, as_stream(stream)>>>(st);
  return check_launch("sweep_begin");
}

int cntgw_gap_blocks(int64_t n) { return gap_blocks(n); }

int cntgw_sweep_gap(cntgw_sweep_state* st, const double* w, const double* pot, const double* tent,
                    int64_t n, double* partials, void* stream) {
  if (!st || !w || !pot || !tent || !partials || n < 1)
    return fail(CNTGW_EINVAL, "sweep_gap: bad arguments");
  sweep_gap_kernel<<<gap_blocks(n), kGapThreads, 0, as_stream(stream)>>>(st, w, pot, tent, n, partials);
  return check_launch("sweep_gap");
}

int cntgw_sweep_finish(cntgw_sweep_state* st, const double* partials_r, int64_t n,
                       const double* partials_c, int64_t m, void* stream) {
  if (!st || !partials_r) return fail(CNTGW_EINVAL, "sweep_finish: bad arguments");
  sweep_finish_kernel<<<1, 1, 0, as_stream(stream)>>>(st, partials_r, gap_blocks(n), partials_c,
                                                       partials_c ? gap_blocks(m) : 0);
  return check_launch("sweep_finish");
}

int cntgw_sweep_apply(const cntgw_sweep_state* st, double* pot, const double* tent, int64_t n,
                      int average, void* stream) {
  if (!st || !pot || !tent || n < 1) return fail(CNTGW_EINVAL, "sweep_apply: bad arguments");
  const int th = 256;
  int64_t b = (n + th - 1) / th;
  if (b > 4 * num_sms()) b = 4 * num_sms();
  sweep_apply_kernel<<<(unsigned)b, th, 0, as_stream(stream)>>>(st, pot, tent, n, average);
  return check_launch("sweep_apply");
}

int cntgw_prep_cols(const cntgw_sweep_state* st, int prec, int kd, int sq_flag, const void* feat,
                    int64_t ld, const void* sq, const double* pot, const double* log2w, int64_t m,
                    void* rec, void* stream) {
  if (!st || !feat || !log2w || !rec || m < 1) return fail(CNTGW_EINVAL, "prep_cols: bad arguments");
  if (sq_flag && !sq) return fail(CNTGW_EINVAL, "prep_cols: sq_flag set without sq values");
  if (prec == CNTGW_F32C) return fail(CNTGW_EINVAL, "prep_cols: CNTGW_F32C columns are packed by cntgw_prep_cols_ctr");
  const int stride = cntgw_col_stride(prec, kd, sq_flag);
  if (stride < 0) return stride;
  const int64_t mpad = cntgw_cols_padded(m);
  const int th = 256;
  const unsigned blocks = (unsigned)((mpad + th - 1) / th);
  const int sqf = sq_flag ? 1 : 0;
  if (prec == CNTGW_TF32X3) {
    const float* f = static_cast<const float*>(feat);
    cudaStream_t s = as_stream(stream);
    if (tc_f16()) {  // absmax of the features (the word after the records), then the fp16 pack
      const size_t rec_bytes = (size_t)mpad * (kd == 8 ? TcLayoutH<8>::kRecBytes : TcLayoutH<16>::kRecBytes);
      uint32_t* absmax = reinterpret_cast<uint32_t*>(static_cast<char*>(rec) + rec_bytes);
      cudaMemsetAsync(absmax, 0, sizeof(uint32_t), s);
      tc_absmax_kernel<<<(unsigned)std::min<int64_t>((m * kd + 1023) / 1024, 4 * num_sms()), 256, 0, s>>>(
          f, ld, kd, m, absmax);
      if (kd == 8)
        prep_cols_tch_kernel<8><<<blocks, th, 0, s>>>(st, f, ld, pot, log2w, m, mpad, static_cast<__half*>(rec),
                                                      absmax);
      else
        prep_cols_tch_kernel<16><<<blocks, th, 0, s>>>(st, f, ld, pot, log2w, m, mpad, static_cast<__half*>(rec),
                                                       absmax);
    } else if (kd == 8)
      prep_cols_tc_kernel<8><<<blocks, th, 0, s>>>(st, f, ld, pot, log2w, m, mpad, static_cast<float*>(rec));
    else
      prep_cols_tc_kernel<16><<<blocks, th, 0, s>>>(st, f, ld, pot, log2w, m, mpad, static_cast<float*>(rec));
    return check_launch("prep_cols_tc");
  }
  if (prec == CNTGW_F32)
    prep_cols_kernel<float><<<blocks, th, 0, as_stream(stream)>>>(
        st, kd, sqf, stride, static_cast<const float*>(feat), ld, static_cast<const float*>(sq), pot,
        log2w, m, mpad, static_cast<float*>(rec));
  else
    prep_cols_kernel<double><<<blocks, th, 0, as_stream(stream)>>>(
        st, kd, sqf, stride, static_cast<const double*>(feat), ld, static_cast<const double*>(sq),
        pot, log2w, m, mpad, static_cast<double*>(rec));
  return check_launch("prep_cols");
}

int cntgw_locality_codes(const double* x, int64_t n, int d, int64_t ld, double* bbox, int64_t* codes,
                         void* stream) {
  if (!x || !bbox || !codes || n < 1 || d < 1 || ld < d) return fail(CNTGW_EINVAL, "locality_codes: bad arguments");
  const int d3 = d < 3 ? d : 3;
  cudaStream_t s = as_stream(stream);
  bbox_kernel<<<1, 1024, 0, s>>>(x, n, d3, ld, bbox);
  morton_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, n, d3, ld, bbox, codes);
  return check_launch("locality_codes");
}

static int ctr_kx(int kd, int sq_flag) {
  if (!kd_supported(kd)) return -1;
  const int kx = kd + (sq_flag ? 1 : 0);
  return kx <= 4 ? 4 : (kx <= 8 ? 8 : -1);
}

size_t cntgw_ctr_rows_bytes(int64_t n, int kd, int sq_flag) {
  const int kx = ctr_kx(kd, sq_flag);
  return (kx < 0 || n < 1) ? 0 : ctr_rows_bytes(n, kx);
}

size_t cntgw_ctr_cols_bytes(int64_t m, int kd, int sq_flag) {
  const int kx = ctr_kx(kd, sq_flag);
  return (kx < 0 || m < 1) ? 0 : ctr_cols_bytes_all(cntgw_cols_padded(m), kx);
}

int cntgw_prep_rows_ctr(int kd, int sq_flag, const double* feat, int64_t ld, const double* sq,
                        const int64_t* order, int64_t n, void* rows, void* stream) {
  if (!feat || !rows || n < 1 || ld < kd) return fail(CNTGW_EINVAL, "prep_rows_ctr: bad arguments");
  if (sq_flag && !sq) return fail(CNTGW_EINVAL, "prep_rows_ctr: sq_flag set without sq values");
  const int kx = ctr_kx(kd, sq_flag);
  if (kx < 0) return fail(CNTGW_EINVAL, "prep_rows_ctr: kd + sq = %d + %d > 8", kd, sq_flag);
  const unsigned g = (unsigned)ctr_groups(n);
  cudaStream_t s = as_stream(stream);
  if (kx == 4)
    prep_rows_ctr_kernel<4><<<g, kCtrRowGroup, 0, s>>>(kd, sq_flag ? 1 : 0, feat, ld, sq, order, n, rows);
  else
    prep_rows_ctr_kernel<8><<<g, kCtrRowGroup, 0, s>>>(kd, sq_flag ? 1 : 0, feat, ld, sq, order, n, rows);
  return check_launch("prep_rows_ctr");
}

int cntgw_prep_cols_ctr(const cntgw_sweep_state* st, int kd, int sq_flag, const double* feat, int64_t ld,
                        const double* sq, const double* pot, const double* log2w, const int64_t* order,
                        int64_t m, void* cols, void* stream) {
  if (!st || !feat || !log2w || !cols || m < 1 || ld < kd)
    return fail(CNTGW_EINVAL, "prep_cols_ctr: bad arguments");
  if (sq_flag && !sq) return fail(CNTGW_EINVAL, "prep_cols_ctr: sq_flag set without sq values");
  const int kx = ctr_kx(kd, sq_flag);
  if (kx < 0) return fail(CNTGW_EINVAL, "prep_cols_ctr: kd + sq = %d + %d > 8", kd, sq_flag);
  const int64_t mpad = cntgw_cols_padded(m);
  const unsigned tiles = (unsigned)(mpad / kColTile);
  cudaStream_t s = as_stream(stream);
  const int sqf = sq_flag ? 1 : 0;
  if (kx == 4) {
    prep_cols_ctr_kernel<4><<<tiles, kColTile, 0, s>>>(st, kd, sqf, feat, ld, sq, pot, log2w, order, m, mpad, cols);
    const CtrCols cv = ctr_cols_view(cols, mpad, 4);
    prep_cols_ctc_kernel<<<(unsigned)(mpad / 256), 256, 0, s>>>(
        cv.rec32, mpad, reinterpret_cast<float*>(static_cast<char*>(cols) + ctr_cols_bytes(mpad, 4)));
  } else
    prep_cols_ctr_kernel<8><<<tiles, kColTile, 0, s>>>(st, kd, sqf, feat, ld, sq, pot, log2w, order, m, mpad, cols);
  return check_launch("prep_cols_ctr");
}

size_t cntgw_softmin_workspace(int prec, int64_t n, int64_t m, int kd, int sq_flag) {
  KernelPick k;
  if (n < 1 || m < 1 || !lookup(prec, kd, sq_flag, &k)) return 0;
  return align256(plan_workspace(plan_softmin(n, m, k), n)) + ctr_plan_bytes(k, n, m) + f64s_plan_bytes(k, n, m);
}

int cntgw_softmin(const cntgw_sweep_state* st, int skip_if_done, int prec, int kd, int sq_flag,
                  const void* row_feat, int64_t ld_row, const void* row_sq, const double* row_add,
                  const void* col_rec, int64_t n, int64_t m, double* out, double* out_max,
                  double* out_sum, void* workspace, size_t workspace_bytes, void* stream) {
  if (!st || !row_feat || !col_rec || n < 1 || m < 1)
    return fail(CNTGW_EINVAL, "softmin: bad arguments (n=%lld m=%lld)", (long long)n, (long long)m);
  if (sq_flag && !row_sq) return fail(CNTGW_EINVAL, "softmin: sq_flag without row_sq");
  if (!out && !(out_max && out_sum)) return fail(CNTGW_EINVAL, "softmin: no output");
  KernelPick k;
  if (!lookup(prec, kd, sq_flag, &k))
    return fail(CNTGW_EINVAL, "softmin: unsupported precision %d / feature width kd=%d", prec, kd);
  cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem);
  const Plan p = plan_softmin(n, m, k);
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
  a.chunk_cols = p.chunk_cols;
  a.nchunks = p.nchunks;
  a.out = out;
  a.out_max = out_max;
  a.out_sum = out_sum;
  {  // fp32 pair-term bound per (row group, column tile) of CNTGW_F32C, log2 units
    const char* e = getenv("CNTGW_CTR_TILE_LIMIT");
    a.ctr_limit = e ? atof(e) : 65536.0;
  }
  const size_t part_bytes = align256(plan_workspace(p, n)),
               plan_bytes = ctr_plan_bytes(k, n, m) + f64s_plan_bytes(k, n, m);
  if (part_bytes + plan_bytes > 0 && (workspace == nullptr || workspace_bytes < part_bytes + plan_bytes))
    return fail(CNTGW_ENOSPACE, "softmin workspace %zu < %zu bytes", workspace_bytes, part_bytes + plan_bytes);
  if (p.nchunks > 1) {
    a.part_max = static_cast<double*>(workspace);
    a.part_sum = a.part_max + (size_t)p.nchunks * n;
  }
  cudaStream_t s = as_stream(stream);
  if (k.ctr_kx > 0 && ctr_plan_bytes(k, n, m) > 0)
    a.ctr_need = ctr_build_plan(k, a, static_cast<char*>(workspace) + part_bytes, s);
  F64sArgs fs{};
  F64sPlanLayout fl{};
  if (k.f64s_tile > 0) {  // CNTGW_F64S: re-vote the plan, then the sweep (measure, or sparse)
    fl = f64s_layout(k, n, m);
    if (p.chunk_cols / k.f64s_tile > 4096)
      return fail(CNTGW_EINVAL, "softmin f64s: %lld stages per column chunk (max 4096)",
                  (long long)(p.chunk_cols / k.f64s_tile));
    const F64sPlan pl = f64s_plan(static_cast<char*>(workspace) + part_bytes, fl);
    fs.tmin = pl.tmin;
    fs.need = pl.need;
    fs.row_order = static_cast<const int64_t*>(row_feat);  // the rows block starts with the order
    fs.replan = pl.flag;
    fs.stages = fl.stages;
    const double* rec = static_cast<const double*>(col_rec);
    if (const int rc = f64s_revote(k, fl, pl, st, rec, kd, sq_flag ? 1 : 0, row_feat, col_rec, n, m, s, 1,
                                   skip_if_done))
      return rc;
    if (env_int("CNTGW_CTR_REUSE", 1) == 0) f64s_begin_kernel<<<1, 1, 0, s>>>(nullptr, 0, pl.key, row_feat, col_rec,
                                                                                n, m, pl.flag, pl.counter, pl.full, pl.sched);
    // (before the probe, which clears *full once its plan stands)
    if (sq_flag && env_int("CNTGW_F64S_DOTZERO", 1))  // does the dot term vanish (Gamma = 0)? (first sweeps)
      f64s_dotzero_kernel<<<2 * num_sms(), 256, 0, s>>>(pl.full, row_feat, n, kd, rec,
                                                        cntgw_col_stride(CNTGW_F64S, kd, 1), m, pl.dotzero);
    else
      cudaMemsetAsync(pl.dotzero, 0xff, 2 * sizeof(int), s);  // (both sides "nonzero")
    if (f64s_probe_enabled(k))
      if (const int rc = f64s_probe(k, fl, pl, st, skip_if_done, rec, kd, sq_flag ? 1 : 0, row_feat, col_rec, n, m, s))
        return rc;
    fs.full = pl.full;
    fs.dotzero = pl.dotzero;
    void* args2[] = {&a, &fs};
    cudaError_t e2 = cudaLaunchKernel(k.fn, dim3(p.row_tiles, p.nchunks), dim3(k.threads), args2, k.smem, s);
    if (e2 != cudaSuccess) {
      cudaGetLastError();
      return fail(CNTGW_ECUDA, "softmin f64s launch: %s", cudaGetErrorString(e2));
    }
    const int64_t mpad = (m + kColTile - 1) / kColTile * kColTile;
    f64s_reduce_kernel<<<(unsigned)fl.row_tiles, 256, f64s_reduce_smem(k, fl.stages), s>>>(
        pl.flag, pl.full, pl.tmin, pl.need, pl.range, n, fl.stages, k.cta_rows, pl.gmin, pl.tstar, pl.rowmin,
        0.f, nullptr);  // (the fp64 kernel measures exact stage minima: no slack)
    f64s_commit_kernel<<<1, 1024, 0, s>>>(pl.flag, st, rec, cntgw_col_stride(CNTGW_F64S, kd, sq_flag),
                                          kd + (sq_flag ? 1 : 0), mpad, pl.c_plan, pl.key, row_feat, col_rec, n, m,
                                          pl.next_measure, pl.counter, pl.sched);
    if (const int rc = check_launch("f64s_commit")) return rc;
    if (p.nchunks > 1) {
      const int th = 256;
      lse_combine_kernel<<<(unsigned)((n + th - 1) / th), th, 0, s>>>(
          st, skip_if_done, prec, a.part_max, a.part_sum, p.nchunks, n, row_add, out, out_max, out_sum);
      return check_launch("lse_combine");
    }
    return CNTGW_OK;
  }
  void* args[] = {&a};
  const cudaError_t e =
      cudaLaunchKernel(k.fn, dim3(p.row_tiles, p.nchunks), dim3(k.threads), args, k.smem, s);
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear, so the failure is not reported again by a later call
    return fail(CNTGW_ECUDA, "softmin launch: %s", cudaGetErrorString(e));
  }
  if (p.nchunks > 1) {
    const int th = 256;
    lse_combine_kernel<<<(unsigned)((n + th - 1) / th), th, 0, s>>>(
        st, skip_if_done, prec, a.part_max, a.part_sum, p.nchunks, n, row_add, out, out_max, out_sum);
    return check_launch("lse_combine");
  }
  return CNTGW_OK;
}

int cntgw_lse_finalize(const cntgw_sweep_state* st, int skip_if_done, int prec, const double* mx,
                       const double* sm, const double* row_add, int64_t n, double* out,
                       void* stream) {
  if (!st || !mx || !sm || !out || n < 1) return fail(CNTGW_EINVAL, "lse_finalize: bad arguments");
  const int th = 256;
  lse_combine_kernel<<<(unsigned)((n + th - 1) / th), th, 0, as_stream(stream)>>>(
      st, skip_if_done, prec, mx, sm, 1, n, row_add, out, nullptr, nullptr);
  return check_launch("lse_finalize");
}

int cntgw_softmin_dense(const cntgw_sweep_state* st, int skip_if_done, const double* cost,
                        int64_t ld, const double* pot, const double* log2w, const double* row_add,
                        int64_t n, int64_t m, double* out, void* stream) {
  if (!st || !cost || !pot || !log2w || !out || n < 1 || m < 1)
    return fail(CNTGW_EINVAL, "softmin_dense: bad arguments");
  const int warps = 8;
  softmin_dense_kernel<<<(unsigned)((n + warps - 1) / warps), warps * 32, 0, as_stream(stream)>>>(
      st, skip_if_done, cost, ld, pot, log2w, row_add, n, m, out);
  return check_launch("softmin_dense");
}

/* ---- CNTGW_F64S plan diagnostics: out[0] needed (row group, stage) pairs of
 * the mask the last sweep used, out[1] all pairs, out[2] bit 0: that sweep
 * measured with the fp64 kernel, bit 1: its plan came from the fp32 probe;
 * out: 3 int64 on the device (out[0] summed) */
int cntgw_f64s_plan_density(int kd, int sq_flag, int64_t n, int64_t m, const void* workspace, int64_t* out,
                            void* stream) {
  KernelPick k;
  if (!workspace || !out || n < 1 || m < 1 || !lookup(CNTGW_F64S, kd, sq_flag, &k))
    return fail(CNTGW_EINVAL, "f64s_plan_density: bad arguments");
  const F64sPlanLayout fl = f64s_layout(k, n, m);
  const size_t part_bytes = align256(plan_workspace(plan_softmin(n, m, k), n));
  const F64sPlan pl = f64s_plan(static_cast<char*>(const_cast<void*>(workspace)) + part_bytes, fl);
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(out, 0, sizeof(int64_t), s);
  f64s_density_kernel<<<148, 256, 0, s>>>(pl.need, fl.row_tiles * (int64_t)fl.stages, pl.flag,
                                          f64s_probe_enabled(k) ? pl.probe_ok : nullptr, out);
  return check_launch("f64s_density");
}

/* Where the measured plan's stage minima live in an F64S workspace (host-side query). */
int cntgw_f64s_plan_layout(int kd, int sq_flag, int64_t n, int64_t m, int64_t* out) {
  KernelPick k;
  if (!out || n < 1 || m < 1 || !lookup(CNTGW_F64S, kd, sq_flag, &k))
    return fail(CNTGW_EINVAL, "f64s_plan_layout: bad arguments");
  const F64sPlanLayout fl = f64s_layout(k, n, m);
  out[0] = (int64_t)align256(plan_workspace(plan_softmin(n, m, k), n));  // tmin: [n][stages] fp32
  out[1] = fl.stages;
  out[2] = k.f64s_tile;
  return CNTGW_OK;
}

/* ---- CNTGW_F64S: the point order of the next loop from the device Gamma ---- */
int cntgw_select_order(const double* gamma, int de, const int64_t* order_if_zero, const int64_t* order_otherwise,
                       int64_t n, int64_t* out, void* stream) {
  if (!gamma || de < 1 || !order_if_zero || !order_otherwise || !out || n < 1)
    return fail(CNTGW_EINVAL, "select_order: bad arguments");
  const int64_t blocks = (n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184;
  select_order_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(gamma, de, order_if_zero, order_otherwise,
                                                                       n, out);
  return check_launch("select_order");
}

/* ---- CNTGW_F64S rows block and ordered column records ---- */
size_t cntgw_f64s_rows_bytes(int64_t n, int kd) { return n < 1 ? 0 : f64s_rows_bytes(n, kd); }

int cntgw_prep_rows_f64s(int kd, int sq_flag, const double* feat, int64_t ld, const double* sq,
                         const int64_t* order, int64_t n, void* rows, void* stream) {
  if (!feat || !rows || n < 1 || !kd_supported(kd) || (sq_flag && !sq))
    return fail(CNTGW_EINVAL, "prep_rows_f64s: bad arguments");
  f64s_prep_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(kd, sq_flag ? 1 : 0, feat,
                                                                                    ld, sq, order, n, rows);
  return check_launch("prep_rows_f64s");
}

int cntgw_prep_cols_f64s(const cntgw_sweep_state* st, int kd, int sq_flag, const double* feat, int64_t ld,
                         const double* sq, const double* pot, const double* log2w, const int64_t* order,
                         int64_t m, void* rec, void* stream) {
  if (!st || !feat || !log2w || !rec || m < 1 || (sq_flag && !sq))
    return fail(CNTGW_EINVAL, "prep_cols_f64s: bad arguments");
  const int stride = cntgw_col_stride(CNTGW_F64S, kd, sq_flag);
  if (stride < 0) return stride;
  const int64_t mpad = cntgw_cols_padded(m);
  prep_cols_kernel<double><<<(unsigned)((mpad + 255) / 256), 256, 0, as_stream(stream)>>>(
      st, kd, sq_flag ? 1 : 0, stride, feat, ld, sq, pot, log2w, m, mpad, static_cast<double*>(rec), order);
  return check_launch("prep_cols_f64s");
}

int cntgw_update_cols_f64s(const cntgw_sweep_state* st, int kd, int sq_flag, const double* feat, int64_t ld,
                           const double* sq, const double* pot, const double* log2w, const int64_t* order,
                           int64_t m, void* rec, void* stream) {
  if (!st || !feat || !log2w || !rec || m < 1 || (sq_flag && !sq))
    return fail(CNTGW_EINVAL, "update_cols_f64s: bad arguments");
  const int stride = cntgw_col_stride(CNTGW_F64S, kd, sq_flag);
  if (stride < 0) return stride;
  const int64_t mpad = cntgw_cols_padded(m);
  prep_cols_kernel<double><<<(unsigned)((mpad + 255) / 256), 256, 0, as_stream(stream)>>>(
      st, kd, sq_flag ? 1 : 0, stride, feat, ld, sq, pot, log2w, m, mpad, static_cast<double*>(rec), order, 1);
  return check_launch("update_cols_f64s");
}

/* ---- K4 on the centred path's block-sparse plan (reduce_ctr.cuh) ---- */
size_t cntgw_plan_reduce_ctr_workspace(int64_t m, int e) {
  const int ep = e <= 4 ? 4 : (e <= 8 ? 8 : (e <= 16 ? 16 : (e <= 32 ? 32 : (e <= 64 ? 64 : -1))));
  if (ep < 0 || e < 1) return 0;
  return (size_t)cntgw_cols_padded(m) * (size_t)((ep + 1 + 1) / 2 * 2) * sizeof(double);
}

int cntgw_plan_reduce_ctr(const cntgw_sweep_state* st, int kd, int sq_flag, int e, const void* ctr_rows,
                          const void* ctr_cols, const int64_t* col_order, const double* row_feat,
                          int64_t ld_row, const double* row_sq, const double* f_tilde, const double* log2a,
                          const double* col_acc, int64_t ld_acc, const double* col_s, int64_t n, int64_t m,
                          double* row_mass, double* pi_y, double* pi_s, int64_t* argmax, void* plan_ws,
                          size_t plan_ws_bytes, void* acc_ws, size_t acc_ws_bytes, void* stream) {
  if (!st || !ctr_rows || !ctr_cols || !row_feat || !f_tilde || !log2a || !col_acc || !col_s || !row_mass ||
      !pi_y || !pi_s || !argmax || n < 1 || m < 1 || e < 1 || (sq_flag && !row_sq))
    return fail(CNTGW_EINVAL, "plan_reduce_ctr: bad arguments");
  KernelPick k;
  if (!lookup(CNTGW_F32C, kd, sq_flag, &k))
    return fail(CNTGW_EINVAL, "plan_reduce_ctr: no centred kernel for kd=%d sq=%d", kd, sq_flag);
  // the opt-in tcgen05 centred kernel (CNTGW_CTR_TC=1) keeps the kx = 4 block
  // layout but has no plan: the pass then visits every tile
  const int kx = k.ctr_kx > 0 ? k.ctr_kx : 4;
  const int ep = e <= 4 ? 4 : (e <= 8 ? 8 : (e <= 16 ? 16 : (e <= 32 ? 32 : (e <= 64 ? 64 : -1))));
  if (ep < 0) return fail(CNTGW_EINVAL, "plan_reduce_ctr: unsupported e=%d", e);
  const size_t acc_need = cntgw_plan_reduce_ctr_workspace(m, e);
  if (!acc_ws || acc_ws_bytes < acc_need)
    return fail(CNTGW_ENOSPACE, "plan_reduce_ctr workspace %zu < %zu", acc_ws_bytes, acc_need);
  const size_t plan_bytes = ctr_plan_bytes(k, n, m);
  const size_t part_bytes = plan_bytes > 0 ? align256(plan_workspace(plan_softmin(n, m, k), n)) : 0;
  if (plan_bytes > 0 && (!plan_ws || plan_ws_bytes < part_bytes + plan_bytes))
    return fail(CNTGW_ENOSPACE, "plan_reduce_ctr: plan workspace %zu < %zu", plan_ws_bytes,
                part_bytes + plan_bytes);
  cudaStream_t s = as_stream(stream);
  SoftminArgs sa{};
  sa.st = st;
  sa.row_feat = ctr_rows;
  sa.col_rec = ctr_cols;
  sa.n = n;
  sa.m = m;
  const uint32_t* need =
      plan_bytes > 0 ? ctr_build_plan(k, sa, static_cast<char*>(plan_ws) + part_bytes, s) : nullptr;
  const int64_t mpad = cntgw_cols_padded(m);
  const int stride = (ep + 1 + 1) / 2 * 2;
  double* acc = static_cast<double*>(acc_ws);
  pack_acc_ordered_kernel<<<(unsigned)((mpad + 255) / 256), 256, 0, s>>>(col_acc, ld_acc, e, ep, stride, col_s,
                                                                          col_order, m, mpad, acc);
  int rc = check_launch("pack_acc_ordered");
  if (rc) return rc;
  PlanReduceCtrArgs a{};
  a.st = st;
  const CtrRows rv = ctr_rows_view(ctr_rows, n, kx);
  a.row_order = rv.order;
  a.col_order = col_order;
  a.row_feat = row_feat;
  a.ld_row = ld_row;
  a.kd = kd;
  a.sq = sq_flag ? 1 : 0;
  a.row_sq = row_sq;
  a.f_tilde = f_tilde;
  a.log2a = log2a;
  a.rec64 = ctr_cols_view(ctr_cols, mpad, kx).rec64;
  a.acc = acc;
  a.need = need;
  a.ctr_r = k.ctr_r > 0 ? k.ctr_r : 1;
  a.n = n;
  a.m = m;
  a.row_mass = row_mass;
  a.pi_y = pi_y;
  a.e_real = e;
  a.pi_s = pi_s;
  a.argmax = argmax;
  const unsigned blocks = (unsigned)ctr_groups(n);
#define PRC(KX_, E_)                                                                    \
  if (kx == KX_ && ep == E_) {                                                         \
    auto kern = plan_reduce_ctr_kernel<KX_, E_, 4>;                                    \
    const size_t smem = CtrReduceSmem<KX_ + 1, E_>::kBytes;                                \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    kern<<<blocks, 128, smem, s>>>(a);                                                 \
    return check_launch("plan_reduce_ctr_kernel");                                     \
  }
  PRC(4, 4) PRC(4, 8) PRC(4, 16) PRC(4, 32) PRC(4, 64)
  PRC(8, 4) PRC(8, 8) PRC(8, 16) PRC(8, 32) PRC(8, 64)
#undef PRC
  return fail(CNTGW_EINVAL, "plan_reduce_ctr: unsupported kx=%d e=%d", kx, e);
}

/* ---- K4 on the CNTGW_F64S measured plan ---- */
int cntgw_plan_reduce_f64s(const cntgw_sweep_state* st, int kd, int sq_flag, int e, const void* f64s_rows,
                           const double* col_rec, const int64_t* col_order, const double* row_feat,
                           int64_t ld_row, const double* row_sq, const double* f_tilde, const double* log2a,
                           const double* col_acc, int64_t ld_acc, const double* col_s, int64_t n, int64_t m,
                           double* row_mass, double* pi_y, double* pi_s, int64_t* argmax, void* plan_ws,
                           size_t plan_ws_bytes, void* acc_ws, size_t acc_ws_bytes, void* stream) {
  if (!st || !f64s_rows || !col_rec || !row_feat || !f_tilde || !log2a || !col_acc || !col_s || !row_mass ||
      !pi_y || !pi_s || !argmax || n < 1 || m < 1 || e < 1 || !sq_flag || !row_sq || !plan_ws)
    return fail(CNTGW_EINVAL, "plan_reduce_f64s: bad arguments");
  KernelPick k;
  if (!lookup(CNTGW_F64S, kd, 1, &k)) return fail(CNTGW_EINVAL, "plan_reduce_f64s: unsupported kd=%d", kd);
  const int ep = e <= 4 ? 4 : (e <= 8 ? 8 : (e <= 16 ? 16 : (e <= 32 ? 32 : (e <= 64 ? 64 : -1))));
  if (ep < 0) return fail(CNTGW_EINVAL, "plan_reduce_f64s: unsupported e=%d", e);
  const size_t acc_need = cntgw_plan_reduce_ctr_workspace(m, e);
  if (!acc_ws || acc_ws_bytes < acc_need)
    return fail(CNTGW_ENOSPACE, "plan_reduce_f64s workspace %zu < %zu", acc_ws_bytes, acc_need);
  const size_t part_bytes = align256(plan_workspace(plan_softmin(n, m, k), n));
  const F64sPlanLayout fl = f64s_layout(k, n, m);
  if (plan_ws_bytes < part_bytes + fl.total)
    return fail(CNTGW_ENOSPACE, "plan_reduce_f64s: plan workspace %zu < %zu", plan_ws_bytes, part_bytes + fl.total);
  cudaStream_t s = as_stream(stream);
  const F64sPlan pl = f64s_plan(static_cast<char*>(plan_ws) + part_bytes, fl);
  const int64_t mpad = cntgw_cols_padded(m);
  // re-vote for the final pair's records; a stale plan (*flag) walks every stage
  if (const int rc = f64s_revote(k, fl, pl, st, col_rec, kd, 1, f64s_rows, col_rec, n, m, s, 0, 0)) return rc;
  const uint8_t* need = pl.need;
  const int* stale = pl.flag;
  const int stride_acc = (ep + 1 + 1) / 2 * 2;
  double* acc = static_cast<double*>(acc_ws);
  pack_acc_ordered_kernel<<<(unsigned)((mpad + 255) / 256), 256, 0, s>>>(col_acc, ld_acc, e, ep, stride_acc, col_s,
                                                                          col_order, m, mpad, acc);
  if (const int rc = check_launch("pack_acc_ordered")) return rc;
  PlanReduceCtrArgs a{};
  a.st = st;
  a.row_order = static_cast<const int64_t*>(f64s_rows);  // the rows block starts with the order
  a.col_order = col_order;
  a.row_feat = row_feat;
  a.ld_row = ld_row;
  a.kd = kd;
  a.sq = 1;
  a.row_sq = row_sq;
  a.f_tilde = f_tilde;
  a.log2a = log2a;
  a.rec64 = col_rec;
  a.acc = acc;
  a.need = nullptr;
  a.ctr_r = 1;
  a.need8 = need;
  a.replan = stale;
  a.grows = k.cta_rows;
  a.n = n;
  a.m = m;
  a.row_mass = row_mass;
  a.pi_y = pi_y;
  a.e_real = e;
  a.pi_s = pi_s;
  a.argmax = argmax;
  const unsigned blocks = (unsigned)ctr_groups(n);
#define PRS(KD_, E_)                                                                                 \
  if (kd == KD_ && ep == E_) {                                                                       \
    constexpr int KX = KD_ + 1, STR = ColLayout<double, KD_, 1>::kStride;                           \
    constexpr int TD = f64s_stage_cols(KD_);                                                         \
    auto kern = plan_reduce_ctr_kernel<KX, E_, 4, STR, TD>;                                          \
    const size_t smem = CtrReduceSmem<STR, E_, TD>::kBytes;                                          \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);              \
    kern<<<blocks, 128, smem, s>>>(a);                                                               \
    return check_launch("plan_reduce_f64s_kernel");                                                  \
  }
  PRS(1, 4) PRS(2, 4) PRS(3, 4) PRS(4, 4) PRS(1, 8) PRS(2, 8) PRS(3, 8) PRS(4, 8) PRS(8, 8)
  PRS(1, 16) PRS(2, 16) PRS(3, 16) PRS(4, 16) PRS(8, 16) PRS(16, 16)
  PRS(1, 32) PRS(2, 32) PRS(3, 32) PRS(4, 32) PRS(8, 32) PRS(16, 32) PRS(32, 32)
  PRS(1, 64) PRS(2, 64) PRS(3, 64) PRS(4, 64) PRS(8, 64) PRS(16, 64) PRS(32, 64) PRS(64, 64)
#undef PRS
  return fail(CNTGW_EINVAL, "plan_reduce_f64s: unsupported kd=%d e=%d", kd, e);
}

}  // extern "C"
