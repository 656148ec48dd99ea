// Row-sharded multi-GPU exchange as C-ABI collectives on the
// caller's stream, so a sharded solve stays one CUDA graph.
//
// The row-sharded g-update (dist.py) leaves every rank with per-column
// partial log-sum-exp pairs (m_j, s_j) over its own rows; the full column
// softmin needs M_j = max_ranks m_j and S_j = sum_ranks s_j 2^(m_j - M_j).
// cntgw_comm_combine_lse does exactly that with two NCCL all-reduces and one
// rescale kernel, all enqueued on `stream`:
//     ncclAllReduce(m -> M, MAX)      (out of place: the local m is kept)
//     s_j <- s_j 2^(m_j - M_j)        (lse_rescale_kernel; an empty partial,
//                                      s_j = 0 or m_j = -inf, contributes 0)
//     ncclAllReduce(s, SUM)           (in place)
// NCCL is resolved at run time from the process (torch loads its bundled
// libnccl.so.2; dlopen returns the same instance), so the library has no
// link-time NCCL dependency and a CPU-only build container can build it.
// Every call is stream-ordered and graph-capturable (NCCL >= 2.9).
#include <dlfcn.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "common.cuh"

using namespace cntgw;

namespace cntgw {
int set_error(int code, const char* msg);
}

struct cntgw_comm {
  ncclComm_t comm;
  int world;
  int rank;
};

namespace {

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return cntgw::set_error(code, buf);
}

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*);
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*comm_destroy)(ncclComm_t);
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t);
  const char* (*error_string)(ncclResult_t);
  ncclResult_t (*get_version)(int*);
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the instance torch already mapped, else the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.get_version = reinterpret_cast<decltype(api.get_version)>(dlsym(h, "ncclGetVersion"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce &&
             api.error_string;
  });
  return api;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return CNTGW_OK;
  return fail(CNTGW_ECUDA, "%s: %s", what, nccl().error_string(r));
}

__global__ void lse_rescale_kernel(const double* __restrict__ m_local, const double* __restrict__ m_glob,
                                   double* __restrict__ s, int64_t n) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double sj = s[j], mj = m_local[j];
  // empty partial (no live row, or every term -inf): contributes nothing
  s[j] = (sj > 0.0 && mj > -CUDART_INF) ? sj * exp2(mj - m_glob[j]) : 0.0;
}

}  // namespace

extern "C" {

int cntgw_comm_id_bytes(void) { return NCCL_UNIQUE_ID_BYTES; }

int cntgw_comm_available(void) { return nccl().ok ? 1 : 0; }

int cntgw_comm_nccl_version(void) {
  int v = 0;
  if (nccl().ok && nccl().get_version) nccl().get_version(&v);
  return v;
}

int cntgw_comm_unique_id(void* id_out) {
  if (!id_out) return fail(CNTGW_EINVAL, "comm_unique_id: null buffer");
  if (!nccl().ok) return fail(CNTGW_ECUDA, "comm_unique_id: libnccl.so.2 not found");
  ncclUniqueId id;
  const int rc = nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  if (rc) return rc;
  memcpy(id_out, &id, sizeof(id));
  return CNTGW_OK;
}

int cntgw_comm_init(cntgw_comm** out, int world, int rank, const void* id) {
  if (!out || !id || world < 1 || rank < 0 || rank >= world)
    return fail(CNTGW_EINVAL, "comm_init: bad arguments (world=%d rank=%d)", world, rank);
  if (!nccl().ok) return fail(CNTGW_ECUDA, "comm_init: libnccl.so.2 not found");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  auto* c = new cntgw_comm{};
  c->world = world;
  c->rank = rank;
  const int rc = nccl_check(nccl().comm_init_rank(&c->comm, world, uid, rank), "ncclCommInitRank");
  if (rc) {
    delete c;
    return rc;
  }
  *out = c;
  return CNTGW_OK;
}

int cntgw_comm_destroy(cntgw_comm* c) {
  if (!c) return CNTGW_OK;
  const int rc = nccl_check(nccl().comm_destroy(c->comm), "ncclCommDestroy");
  delete c;
  return rc;
}

/* op: 0 = sum, 1 = max; fp64; send == recv for in place. */
int cntgw_comm_allreduce(cntgw_comm* c, const double* send, double* recv, int64_t count, int op,
                         void* stream) {
  if (!c || !send || !recv || count < 1 || op < 0 || op > 1)
    return fail(CNTGW_EINVAL, "comm_allreduce: bad arguments");
  return nccl_check(nccl().all_reduce(send, recv, (size_t)count, ncclFloat64, op ? ncclMax : ncclSum, c->comm,
                                      reinterpret_cast<cudaStream_t>(stream)),
                    "ncclAllReduce");
}

int cntgw_lse_rescale(const double* m_local, const double* m_glob, double* s, int64_t n, void* stream) {
  if (!m_local || !m_glob || !s || n < 1) return fail(CNTGW_EINVAL, "lse_rescale: bad arguments");
  lse_rescale_kernel<<<(unsigned)((n + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      m_local, m_glob, s, n);
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(CNTGW_ECUDA, "lse_rescale: %s", cudaGetErrorString(e));
  }
  return CNTGW_OK;
}

int cntgw_comm_combine_lse(cntgw_comm* c, const double* m_local, double* m_glob, double* s, int64_t n,
                           void* stream) {
  int rc = cntgw_comm_allreduce(c, m_local, m_glob, n, 1, stream);
  if (rc) return rc;
  rc = cntgw_lse_rescale(m_local, m_glob, s, n, stream);
  if (rc) return rc;
  return cntgw_comm_allreduce(c, s, s, n, 0, stream);
}

}  // extern "C"
