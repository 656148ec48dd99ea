// Device-resident outer loop: the CNT-GW outer-step control as a kernel and
// CUDA-graph conditional WHILE nodes (CUDA >= 12.4) so that an entire solve —
// every outer step and every (data-dependently terminated) Sinkhorn sweep —
// is one graph launch. Declarations: include/cntgw_b200.h.
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

int check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(CNTGW_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  }
  return CNTGW_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void outer_init_kernel(cntgw_outer_state* os, double constant, double eps_outer,
                                  double delta_outer, int max_outer) {
  os->constant = constant;
  os->eps_outer = eps_outer;
  os->delta_outer = delta_outer;
  os->prev_objective = 0.0;
  os->t0_ns = (double)globaltimer();
  os->max_outer = max_outer;
  os->step = 0;
  os->ups = 0;
  os->done = 0;
  os->converged = 0;
  os->error = 0;
  os->has_prev = 0;
}

// One outer step's bookkeeping (reference solvers.py:330-334 and the stop rule
// and divergence guard of solvers.py:579-612), from the fp64 reductions.
__global__ void outer_finish_kernel(cntgw_outer_state* os, const cntgw_sweep_state* st,
                                    const double* acc_rows, const double* acc_cols, double* gamma,
                                    double* gamma_prev, int de, double* trace) {
  __shared__ double red[3][32];
  if (os->done) return;
  const double* gnext = acc_rows + 16;
  double sq = 0.0, cross = 0.0, diff = 0.0;
  for (int k = threadIdx.x; k < de; k += blockDim.x) {
    const double a = gamma[k], b = gnext[k];
    sq += b * b;
    cross += a * b;
    diff += (b - a) * (b - a);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sq += __shfl_down_sync(0xffffffffu, sq, o);
    cross += __shfl_down_sync(0xffffffffu, cross, o);
    diff += __shfl_down_sync(0xffffffffu, diff, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = sq;
    red[1][w] = cross;
    red[2][w] = diff;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    sq = cross = diff = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      sq += red[0][i];
      cross += red[1][i];
      diff += red[2][i];
    }
    const double sigma_ss = acc_rows[3];
    const double plan_lin = acc_rows[0] + acc_cols[0] + 2.0 * cross - acc_rows[1] - acc_cols[1] +
                            2.0 * sigma_ss;
    const double kl = plan_lin / st->eps_n;
    const double obj =
        os->constant + 8.0 * (-sq + (os->eps_outer / 8.0) * kl - 2.0 * sigma_ss);
    const double err = acc_rows[2] + acc_cols[2];
    const int k = os->step;
    double* row = trace + 5 * k;
    row[0] = obj;
    row[1] = sqrt(diff);
    row[2] = err;
    row[3] = (double)st->applied;
    row[4] = ((double)globaltimer() - os->t0_ns) * 1e-9;
    os->step = k + 1;
    if (os->has_prev) {
      const double change = os->prev_objective - obj;
      if (fabs(change) < os->delta_outer) {
        os->converged = 1;
        os->done = 1;
      } else if (change < 0.0) {
        if (++os->ups >= 5) {
          os->error = 1;  // SolverError: objective increased 5 outer steps in a row
          os->done = 1;
        }
      } else {
        os->ups = 0;
      }
    }
    os->prev_objective = obj;
    os->has_prev = 1;
    if (os->step >= os->max_outer) os->done = 1;
  }
  __syncthreads();
  // Gamma_t -> coupling operator, Gamma_{t+1} -> next step's operator
  for (int k = threadIdx.x; k < de; k += blockDim.x) {
    gamma_prev[k] = gamma[k];
    gamma[k] = gnext[k];
  }
}

__global__ void set_condition_kernel(cudaGraphConditionalHandle h, const int32_t* done) {
  cudaGraphSetConditional(h, *done ? 0u : 1u);
}

// A conditional's default value is assigned once per graph LAUNCH, so a WHILE
// nested in another loop body must be re-armed every time the body runs.
__global__ void arm_condition_kernel(cudaGraphConditionalHandle h) { cudaGraphSetConditional(h, 1u); }

}  // namespace

extern "C" {

int cntgw_outer_state_size(void) { return (int)sizeof(cntgw_outer_state); }

int cntgw_outer_init(cntgw_outer_state* os, double constant, double eps_outer, double delta_outer,
                     int max_outer, void* stream) {
  if (!os || max_outer < 1) return fail(CNTGW_EINVAL, "outer_init: bad arguments");
  outer_init_kernel<<<1, 1, 0, as_stream(stream)>>>(os, constant, eps_outer, delta_outer, max_outer);
  return check_cuda(cudaPeekAtLastError(), "outer_init");
}

int cntgw_outer_finish(cntgw_outer_state* os, const cntgw_sweep_state* st, const double* acc_rows,
                       const double* acc_cols, double* gamma, double* gamma_prev, int de,
                       double* trace, void* stream) {
  if (!os || !st || !acc_rows || !acc_cols || !gamma || !gamma_prev || !trace || de < 1)
    return fail(CNTGW_EINVAL, "outer_finish: bad arguments");
  outer_finish_kernel<<<1, 256, 0, as_stream(stream)>>>(os, st, acc_rows, acc_cols, gamma,
                                                         gamma_prev, de, trace);
  return check_cuda(cudaPeekAtLastError(), "outer_finish");
}

int cntgw_graph_begin(void* stream) {
  return check_cuda(cudaStreamBeginCapture(as_stream(stream), cudaStreamCaptureModeRelaxed),
                    "cudaStreamBeginCapture");
}

int cntgw_graph_while_begin(void* stream, void* body_stream, uint64_t* handle_out) {
  if (!handle_out) return fail(CNTGW_EINVAL, "graph_while_begin: null handle");
  cudaStream_t s = as_stream(stream);
  cudaStreamCaptureStatus status;
  cudaGraph_t graph;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  int rc = check_cuda(cudaStreamGetCaptureInfo(s, &status, nullptr, &graph, &deps, &ndeps),
                      "cudaStreamGetCaptureInfo");
  if (rc) return rc;
  if (status != cudaStreamCaptureStatusActive)
    return fail(CNTGW_EINVAL, "graph_while_begin: stream is not capturing");
  cudaGraphConditionalHandle h;
  rc = check_cuda(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault),
                  "cudaGraphConditionalHandleCreate");
  if (rc) return rc;
  arm_condition_kernel<<<1, 1, 0, s>>>(h);  // re-armed on every pass of an enclosing body
  rc = check_cuda(cudaPeekAtLastError(), "arm_condition");
  if (rc) return rc;
  rc = check_cuda(cudaStreamGetCaptureInfo(s, &status, nullptr, &graph, &deps, &ndeps),
                  "cudaStreamGetCaptureInfo");
  if (rc) return rc;
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  rc = check_cuda(cudaGraphAddNode(&node, graph, deps, ndeps, &p), "cudaGraphAddNode(while)");
  if (rc) return rc;
  rc = check_cuda(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies),
                  "cudaStreamUpdateCaptureDependencies");
  if (rc) return rc;
  cudaGraph_t body = p.conditional.phGraph_out[0];
  rc = check_cuda(cudaStreamBeginCaptureToGraph(as_stream(body_stream), body, nullptr, nullptr, 0,
                                                cudaStreamCaptureModeRelaxed),
                  "cudaStreamBeginCaptureToGraph");
  if (rc) return rc;
  *handle_out = (uint64_t)h;
  return CNTGW_OK;
}

int cntgw_graph_while_end(void* body_stream) {
  cudaGraph_t g;
  return check_cuda(cudaStreamEndCapture(as_stream(body_stream), &g), "cudaStreamEndCapture(body)");
}

int cntgw_graph_set_condition(uint64_t handle, const int32_t* done_flag, void* stream) {
  if (!done_flag) return fail(CNTGW_EINVAL, "graph_set_condition: null flag");
  set_condition_kernel<<<1, 1, 0, as_stream(stream)>>>((cudaGraphConditionalHandle)handle, done_flag);
  return check_cuda(cudaPeekAtLastError(), "set_condition");
}

int cntgw_graph_end(void* stream, void** exec_out) {
  if (!exec_out) return fail(CNTGW_EINVAL, "graph_end: null output");
  cudaGraph_t g;
  int rc = check_cuda(cudaStreamEndCapture(as_stream(stream), &g), "cudaStreamEndCapture");
  if (rc) return rc;
  cudaGraphExec_t exec;
  rc = check_cuda(cudaGraphInstantiate(&exec, g, 0), "cudaGraphInstantiate");
  cudaGraphDestroy(g);
  if (rc) return rc;
  *exec_out = (void*)exec;
  return CNTGW_OK;
}

int cntgw_graph_launch(void* exec, void* stream) {
  if (!exec) return fail(CNTGW_EINVAL, "graph_launch: null graph");
  return check_cuda(cudaGraphLaunch((cudaGraphExec_t)exec, as_stream(stream)), "cudaGraphLaunch");
}

int cntgw_graph_destroy(void* exec) {
  if (!exec) return CNTGW_OK;
  return check_cuda(cudaGraphExecDestroy((cudaGraphExec_t)exec), "cudaGraphExecDestroy");
}

}  // extern "C"
