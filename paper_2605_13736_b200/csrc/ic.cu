// ic.cu — inertia correction of a scenario batch ON THE DEVICE (SURVEY §8(f)
// NEXT-1; "the regularization is performed repeatedly for
// increasingly large multiples until the linear solver reports that inertia for
// (5) is (n,0,m)", by PAPER.md:191 (n_d, 0, m) for the condensed matrix).
//
// Per scenario the multiples of the cited Algorithm IC (reading R22) run as a
// small state machine on the device, one step per trial round:
//   phase 0  the (0, 0) trial was evaluated: accept, or
//            delta_c = delta_c_bar mu^kappa_c iff zero eigenvalues were seen,
//            delta_w = delta_w0 (delta_w_last = 0) or max(delta_w_min, kappa_w_minus delta_w_last);
//   phase 1  a delta_w > 0 trial was evaluated: accept (delta_w_last = delta_w), or
//            delta_w *= kappa_w_plus_first (delta_w_last = 0) / kappa_w_plus; above
//            delta_w_max -> SINGULAR;
//   phase 2  accepted; 3 failed (singular); 4 data error (status set by condense/factor).
// active[s] = 1 exactly for the scenarios that need another trial: the batched
// condense and factor re-run only those (mask), the others keep their outputs.
// `mds_ic_graph_create` builds the whole loop as ONE CUDA graph: the first trial
// of every scenario, then a conditional WHILE node whose body (masked condense +
// masked factor + the step kernel) repeats while any scenario is active; the
// step kernel sets the loop condition with cudaGraphSetConditional.  No host
// round trip per trial.
#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include "common.cuh"

namespace {
struct IcState {
  double* dw;
  double* dc;
  double* dw_last;
  int32_t* phase;
  int32_t* active;
  int32_t* ntrial;
  int32_t* any;
};

__global__ void k_ic_begin(int64_t batch, IcState S) {
  pdl_wait();
  pdl_trigger();
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < batch; s += (int64_t)gridDim.x * blockDim.x) {
    S.dw[s] = 0.0;
    S.dc[s] = 0.0;
    S.phase[s] = 0;
    S.active[s] = 1;
    S.ntrial[s] = 1;
  }
}

__global__ void __launch_bounds__(1024) k_ic_step(int64_t batch, int64_t n_d, int64_t m, const mds_inertia* ine,
                                                 int32_t* status, const double* mu_arr, double mu,
                                                 mds_ic_params P, IcState S, cudaGraphConditionalHandle h, int use_h) {
  pdl_wait();
  pdl_trigger();
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  int mine = 0;
  for (int64_t s = threadIdx.x; s < batch; s += blockDim.x) {
    if (!S.active[s]) continue;
    const mds_inertia in = ine[s];
    const bool ok = in.pos == n_d && in.zero == 0 && in.neg == m;
    int act = 0;
    if (status[s] != 0) {
      S.phase[s] = 4;                                            // data error: no escalation can fix it
    } else if (S.phase[s] == 0) {
      if (ok) {
        S.phase[s] = 2;
      } else {
        const double mus = mu_arr ? mu_arr[s] : mu;
        S.dc[s] = in.zero > 0 ? P.delta_c_bar * pow(mus, P.kappa_c) : 0.0;                          // IC-2
        S.dw[s] = S.dw_last[s] == 0.0 ? P.delta_w0 : fmax(P.delta_w_min, P.kappa_w_minus * S.dw_last[s]);   // IC-3
        S.phase[s] = 1;
        act = 1;
      }
    } else {
      if (ok) {
        S.dw_last[s] = S.dw[s];                                  // IC-4
        S.phase[s] = 2;
      } else {
        S.dw[s] *= S.dw_last[s] == 0.0 ? P.kappa_w_plus_first : P.kappa_w_plus;    // IC-5
        if (S.dw[s] > P.delta_w_max) {
          S.phase[s] = 3;                                        // IC-6: singular, the solve skips it
          status[s] = MDS_ERR_SINGULAR;
        } else {
          act = 1;
        }
      }
    }
    S.active[s] = act;
    if (act) S.ntrial[s] += 1;
    mine |= act;
  }
  if (mine) atomicOr(&any, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    *S.any = any;
    if (use_h) cudaGraphSetConditional(h, any ? 1u : 0u);
  }
}

IcState state_of(const mds_ic_state* st) {
  IcState S;
  S.dw = st->delta_w; S.dc = st->delta_c; S.dw_last = st->delta_w_last; S.phase = st->phase;
  S.active = st->active; S.ntrial = st->ntrial; S.any = st->any_active;
  return S;
}
bool state_ok(const mds_ic_state* st) {
  return st && st->delta_w && st->delta_c && st->delta_w_last && st->phase && st->active && st->ntrial &&
         st->any_active;
}
}  // namespace

extern "C" int mds_ic_begin_batched(int64_t batch, const mds_ic_state* st, void* stream) {
  if (batch < 0 || !state_ok(st)) return MDS_ERR_ARG;
  if (batch == 0) return MDS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  MDS_LAUNCH(PC_VECTORS, s, MDS_CUDA_TRY(launch_pdl(k_ic_begin, dim3((unsigned)std::min<int64_t>(mds_cdiv(batch, 256), 64)),
                                                    dim3(256), 0, s, batch, state_of(st))));
  return MDS_OK;
}

static int ic_step(int64_t batch, int64_t n_d, int64_t m, const mds_inertia* inertia, int32_t* status,
                   const double* mu_arr, double mu, const mds_ic_params* params, const mds_ic_state* st,
                   cudaGraphConditionalHandle h, int use_h, cudaStream_t s) {
  if (batch < 0 || n_d < 0 || m < 0 || !inertia || !status || !params || !state_ok(st)) return MDS_ERR_ARG;
  if (batch == 0) return MDS_OK;
  MDS_LAUNCH(PC_VECTORS, s, MDS_CUDA_TRY(launch_pdl(k_ic_step, dim3(1), dim3(1024), 0, s, batch, n_d, m, inertia, status,
                                                    mu_arr, mu, *params, state_of(st), h, use_h)));
  return MDS_OK;
}

extern "C" int mds_ic_step_batched(int64_t batch, int64_t n_d, int64_t m, const mds_inertia* inertia,
                                   int32_t* status, const double* mu_arr, double mu,
                                   const mds_ic_params* params, const mds_ic_state* st, void* stream) {
  return ic_step(batch, n_d, m, inertia, status, mu_arr, mu, params, st, 0, 0, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// The whole correction loop as one CUDA graph (conditional WHILE node).
struct mds_ic_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

extern MdsVariant g_mds_var;

extern "C" int mds_ic_graph_create(const mds_plan* plan, const mds_condense_batched_args* ca,
                                   const mds_factor_batched_args* fa, int64_t n_d, int64_t m, const double* mu_arr,
                                   double mu, const mds_ic_params* params, const mds_ic_state* st,
                                   mds_ic_graph** out) {
  if (!plan || !ca || !fa || !params || !state_ok(st) || !out || ca->batch != fa->batch || ca->batch < 1)
    return MDS_ERR_ARG;
  const int64_t B = ca->batch;
  mds_ic_graph* G = new (std::nothrow) mds_ic_graph();
  if (!G) return MDS_ERR_ARG;
  cudaStream_t cs = nullptr;
  int rc = MDS_OK;
  const int saved_pdl = g_mds_var.no_pdl;
  auto fail = [&](int code) {
    g_mds_var.no_pdl = saved_pdl;
    if (cs) cudaStreamDestroy(cs);
    if (G->exec) cudaGraphExecDestroy(G->exec);
    if (G->graph) cudaGraphDestroy(G->graph);
    delete G;
    return code;
  };
  auto trial = [&](const int32_t* active) -> int {
    int r = mds_condense_batched(plan, B, ca->js_val, ca->str_val, ca->h_ss, ca->str_hss, ca->sigma_s, ca->str_sig,
                                 ca->H_dd, ca->ldh, ca->str_H, ca->sigma_d, ca->str_sd, ca->J_d, ca->ldj, ca->str_J,
                                 ca->d_h, ca->str_dh, st->delta_w, st->delta_c, ca->r, ca->str_r, ca->M, ca->ldm,
                                 ca->str_M, ca->rhs_c, ca->str_rhs, ca->w_out, ca->str_w, ca->anorm_out, ca->status,
                                 active, ca->work, ca->work_bytes, cs);
    if (r) return r;
    return mds_factor_batched(B, fa->N, ca->M, ca->ldm, ca->str_M, fa->piv, fa->str_piv, fa->zero_tol, ca->anorm_out,
                              fa->inertia_dev, ca->status, active, fa->work, fa->work_bytes, cs);
  };
  if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return fail(MDS_ERR_CUDA);
  // (programmatic-dependent-launch edges are not used inside the loop body)
  g_mds_var.no_pdl = 1;
  if (cudaGraphCreate(&G->graph, 0) != cudaSuccess) return fail(MDS_ERR_CUDA);
  cudaGraphConditionalHandle h;
  if (cudaGraphConditionalHandleCreate(&h, G->graph, 0, 0) != cudaSuccess) return fail(MDS_ERR_CUDA);
  // prologue: reset, first trial of every scenario, first step (sets the loop condition)
  if (cudaStreamBeginCaptureToGraph(cs, G->graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return fail(MDS_ERR_CUDA);
  rc = mds_ic_begin_batched(B, st, cs);
  if (!rc) rc = trial(nullptr);
  if (!rc) rc = ic_step(B, n_d, m, fa->inertia_dev, ca->status, mu_arr, mu, params, st, h, 1, cs);
  cudaGraph_t tmp = nullptr;
  if (cudaStreamEndCapture(cs, &tmp) != cudaSuccess || rc) return fail(rc ? rc : MDS_ERR_CUDA);
  // the conditional WHILE node after the prologue's leaf nodes
  size_t nleaf = 0;
  if (cudaGraphGetNodes(G->graph, nullptr, &nleaf) != cudaSuccess) return fail(MDS_ERR_CUDA);
  std::vector<cudaGraphNode_t> nodes(nleaf);
  cudaGraphGetNodes(G->graph, nodes.data(), &nleaf);
  std::vector<cudaGraphNode_t> leaves;
  for (auto n : nodes) {
    size_t nd = 0;
    cudaGraphNodeGetDependentNodes(n, nullptr, &nd);
    if (nd == 0) leaves.push_back(n);
  }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cnode;
  if (cudaGraphAddNode(&cnode, G->graph, leaves.data(), leaves.size(), &cp) != cudaSuccess) return fail(MDS_ERR_CUDA);
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  if (cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return fail(MDS_ERR_CUDA);
  rc = trial(st->active);
  if (!rc) rc = ic_step(B, n_d, m, fa->inertia_dev, ca->status, mu_arr, mu, params, st, h, 1, cs);
  cudaGraph_t tmp2 = nullptr;
  if (cudaStreamEndCapture(cs, &tmp2) != cudaSuccess || rc) return fail(rc ? rc : MDS_ERR_CUDA);
  g_mds_var.no_pdl = saved_pdl;
  if (cudaGraphInstantiate(&G->exec, G->graph, 0) != cudaSuccess) return fail(MDS_ERR_CUDA);
  cudaStreamDestroy(cs);
  *out = G;
  return MDS_OK;
}

extern "C" int mds_ic_graph_launch(mds_ic_graph* G, void* stream) {
  if (!G || !G->exec) return MDS_ERR_ARG;
  MDS_CUDA_TRY(cudaGraphLaunch(G->exec, (cudaStream_t)stream));
  return MDS_OK;
}

extern "C" int mds_ic_graph_destroy(mds_ic_graph* G) {
  if (!G) return MDS_ERR_ARG;
  if (G->exec) cudaGraphExecDestroy(G->exec);
  if (G->graph) cudaGraphDestroy(G->graph);
  delete G;
  return MDS_OK;
}
