// CUDA-graph capture of a 1F1B step (include/ppc.h ppc_graph_*).  The captured kernels take
// sequence numbers relative to per-comm device counters (SeqRef in ppc_internal.h); each
// launch sets the counters to the host's current sequence numbers, replays the graph and
// advances the host counters by the step's message counts.
#include <vector>

#include "ppc_comm_impl.h"

struct ppc_graph {
  std::vector<ppc_comm*> comms;
  std::vector<cudaStream_t> streams;
  std::vector<uint64_t> dsend[2], drecv[2];       // per comm, messages per step
  std::vector<cudaEvent_t> ev;                    // prologue joins
  std::vector<cudaEvent_t> captured;              // events referenced by the graph's nodes
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

namespace {

// Events recorded inside a capture become graph nodes and can no longer be waited on by
// eager work; the graph keeps them (they must outlive it) and the comm gets fresh ones.
cudaError_t swap_events(ppc_comm* c, std::vector<cudaEvent_t>& keep) {
  auto swap = [&](cudaEvent_t& e) -> cudaError_t {
    if (!e) return cudaSuccess;
    keep.push_back(e);
    return cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  };
  StepBufs& sb = c->sb;
  cudaError_t r = swap(sb.ready);
  for (int d = 0; d < 2; ++d) {
    if (!r) r = swap(sb.join[d]);
    for (int i = 0; i < 2 && !r; ++i) {
      r = swap(sb.rfree[d][i]);
      if (!r) r = swap(sb.ofree[d][i]);
      if (!r) r = swap(sb.dready[d][i]);
      if (!r) r = swap(sb.cons_r[d][i]);
      if (!r) r = swap(sb.cons_o[d][i]);
    }
    for (auto& e : c->ch[d].sent_ev) if (!r) r = swap(e);
    for (auto& e : c->ch[d].recvd_ev) if (!r) r = swap(e);
  }
  return r;
}

void reset_step_state(ppc_comm* c) {
  StepBufs& sb = c->sb;
  for (int d = 0; d < 2; ++d)
    for (int i = 0; i < 2; ++i) {
      sb.rpending[d][i] = sb.opending[d][i] = false;
      sb.held_r[d][i] = sb.held_o[d][i] = false;
      sb.cwait_r[d][i] = sb.cwait_o[d][i] = false;
    }
}

}  // namespace

extern "C" {

ppc_status_t ppc_graph_create(ppc_comm_t* const* comms, int n, const ppc_step_t* steps,
                              const cudaStream_t* streams, ppc_graph_t** out) {
  if (!comms || !steps || !streams || !out || n < 1) return PPC_ERR_INVALID_ARG;
  *out = nullptr;
  for (int k = 0; k < n; ++k) {
    ppc_status_t st = check_live(comms[k]);
    if (st) return st;
    if (comms[k]->device < 0) return PPC_ERR_STATE;
    if (comms[k]->cfg.engine == PPC_ENGINE_CE) return PPC_ERR_INVALID_ARG;
    // the step's buffers must already exist (one eager step first): no allocation in capture
    const size_t need = std::max<size_t>(std::max(steps[k].fwd_bytes, steps[k].bwd_bytes), 256);
    if (comms[k]->sb.bytes < need) return PPC_ERR_STATE;
  }
  if (n == 1 && comms[0]->local_mode && comms[0]->cfg.pp > 1) return PPC_ERR_INVALID_ARG;
  ppc_graph* g = new ppc_graph();
  g->comms.assign(comms, comms + n);
  g->streams.assign(streams, streams + n);
  std::vector<int> saved_trace(n);
  // quiesce: eager work must not be referenced from inside the capture
  for (int k = 0; k < n; ++k) {
    ppc_comm* c = comms[k];
    DeviceGuard dg(c->device);
    if (cudaDeviceSynchronize() != cudaSuccess) { delete g; return PPC_ERR_CUDA; }
    if (!c->dseq && cudaMalloc(&c->dseq, 4 * sizeof(uint64_t)) != cudaSuccess) {
      delete g;
      return PPC_ERR_CUDA;
    }
    reset_step_state(c);
    saved_trace[k] = c->cfg.trace;
    c->cfg.trace = 0;                         // no per-launch events / records in the graph
    for (int d = 0; d < 2; ++d) {
      c->cap_send[d] = c->ch[d].send_seq;
      c->cap_recv[d] = c->ch[d].recv_seq;
    }
  }
  for (int k = 0; k < n; ++k) comms[k]->capturing = true;
  auto finish = [&](ppc_status_t st) {
    for (int k = 0; k < n; ++k) {
      ppc_comm* c = comms[k];
      for (int d = 0; d < 2; ++d) {
        g->dsend[d].push_back(c->ch[d].send_seq - c->cap_send[d]);
        g->drecv[d].push_back(c->ch[d].recv_seq - c->cap_recv[d]);
        c->ch[d].send_seq = c->cap_send[d];   // the capture ran nothing: roll back
        c->ch[d].recv_seq = c->cap_recv[d];
      }
      c->capturing = false;
      c->cfg.trace = saved_trace[k];
      reset_step_state(c);
      DeviceGuard dgk(c->device);
      if (swap_events(c, g->captured) != cudaSuccess && !st) st = PPC_ERR_CUDA;
    }
    return st;
  };
  DeviceGuard dg0(comms[0]->device);
  cudaStream_t s0 = streams[0];
  if (cudaStreamBeginCapture(s0, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    finish(PPC_ERR_CUDA);
    delete g;
    return PPC_ERR_CUDA;
  }
  ppc_status_t st = PPC_OK;
  // fork every stage stream into the capture
  cudaEvent_t fork = nullptr;
  if (cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(fork, s0) != cudaSuccess)
    st = PPC_ERR_CUDA;
  for (int k = 1; k < n && !st; ++k)
    if (cudaStreamWaitEvent(streams[k], fork, 0) != cudaSuccess) st = PPC_ERR_CUDA;
  if (!st) st = n == 1 ? ppc_step_1f1b(comms[0], &steps[0], s0)
                       : ppc_step_1f1b_local(comms, n, steps, streams);
  // join them back
  std::vector<cudaEvent_t> joins(n, nullptr);
  for (int k = 1; k < n && !st; ++k) {
    DeviceGuard dg(comms[k]->device);
    if (cudaEventCreateWithFlags(&joins[k], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(joins[k], streams[k]) != cudaSuccess ||
        cudaStreamWaitEvent(s0, joins[k], 0) != cudaSuccess)
      st = PPC_ERR_CUDA;
  }
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(s0, &graph);
  if (getenv("PPC_DEBUG") && (st || ec != cudaSuccess))
    fprintf(stderr, "ppc: graph capture step=%d end=%s\n", (int)st, cudaGetErrorString(ec));
  if (!st && ec != cudaSuccess) st = PPC_ERR_CUDA;
  if (fork) cudaEventDestroy(fork);
  for (cudaEvent_t e : joins) if (e) cudaEventDestroy(e);
  st = finish(st);
  if (!st) {
    const cudaError_t ei = cudaGraphInstantiate(&g->exec, graph, 0);
    if (ei != cudaSuccess) {
      if (getenv("PPC_DEBUG")) fprintf(stderr, "ppc: graph instantiate %s\n", cudaGetErrorString(ei));
      st = PPC_ERR_CUDA;
    }
  }
  g->graph = graph;
  if (st) {
    cudaGetLastError();
    ppc_graph_destroy(g);
    return st;
  }
  for (int k = 0; k < n; ++k) {
    cudaEvent_t e = nullptr;
    DeviceGuard dg(comms[k]->device);
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      ppc_graph_destroy(g);
      return PPC_ERR_CUDA;
    }
    g->ev.push_back(e);
  }
  *out = g;
  return PPC_OK;
}

ppc_status_t ppc_graph_launch(ppc_graph_t* g) {
  if (!g || !g->exec) return PPC_ERR_INVALID_ARG;
  const int n = (int)g->comms.size();
  for (int k = 0; k < n; ++k) {
    ppc_status_t st = check_live(g->comms[k]);
    if (st) return st;
  }
  // prologue: every comm's device sequence bases = its host counters, ordered before s0
  for (int k = 0; k < n; ++k) {
    ppc_comm* c = g->comms[k];
    DeviceGuard dg(c->device);
    CK(launch_set_seq(c->dseq, c->ch[0].send_seq, c->ch[1].send_seq, c->ch[0].recv_seq,
                      c->ch[1].recv_seq, g->streams[k]));
    if (k > 0) {
      CK(cudaEventRecord(g->ev[k], g->streams[k]));
      DeviceGuard d0(g->comms[0]->device);
      CK(cudaStreamWaitEvent(g->streams[0], g->ev[k], 0));
    }
  }
  {
    DeviceGuard d0(g->comms[0]->device);
    CK(cudaGraphLaunch(g->exec, g->streams[0]));
  }
  for (int k = 0; k < n; ++k)
    for (int d = 0; d < 2; ++d) {
      g->comms[k]->ch[d].send_seq += g->dsend[d][k];
      g->comms[k]->ch[d].recv_seq += g->drecv[d][k];
    }
  return PPC_OK;
}

ppc_status_t ppc_graph_destroy(ppc_graph_t* g) {
  if (!g) return PPC_ERR_INVALID_ARG;
  if (!g->comms.empty()) {
    DeviceGuard dg(g->comms[0]->device);
    cudaDeviceSynchronize();
  }
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  for (cudaEvent_t e : g->ev) if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : g->captured) if (e) cudaEventDestroy(e);
  delete g;
  return PPC_OK;
}

}  // extern "C"
