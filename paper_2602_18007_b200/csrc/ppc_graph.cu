// CUDA-graph capture of a 1F1B step (include/ppc.h ppc_graph_*).  The captured kernels take
// sequence numbers relative to per-comm device counters (SeqRef in ppc_internal.h); each
// launch sets the counters to the host's current sequence numbers, replays the graph and
// advances the host counters by the step's message counts.
//
// The step is captured on private per-stage streams (any caller stream works, including the
// legacy default stream, which cannot be captured): a launch orders the private streams
// after the caller's streams and the caller's streams after the replay.
#include <vector>

#include "ppc_comm_impl.h"

struct ppc_graph {
  std::vector<ppc_comm*> comms;
  std::vector<cudaStream_t> user;                 // caller streams, one per stage
  std::vector<cudaStream_t> cap;                  // private capture / launch streams
  std::vector<uint64_t> dsend[2], drecv[2];       // per comm, messages per step
  std::vector<cudaEvent_t> ev_in, ev_pro;         // caller -> launch, prologue joins
  cudaEvent_t ev_out = nullptr;                   // launch -> callers
  std::vector<cudaEvent_t> captured;              // events referenced by the graph's nodes
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  unsigned long long kernels = 0;                 // libppc kernel nodes (ppc_launch_count)
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
    if (!r) r = swap(c->zc_ev[d]);
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

cudaEvent_t new_event() {
  cudaEvent_t e = nullptr;
  if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
  return e;
}

#define GDBG(...) do { if (getenv("PPC_DEBUG")) fprintf(stderr, __VA_ARGS__); } while (0)

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
  g->user.assign(streams, streams + n);
  auto fail = [&](ppc_status_t st) {
    ppc_graph_destroy(g);
    return st;
  };
  // private streams and events; quiesce: eager work must not be referenced by the capture
  for (int k = 0; k < n; ++k) {
    ppc_comm* c = comms[k];
    DeviceGuard dg(c->device);
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return fail(PPC_ERR_CUDA);
    g->cap.push_back(s);
    g->ev_in.push_back(new_event());
    g->ev_pro.push_back(new_event());
    if (!g->ev_in.back() || !g->ev_pro.back()) return fail(PPC_ERR_CUDA);
    if (cudaDeviceSynchronize() != cudaSuccess) return fail(PPC_ERR_CUDA);
    if (!c->dseq && cudaMalloc(&c->dseq, 4 * sizeof(uint64_t)) != cudaSuccess)
      return fail(PPC_ERR_CUDA);
  }
  {
    DeviceGuard dg(comms[0]->device);
    if (!(g->ev_out = new_event())) return fail(PPC_ERR_CUDA);
  }
  std::vector<int> saved_trace(n);
  for (int k = 0; k < n; ++k) {
    ppc_comm* c = comms[k];
    reset_step_state(c);
    saved_trace[k] = c->cfg.trace;
    c->cfg.trace &= 1;   // records stay (each replay rewrites them); no per-launch events
    for (int d = 0; d < 2; ++d) {
      c->cap_send[d] = c->ch[d].send_seq;
      c->cap_recv[d] = c->ch[d].recv_seq;
    }
    c->capturing = true;
  }
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
  cudaStream_t s0 = g->cap[0];
  const unsigned long long launches0 = g_launches.load();
  cudaError_t e = cudaStreamBeginCapture(s0, cudaStreamCaptureModeRelaxed);
  if (e != cudaSuccess) {
    GDBG("ppc: graph begin capture %s\n", cudaGetErrorString(e));
    finish(PPC_ERR_CUDA);
    return fail(PPC_ERR_CUDA);
  }
  ppc_status_t st = PPC_OK;
  cudaEvent_t fork = new_event();             // fork every stage stream into the capture
  if (!fork || cudaEventRecord(fork, s0) != cudaSuccess) st = PPC_ERR_CUDA;
  for (int k = 1; k < n && !st; ++k)
    if (cudaStreamWaitEvent(g->cap[k], fork, 0) != cudaSuccess) st = PPC_ERR_CUDA;
  if (!st) st = n == 1 ? ppc_step_1f1b(comms[0], &steps[0], s0)
                       : ppc_step_1f1b_local(comms, n, steps, g->cap.data());
  if (st) GDBG("ppc: graph capture of the step failed: %d\n", (int)st);
  std::vector<cudaEvent_t> joins(n, nullptr);  // join them back
  for (int k = 1; k < n && !st; ++k) {
    DeviceGuard dg(comms[k]->device);
    if (!(joins[k] = new_event()) || cudaEventRecord(joins[k], g->cap[k]) != cudaSuccess ||
        cudaStreamWaitEvent(s0, joins[k], 0) != cudaSuccess)
      st = PPC_ERR_CUDA;
  }
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(s0, &graph);
  if (e != cudaSuccess) GDBG("ppc: graph end capture %s\n", cudaGetErrorString(e));
  if (!st && e != cudaSuccess) st = PPC_ERR_CUDA;
  if (fork) cudaEventDestroy(fork);
  for (cudaEvent_t j : joins) if (j) cudaEventDestroy(j);
  st = finish(st);
  g->kernels = g_launches.load() - launches0;   // captured, not run: counted per replay
  g_launches.fetch_sub(g->kernels);
  g->graph = graph;
  if (!st) {
    e = cudaGraphInstantiate(&g->exec, graph, 0);
    if (e != cudaSuccess) {
      GDBG("ppc: graph instantiate %s\n", cudaGetErrorString(e));
      st = PPC_ERR_CUDA;
    }
  }
  if (st) {
    cudaGetLastError();
    return fail(st);
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
  // prologue on the private streams: after the caller's work, set the device sequence
  // bases of every comm to its host counters, all joined into cap[0]
  for (int k = 0; k < n; ++k) {
    ppc_comm* c = g->comms[k];
    DeviceGuard dg(c->device);
    CK(cudaEventRecord(g->ev_in[k], g->user[k]));
    CK(cudaStreamWaitEvent(g->cap[k], g->ev_in[k], 0));
    CK(launch_set_seq(c->dseq, c->ch[0].send_seq, c->ch[1].send_seq, c->ch[0].recv_seq,
                      c->ch[1].recv_seq, g->cap[k]));
    if (k > 0) {
      CK(cudaEventRecord(g->ev_pro[k], g->cap[k]));
      DeviceGuard d0(g->comms[0]->device);
      CK(cudaStreamWaitEvent(g->cap[0], g->ev_pro[k], 0));
    }
  }
  {
    DeviceGuard d0(g->comms[0]->device);
    CK(cudaGraphLaunch(g->exec, g->cap[0]));
    g_launches.fetch_add(g->kernels);
    CK(cudaEventRecord(g->ev_out, g->cap[0]));
  }
  for (int k = 0; k < n; ++k) {                 // the caller's streams continue after it
    DeviceGuard dg(g->comms[k]->device);
    CK(cudaStreamWaitEvent(g->user[k], g->ev_out, 0));
    for (int d = 0; d < 2; ++d) {
      g->comms[k]->ch[d].send_seq += g->dsend[d][k];
      g->comms[k]->ch[d].recv_seq += g->drecv[d][k];
    }
  }
  return PPC_OK;
}

ppc_status_t ppc_graph_destroy(ppc_graph_t* g) {
  if (!g) return PPC_ERR_INVALID_ARG;
  for (ppc_comm* c : g->comms) {
    DeviceGuard dg(c->device);
    cudaDeviceSynchronize();
  }
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  for (cudaEvent_t e : g->ev_in) if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : g->ev_pro) if (e) cudaEventDestroy(e);
  if (g->ev_out) cudaEventDestroy(g->ev_out);
  for (cudaEvent_t e : g->captured) if (e) cudaEventDestroy(e);
  for (cudaStream_t s : g->cap) if (s) cudaStreamDestroy(s);
  delete g;
  return PPC_OK;
}

}  // extern "C"
