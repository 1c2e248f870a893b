// 1F1B step driver (§8(a) row a7): per op recv -> stage fn -> send, host only enqueues.
// Op order = ppc_schedule_1f1b (R2).  Receives and stage compute
// run on the caller's stream; sends run on the comm's per-direction side streams so that
// a middle stage's FWD and BWD transfers overlap each other and the next op (the full-
// duplex NVLink steady state).  Buffer reuse across streams is ordered by events.
#include "ppc_comm_impl.h"

namespace {

bool is_host_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
}

ppc_status_t ensure_bufs(ppc_comm* c, size_t bytes) {
  StepBufs& sb = c->sb;
  if (!sb.ready) {
    CK(cudaEventCreateWithFlags(&sb.ready, cudaEventDisableTiming));
    for (int d = 0; d < 2; ++d) {
      CK(cudaEventCreateWithFlags(&sb.join[d], cudaEventDisableTiming));
      for (int i = 0; i < 2; ++i) {
        CK(cudaEventCreateWithFlags(&sb.rfree[d][i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&sb.ofree[d][i], cudaEventDisableTiming));
      }
    }
  }
  if (bytes <= sb.bytes) return PPC_OK;
  CK(cudaDeviceSynchronize());
  for (int d = 0; d < 2; ++d)
    for (int i = 0; i < 2; ++i) {
      if (sb.rbuf[d][i]) cudaFree(sb.rbuf[d][i]);
      if (sb.obuf[d][i]) cudaFree(sb.obuf[d][i]);
      sb.rbuf[d][i] = sb.obuf[d][i] = nullptr;
      CK(cudaMalloc(&sb.rbuf[d][i], bytes));
      CK(cudaMalloc(&sb.obuf[d][i], bytes));
      CK(cudaMemset(sb.obuf[d][i], 0, bytes));
      sb.rpending[d][i] = sb.opending[d][i] = false;
    }
  sb.bytes = bytes;
  return PPC_OK;
}

// Resumable enqueuer of one stage's step.  advance() enqueues ops until done or until a
// virtual-stage send/recv reports PPC_ERR_WOULD_BLOCK (then the caller retries later).
struct Stepper {
  ppc_comm* c = nullptr;
  const ppc_step_t* st = nullptr;
  cudaStream_t cs = nullptr;
  int S = 1, s = 0;
  std::vector<ppc_op_t> ops;
  size_t i = 0;
  int phase = 0;
  const void* in = nullptr;
  const void* send_src = nullptr;
  cudaEvent_t send_free = nullptr;
  bool* send_pending = nullptr;
  bool direct = false;          // the receive landed in the terminal destination already

  ppc_status_t init(ppc_comm* comm, const ppc_step_t* step, cudaStream_t stream) {
    c = comm;
    st = step;
    cs = stream;
    if (!c || !st || st->M < 1) return PPC_ERR_INVALID_ARG;
    S = c->cfg.pp;
    s = c->pp_i;
    ops.resize(2 * (size_t)st->M);
    int n = 0;
    ppc_status_t r = ppc_schedule_1f1b(S, s, st->M, ops.data(), &n);
    if (r) return r;
    ops.resize(n);
    return ensure_bufs(c, std::max<size_t>(std::max(st->fwd_bytes, st->bwd_bytes), 256));
  }

  bool done() const { return i == ops.size(); }

  ppc_status_t advance(bool* progressed) {
    StepBufs& sb = c->sb;
    while (i < ops.size()) {
      const int kind = ops[i].kind, m = ops[i].mb, d = kind;   // F travels FWD, B travels BWD
      const size_t bytes = kind == 0 ? st->fwd_bytes : st->bwd_bytes;
      const bool has_in = kind == 0 ? s > 0 : s < S - 1;
      const bool has_out = kind == 0 ? s < S - 1 : s > 0;
      const int bi = m & 1;
      if (phase == 0) {                                  // input
        direct = false;
        if (has_in) {
          // terminal identity op with a device destination: receive straight into it
          void* const* dsts = kind == 0 ? st->y : st->dx;
          void* dst = (!has_out && !(kind == 0 ? st->fwd : st->bwd) && dsts) ? dsts[m] : nullptr;
          if (dst && is_host_ptr(dst)) dst = nullptr;
          uint8_t* r = dst ? static_cast<uint8_t*>(dst) : sb.rbuf[d][bi];
          if (!dst && sb.rpending[d][bi]) CK(cudaStreamWaitEvent(cs, sb.rfree[d][bi], 0));
          ppc_status_t rs = ppc_pp_recv(c, (ppc_dir_t)d, r, bytes, m, cs);
          if (rs == PPC_ERR_WOULD_BLOCK) return PPC_OK;
          if (rs) return rs;
          if (!dst) sb.rpending[d][bi] = false;
          direct = dst != nullptr;
          in = r;
        } else {
          const void* const* srcs = kind == 0 ? st->x : st->g;
          in = srcs ? srcs[m] : nullptr;
          if (in && is_host_ptr(in)) {
            uint8_t* r = sb.rbuf[d][bi];
            if (sb.rpending[d][bi]) CK(cudaStreamWaitEvent(cs, sb.rfree[d][bi], 0));
            sb.rpending[d][bi] = false;
            CK(cudaMemcpyAsync(r, in, bytes, cudaMemcpyHostToDevice, cs));
            in = r;
          }
        }
        *progressed = true;
        phase = 1;
      }
      if (phase == 1) {                                  // stage compute
        ppc_stage_fn fn = kind == 0 ? st->fwd : st->bwd;
        void* user = kind == 0 ? st->fwd_user : st->bwd_user;
        if (has_out) {
          if (fn) {
            uint8_t* o = sb.obuf[d][bi];
            if (sb.opending[d][bi]) CK(cudaStreamWaitEvent(cs, sb.ofree[d][bi], 0));
            if (fn(user, m, in, o, in ? bytes : 0, bytes, cs) != 0) return PPC_ERR_INVALID_ARG;
            send_src = o;
            send_free = sb.ofree[d][bi];
            send_pending = &sb.opending[d][bi];
          } else if (in == sb.rbuf[d][bi]) {
            send_src = in;
            send_free = sb.rfree[d][bi];
            send_pending = &sb.rpending[d][bi];
          } else if (in) {                               // caller's device buffer
            send_src = in;
            send_free = nullptr;
            send_pending = nullptr;
          } else {                                       // no input given: scratch contents
            send_src = sb.obuf[d][bi];
            send_free = sb.ofree[d][bi];
            send_pending = &sb.opending[d][bi];
            if (sb.opending[d][bi]) CK(cudaStreamWaitEvent(cs, sb.ofree[d][bi], 0));
          }
          CK(cudaEventRecord(sb.ready, cs));
          CK(cudaStreamWaitEvent(c->side[d], sb.ready, 0));
        } else {
          void* const* dsts = kind == 0 ? st->y : st->dx;
          void* dst = dsts ? dsts[m] : nullptr;
          if (fn) {
            const bool host = dst && is_host_ptr(dst);
            uint8_t* o = sb.obuf[d][bi];
            if (sb.opending[d][bi]) {
              CK(cudaStreamWaitEvent(cs, sb.ofree[d][bi], 0));
              sb.opending[d][bi] = false;
            }
            void* target = (dst && !host) ? dst : o;
            if (fn(user, m, in, target, in ? bytes : 0, bytes, cs) != 0) return PPC_ERR_INVALID_ARG;
            if (host) CK(cudaMemcpyAsync(dst, o, bytes, cudaMemcpyDeviceToHost, cs));
          } else if (dst && in && bytes && !direct) {
            CK(cudaMemcpyAsync(dst, in, bytes, cudaMemcpyDefault, cs));
          }
        }
        *progressed = true;
        phase = 2;
      }
      if (phase == 2) {                                  // send
        if (has_out) {
          ppc_status_t ss = ppc_pp_send(c, (ppc_dir_t)d, send_src, bytes, m, c->side[d]);
          if (ss == PPC_ERR_WOULD_BLOCK) return PPC_OK;
          if (ss) return ss;
          if (send_free) {
            CK(cudaEventRecord(send_free, c->side[d]));
            *send_pending = true;
          }
        }
        *progressed = true;
        phase = 0;
        ++i;
      }
    }
    return PPC_OK;
  }

  ppc_status_t finish() {
    for (int d = 0; d < 2; ++d) {
      CK(cudaEventRecord(c->sb.join[d], c->side[d]));
      CK(cudaStreamWaitEvent(cs, c->sb.join[d], 0));
    }
    return PPC_OK;
  }
};

}  // namespace

extern "C" ppc_status_t ppc_step_1f1b(ppc_comm_t* c, const ppc_step_t* st, cudaStream_t s) {
  ppc_status_t r = check_live(c);
  if (r) return r;
  if (c->device < 0) return PPC_ERR_STATE;
  if (c->local_mode) return PPC_ERR_INVALID_ARG;     // virtual stages: ppc_step_1f1b_local
  DeviceGuard g(c->device);
  Stepper sp;
  if ((r = sp.init(c, st, s))) return r;
  while (!sp.done()) {
    bool prog = false;
    if ((r = sp.advance(&prog))) return r;
    if (!prog) return PPC_ERR_STATE;
  }
  return sp.finish();
}

extern "C" ppc_status_t ppc_step_1f1b_local(ppc_comm_t* const* comms, int S,
                                            const ppc_step_t* steps,
                                            const cudaStream_t* streams) {
  if (!comms || !steps || !streams || S < 1) return PPC_ERR_INVALID_ARG;
  std::vector<Stepper> sp(S);
  for (int k = 0; k < S; ++k) {
    ppc_status_t r = check_live(comms[k]);
    if (r) return r;
    if (comms[k]->cfg.pp != S || comms[k]->pp_i != k) return PPC_ERR_INVALID_ARG;
    if (S > 1 && !comms[k]->local_mode) return PPC_ERR_INVALID_ARG;
    if (steps[k].M != steps[0].M) return PPC_ERR_INVALID_ARG;
    DeviceGuard g(comms[k]->device);
    if ((r = sp[k].init(comms[k], &steps[k], streams[k]))) return r;
  }
  // round-robin: a dependency-respecting enqueue order (every recv after its send)
  for (;;) {
    bool all = true, prog = false;
    for (int k = 0; k < S; ++k) {
      if (sp[k].done()) continue;
      DeviceGuard g(comms[k]->device);
      ppc_status_t r = sp[k].advance(&prog);
      if (r) return r;
      all = all && sp[k].done();
    }
    if (all) break;
    if (!prog) return PPC_ERR_STATE;
  }
  for (int k = 0; k < S; ++k) {
    DeviceGuard g(comms[k]->device);
    ppc_status_t r = sp[k].finish();
    if (r) return r;
  }
  return PPC_OK;
}
