// 1F1B step driver (§8(a) row a7): per op recv -> stage fn -> send, host only enqueues.
// Op order = ppc_schedule_1f1b (R2).  Receives and stage compute
// run on the caller's stream; sends run on the comm's per-direction side streams so that
// a middle stage's FWD and BWD transfers overlap each other and the next op (the full-
// duplex NVLink steady state).  Buffer reuse across streams is ordered by events.
//
// Direct mode (virtual stages sharing one GPU): the driver sees every stage,
// so a message is handed over as (pointer, ready event) and the receiving stage makes the
// ONE copy into its destination; the sending stage's buffer is held until that copy is
// enqueued and reused only after it completes.  One HBM copy per message instead of the
// ring's two (push into the slot + copy-out).  PPC_LOCAL_DIRECT=0 selects the ring path.
#include <deque>

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
    CK(cudaEventCreateWithFlags(&sb.xgo, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sb.xdone, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sb.dgo, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sb.djoin, cudaEventDisableTiming));
    for (int d = 0; d < 2; ++d) {
      CK(cudaEventCreateWithFlags(&sb.join[d], cudaEventDisableTiming));
      for (int i = 0; i < 2; ++i) {
        CK(cudaEventCreateWithFlags(&sb.rfree[d][i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&sb.ofree[d][i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&sb.dready[d][i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&sb.cons_r[d][i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&sb.cons_o[d][i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&sb.dfree_r[d][i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&sb.dfree_o[d][i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&sb.hdone[d][i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&sb.rlast[d][i], cudaEventDisableTiming));
      }
    }
  }
  if (bytes <= sb.bytes) return PPC_OK;
  // only freeing old scratch needs the device idle (the first call allocates nothing that is
  // in use; with cfg.local_spin another stage of this process may already be spinning)
  if (!sb.in_arena && sb.rbuf[0][0]) CK(cudaDeviceSynchronize());
  // messages up to max_msg_bytes: the arena's step region (zeroed at create; a peer can
  // pull a forwarded message from it, zero-copy); larger scratch falls back to cudaMalloc
  const bool arena = c->arena && bytes <= c->lay.stride;
  for (int d = 0; d < 2; ++d)
    for (int i = 0; i < 2; ++i) {
      if (!sb.in_arena) {
        if (sb.rbuf[d][i]) cudaFree(sb.rbuf[d][i]);
        if (sb.obuf[d][i]) cudaFree(sb.obuf[d][i]);
      }
      sb.rbuf[d][i] = sb.obuf[d][i] = nullptr;
      if (arena) {
        sb.rbuf[d][i] = c->arena + c->lay.step + (size_t)((0 * 2 + d) * 2 + i) * c->lay.stride;
        sb.obuf[d][i] = c->arena + c->lay.step + (size_t)((1 * 2 + d) * 2 + i) * c->lay.stride;
      } else {
        CK(cudaMalloc(&sb.rbuf[d][i], bytes));
        CK(cudaMalloc(&sb.obuf[d][i], bytes));
        CK(cudaMemset(sb.obuf[d][i], 0, bytes));
      }
      sb.rpending[d][i] = sb.opending[d][i] = false;
    }
  sb.in_arena = arena;
  sb.bytes = arena ? c->lay.stride : bytes;
  return PPC_OK;
}

// A message handed from one virtual stage to the next in direct mode.
struct Pending {
  const void* src;
  size_t bytes;
  long long mb;
  cudaEvent_t ready;      // src is complete once this fires
  cudaEvent_t consumed;   // recorded by the receiver after its copy (nullptr: user buffer)
  bool* held;
  bool* cwait;
};
using Mailbox = std::deque<Pending>;

// Resumable enqueuer of one stage's step.  advance() enqueues ops until done or until a
// virtual-stage send/recv cannot proceed yet (then the caller retries later).
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
  int send_buf = 0;             // direct mode: 0 = user buffer, 1 = rbuf, 2 = obuf
  bool direct = false;          // the receive landed in the terminal destination already
  bool zc_send = false;         // this op's send source is a registered buffer
  bool zc_cs = false;           // ... and it is published from the compute stream
  bool used_zcw[2] = {false, false};
  // direct mode: inbox[d] = messages sent to this stage in direction d; out[d] = receiver's
  Mailbox* inbox[2] = {nullptr, nullptr};
  Mailbox* outbox[2] = {nullptr, nullptr};
  bool fused_next = false;      // the next op's send was fused into this op's receive
  bool inplace_sent = false;    // this op's stage fn produced straight into the peer's slot
  bool used_ds = false;         // a terminal output went to host memory through sb.ds
  bool dmode = false;
  cudaStream_t xq = nullptr;    // direct mode: the GPU's transfer queue (nullptr: own stream)
  // PPC_STEP_BATCH=1 (one process per GPU): consecutive terminal receives (identity stage,
  // device destination — with the next op's zero-copy publication fused in or not) whose
  // ops enqueue nothing else on the compute stream are collected and launched as ONE
  // batched-receive grid (ppc_impl_recv_launch_batch), so the receiving CTAs flow from one
  // message to the next without a kernel boundary.  Their rendezvous commits and completion
  // bookkeeping follow the grid.
  // Rendezvous commits of zero-copy sends from the caller's own buffers (x / g: never
  // rewritten inside the step) are deferred to the step's end — one bounded credit wait per
  // direction for the highest seq (credits are monotone and returned in order) instead of an
  // event record on the compute stream + a wait kernel per message, so consecutive receive
  // kernels on the compute stream stay PDL-chained.  Sends from the double-buffered step
  // buffers keep their per-message commit (the buffer is reused two micro-batches later).
  ZcSend last_commit[2];
  bool has_last_commit[2] = {false, false};
  void defer_commit(const ZcSend& z) {
    last_commit[z.d] = z;
    has_last_commit[z.d] = true;
  }

  // Chained receives (PPC_RECV_CHAIN): a terminal receive into a device destination whose
  // kernel also carries the next op's publication enqueues nothing else on the compute
  // stream, and neither does that next (fused source) op; so when the op after it is a
  // receive again, the last thing on the stream is the previous receive's kernel, and the
  // new receive may start on that kernel's posted completion (ppc_impl_recv_ex prev).
  RecvChainRef chain_prev{0, 0};
  size_t chain_op = (size_t)-1;   // op index of that receive; chained iff i == chain_op + 2

  bool batching = false;
  std::vector<RecvArgs> pend;
  std::vector<std::pair<int, uint64_t>> pend_done;   // (dir, seq)
  std::vector<ZcSend> pend_commit;

  ppc_status_t flush() {
    if (pend.empty()) return PPC_OK;
    for (size_t b = 0; b < pend.size(); b += kMaxBatch) {
      const int n = (int)std::min<size_t>(kMaxBatch, pend.size() - b);
      if (ppc_status_t st = ppc_impl_recv_launch_batch(c, pend.data() + b, n, cs)) return st;
    }
    for (auto& dq : pend_done)
      if (ppc_status_t st = ppc_impl_recv_done(c, (ppc_dir_t)dq.first, dq.second, cs)) return st;
    for (const ZcSend& z : pend_commit) defer_commit(z);
    pend.clear();
    pend_done.clear();
    pend_commit.clear();
    return PPC_OK;
  }

  // the op's input is a terminal identity receive into a device destination
  bool terminal_recv(int kind, int m) const {
    const bool has_in = kind == 0 ? s > 0 : s < S - 1;
    const bool has_out = kind == 0 ? s < S - 1 : s > 0;
    void* const* dsts = kind == 0 ? st->y : st->dx;
    return has_in && !has_out && !(kind == 0 ? st->fwd : st->bwd) && dsts && dsts[m] &&
           !is_host_ptr(dsts[m]);
  }

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

  // before stream q writes rbuf / obuf [d][bi]: wait for a pending device->host read of it
  ppc_status_t before_write(int kind, int d, int bi, cudaStream_t q) {
    StepBufs& sb = c->sb;
    bool* pend = kind == 1 ? &sb.dpend_r[d][bi] : &sb.dpend_o[d][bi];
    if (*pend) {
      CK(cudaStreamWaitEvent(q, kind == 1 ? sb.dfree_r[d][bi] : sb.dfree_o[d][bi], 0));
      *pend = false;
    }
    return PPC_OK;
  }

  // the compute stream just read `in`: if it is the staging buffer rbuf [d][bi], the next
  // host->device staging into it (on hs) must wait for this point
  ppc_status_t mark_read(const void* in, int d, int bi) {
    StepBufs& sb = c->sb;
    if (in && in == sb.rbuf[d][bi]) {
      CK(cudaEventRecord(sb.rlast[d][bi], cs));
      sb.rlast_set[d][bi] = true;
    }
    return PPC_OK;
  }

  // terminal output to host memory: copy on the D2H stream (kind: 1 = src is rbuf [d][bi],
  // 2 = obuf [d][bi], 0 = a caller buffer)
  ppc_status_t d2h(void* dst, const void* src, size_t bytes, int kind, int d, int bi) {
    StepBufs& sb = c->sb;
    if (!sb.ds) CK(cudaStreamCreateWithFlags(&sb.ds, cudaStreamNonBlocking));   // first use
    CK(cudaEventRecord(sb.dgo, cs));
    CK(cudaStreamWaitEvent(sb.ds, sb.dgo, 0));
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, sb.ds));
    if (kind == 1) {
      CK(cudaEventRecord(sb.dfree_r[d][bi], sb.ds));
      sb.dpend_r[d][bi] = true;
    } else if (kind == 2) {
      CK(cudaEventRecord(sb.dfree_o[d][bi], sb.ds));
      sb.dpend_o[d][bi] = true;
    }
    used_ds = true;
    return PPC_OK;
  }

  // Fusion of "terminal receive, then a zero-copy send with no stage compute in between"
  // (both ends of a comm-only PP2 step: F_m lands in y[m], then B_m leaves from g[m]).
  // The next op is a source op (no input, no stage function) whose registered source is
  // published from the compute stream: its publication then rides on this receive's
  // kernel (the last CTA writes the header right after the credit), saving one kernel
  // boundary on the critical path.  The order of the two ops is unchanged.
  // PPC_FUSE_PUBLISH=0 disables it.
  bool fusable_next(ZcSend* z) {
    if (i + 1 >= ops.size() || c->zc_side || !c->fuse_publish) return false;
    const int kind = ops[i + 1].kind, m = ops[i + 1].mb;
    const bool has_in = kind == 0 ? s > 0 : s < S - 1;
    const bool has_out = kind == 0 ? s < S - 1 : s > 0;
    if (has_in || !has_out || (kind == 0 ? st->fwd : st->bwd)) return false;
    const void* const* srcs = kind == 0 ? st->x : st->g;
    const void* src = srcs ? srcs[m] : nullptr;
    const size_t bytes = kind == 0 ? st->fwd_bytes : st->bwd_bytes;
    if (!src || !bytes || is_host_ptr(src) || !ppc_impl_is_zero_copy(c, src, bytes)) return false;
    return ppc_impl_zc_prepare(c, (ppc_dir_t)kind, src, bytes, m, z) == PPC_OK;
  }

  // direct mode: may the stage overwrite its buffer (kind 1 = rbuf, 2 = obuf) [d][bi]?
  // false = the receiving stage has not enqueued its copy yet (caller returns, retries).
  bool reuse_ok(int kind, int d, int bi, ppc_status_t* err, cudaStream_t q = nullptr) {
    StepBufs& sb = c->sb;
    bool* held = kind == 1 ? &sb.held_r[d][bi] : &sb.held_o[d][bi];
    bool* cw = kind == 1 ? &sb.cwait_r[d][bi] : &sb.cwait_o[d][bi];
    if (*held) return false;
    if (*cw) {
      cudaEvent_t e = kind == 1 ? sb.cons_r[d][bi] : sb.cons_o[d][bi];
      if (cudaStreamWaitEvent(q ? q : cs, e, 0) != cudaSuccess) { *err = PPC_ERR_CUDA; return false; }
      *cw = false;
    }
    return true;
  }

  ppc_status_t advance(bool* progressed) {
    StepBufs& sb = c->sb;
    while (i < ops.size()) {
      const int kind = ops[i].kind, m = ops[i].mb, d = kind;   // F travels FWD, B travels BWD
      const size_t bytes = kind == 0 ? st->fwd_bytes : st->bwd_bytes;
      const bool has_in = kind == 0 ? s > 0 : s < S - 1;
      const bool has_out = kind == 0 ? s < S - 1 : s > 0;
      const int bi = m & 1;
      // batched terminal receives: anything else that enqueues on the compute stream first
      // launches the pending batch (a fused source op enqueues nothing there)
      const bool batchable = batching && phase == 0 && terminal_recv(kind, m);
      if (batching && phase == 0 && !batchable && !fused_next)
        if (ppc_status_t fs = flush()) return fs;
      if (batchable) {
        void* dst = (kind == 0 ? st->y : st->dx)[m];
        ZcSend z;
        const bool fuse = fusable_next(&z);
        RecvArgs ra;
        if (ppc_status_t rs = ppc_impl_recv_prepare(c, (ppc_dir_t)d, dst, bytes, m, cs,
                                                    fuse ? &z.p : nullptr, &ra))
          return rs;
        pend.push_back(ra);
        pend_done.push_back({d, c->ch[d].recv_seq});
        if (fuse) {
          pend_commit.push_back(z);
          fused_next = true;
        }
        direct = true;
        in = dst;
        *progressed = true;
        phase = 1;
      }
      if (phase == 0) {                                  // input
        direct = false;
        if (has_in) {
          // terminal identity op with a device destination: receive straight into it
          void* const* dsts = kind == 0 ? st->y : st->dx;
          void* dst = (!has_out && !(kind == 0 ? st->fwd : st->bwd) && dsts) ? dsts[m] : nullptr;
          if (dst && is_host_ptr(dst)) dst = nullptr;
          uint8_t* r = dst ? static_cast<uint8_t*>(dst) : sb.rbuf[d][bi];
          if (dmode) {
            Mailbox& box = *inbox[d];
            if (box.empty()) return PPC_OK;                       // sender not there yet
            ppc_status_t e = PPC_OK;
            if (!dst && !reuse_ok(1, d, bi, &e)) return e;
            Pending p = box.front();
            if (p.bytes != bytes) return PPC_ERR_SIZE_MISMATCH;
            if (p.mb != m) return PPC_ERR_ORDER;
            box.pop_front();
            // with PPC_LOCAL_QUEUE the copy runs on the GPU's single transfer queue (xq);
            // the queue order (the round-robin enqueue order) respects every dependency
            cudaStream_t q = xq ? xq : cs;
            if (!dst)
              if (ppc_status_t w = before_write(1, d, bi, cs)) return w;
            if (xq) {
              CK(cudaEventRecord(sb.xgo, cs));
              CK(cudaStreamWaitEvent(xq, sb.xgo, 0));
            }
            CK(cudaStreamWaitEvent(q, p.ready, 0));
            const uint64_t ch = c->chunk;
            const int grid = env_int("PPC_COPY_CTAS", 296);   // 2 per SM (copy_kernel)
            if (ppc_status_t ts = time_mark(c, 0, q, true)) return ts;
            CK(launch_copy(r, p.src, bytes, ch, grid, q));
            if (ppc_status_t ts = time_mark(c, 0, q, false)) return ts;
            if (xq) {
              CK(cudaEventRecord(sb.xdone, xq));
              CK(cudaStreamWaitEvent(cs, sb.xdone, 0));
            }
            if (p.consumed) {
              CK(cudaEventRecord(p.consumed, cs));
              *p.held = false;
              *p.cwait = true;
            }
          } else {
            if (!dst && sb.rpending[d][bi]) CK(cudaStreamWaitEvent(cs, sb.rfree[d][bi], 0));
            if (!dst)
              if (ppc_status_t w = before_write(1, d, bi, cs)) return w;
            ZcSend z;
            const bool fuse = dst && fusable_next(&z);
            const bool chained = chain_op != (size_t)-1 && i == chain_op + 2;
            ppc_status_t rs = ppc_impl_recv_ex(c, (ppc_dir_t)d, r, bytes, m, cs,
                                               fuse ? &z.p : nullptr,
                                               chained ? &chain_prev : nullptr);
            if (rs == PPC_ERR_WOULD_BLOCK) return PPC_OK;
            if (rs) return rs;
            if (!dst) sb.rpending[d][bi] = false;
            chain_op = (size_t)-1;
            if (fuse) {   // the next op's send was published by this receive's kernel
              defer_commit(z);
              fused_next = true;
              chain_prev = {d, c->ch[d].recv_seq};   // dst: terminal, nothing follows on cs
              chain_op = i;
            }
          }
          direct = dst != nullptr;
          in = r;
        } else {
          const void* const* srcs = kind == 0 ? st->x : st->g;
          in = srcs ? srcs[m] : nullptr;
          if (in && is_host_ptr(in)) {
            // stage the host input on hs, ahead of the compute stream: wait only until the
            // staging buffer's previous contents are consumed (send done / copied by the next
            // virtual stage / read by this stage's fn / read by a device->host copy)
            uint8_t* r = sb.rbuf[d][bi];
            if (!sb.hs) CK(cudaStreamCreateWithFlags(&sb.hs, cudaStreamNonBlocking));
            cudaStream_t q = sb.hs;
            if (dmode) {
              ppc_status_t e = PPC_OK;
              if (!reuse_ok(1, d, bi, &e, q)) return e;
            } else if (sb.rpending[d][bi]) {
              CK(cudaStreamWaitEvent(q, sb.rfree[d][bi], 0));
            }
            sb.rpending[d][bi] = false;
            if (sb.rlast_set[d][bi]) {
              CK(cudaStreamWaitEvent(q, sb.rlast[d][bi], 0));
              sb.rlast_set[d][bi] = false;
            }
            if (ppc_status_t w = before_write(1, d, bi, q)) return w;
            CK(cudaMemcpyAsync(r, in, bytes, cudaMemcpyHostToDevice, q));
            CK(cudaEventRecord(sb.hdone[d][bi], q));
            CK(cudaStreamWaitEvent(cs, sb.hdone[d][bi], 0));
            in = r;
          }
        }
        *progressed = true;
        phase = 1;
      }
      if (phase == 1) {                                  // stage compute
        ppc_stage_fn fn = kind == 0 ? st->fwd : st->bwd;
        void* user = kind == 0 ? st->fwd_user : st->bwd_user;
        if (has_out && fn && bytes && c->step_inplace && !dmode && !c->capturing) {
          // produce in place: the stage fn writes the boundary tensor straight into the
          // receiver's ring slot (ppc_pp_send_begin / _end on the compute stream), so no
          // send pass re-reads it from HBM
          ppc_slot_t sl;
          ppc_status_t bs = ppc_pp_send_begin(c, (ppc_dir_t)d, bytes, m, cs, &sl);
          if (bs == PPC_ERR_WOULD_BLOCK) return PPC_OK;
          if (bs) return bs;
          if (fn(user, m, in, sl.payload, in ? bytes : 0, bytes, cs) != 0) return PPC_ERR_INVALID_ARG;
          mark_read(in, d, bi);
          if (ppc_status_t es = ppc_pp_send_end(c, (ppc_dir_t)d, 0, cs)) return es;
          inplace_sent = true;
        } else if (has_out) {
          if (fn || !in) {
            if (dmode) {
              ppc_status_t e = PPC_OK;
              if (!reuse_ok(2, d, bi, &e)) return e;
            } else if (sb.opending[d][bi]) {
              CK(cudaStreamWaitEvent(cs, sb.ofree[d][bi], 0));
            }
            uint8_t* o = sb.obuf[d][bi];
            if (ppc_status_t w = before_write(2, d, bi, cs)) return w;
            if (fn && fn(user, m, in, o, in ? bytes : 0, bytes, cs) != 0) return PPC_ERR_INVALID_ARG;
            mark_read(in, d, bi);
            send_src = o;          // no input and no fn: scratch contents
            send_free = sb.ofree[d][bi];
            send_pending = &sb.opending[d][bi];
            send_buf = 2;
          } else if (in == sb.rbuf[d][bi]) {
            send_src = in;
            send_free = sb.rfree[d][bi];
            send_pending = &sb.rpending[d][bi];
            send_buf = 1;
          } else {                                       // caller's device buffer
            send_src = in;
            send_free = nullptr;
            send_pending = nullptr;
            send_buf = 0;
          }
          // zero-copy sends publish from the send stream by default, so that the next op's
          // receive kernel is not queued behind the publication on the compute stream (it is
          // resident and spinning when its header lands); PPC_ZC_SIDE=0 publishes on the
          // compute stream instead.  Consumption is always awaited on the send stream.
          zc_send = !dmode && ppc_impl_is_zero_copy(c, send_src, bytes);
          zc_cs = zc_send && !c->zc_side;
          if (!dmode && !zc_cs) {
            CK(cudaEventRecord(sb.ready, cs));
            CK(cudaStreamWaitEvent(c->side[d], sb.ready, 0));
          }
        } else {
          void* const* dsts = kind == 0 ? st->y : st->dx;
          void* dst = dsts ? dsts[m] : nullptr;
          if (fn) {
            const bool host = dst && is_host_ptr(dst);
            if (dmode) {
              ppc_status_t e = PPC_OK;
              if (!reuse_ok(2, d, bi, &e)) return e;
            } else if (sb.opending[d][bi]) {
              CK(cudaStreamWaitEvent(cs, sb.ofree[d][bi], 0));
              sb.opending[d][bi] = false;
            }
            uint8_t* o = sb.obuf[d][bi];
            void* target = (dst && !host) ? dst : o;
            if (target == o)
              if (ppc_status_t w = before_write(2, d, bi, cs)) return w;
            if (fn(user, m, in, target, in ? bytes : 0, bytes, cs) != 0) return PPC_ERR_INVALID_ARG;
            mark_read(in, d, bi);
            if (host)
              if (ppc_status_t w = d2h(dst, o, bytes, 2, d, bi)) return w;
          } else if (dst && in && bytes && !direct) {
            if (is_host_ptr(dst)) {
              if (ppc_status_t w = d2h(dst, in, bytes, in == sb.rbuf[d][bi] ? 1 : 0, d, bi)) return w;
            } else {
              CK(cudaMemcpyAsync(dst, in, bytes, cudaMemcpyDefault, cs));
            }
          }
        }
        *progressed = true;
        phase = 2;
      }
      if (phase == 2) {                                  // send
        if (has_out && fused_next) {
          fused_next = false;                            // already published (fusion)
        } else if (has_out && inplace_sent) {
          inplace_sent = false;                          // produced into the slot
        } else if (has_out) {
          if (dmode) {
            // hand the buffer to the next stage: it makes the one copy
            cudaEvent_t rdy = sb.dready[d][bi];
            CK(cudaEventRecord(rdy, cs));
            Pending p{send_src, bytes, (long long)m, rdy, nullptr, nullptr, nullptr};
            if (send_buf == 1) {
              p.consumed = sb.cons_r[d][bi];
              p.held = &sb.held_r[d][bi];
              p.cwait = &sb.cwait_r[d][bi];
            } else if (send_buf == 2) {
              p.consumed = sb.cons_o[d][bi];
              p.held = &sb.held_o[d][bi];
              p.cwait = &sb.cwait_o[d][bi];
            }
            if (p.held) *p.held = true;
            outbox[d]->push_back(p);
          } else {
            // zero-copy: the buffer is free once consumed, awaited on zcw[d] off the
            // publication stream so the next publication is not queued behind it
            if (zc_send && !zc_cs && !c->zcw[d]) {      // first zero-copy send off cs
              int lo = 0, hi = 0;
              cudaDeviceGetStreamPriorityRange(&lo, &hi);
              CK(cudaStreamCreateWithPriority(&c->zcw[d], cudaStreamNonBlocking, hi));
            }
            cudaStream_t s_pub = zc_cs ? cs : c->side[d];
            cudaStream_t s_done = zc_send ? (zc_cs ? c->side[d] : c->zcw[d]) : c->side[d];
            if (zc_cs && send_buf == 0) {      // caller's buffer: publish now, commit at the end
              ZcSend z;
              if (ppc_status_t ps = ppc_impl_zc_prepare(c, (ppc_dir_t)d, send_src, bytes, m, &z))
                return ps;
              if (ppc_status_t ts = time_mark(c, 0, cs, true)) return ts;
              CK(launch_publish(z.p, cs));
              if (ppc_status_t ts = time_mark(c, 0, cs, false)) return ts;
              defer_commit(z);
              *progressed = true;
              phase = 0;
              ++i;
              continue;
            }
            ppc_status_t ss = ppc_impl_send_ex(c, (ppc_dir_t)d, send_src, bytes, m, s_pub, s_done);
            if (ss == PPC_ERR_WOULD_BLOCK) return PPC_OK;
            if (ss) return ss;
            if (s_done == c->zcw[d]) used_zcw[d] = true;
            if (send_free) {
              CK(cudaEventRecord(send_free, s_done));
              *send_pending = true;
            }
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
    if (ppc_status_t fs = flush()) return fs;
    for (int d = 0; d < 2; ++d)                  // the deferred rendezvous: one wait per dir
      if (has_last_commit[d]) {
        if (ppc_status_t ws = ppc_impl_zc_commit(c, last_commit[d], cs, c->side[d])) return ws;
        has_last_commit[d] = false;
      }
    if (used_ds) {                 // host outputs complete with the step
      CK(cudaEventRecord(c->sb.djoin, c->sb.ds));
      CK(cudaStreamWaitEvent(cs, c->sb.djoin, 0));
    }
    if (dmode) return PPC_OK;
    for (int d = 0; d < 2; ++d) {
      // join only the send streams this stage used (an unused one is not part of a graph
      // capture, and waiting on it from the capturing stream would be illegal)
      if (!(d == 0 ? s < S - 1 : s > 0)) continue;
      CK(cudaEventRecord(c->sb.join[d], c->side[d]));
      CK(cudaStreamWaitEvent(cs, c->sb.join[d], 0));
      if (used_zcw[d]) {
        CK(cudaEventRecord(c->sb.join[d], c->zcw[d]));
        CK(cudaStreamWaitEvent(cs, c->sb.join[d], 0));
      }
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
  sp.batching = env_int("PPC_STEP_BATCH", 0) != 0;
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
  bool same_device = true;
  for (int k = 0; k < S; ++k) {
    ppc_status_t r = check_live(comms[k]);
    if (r) return r;
    if (comms[k]->cfg.pp != S || comms[k]->pp_i != k) return PPC_ERR_INVALID_ARG;
    if (S > 1 && !comms[k]->local_mode) return PPC_ERR_INVALID_ARG;
    if (steps[k].M != steps[0].M) return PPC_ERR_INVALID_ARG;
    same_device = same_device && comms[k]->device == comms[0]->device;
    DeviceGuard g(comms[k]->device);
    if ((r = sp[k].init(comms[k], &steps[k], streams[k]))) return r;
  }
  // mailboxes of the direct (single-copy) mode: box[k][d] = messages into stage k, dir d
  std::vector<Mailbox> box(2 * S);
  const bool dmode = S > 1 && same_device && env_int("PPC_LOCAL_DIRECT", 1) != 0;
  cudaStream_t xq = nullptr;
  // PPC_LOCAL_QUEUE=1: all copies of the GPU on one transfer queue.  Measured slower than
  // letting each stage copy on its own stream (C2: 219 vs 188 us per step,
  // profiles/r34_n1_queue.jsonl): one 32 MiB copy alone does not saturate HBM, two
  // concurrent ones do.  Kept as an option; off by default.
  if (dmode && env_int("PPC_LOCAL_QUEUE", 0) != 0) {
    ppc_comm* c0 = comms[0];
    DeviceGuard g(c0->device);
    if (!c0->sb.xq) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      CK(cudaStreamCreateWithPriority(&c0->sb.xq, cudaStreamNonBlocking, hi));
    }
    xq = c0->sb.xq;
  }
  for (int k = 0; k < S && dmode; ++k) {
    sp[k].dmode = true;
    sp[k].xq = xq;
    sp[k].inbox[0] = &box[2 * k + 0];
    sp[k].inbox[1] = &box[2 * k + 1];
    sp[k].outbox[0] = k + 1 < S ? &box[2 * (k + 1) + 0] : nullptr;
    sp[k].outbox[1] = k > 0 ? &box[2 * (k - 1) + 1] : nullptr;
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
