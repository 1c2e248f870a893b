// Private definitions shared by the libppc host translation units (not part of the ABI).
#pragma once
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>
#include <cuda.h>
#include <nccl.h>
#include <unistd.h>

#include "ppc.h"
#include "ppc_internal.h"

using namespace ppc;

namespace ppc_impl {

constexpr uint32_t kBlobMagic = 0x50504342u;   // "BCPP"
constexpr uint32_t kBlobVersion = 1;
constexpr size_t kAlign = 4096;
constexpr int kTraceCap = 8192;
constexpr int kDbgCtas = 128;      // PPC_DBG_STAMPS: stamp rows per receive launch
constexpr int kDbgLaunches = 4096;

inline size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Blob {
  uint32_t magic, version;
  int32_t rank, world, device, pid;
  int32_t tp, pp, dp, K;
  uint64_t max_msg, chunk, arena_bytes;
  uint64_t host_hash;
  uint64_t arena_ptr;    // raw pointer (same-process mapping)
  uint64_t comm_ptr;     // ppc_comm* (same-process virtual stages)
  char busid[32];
  cudaIpcMemHandle_t ipc;
  int32_t has_arena;
  uint8_t pad[PPC_BLOB_BYTES - 4 * 2 - 4 * 8 - 8 * 6 - 32 - sizeof(cudaIpcMemHandle_t) - 4];
};
static_assert(sizeof(Blob) == PPC_BLOB_BYTES, "blob size");

// Byte offsets of this rank's shared arena (identical geometry on every rank).
struct Layout {
  size_t stride = 0;             // slot payload stride
  size_t payload[2] = {}, hdr[2] = {}, hdr_flag[2] = {}, flags[2] = {}, credit[2] = {},
         done[2] = {}, push_done[2] = {}, gdone[2] = {};
  size_t step = 0;               // step driver buffers: [recv|out][dir][2] x stride
  size_t total = 0;
  uint32_t max_chunks = 0;
  void build(int K, size_t max_msg, size_t chunk) {
    stride = round_up(std::max<size_t>(max_msg, 1), kAlign);
    max_chunks = (uint32_t)((max_msg + chunk - 1) / chunk);
    size_t off = 0;
    for (int d = 0; d < 2; ++d) { payload[d] = off; off += (size_t)K * stride; }
    // the step driver's receive / output buffers, so a middle stage can forward a message
    // zero-copy (the next stage pulls it from this arena, already mapped there)
    step = off;
    off += 8 * stride;
    for (int d = 0; d < 2; ++d) { hdr[d] = off; off = round_up(off + (size_t)K * 64, 256); }
    for (int d = 0; d < 2; ++d) { hdr_flag[d] = off; off = round_up(off + (size_t)K * 8, 256); }
    for (int d = 0; d < 2; ++d) {
      flags[d] = off;
      off = round_up(off + (size_t)K * std::max<uint32_t>(max_chunks, 1) * 8, 256);
    }
    for (int d = 0; d < 2; ++d) { credit[d] = off; off += 256; }
    // per slot: the receive's arrival counter, then (K further) its pull-unit claim counter
    for (int d = 0; d < 2; ++d) { done[d] = off; off = round_up(off + (size_t)K * 8, 256); }
    for (int d = 0; d < 2; ++d) { push_done[d] = off; off += 256; }
    // TP-sliced receives: receivers of one stage count finished pulls here (monotone)
    for (int d = 0; d < 2; ++d) { gdone[d] = off; off += 256; }
    total = round_up(off, kAlign);
  }
};

struct Chan {
  // sending side of direction d (we -> peer_out)
  int peer_out = -1;
  uint8_t* o_payload = nullptr;
  SlotHeader* o_hdr = nullptr;
  uint64_t* o_hdr_flag = nullptr;
  uint64_t* o_flags = nullptr;
  uint64_t* credit = nullptr;        // ours; the receiver writes it
  uint32_t* push_done = nullptr;
  uint64_t send_seq = 0;
  uint64_t open_seq = 0;             // ppc_pp_send_begin .. _end in progress (0 = none)
  uint32_t open_chunks = 0;
  ppc_record_t* open_rec = nullptr;
  ppc_comm* out_comm = nullptr;      // same-process peer
  // receiving side of direction d (peer_in -> we)
  int peer_in = -1;
  uint8_t* i_payload = nullptr;
  SlotHeader* i_hdr = nullptr;
  uint64_t* i_hdr_flag = nullptr;
  uint64_t* i_flags = nullptr;
  uint32_t* i_done = nullptr;
  uint64_t* peer_credit = nullptr;   // in the sender's arena
  const uint8_t* i_arena = nullptr;  // the sender's arena (zero-copy from its step buffers)
  uint64_t recv_seq = 0;
  ppc_comm* in_comm = nullptr;
  // virtual-stage mode: stream ordering through events
  std::vector<cudaEvent_t> sent_ev, recvd_ev;
};

struct StepBufs {
  size_t bytes = 0;
  uint8_t* rbuf[2][2] = {};     // [dir][i] recv landing
  uint8_t* obuf[2][2] = {};     // [dir][i] stage output
  uint8_t* hbuf[2][2] = {};     // [dir][i] staging for host inputs / outputs
  bool in_arena = false;        // rbuf / obuf are the arena's step region (not freed here)
  // device->host copies of terminal outputs run on ds (overlapping the next op's host->device
  // copy and transfers); dfree_[ro] = that copy finished reading rbuf / obuf [dir][i]
  cudaStream_t ds = nullptr;
  cudaEvent_t dgo = nullptr, djoin = nullptr, dfree_r[2][2] = {}, dfree_o[2][2] = {};
  bool dpend_r[2][2] = {}, dpend_o[2][2] = {};
  // host->device staging of host inputs runs ahead on hs: it waits only for the staging
  // buffer rbuf [dir][i] to be free (rfree / rlast / cons), not for the compute stream;
  // hdone = staged, rlast = the compute stream's last read of rbuf [dir][i] (a stage fn)
  cudaStream_t hs = nullptr;
  cudaEvent_t hdone[2][2] = {}, rlast[2][2] = {};
  bool rlast_set[2][2] = {};
  cudaEvent_t rfree[2][2] = {}, ofree[2][2] = {}, ready = nullptr, join[2] = {};
  bool rpending[2][2] = {}, opending[2][2] = {};
  // direct (single-copy) mode of same-GPU virtual stages: [dir][i] of the buffer handed to
  // the receiving stage; held = posted, receiver has not enqueued its copy yet;
  // cwait = copy enqueued, wait `cons` before overwriting
  cudaEvent_t dready[2][2] = {}, cons_r[2][2] = {}, cons_o[2][2] = {};
  bool held_r[2][2] = {}, held_o[2][2] = {}, cwait_r[2][2] = {}, cwait_o[2][2] = {};
  // direct mode, one transfer queue per GPU: xgo = the receiving stage is ready for the
  // copy (recorded on its stream), xdone = the copy finished (recorded on the queue)
  cudaEvent_t xgo = nullptr, xdone = nullptr;
  cudaStream_t xq = nullptr;    // the queue (owned by stage 0's comm; others borrow it)
};

}  // namespace ppc_impl

using namespace ppc_impl;

struct ppc_comm {
  ppc_config_t cfg{};
  int world = 0, rank = 0, device = -1;
  int pp_i = 0, dp_i = 0, tp_i = 0;
  int K = 2;
  size_t chunk = 1 << 20;
  unsigned long long timeout_ns = 10000000000ull;
  Layout lay;
  uint8_t* arena = nullptr;
  ErrHost* err_host = nullptr;     // mapped host record (polled by the host)
  ErrWord* err_dev = nullptr;      // device claim word + the record's device pointer
  // chained receives: per direction, the highest seq whose receive finished its data phase
  // (device memory, monotone); chain_* = the receive last enqueued by the step driver
  uint64_t* rchain = nullptr;
  bool recv_chain = true;          // PPC_RECV_CHAIN (default on)
  bool pub_b0 = true;              // PPC_PUB_BLOCK0: block 0 releases a fused publication
  bool pull_dyn = true;            // PPC_PULL_DYN: zero-copy pulls claim 4 KiB units per warp
  bool connected = false, poisoned = false, local_mode = false;
  bool sys_scope = true;   // a PP neighbour is another GPU: .sys fences, NVLink-sized grids
  int spin_cap = 64;       // max CTAs of a spinning grid (8 when a peer shares our GPU in
                           // this process: cfg.local_spin, every stage must stay resident)
  Chan ch[2];
  std::vector<void*> opened;          // IPC-opened peer arenas
  ncclComm_t nccl[2] = {nullptr, nullptr};
  std::vector<int> members[3];
  cudaStream_t side[2] = {nullptr, nullptr};   // send streams of the step driver
  cudaStream_t zcw[2] = {nullptr, nullptr};    // step driver: zero-copy consumption waits
  cudaStream_t gcw[2] = {nullptr, nullptr};    // TP-sliced gathers: credit releases
  cudaEvent_t g_ev[2] = {nullptr, nullptr};
  bool step_inplace = false;                   // step driver: stage fns produce into the slot
  bool zc_side = false;                        // step driver publishes zero-copy on side[d]
  bool fuse_publish = true;                    // step driver: publish from the prior receive
  bool zc_stepbufs = true;                     // step driver buffers are zero-copy sources
  // CE engine channel streams, one set per direction: a middle stage's FWD and BWD copies
  // must not queue behind each other (a FWD copy waiting for its credit would hold up the
  // BWD copy the other neighbour needs — a false dependency the 1F1B order does not have)
  cudaStream_t ce[2][8] = {};
  cudaEvent_t ce_fork[2] = {}, ce_join[2][8] = {};
  ppc_record_t* trace_dev = nullptr;
  int trace_n = 0;
  // cfg.trace bit 1: event pairs around send (0) / recv (1) launches
  std::vector<cudaEvent_t> tev[2];
  size_t tev_n[2] = {0, 0};
  StepBufs sb;
  uint8_t* hx_buf = nullptr;      // hetero allreduce receive scratch (max_msg bytes)
  // zero-copy registrations: mine (index = segment id) and the neighbours' mapped bases
  struct Reg { uintptr_t base; size_t size; };
  std::vector<Reg> regs;
  // device [2][tp][kMaxSeg]: side 0 = ranks of the previous stage (FWD in), 1 = next stage;
  // index tp_i of the sending rank (own PP neighbour = own tp_i)
  uint64_t* seg_tab = nullptr;
  std::vector<void*> reg_opened;
  std::vector<uint8_t*> tp_arena;   // arenas of this stage's TP group, by tp index (gather)
  // CUDA-graph capture (ppc_graph_create): sends / receives enqueued while capturing use
  // sequence numbers relative to cap_*; dseq = {send FWD, send BWD, recv FWD, recv BWD}
  // device bases, set before each graph launch
  cudaEvent_t zc_ev[2] = {nullptr, nullptr};   // publication -> rendezvous-wait stream
  uint64_t gcount[2] = {0, 0};                 // TP-sliced gathers received per direction
  bool capturing = false;
  uint64_t cap_send[2] = {0, 0}, cap_recv[2] = {0, 0};
  uint64_t* dseq = nullptr;
  // PPC_DBG_STAMPS: recv_kernel per-CTA stamps, kDbgCtas x 4 per launch, and per launch
  // (seq, dir, grid) on the host
  uint64_t* dbg = nullptr;
  std::vector<long long> dbg_meta;
  Blob blob{};
};

// A zero-copy send split in two (step driver fusion): the prepared publication, then the
// rendezvous wait for its consumption.
struct ZcSend {
  PublishArgs p;
  uint64_t target;          // credit to wait for (relative to *base when capturing)
  const uint64_t* base;
  ppc_dir_t d;
};

// internal entry points shared by the host translation units (not in the C ABI header)
extern "C" {
ppc_status_t ppc_impl_send_ex(ppc_comm_t* c, ppc_dir_t d, const void* buf, size_t bytes,
                              long long mb, cudaStream_t s, cudaStream_t s_wait);
int ppc_impl_is_zero_copy(const ppc_comm_t* c, const void* buf, size_t bytes);
// bookkeeping + publication arguments of a zero-copy send, without launching anything
ppc_status_t ppc_impl_zc_prepare(ppc_comm_t* c, ppc_dir_t d, const void* buf, size_t bytes,
                                 long long mb, ZcSend* z);
// rendezvous wait of a published zero-copy send on s_wait (after the work queued on s)
ppc_status_t ppc_impl_zc_commit(ppc_comm_t* c, const ZcSend& z, cudaStream_t s,
                                cudaStream_t s_wait);
// The receive a chained receive starts behind (its direction and absolute seq).
struct RecvChainRef {
  int dir;
  uint64_t seq;
};
// ppc_pp_recv whose kernel also publishes `pub` after completing (nullptr: plain receive).
// prev != nullptr: the caller guarantees that the last thing it enqueued on s is that
// receive's kernel (nothing in between), so this one may start on its posted completion.
ppc_status_t ppc_impl_recv_ex(ppc_comm_t* c, ppc_dir_t d, void* buf, size_t bytes,
                              long long mb, cudaStream_t s, const PublishArgs* pub,
                              const RecvChainRef* prev = nullptr);
// the same split in three: arguments + bookkeeping, one grid for n prepared receives, and
// the per-message completion bookkeeping (virtual stages: the recvd event)
ppc_status_t ppc_impl_recv_prepare(ppc_comm_t* c, ppc_dir_t d, void* buf, size_t bytes,
                                   long long mb, cudaStream_t s, const PublishArgs* pub,
                                   RecvArgs* out, const RecvChainRef* prev = nullptr);
ppc_status_t ppc_impl_recv_launch_batch(ppc_comm_t* c, const RecvArgs* as, int n,
                                        cudaStream_t s);
ppc_status_t ppc_impl_recv_done(ppc_comm_t* c, ppc_dir_t d, uint64_t seq, cudaStream_t s);
}

namespace ppc_impl {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (dev >= 0) {
      cudaGetDevice(&prev);
      if (prev != dev) cudaSetDevice(dev); else prev = -1;
    }
  }
  ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      if (getenv("PPC_DEBUG")) fprintf(stderr, "ppc: %s -> %s (%s:%d)\n", #x,     \
                                       cudaGetErrorString(e_), __FILE__, __LINE__); \
      return PPC_ERR_CUDA;                                                       \
    }                                                                            \
  } while (0)

inline uint64_t host_hash() {
  char h[256] = {};
  gethostname(h, sizeof(h) - 1);
  uint64_t x = 1469598103934665603ull;
  for (char* p = h; *p; ++p) x = (x ^ (uint8_t)*p) * 1099511628211ull;
  return x;
}

inline ppc_status_t check_live(ppc_comm* c) {
  if (!c || !c->connected) return PPC_ERR_STATE;
  if (c->poisoned) return PPC_ERR_STATE;
  if (c->err_host && ((volatile ErrHost*)c->err_host)->code != 0) {
    c->poisoned = true;
    return PPC_ERR_STATE;
  }
  return PPC_OK;
}

// cfg.trace bit 1: record the event opening (begin) / closing (!begin) a timed launch
inline ppc_status_t time_mark(ppc_comm* c, int kind, cudaStream_t s, bool begin) {
  if (!(c->cfg.trace & 2)) return PPC_OK;
  std::vector<cudaEvent_t>& v = c->tev[kind];
  size_t& n = c->tev_n[kind];
  if (begin && n + 2 > 2 * 4096) return PPC_OK;        // list full: stop timing
  if (!begin && (n & 1) == 0) return PPC_OK;           // begin was skipped
  if (n == v.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    v.push_back(e);
  }
  CK(cudaEventRecord(v[n], s));
  ++n;
  return PPC_OK;
}

inline int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}
// Send-side grid: SM push / PULL staging CTAs (MPDT channels x CTAs per channel).
inline int push_grid(const ppc_comm* c, uint32_t n_chunks) {
  if (n_chunks == 0) return 1;
  int per = c->cfg.cta_per_channel;
  int chans = std::max(1, c->cfg.channels);
  int g = per > 0 ? per * chans : (c->sys_scope ? c->spin_cap * chans : 296);
  if (c->cfg.engine == PPC_ENGINE_PULL && c->sys_scope)
    g = env_int("PPC_STAGE_CTAS", 128);          // local staging copy: HBM-bound, wide
  if (c->sys_scope) g = std::min(g, c->spin_cap * chans);
  return (int)std::max<uint32_t>(1, std::min<uint32_t>(n_chunks, (uint32_t)g));
}
// Receive-side grid: copy-out CTAs (SM/CE) or pulling CTAs (PULL).
inline int recv_grid(const ppc_comm* c, uint32_t n_chunks) {
  if (n_chunks == 0) return 1;
  int g = c->sys_scope ? 64 : 296;
  if (c->cfg.engine == PPC_ENGINE_PULL && c->sys_scope && c->cfg.cta_per_channel > 0)
    g = c->cfg.cta_per_channel * std::max(1, c->cfg.channels);      // the pulling CTAs
  g = env_int("PPC_RECV_CTAS", g);
  if (c->sys_scope) g = std::min(g, c->spin_cap);
  return (int)std::max<uint32_t>(1, std::min<uint32_t>(n_chunks, (uint32_t)g));
}

}  // namespace ppc_impl
