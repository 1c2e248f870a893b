// libppc host side: comm lifecycle (Resource Discovery / Topology Awareness, PAPER.md
// §2.2), DCBS groups, the pp_send / pp_recv enqueue logic
// (P:L53), the 1F1B step driver and diagnostics.  The host only enqueues: every
// wait on a peer happens on the device (flags/credits) or, for virtual stages sharing one
// GPU in one process, through CUDA events.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>
#include <unistd.h>

#include "ppc.h"
#include "ppc_internal.h"
#include "ppc_comm_impl.h"

using namespace ppc;

namespace {


ppc_record_t* next_record(ppc_comm* c) {
  // the kernel that stamps the times also writes the record's metadata
  if (!c->cfg.trace || !c->trace_dev || c->trace_n >= kTraceCap) return nullptr;
  return c->trace_dev + c->trace_n++;
}

struct RegBlob {
  uint32_t magic;
  int32_t rank, pid;
  uint32_t seg;
  uint64_t base, size, host_hash;
  cudaIpcMemHandle_t ipc;
  uint8_t pad[PPC_REG_BLOB_BYTES - 4 * 4 - 8 * 3 - sizeof(cudaIpcMemHandle_t)];
};
static_assert(sizeof(RegBlob) == PPC_REG_BLOB_BYTES, "reg blob size");
constexpr uint32_t kRegMagic = 0x52435050u;   // "PPCR"

// Allocation range of a device pointer (driver API through the runtime's entry point, so
// libppc does not link libcuda directly).
bool alloc_range(const void* p, uintptr_t* base, size_t* size) {
  using Fn = CUresult (*)(void*, CUpointer_attribute, CUdeviceptr);
  static Fn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuPointerGetAttribute", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f)
      return false;
    fn = reinterpret_cast<Fn>(f);
  }
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, (CUdeviceptr)(uintptr_t)p) != CUDA_SUCCESS ||
      fn(&sz, CU_POINTER_ATTRIBUTE_RANGE_SIZE, (CUdeviceptr)(uintptr_t)p) != CUDA_SUCCESS)
    return false;
  *base = (uintptr_t)b;
  *size = sz;
  return true;
}

// Zero-copy source lookup: index of the registered segment holding [p, p+bytes), or
// kArenaSeg for the step driver's buffers in our own arena (PPC_ZC_STEPBUFS), else -1.
int find_reg(const ppc_comm* c, const void* p, size_t bytes, uint64_t* off) {
  const uintptr_t a = (uintptr_t)p;
  if (c->arena && c->zc_stepbufs) {
    const uintptr_t s0 = (uintptr_t)c->arena + c->lay.step;
    if (a >= s0 && a + bytes <= s0 + 8 * c->lay.stride) {
      *off = a - (uintptr_t)c->arena;
      return (int)kArenaSeg;
    }
  }
  for (size_t i = 0; i < c->regs.size(); ++i) {
    const auto& r = c->regs[i];
    if (a >= r.base && a + bytes <= r.base + r.size) {
      *off = a - r.base;
      return (int)i;
    }
  }
  return -1;
}
}  // namespace

extern "C" {

size_t ppc_struct_size(int which) {
  switch (which) {
    case 0: return sizeof(ppc_config_t);
    case 1: return sizeof(ppc_step_t);
    case 2: return sizeof(ppc_record_t);
    case 3: return sizeof(ppc_op_t);
    case 4: return sizeof(ppc_slot_t);
  }
  return 0;
}

const char* ppc_status_str(ppc_status_t st) {
  switch (st) {
    case PPC_OK: return "PPC_OK";
    case PPC_ERR_INVALID_ARG: return "PPC_ERR_INVALID_ARG";
    case PPC_ERR_GRID_MISMATCH: return "PPC_ERR_GRID_MISMATCH";
    case PPC_ERR_RANK_OUT_OF_RANGE: return "PPC_ERR_RANK_OUT_OF_RANGE";
    case PPC_ERR_SELF_SEND: return "PPC_ERR_SELF_SEND";
    case PPC_ERR_NO_NEIGHBOR: return "PPC_ERR_NO_NEIGHBOR";
    case PPC_ERR_TOO_LARGE: return "PPC_ERR_TOO_LARGE";
    case PPC_ERR_SIZE_MISMATCH: return "PPC_ERR_SIZE_MISMATCH";
    case PPC_ERR_ORDER: return "PPC_ERR_ORDER";
    case PPC_ERR_TIMEOUT: return "PPC_ERR_TIMEOUT";
    case PPC_ERR_BACKEND: return "PPC_ERR_BACKEND";
    case PPC_ERR_CUDA: return "PPC_ERR_CUDA";
    case PPC_ERR_NCCL: return "PPC_ERR_NCCL";
    case PPC_ERR_STATE: return "PPC_ERR_STATE";
    case PPC_ERR_WOULD_BLOCK: return "PPC_ERR_WOULD_BLOCK";
  }
  return "PPC_ERR_UNKNOWN";
}

ppc_status_t ppc_schedule_1f1b(int S, int s, int M, ppc_op_t* ops, int* n_ops) {
  if (S < 1 || s < 0 || s >= S || M < 1 || !ops || !n_ops) return PPC_ERR_INVALID_ARG;
  const int w = std::min(S - s - 1, M);
  int n = 0;
  for (int m = 0; m < w; ++m) ops[n++] = {0, m};
  for (int i = 0; i < M - w; ++i) {
    ops[n++] = {0, w + i};
    ops[n++] = {1, i};
  }
  for (int m = M - w; m < M; ++m) ops[n++] = {1, m};
  *n_ops = n;
  return PPC_OK;
}

ppc_status_t ppc_create(const ppc_config_t* cfg, int world, int rank, int cuda_device,
                        ppc_comm_t** out) {
  if (!cfg || !out) return PPC_ERR_INVALID_ARG;
  *out = nullptr;
  if (world < 1) return PPC_ERR_INVALID_ARG;
  if (cfg->tp < 1 || cfg->pp < 1 || cfg->dp < 1 || cfg->tp * cfg->pp * cfg->dp != world)
    return PPC_ERR_GRID_MISMATCH;
  if (rank < 0 || rank >= world) return PPC_ERR_RANK_OUT_OF_RANGE;
  if (cfg->ring_slots < 0 || cfg->ring_slots > kMaxSlots || cfg->channels < 0 ||
      cfg->channels > 8 || cfg->cta_per_channel < 0 || cfg->cta_per_channel > 1024 ||
      (cfg->engine != PPC_ENGINE_SM && cfg->engine != PPC_ENGINE_CE &&
       cfg->engine != PPC_ENGINE_PULL) ||
      (cfg->chunk_bytes % 4096) != 0 || cfg->max_msg_bytes == 0 ||
      cfg->max_msg_bytes > (1ull << 40))
    return PPC_ERR_INVALID_ARG;
  ppc_comm* c = new ppc_comm();
  c->cfg = *cfg;
  c->world = world;
  c->rank = rank;
  c->device = cuda_device;
  // default K = pp + 1: under 1F1B stage s never has more than min(S - s, M) unconsumed
  // messages per boundary, so sends never wait for a slot
  c->K = cfg->ring_slots ? cfg->ring_slots : std::min(cfg->pp + 1, kMaxSlots);
  c->chunk = cfg->chunk_bytes ? cfg->chunk_bytes : (1u << 20);
  c->timeout_ns = cfg->timeout_ns ? cfg->timeout_ns : 10000000000ull;
  if (c->cfg.channels == 0) c->cfg.channels = 1;
  c->zc_side = env_int("PPC_ZC_SIDE", 0) != 0;
  c->fuse_publish = env_int("PPC_FUSE_PUBLISH", 1) != 0;
  c->recv_chain = env_int("PPC_RECV_CHAIN", 1) != 0;
  c->pub_b0 = env_int("PPC_PUB_BLOCK0", 1) != 0;
  c->pull_dyn = env_int("PPC_PULL_DYN", 1) != 0;
  c->zc_stepbufs = env_int("PPC_ZC_STEPBUFS", 1) != 0;
  c->step_inplace = env_int("PPC_STEP_INPLACE", 0) != 0;
  ppc::g_pdl = env_int("PPC_PDL", 1) != 0 ? 1 : 0;
  ppc::g_recv_early = env_int("PPC_RECV_EARLY", 0) != 0 ? 1 : 0;
  ppc::g_copy_tma_ctas = std::max(0, env_int("PPC_COPY_TMA_CTAS", 0));
  ppc::g_wait_value = env_int("PPC_WAIT_VALUE", 0) != 0 ? 1 : 0;
  ppc::kMaxSpinGrid = std::max(1, env_int("PPC_SPIN_GRID_CAP", 64));
  c->spin_cap = ppc::kMaxSpinGrid;
  const int tp = cfg->tp, dp = cfg->dp;
  c->pp_i = rank / (tp * dp);
  c->dp_i = (rank % (tp * dp)) / tp;
  c->tp_i = rank % tp;
  for (int t = 0; t < tp; ++t) c->members[PPC_GROUP_TP].push_back(c->pp_i * tp * dp + c->dp_i * tp + t);
  for (int d = 0; d < dp; ++d) c->members[PPC_GROUP_DP].push_back(c->pp_i * tp * dp + d * tp + c->tp_i);
  for (int p = 0; p < cfg->pp; ++p) c->members[PPC_GROUP_PP].push_back(p * tp * dp + c->dp_i * tp + c->tp_i);
  c->lay.build(c->K, cfg->max_msg_bytes, c->chunk);

  Blob& b = c->blob;
  memset(&b, 0, sizeof(b));
  b.magic = kBlobMagic;
  b.version = kBlobVersion;
  b.rank = rank;
  b.world = world;
  b.device = cuda_device;
  b.pid = (int32_t)getpid();
  b.tp = cfg->tp; b.pp = cfg->pp; b.dp = cfg->dp; b.K = c->K;
  b.max_msg = cfg->max_msg_bytes;
  b.chunk = c->chunk;
  b.arena_bytes = c->lay.total;
  b.host_hash = host_hash();
  b.comm_ptr = (uint64_t)(uintptr_t)c;

  if (cuda_device >= 0) {
    DeviceGuard g(cuda_device);
    auto fail = [&](ppc_status_t st) { ppc_destroy(c); return st; };
    if (cudaSetDevice(cuda_device) != cudaSuccess) return fail(PPC_ERR_CUDA);
    if (preload_kernels() != cudaSuccess) return fail(PPC_ERR_CUDA);   // no lazy loads later
    if (cudaMalloc(&c->arena, c->lay.total) != cudaSuccess) return fail(PPC_ERR_CUDA);
    if (cudaMemset(c->arena, 0, c->lay.total) != cudaSuccess) return fail(PPC_ERR_CUDA);
    // the same for the driver's device-to-device copy (CE engine, host staging): its first
    // use must not be a lazy load that waits for a device on which a receive is spinning
    if (cudaMemcpy(c->arena + c->lay.step, c->arena, 64, cudaMemcpyDeviceToDevice) != cudaSuccess)
      return fail(PPC_ERR_CUDA);
    if (cudaHostAlloc(&c->err_host, sizeof(ErrHost), cudaHostAllocMapped) != cudaSuccess)
      return fail(PPC_ERR_CUDA);
    memset(c->err_host, 0, sizeof(ErrHost));
    {
      ErrWord w{};
      if (cudaHostGetDevicePointer((void**)&w.host, c->err_host, 0) != cudaSuccess ||
          cudaMalloc(&c->err_dev, sizeof(ErrWord)) != cudaSuccess ||
          cudaMemcpy(c->err_dev, &w, sizeof(w), cudaMemcpyHostToDevice) != cudaSuccess)
        return fail(PPC_ERR_CUDA);
    }
    if (cudaMalloc(&c->rchain, 2 * sizeof(uint64_t)) != cudaSuccess ||
        cudaMemset(c->rchain, 0, 2 * sizeof(uint64_t)) != cudaSuccess)
      return fail(PPC_ERR_CUDA);
    if (cudaIpcGetMemHandle(&b.ipc, c->arena) != cudaSuccess) return fail(PPC_ERR_CUDA);
    if (cudaDeviceGetPCIBusId(b.busid, sizeof(b.busid), cuda_device) != cudaSuccess)
      return fail(PPC_ERR_CUDA);
    // send streams (side, CE channels) are created in ppc_connect for the directions that
    // have a neighbour, the zero-copy wait streams on first use: a process that drives many
    // comms (virtual stages) must stay under CUDA_DEVICE_MAX_CONNECTIONS hardware queues, or
    // aliased streams add false dependencies behind spinning kernels
    if (cfg->trace && cudaMalloc(&c->trace_dev, sizeof(ppc_record_t) * kTraceCap) != cudaSuccess)
      return fail(PPC_ERR_CUDA);
    if (env_int("PPC_DBG_STAMPS", 0)) {
      const size_t nb = sizeof(uint64_t) * 4 * kDbgCtas * kDbgLaunches;
      if (cudaMalloc(&c->dbg, nb) != cudaSuccess || cudaMemset(c->dbg, 0, nb) != cudaSuccess)
        return fail(PPC_ERR_CUDA);
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return fail(PPC_ERR_CUDA);
    b.arena_ptr = (uint64_t)(uintptr_t)c->arena;
    b.has_arena = 1;
  }
  *out = c;
  return PPC_OK;
}

ppc_status_t ppc_export(ppc_comm_t* c, void* blob, size_t* blob_bytes) {
  if (!c || !blob_bytes) return PPC_ERR_INVALID_ARG;
  if (!blob) {
    *blob_bytes = PPC_BLOB_BYTES;
    return PPC_OK;
  }
  if (*blob_bytes < PPC_BLOB_BYTES) return PPC_ERR_INVALID_ARG;
  memcpy(blob, &c->blob, PPC_BLOB_BYTES);
  *blob_bytes = PPC_BLOB_BYTES;
  return PPC_OK;
}

ppc_status_t ppc_nccl_unique_id(void* out128) {
  if (!out128) return PPC_ERR_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return PPC_ERR_NCCL;
  static_assert(sizeof(id) == 128, "nccl id");
  memcpy(out128, &id, 128);
  return PPC_OK;
}

static ppc_status_t map_peer(ppc_comm* c, const Blob& pb, uint8_t** base) {
  if (!pb.has_arena) return PPC_ERR_STATE;
  if (pb.pid == c->blob.pid && pb.host_hash == c->blob.host_hash) {
    *base = (uint8_t*)(uintptr_t)pb.arena_ptr;      // same process: raw UVA pointer
    return PPC_OK;
  }
  void* p = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, pb.ipc, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    if (getenv("PPC_DEBUG")) fprintf(stderr, "ppc: IPC open rank %d: %s\n", pb.rank, cudaGetErrorString(e));
    return PPC_ERR_CUDA;
  }
  c->opened.push_back(p);
  *base = (uint8_t*)p;
  return PPC_OK;
}

ppc_status_t ppc_connect(ppc_comm_t* c, const void* all_blobs, size_t blob_bytes,
                         const void* nccl_ids, int n_ids) {
  if (!c || !all_blobs || blob_bytes != PPC_BLOB_BYTES || n_ids < 0 || n_ids > 2 ||
      (n_ids > 0 && !nccl_ids))
    return PPC_ERR_INVALID_ARG;
  if (c->connected) return PPC_ERR_STATE;
  const Blob* B = static_cast<const Blob*>(all_blobs);
  for (int r = 0; r < c->world; ++r) {
    const Blob& b = B[r];
    if (b.magic != kBlobMagic || b.version != kBlobVersion || b.world != c->world ||
        b.tp != c->cfg.tp || b.pp != c->cfg.pp || b.dp != c->cfg.dp || b.K != c->K ||
        b.max_msg != c->cfg.max_msg_bytes || b.chunk != c->chunk)
      return PPC_ERR_INVALID_ARG;
    if (b.rank != r) return PPC_ERR_RANK_OUT_OF_RANGE;
  }
  const int tpdp = c->cfg.tp * c->cfg.dp;
  const int prev = c->pp_i > 0 ? c->rank - tpdp : -1;
  const int next = c->pp_i < c->cfg.pp - 1 ? c->rank + tpdp : -1;
  for (int nb : {prev, next}) {
    if (nb < 0) continue;
    const Blob& pb = B[nb];
    if (pb.comm_ptr == c->blob.comm_ptr && pb.pid == c->blob.pid &&
        pb.host_hash == c->blob.host_hash)
      return PPC_ERR_SELF_SEND;
  }
  c->ch[PPC_FWD].peer_out = next;
  c->ch[PPC_FWD].peer_in = prev;
  c->ch[PPC_BWD].peer_out = prev;
  c->ch[PPC_BWD].peer_in = next;
  if (c->device >= 0) {
    DeviceGuard g(c->device);
    // same-process neighbours <=> virtual stages on one GPU (events order the streams)
    int same = 0, cross = 0;
    for (int nb : {prev, next}) {
      if (nb < 0) continue;
      if (B[nb].pid == c->blob.pid && B[nb].host_hash == c->blob.host_hash) ++same; else ++cross;
    }
    if (same && cross) return PPC_ERR_INVALID_ARG;
    // cfg.local_spin: same-process neighbours run the cross-process protocol (device spins)
    c->local_mode = same > 0 && !c->cfg.local_spin;
    // virtual stages may also sit on different GPUs of this process (used to profile the
    // NVLink push without cross-process spins): enable peer access, keep .sys scope
    c->sys_scope = !c->local_mode;
    // a spinning grid must never starve the peer it waits for: stages of this process that
    // share our GPU get small spinning grids (other processes time-slice the GPU instead)
    for (int r = 0; r < c->world; ++r)
      if (r != c->rank && B[r].pid == c->blob.pid && B[r].host_hash == c->blob.host_hash &&
          B[r].device == c->device)
        c->spin_cap = 8;
    for (int nb : {prev, next}) {
      if (nb < 0 || B[nb].pid != c->blob.pid || B[nb].host_hash != c->blob.host_hash ||
          B[nb].device == c->device)
        continue;
      c->sys_scope = true;
      cudaError_t e = cudaDeviceEnablePeerAccess(B[nb].device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else CK(e);
    }
    uint8_t* base_prev = nullptr;
    uint8_t* base_next = nullptr;
    if (prev >= 0) { ppc_status_t st = map_peer(c, B[prev], &base_prev); if (st) return st; }
    if (next >= 0) { ppc_status_t st = map_peer(c, B[next], &base_next); if (st) return st; }
    // TP group of this stage: their arenas hold the headers of the slices they receive
    // (TP-sliced gathers, ppc_pp_recv_gather)
    c->tp_arena.assign(c->cfg.tp, nullptr);
    for (int t = 0; t < c->cfg.tp; ++t) {
      const int r = c->members[PPC_GROUP_TP][t];
      if (r == c->rank) { c->tp_arena[t] = c->arena; continue; }
      ppc_status_t st = map_peer(c, B[r], &c->tp_arena[t]);
      if (st) return st;
    }
    const Layout& L = c->lay;
    for (int d = 0; d < 2; ++d) {
      Chan& h = c->ch[d];
      uint8_t* ob = (h.peer_out == next) ? base_next : base_prev;
      uint8_t* ib = (h.peer_in == next) ? base_next : base_prev;
      h.credit = (uint64_t*)(c->arena + L.credit[d]);
      h.push_done = (uint32_t*)(c->arena + L.push_done[d]);
      if (h.peer_out >= 0) {
        // PULL: the ring slot of an outgoing message lives in the SENDER's arena
        h.o_payload = (c->cfg.engine == PPC_ENGINE_PULL ? c->arena : ob) + L.payload[d];
        h.o_hdr = (SlotHeader*)(ob + L.hdr[d]);
        h.o_hdr_flag = (uint64_t*)(ob + L.hdr_flag[d]);
        h.o_flags = (uint64_t*)(ob + L.flags[d]);
        if (c->local_mode) h.out_comm = (ppc_comm*)(uintptr_t)B[h.peer_out].comm_ptr;
      }
      if (h.peer_in >= 0) {
        h.i_payload = (c->cfg.engine == PPC_ENGINE_PULL ? ib : c->arena) + L.payload[d];
        h.i_hdr = (SlotHeader*)(c->arena + L.hdr[d]);
        h.i_hdr_flag = (uint64_t*)(c->arena + L.hdr_flag[d]);
        h.i_flags = (uint64_t*)(c->arena + L.flags[d]);
        h.i_done = (uint32_t*)(c->arena + L.done[d]);
        h.peer_credit = (uint64_t*)(ib + L.credit[d]);
        h.i_arena = ib;
        if (c->local_mode) h.in_comm = (ppc_comm*)(uintptr_t)B[h.peer_in].comm_ptr;
      }
      if (c->local_mode) {
        h.sent_ev.assign(c->K, nullptr);
        h.recvd_ev.assign(c->K, nullptr);
        for (int k = 0; k < c->K; ++k) {
          CK(cudaEventCreateWithFlags(&h.sent_ev[k], cudaEventDisableTiming));
          CK(cudaEventCreateWithFlags(&h.recvd_ev[k], cudaEventDisableTiming));
        }
      }
    }
    {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      for (int d = 0; d < 2; ++d) {
        if (c->ch[d].peer_out < 0) continue;
        if (!c->side[d]) CK(cudaStreamCreateWithPriority(&c->side[d], cudaStreamNonBlocking, hi));
        if (c->cfg.engine != PPC_ENGINE_CE) continue;
        for (int i = 0; i < c->cfg.channels; ++i) {
          if (!c->ce[d][i]) CK(cudaStreamCreateWithPriority(&c->ce[d][i], cudaStreamNonBlocking, hi));
          if (!c->ce_join[d][i]) CK(cudaEventCreateWithFlags(&c->ce_join[d][i], cudaEventDisableTiming));
        }
        if (!c->ce_fork[d]) CK(cudaEventCreateWithFlags(&c->ce_fork[d], cudaEventDisableTiming));
      }
    }
    // DCBS: TP and DP groups on NCCL; PP stays on the peer kernels
    const ncclUniqueId* ids = static_cast<const ncclUniqueId*>(nccl_ids);
    for (int gi = 0; gi < n_ids; ++gi) {
      const std::vector<int>& mem = c->members[gi];
      // PPC_NCCL_SINGLETON=1 (tests): a one-rank group gets its own one-rank communicator
      // too, so the NCCL init and allreduce path runs where ranks share one GPU (NCCL
      // refuses two ranks of one communicator on one GPU); a zero id = no communicator
      static const ncclUniqueId kZero{};
      if (mem.size() < 2 && (!env_int("PPC_NCCL_SINGLETON", 0) ||
                             memcmp(&ids[gi], &kZero, sizeof(kZero)) == 0))
        continue;
      const int r = (int)(std::find(mem.begin(), mem.end(), c->rank) - mem.begin());
      if (ncclCommInitRank(&c->nccl[gi], (int)mem.size(), ids[gi], r) != ncclSuccess)
        return PPC_ERR_NCCL;
    }
  }
  c->connected = true;
  return PPC_OK;
}

ppc_status_t ppc_group(const ppc_comm_t* c, ppc_group_t g, int* members, int* n,
                       ppc_backend_t* backend) {
  if (!c || !n || g < PPC_GROUP_TP || g > PPC_GROUP_PP) return PPC_ERR_INVALID_ARG;
  const std::vector<int>& m = c->members[g];
  if (members) {
    if (*n < (int)m.size()) return PPC_ERR_INVALID_ARG;
    std::copy(m.begin(), m.end(), members);
  }
  *n = (int)m.size();
  if (backend) *backend = g == PPC_GROUP_PP ? PPC_BACKEND_PEER : PPC_BACKEND_NCCL;
  return PPC_OK;
}

int ppc_impl_is_zero_copy(const ppc_comm_t* c, const void* buf, size_t bytes) {
  uint64_t off = 0;
  return c && !c->local_mode && bytes > 0 && buf && find_reg(c, buf, bytes, &off) != -1;
}

}  // extern "C"

namespace {
// Publication of zero-copy send `seq` (the record times the publication; the receiver's
// record times the data).
void fill_publish(ppc_comm* c, ppc_dir_t d, uint64_t seq, uint64_t need, size_t bytes,
                  long long mb, int zc_seg, uint64_t zc_off, ppc_record_t* rec, ZcSend* z) {
  Chan& h = c->ch[d];
  const int slot = (int)(seq % c->K);
  PublishArgs& p = z->p;
  p = PublishArgs{};
  p.rec = rec;
  p.rec_src = c->rank;
  p.rec_dst = h.peer_out;
  p.hdr = h.o_hdr + slot;
  p.hdr_flag = h.o_hdr_flag + slot;
  p.credit = h.credit;
  p.need_credit = need;
  p.bytes = bytes;
  p.seq = seq;
  p.src_off = zc_off;
  p.mb = mb;
  p.src_seg = (uint32_t)zc_seg;
  p.dir = d;
  p.boundary = (uint32_t)(d == PPC_FWD ? c->pp_i : c->pp_i - 1);
  static const int gpu_fence = [] {
    const char* v = getenv("PPC_PUB_FENCE");
    return v && strcmp(v, "gpu") == 0 ? 1 : 0;
  }();
  p.gpu_fence = (uint32_t)gpu_fence;
  p.err = c->err_dev;
  p.timeout_ns = c->timeout_ns;
  z->d = d;
  z->base = nullptr;
  z->target = seq;
  if (c->capturing) {             // graph: relative seq, slot resolved on device
    z->base = c->dseq + d;
    p.sr = {z->base, 0, (uint32_t)c->K, 0, c->local_mode ? 0u : 1u, 0};
    p.seq = z->target = seq - c->cap_send[d];
    p.hdr = h.o_hdr;
    p.hdr_flag = h.o_hdr_flag;
  }
}
}  // namespace

extern "C" {

ppc_status_t ppc_impl_zc_commit(ppc_comm_t* c, const ZcSend& z, cudaStream_t s,
                                cudaStream_t s_wait) {
  if (s_wait != s) {
    if (!c->zc_ev[z.d]) CK(cudaEventCreateWithFlags(&c->zc_ev[z.d], cudaEventDisableTiming));
    CK(cudaEventRecord(c->zc_ev[z.d], s));
    CK(cudaStreamWaitEvent(s_wait, c->zc_ev[z.d], 0));
  }
  // rendezvous: the buffer may be reused once the receiver consumed it
  CK(launch_wait_credit(c->ch[z.d].credit, z.target, c->err_dev, c->timeout_ns, s_wait, z.base));
  return PPC_OK;
}

ppc_status_t ppc_impl_zc_prepare(ppc_comm_t* c, ppc_dir_t d, const void* buf, size_t bytes,
                                 long long mb, ZcSend* z) {
  ppc_status_t st = check_live(c);
  if (st) return st;
  if (d != PPC_FWD && d != PPC_BWD) return PPC_ERR_INVALID_ARG;
  if (mb < 0 || bytes == 0 || !buf || !z) return PPC_ERR_INVALID_ARG;
  Chan& h = c->ch[d];
  if (h.peer_out < 0) return PPC_ERR_NO_NEIGHBOR;
  if (bytes > c->cfg.max_msg_bytes) return PPC_ERR_TOO_LARGE;
  if (c->device < 0 || c->local_mode || h.open_seq) return PPC_ERR_STATE;
  uint64_t zc_off = 0;
  const int zc_seg = find_reg(c, buf, bytes, &zc_off);
  if (zc_seg == -1) return PPC_ERR_INVALID_ARG;
  const uint64_t seq = h.send_seq + 1;
  const uint64_t need = seq > (uint64_t)c->K ? seq - c->K : 0;
  fill_publish(c, d, seq, need, bytes, mb, zc_seg, zc_off, next_record(c), z);
  h.send_seq = seq;
  return PPC_OK;
}

ppc_status_t ppc_pp_send(ppc_comm_t* c, ppc_dir_t d, const void* buf, size_t bytes,
                         long long mb, cudaStream_t s) {
  return ppc_impl_send_ex(c, d, buf, bytes, mb, s, s);
}

// s: the data mover / publication; s_wait: the zero-copy rendezvous wait (the step driver
// publishes on its send stream and waits for consumption on a third stream, ppc_step.cu)
ppc_status_t ppc_impl_send_ex(ppc_comm_t* c, ppc_dir_t d, const void* buf, size_t bytes,
                              long long mb, cudaStream_t s, cudaStream_t s_wait) {
  ppc_status_t st = check_live(c);
  if (st) return st;
  if (d != PPC_FWD && d != PPC_BWD) return PPC_ERR_INVALID_ARG;
  if (mb < 0 || (bytes > 0 && !buf)) return PPC_ERR_INVALID_ARG;
  Chan& h = c->ch[d];
  if (h.peer_out < 0) return PPC_ERR_NO_NEIGHBOR;
  if (bytes > c->cfg.max_msg_bytes) return PPC_ERR_TOO_LARGE;
  if (c->device < 0 || h.open_seq) return PPC_ERR_STATE;
  DeviceGuard g(c->device);
  const uint64_t seq = h.send_seq + 1;
  const int slot = (int)(seq % c->K);
  uint64_t need = seq > (uint64_t)c->K ? seq - c->K : 0;
  if (c->local_mode) {
    if (need) {
      Chan& rh = h.out_comm->ch[d];
      if (rh.recv_seq < need) return PPC_ERR_WOULD_BLOCK;
      // while capturing a graph, a recv enqueued before the capture belongs to an earlier
      // (already serialised) launch: no edge
      if (!(c->capturing && need <= h.out_comm->cap_recv[d]))
        CK(cudaStreamWaitEvent(s, rh.recvd_ev[slot], 0));
    }
    need = 0;   // ordered by the event; the kernel does not spin on the same GPU
  }
  const uint32_t n_chunks = (uint32_t)((bytes + c->chunk - 1) / c->chunk);
  const int boundary = d == PPC_FWD ? c->pp_i : c->pp_i - 1;
  ppc_record_t* rec = next_record(c);
  uint8_t* dst = h.o_payload + (size_t)slot * c->lay.stride;
  uint64_t* flags = h.o_flags + (size_t)slot * std::max<uint32_t>(c->lay.max_chunks, 1);
  if (ppc_status_t ts = time_mark(c, 0, s, true)) return ts;
  uint64_t zc_off = 0;
  const int zc_seg = (!c->local_mode && bytes > 0) ? find_reg(c, buf, bytes, &zc_off) : -1;
  if (zc_seg != -1) {              // registered buffer: publish it, the receiver pulls it
    ZcSend z;
    fill_publish(c, d, seq, need, bytes, mb, zc_seg, zc_off, rec, &z);
    CK(launch_publish(z.p, s));
    // public call with cfg.zc_async: complete at publication (ppc_pp_wait_consumed waits)
    const bool async = c->cfg.zc_async && s_wait == s;
    if (!async)
      if (ppc_status_t ws = ppc_impl_zc_commit(c, z, s, s_wait)) return ws;
  } else if (c->cfg.engine != PPC_ENGINE_CE || bytes == 0) {  // SM push, or PULL's staging
    PushArgs a{};
    a.src = static_cast<const uint8_t*>(buf);
    a.dst = dst;
    a.hdr = h.o_hdr + slot;
    a.hdr_flag = h.o_hdr_flag + slot;
    a.flags = flags;
    a.credit = h.credit;
    a.need_credit = need;
    a.bytes = bytes;
    a.chunk = c->chunk;
    a.n_chunks = n_chunks;
    a.seq = seq;
    a.mb = mb;
    a.step = 0;
    a.dir = d;
    a.boundary = (uint32_t)boundary;
    a.err = c->err_dev;
    a.timeout_ns = c->timeout_ns;
    a.rec = rec;
    a.rec_src = c->rank;
    a.rec_dst = h.peer_out;
    a.done = h.push_done;
    a.channels = (uint32_t)std::max(1, c->cfg.channels);
    if (c->capturing) {           // graph: relative seq, slot resolved on device
      a.sr = {c->dseq + d, (uint64_t)c->lay.stride, (uint32_t)c->K,
              std::max<uint32_t>(c->lay.max_chunks, 1), c->local_mode ? 0u : 1u, 0};
      a.seq = seq - c->cap_send[d];
      a.dst = h.o_payload;
      a.hdr = h.o_hdr;
      a.hdr_flag = h.o_hdr_flag;
      a.flags = h.o_flags;
    }
    CK(launch_push(a, push_grid(c, n_chunks), c->sys_scope, env_int("PPC_PUSH_WS", 1) != 0, s));
  } else {
    if (c->capturing) return PPC_ERR_INVALID_ARG;       // CE copies are not graph-relocatable
    CeHeadArgs a{};
    a.hdr = h.o_hdr + slot;
    a.hdr_flag = h.o_hdr_flag + slot;
    a.credit = h.credit;
    a.need_credit = need;
    a.bytes = bytes;
    a.seq = seq;
    a.step = 0;
    a.mb = mb;
    a.dir = d;
    a.boundary = (uint32_t)boundary;
    a.err = c->err_dev;
    a.timeout_ns = c->timeout_ns;
    a.rec = rec;
    a.rec_src = c->rank;
    a.rec_dst = h.peer_out;
    CK(launch_ce_head(a, s));
    CK(cudaEventRecord(c->ce_fork[d], s));
    const int C = std::min<int>(c->cfg.channels, (int)n_chunks);
    for (int i = 0; i < C; ++i) {
      const uint32_t c0 = (uint32_t)((uint64_t)n_chunks * i / C);
      const uint32_t c1 = (uint32_t)((uint64_t)n_chunks * (i + 1) / C);
      const size_t off = (size_t)c0 * c->chunk;
      const size_t len = std::min<size_t>((size_t)c1 * c->chunk, bytes) - off;
      CK(cudaStreamWaitEvent(c->ce[d][i], c->ce_fork[d], 0));
      CK(cudaMemcpyAsync(dst + off, static_cast<const uint8_t*>(buf) + off, len,
                         cudaMemcpyDeviceToDevice, c->ce[d][i]));
      CK(launch_ce_flags(flags, c0, c1, seq, i == C - 1 ? rec : nullptr, c->ce[d][i]));
      CK(cudaEventRecord(c->ce_join[d][i], c->ce[d][i]));
      CK(cudaStreamWaitEvent(s, c->ce_join[d][i], 0));
    }
  }
  // zero-copy: the send completes when the receiver has pulled it (on s_wait)
  if (ppc_status_t ts = time_mark(c, 0, zc_seg >= 0 ? s_wait : s, false)) return ts;
  h.send_seq = seq;
  if (c->local_mode) CK(cudaEventRecord(h.sent_ev[slot], s));
  return PPC_OK;
}

// Produce-in-place send (ppc.h): the CE engine's signalling (credit + header kernel before,
// flags kernel after) around the caller's producer kernels instead of a copy.
ppc_status_t ppc_pp_send_begin(ppc_comm_t* c, ppc_dir_t d, size_t bytes, long long mb,
                               cudaStream_t s, ppc_slot_t* out) {
  ppc_status_t st = check_live(c);
  if (st) return st;
  if (d != PPC_FWD && d != PPC_BWD) return PPC_ERR_INVALID_ARG;
  if (mb < 0 || bytes == 0 || !out) return PPC_ERR_INVALID_ARG;
  Chan& h = c->ch[d];
  if (h.peer_out < 0) return PPC_ERR_NO_NEIGHBOR;
  if (bytes > c->cfg.max_msg_bytes) return PPC_ERR_TOO_LARGE;
  if (c->device < 0 || h.open_seq) return PPC_ERR_STATE;
  if (c->capturing) return PPC_ERR_INVALID_ARG;
  DeviceGuard g(c->device);
  const uint64_t seq = h.send_seq + 1;
  const int slot = (int)(seq % c->K);
  uint64_t need = seq > (uint64_t)c->K ? seq - c->K : 0;
  if (c->local_mode) {
    if (need) {
      Chan& rh = h.out_comm->ch[d];
      if (rh.recv_seq < need) return PPC_ERR_WOULD_BLOCK;
      CK(cudaStreamWaitEvent(s, rh.recvd_ev[slot], 0));
    }
    need = 0;
  }
  const uint32_t n_chunks = (uint32_t)((bytes + c->chunk - 1) / c->chunk);
  CeHeadArgs a{};
  a.hdr = h.o_hdr + slot;
  a.hdr_flag = h.o_hdr_flag + slot;
  a.credit = h.credit;
  a.need_credit = need;
  a.bytes = bytes;
  a.seq = seq;
  a.step = 0;
  a.mb = mb;
  a.dir = d;
  a.boundary = (uint32_t)(d == PPC_FWD ? c->pp_i : c->pp_i - 1);
  a.err = c->err_dev;
  a.timeout_ns = c->timeout_ns;
  a.rec = next_record(c);
  a.rec_src = c->rank;
  a.rec_dst = h.peer_out;
  CK(launch_ce_head(a, s, true));
  out->payload = h.o_payload + (size_t)slot * c->lay.stride;
  out->flags = reinterpret_cast<unsigned long long*>(
      h.o_flags + (size_t)slot * std::max<uint32_t>(c->lay.max_chunks, 1));
  out->seq = seq;
  out->bytes = bytes;
  out->chunk_bytes = c->chunk;
  out->n_chunks = n_chunks;
  h.open_seq = seq;
  h.open_chunks = n_chunks;
  h.open_rec = a.rec;
  return PPC_OK;
}

ppc_status_t ppc_pp_send_end(ppc_comm_t* c, ppc_dir_t d, int flags_released, cudaStream_t s) {
  ppc_status_t st = check_live(c);
  if (st) return st;
  if (d != PPC_FWD && d != PPC_BWD) return PPC_ERR_INVALID_ARG;
  Chan& h = c->ch[d];
  if (!h.open_seq) return PPC_ERR_STATE;
  DeviceGuard g(c->device);
  const uint64_t seq = h.open_seq;
  const int slot = (int)(seq % c->K);
  uint64_t* flags = h.o_flags + (size_t)slot * std::max<uint32_t>(c->lay.max_chunks, 1);
  if (!flags_released || h.open_rec)       // flags, or just the trace end stamp
    CK(launch_ce_flags(flags, 0, flags_released ? 0 : h.open_chunks, seq, h.open_rec, s, true));
  h.send_seq = seq;
  h.open_seq = 0;
  h.open_rec = nullptr;
  if (c->local_mode) CK(cudaEventRecord(h.sent_ev[slot], s));
  return PPC_OK;
}

ppc_status_t ppc_pp_recv(ppc_comm_t* c, ppc_dir_t d, void* buf, size_t bytes, long long mb,
                         cudaStream_t s) {
  return ppc_impl_recv_ex(c, d, buf, bytes, mb, s, nullptr);
}

// Arguments of the next receive of direction d (bookkeeping included: recv_seq advances,
// trace record taken).  pub != nullptr: the receive kernel also publishes that (prepared)
// zero-copy send once this receive has completed (step driver fusion, ppc_step.cu).
// Virtual stages: the stream waits for the matching send's event first.
ppc_status_t ppc_impl_recv_prepare(ppc_comm_t* c, ppc_dir_t d, void* buf, size_t bytes,
                                   long long mb, cudaStream_t s, const PublishArgs* pub,
                                   RecvArgs* out, const RecvChainRef* prev) {
  ppc_status_t st = check_live(c);
  if (st) return st;
  if (d != PPC_FWD && d != PPC_BWD) return PPC_ERR_INVALID_ARG;
  if (mb < 0 || (bytes > 0 && !buf)) return PPC_ERR_INVALID_ARG;
  Chan& h = c->ch[d];
  if (h.peer_in < 0) return PPC_ERR_NO_NEIGHBOR;
  if (bytes > c->cfg.max_msg_bytes) return PPC_ERR_TOO_LARGE;
  if (c->device < 0) return PPC_ERR_STATE;
  if (pub && c->local_mode) return PPC_ERR_STATE;
  const uint64_t seq = h.recv_seq + 1;
  const int slot = (int)(seq % c->K);
  if (c->local_mode) {
    Chan& sh = h.in_comm->ch[d];
    if (sh.send_seq < seq) return PPC_ERR_WOULD_BLOCK;
    if (!(c->capturing && seq <= h.in_comm->cap_send[d]))
      CK(cudaStreamWaitEvent(s, sh.sent_ev[slot], 0));
  }
  const uint32_t n_chunks = (uint32_t)((bytes + c->chunk - 1) / c->chunk);
  RecvArgs& a = *out;
  a = RecvArgs{};
  a.dst = static_cast<uint8_t*>(buf);
  a.src = h.i_payload + (size_t)slot * c->lay.stride;
  a.hdr = h.i_hdr + slot;
  a.hdr_flag = h.i_hdr_flag + slot;
  a.flags = h.i_flags + (size_t)slot * std::max<uint32_t>(c->lay.max_chunks, 1);
  a.peer_credit = h.peer_credit;
  a.done = h.i_done + slot;
  a.next = h.i_done + c->K + slot;
  a.dyn = c->pull_dyn ? 1u : 0u;
  a.bytes = bytes;
  a.chunk = c->chunk;
  a.n_chunks = n_chunks;
  a.seq = seq;
  a.mb = mb;
  a.err = c->err_dev;
  a.timeout_ns = c->timeout_ns;
  a.rec = next_record(c);
  a.rec_src = h.peer_in;
  a.rec_dst = c->rank;
  a.seg_tab = c->seg_tab
      ? c->seg_tab + ((size_t)(d == PPC_FWD ? 0 : 1) * c->cfg.tp + c->tp_i) * kMaxSeg : nullptr;
  a.peer_arena = h.i_arena;
  a.channels = c->cfg.engine == PPC_ENGINE_CE ? 1u : (uint32_t)std::max(1, c->cfg.channels);
  if (pub) {
    a.has_pub = 1;
    a.pub_b0 = c->pub_b0 ? 1u : 0u;
    a.pub = *pub;
  }
  if (c->recv_chain && !c->local_mode) {
    a.chain_post = c->rchain + d;
    if (prev && c->cfg.engine != PPC_ENGINE_CE) {
      a.chain_wait = c->rchain + prev->dir;
      a.chain_seq = prev->seq;
      if (c->capturing) {         // the predecessor's seq relative to its graph base
        if (prev->seq <= c->cap_recv[prev->dir]) {
          a.chain_wait = nullptr;   // captured before this graph: plain PDL wait
        } else {
          a.chain_base = c->dseq + 2 + prev->dir;
          a.chain_seq = prev->seq - c->cap_recv[prev->dir];
        }
      }
    }
  }
  if (c->capturing) {             // graph: relative seq, slot resolved on device
    a.sr = {c->dseq + 2 + d, (uint64_t)c->lay.stride, (uint32_t)c->K,
            std::max<uint32_t>(c->lay.max_chunks, 1), 0, 0};
    a.seq = seq - c->cap_recv[d];
    a.src = h.i_payload;
    a.hdr = h.i_hdr;
    a.hdr_flag = h.i_hdr_flag;
    a.flags = h.i_flags;
    a.done = h.i_done;
    a.next = h.i_done + c->K;
  }
  if (c->dbg && c->dbg_meta.size() / 3 < (size_t)kDbgLaunches) {   // graph: last replay's
    a.dbg = c->dbg + (c->dbg_meta.size() / 3) * 4 * kDbgCtas;
    c->dbg_meta.push_back((long long)seq);
    c->dbg_meta.push_back(d);
    c->dbg_meta.push_back(std::min<long long>(recv_grid(c, n_chunks) + (pub ? 1 : 0), kDbgCtas));
  }
  h.recv_seq = seq;
  return PPC_OK;
}

// After the receive kernel of direction d (seq = the channel's current recv_seq) is enqueued.
ppc_status_t ppc_impl_recv_done(ppc_comm_t* c, ppc_dir_t d, uint64_t seq, cudaStream_t s) {
  if (c->local_mode) CK(cudaEventRecord(c->ch[d].recvd_ev[seq % c->K], s));
  return PPC_OK;
}

ppc_status_t ppc_impl_recv_ex(ppc_comm_t* c, ppc_dir_t d, void* buf, size_t bytes,
                              long long mb, cudaStream_t s, const PublishArgs* pub,
                              const RecvChainRef* prev) {
  if (!c) return PPC_ERR_STATE;
  DeviceGuard g(c->device);
  RecvArgs a;
  ppc_status_t st = ppc_impl_recv_prepare(c, d, buf, bytes, mb, s, pub, &a, prev);
  if (st) return st;
  if (ppc_status_t ts = time_mark(c, 1, s, true)) return ts;
  CK(launch_recv(a, recv_grid(c, a.n_chunks), c->sys_scope, s));
  if (ppc_status_t ts = time_mark(c, 1, s, false)) return ts;
  return ppc_impl_recv_done(c, d, c->ch[d].recv_seq, s);
}

// A batch of prepared receives (each possibly with a fused publication) in ONE grid.
ppc_status_t ppc_impl_recv_launch_batch(ppc_comm_t* c, const RecvArgs* as, int n,
                                        cudaStream_t s) {
  if (n < 1 || n > kMaxBatch) return PPC_ERR_INVALID_ARG;
  DeviceGuard g(c->device);
  static thread_local RecvBatch b;       // ~6 KiB: kept off the stack
  b.n = (uint32_t)n;
  uint32_t max_chunks = 1;
  for (int i = 0; i < n; ++i) {
    b.a[i] = as[i];
    max_chunks = std::max(max_chunks, as[i].n_chunks);
  }
  if (ppc_status_t ts = time_mark(c, 1, s, true)) return ts;
  CK(launch_recv_batch(b, recv_grid(c, max_chunks), c->sys_scope, s));
  if (ppc_status_t ts = time_mark(c, 1, s, false)) return ts;
  return PPC_OK;
}

ppc_status_t ppc_pp_recv_batch(ppc_comm_t* c, ppc_dir_t d, void* const* bufs,
                               const size_t* bytes, int n, long long mb0, cudaStream_t s) {
  ppc_status_t st = check_live(c);
  if (st) return st;
  if (d != PPC_FWD && d != PPC_BWD) return PPC_ERR_INVALID_ARG;
  if (n < 1 || n > kMaxBatch || !bufs || !bytes || mb0 < 0) return PPC_ERR_INVALID_ARG;
  Chan& h = c->ch[d];
  if (h.peer_in < 0) return PPC_ERR_NO_NEIGHBOR;
  for (int i = 0; i < n; ++i) {        // every argument error before anything is enqueued
    if (bytes[i] > 0 && !bufs[i]) return PPC_ERR_INVALID_ARG;
    if (bytes[i] > c->cfg.max_msg_bytes) return PPC_ERR_TOO_LARGE;
  }
  if (c->device < 0) return PPC_ERR_STATE;
  if (c->local_mode && h.in_comm->ch[d].send_seq < h.recv_seq + n) return PPC_ERR_WOULD_BLOCK;
  DeviceGuard g(c->device);
  RecvArgs as[kMaxBatch];
  for (int i = 0; i < n; ++i)
    if ((st = ppc_impl_recv_prepare(c, d, bufs[i], bytes[i], mb0 + i, s, nullptr, &as[i])))
      return st;
  if ((st = ppc_impl_recv_launch_batch(c, as, n, s))) return st;
  for (int i = 0; i < n; ++i)
    if ((st = ppc_impl_recv_done(c, d, h.recv_seq - n + 1 + i, s))) return st;
  return PPC_OK;
}

ppc_status_t ppc_pp_recv_gather(ppc_comm_t* c, ppc_dir_t d, void* buf, size_t total_bytes,
                                long long mb, cudaStream_t s) {
  ppc_status_t st = check_live(c);
  if (st) return st;
  if (d != PPC_FWD && d != PPC_BWD) return PPC_ERR_INVALID_ARG;
  const int tp = c->cfg.tp;
  if (mb < 0 || !buf || total_bytes == 0 || total_bytes % tp != 0 || tp > kMaxTp)
    return PPC_ERR_INVALID_ARG;
  Chan& h = c->ch[d];
  if (h.peer_in < 0) return PPC_ERR_NO_NEIGHBOR;
  const size_t slice = total_bytes / tp;
  if (slice > c->cfg.max_msg_bytes) return PPC_ERR_TOO_LARGE;
  if (c->device < 0 || c->local_mode || c->capturing) return PPC_ERR_STATE;
  if (!c->seg_tab || (int)c->tp_arena.size() != tp) return PPC_ERR_STATE;   // no imports
  DeviceGuard g(c->device);
  const uint64_t seq = h.recv_seq + 1;
  const int slot = (int)(seq % c->K);
  const Layout& L = c->lay;
  const int side = d == PPC_FWD ? 0 : 1;
  GatherArgs a{};
  a.dst = static_cast<uint8_t*>(buf);
  a.slice_bytes = slice;
  a.chunk = c->chunk;
  a.n_chunks = (uint32_t)((slice + c->chunk - 1) / c->chunk);
  a.tp = (uint32_t)tp;
  a.my_tp = (uint32_t)c->tp_i;
  a.seq = seq;
  a.gtarget = (uint64_t)tp * (c->gcount[d] + 1);
  a.mb = mb;
  for (int t = 0; t < tp; ++t) {
    uint8_t* ar = c->tp_arena[t];
    a.hdr[t] = reinterpret_cast<const SlotHeader*>(ar + L.hdr[d]) + slot;
    a.hdr_flag[t] = reinterpret_cast<const uint64_t*>(ar + L.hdr_flag[d]) + slot;
    a.seg_tab[t] = c->seg_tab + ((size_t)side * tp + t) * kMaxSeg;
    a.gdone[t] = reinterpret_cast<unsigned long long*>(ar + L.gdone[d]);
  }
  a.peer_credit = h.peer_credit;
  a.done = h.i_done + slot;
  a.err = c->err_dev;
  a.timeout_ns = c->timeout_ns;
  const int grid = (int)std::max<uint32_t>(1, std::min<uint32_t>(a.tp * a.n_chunks, (uint32_t)c->spin_cap));
  if (ppc_status_t ts = time_mark(c, 1, s, true)) return ts;
  CK(launch_gather(a, grid, s));
  if (ppc_status_t ts = time_mark(c, 1, s, false)) return ts;
  // the credit waits for the OTHER receivers' pulls of our sender's slice: on the direction's
  // side stream (after this gather), not on s
  if (!c->gcw[d]) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    CK(cudaStreamCreateWithPriority(&c->gcw[d], cudaStreamNonBlocking, hi));
  }
  if (!c->g_ev[d]) CK(cudaEventCreateWithFlags(&c->g_ev[d], cudaEventDisableTiming));
  CK(cudaEventRecord(c->g_ev[d], s));
  CK(cudaStreamWaitEvent(c->gcw[d], c->g_ev[d], 0));
  CK(launch_gather_credit(a, c->gcw[d]));
  h.recv_seq = seq;
  c->gcount[d] += 1;
  return PPC_OK;
}

ppc_status_t ppc_pp_wait_consumed(ppc_comm_t* c, ppc_dir_t d, cudaStream_t s) {
  ppc_status_t st = check_live(c);
  if (st) return st;
  if (d != PPC_FWD && d != PPC_BWD) return PPC_ERR_INVALID_ARG;
  Chan& h = c->ch[d];
  if (h.peer_out < 0) return PPC_ERR_NO_NEIGHBOR;
  if (c->device < 0) return PPC_ERR_STATE;
  if (h.send_seq == 0) return PPC_OK;
  DeviceGuard g(c->device);
  if (c->local_mode) {
    Chan& rh = h.out_comm->ch[d];
    if (rh.recv_seq < h.send_seq) return PPC_ERR_WOULD_BLOCK;
    if (!(c->capturing && h.send_seq <= h.out_comm->cap_recv[d]))
      CK(cudaStreamWaitEvent(s, rh.recvd_ev[h.send_seq % c->K], 0));
    return PPC_OK;
  }
  if (c->capturing)
    CK(launch_wait_credit(h.credit, h.send_seq - c->cap_send[d], c->err_dev, c->timeout_ns, s,
                          c->dseq + d));
  else
    CK(launch_wait_credit(h.credit, h.send_seq, c->err_dev, c->timeout_ns, s));
  return PPC_OK;
}

ppc_status_t ppc_allreduce(ppc_comm_t* c, ppc_group_t g, void* buf, size_t count,
                           int nccl_dtype, cudaStream_t s) {
  ppc_status_t st = check_live(c);
  if (st) return st;
  if (g == PPC_GROUP_PP) return PPC_ERR_BACKEND;      // DCBS: PP is not a collective group
  if (g != PPC_GROUP_TP && g != PPC_GROUP_DP) return PPC_ERR_INVALID_ARG;
  if (count && !buf) return PPC_ERR_INVALID_ARG;
  if (count == 0) return PPC_OK;
  if (c->members[g].size() < 2 && !c->nccl[g]) return PPC_OK;    // group of one: identity
  if (!c->nccl[g]) return PPC_ERR_STATE;
  DeviceGuard gd(c->device);
  if (ncclAllReduce(buf, buf, count, (ncclDataType_t)nccl_dtype, ncclSum, c->nccl[g], s) !=
      ncclSuccess)
    return PPC_ERR_NCCL;
  return PPC_OK;
}


ppc_status_t ppc_register(ppc_comm_t* c, const void* ptr, size_t bytes, void* blob,
                          size_t* blob_bytes) {
  if (!c || !ptr || !blob || !blob_bytes || *blob_bytes < PPC_REG_BLOB_BYTES)
    return PPC_ERR_INVALID_ARG;
  if (c->device < 0) return PPC_ERR_STATE;
  DeviceGuard g(c->device);
  uintptr_t base = 0;
  size_t size = 0;
  if (!alloc_range(ptr, &base, &size) || (uintptr_t)ptr + bytes > base + size)
    return PPC_ERR_INVALID_ARG;
  RegBlob rb{};
  rb.magic = kRegMagic;
  rb.rank = c->rank;
  rb.pid = c->blob.pid;
  rb.host_hash = c->blob.host_hash;
  rb.base = base;
  rb.size = size;
  int seg = -1;
  for (size_t i = 0; i < c->regs.size(); ++i)
    if (c->regs[i].base == base) seg = (int)i;
  if (seg < 0) {
    if ((int)c->regs.size() >= kMaxSeg) return PPC_ERR_TOO_LARGE;
    seg = (int)c->regs.size();
    c->regs.push_back({base, size});
  }
  rb.seg = (uint32_t)seg;
  CK(cudaIpcGetMemHandle(&rb.ipc, (void*)base));
  memcpy(blob, &rb, sizeof(rb));
  *blob_bytes = PPC_REG_BLOB_BYTES;
  return PPC_OK;
}

ppc_status_t ppc_register_import(ppc_comm_t* c, const void* blob, size_t blob_bytes) {
  if (!c || !blob || blob_bytes != PPC_REG_BLOB_BYTES) return PPC_ERR_INVALID_ARG;
  if (!c->connected || c->device < 0) return PPC_ERR_STATE;
  RegBlob rb;
  memcpy(&rb, blob, sizeof(rb));
  if (rb.magic != kRegMagic || rb.seg >= (uint32_t)kMaxSeg || rb.rank < 0 || rb.rank >= c->world)
    return PPC_ERR_INVALID_ARG;
  // senders we may pull from: every rank of an adjacent stage with our dp index (its own PP
  // neighbour, or a TP peer of it for TP-sliced gathers)
  const int tp = c->cfg.tp, dp = c->cfg.dp;
  const int r_pp = rb.rank / (tp * dp), r_dp = (rb.rank % (tp * dp)) / tp, r_tp = rb.rank % tp;
  const int side = r_dp != c->dp_i ? -1 : (r_pp == c->pp_i - 1 ? 0 : (r_pp == c->pp_i + 1 ? 1 : -1));
  if (side < 0) return PPC_OK;                                   // not an adjacent stage
  DeviceGuard g(c->device);
  const size_t tab = (size_t)2 * tp * kMaxSeg * sizeof(uint64_t);
  if (!c->seg_tab) {
    CK(cudaMalloc(&c->seg_tab, tab));
    CK(cudaMemset(c->seg_tab, 0, tab));
  }
  uint64_t mapped = 0;
  if (rb.pid == c->blob.pid && rb.host_hash == c->blob.host_hash) {
    mapped = rb.base;                                            // same process: UVA pointer
  } else {
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, rb.ipc, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      if (getenv("PPC_DEBUG")) fprintf(stderr, "ppc: reg import %s\n", cudaGetErrorString(e));
      return PPC_ERR_CUDA;
    }
    c->reg_opened.push_back(p);
    mapped = (uint64_t)(uintptr_t)p;
  }
  CK(cudaMemcpy(c->seg_tab + ((size_t)side * tp + r_tp) * kMaxSeg + rb.seg, &mapped,
                sizeof(mapped), cudaMemcpyHostToDevice));
  return PPC_OK;
}

ppc_status_t ppc_hetero_allreduce(ppc_comm_t* c, void* buf, size_t count, int nccl_dtype,
                                  cudaStream_t s) {
  ppc_status_t st = check_live(c);
  if (st) return st;
  if (c->device < 0 || c->local_mode) return PPC_ERR_STATE;
  int kind, esize;
  switch (nccl_dtype) {
    case ncclFloat32: kind = 0; esize = 4; break;
    case ncclFloat16: kind = 1; esize = 2; break;
    case ncclBfloat16: kind = 2; esize = 2; break;
    case ncclInt32: kind = 3; esize = 4; break;
    default: return PPC_ERR_INVALID_ARG;
  }
  if (count == 0) return PPC_OK;
  if (!buf) return PPC_ERR_INVALID_ARG;
  const size_t bytes = count * (size_t)esize;
  if (bytes > c->cfg.max_msg_bytes) return PPC_ERR_TOO_LARGE;
  DeviceGuard g(c->device);
  const bool multi_dp = c->members[PPC_GROUP_DP].size() > 1;
  if (multi_dp && !c->nccl[PPC_GROUP_DP]) return PPC_ERR_STATE;
  // (1) intra-subgroup aggregation with the vendor CCL
  if (multi_dp && ncclAllReduce(buf, buf, count, (ncclDataType_t)nccl_dtype, ncclSum,
                                c->nccl[PPC_GROUP_DP], s) != ncclSuccess)
    return PPC_ERR_NCCL;
  // (2) cross-subgroup exchange of the intermediate results between leaders, P2P path
  const int S = c->cfg.pp, sidx = c->pp_i;
  const long long tag = 0x7FFFFFFFll;
  if (c->dp_i == 0 && S > 1) {
    if (!c->hx_buf) CK(cudaMalloc(&c->hx_buf, c->cfg.max_msg_bytes));
    if (sidx > 0) {                                   // partial sum of stages < sidx
      if ((st = ppc_pp_recv(c, PPC_FWD, c->hx_buf, bytes, tag, s))) return st;
      CK(launch_add(buf, c->hx_buf, count, kind, s));
    }
    if (sidx < S - 1) {
      if ((st = ppc_pp_send(c, PPC_FWD, buf, bytes, tag, s))) return st;
      if ((st = ppc_pp_recv(c, PPC_BWD, buf, bytes, tag, s))) return st;   // the total
    }
    if (sidx > 0 && (st = ppc_pp_send(c, PPC_BWD, buf, bytes, tag, s))) return st;
  }
  // (3) intra-subgroup broadcast from the leader (DP rank 0)
  if (multi_dp && ncclBroadcast(buf, buf, count, (ncclDataType_t)nccl_dtype, 0,
                                c->nccl[PPC_GROUP_DP], s) != ncclSuccess)
    return PPC_ERR_NCCL;
  return PPC_OK;
}

ppc_status_t ppc_error_info(ppc_comm_t* c, unsigned* seq, unsigned* info) {
  if (!c || !seq || !info) return PPC_ERR_INVALID_ARG;
  if (!c->err_host) { *seq = *info = 0; return PPC_OK; }
  const volatile ErrHost* e = c->err_host;
  *seq = e->seq;
  *info = e->info;
  return (ppc_status_t)e->code;
}

ppc_status_t ppc_poll(ppc_comm_t* c) {
  if (!c) return PPC_ERR_INVALID_ARG;
  if (!c->err_host) return PPC_OK;
  const unsigned code = ((volatile ErrHost*)c->err_host)->code;
  if (code) c->poisoned = true;
  return (ppc_status_t)code;
}

ppc_status_t ppc_trace(ppc_comm_t* c, ppc_record_t* out, int* n) {
  if (!c || !n || (*n > 0 && !out)) return PPC_ERR_INVALID_ARG;
  if (!c->trace_dev) { *n = 0; return PPC_OK; }
  DeviceGuard g(c->device);
  CK(cudaDeviceSynchronize());
  const int k = std::min(*n, c->trace_n);
  if (k > 0) CK(cudaMemcpy(out, c->trace_dev, sizeof(ppc_record_t) * k, cudaMemcpyDeviceToHost));
  *n = k;
  return PPC_OK;
}

ppc_status_t ppc_debug_stamps(ppc_comm_t* c, unsigned long long* stamps, long long* meta,
                              int* n) {
  if (!c || !n || (*n > 0 && (!stamps || !meta))) return PPC_ERR_INVALID_ARG;
  if (!c->dbg) { *n = 0; return PPC_OK; }
  DeviceGuard g(c->device);
  CK(cudaDeviceSynchronize());
  const int k = std::min(*n, (int)(c->dbg_meta.size() / 3));
  if (k > 0) {
    CK(cudaMemcpy(stamps, c->dbg, sizeof(uint64_t) * 4 * kDbgCtas * k, cudaMemcpyDeviceToHost));
    std::copy(c->dbg_meta.begin(), c->dbg_meta.begin() + 3 * k, meta);
  }
  *n = k;
  return PPC_OK;
}

ppc_status_t ppc_kernel_times(ppc_comm_t* c, int kind, float* ms, int* n) {
  if (!c || !n || (kind != 0 && kind != 1) || (*n > 0 && !ms)) return PPC_ERR_INVALID_ARG;
  if (c->device < 0) { *n = 0; return PPC_OK; }
  DeviceGuard g(c->device);
  CK(cudaDeviceSynchronize());
  const int pairs = (int)(c->tev_n[kind] / 2);
  const int k = std::min(*n, pairs);
  for (int i = 0; i < k; ++i)
    CK(cudaEventElapsedTime(&ms[i], c->tev[kind][2 * i], c->tev[kind][2 * i + 1]));
  c->tev_n[kind] = 0;
  *n = k;
  return PPC_OK;
}

ppc_status_t ppc_set_trace(ppc_comm_t* c, int trace) {
  if (!c || trace < 0 || trace > 3) return PPC_ERR_INVALID_ARG;
  if ((trace & 1) && !c->trace_dev) return PPC_ERR_STATE;
  c->cfg.trace = trace;
  return PPC_OK;
}

ppc_status_t ppc_disconnect(ppc_comm_t* c) {
  if (!c) return PPC_ERR_INVALID_ARG;
  DeviceGuard g(c->device);
  if (c->device >= 0) cudaDeviceSynchronize();
  for (int i = 0; i < 2; ++i)
    if (c->nccl[i]) { ncclCommDestroy(c->nccl[i]); c->nccl[i] = nullptr; }
  for (void* p : c->reg_opened) cudaIpcCloseMemHandle(p);
  c->reg_opened.clear();
  for (void* p : c->opened) cudaIpcCloseMemHandle(p);
  c->opened.clear();
  for (int d = 0; d < 2; ++d) {
    for (cudaEvent_t e : c->ch[d].sent_ev) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ch[d].recvd_ev) if (e) cudaEventDestroy(e);
    c->ch[d].sent_ev.clear();
    c->ch[d].recvd_ev.clear();
  }
  c->connected = false;
  return PPC_OK;
}

ppc_status_t ppc_destroy(ppc_comm_t* c) {
  if (!c) return PPC_ERR_INVALID_ARG;
  if (c->connected) ppc_disconnect(c);
  if (c->device >= 0) {
    DeviceGuard g(c->device);
    cudaDeviceSynchronize();
    StepBufs& sb = c->sb;
    for (int d = 0; d < 2; ++d)
      for (int i = 0; i < 2; ++i) {
        if (sb.rbuf[d][i] && !sb.in_arena) cudaFree(sb.rbuf[d][i]);
        if (sb.obuf[d][i] && !sb.in_arena) cudaFree(sb.obuf[d][i]);
        if (sb.hbuf[d][i]) cudaFree(sb.hbuf[d][i]);
        if (sb.rfree[d][i]) cudaEventDestroy(sb.rfree[d][i]);
        if (sb.ofree[d][i]) cudaEventDestroy(sb.ofree[d][i]);
      }
    if (sb.ready) cudaEventDestroy(sb.ready);
    if (sb.xgo) cudaEventDestroy(sb.xgo);
    if (sb.xdone) cudaEventDestroy(sb.xdone);
    if (sb.xq) cudaStreamDestroy(sb.xq);
    if (sb.ds) cudaStreamDestroy(sb.ds);
    if (sb.hs) cudaStreamDestroy(sb.hs);
    if (sb.dgo) cudaEventDestroy(sb.dgo);
    if (sb.djoin) cudaEventDestroy(sb.djoin);
    for (int d = 0; d < 2; ++d)
      for (int i = 0; i < 2; ++i) {
        if (sb.dfree_r[d][i]) cudaEventDestroy(sb.dfree_r[d][i]);
        if (sb.dfree_o[d][i]) cudaEventDestroy(sb.dfree_o[d][i]);
        if (sb.hdone[d][i]) cudaEventDestroy(sb.hdone[d][i]);
        if (sb.rlast[d][i]) cudaEventDestroy(sb.rlast[d][i]);
      }
    for (int d = 0; d < 2; ++d) if (sb.join[d]) cudaEventDestroy(sb.join[d]);
    for (int d = 0; d < 2; ++d) {
      if (c->side[d]) cudaStreamDestroy(c->side[d]);
      if (c->zcw[d]) cudaStreamDestroy(c->zcw[d]);
    }
    for (int d = 0; d < 2; ++d) {
      for (int i = 0; i < 8; ++i) {
        if (c->ce[d][i]) cudaStreamDestroy(c->ce[d][i]);
        if (c->ce_join[d][i]) cudaEventDestroy(c->ce_join[d][i]);
      }
      if (c->ce_fork[d]) cudaEventDestroy(c->ce_fork[d]);
    }
    if (c->trace_dev) cudaFree(c->trace_dev);
    if (c->dbg) cudaFree(c->dbg);
    for (int k = 0; k < 2; ++k)
      for (cudaEvent_t e : c->tev[k]) cudaEventDestroy(e);
    if (c->hx_buf) cudaFree(c->hx_buf);
    if (c->seg_tab) cudaFree(c->seg_tab);
    if (c->dseq) cudaFree(c->dseq);
    for (int d = 0; d < 2; ++d) {
      if (c->zc_ev[d]) cudaEventDestroy(c->zc_ev[d]);
      if (c->g_ev[d]) cudaEventDestroy(c->g_ev[d]);
      if (c->gcw[d]) cudaStreamDestroy(c->gcw[d]);
    }
    if (c->arena) cudaFree(c->arena);
    if (c->err_host) cudaFreeHost(c->err_host);
    if (c->err_dev) cudaFree(c->err_dev);
    if (c->rchain) cudaFree(c->rchain);
  }
  delete c;
  return PPC_OK;
}

}  // extern "C"
