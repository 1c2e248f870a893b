// CPU-Forwarding baseline B1 (include/ppcb.h; §2.1): D2H into
// a pinned /dev/shm ring shared by sender and receiver processes, host-side per-chunk flags,
// H2D on the receiver; `channels` host threads move disjoint chunks in parallel.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include "ppcb.h"

namespace {

constexpr uint32_t kMagic = 0x42435050u;   // "PPCB"
constexpr size_t kPage = 4096;

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct alignas(64) SlotHdr {
  std::atomic<uint64_t> seq;
  uint64_t bytes;
  int64_t mb;
};

struct alignas(64) ShmHdr {
  uint32_t magic;
  int32_t K;
  uint64_t max_msg, chunk, max_chunks, data_off, stride, total;
  alignas(64) std::atomic<uint64_t> credit;
};

size_t flags_off() { return round_up(sizeof(ShmHdr), 64); }

}  // namespace

struct ppcb_comm {
  std::string name;
  bool sender = false;
  int device = 0, channels = 1, K = 2;
  size_t max_msg = 0, chunk = 0, max_chunks = 0, stride = 0, total = 0, data_off = 0;
  unsigned timeout_ms = 10000;
  uint8_t* base = nullptr;
  bool registered = false;
  uint64_t seq = 0;
  std::vector<cudaStream_t> st;
  cudaEvent_t ev = nullptr;

  ShmHdr* hdr() { return reinterpret_cast<ShmHdr*>(base); }
  SlotHdr* slot_hdr(int k) {
    return reinterpret_cast<SlotHdr*>(base + flags_off()) + k;
  }
  std::atomic<uint64_t>* flags(int k) {
    uint8_t* p = base + flags_off() + round_up(sizeof(SlotHdr) * K, 64);
    return reinterpret_cast<std::atomic<uint64_t>*>(p) + (size_t)k * max_chunks;
  }
  uint8_t* data(int k) { return base + data_off + (size_t)k * stride; }
};

namespace {

bool wait_geq(const std::atomic<uint64_t>& a, uint64_t v, unsigned timeout_ms) {
  auto t0 = std::chrono::steady_clock::now();
  int spins = 0;
  while ((int64_t)(a.load(std::memory_order_acquire) - v) < 0) {
    if (++spins > 1000) {
      std::this_thread::yield();
      if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms)) return false;
      spins = 0;
    }
  }
  return true;
}

ppc_status_t map_shm(ppcb_comm* c, bool create) {
  const size_t hdr_bytes = flags_off() + round_up(sizeof(SlotHdr) * c->K, 64) +
                           (size_t)c->K * c->max_chunks * 8;
  c->data_off = round_up(hdr_bytes, kPage);
  c->stride = round_up(c->max_msg, kPage);
  c->total = c->data_off + (size_t)c->K * c->stride;
  int fd = shm_open(c->name.c_str(), create ? (O_CREAT | O_RDWR | O_TRUNC) : O_RDWR, 0600);
  if (fd < 0) return PPC_ERR_STATE;
  if (create && ftruncate(fd, (off_t)c->total) != 0) { close(fd); return PPC_ERR_STATE; }
  void* p = mmap(nullptr, c->total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return PPC_ERR_STATE;
  c->base = static_cast<uint8_t*>(p);
  if (create) {
    memset(c->base, 0, c->data_off);
    ShmHdr* h = c->hdr();
    h->K = c->K;
    h->max_msg = c->max_msg;
    h->chunk = c->chunk;
    h->max_chunks = c->max_chunks;
    h->data_off = c->data_off;
    h->stride = c->stride;
    h->total = c->total;
    std::atomic_thread_fence(std::memory_order_release);
    h->magic = kMagic;
  } else {
    ShmHdr* h = c->hdr();
    if (h->magic != kMagic || h->K != c->K || h->max_msg != c->max_msg || h->chunk != c->chunk)
      return PPC_ERR_INVALID_ARG;
  }
  if (cudaHostRegister(c->base + c->data_off, (size_t)c->K * c->stride, cudaHostRegisterPortable) !=
      cudaSuccess)
    return PPC_ERR_CUDA;
  c->registered = true;
  return PPC_OK;
}

}  // namespace

extern "C" {

ppc_status_t ppcb_create(const char* tag, int is_sender, size_t max_msg, size_t chunk, int K,
                         int channels, int device, unsigned timeout_ms, ppcb_comm_t** out) {
  if (!tag || !out || max_msg == 0 || chunk == 0 || K < 1 || channels < 1 || channels > 16)
    return PPC_ERR_INVALID_ARG;
  ppcb_comm* c = new ppcb_comm();
  c->name = std::string("/ppcb_") + tag;
  c->sender = is_sender != 0;
  c->device = device;
  c->channels = channels;
  c->K = K;
  c->max_msg = max_msg;
  c->chunk = chunk;
  c->max_chunks = (max_msg + chunk - 1) / chunk;
  c->timeout_ms = timeout_ms ? timeout_ms : 10000;
  if (cudaSetDevice(device) != cudaSuccess) { delete c; return PPC_ERR_CUDA; }
  c->st.resize(channels);
  for (auto& s : c->st)
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) { ppcb_destroy(c); return PPC_ERR_CUDA; }
  if (cudaEventCreateWithFlags(&c->ev, cudaEventDisableTiming) != cudaSuccess) { ppcb_destroy(c); return PPC_ERR_CUDA; }
  if (c->sender) {
    ppc_status_t st = map_shm(c, true);
    if (st) { ppcb_destroy(c); return st; }
  }
  *out = c;
  return PPC_OK;
}

ppc_status_t ppcb_connect(ppcb_comm_t* c) {
  if (!c) return PPC_ERR_INVALID_ARG;
  if (c->sender || c->base) return PPC_OK;
  cudaSetDevice(c->device);
  return map_shm(c, false);
}

ppc_status_t ppcb_send(ppcb_comm_t* c, const void* buf, size_t bytes, long long mb, cudaStream_t s) {
  if (!c || !c->sender || !c->base || (bytes && !buf) || mb < 0) return PPC_ERR_INVALID_ARG;
  if (bytes > c->max_msg) return PPC_ERR_TOO_LARGE;
  cudaSetDevice(c->device);
  const uint64_t seq = c->seq + 1;
  const int k = (int)(seq % c->K);
  if (seq > (uint64_t)c->K && !wait_geq(c->hdr()->credit, seq - c->K, c->timeout_ms))
    return PPC_ERR_TIMEOUT;
  if (cudaEventRecord(c->ev, s) != cudaSuccess) return PPC_ERR_CUDA;
  SlotHdr* sh = c->slot_hdr(k);
  sh->bytes = bytes;
  sh->mb = mb;
  sh->seq.store(seq, std::memory_order_release);
  const size_t n = (bytes + c->chunk - 1) / c->chunk;
  std::atomic<uint64_t>* fl = c->flags(k);
  uint8_t* dst = c->data(k);
  std::atomic<int> err{0};
  auto work = [&](int t) {
    cudaSetDevice(c->device);
    if (cudaStreamWaitEvent(c->st[t], c->ev, 0) != cudaSuccess) { err = PPC_ERR_CUDA; return; }
    for (size_t ci = t; ci < n; ci += c->channels) {
      const size_t off = ci * c->chunk, len = std::min(c->chunk, bytes - off);
      if (cudaMemcpyAsync(dst + off, static_cast<const uint8_t*>(buf) + off, len,
                          cudaMemcpyDeviceToHost, c->st[t]) != cudaSuccess ||
          cudaStreamSynchronize(c->st[t]) != cudaSuccess) {
        err = PPC_ERR_CUDA;
        return;
      }
      fl[ci].store(seq, std::memory_order_release);
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < c->channels; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  if (err) return (ppc_status_t)err.load();
  c->seq = seq;
  return PPC_OK;
}

ppc_status_t ppcb_recv(ppcb_comm_t* c, void* buf, size_t bytes, long long mb, cudaStream_t s) {
  if (!c || c->sender || !c->base || (bytes && !buf) || mb < 0) return PPC_ERR_INVALID_ARG;
  if (bytes > c->max_msg) return PPC_ERR_TOO_LARGE;
  cudaSetDevice(c->device);
  const uint64_t seq = c->seq + 1;
  const int k = (int)(seq % c->K);
  SlotHdr* sh = c->slot_hdr(k);
  if (!wait_geq(sh->seq, seq, c->timeout_ms)) return PPC_ERR_TIMEOUT;
  if (sh->seq.load(std::memory_order_acquire) != seq || sh->mb != mb) return PPC_ERR_ORDER;
  if (sh->bytes != bytes) return PPC_ERR_SIZE_MISMATCH;
  if (cudaEventRecord(c->ev, s) != cudaSuccess) return PPC_ERR_CUDA;
  const size_t n = (bytes + c->chunk - 1) / c->chunk;
  std::atomic<uint64_t>* fl = c->flags(k);
  const uint8_t* src = c->data(k);
  std::atomic<int> err{0};
  auto work = [&](int t) {
    cudaSetDevice(c->device);
    if (cudaStreamWaitEvent(c->st[t], c->ev, 0) != cudaSuccess) { err = PPC_ERR_CUDA; return; }
    for (size_t ci = t; ci < n; ci += c->channels) {
      if (!wait_geq(fl[ci], seq, c->timeout_ms)) { err = PPC_ERR_TIMEOUT; return; }
      const size_t off = ci * c->chunk, len = std::min(c->chunk, bytes - off);
      if (cudaMemcpyAsync(static_cast<uint8_t*>(buf) + off, src + off, len, cudaMemcpyHostToDevice,
                          c->st[t]) != cudaSuccess) {
        err = PPC_ERR_CUDA;
        return;
      }
    }
    if (cudaStreamSynchronize(c->st[t]) != cudaSuccess) err = PPC_ERR_CUDA;
  };
  std::vector<std::thread> th;
  for (int t = 1; t < c->channels; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  if (err) return (ppc_status_t)err.load();
  c->hdr()->credit.store(seq, std::memory_order_release);
  c->seq = seq;
  return PPC_OK;
}

ppc_status_t ppcb_destroy(ppcb_comm_t* c) {
  if (!c) return PPC_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  if (c->registered) cudaHostUnregister(c->base + c->data_off);
  if (c->base) munmap(c->base, c->total);
  if (c->sender) shm_unlink(c->name.c_str());
  for (auto s : c->st) if (s) cudaStreamDestroy(s);
  if (c->ev) cudaEventDestroy(c->ev);
  delete c;
  return PPC_OK;
}

}  // extern "C"
