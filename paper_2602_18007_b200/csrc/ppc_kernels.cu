// sm_100a kernels of the stage-boundary transfer (K9 push, K10 recv, K12 CE signalling)
// and the test kernels (K14: SplitMix64 fill, XOR stage proxy).
//
// Memory-ordering protocol:
//   sender, per chunk:   data stores -> fence.acq_rel.sys (every thread) -> bar.sync ->
//                        st.release.sys flags[c] = seq (thread 0)
//   receiver, per chunk: ld.acquire.sys flags[c] >= seq (thread 0) -> bar.sync ->
//                        L1-bypassing (.cg) loads of the slot
//   credit:              receiver's last CTA -> st.release.sys credit = seq (sender memory);
//                        sender waits ld.acquire.sys credit >= seq - K before writing a slot.
// Flags and credits are monotone u64 sequence numbers (never reset); every wait compares
// wrap-safe and is bounded by %globaltimer (§4.3 P:L211 hangs).
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include "ppc_internal.h"

namespace ppc {

// kernels this process enqueued through libppc (ppc_launch_count): every launch site bumps it;
// a graph capture's launches are moved from it into the graph, which adds them per replay
std::atomic<unsigned long long> g_launches{0};
int g_pdl = 1;   // programmatic dependent launch for transport kernels (PPC_PDL, ppc_create)
int g_recv_early = 0;   // receive looks for its publication before griddepcontrol.wait (PPC_RECV_EARLY)
int g_copy_tma_ctas = 0;   // virtual-stage copy: TMA bulk grid; 0 = SIMT copy_kernel (PPC_COPY_TMA_CTAS)

// Programmatic dependent launch (PDL): a transport kernel launched right behind another one
// on the same stream may be scheduled while its predecessor still runs.  griddepcontrol.wait
// returns once every prerequisite grid has completed and its memory is visible, so nothing
// below it can observe a partial predecessor; launch_dependents then lets the NEXT kernel
// get resident early.  Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// A PDL dependent may be resident before its predecessor ends, and CTAs of it that do not
// fit yet stay pending.  A spinning transport kernel must never be pending behind its
// predecessor: pending CTAs can hold up other kernels on the GPU (measured: a bidirectional
// zero-copy stream of 128-CTA receives timed out when a receive grid could not be resident
// next to the one before it), and the kernel a spinning predecessor waits for may be the
// peer's.  So a spinning kernel gets PDL only if two of its grids fit on the GPU at once
// (occupancy x SMs >= 2 x grid); kernels that never spin (copy, 1-thread kernels) always.
// CTAs of kernel k (block threads) that can be resident on the current GPU at once
// (occupancy x SMs), cached; 0 if unknown.
template <typename... KArgs>
unsigned resident_capacity(void (*k)(KArgs...), unsigned block) {
  struct Entry { const void* k; unsigned block; int dev, cap; };
  static thread_local Entry cache[16];
  static thread_local int used = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  for (int i = 0; i < used; ++i)
    if (cache[i].k == (const void*)k && cache[i].block == block && cache[i].dev == dev)
      return (unsigned)cache[i].cap;
  int per_sm = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, (int)block, 0) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  const Entry e{(const void*)k, block, dev, per_sm * sms};
  cache[used < 16 ? used++ : 15] = e;
  return (unsigned)e.cap;
}
template <typename... KArgs>
bool pdl_fits(void (*k)(KArgs...), unsigned grid, unsigned block) {
  return 2 * grid <= resident_capacity(k, block);
}
// A spinning grid must be resident as a whole: CTAs left pending behind it can hold up the
// kernels its peer is waiting for (see above).  Grids are grid-strided, so any size works.
template <typename... KArgs>
int fit_grid(void (*k)(KArgs...), int grid, unsigned block) {
  const unsigned cap = resident_capacity(k, block);
  return (cap && (unsigned)grid > cap) ? (int)cap : grid;
}
// Cap of cross-GPU spinning grids.  Round 1 measured a bidirectional zero-copy stream
// stalling once the receive CTAs in flight exceeded the SM count (profiles/r47_zc_bidir.log);
// the cause was a lazy module load waiting for an idle device behind spinning receives
// (ppc_create now preloads every kernel): the same stream runs clean with 96, 128, 148 and
// 256-CTA grids, with and without PDL (profiles/round2/p44_zc_bidir_grids/).  64 stays the
// default because it is the fastest grid for pulls with both directions loaded
// (profiles/round2/p24_bidir_probe.jsonl: 596 GB/s at 64 vs 556-560 at 96 / 148).
int kMaxSpinGrid = 64;   // PPC_SPIN_GRID_CAP

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*k)(KArgs...), unsigned grid, unsigned block, cudaStream_t s,
                     bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (g_pdl && pdl) ? 1 : 0;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Scope-templated variants: kSys = peer GPU over NVLink (.sys); !kSys = virtual stages on
// one GPU, where the consumer is on the same device (.gpu is enough and cheaper).
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
template <bool kSys>
__device__ __forceinline__ uint64_t ld_acq(const uint64_t* p) {
  return kSys ? ld_acquire_sys(p) : ld_acquire_gpu(p);
}
template <bool kSys>
__device__ __forceinline__ void st_rel(uint64_t* p, uint64_t v) {
  if (kSys) st_release_sys(p, v); else st_release_gpu(p, v);
}
template <bool kSys>
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  if (kSys) st_relaxed_sys(p, v); else st_relaxed_gpu(p, v);
}
template <bool kSys>
__device__ __forceinline__ void fence_rel() {
  if (kSys) fence_acq_rel_sys(); else asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
// streaming read of data nobody writes during the kernel (user source buffer)
__device__ __forceinline__ uint4 ld_src(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// coherent read (L2) of ring data written by another GPU / kernel
__device__ __forceinline__ uint4 ld_ring(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_data(uint4* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}

__device__ __forceinline__ void latch(ErrWord* e, unsigned code, uint64_t seq, unsigned info) {
  // first failure wins (ErrWord): claim in device memory, then the mapped host record with
  // its code stored last; any error poisons the comm
  if (atomicCAS(&e->claim, 0u, 1u) != 0u) return;
  volatile ErrHost* v = e->host;
  v->seq = (unsigned)seq;
  v->info = info;
  __threadfence_system();
  v->code = code;
  __threadfence_system();
}

// PPC_DBG_STAMPS: %globaltimer (low 48 bits) with the SM id in the top 16 bits
__device__ __forceinline__ uint64_t dbg_stamp_sm() {
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  return ((uint64_t)smid << 48) | (globaltimer() & 0xFFFFFFFFFFFFull);
}

// Wait until *p >= target (wrap-safe); false on timeout.
// A latched error poisons the comm (ErrWord): every other bounded wait of the comm gives up
// at its next check instead of running into its own deadline, so one failure does not
// cost one timeout per queued kernel.
__device__ __forceinline__ bool err_claimed(const ErrWord* e) {
  return e && *reinterpret_cast<const volatile unsigned*>(&e->claim) != 0u;
}
template <bool kSys = true>
__device__ __forceinline__ bool wait_geq(const uint64_t* p, uint64_t target, uint64_t deadline,
                                         const ErrWord* err) {
  uint64_t v = ld_acq<kSys>(p);
  int spins = 0;
  while ((int64_t)(v - target) < 0) {
    if (((++spins) & 63) == 0 && (globaltimer() > deadline || err_claimed(err))) return false;
    __nanosleep(32);
    v = ld_acq<kSys>(p);
  }
  return true;
}

// Copy `len` bytes with the CTA's threads: 16-byte vectors, UNROLL loads in flight per
// thread before their stores; byte loop for misaligned buffers and the ragged tail.
// 32-byte vectors (sm_100 LDG/STG.256)
struct __align__(32) V32 {
  uint4 lo, hi;
};
__device__ __forceinline__ V32 ld_src(const V32* p) {
  V32 r;
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.lo.x), "=r"(r.lo.y), "=r"(r.lo.z), "=r"(r.lo.w), "=r"(r.hi.x),
                 "=r"(r.hi.y), "=r"(r.hi.z), "=r"(r.hi.w) : "l"(p));
  return r;
}
__device__ __forceinline__ V32 ld_ring(const V32* p) {
  V32 r;
  asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.lo.x), "=r"(r.lo.y), "=r"(r.lo.z), "=r"(r.lo.w), "=r"(r.hi.x),
                 "=r"(r.hi.y), "=r"(r.hi.z), "=r"(r.hi.w) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_data(V32* p, const V32& v) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.lo.x),
               "r"(v.lo.y), "r"(v.lo.z), "r"(v.lo.w), "r"(v.hi.x), "r"(v.hi.y), "r"(v.hi.z),
               "r"(v.hi.w) : "memory");
}

// Vector body of a CTA copy: VT = uint4 (16 B) or V32 (32 B), U vectors in flight per
// thread (all loads issued before their stores).
template <bool kRingSrc, typename VT, int U>
__device__ __forceinline__ uint64_t cta_copy_body(uint8_t* __restrict__ dst,
                                                  const uint8_t* __restrict__ src, uint64_t len,
                                                  uint64_t tid, uint64_t nt) {
  const uint64_t nv = len / sizeof(VT);
  const VT* s = reinterpret_cast<const VT*>(src);
  VT* d = reinterpret_cast<VT*>(dst);
  uint64_t i = tid;
  for (; i + (U - 1) * nt < nv; i += nt * U) {
    VT v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) v[j] = kRingSrc ? ld_ring(s + i + j * nt) : ld_src(s + i + j * nt);
#pragma unroll
    for (int j = 0; j < U; ++j) st_data(d + i + j * nt, v[j]);
  }
  for (; i < nv; i += nt) st_data(d + i, kRingSrc ? ld_ring(s + i) : ld_src(s + i));
  return nv * sizeof(VT);
}

template <bool kRingSrc>
__device__ __forceinline__ void cta_copy(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                         uint64_t len, uint64_t tid = threadIdx.x,
                                         uint64_t nt = blockDim.x) {
  uint64_t body = 0;
  const uintptr_t al = (uintptr_t)dst | (uintptr_t)src;
  if ((al & 31) == 0) {
    body = cta_copy_body<kRingSrc, V32, 4>(dst, src, len, tid, nt);
    if (len - body >= 16)
      body += cta_copy_body<kRingSrc, uint4, 1>(dst + body, src + body, len - body, tid, nt);
  } else if ((al & 15) == 0) {
    body = cta_copy_body<kRingSrc, uint4, 8>(dst, src, len, tid, nt);
  }
  for (uint64_t k = body + tid; k < len; k += nt) {
    uint8_t b;
    if (kRingSrc) {
      b = *reinterpret_cast<const volatile uint8_t*>(src + k);
    } else {
      b = src[k];
    }
    dst[k] = b;
  }
}

// ---------------------------------------------------------------- MPDT channels
// The paper splits one message across several NICs (Multi-NIC Parallel Data Transfer).  Here
// a message's chunks are split into C contiguous ranges ("channels"), each moved by its own
// group of CTAs: CTA b of `workers` serves channel b % C and walks chunks [c0, c1) of that
// channel with a stride of the channel's CTA count.  C = 1 is the plain grid stride.
struct ChanIter {
  uint32_t first, end, step;
};
__device__ __forceinline__ ChanIter chan_iter(uint32_t n_chunks, uint32_t C, uint32_t b,
                                              uint32_t workers) {
  C = max(1u, min(C, workers));
  const uint32_t ch = b % C;
  const uint32_t ctas = (workers - ch + C - 1) / C;          // CTAs serving channel ch
  const uint32_t c0 = (uint32_t)((uint64_t)n_chunks * ch / C);
  const uint32_t c1 = (uint32_t)((uint64_t)n_chunks * (ch + 1) / C);
  return {c0 + b / C, c1, ctas};
}

// ---------------------------------------------------------------- graph-replay resolution
// (SeqRef): absolute seq and slot pointers from the device sequence base.
__device__ __forceinline__ PushArgs resolve(PushArgs a) {
  if (a.sr.base) {
    a.seq += *a.sr.base;
    const uint64_t slot = a.seq % a.sr.K;
    a.dst += slot * a.sr.stride;
    a.hdr += slot;
    a.hdr_flag += slot;
    a.flags += slot * a.sr.fstride;
    a.need_credit = (a.sr.wait_credit && a.seq > a.sr.K) ? a.seq - a.sr.K : 0;
  }
  return a;
}
__device__ __forceinline__ RecvArgs resolve(RecvArgs a) {
  if (a.sr.base) {
    a.seq += *a.sr.base;
    const uint64_t slot = a.seq % a.sr.K;
    a.src += slot * a.sr.stride;
    a.hdr += slot;
    a.hdr_flag += slot;
    a.flags += slot * a.sr.fstride;
    a.done += slot;
    a.next += slot;
  }
  return a;
}
__device__ __forceinline__ PublishArgs resolve(PublishArgs a) {
  if (a.sr.base) {
    a.seq += *a.sr.base;
    const uint64_t slot = a.seq % a.sr.K;
    a.hdr += slot;
    a.hdr_flag += slot;
    a.need_credit = (a.sr.wait_credit && a.seq > a.sr.K) ? a.seq - a.sr.K : 0;
  }
  return a;
}

// ---------------------------------------------------------------- K9: push (SM engine)
template <bool kSys>
__global__ void __launch_bounds__(kThreads) push_kernel(PushArgs a0) {
  pdl_enter();
  const PushArgs a = resolve(a0);
  uint64_t deadline = 0;
  int fail = 0;
  if (threadIdx.x == 0) {
    const uint64_t t0 = globaltimer();
    deadline = t0 + a.timeout_ns;
    if (a.rec && blockIdx.x == 0)
      fill_record(a.rec, (long long)t0, a.rec_src, a.rec_dst, a.dir, 0, a.seq, a.mb, a.bytes);
    if (a.need_credit && !wait_geq<kSys>(a.credit, a.need_credit, deadline, a.err)) {
      latch(a.err, PPC_ERR_TIMEOUT, a.seq, a.dir);
      fail = 1;
    } else if (blockIdx.x == 0) {
      SlotHeader h = {};
      h.magic = kMagic;
      h.dir = (uint8_t)a.dir;
      h.boundary = (uint8_t)a.boundary;
      h.bytes = a.bytes;
      h.seq = a.seq;
      h.mb = a.mb;
      h.step = a.step;
      const uint4* hs = reinterpret_cast<const uint4*>(&h);
      uint4* hd = reinterpret_cast<uint4*>(a.hdr);
#pragma unroll
      for (int j = 0; j < 4; ++j) st_data(hd + j, hs[j]);
      st_rel<kSys>(a.hdr_flag, a.seq);
    }
  }
  if (__syncthreads_or(fail)) return;
  const ChanIter it = chan_iter(a.n_chunks, a.channels, blockIdx.x, gridDim.x);
  for (uint32_t c = it.first; c < it.end; c += it.step) {
    const uint64_t off = (uint64_t)c * a.chunk;
    const uint64_t len = min(a.chunk, a.bytes - off);
    cta_copy<false>(a.dst + off, a.src + off, len);
    // bar.sync orders every thread's stores before thread 0's release; the release
    // (fence.acq_rel + strong store, cumulative) publishes them to the peer.  One fence per
    // CTA-chunk instead of one per thread (profiles/r1_nvlink_probe.md: +6-15% at 32 MiB).
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_rel<kSys>();
      st_rel<kSys>(a.flags + c, a.seq);
    }
  }
  if (a.rec) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(a.done, 1u) == gridDim.x - 1) {
        *a.done = 0;
        a.rec->t_end_ns = (long long)globaltimer();
      }
    }
  }
}

// ---------------------------------------------------------------- K9': warp-specialised push
// Warp 0 signals, warps 1..16 copy.  Copy warps stream chunk after chunk and hand each
// finished chunk to the signal warp through a ring of shared-memory mbarriers (arrive =
// release.cta); the signal warp waits (acquire.cta), issues the system-scope release fence
// and the flag store for that chunk while the copy warps are already moving the next one.
// So the NVLink round trip of the release fence is off the copy path and chunks can be
// small (receiver copy-out pipelines behind them) without paying a CTA-wide stall per chunk.
constexpr int kWsCopyWarps = 16;
constexpr int kWsThreads = 32 * (kWsCopyWarps + 1);
constexpr int kWsRing = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* m) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(m)), "r"(parity) : "memory");
}

template <bool kSys>
__global__ void __launch_bounds__(kWsThreads) push_ws_kernel(PushArgs a0) {
  pdl_enter();
  const PushArgs a = resolve(a0);
  __shared__ __align__(8) uint64_t full[kWsRing], empty[kWsRing];
  uint64_t deadline = 0;
  int fail = 0;
  if (threadIdx.x == 0) {
    const uint64_t t0 = globaltimer();
    deadline = t0 + a.timeout_ns;
    if (a.rec && blockIdx.x == 0)
      fill_record(a.rec, (long long)t0, a.rec_src, a.rec_dst, a.dir, 0, a.seq, a.mb, a.bytes);
    for (int b = 0; b < kWsRing; ++b) {
      mbar_init(&full[b], kWsCopyWarps);
      mbar_init(&empty[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (a.need_credit && !wait_geq<kSys>(a.credit, a.need_credit, deadline, a.err)) {
      latch(a.err, PPC_ERR_TIMEOUT, a.seq, a.dir);
      fail = 1;
    } else if (blockIdx.x == 0) {
      SlotHeader h = {};
      h.magic = kMagic;
      h.dir = (uint8_t)a.dir;
      h.boundary = (uint8_t)a.boundary;
      h.bytes = a.bytes;
      h.seq = a.seq;
      h.mb = a.mb;
      h.step = a.step;
      const uint4* hs = reinterpret_cast<const uint4*>(&h);
      uint4* hd = reinterpret_cast<uint4*>(a.hdr);
#pragma unroll
      for (int j = 0; j < 4; ++j) st_data(hd + j, hs[j]);
      st_rel<kSys>(a.hdr_flag, a.seq);
    }
  }
  if (__syncthreads_or(fail)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ChanIter it = chan_iter(a.n_chunks, a.channels, blockIdx.x, gridDim.x);
  uint32_t i = 0;
  if (warp == 0) {                                   // signal warp
    if (lane == 0) {
      for (uint32_t c = it.first; c < it.end; c += it.step, ++i) {
        const int b = i % kWsRing;
        mbar_wait(&full[b], (i / kWsRing) & 1);
        fence_rel<kSys>();
        st_rel<kSys>(a.flags + c, a.seq);
        mbar_arrive(&empty[b]);
      }
    }
  } else {                                           // copy warps
    const uint64_t tid = threadIdx.x - 32, nt = 32 * kWsCopyWarps;
    for (uint32_t c = it.first; c < it.end; c += it.step, ++i) {
      const int b = i % kWsRing;
      if (i >= kWsRing) mbar_wait(&empty[b], ((i / kWsRing) - 1) & 1);
      const uint64_t off = (uint64_t)c * a.chunk;
      const uint64_t len = min(a.chunk, a.bytes - off);
      cta_copy<false>(a.dst + off, a.src + off, len, tid, nt);
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[b]);
    }
  }
  if (a.rec) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(a.done, 1u) == gridDim.x - 1) {
        *a.done = 0;
        a.rec->t_end_ns = (long long)globaltimer();
      }
    }
  }
}

// zero-copy publication (publish_kernel; fused into recv_kernel by the step driver).
// Header phase: wait for the slot's credit, write the 64-B header into the receiver's slot.
// Flag phase: st.release.sys of the header flag (cumulative over the header and over the
// producer's writes to the buffer).  false = the credit wait timed out (error latched).
__device__ __forceinline__ bool publish_header(const PublishArgs& a) {
  if (a.need_credit && !wait_geq(a.credit, a.need_credit, globaltimer() + a.timeout_ns, a.err)) {
    latch(a.err, PPC_ERR_TIMEOUT, a.seq, a.dir);
    return false;
  }
  SlotHeader h = {};
  h.magic = kMagic;
  h.dir = (uint8_t)a.dir;
  h.boundary = (uint8_t)a.boundary;
  h.flags = kHdrZeroCopy;
  h.bytes = a.bytes;
  h.seq = a.seq;
  h.mb = a.mb;
  h.src_off = a.src_off;
  h.src_seg = a.src_seg;
  const uint4* hs = reinterpret_cast<const uint4*>(&h);
  uint4* hd = reinterpret_cast<uint4*>(a.hdr);
#pragma unroll
  for (int j = 0; j < 4; ++j) st_data(hd + j, hs[j]);
  return true;
}
__device__ __forceinline__ void publish_flag(const PublishArgs& a, uint64_t t0) {
  st_release_sys(a.hdr_flag, a.seq);
  if (a.rec) {
    fill_record(a.rec, (long long)t0, a.rec_src, a.rec_dst, (int)a.dir, 0, a.seq, a.mb, a.bytes);
    a.rec->t_end_ns = (long long)globaltimer();
  }
}
__device__ __forceinline__ void publish_body(const PublishArgs& a) {
  const uint64_t t0 = globaltimer();
  if (publish_header(a)) publish_flag(a, t0);
}

// ---------------------------------------------------------------- K10: recv + copy-out
// The 64-B slot header read in ONE round trip (two 32-B L2 loads issued together) after the
// header flag's acquire, instead of a chain of dependent volatile field loads.
struct HdrView {
  uint32_t magic, flags, src_seg;
  uint64_t bytes, seq, src_off;
  int64_t mb;
};
__device__ __forceinline__ HdrView read_header(const SlotHeader* hp) {
  const V32* v = reinterpret_cast<const V32*>(hp);
  const V32 a = ld_ring(v), b = ld_ring(v + 1);
  HdrView h;
  h.magic = a.lo.x;                                    // u32 magic | u8 dir | u8 bnd | u16 flags
  h.flags = a.lo.y >> 16;
  h.bytes = (uint64_t)a.lo.z | (uint64_t)a.lo.w << 32;
  h.seq = (uint64_t)a.hi.x | (uint64_t)a.hi.y << 32;
  h.mb = (int64_t)((uint64_t)a.hi.z | (uint64_t)a.hi.w << 32);
  h.src_off = (uint64_t)b.lo.z | (uint64_t)b.lo.w << 32;   // b: step | src_off | src_seg | pad
  h.src_seg = b.hi.x;
  return h;
}
static_assert(offsetof(SlotHeader, flags) == 6 && offsetof(SlotHeader, bytes) == 8 &&
              offsetof(SlotHeader, seq) == 16 && offsetof(SlotHeader, mb) == 24 &&
              offsetof(SlotHeader, src_off) == 40 && offsetof(SlotHeader, src_seg) == 48,
              "read_header decodes the SlotHeader layout");

// Fused publication.  Its arguments are read from the grid-constant parameter space right
// where they are used, so none of them stays live in registers across the copy loop
// (a local copy of them had pushed the kernel to 110 registers, one CTA per SM).
__device__ __forceinline__ bool fused_publish_header(const PublishArgs* p0) {
  const bool ok = publish_header(resolve(*p0));
  __threadfence_system();
  return ok;
}
// one system fence, then two relaxed stores: the next op's header flag first (it is on the
// critical path), then this receive's credit.  A second release would wait for the first
// store's NVLink acknowledgement.
__device__ __forceinline__ void fused_publish_flag(const PublishArgs* p0, uint64_t* credit,
                                                  uint64_t seq, bool fenced = false) {
  uint64_t pseq = p0->seq;
  uint64_t* flag = p0->hdr_flag;
  if (p0->sr.base) {                  // graph replay: resolve seq and slot (as resolve())
    pseq += *p0->sr.base;
    flag += pseq % p0->sr.K;
  }
  const uint64_t t0 = globaltimer();
  // PPC_PUB_FENCE=gpu: block 0's header stores were already fenced at system scope before
  // its arrival on the done counter (fused_publish_header), every CTA's pulled loads have
  // returned before its arrival, and this CTA saw all arrivals — so only gpu-scope ordering
  // is left to establish here.  Opt-in A/B; the default keeps the full
  // system-scope release.
  // fenced: the caller is block 0, whose own system fence after the header stores
  // (fused_publish_header) already orders them before these stores
  if (!fenced) {
    if (p0->gpu_fence) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    else fence_acq_rel_sys();
  }
  st_relaxed_sys(flag, pseq);
  st_relaxed_sys(credit, seq);
  if (ppc_record_t* r = p0->rec) {
    fill_record(r, (long long)t0, p0->rec_src, p0->rec_dst, (int)p0->dir, 0, pseq, p0->mb,
                p0->bytes);
    r->t_end_ns = (long long)globaltimer();
  }
}

// mapped base of a zero-copy source segment on this GPU; 0 if never imported
__device__ __forceinline__ uint64_t zc_base(const RecvArgs& a, uint32_t seg) {
  return seg == kArenaSeg ? (uint64_t)(uintptr_t)a.peer_arena
       : (a.seg_tab && seg < (uint32_t)kMaxSeg) ? a.seg_tab[seg] : 0;
}
constexpr int kEarlyV = 4;                    // V32 vectors per thread pulled early (64 KiB/CTA)
constexpr uint32_t kPullUnit = 4096;          // PPC_PULL_DYN: bytes per warp claim (4 V32 / lane)

// Chained receive entry (RecvArgs::chain_wait): instead of griddepcontrol.wait (which
// returns only after the predecessor grid has exited — its last CTA's publication fence
// included — and PDL has released us), thread 0 waits (bounded) until the predecessor
// receive has posted the end of its data phase; only then may the NEXT kernel get resident,
// so at most two receive grids are resident at a time, as with plain PDL.  The
// predecessor's sequence base (graph replay) was written by set_seq_kernel, which
// completed before the predecessor passed its own griddepcontrol.wait and therefore before
// we could be launched.  false: timed out (error latched).
__device__ __forceinline__ bool chain_enter(const RecvArgs& a0) {
  int fail = 0;
  if (threadIdx.x == 0) {
    const uint64_t target = a0.chain_seq + (a0.chain_base ? *a0.chain_base : 0);
    if (!wait_geq<false>(a0.chain_wait, target, globaltimer() + a0.timeout_ns, a0.err)) {
      latch(a0.err, PPC_ERR_TIMEOUT, a0.seq, 0x700u);
      fail = 1;
    }
  }
  fail = __syncthreads_or(fail);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  return !fail;
}
// block 0 of a kPub receive: wait (bounded) until the n worker CTAs have arrived
__device__ __forceinline__ bool wait_arrivals(const uint32_t* done, uint32_t n, uint64_t deadline,
                                              const ErrWord* err) {
  int spins = 0;
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done) : "memory");
    if (v >= n) return true;
    if (((++spins) & 255) == 0 && (globaltimer() > deadline || err_claimed(err))) return false;
  }
}
// end of a receive's data phase (its last CTA, after the done count): post its seq
__device__ __forceinline__ void chain_post(const RecvArgs& a) {
  if (a.chain_post)
    atomicMax(reinterpret_cast<unsigned long long*>(a.chain_post), (unsigned long long)a.seq);
}

// kPub: the variant with the fused publication (step driver, terminal receives of a
// comm-only PP2 step).  Both variants need ~90 registers: one 512-thread CTA per SM.
template <bool kSys, bool kPub, bool kEarly = false>
__global__ void __launch_bounds__(kThreads) recv_kernel(const __grid_constant__ RecvArgs a0) {
  __shared__ const uint8_t* s_zc_src;   // zero-copy: the sender's buffer, mapped here
  __shared__ const uint8_t* s_early_src;
  __shared__ uint64_t s_early_seq;
  // Early phase (kEarly: PPC_RECV_EARLY, PDL only; its own instantiation, the early
  // registers would halve the occupancy of the plain kernel): before griddepcontrol.wait, ONE look (no spin) at this
  // message's header.  If its zero-copy publication is already there, the CTA pulls the
  // first 64 KiB of its first chunk into registers while the predecessor drains.  Only
  // peer-published data is read here; nothing is written.  The graph's sequence base may
  // still be stale (set_seq_kernel is a predecessor), so after the wait the early result is
  // used only if the resolved seq is the same.
  V32 pre[kEarlyV];
  bool pre_ok = false;
  if (kEarly) {
    if (threadIdx.x == 0) {
      s_early_src = nullptr;
      const RecvArgs e = resolve(a0);
      if ((int64_t)(ld_acq<kSys>(e.hdr_flag) - e.seq) >= 0) {
        const volatile SlotHeader* h = e.hdr;
        if (h->magic == kMagic && h->seq == e.seq && h->mb == e.mb && h->bytes == e.bytes &&
            (h->flags & kHdrZeroCopy)) {
          const uint64_t base = zc_base(e, h->src_seg);
          if (base) {
            s_early_src = reinterpret_cast<const uint8_t*>(base + h->src_off);
            s_early_seq = e.seq;
          }
        }
      }
    }
    __syncthreads();
    const uint32_t c_first = chan_iter(a0.n_chunks, a0.channels, blockIdx.x, gridDim.x).first;
    const uint64_t off = (uint64_t)c_first * a0.chunk;
    if (s_early_src && c_first < chan_iter(a0.n_chunks, a0.channels, blockIdx.x, gridDim.x).end &&
        min(a0.chunk, a0.bytes - off) >= (uint64_t)kEarlyV * kThreads * sizeof(V32) &&
        (((uintptr_t)(a0.dst + off) | (uintptr_t)(s_early_src + off)) & 31) == 0) {
      const V32* src = reinterpret_cast<const V32*>(s_early_src + off);
#pragma unroll
      for (int j = 0; j < kEarlyV; ++j) pre[j] = ld_ring(src + threadIdx.x + j * kThreads);
      pre_ok = true;
    }
  }
  if (!kEarly && a0.chain_wait) {
    if (!chain_enter(a0)) return;
  } else {
    pdl_enter();
  }
  // PPC_DBG_STAMPS (diagnostics): per CTA [0] released by griddepcontrol.wait (or the
  // chain), [1] header seen, [2] first chunk moved, [3] done
  uint64_t* const dbg = a0.dbg ? a0.dbg + 4 * blockIdx.x : nullptr;
  if (dbg && threadIdx.x == 0) dbg[0] = globaltimer();
  const RecvArgs a = resolve(a0);
  uint64_t deadline = 0;
  int fail = 0;
  if (kEarly && threadIdx.x == 0 && s_early_src && s_early_seq == a.seq) {
    // header already checked in the early phase (same seq, so the same slot and message)
    s_zc_src = s_early_src;
    if (a.rec && blockIdx.x == 0) {  // dir -2 in the record: the early look hit (ppc_trace)
      fill_record(a.rec, (long long)globaltimer(), a.rec_src, a.rec_dst, -2, 1, a.seq, a.mb, a.bytes);
      a.rec->t_start_ns = (long long)globaltimer();
    }
    if (kPub && blockIdx.x == 0 && !fused_publish_header(&a0.pub)) fail = 1;
  } else if (threadIdx.x == 0) {
    const uint64_t t0 = globaltimer();
    deadline = t0 + a.timeout_ns;
    s_zc_src = nullptr;
    if (a.rec && blockIdx.x == 0)
      fill_record(a.rec, (long long)t0, a.rec_src, a.rec_dst, -1, 1, a.seq, a.mb, a.bytes);
    // fused publication, header phase: written now (the slot is free once its credit is
    // in), so its NVLink round trip overlaps this receive; the system fence orders it
    // before the flag the last CTA releases (ordered after us through the done counter)
    if (kPub && blockIdx.x == 0 && !fused_publish_header(&a0.pub)) fail = 1;
    if (fail) {
    } else if (!wait_geq<kSys>(a.hdr_flag, a.seq, deadline, a.err)) {
      latch(a.err, PPC_ERR_TIMEOUT, a.seq, 0x100u);
      fail = 1;
    } else {
      const HdrView h = read_header(a.hdr);
      if (h.magic != kMagic || h.seq != a.seq || h.mb != a.mb) {
        latch(a.err, PPC_ERR_ORDER, a.seq, 0x100u);
        fail = 1;
      } else if (h.bytes != a.bytes) {
        latch(a.err, PPC_ERR_SIZE_MISMATCH, a.seq, 0x100u);
        fail = 1;
      } else if (h.flags & kHdrZeroCopy) {
        const uint32_t seg = h.src_seg;
        const uint64_t base = zc_base(a, seg);
        if (!base) {                   // the receiver never imported that registration
          latch(a.err, PPC_ERR_ORDER, a.seq, 0x300u | seg << 12);
          fail = 1;
        } else {
          s_zc_src = reinterpret_cast<const uint8_t*>(base + h.src_off);
          // trace: a zero-copy receive starts moving data when the publication is seen
          if (a.rec && blockIdx.x == 0) a.rec->t_start_ns = (long long)globaltimer();
        }
      }
    }
  }
  if (__syncthreads_or(fail)) return;
  if (dbg && threadIdx.x == 0) dbg[1] = globaltimer();
  const uint8_t* zc_src = s_zc_src;
  // the early pull is valid only for the message resolved now (CTA-uniform condition)
  const bool use_pre = kEarly && pre_ok && zc_src == s_early_src && s_early_seq == a.seq;
  // fused publication: block 0 spends the start on the next op's header (credit wait, NVLink
  // stores, system fence); it carries no chunks, else it would be the tail CTA whose
  // completion gates the publication (launch_recv adds one CTA for it)
  const uint32_t w0 = (kPub && !kEarly) ? 1u : 0u;
  if (!kEarly && zc_src && a.dyn) {
    // PPC_PULL_DYN: every warp of the worker CTAs claims 4 KiB units of the message from the
    // slot's counter (claim of the next unit in flight with the current unit's loads), so
    // CTAs on SMs with faster NVLink paths take more units and all finish together —
    // with static chunk ranges the first and last CTA finish ~7 us apart
    if (blockIdx.x >= w0) {
      const uint32_t lane = threadIdx.x & 31;
      const uint64_t n_units = (a.bytes + kPullUnit - 1) / kPullUnit;
      uint32_t u = lane == 0 ? atomicAdd(a.next, 1u) : 0u;
      u = __shfl_sync(0xffffffffu, u, 0);
      bool first = true;
      while (u < n_units) {
        const uint32_t nx = lane == 0 ? atomicAdd(a.next, 1u) : 0u;
        const uint64_t off = (uint64_t)u * kPullUnit;
        cta_copy<true>(a.dst + off, zc_src + off, min((uint64_t)kPullUnit, a.bytes - off), lane, 32);
        if (dbg && threadIdx.x == 0 && first) dbg[2] = dbg_stamp_sm();
        first = false;
        u = __shfl_sync(0xffffffffu, nx, 0);
      }
    }
  }
  const ChanIter it = (blockIdx.x >= w0 && !(!kEarly && zc_src && a.dyn))
      ? chan_iter(a.n_chunks, a.channels, blockIdx.x - w0, gridDim.x - w0) : ChanIter{0, 0, 1};
  for (uint32_t c = it.first; c < it.end; c += it.step) {
    const uint64_t off = (uint64_t)c * a.chunk;
    const uint64_t len = min(a.chunk, a.bytes - off);
    if (zc_src) {                      // payload complete at publication: pull it over NVLink
      uint64_t skip = 0;
      if (use_pre && c == it.first) {
        V32* d = reinterpret_cast<V32*>(a.dst + off);
#pragma unroll
        for (int j = 0; j < kEarlyV; ++j) st_data(d + threadIdx.x + j * kThreads, pre[j]);
        skip = (uint64_t)kEarlyV * kThreads * sizeof(V32);
      }
      cta_copy<true>(a.dst + off + skip, zc_src + off + skip, len - skip);
      if (dbg && threadIdx.x == 0 && c == it.first) dbg[2] = dbg_stamp_sm();
      continue;
    }
    int f = 0;
    if (threadIdx.x == 0 && !wait_geq<kSys>(a.flags + c, a.seq, deadline, a.err)) {
      latch(a.err, PPC_ERR_TIMEOUT, a.seq, 0x100u | c << 12);
      f = 1;
    }
    if (__syncthreads_or(f)) return;
    cta_copy<true>(a.dst + off, a.src + off, len);
  }
  __threadfence();                 // slot reads + user-buffer writes before the credit
  __syncthreads();
  if (dbg && threadIdx.x == 0) dbg[3] = globaltimer();
  if (kPub && !kEarly && a0.pub_b0 && threadIdx.x == 0) {
    // The publication is released by block 0, not by the last worker: block 0 fenced its
    // header stores at system scope when it wrote them (off the critical path), so once every
    // worker has arrived it stores the flag and the credit without a second system fence —
    // a fence.sys in the last worker (which has just stored its share of the message) is
    // ~1.3 us on the 1F1B critical path.  Workers' pulls are complete (loads returned) at
    // arrival; the published payload was written by earlier kernels.
    if (blockIdx.x != 0) {
      atomicAdd(a.done, 1u);
    } else if (!wait_arrivals(a.done, gridDim.x - 1, deadline, a.err)) {
      latch(a.err, PPC_ERR_TIMEOUT, a.seq, 0x800u);
    } else {
      *a.done = 0;                 // next use of this slot is stream-ordered after us
      *a.next = 0;                 // every claim (one past the end per warp) is in
      __threadfence();
      chain_post(a);
      fused_publish_flag(&a0.pub, a.peer_credit, a.seq, true);
      if (a.rec) a.rec->t_end_ns = (long long)globaltimer();
    }
  } else if (threadIdx.x == 0) {
    if (atomicAdd(a.done, 1u) == gridDim.x - 1) {
      *a.done = 0;                 // next use of this slot is stream-ordered after us
      *a.next = 0;
      __threadfence();
      chain_post(a);               // a chained successor may start now (before our fence)
      if (kPub) {
        fused_publish_flag(&a0.pub, a.peer_credit, a.seq);
      } else {
        st_rel<kSys>(a.peer_credit, a.seq);
      }
      if (a.rec) a.rec->t_end_ns = (long long)globaltimer();
    }
  }
}

// ---------------------------------------------------------------- K10b: batched receive
// ppc_pp_recv_batch: ONE grid receives n consecutive messages of a direction.  Every CTA
// walks the messages in order and moves on to message i+1 as soon as its own share of
// message i is done, so the tail of one message overlaps the ramp of the next (no grid-wide
// drain + relaunch per message, which costs several us at NVLink rates).  Per message the
// protocol is recv_kernel's: thread 0 acquires the header flag (bounded), checks the header,
// the CTA pulls its chunks (zero-copy) or copies them out behind the chunk flags (ring);
// the CTA that completes the message's count releases its credit.  Credits leave in message
// order without extra waiting: the last CTA of message i+1 counted itself after finishing
// message i, which it did after its own arrival on i (fence + atomic chain), so credit i is
// stored before credit i+1.
// kPub (the step driver's batched terminal receives): message i may carry a fused
// publication of the stage's next zero-copy send, exactly as recv_kernel<kSys, true>: block 0
// writes its header when it reaches message i (and carries no chunks), the message's last
// CTA releases its header flag together with the receive's credit.
template <bool kSys, bool kPub>
__global__ void __launch_bounds__(kThreads) recv_batch_kernel(const __grid_constant__ RecvBatch b) {
  __shared__ const uint8_t* s_zc_src;
  pdl_enter();
  const uint32_t w0 = kPub ? 1u : 0u;            // block 0: publication headers only
  const uint32_t workers = gridDim.x - w0;
  for (uint32_t i = 0; i < b.n; ++i) {
    const RecvArgs a = resolve(b.a[i]);
    uint64_t* const dbg = a.dbg ? a.dbg + 4 * blockIdx.x : nullptr;   // PPC_DBG_STAMPS
    if (dbg && threadIdx.x == 0) dbg[0] = globaltimer();
    int fail = 0;
    uint64_t deadline = 0;
    if (threadIdx.x == 0) {
      const uint64_t t0 = globaltimer();
      deadline = t0 + a.timeout_ns;
      s_zc_src = nullptr;
      if (a.rec && blockIdx.x == 0)
        fill_record(a.rec, (long long)t0, a.rec_src, a.rec_dst, -1, 1, a.seq, a.mb, a.bytes);
      if (kPub && blockIdx.x == 0 && a.has_pub && !fused_publish_header(&b.a[i].pub)) {
        fail = 1;
      } else if (!wait_geq<kSys>(a.hdr_flag, a.seq, deadline, a.err)) {
        latch(a.err, PPC_ERR_TIMEOUT, a.seq, 0x100u);
        fail = 1;
      } else {
        const HdrView h = read_header(a.hdr);
        if (h.magic != kMagic || h.seq != a.seq || h.mb != a.mb) {
          latch(a.err, PPC_ERR_ORDER, a.seq, 0x100u);
          fail = 1;
        } else if (h.bytes != a.bytes) {
          latch(a.err, PPC_ERR_SIZE_MISMATCH, a.seq, 0x100u);
          fail = 1;
        } else if (h.flags & kHdrZeroCopy) {
          const uint64_t base = zc_base(a, h.src_seg);
          if (!base) {
            latch(a.err, PPC_ERR_ORDER, a.seq, 0x300u | h.src_seg << 12);
            fail = 1;
          } else {
            s_zc_src = reinterpret_cast<const uint8_t*>(base + h.src_off);
            if (a.rec && blockIdx.x == 0) a.rec->t_start_ns = (long long)globaltimer();
          }
        }
      }
    }
    if (__syncthreads_or(fail)) return;
    if (dbg && threadIdx.x == 0) dbg[1] = globaltimer();
    const uint8_t* zc_src = s_zc_src;
    if (blockIdx.x >= w0 && zc_src && a.dyn) {
      // dynamic pull units (PPC_PULL_DYN, as recv_kernel): warps claim 4 KiB units of
      // message i; a CTA whose warps find none left moves on to message i + 1
      const uint32_t lane = threadIdx.x & 31;
      const uint64_t n_units = (a.bytes + kPullUnit - 1) / kPullUnit;
      uint32_t u = lane == 0 ? atomicAdd(a.next, 1u) : 0u;
      u = __shfl_sync(0xffffffffu, u, 0);
      while (u < n_units) {
        const uint32_t nx = lane == 0 ? atomicAdd(a.next, 1u) : 0u;
        const uint64_t off = (uint64_t)u * kPullUnit;
        cta_copy<true>(a.dst + off, zc_src + off, min((uint64_t)kPullUnit, a.bytes - off), lane, 32);
        u = __shfl_sync(0xffffffffu, nx, 0);
      }
    } else if (blockIdx.x >= w0) {
      // rotate the chunk ownership per message so the CTAs that carried the last chunks of
      // one message start the next one early
      const uint32_t wid = blockIdx.x - w0;
      const uint32_t first = (wid + i * (a.n_chunks % workers)) % workers;
      for (uint32_t c = first; c < a.n_chunks; c += workers) {
        const uint64_t off = (uint64_t)c * a.chunk;
        const uint64_t len = min(a.chunk, a.bytes - off);
        if (zc_src) {
          cta_copy<true>(a.dst + off, zc_src + off, len);
          if (dbg && threadIdx.x == 0 && c == first) dbg[2] = dbg_stamp_sm();
          continue;
        }
        int f = 0;
        if (threadIdx.x == 0 && !wait_geq<kSys>(a.flags + c, a.seq, deadline, a.err)) {
          latch(a.err, PPC_ERR_TIMEOUT, a.seq, 0x100u | c << 12);
          f = 1;
        }
        if (__syncthreads_or(f)) return;
        cta_copy<true>(a.dst + off, a.src + off, len);
      }
    }
    __threadfence();
    __syncthreads();
    if (dbg && threadIdx.x == 0) dbg[3] = globaltimer();
    if (threadIdx.x == 0) {
      if (atomicAdd(a.done, 1u) == gridDim.x - 1) {
        *a.done = 0;
        *a.next = 0;
        __threadfence();
        chain_post(a);
        if (kPub && a.has_pub) {
          fused_publish_flag(&b.a[i].pub, a.peer_credit, a.seq);
        } else {
          st_rel<kSys>(a.peer_credit, a.seq);
        }
        if (a.rec) a.rec->t_end_ns = (long long)globaltimer();
      }
    }
  }
}

cudaError_t launch_recv_batch(const RecvBatch& b, int grid, bool sys, cudaStream_t s) {
  bool pub = false;
  for (uint32_t i = 0; i < b.n; ++i) pub = pub || b.a[i].has_pub;
  auto k = pub ? (sys ? recv_batch_kernel<true, true> : recv_batch_kernel<false, true>)
               : (sys ? recv_batch_kernel<true, false> : recv_batch_kernel<false, false>);
  if (sys) grid = std::min(grid, kMaxSpinGrid);
  grid = fit_grid(k, grid + (pub ? 1 : 0), kThreads);
  return launch_k(k, grid, kThreads, s, pdl_fits(k, grid, kThreads), b);
}

// ---------------------------------------------------------------- TP-sliced gather (NEXT-1)
__global__ void __launch_bounds__(kThreads) gather_kernel(GatherArgs a) {
  pdl_enter();
  __shared__ const uint8_t* s_src[kMaxTp];
  const uint64_t deadline = globaltimer() + a.timeout_ns;
  if (threadIdx.x == 0)
    for (uint32_t t = 0; t < a.tp; ++t) s_src[t] = nullptr;
  __syncthreads();
  // every CTA pulls (slice, chunk) units of all TP senders over NVLink into its slot of dst.
  // Units interleave the senders (consecutive units come from different senders) and each
  // receiver starts at its own TP index, so at any time a receiver pulls from every sender
  // and every sender serves every receiver — not all receivers draining sender 0 first
  // (measured: 322 GB/s per receiver sender-major vs the replicated boundary's 607).  A
  // sender's header (published in that sender's PP peer's arena) is acquired when the CTA
  // first needs a unit of it, so pulling from the own sender (header in our arena) starts
  // before the other senders' publications are seen.
  const uint32_t units = a.tp * a.n_chunks;
  for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
    const uint32_t t = (u + a.my_tp) % a.tp, c = u / a.tp;
    // every thread reads s_src[t] before thread 0 may set it below: a warp still finishing
    // the previous unit's copy must not see it already set and skip the barrier the others
    // wait at (cta_copy has no barrier, so warps drift apart by a loaded NVLink round trip)
    const bool need = !s_src[t];
    __syncthreads();
    if (need) {
      int fail = 0;
      if (threadIdx.x == 0) {
        if (!wait_geq<true>(a.hdr_flag[t], a.seq, deadline, a.err)) {
          latch(a.err, PPC_ERR_TIMEOUT, a.seq, 0x400u | t << 12);
          fail = 1;
        } else {
          const HdrView h = read_header(a.hdr[t]);
          if (h.magic != kMagic || h.seq != a.seq || h.mb != a.mb || !(h.flags & kHdrZeroCopy)) {
            latch(a.err, PPC_ERR_ORDER, a.seq, 0x400u | t << 12);
            fail = 1;
          } else if (h.bytes != a.slice_bytes) {
            latch(a.err, PPC_ERR_SIZE_MISMATCH, a.seq, 0x400u | t << 12);
            fail = 1;
          } else {
            const uint64_t base = h.src_seg < (uint32_t)kMaxSeg ? a.seg_tab[t][h.src_seg] : 0;
            if (!base) {
              latch(a.err, PPC_ERR_ORDER, a.seq, 0x500u | t << 12);
              fail = 1;
            } else {
              s_src[t] = reinterpret_cast<const uint8_t*>(base + h.src_off);
            }
          }
        }
      }
      if (__syncthreads_or(fail)) return;
    }
    const uint64_t off = (uint64_t)c * a.chunk;
    const uint64_t len = min(a.chunk, a.slice_bytes - off);
    cta_copy<true>(a.dst + (uint64_t)t * a.slice_bytes + off, s_src[t] + off, len);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(a.done, 1u) == gridDim.x - 1) {
    *a.done = 0;
    __threadfence_system();
    for (uint32_t t = 0; t < a.tp; ++t) atomicAdd_system(a.gdone[t], 1ull);   // "pulled"
    // our sender's slice may be reused once EVERY receiver of the stage has pulled it: that
    // wait (and the credit) is gather_credit_kernel's, on a side stream, so the next gather
    // on this stream does not queue behind the slowest receiver
  }
}

// The credit of a TP-sliced gather: once every receiver of the stage counted its pull of our
// sender's slice (gdone >= gtarget), release the sender's credit.  One thread, bounded.
__global__ void gather_credit_kernel(const unsigned long long* gdone, uint64_t gtarget,
                                     uint64_t* peer_credit, uint64_t seq, ErrWord* err,
                                     uint64_t timeout_ns) {
  pdl_enter();
  if (!wait_geq<true>(reinterpret_cast<const uint64_t*>(gdone), gtarget,
                      globaltimer() + timeout_ns, err)) {
    latch(err, PPC_ERR_TIMEOUT, seq, 0x600u);
    return;
  }
  st_release_sys(peer_credit, seq);
}

cudaError_t launch_gather_credit(const GatherArgs& a, cudaStream_t s) {
  return launch_k(gather_credit_kernel, 1, 1, s, true,
                  static_cast<const unsigned long long*>(a.gdone[a.my_tp]), a.gtarget,
                  a.peer_credit, a.seq, a.err, a.timeout_ns);
}

cudaError_t launch_gather(const GatherArgs& a, int grid, cudaStream_t s) {
  grid = fit_grid(gather_kernel, std::min(grid, kMaxSpinGrid), kThreads);
  return launch_k(gather_kernel, grid, kThreads, s, pdl_fits(gather_kernel, grid, kThreads), a);
}

// ---------------------------------------------------------------- zero-copy publication
// The payload stays in the sender's registered buffer; one thread waits for the slot's
// credit and publishes (segment, offset) in the receiver's slot header.  The stream then
// waits for the receiver's credit (launch_wait_credit) before the buffer may be reused.
__global__ void publish_kernel(PublishArgs a0) {
  pdl_enter();
  publish_body(resolve(a0));
}

cudaError_t launch_publish(const PublishArgs& a, cudaStream_t s) {
  return launch_k(publish_kernel, 1, 1, s, true, a);
}

// ---------------------------------------------------------------- K12: CE signalling
__global__ void ce_head_kernel(CeHeadArgs a) {
  pdl_enter();
  const uint64_t t0 = globaltimer();
  if (a.rec) fill_record(a.rec, (long long)t0, a.rec_src, a.rec_dst, a.dir, 0, a.seq, a.mb, a.bytes);
  if (a.need_credit && !wait_geq(a.credit, a.need_credit, t0 + a.timeout_ns, a.err)) {
    latch(a.err, PPC_ERR_TIMEOUT, a.seq, a.dir);
    return;
  }
  SlotHeader h = {};
  h.magic = kMagic;
  h.dir = (uint8_t)a.dir;
  h.boundary = (uint8_t)a.boundary;
  h.bytes = a.bytes;
  h.seq = a.seq;
  h.mb = a.mb;
  h.step = a.step;
  const uint4* hs = reinterpret_cast<const uint4*>(&h);
  uint4* hd = reinterpret_cast<uint4*>(a.hdr);
#pragma unroll
  for (int j = 0; j < 4; ++j) st_data(hd + j, hs[j]);
  st_release_sys(a.hdr_flag, a.seq);
}

// Runs after the copy engine finished this channel's bytes (stream order).
__global__ void ce_flags_kernel(uint64_t* flags, uint32_t c0, uint32_t c1, uint64_t seq,
                                ppc_record_t* rec) {
  pdl_enter();
  fence_acq_rel_sys();
  for (uint32_t c = c0 + threadIdx.x; c < c1; c += blockDim.x) st_release_sys(flags + c, seq);
  if (rec && threadIdx.x == 0) rec->t_end_ns = (long long)globaltimer();
}

// Wait until the receiver consumed `target` (credit protocol), bounded.
__global__ void wait_credit_kernel(const uint64_t* credit, uint64_t target, ErrWord* err,
                                   uint64_t timeout_ns, const uint64_t* seq_base) {
  pdl_enter();
  if (seq_base) target += *seq_base;
  if (!wait_geq(credit, target, globaltimer() + timeout_ns, err)) latch(err, PPC_ERR_TIMEOUT, target, 0x200u);
}

__global__ void set_seq_kernel(uint64_t* seq, uint64_t v0, uint64_t v1, uint64_t v2, uint64_t v3) {
  seq[0] = v0;
  seq[1] = v1;
  seq[2] = v2;
  seq[3] = v3;
}

cudaError_t launch_set_seq(uint64_t* seq, uint64_t v0, uint64_t v1, uint64_t v2, uint64_t v3,
                           cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  set_seq_kernel<<<1, 1, 0, s>>>(seq, v0, v1, v2, v3);
  return cudaGetLastError();
}

template <typename T>
__global__ void add_kernel(T* __restrict__ dst, const T* __restrict__ src, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = dst[i] + src[i];
}

cudaError_t launch_add(void* dst, const void* src, size_t count, int dtype, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  const int grid = (int)std::min<size_t>((count + 255) / 256, 148 * 8);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  switch (dtype) {
    case 0: add_kernel<float><<<grid, 256, 0, s>>>((float*)dst, (const float*)src, count); break;
    case 1: add_kernel<__half><<<grid, 256, 0, s>>>((__half*)dst, (const __half*)src, count); break;
    case 2:
      add_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((__nv_bfloat16*)dst,
                                                     (const __nv_bfloat16*)src, count);
      break;
    case 3: add_kernel<int32_t><<<grid, 256, 0, s>>>((int32_t*)dst, (const int32_t*)src, count); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// K11: same-GPU single copy.  32-B aligned buffers: grid-stride over 32-B vectors with
// kCopyU predicated loads in flight per thread before their stores, so every size spreads
// evenly over the grid in one pass (no dependent load->store tail per thread, no partial
// last wave of chunks); otherwise per-CTA chunks of `chunk` bytes (cta_copy handles any
// alignment).
constexpr int kCopyU = 4;
__global__ void __launch_bounds__(kThreads, 2) copy_kernel(uint8_t* dst, const uint8_t* src,
                                                        uint64_t bytes, uint64_t chunk) {
  pdl_enter();
  if ((((uintptr_t)dst | (uintptr_t)src) & 31) != 0) {
    const uint64_t n = (bytes + chunk - 1) / chunk;
    for (uint64_t c = blockIdx.x; c < n; c += gridDim.x) {
      const uint64_t off = c * chunk;
      cta_copy<false>(dst + off, src + off, min(chunk, bytes - off));
    }
    return;
  }
  const uint64_t nv = bytes / sizeof(V32);
  const V32* s = reinterpret_cast<const V32*>(src);
  V32* d = reinterpret_cast<V32*>(dst);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (uint64_t b = t; b < nv; b += kCopyU * stride) {
    V32 v[kCopyU];
#pragma unroll
    for (int j = 0; j < kCopyU; ++j)
      if (b + j * stride < nv) v[j] = ld_src(s + b + j * stride);
#pragma unroll
    for (int j = 0; j < kCopyU; ++j)
      if (b + j * stride < nv) st_data(d + b + j * stride, v[j]);
  }
  for (uint64_t k = nv * sizeof(V32) + t; k < bytes; k += stride) dst[k] = src[k];
}

// K11 (TMA engine): the same copy through shared memory with bulk async copies
// (cp.async.bulk global->shared completing on an mbarrier, shared->global in bulk groups).
// One elected thread per CTA drives a kTmaStages-deep ring of kTmaTile-byte tiles; each CTA
// owns a contiguous range of tiles.  Tile i+kTmaStages-1 is loaded into the stage tile i-1
// used once that tile's store has finished reading shared memory (wait_group.read 1), so the
// newest store and kTmaStages-1 loads stay in flight.  Needs 16-B aligned dst/src (bulk
// copies move 16-B multiples); the last (bytes % 16) bytes are copied by thread 0 of the
// last CTA.  Measured alone (tools/nvlink_probe hbm, profiles/r55_hbm_copy_probe.jsonl):
// 8.3 us per 32 MiB vs 9.1 us for the SIMT copy at 148 CTAs; ncu in the step 11.1 vs
// 11.8 us.  Inside the N=1 step, where F and B copies overlap, the SIMT copy is faster
// (188.5 vs 190.9-193.9 us per step, profiles/r56_copy_engine_ab.jsonl), so it stays the
// default and this engine is opt-in (PPC_COPY_TMA_CTAS > 0).
constexpr int kTmaStages = 6;
constexpr uint32_t kTmaTile = 16u << 10;
constexpr uint32_t kTmaSmem = kTmaStages * kTmaTile;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void tma_ld(void* sdst, const void* gsrc, uint32_t n, uint64_t* mbar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_addr(mbar)), "r"(n) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_addr(sdst)), "l"(gsrc), "r"(n), "r"(smem_addr(mbar)) : "memory");
}
__device__ __forceinline__ void tma_st(void* gdst, const void* ssrc, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               ::"l"(gdst), "r"(smem_addr(ssrc)), "r"(n) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* mbar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(mbar)), "r"(phase) : "memory");
}

__global__ void __launch_bounds__(32) copy_tma_kernel(uint8_t* dst, const uint8_t* src,
                                                      uint64_t bytes) {
  extern __shared__ __align__(128) uint8_t tiles[];
  __shared__ __align__(8) uint64_t mbar[kTmaStages];
  pdl_enter();
  if (threadIdx.x != 0) return;
  const uint64_t body = bytes & ~15ull;
  if (blockIdx.x == gridDim.x - 1)
    for (uint64_t k = body; k < bytes; ++k) dst[k] = src[k];
  const uint64_t ntiles = (body + kTmaTile - 1) / kTmaTile;
  const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * per, t1 = min(ntiles, t0 + per);
  if (t0 >= t1) return;
  const uint64_t n = t1 - t0;
  auto len = [&](uint64_t t) { return (uint32_t)min((uint64_t)kTmaTile, body - t * kTmaTile); };
  for (int k = 0; k < kTmaStages; ++k)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&mbar[k])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  for (uint64_t j = 0; j < n && j < (uint64_t)kTmaStages; ++j)
    tma_ld(tiles + j * kTmaTile, src + (t0 + j) * kTmaTile, len(t0 + j), &mbar[j]);
  for (uint64_t i = 0; i < n; ++i) {
    const int st = (int)(i % kTmaStages);
    mbar_wait_parity(&mbar[st], (uint32_t)((i / kTmaStages) & 1));
    tma_st(dst + (t0 + i) * kTmaTile, tiles + st * kTmaTile, len(t0 + i));
    const uint64_t j = i - 1 + kTmaStages;   // refill the stage tile i-1 used
    if (i >= 1 && j < n) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      const int sj = (int)((i - 1) % kTmaStages);
      tma_ld(tiles + sj * kTmaTile, src + (t0 + j) * kTmaTile, len(t0 + j), &mbar[sj]);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


cudaError_t launch_copy(void* dst, const void* src, uint64_t bytes, uint64_t chunk, int grid,
                        cudaStream_t s) {
  if (bytes == 0) return cudaSuccess;
  if (g_copy_tma_ctas > 0 && bytes >= 16 && (((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const uint64_t ntiles = ((bytes & ~15ull) + kTmaTile - 1) / kTmaTile;
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g_copy_tma_ctas, ntiles));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = kTmaSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_pdl ? 1 : 0;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaLaunchKernelEx(&cfg, copy_tma_kernel, static_cast<uint8_t*>(dst),
                              static_cast<const uint8_t*>(src), bytes);
  }
  return launch_k(copy_kernel, grid, kThreads, s, true, static_cast<uint8_t*>(dst),
                  static_cast<const uint8_t*>(src), bytes, chunk);
}

// PPC_WAIT_VALUE=1 (opt-in, eager enqueues only): the credit wait becomes a stream memory
// operation, cuStreamWaitValue64(GEQ) — zero SMs, no kernel.  It cannot be bounded (no
// timeout: a lost credit hangs the stream instead of latching PPC_ERR_TIMEOUT), and
// its value is fixed at enqueue, so graph captures (device-relative sequence numbers) keep
// the bounded 1-thread kernel.  Measured against the kernel in DESIGN.md §7.
int g_wait_value = 0;
namespace {
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
WaitValueFn wait_value_fn() {
  static WaitValueFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (WaitValueFn) nullptr;
    return reinterpret_cast<WaitValueFn>(f);
  }();
  return fn;
}
}  // namespace

cudaError_t launch_wait_credit(const uint64_t* credit, uint64_t target, ErrWord* err,
                               uint64_t timeout_ns, cudaStream_t s, const uint64_t* seq_base) {
  if (g_wait_value && !seq_base) {
    if (WaitValueFn fn = wait_value_fn()) {
      return fn((CUstream)s, (CUdeviceptr)(uintptr_t)credit, (cuuint64_t)target,
                CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS ? cudaSuccess : cudaErrorUnknown;
    }
  }
  return launch_k(wait_credit_kernel, 1, 1, s, true, credit, target, err, timeout_ns, seq_base);
}

cudaError_t launch_push(const PushArgs& a, int grid, bool sys, bool ws, cudaStream_t s) {
  if (ws) {
    auto k = sys ? push_ws_kernel<true> : push_ws_kernel<false>;
    grid = fit_grid(k, grid, kWsThreads);
    return launch_k(k, grid, kWsThreads, s, pdl_fits(k, grid, kWsThreads), a);
  }
  auto k = sys ? push_kernel<true> : push_kernel<false>;
  grid = fit_grid(k, grid, kThreads);
  return launch_k(k, grid, kThreads, s, pdl_fits(k, grid, kThreads), a);
}
cudaError_t launch_recv(const RecvArgs& a, int grid, bool sys, cudaStream_t s) {
  auto k = a.has_pub ? (sys ? recv_kernel<true, true> : recv_kernel<false, true>)
                     : (sys ? recv_kernel<true, false> : recv_kernel<false, false>);
  if (sys) grid = std::min(grid, kMaxSpinGrid);
  grid = fit_grid(k, grid, kThreads);
  if (sys && g_pdl && g_recv_early) {   // zero-copy pulls over NVLink; without PDL nothing runs early
    auto ke = a.has_pub ? recv_kernel<true, true, true> : recv_kernel<true, false, true>;
    if (pdl_fits(ke, grid, kThreads)) return launch_k(ke, grid, kThreads, s, true, a);
  }
  if (a.has_pub) grid = fit_grid(k, grid + 1, kThreads);   // + the header-only block 0
  const bool pdl = pdl_fits(k, grid, kThreads);
  return launch_k(k, grid, kThreads, s, pdl, a);
}
cudaError_t launch_ce_head(const CeHeadArgs& a, cudaStream_t s, bool pdl) {
  return launch_k(ce_head_kernel, 1, 1, s, pdl, a);
}
cudaError_t launch_ce_flags(uint64_t* flags, uint32_t c0, uint32_t c1, uint64_t seq,
                            ppc_record_t* rec, cudaStream_t s, bool pdl) {
  return launch_k(ce_flags_kernel, 1, 32, s, pdl, flags, c0, c1, seq, rec);
}

// Force-load every transport kernel on the current device.  With lazy module loading
// (CUDA_MODULE_LOADING=LAZY, the CUDA 12 default) the first launch of a kernel loads it,
// and that load can wait for the device to go idle: a rank whose wait_credit_kernel is
// spinning on a peer would then block the peer's first receive launch until the wait
// times out.  Touching the functions up front (cudaFuncGetAttributes loads them) keeps
// every later launch free of module loads.
__global__ void __launch_bounds__(kWsThreads) xor_send_kernel(uint8_t* out, uint64_t* flags,
                                                              uint64_t seq, const uint8_t* in,
                                                              uint64_t bytes, uint64_t chunk,
                                                              uint32_t n_chunks, uint64_t key);
__global__ void splitmix_xor_kernel(uint8_t* out, const uint8_t* in, uint64_t bytes, uint64_t key);
cudaError_t preload_kernels() {
  cudaFuncAttributes fa;
  const void* fns[] = {
      (const void*)push_kernel<true>,      (const void*)push_kernel<false>,
      (const void*)push_ws_kernel<true>,   (const void*)push_ws_kernel<false>,
      (const void*)recv_kernel<true, false>, (const void*)recv_kernel<false, false>,
      (const void*)recv_kernel<true, false, true>, (const void*)recv_kernel<true, true, true>,
      (const void*)recv_kernel<true, true>,  (const void*)recv_kernel<false, true>,
      (const void*)recv_batch_kernel<true, false>, (const void*)recv_batch_kernel<false, false>,
      (const void*)recv_batch_kernel<true, true>, (const void*)recv_batch_kernel<false, true>,
      (const void*)gather_kernel,          (const void*)publish_kernel,
      (const void*)gather_credit_kernel,
      (const void*)ce_head_kernel,         (const void*)ce_flags_kernel,
      (const void*)wait_credit_kernel,     (const void*)set_seq_kernel,
      (const void*)add_kernel<float>,      (const void*)add_kernel<__half>,
      (const void*)add_kernel<__nv_bfloat16>, (const void*)add_kernel<int32_t>,
      (const void*)copy_kernel,            (const void*)xor_send_kernel,
      (const void*)splitmix_xor_kernel,
  };
  for (const void* f : fns) {
    const cudaError_t e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return e;
  }
  return cudaFuncSetAttribute(copy_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)kTmaSmem);
}

// ---------------------------------------------------------------- K14: test kernels
// SplitMix64 (synth/payload.py, implemented independently here):
//   key = seed<<48 ^ step<<32 ^ boundary<<24 ^ dir<<23 ^ mb ; base = mix(key + G)
//   word[w] = mix(base + (w+1)*G)
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t payload_key(int seed, int step, int boundary, int dir,
                                                long long mb) {
  return ((uint64_t)(uint32_t)seed << 48) ^ ((uint64_t)(uint32_t)step << 32) ^
         ((uint64_t)(uint32_t)boundary << 24) ^ ((uint64_t)(uint32_t)dir << 23) ^ (uint64_t)mb;
}

// out = in XOR stream (in == nullptr: out = stream).  Whole words as u64, ragged tail bytewise.
__global__ void splitmix_xor_kernel(uint8_t* out, const uint8_t* in, uint64_t bytes, uint64_t key) {
  const uint64_t base = mix64(key + kGamma);
  const uint64_t nw = bytes >> 3;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const bool aligned = ((((uintptr_t)out) | ((uintptr_t)in)) & 7) == 0;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += stride) {
    uint64_t v = mix64(base + (w + 1) * kGamma);
    if (aligned) {
      if (in) v ^= reinterpret_cast<const uint64_t*>(in)[w];
      reinterpret_cast<uint64_t*>(out)[w] = v;
    } else {
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        uint8_t x = (uint8_t)(v >> (8 * b));
        if (in) x ^= in[w * 8 + b];
        out[w * 8 + b] = x;
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (bytes & 7)) {
    const uint64_t v = mix64(base + (nw + 1) * kGamma);
    for (uint64_t k = nw * 8; k < bytes; ++k) {
      uint8_t x = (uint8_t)(v >> (8 * (k & 7)));
      if (in) x ^= in[k];
      out[k] = x;
    }
  }
}

// The XOR stage proxy fused with its send (ppc_stage_xor_send): the stage's output goes
// straight into the receiver's slot over NVLink, so the receiver copies chunk c out while
// later chunks are still being produced.  Warp-specialised like push_ws_kernel: warps 1..16
// compute out = in ^ stream and store it with 32-B vectors (st.global.v8, 4 stream words
// per thread per step), chunk after chunk of the CTA's chunks; each finished chunk is handed
// through an mbarrier ring to warp 0, which issues fence.acq_rel.sys + st.release.sys of
// that chunk's flag while the copy warps already store the next chunk (r1: CTA per chunk,
// 16-B stores, a CTA-wide barrier + fence before every flag: 537 GB/s).
__global__ void __launch_bounds__(kWsThreads) xor_send_kernel(uint8_t* out, uint64_t* flags,
                                                              uint64_t seq, const uint8_t* in,
                                                              uint64_t bytes, uint64_t chunk,
                                                              uint32_t n_chunks, uint64_t key) {
  pdl_enter();                     // the slot's credit wait (ce_head_kernel) has completed
  __shared__ __align__(8) uint64_t full[kWsRing], empty[kWsRing];
  if (threadIdx.x == 0) {
    for (int b = 0; b < kWsRing; ++b) {
      mbar_init(&full[b], kWsCopyWarps);
      mbar_init(&empty[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t base = mix64(key + kGamma);
  const bool vec = ((((uintptr_t)out) | ((uintptr_t)in)) & 31) == 0 && (chunk & 31) == 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t i = 0;
  if (warp == 0) {                                   // signal warp
    if (lane == 0) {
      for (uint32_t c = blockIdx.x; c < n_chunks; c += gridDim.x, ++i) {
        const int b = i % kWsRing;
        mbar_wait(&full[b], (i / kWsRing) & 1);
        fence_acq_rel_sys();
        st_release_sys(flags + c, seq);
        mbar_arrive(&empty[b]);
      }
    }
    return;
  }
  const uint64_t tid = threadIdx.x - 32, nt = 32 * kWsCopyWarps;
  for (uint32_t c = blockIdx.x; c < n_chunks; c += gridDim.x, ++i) {
    const int b = i % kWsRing;
    if (i >= kWsRing) mbar_wait(&empty[b], ((i / kWsRing) - 1) & 1);
    const uint64_t off = (uint64_t)c * chunk, end = min(off + chunk, bytes);
    uint64_t k = off;
    if (vec) {                     // 4-word quads (w .. w+3), w a multiple of 4, in the chunk
      const uint64_t nq = (end - off) / 32;
      for (uint64_t q = tid; q < nq; q += nt) {
        const uint64_t w = off / 8 + 4 * q;
        uint64_t v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = mix64(base + (w + 1 + j) * kGamma);
        if (in) {
          const V32 x = ld_src(reinterpret_cast<const V32*>(in + 8 * w));
          v[0] ^= (uint64_t)x.lo.x | (uint64_t)x.lo.y << 32;
          v[1] ^= (uint64_t)x.lo.z | (uint64_t)x.lo.w << 32;
          v[2] ^= (uint64_t)x.hi.x | (uint64_t)x.hi.y << 32;
          v[3] ^= (uint64_t)x.hi.z | (uint64_t)x.hi.w << 32;
        }
        V32 y;
        y.lo = make_uint4((uint32_t)v[0], (uint32_t)(v[0] >> 32), (uint32_t)v[1], (uint32_t)(v[1] >> 32));
        y.hi = make_uint4((uint32_t)v[2], (uint32_t)(v[2] >> 32), (uint32_t)v[3], (uint32_t)(v[3] >> 32));
        st_data(reinterpret_cast<V32*>(out + 8 * w), y);
      }
      k = off + nq * 32;
    }
    for (uint64_t bb = k + tid; bb < end; bb += nt) {   // bytewise remainder
      const uint64_t v = mix64(base + (bb / 8 + 1) * kGamma);
      uint8_t x = (uint8_t)(v >> (8 * (bb & 7)));
      if (in) x ^= in[bb];
      out[bb] = x;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&full[b]);
  }
}

}  // namespace ppc

extern "C" ppc_status_t ppc_stage_xor_send(const ppc_slot_t* slot, const ppc_xor_ctx_t* ctx,
                                           int mb, const void* in, size_t bytes,
                                           cudaStream_t s) {
  if (!slot || !ctx || !slot->payload || !slot->flags || bytes == 0 || bytes != slot->bytes ||
      slot->chunk_bytes == 0 || slot->n_chunks != (bytes + slot->chunk_bytes - 1) / slot->chunk_bytes)
    return PPC_ERR_INVALID_ARG;
  // two 544-thread CTAs per SM; a CTA walks several chunks when there are more than that
  static const int max_grid = [] {
    const char* v = getenv("PPC_XOR_SEND_CTAS");
    return v && *v ? std::max(1, atoi(v)) : 296;
  }();
  const int grid = (int)std::min<uint32_t>(slot->n_chunks, (uint32_t)max_grid);
  const cudaError_t e = ppc::launch_k(
      ppc::xor_send_kernel, grid, ppc::kWsThreads, s, true, static_cast<uint8_t*>(slot->payload),
      reinterpret_cast<uint64_t*>(slot->flags), (uint64_t)slot->seq,
      static_cast<const uint8_t*>(in), (uint64_t)bytes, (uint64_t)slot->chunk_bytes,
      (uint32_t)slot->n_chunks,
      ppc::payload_key(ctx->seed ^ 0x8000, ctx->step, ctx->stage, ctx->dir, mb));
  return e == cudaSuccess ? PPC_OK : PPC_ERR_CUDA;
}

extern "C" ppc_status_t ppc_fill_payload(void* buf, size_t bytes, int seed, int step,
                                         int boundary, int dir, long long mb, cudaStream_t s) {
  if (bytes == 0) return PPC_OK;
  if (!buf || seed < 0 || seed >= (1 << 16) || step < 0 || step >= (1 << 16) || boundary < 0 ||
      boundary > 255 || (dir != 0 && dir != 1) || mb < 0 || mb >= (1ll << 23))
    return PPC_ERR_INVALID_ARG;
  const uint64_t nw = (bytes + 7) / 8;
  const int grid = (int)std::min<uint64_t>((nw + 255) / 256, 148ull * 8);
  ppc::g_launches.fetch_add(1, std::memory_order_relaxed);
  ppc::splitmix_xor_kernel<<<grid, 256, 0, s>>>(static_cast<uint8_t*>(buf), nullptr, bytes,
                                               ppc::payload_key(seed, step, boundary, dir, mb));
  return cudaGetLastError() == cudaSuccess ? PPC_OK : PPC_ERR_CUDA;
}

extern "C" int ppc_stage_xor(void* user, int mb, const void* in, void* out, size_t in_bytes,
                             size_t out_bytes, cudaStream_t s) {
  const ppc_xor_ctx_t* c = static_cast<const ppc_xor_ctx_t*>(user);
  if (!c || !out || (in && in_bytes != out_bytes)) return PPC_ERR_INVALID_ARG;
  if (out_bytes == 0) return PPC_OK;
  const uint64_t nw = (out_bytes + 7) / 8;
  const int grid = (int)std::min<uint64_t>((nw + 255) / 256, 148ull * 8);
  ppc::g_launches.fetch_add(1, std::memory_order_relaxed);
  ppc::splitmix_xor_kernel<<<grid, 256, 0, s>>>(
      static_cast<uint8_t*>(out), static_cast<const uint8_t*>(in), out_bytes,
      ppc::payload_key(c->seed ^ 0x8000, c->step, c->stage, c->dir, mb));
  return cudaGetLastError() == cudaSuccess ? PPC_OK : PPC_ERR_CUDA;
}

extern "C" unsigned long long ppc_launch_count(void) {
  return ppc::g_launches.load(std::memory_order_relaxed);
}
