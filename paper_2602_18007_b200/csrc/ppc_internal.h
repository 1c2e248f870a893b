// Internal declarations of libppc (not part of the C ABI).
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>
#include "ppc.h"

namespace ppc {

constexpr uint32_t kMagic = 0x48435043u;     // SPEC.md S:L403 chunk-header magic, reused
constexpr int kThreads = 512;                // CTA size of the copy kernels
constexpr int kMaxSlots = 64;
constexpr int kMaxSeg = 256;                 // registered send buffers per peer
constexpr uint16_t kHdrZeroCopy = 1;         // header flag: payload is in a registered buffer
constexpr uint32_t kArenaSeg = 0xFFFFFFFFu;  // zero-copy src_seg: the sender's own arena
                                             // (the step driver's buffers live there)

// 64-byte slot header, little-endian.  Ring path: the payload is in
// the slot.  Zero-copy path (flags & kHdrZeroCopy): the payload stays in the sender's
// registered buffer (segment src_seg, offset src_off) and the receiver pulls it.
struct __align__(64) SlotHeader {
  uint32_t magic;
  uint8_t dir, boundary;
  uint16_t flags;
  uint64_t bytes;
  uint64_t seq;
  int64_t mb;
  uint64_t step;
  uint64_t src_off;
  uint32_t src_seg;
  uint8_t pad[12];
};
static_assert(sizeof(SlotHeader) == 64, "slot header is 64 B");

// Sticky error record in mapped host memory (the host polls it without synchronising):
// code = status, seq = message seq, info = where (see ppc_error_info).
struct ErrHost {
  unsigned code, seq, info, pad;
};
// What the kernels get: a claim word in DEVICE memory plus the mapped host record.  The first
// failing thread wins the claim (atomicCAS; every kernel that latches into a comm's record
// runs on that comm's device), then writes seq and info and, after a system fence, code —
// so the record is never torn and the host never sees a code without its seq / info.
struct ErrWord {
  unsigned claim, pad;
  ErrHost* host;      // device pointer of the mapped host record
};

// Graph-capturable sequence numbers.  base == nullptr: `seq` in the kernel args is absolute
// and every slot pointer is already resolved by the host.  Otherwise (a captured CUDA graph)
// seq = args.seq + *base, where *base is a device counter set before each graph launch, and
// the kernel resolves the slot (seq % K) pointers from the slot-0 bases itself.
struct SeqRef {
  const uint64_t* base;
  uint64_t stride;             // payload bytes per slot
  uint32_t K, fstride;         // slots; chunk flags per slot
  uint32_t wait_credit;        // wait credit >= seq - K (cross-GPU) or not (virtual stages)
  uint32_t pad;
};

struct PushArgs {
  SeqRef sr;
  const uint8_t* src;
  uint8_t* dst;                 // peer (or local) slot payload
  SlotHeader* hdr;              // peer slot header
  uint64_t* hdr_flag;           // peer: = seq once the header is written
  uint64_t* flags;              // peer: flags[c] = seq once chunk c is written
  const uint64_t* credit;       // local: last seq the receiver consumed
  uint64_t need_credit;         // wait until credit >= need_credit (0: no wait)
  uint64_t bytes, chunk;
  uint32_t n_chunks;
  uint64_t seq;
  int64_t mb;
  uint64_t step;
  uint32_t dir, boundary;
  ErrWord* err;
  uint64_t timeout_ns;
  ppc_record_t* rec;            // trace record or nullptr
  int rec_src, rec_dst;
  uint32_t* done;               // completion counter (trace only)
  uint32_t channels;            // MPDT channels: contiguous chunk ranges per CTA group
};

// Zero-copy publication of a registered send buffer: credit wait, header, header flag.
struct PublishArgs {
  SeqRef sr;
  SlotHeader* hdr;
  uint64_t* hdr_flag;
  const uint64_t* credit;
  uint64_t need_credit;
  uint64_t bytes, seq, src_off;
  int64_t mb;
  uint32_t src_seg, dir, boundary;
  uint32_t gpu_fence;             // PPC_PUB_FENCE=gpu (opt-in): fused flag release without the
                                  // system fence (the header was already fenced by block 0)
  ErrWord* err;
  uint64_t timeout_ns;
  ppc_record_t* rec;              // trace: publish kernel entry .. header flag stored
  int rec_src, rec_dst;
};

struct RecvArgs {
  SeqRef sr;
  uint8_t* dst;                 // user buffer
  const uint8_t* src;           // local slot payload
  const SlotHeader* hdr;
  const uint64_t* hdr_flag;
  const uint64_t* flags;
  uint64_t* peer_credit;        // sender's credit word (peer memory)
  uint32_t* done;               // local completion counter of this slot
  uint32_t* next;               // zero-copy pull: unit claim counter of this slot (dyn)
  uint32_t dyn;                 // zero-copy pull: warps claim 4 KiB units (PPC_PULL_DYN)
  uint64_t bytes, chunk;
  uint32_t n_chunks;
  uint64_t seq;
  int64_t mb;
  ErrWord* err;
  uint64_t timeout_ns;
  ppc_record_t* rec;
  int rec_src, rec_dst;
  const uint64_t* seg_tab;      // zero-copy: mapped bases of the sender's registered buffers
  const uint8_t* peer_arena;    // zero-copy from the sender's arena (src_seg == kArenaSeg)
  uint32_t channels;            // MPDT channels of the pulling / copy-out CTAs
  uint64_t* dbg;                // PPC_DBG_STAMPS: 4 %globaltimer stamps per CTA, or nullptr
  // fused publication (step driver): when has_pub, the last CTA publishes `pub` (the next
  // op's zero-copy send) right after releasing this receive's credit
  uint32_t has_pub;
  uint32_t pub_b0;              // the publication is released by block 0 (PPC_PUB_BLOCK0)
  PublishArgs pub;
  // chained receives (step driver, PPC_RECV_CHAIN): a receive whose stream predecessor is
  // another receive starts when that one has finished its data phase — posted as its
  // resolved seq in a local per-direction word — instead of at griddepcontrol.wait, i.e.
  // after the predecessor grid's exit and PDL release (and off its publication fence)
  uint64_t* chain_post;         // this receive's direction word (atomicMax of its seq), or nullptr
  const uint64_t* chain_wait;   // the predecessor's direction word, or nullptr (plain PDL wait)
  const uint64_t* chain_base;   // graph capture: the predecessor's sequence base, else nullptr
  uint64_t chain_seq;           // the predecessor's seq (relative to *chain_base when set)
};
extern int g_recv_early;
cudaError_t launch_publish(const PublishArgs& a, cudaStream_t s);

// ppc_pp_recv_batch: n consecutive receives of one direction in one grid (kernel parameter
// space holds the descriptors: n x sizeof(RecvArgs) <= ~8 KiB).
constexpr int kMaxBatch = 16;
struct RecvBatch {
  uint32_t n, pad;
  RecvArgs a[kMaxBatch];
};
cudaError_t launch_recv_batch(const RecvBatch& b, int grid, bool sys, cudaStream_t s);

// TP-sliced receive with a fused all-gather (ppc_pp_recv_gather).
constexpr int kMaxTp = 8;
struct GatherArgs {
  uint8_t* dst;
  uint64_t slice_bytes, chunk;
  uint32_t n_chunks, tp, my_tp;   // chunks per slice
  uint64_t seq, gtarget;          // gtarget = tp x gathers so far on this channel
  int64_t mb;
  const SlotHeader* hdr[kMaxTp];  // this seq's slot header in receiver t's arena
  const uint64_t* hdr_flag[kMaxTp];
  const uint64_t* seg_tab[kMaxTp];
  unsigned long long* gdone[kMaxTp];   // receiver t's finished-pull counter
  uint64_t* peer_credit;          // our own sender's credit word
  uint32_t* done;                 // our slot completion counter
  ErrWord* err;
  uint64_t timeout_ns;
};
cudaError_t launch_gather(const GatherArgs& a, int grid, cudaStream_t s);
// the gather's credit: waits (1 thread, bounded) until every receiver pulled our sender's
// slice, then releases the sender's credit; enqueued on a side stream after the gather
cudaError_t launch_gather_credit(const GatherArgs& a, cudaStream_t s);


// CE engine pieces: header/credit kernel before the copies, flag kernel after each.
struct CeHeadArgs {
  SlotHeader* hdr;
  uint64_t* hdr_flag;
  const uint64_t* credit;
  uint64_t need_credit;
  uint64_t bytes, seq, step;
  int64_t mb;
  uint32_t dir, boundary;
  ErrWord* err;
  uint64_t timeout_ns;
  ppc_record_t* rec;
  int rec_src, rec_dst;
};

__device__ __forceinline__ void fill_record(ppc_record_t* r, long long t0, int src, int dst,
                                            int dir, int kind, uint64_t seq, int64_t mb,
                                            uint64_t bytes) {
  r->t_start_ns = t0;
  r->t_end_ns = 0;
  r->src = src;
  r->dst = dst;
  r->dir = dir;
  r->kind = kind;
  r->seq = (long long)seq;
  r->mb = mb;
  r->bytes = (long long)bytes;
}

cudaError_t launch_push(const PushArgs& a, int grid, bool sys, bool ws, cudaStream_t s);
// dst[i] += src[i] for the hetero allreduce (dtype: 0 f32, 1 f16, 2 bf16, 3 i32).
cudaError_t launch_add(void* dst, const void* src, size_t count, int dtype, cudaStream_t s);
// Same-GPU single copy (direct mode of virtual stages): dst <- src, `bytes`, CTA chunks.
cudaError_t launch_copy(void* dst, const void* src, uint64_t bytes, uint64_t chunk, int grid,
                        cudaStream_t s);
// load every transport kernel on the current device now (see ppc_kernels.cu)
cudaError_t preload_kernels();
// launch transport kernels with programmatic dependent launch (ppc_kernels.cu); set from
// PPC_PDL by ppc_create
extern int g_pdl;
extern int kMaxSpinGrid;   // cap of cross-GPU spinning grids (64; PPC_SPIN_GRID_CAP)
extern int g_copy_tma_ctas;
extern int g_wait_value;       // PPC_WAIT_VALUE: eager credit waits as cuStreamWaitValue64
extern std::atomic<unsigned long long> g_launches;   // ppc_launch_count
// wait until *credit >= target (+ *seq_base when seq_base != nullptr: graph replay)
cudaError_t launch_wait_credit(const uint64_t* credit, uint64_t target, ErrWord* err,
                               uint64_t timeout_ns, cudaStream_t s,
                               const uint64_t* seq_base = nullptr);
// graph launch prologue: seq[0..3] = v[0..3]
cudaError_t launch_set_seq(uint64_t* seq, uint64_t v0, uint64_t v1, uint64_t v2, uint64_t v3,
                           cudaStream_t s);
cudaError_t launch_recv(const RecvArgs& a, int grid, bool sys, cudaStream_t s);
cudaError_t launch_ce_head(const CeHeadArgs& a, cudaStream_t s, bool pdl = false);
cudaError_t launch_ce_flags(uint64_t* flags, uint32_t c0, uint32_t c1, uint64_t seq,
                            ppc_record_t* rec, cudaStream_t s, bool pdl = false);

}  // namespace ppc
