/* ppc.h — pipeline-parallel stage-boundary transfer for B200 (sm_100a).  C ABI.
 *
 * The path (§2.2): per micro-batch, stage s sends its activation to
 * stage s+1 (FWD) and stage s+1 later sends the activation-gradient back (BWD), under a
 * non-interleaved 1F1B schedule (BASELINE.json north_star).  The paper's
 * Device-Direct idea — "the host manages control operations ... the data path remains
 * entirely on-device" — is rebuilt as sm_100a kernels that write the user buffer
 * straight into the receiver's ring slot over NVLink 5 (one pass; the paper's
 * user->chunk D2D, GDR, RDMA and chunk->user copies collapse into one peer write plus a
 * chunk-pipelined receiver copy-out).  Events (flags, credits) are handled on device;
 * the host thread only enqueues.
 *
 * Conventions
 *  - Every call runs on the calling host thread and never blocks on the GPU (stream
 *    ordered, like NCCL) unless stated.  Every call returns ppc_status_t; no exception
 *    crosses the ABI.  A ppc_comm_t is not thread-safe.
 *  - Pointers: "device" = CUDA device pointer on the comm's device; "host" = ordinary or
 *    pinned host memory.  Buffers stay owned by the caller and must stay valid until the
 *    stream reaches the operation (NCCL semantics).  libppc owns its rings, flags,
 *    credits, NCCL communicators and IPC mappings (allocated with cudaMalloc, outside any
 *    caching allocator, so CUDA IPC handles name whole allocations).
 *  - Errors: argument/state errors return synchronously and enqueue nothing.
 *    Device-detected errors (SIZE_MISMATCH, ORDER, TIMEOUT) latch a sticky error word
 *    in mapped host memory; ppc_poll returns it and every later call fails with
 *    PPC_ERR_STATE.  Recovery = ppc_disconnect on every rank, a caller barrier,
 *    ppc_destroy, then a fresh ppc_create.
 *  - Every device wait is bounded by cfg.timeout_ns (%globaltimer); no unbounded spin
 *    (§4.3: "training frequently encountered hang issues").  Once an
 *    error is latched on a comm, its other device waits give up at their next check
 *    instead of each running into its own timeout.
 *
 * Environment (read by ppc_create / the step driver; defaults are the measured best,
 * DESIGN.md §6-7):
 *   PPC_PDL=1            programmatic dependent launch of the transport kernels
 *   PPC_RECV_EARLY=0     cross-GPU receives (with PDL) look once for their zero-copy
 *                        publication before waiting on the predecessor kernel and pull the
 *                        first 64 KiB of each CTA's first chunk into registers meanwhile
 *   PPC_FUSE_PUBLISH=1   step driver: a zero-copy source op's publication rides on the
 *                        preceding terminal receive kernel
 *   PPC_PUB_BLOCK0=1     that fused publication's flag is released by the receive's block 0
 *                        (header already fenced at system scope) once every worker CTA has
 *                        arrived, instead of by the last worker behind a second system fence
 *   PPC_PULL_DYN=1       zero-copy pulls: every warp claims 4 KiB units of the message from
 *                        a per-slot counter (CTAs with faster NVLink paths take more) instead
 *                        of static chunk ranges per CTA (cfg.channels does not apply then)
 *   PPC_RECV_CHAIN=1     step driver: a receive enqueued right behind another receive starts
 *                        on that receive's posted end of data phase (a local device word)
 *                        instead of at griddepcontrol.wait (its grid exit + PDL release)
 *   PPC_ZC_SIDE=0        step driver: publish zero-copy sends on the send stream instead
 *                        of the compute stream
 *   PPC_ZC_STEPBUFS=1    the step driver's buffers (in the arena) are zero-copy sources
 *   PPC_STEP_INPLACE=0   step driver: a stage fn whose output is sent writes it straight
 *                        into the receiver's ring slot (ppc_pp_send_begin / _end) instead
 *                        of a local buffer that a send then moves (not in graph capture
 *                        or the virtual-stage direct mode)
 *   PPC_LOCAL_DIRECT=1   virtual stages: single-copy hand-off instead of the ring
 *   PPC_LOCAL_QUEUE=0    virtual stages: serialise all copies of the GPU on one queue
 *   PPC_COPY_CTAS=296    virtual stages: CTAs of the SIMT hand-off copy kernel
 *   PPC_COPY_TMA_CTAS=0  virtual stages: >0 selects the TMA bulk hand-off copy with that
 *                        many CTAs (16-B aligned buffers); 0 = the SIMT copy kernel
 *                        (faster inside the overlapped step, profiles/r56_copy_engine_ab.jsonl)
 *   PPC_STEP_BATCH=0     step driver (one process per GPU): the step's terminal receives (and
 *                        their fused publications) as one batched-receive grid per step
 *   PPC_PUB_FENCE=sys    fused publication flag release behind a system-scope fence; "gpu"
 *                        uses a gpu-scope fence (−1 % N=2 step, outside the PTX model's
 *                        guarantee for the peer — opt-in)
 *   PPC_DBG_STAMPS=0     per-CTA receive-kernel stamps for ppc_debug_stamps (diagnostics)
 *   PPC_WAIT_VALUE=0     eager credit waits (zero-copy rendezvous, ppc_pp_wait_consumed) as
 *                        cuStreamWaitValue64 instead of the bounded 1-thread kernel: zero SMs,
 *                        but UNBOUNDED (no timeout) — measured opt-in, DESIGN.md §7
 *   PPC_XOR_SEND_CTAS=296  grid cap of the fused XOR-send kernel
 *   PPC_SPIN_GRID_CAP=64 cap of cross-GPU spinning grids (receive / push / gather); larger
 *                        grids are safe since kernels are preloaded, 64 is the fastest
 *   PPC_NCCL_SINGLETON=0 tests: one-rank TP / DP groups get one-rank NCCL communicators too
 *   PPC_RECV_CTAS, PPC_STAGE_CTAS, PPC_PUSH_WS=1   grid / kernel-variant overrides
 */
#ifndef PPC_H_
#define PPC_H_

#include <stddef.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PPC_OK = 0,
  PPC_ERR_INVALID_ARG = 1,       /* null pointer, bad dir, mb < 0, misconfigured cfg           */
  PPC_ERR_GRID_MISMATCH = 2,     /* tp*pp*dp != world      */
  PPC_ERR_RANK_OUT_OF_RANGE = 3, /* rank not in [0, world)       */
  PPC_ERR_SELF_SEND = 4,         /* a PP neighbour's blob names the caller's own rank */
  PPC_ERR_NO_NEIGHBOR = 5,       /* FWD send on the last stage / BWD send on stage 0           */
  PPC_ERR_TOO_LARGE = 6,         /* bytes > cfg.max_msg_bytes                                   */
  PPC_ERR_SIZE_MISMATCH = 7,     /* async: header bytes != recv bytes      */
  PPC_ERR_ORDER = 8,             /* async: header seq/mb != expected (exactly once, in order)  */
  PPC_ERR_TIMEOUT = 9,           /* async: a bounded device wait expired      */
  PPC_ERR_BACKEND = 10,          /* DCBS rule: custom path requested for TP/DP      */
  PPC_ERR_CUDA = 11,
  PPC_ERR_NCCL = 12,
  PPC_ERR_STATE = 13,            /* not connected, destroyed, or poisoned by an async error    */
  PPC_ERR_WOULD_BLOCK = 14       /* virtual-stage (same-process) mode only: the matching send /
                                    the slot's previous recv is not enqueued yet; nothing was
                                    enqueued, retry after enqueueing the peer's op            */
} ppc_status_t;

typedef enum { PPC_FWD = 0, PPC_BWD = 1 } ppc_dir_t;     /* FWD: s -> s+1 ; BWD: s+1 -> s */
/* Data movers (the MPDT analogue):
 *  SM   : the sender's CTAs load the user buffer and STORE it into the receiver's ring
 *         over NVLink; the receiver copies the slot out (chunk-pipelined).
 *  CE   : the sender's copy engines (cudaMemcpyAsync on `channels` streams) write the
 *         receiver's ring; zero SMs for the data.
 *  PULL : the sender copies the user buffer into its OWN ring (local HBM) and releases
 *         per-chunk flags in the receiver's memory; the receiver's CTAs LOAD each chunk over
 *         NVLink straight into its user buffer (no copy-out; peer loads outrun peer stores
 *         on B200, see profiles/). */
typedef enum { PPC_ENGINE_SM = 0, PPC_ENGINE_CE = 1, PPC_ENGINE_PULL = 2 } ppc_engine_t;
typedef enum { PPC_GROUP_TP = 0, PPC_GROUP_DP = 1, PPC_GROUP_PP = 2 } ppc_group_t;
typedef enum { PPC_BACKEND_NCCL = 0, PPC_BACKEND_PEER = 1, PPC_BACKEND_NONE = 2 } ppc_backend_t;

typedef struct {
  int tp, pp, dp;               /* grid; rank = pp_i*(tp*dp) + dp_i*tp + tp_i */
  size_t max_msg_bytes;         /* ring slot payload capacity                                  */
  int ring_slots;               /* K; 0 => pp + 1 (1F1B occupancy bound + 1: sends never wait
                                   for a slot; SPEC's double buffering is K = 2)        */
  int channels;                 /* MPDT analogue: a message's chunks split into this
                                   many contiguous ranges, each moved by its own CTA group (SM
                                   push, PULL staging and pulls, zero-copy pulls) or its own
                                   copy-engine stream (CE engine); 1..8; 0 => 1               */
  size_t chunk_bytes;           /* flag granularity, multiple of 4096; 0 => 1 MiB              */
  ppc_engine_t engine;          /* data mover for sends                                        */
  int cta_per_channel;          /* SM engine CTAs per channel; 0 => auto                       */
  unsigned long long timeout_ns;/* bound of every device wait; 0 => 10 s                       */
  int trace;                    /* bit 0: %globaltimer records per transfer (ppc_trace);
                                   bit 1: CUDA-event pair around every send / recv launch on
                                   its stream (ppc_kernel_times)                               */
  int zc_async;                 /* 1: a zero-copy ppc_pp_send completes at publication, so
                                   consecutive sends on one stream overlap; the caller keeps
                                   the buffer unchanged until ppc_pp_wait_consumed (like an
                                   MPI_Isend / MPI_Wait pair).  0: rendezvous (default)        */
  int local_spin;               /* comms of ONE process (virtual stages, ppc_connect with blobs
                                   of the same pid): 0 => CUDA events order the stages (the
                                   virtual-stage mode, ppc_step_1f1b_local); 1 => the comms
                                   behave exactly like one process per GPU — device flag /
                                   credit / header spins with .sys scope, zero-copy
                                   registrations, publication, TP gathers, the per-rank step
                                   driver ppc_step_1f1b on each comm (the host never blocks,
                                   so S comms are stepped one after another from one thread).
                                   Spinning grids of stages sharing a GPU are capped at 8
                                   CTAs so every stage stays resident.  Lets one GPU exercise
                                   the whole cross-process protocol (tests, smoke)          */
} ppc_config_t;

typedef struct ppc_comm ppc_comm_t;

typedef struct { int kind; /* 0 = F, 1 = B */ int mb; } ppc_op_t;

typedef struct {
  long long t_start_ns, t_end_ns;   /* %globaltimer of the first CTA start / last CTA end     */
  int src, dst, dir, kind;          /* kind: 0 = send, 1 = recv; a recv's dir is -1, or -2 when
                                       PPC_RECV_EARLY's early look found the publication      */
  long long seq, mb, bytes;
} ppc_record_t;

/* Stage compute callback of the 1F1B driver.  Enqueue work on `s` that reads `in`
 * (in_bytes) and writes `out` (out_bytes); return 0 on success.  in == NULL on stage 0's F
 * when no stage input is given; out may alias nothing else. */
typedef int (*ppc_stage_fn)(void* user, int mb, const void* in, void* out,
                            size_t in_bytes, size_t out_bytes, cudaStream_t s);

/* One 1F1B step (ppc_step_1f1b).  fwd/bwd NULL => identity stage (out = in).  x/g/y/dx
 * entries may be host or device pointers.  Host (pinned for full speed) => copied inside
 * the step: inputs are staged into the step buffers on an internal host->device stream that
 * runs ahead as soon as a staging buffer is free, outputs leave on an internal
 * device->host stream; both complete within the step's stream order on `s`. */
typedef struct {
  int M;                         /* micro-batches                                            */
  size_t fwd_bytes, bwd_bytes;   /* boundary activation / gradient bytes per micro-batch      */
  ppc_stage_fn fwd, bwd;
  void* fwd_user;                /* passed to fwd                                            */
  void* bwd_user;                /* passed to bwd                                            */
  const void* const* x;          /* [M] stage-0 F inputs (used when s == 0), may be NULL      */
  const void* const* g;          /* [M] last-stage B inputs (used when s == S-1), may be NULL */
  void* const* y;                /* [M] last-stage F outputs (s == S-1), may be NULL          */
  void* const* dx;               /* [M] stage-0 B outputs (s == 0), may be NULL               */
} ppc_step_t;

/* ---- lifecycle (§2.2 Initialization Phase) ---------------------------- */

/* Resource Discovery: validate the grid (PPC_ERR_GRID_MISMATCH), allocate this rank's
 * incoming rings (K slots x (64 B header + max_msg_bytes)), flags, credits and the mapped
 * error word on `cuda_device`.  cuda_device = -1 creates a host-only comm (no device
 * memory; group logic and blob exchange only — used by CPU tests). */
ppc_status_t ppc_create(const ppc_config_t* cfg, int world, int rank, int cuda_device,
                        ppc_comm_t** out);

/* Topology Awareness blob of this rank (rank, device, PCI bus id, pid, IPC handle of the
 * ring arena, geometry).  blob may be NULL to query *blob_bytes (fixed PPC_BLOB_BYTES). */
#define PPC_BLOB_BYTES 512
ppc_status_t ppc_export(ppc_comm_t* c, void* blob, size_t* blob_bytes);

/* Open the PP neighbours' rings from the all-gathered blobs (world x blob_bytes, rank
 * order) and, for TP/DP groups of size > 1, init NCCL communicators (DCBS)
 * from nccl_ids = [tp_id, dp_id] (each 128 B, made by the group's lowest rank with
 * ppc_nccl_unique_id).  Blobs of the same process (virtual stages on one GPU) are mapped
 * by raw pointer instead of IPC.  n_ids = 0 skips NCCL. */
ppc_status_t ppc_connect(ppc_comm_t* c, const void* all_blobs, size_t blob_bytes,
                         const void* nccl_ids, int n_ids);

ppc_status_t ppc_nccl_unique_id(void* out128);

/* Members (rank order) and backend of this rank's group g: TP/DP -> NCCL, PP -> PEER. */
ppc_status_t ppc_group(const ppc_comm_t* c, ppc_group_t g, int* members, int* n,
                       ppc_backend_t* backend);

/* ---- data path (§2.2 Communication Phase, Heterogeneous P2P) ----------- */

/* Send `bytes` of device buffer `buf` to the PP neighbour in direction d as micro-batch
 * `mb`.  Enqueued on `s`: waits (on device) for the slot's credit, writes the 64-B header
 * and the payload into the neighbour's ring slot seq % K, releases per-chunk flags.
 * Errors: PPC_ERR_NO_NEIGHBOR, PPC_ERR_TOO_LARGE, PPC_ERR_INVALID_ARG. */
ppc_status_t ppc_pp_send(ppc_comm_t* c, ppc_dir_t d, const void* buf, size_t bytes,
                         long long mb, cudaStream_t s);

/* Receive the next message of direction d into device buffer `buf`.  Enqueued on `s`:
 * per chunk waits for the flag, checks the header (bytes -> SIZE_MISMATCH, seq/mb ->
 * ORDER), copies slot -> buf, and after the last chunk returns the credit to the sender. */
ppc_status_t ppc_pp_recv(ppc_comm_t* c, ppc_dir_t d, void* buf, size_t bytes,
                         long long mb, cudaStream_t s);

/* Enqueue on `s` a (bounded) device wait until the peer has consumed every message sent so
 * far in direction d, i.e. its credit reached the last send's seq: afterwards the data is
 * in the receiver's user buffer.  Used to time transfers end to end from the sender. */
ppc_status_t ppc_pp_wait_consumed(ppc_comm_t* c, ppc_dir_t d, cudaStream_t s);

/* Produce-in-place send: the stage's producing kernel writes the message straight into the
 * receiver's ring slot over NVLink, so no separate send pass reads it back from HBM (the
 * compute step fused with the transfer; P:L53's device-direct path without its staging
 * copies).  ppc_pp_send_begin enqueues on s the slot's credit wait (bounded; a timeout
 * latches PPC_ERR_TIMEOUT) and the 64-B header, and returns in *slot where to write:
 *   payload   the receiver's slot (peer memory, a device pointer valid on the caller's GPU;
 *             write [0, bytes) only, from kernels enqueued on s after this call)
 *   flags     n_chunks per-chunk flags in the receiver's memory; chunk i covers
 *             [i*chunk_bytes, min((i+1)*chunk_bytes, bytes))
 *   seq       the value that marks a chunk complete
 * A producer that signals itself stores chunk i, then (one thread, after a CTA barrier)
 * fence.acq_rel.sys + st.release.sys flags[i] = seq — the receiver copies chunk i out as
 * soon as its flag lands.  ppc_pp_send_end(flags_released = 0) enqueues one kernel that
 * releases every flag after the producer's kernels (stream order); flags_released = 1
 * means the producer released all of them.  One begin/end pair open per direction;
 * bytes == 0 or > max_msg_bytes, a second begin, or an end without begin fail synchronously
 * (PPC_ERR_INVALID_ARG / PPC_ERR_TOO_LARGE / PPC_ERR_STATE).  Not capturable into a step
 * graph (the slot address depends on the sequence number): PPC_ERR_INVALID_ARG. */
typedef struct {
  void* payload;
  unsigned long long* flags;
  unsigned long long seq;
  size_t bytes, chunk_bytes;
  unsigned int n_chunks;
} ppc_slot_t;
ppc_status_t ppc_pp_send_begin(ppc_comm_t* c, ppc_dir_t d, size_t bytes, long long mb,
                               cudaStream_t s, ppc_slot_t* slot);
ppc_status_t ppc_pp_send_end(ppc_comm_t* c, ppc_dir_t d, int flags_released, cudaStream_t s);

/* Zero-copy send buffers.  ppc_register(c, ptr, bytes) registers the device allocation that
 * contains [ptr, ptr+bytes) (one CUDA IPC handle per allocation) and returns a blob of
 * PPC_REG_BLOB_BYTES; the caller gives every PP neighbour the blob (control plane, e.g. a
 * gloo all-gather) and the neighbour calls ppc_register_import.  Afterwards ppc_pp_send from
 * a registered range moves no data on the sender: it publishes (segment, offset) in the
 * receiver's slot header and the receiver's CTAs LOAD the payload over NVLink straight into
 * their user buffer (one pass, no ring copy).  The send completes on its stream only when
 * the receiver has consumed the message (rendezvous), so the buffer may be reused after it
 * — unless cfg.zc_async, where it completes at publication and ppc_pp_wait_consumed marks
 * the point after which the buffers of all earlier sends may be reused.
 * Blobs of non-neighbours are accepted and ignored.  Up to 256 registrations per comm. */
#define PPC_REG_BLOB_BYTES 128
ppc_status_t ppc_register(ppc_comm_t* c, const void* ptr, size_t bytes, void* blob,
                          size_t* blob_bytes);
ppc_status_t ppc_register_import(ppc_comm_t* c, const void* blob, size_t blob_bytes);

/* Batched receive: the next n (1..16) messages of direction d into bufs[i] (bytes[i] each,
 * micro-batch mb0 + i), exactly as n consecutive ppc_pp_recv calls — but in ONE grid whose
 * CTAs move on to message i+1 as soon as their share of message i is done, so consecutive
 * messages overlap their ramp and tail instead of paying a kernel boundary each (a stream
 * of messages: the C5 sweep, a stage receiving several micro-batches back to back).  Credits
 * are returned per message, in order; the n buffers must not overlap (CTAs of one grid may
 * write messages i and i+1 at the same time).  Errors as ppc_pp_recv (per message).  In the
 * virtual-stage mode all n sends must already be enqueued (else PPC_ERR_WOULD_BLOCK). */
ppc_status_t ppc_pp_recv_batch(ppc_comm_t* c, ppc_dir_t d, void* const* bufs,
                               const size_t* bytes, int n, long long mb0, cudaStream_t s);

/* TP-sliced boundary with a fused all-gather (BJ configs[2], PP x TP):
 * every TP rank of the sending stage sends only its 1/TP slice (ppc_pp_send of slice bytes
 * from a REGISTERED buffer); every TP rank of the receiving stage calls ppc_pp_recv_gather
 * with the full size and receives all TP slices, in tp order, pulled over NVLink straight
 * from the senders' buffers — no separate all-gather.  The receivers of one stage count
 * their finished pulls in each other's memory; each then returns its own sender's credit,
 * so a sender reuses its slice only after every receiver pulled it.  Registration blobs of
 * every rank of the adjacent stage must be imported (ppc_register_import accepts them).
 * total_bytes must be a multiple of tp.  One process per GPU only. */
ppc_status_t ppc_pp_recv_gather(ppc_comm_t* c, ppc_dir_t d, void* buf, size_t total_bytes,
                                long long mb, cudaStream_t s);

/* Pure: the 1F1B op list of stage s (of S) over M micro-batches; ops has room for 2M.
 * w = min(S-s-1, M) forwards, then M-w (F, B) pairs, then w backwards. */
ppc_status_t ppc_schedule_1f1b(int S, int s, int M, ppc_op_t* ops, int* n_ops);

/* One 1F1B step of this rank's stage: per op recv -> stage fn -> send, with sends on
 * internal streams; returns after enqueueing everything on `s` (host never blocks). */
ppc_status_t ppc_step_1f1b(ppc_comm_t* c, const ppc_step_t* st, cudaStream_t s);

/* The same for S virtual stages created in this process (one GPU; ranks 0..S-1 of a
 * pp = S grid): interleaves the stages' ops in a dependency-respecting enqueue order.
 * comms[i], steps[i] and streams[i] belong to stage i. */
ppc_status_t ppc_step_1f1b_local(ppc_comm_t* const* comms, int S, const ppc_step_t* steps,
                                 const cudaStream_t* streams);

/* CUDA-graph capture of one 1F1B step (streams and graphs instead of per-op launches).
 * n == 1: comms[0] is a one-process-per-GPU comm, the step is ppc_step_1f1b(comms[0],
 * &steps[0], streams[0]); n == S: virtual stages, ppc_step_1f1b_local(comms, S, steps,
 * streams).  Every kernel of the captured step reads its sequence number relative to a
 * device counter that ppc_graph_launch sets, so one graph replays every later step; the
 * host counters advance per launch exactly as an eager step would.  The step arguments'
 * buffers must stay valid for the graph's lifetime.  Not capturable: the CE engine.  Before
 * creating, the devices are synchronised; launches are serialised on streams[0]. */
typedef struct ppc_graph ppc_graph_t;
ppc_status_t ppc_graph_create(ppc_comm_t* const* comms, int n, const ppc_step_t* steps,
                              const cudaStream_t* streams, ppc_graph_t** out);
ppc_status_t ppc_graph_launch(ppc_graph_t* g);
ppc_status_t ppc_graph_destroy(ppc_graph_t* g);

/* DCBS TP/DP traffic on NCCL: in-place sum allreduce over group g.
 * PPC_ERR_BACKEND for g == PPC_GROUP_PP. nccl_dtype is an ncclDataType_t value. */
ppc_status_t ppc_allreduce(ppc_comm_t* c, ppc_group_t g, void* buf, size_t count,
                           int nccl_dtype, cudaStream_t s);

/* Heterogeneous-collective composition (§2.2):
 * in-place sum allreduce over ALL ranks of this rank's tensor-parallel slice (every rank
 * with the same tp_i), composed as (1) a vendor-CCL (NCCL) allreduce inside each
 * homogeneous subgroup = this stage's DP group, (2) the cross-subgroup exchange of the
 * intermediate results between the subgroup leaders (dp_i = 0) over the PP peer path
 * (libppc send/recv along the stage chain: reduce forward, result backward), (3) an NCCL
 * broadcast from the leader inside each subgroup.  count * element size <= max_msg_bytes.
 * nccl_dtype: ncclFloat32 (7), ncclFloat16 (6), ncclBfloat16 (9) or ncclInt32 (2).
 * One process per GPU only (not virtual stages). */
ppc_status_t ppc_hetero_allreduce(ppc_comm_t* c, void* buf, size_t count, int nccl_dtype,
                                  cudaStream_t s);

/* ---- diagnostics and teardown ---------------------------------------------------------- */
ppc_status_t ppc_poll(ppc_comm_t* c);              /* non-blocking read of the error word  */
/* Details of a latched device error: the message seq and where (0x1xx receive header or
 * chunk wait, 0x2xx credit wait, 0x3xx zero-copy lookup, 0x4xx-0x6xx TP gather; chunk or
 * tp index in bits 12+; a send's timeout reports its direction). */
ppc_status_t ppc_error_info(ppc_comm_t* c, unsigned* seq, unsigned* info);
ppc_status_t ppc_trace(ppc_comm_t* c, ppc_record_t* out, int* n);  /* synchronizes the device;
                                                      *n in: capacity, out: records written */
/* Device durations (ms) of the send (kind 0) or recv (kind 1) launches enqueued since the
 * last call, from the CUDA-event pairs of cfg.trace bit 1, in launch order; synchronizes
 * the device.  *n in: capacity, out: entries written.  Resets the list. */
ppc_status_t ppc_kernel_times(ppc_comm_t* c, int kind, float* ms, int* n);
/* Diagnostics (PPC_DBG_STAMPS=1 at ppc_create): per eager receive launch (the first 4096),
 * 128 CTA rows x 4 %globaltimer stamps — [0] released by griddepcontrol.wait, [1] header seen,
 * [2] first chunk moved (zero-copy pulls; SM id in bits 48-63, the timer's low 48 bits below),
 * [3] CTA done (0 = not reached / CTA absent) — and
 * meta = (seq, dir, grid) per launch; synchronizes the device.  *n in: capacity in launches,
 * out: launches returned.  stamps has room for *n x 512 values, meta for *n x 3. */
ppc_status_t ppc_debug_stamps(ppc_comm_t* c, unsigned long long* stamps, long long* meta, int* n);
/* Switch cfg.trace bits at run time (bit 0 only if the comm was created with it). */
ppc_status_t ppc_set_trace(ppc_comm_t* c, int trace);
ppc_status_t ppc_disconnect(ppc_comm_t* c);        /* phase 1: close peer handles, NCCL    */
ppc_status_t ppc_destroy(ppc_comm_t* c);           /* phase 2 (after a caller barrier)     */
const char* ppc_status_str(ppc_status_t st);
/* Kernels libppc enqueued in this process so far (transport, stage proxy and fill kernels;
 * a CUDA graph's kernel nodes count once per ppc_graph_launch).  Copy-engine copies are not
 * kernels and are not counted.  Thread-safe, monotone. */
unsigned long long ppc_launch_count(void);
/* sizeof of the ABI structs, for bindings to check their layouts: which = 0 ppc_config_t,
 * 1 ppc_step_t, 2 ppc_record_t, 3 ppc_op_t, 4 ppc_slot_t; 0 for any other value. */
size_t ppc_struct_size(int which);

/* ---- test/bench kernels (K14); not part of the transfer path --------------------------- */
/* Fill `bytes` of device buffer with the synth/payload.py SplitMix64 stream of key
 * (seed, step, boundary, dir, mb). */
ppc_status_t ppc_fill_payload(void* buf, size_t bytes, int seed, int step, int boundary,
                              int dir, long long mb, cudaStream_t s);
/* ppc_stage_fn: out = in XOR mask(stage, dir, mb) (synth/payload.proxy_mask, seed tagged
 * with 0x8000); `user` must point to a ppc_xor_ctx_t.  in == NULL reads zeros. */
typedef struct { int seed, step, stage, dir; } ppc_xor_ctx_t;
int ppc_stage_xor(void* user, int mb, const void* in, void* out, size_t in_bytes,
                  size_t out_bytes, cudaStream_t s);
/* The XOR stage proxy fused with its send (the produce-in-place pattern above): computes
 * out = in XOR stream(ctx, mb) exactly as ppc_stage_xor and stores it straight into
 * slot->payload, releasing each chunk's flag as soon as that chunk is written (call
 * ppc_pp_send_end with flags_released = 1 afterwards).  bytes must equal slot->bytes. */
ppc_status_t ppc_stage_xor_send(const ppc_slot_t* slot, const ppc_xor_ctx_t* ctx, int mb,
                                const void* in, size_t bytes, cudaStream_t s);

#ifdef __cplusplus
}
#endif
#endif /* PPC_H_ */
