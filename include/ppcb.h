/* ppcb.h — CPU-Forwarding baseline (BASELINE.json north_star: "kept only as the measured
 * baseline").  Separate library (libppcb.so) so libppc has no CPU path.
 *
 * PAPER.md §2.1: "this approach relies on global GPU data being routed through the CPU"
 * with "explicit data copy logic between GPU and CPU buffers during P2P operations"
 * (P:L47); the optimised variant ("DCBS&MPDT") parallelises the transfer.
 * B1 here: the sender copies D2H into a pinned ring shared by the two processes through
 * /dev/shm (cudaHostRegister'ed by both), publishes per-chunk sequence flags in shared
 * host memory, and the receiver copies H2D as chunks land.  `channels` host threads (each
 * with its own CUDA stream) move disjoint chunks in parallel (the MPDT analogue).  Calls
 * BLOCK the host until the bytes are in the shared ring (send) or in device memory (recv),
 * like the Megatron/Gloo P2P they model.  Same ring protocol as libppc: slot = seq % K,
 * per-chunk flags = seq, credit = last consumed seq, every wait bounded (timeout_ms).
 */
#ifndef PPCB_H_
#define PPCB_H_

#include <stddef.h>
#include <cuda_runtime_api.h>
#include "ppc.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ppcb_comm ppcb_comm_t;

/* One directed link src -> dst of a pair.  The side with is_sender = 1 creates the shared
 * ring "/ppcb_<tag>" (K slots x max_msg bytes + flags); the receiver opens it in
 * ppcb_connect after a caller barrier.  device: the caller's GPU. */
ppc_status_t ppcb_create(const char* tag, int is_sender, size_t max_msg, size_t chunk, int K,
                         int channels, int device, unsigned timeout_ms, ppcb_comm_t** out);
ppc_status_t ppcb_connect(ppcb_comm_t* c);
/* Blocking: waits for the slot's credit, D2H of every chunk (device buffer `buf`, after the
 * work already enqueued on s), publishes the chunk flags. */
ppc_status_t ppcb_send(ppcb_comm_t* c, const void* buf, size_t bytes, long long mb, cudaStream_t s);
/* Blocking: waits for each chunk flag, H2D into device buffer `buf`, returns the credit.
 * Checks the slot header: bytes (PPC_ERR_SIZE_MISMATCH), mb (PPC_ERR_ORDER). */
ppc_status_t ppcb_recv(ppcb_comm_t* c, void* buf, size_t bytes, long long mb, cudaStream_t s);
ppc_status_t ppcb_destroy(ppcb_comm_t* c);

#ifdef __cplusplus
}
#endif
#endif /* PPCB_H_ */
