/* ppc_toy.h — stage compute of the C1 toy pipeline (BASELINE.json configs[0]) on the GPU.
 *
 * Not part of the transfer path: these are the ppc_stage_fn callbacks a user model plugs into
 * ppc_step_1f1b, used to check the BJ gate "within 1e-3 relative error (bf16) on the
 * toy-model loss" end to end through the transfer kernels.  The model follows
 * oracle/toy.py (R11): 2 stages x 2 layers, z_l = h_l W_l + b_l, tanh on all but
 * the last layer, L = (1/M) sum_m mean((Y_m - T_m)^2), gradients accumulated over m in
 * ascending order, SGD at the end of the step.  fp32 arithmetic with a fixed summation order
 * (one thread per output, k ascending), so a pipelined and an un-pipelined GPU run of the
 * same kernels are bitwise identical.
 *
 * Boundary tensor: [rows, width] fp32 (boundary_bf16 = 0) or bf16 round-to-nearest-even
 * (boundary_bf16 = 1; message bytes = rows*width*2).
 */
#ifndef PPC_TOY_H_
#define PPC_TOY_H_

#include <stddef.h>
#include <cuda_runtime_api.h>
#include "ppc.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ppc_toy ppc_toy_t;

/* stage 0 or 1 of the 2-stage toy; M micro-batches of [rows, width]. Allocates on `device`. */
ppc_status_t ppc_toy_create(int stage, int rows, int width, int M, float lr, int boundary_bf16,
                            int device, ppc_toy_t** out);
/* Host fp32 parameters of this stage's two layers: W [2][width][width] row-major (h @ W),
 * b [2][width].  Stage 0 holds layers 0, 1; stage 1 holds layers 2, 3. Synchronous. */
ppc_status_t ppc_toy_set_params(ppc_toy_t* t, const float* W, const float* b);
ppc_status_t ppc_toy_get_params(ppc_toy_t* t, float* W, float* b);
/* Host fp32 micro-batch data [M][rows][width]: inputs X (stage 0) or targets T (stage 1). */
ppc_status_t ppc_toy_set_data(ppc_toy_t* t, const float* data);
/* ppc_stage_fn callbacks; user = the ppc_toy_t of the stage. */
int ppc_toy_fwd(void* user, int mb, const void* in, void* out, size_t in_bytes, size_t out_bytes,
                cudaStream_t s);
int ppc_toy_bwd(void* user, int mb, const void* in, void* out, size_t in_bytes, size_t out_bytes,
                cudaStream_t s);
/* End of step: SGD update p -= lr * grad, grads zeroed (enqueued on s). */
ppc_status_t ppc_toy_step_end(ppc_toy_t* t, cudaStream_t s);
/* Stage 1: the step's loss (1/M) sum_m loss_m, summed in ascending m; synchronizes s. */
ppc_status_t ppc_toy_loss(ppc_toy_t* t, cudaStream_t s, double* loss);
/* Boundary message bytes (rows*width*4, or *2 with a bf16 boundary). */
size_t ppc_toy_boundary_bytes(const ppc_toy_t* t);
ppc_status_t ppc_toy_destroy(ppc_toy_t* t);

#ifdef __cplusplus
}
#endif
#endif /* PPC_TOY_H_ */
