// C1 toy pipeline stage compute (include/ppc_toy.h): fp32 MLP layers with a fixed
// summation order.  Follows oracle/toy.py (R11); not part of the transfer path.
#include <cstdint>
#include <cstring>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ppc_toy.h"

namespace {

constexpr int T = 16;   // GEMM tile

enum Epi { kNone = 0, kTanh = 1, kDTanh = 2 };   // kDTanh: v *= (1 - H^2)

// C[MxN] (=|+=) op(A) op(B) (+ bias), one thread per output, k ascending (deterministic).
// TA: A stored [K][M]; TB: B stored [N][K].
template <bool TA, bool TB>
__global__ void gemm_kernel(const float* __restrict__ A, const float* __restrict__ B,
                            float* __restrict__ C, int M, int N, int K,
                            const float* __restrict__ bias, int epi, const float* __restrict__ H,
                            int accumulate) {
  __shared__ float As[T][T + 1];
  __shared__ float Bs[T][T + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int i = blockIdx.y * T + ty, j = blockIdx.x * T + tx;
  float acc = 0.f;
  for (int k0 = 0; k0 < K; k0 += T) {
    const int ka = k0 + tx, kb = k0 + ty;
    float a = 0.f, b = 0.f;
    if (i < M && ka < K) a = TA ? A[(size_t)ka * M + i] : A[(size_t)i * K + ka];
    if (j < N && kb < K) b = TB ? B[(size_t)j * K + kb] : B[(size_t)kb * N + j];
    As[ty][tx] = a;
    Bs[ty][tx] = b;
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < T; ++kk) acc = fmaf(As[ty][kk], Bs[kk][tx], acc);
    __syncthreads();
  }
  if (i >= M || j >= N) return;
  float v = acc;
  if (bias) v += bias[j];
  if (epi == kTanh) v = tanhf(v);
  if (epi == kDTanh) {
    const float h = H[(size_t)i * N + j];
    v = v * (1.f - h * h);
  }
  float* c = C + (size_t)i * N + j;
  *c = accumulate ? *c + v : v;
}

// gb[j] += sum_r dz[r][j], r ascending
__global__ void colsum_kernel(const float* __restrict__ dz, float* __restrict__ gb, int rows, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  float s = 0.f;
  for (int r = 0; r < rows; ++r) s += dz[(size_t)r * n + j];
  gb[j] = gb[j] + s;
}

// dY = 2 (y - t) / (rows * width * M)
__global__ void dloss_kernel(const float* y, const float* t, float* dy, size_t n, float scale) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dy[i] = 2.f * (y[i] - t[i]) / scale;
}

// out = a * (1 - h^2)
__global__ void dtanh_kernel(const float* a, const float* h, float* out, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] * (1.f - h[i] * h[i]);
}

// loss = mean((y - t)^2): fixed strided partial sums + fixed tree (one block of 256)
__global__ void loss_kernel(const float* y, const float* t, float* loss, size_t n) {
  __shared__ float sm[256];
  float s = 0.f;
  for (size_t i = threadIdx.x; i < n; i += 256) {
    const float d = y[i] - t[i];
    s = fmaf(d, d, s);
  }
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = sm[0] / (float)n;
}

__global__ void sgd_kernel(float* p, float* g, size_t n, float lr) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    p[i] = p[i] - lr * g[i];
    g[i] = 0.f;
  }
}

__global__ void to_bf16_kernel(const float* x, __nv_bfloat16* o, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = __float2bfloat16_rn(x[i]);
}
__global__ void from_bf16_kernel(const __nv_bfloat16* x, float* o, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = __bfloat162float(x[i]);
}

inline int blocks(size_t n, int b = 256) { return (int)((n + b - 1) / b); }

template <bool TA, bool TB>
void gemm(const float* A, const float* B, float* C, int M, int N, int K, const float* bias, int epi,
          const float* H, int acc, cudaStream_t s) {
  dim3 blk(T, T), grd((N + T - 1) / T, (M + T - 1) / T);
  gemm_kernel<TA, TB><<<grd, blk, 0, s>>>(A, B, C, M, N, K, bias, epi, H, acc);
}

}  // namespace

struct ppc_toy {
  int stage, rows, width, M, bf16, device;
  float lr;
  size_t act;                 // rows * width
  float *W[2], *b[2], *gW[2], *gb[2];
  float* data;                // X (stage 0) or T (stage 1): [M][rows][width]
  float *h1, *a, *h3, *y;     // caches [M][rows][width]
  float *ain, *dy, *dz, *dz2, *tmp;
  float* loss;                // [M]
  float* bnd;                 // fp32 boundary scratch
};

extern "C" {

ppc_status_t ppc_toy_create(int stage, int rows, int width, int M, float lr, int boundary_bf16,
                            int device, ppc_toy_t** out) {
  if (!out || (stage != 0 && stage != 1) || rows < 1 || width < 1 || M < 1) return PPC_ERR_INVALID_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return PPC_ERR_CUDA;
  ppc_toy* t = new ppc_toy();
  t->stage = stage; t->rows = rows; t->width = width; t->M = M; t->lr = lr;
  t->bf16 = boundary_bf16; t->device = device;
  t->act = (size_t)rows * width;
  const size_t ww = (size_t)width * width;
  bool ok = true;
  auto al = [&](float** p, size_t n) {
    ok = ok && cudaMalloc(p, n * sizeof(float)) == cudaSuccess &&
         cudaMemset(*p, 0, n * sizeof(float)) == cudaSuccess;
  };
  for (int l = 0; l < 2; ++l) {
    al(&t->W[l], ww); al(&t->gW[l], ww); al(&t->b[l], width); al(&t->gb[l], width);
  }
  al(&t->data, t->act * M);
  al(&t->h1, t->act * M); al(&t->a, t->act * M); al(&t->h3, t->act * M); al(&t->y, t->act * M);
  al(&t->ain, t->act * M);
  al(&t->dy, t->act); al(&t->dz, t->act); al(&t->dz2, t->act); al(&t->tmp, t->act);
  al(&t->bnd, t->act);
  al(&t->loss, M);
  if (!ok) { ppc_toy_destroy(t); return PPC_ERR_CUDA; }
  *out = t;
  return PPC_OK;
}

ppc_status_t ppc_toy_set_params(ppc_toy_t* t, const float* W, const float* b) {
  if (!t || !W || !b) return PPC_ERR_INVALID_ARG;
  cudaSetDevice(t->device);
  const size_t ww = (size_t)t->width * t->width;
  for (int l = 0; l < 2; ++l) {
    if (cudaMemcpy(t->W[l], W + l * ww, ww * 4, cudaMemcpyHostToDevice) ||
        cudaMemcpy(t->b[l], b + l * t->width, t->width * 4, cudaMemcpyHostToDevice))
      return PPC_ERR_CUDA;
  }
  return PPC_OK;
}

ppc_status_t ppc_toy_get_params(ppc_toy_t* t, float* W, float* b) {
  if (!t || !W || !b) return PPC_ERR_INVALID_ARG;
  cudaSetDevice(t->device);
  if (cudaDeviceSynchronize()) return PPC_ERR_CUDA;
  const size_t ww = (size_t)t->width * t->width;
  for (int l = 0; l < 2; ++l) {
    if (cudaMemcpy(W + l * ww, t->W[l], ww * 4, cudaMemcpyDeviceToHost) ||
        cudaMemcpy(b + l * t->width, t->b[l], t->width * 4, cudaMemcpyDeviceToHost))
      return PPC_ERR_CUDA;
  }
  return PPC_OK;
}

ppc_status_t ppc_toy_set_data(ppc_toy_t* t, const float* data) {
  if (!t || !data) return PPC_ERR_INVALID_ARG;
  cudaSetDevice(t->device);
  return cudaMemcpy(t->data, data, t->act * t->M * 4, cudaMemcpyHostToDevice) ? PPC_ERR_CUDA : PPC_OK;
}

size_t ppc_toy_boundary_bytes(const ppc_toy_t* t) { return t ? t->act * (t->bf16 ? 2 : 4) : 0; }

static void emit_boundary(ppc_toy* t, const float* v, void* out, cudaStream_t s) {
  if (!out) return;
  if (t->bf16) to_bf16_kernel<<<blocks(t->act), 256, 0, s>>>(v, (__nv_bfloat16*)out, t->act);
  else cudaMemcpyAsync(out, v, t->act * 4, cudaMemcpyDeviceToDevice, s);
}

static void take_boundary(ppc_toy* t, const void* in, float* dst, cudaStream_t s) {
  if (t->bf16) from_bf16_kernel<<<blocks(t->act), 256, 0, s>>>((const __nv_bfloat16*)in, dst, t->act);
  else cudaMemcpyAsync(dst, in, t->act * 4, cudaMemcpyDeviceToDevice, s);
}

int ppc_toy_fwd(void* user, int mb, const void* in, void* out, size_t, size_t, cudaStream_t s) {
  ppc_toy* t = static_cast<ppc_toy*>(user);
  if (!t || mb < 0 || mb >= t->M) return PPC_ERR_INVALID_ARG;
  const int R = t->rows, Wd = t->width;
  const size_t o = (size_t)mb * t->act;
  if (t->stage == 0) {
    gemm<false, false>(t->data + o, t->W[0], t->h1 + o, R, Wd, Wd, t->b[0], kTanh, nullptr, 0, s);
    gemm<false, false>(t->h1 + o, t->W[1], t->a + o, R, Wd, Wd, t->b[1], kTanh, nullptr, 0, s);
    emit_boundary(t, t->a + o, out, s);
  } else {
    if (!in) return PPC_ERR_INVALID_ARG;
    take_boundary(t, in, t->ain + o, s);
    gemm<false, false>(t->ain + o, t->W[0], t->h3 + o, R, Wd, Wd, t->b[0], kTanh, nullptr, 0, s);
    gemm<false, false>(t->h3 + o, t->W[1], t->y + o, R, Wd, Wd, t->b[1], kNone, nullptr, 0, s);
    loss_kernel<<<1, 256, 0, s>>>(t->y + o, t->data + o, t->loss + mb, t->act);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : PPC_ERR_CUDA;
}

int ppc_toy_bwd(void* user, int mb, const void* in, void* out, size_t, size_t, cudaStream_t s) {
  ppc_toy* t = static_cast<ppc_toy*>(user);
  if (!t || mb < 0 || mb >= t->M) return PPC_ERR_INVALID_ARG;
  const int R = t->rows, Wd = t->width;
  const size_t o = (size_t)mb * t->act;
  if (t->stage == 1) {
    // dY, layer 3 (linear), layer 2 (tanh), boundary gradient
    dloss_kernel<<<blocks(t->act), 256, 0, s>>>(t->y + o, t->data + o, t->dy, t->act,
                                                (float)t->act * (float)t->M);
    gemm<true, false>(t->h3 + o, t->dy, t->gW[1], Wd, Wd, R, nullptr, kNone, nullptr, 1, s);
    colsum_kernel<<<blocks(Wd), 256, 0, s>>>(t->dy, t->gb[1], R, Wd);
    gemm<false, true>(t->dy, t->W[1], t->dz, R, Wd, Wd, nullptr, kDTanh, t->h3 + o, 0, s);
    gemm<true, false>(t->ain + o, t->dz, t->gW[0], Wd, Wd, R, nullptr, kNone, nullptr, 1, s);
    colsum_kernel<<<blocks(Wd), 256, 0, s>>>(t->dz, t->gb[0], R, Wd);
    gemm<false, true>(t->dz, t->W[0], t->tmp, R, Wd, Wd, nullptr, kNone, nullptr, 0, s);
    emit_boundary(t, t->tmp, out, s);
  } else {
    if (!in) return PPC_ERR_INVALID_ARG;
    take_boundary(t, in, t->bnd, s);
    dtanh_kernel<<<blocks(t->act), 256, 0, s>>>(t->bnd, t->a + o, t->dz, t->act);
    gemm<true, false>(t->h1 + o, t->dz, t->gW[1], Wd, Wd, R, nullptr, kNone, nullptr, 1, s);
    colsum_kernel<<<blocks(Wd), 256, 0, s>>>(t->dz, t->gb[1], R, Wd);
    gemm<false, true>(t->dz, t->W[1], t->dz2, R, Wd, Wd, nullptr, kDTanh, t->h1 + o, 0, s);
    gemm<true, false>(t->data + o, t->dz2, t->gW[0], Wd, Wd, R, nullptr, kNone, nullptr, 1, s);
    colsum_kernel<<<blocks(Wd), 256, 0, s>>>(t->dz2, t->gb[0], R, Wd);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : PPC_ERR_CUDA;
}

ppc_status_t ppc_toy_step_end(ppc_toy_t* t, cudaStream_t s) {
  if (!t) return PPC_ERR_INVALID_ARG;
  cudaSetDevice(t->device);
  const size_t ww = (size_t)t->width * t->width;
  for (int l = 0; l < 2; ++l) {
    sgd_kernel<<<blocks(ww), 256, 0, s>>>(t->W[l], t->gW[l], ww, t->lr);
    sgd_kernel<<<blocks(t->width), 256, 0, s>>>(t->b[l], t->gb[l], t->width, t->lr);
  }
  return cudaGetLastError() == cudaSuccess ? PPC_OK : PPC_ERR_CUDA;
}

ppc_status_t ppc_toy_loss(ppc_toy_t* t, cudaStream_t s, double* loss) {
  if (!t || !loss || t->stage != 1) return PPC_ERR_INVALID_ARG;
  cudaSetDevice(t->device);
  std::vector<float> l(t->M);
  if (cudaStreamSynchronize(s) ||
      cudaMemcpy(l.data(), t->loss, t->M * sizeof(float), cudaMemcpyDeviceToHost))
    return PPC_ERR_CUDA;
  double acc = 0.0;
  for (int m = 0; m < t->M; ++m) acc += (double)l[m] / t->M;
  *loss = acc;
  return PPC_OK;
}

ppc_status_t ppc_toy_destroy(ppc_toy_t* t) {
  if (!t) return PPC_ERR_INVALID_ARG;
  cudaSetDevice(t->device);
  cudaDeviceSynchronize();
  float* ps[] = {t->W[0], t->W[1], t->b[0], t->b[1], t->gW[0], t->gW[1], t->gb[0], t->gb[1],
                 t->data, t->h1, t->a, t->h3, t->y, t->ain, t->dy, t->dz, t->dz2, t->tmp,
                 t->bnd, t->loss};
  for (float* p : ps) if (p) cudaFree(p);
  delete t;
  return PPC_OK;
}

}  // extern "C"
