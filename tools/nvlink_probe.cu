// NVLink data-mover probe (one process, two GPUs with peer access): which way of moving a
// stage-boundary message GPU0 -> GPU1 is fastest on B200?
//   store  : SM kernel, local 16/32-byte loads -> peer stores (push; current K9 design)
//   load   : SM kernel on GPU1, peer loads from GPU0 -> local stores (pull)
//   tma_st : TMA bulk global(local)->smem->global(peer) per CTA (push)
//   tma_ld : TMA bulk global(peer)->smem->global(local) per CTA on GPU1 (pull)
//   ce     : cudaMemcpyPeerAsync
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o nvlink_probe nvlink_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); exit(1);} } while (0)

struct __align__(32) V32 { uint4 lo, hi; };

__device__ __forceinline__ V32 ld32(const V32* p) {
  V32 r;
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.lo.x), "=r"(r.lo.y), "=r"(r.lo.z), "=r"(r.lo.w), "=r"(r.hi.x),
                 "=r"(r.hi.y), "=r"(r.hi.z), "=r"(r.hi.w) : "l"(p));
  return r;
}
__device__ __forceinline__ V32 ld32_cg(const V32* p) {
  V32 r;
  asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.lo.x), "=r"(r.lo.y), "=r"(r.lo.z), "=r"(r.lo.w), "=r"(r.hi.x),
                 "=r"(r.hi.y), "=r"(r.hi.z), "=r"(r.hi.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st32(V32* p, const V32& v) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.lo.x),
               "r"(v.lo.y), "r"(v.lo.z), "r"(v.lo.w), "r"(v.hi.x), "r"(v.hi.y), "r"(v.hi.z),
               "r"(v.hi.w) : "memory");
}

// contiguous per-CTA ranges, U vectors in flight per thread
template <int U, bool PEER_SRC>
__global__ void __launch_bounds__(512) simt_copy(V32* dst, const V32* src, size_t nv) {
  const size_t per = (nv + gridDim.x - 1) / gridDim.x;
  const size_t b = blockIdx.x * per, e = min(nv, b + per);
  size_t i = b + threadIdx.x;
  const size_t nt = blockDim.x;
  for (; i + (U - 1) * nt < e; i += nt * U) {
    V32 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) v[j] = PEER_SRC ? ld32_cg(src + i + j * nt) : ld32(src + i + j * nt);
#pragma unroll
    for (int j = 0; j < U; ++j) st32(dst + i + j * nt, v[j]);
  }
  for (; i < e; i += nt) st32(dst + i, PEER_SRC ? ld32_cg(src + i) : ld32(src + i));
}

// The K9 push pattern: chunk per CTA iteration, then fence + flag (fence by all threads or
// by thread 0 only after the barrier), to isolate the cost of the release protocol.
template <int U, bool ALL_FENCE>
__global__ void __launch_bounds__(512) simt_store_flagged(V32* dst, const V32* src, size_t nv,
                                                          size_t chunk_v, uint64_t* flags, uint64_t seq) {
  const size_t nchunks = (nv + chunk_v - 1) / chunk_v;
  const size_t nt = blockDim.x;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const size_t b = c * chunk_v, e = min(nv, b + chunk_v);
    size_t i = b + threadIdx.x;
    for (; i + (U - 1) * nt < e; i += nt * U) {
      V32 v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) v[j] = ld32(src + i + j * nt);
#pragma unroll
      for (int j = 0; j < U; ++j) st32(dst + i + j * nt, v[j]);
    }
    for (; i < e; i += nt) st32(dst + i, ld32(src + i));
    if (ALL_FENCE) asm volatile("fence.acq_rel.sys;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      if (!ALL_FENCE) asm volatile("fence.acq_rel.sys;" ::: "memory");
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(flags + c), "l"(seq) : "memory");
    }
  }
}

// ---- TMA bulk pipeline: one elected thread per CTA, S stages of T bytes in shared memory
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(m)), "r"(phase) : "memory");
}
__device__ __forceinline__ void tma_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void tma_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void tma_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void tma_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int S>
__global__ void tma_copy(uint8_t* dst, const uint8_t* src, size_t bytes, uint32_t tile) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t mbar[S];
  if (threadIdx.x != 0) return;
  const size_t ntiles = (bytes + tile - 1) / tile;
  const size_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const size_t t0 = blockIdx.x * per, t1 = min(ntiles, t0 + per);
  if (t0 >= t1) return;
  for (int s = 0; s < S; ++s) mbar_init(&mbar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t n = t1 - t0;
  auto len_of = [&](size_t t) { return (uint32_t)min((size_t)tile, bytes - t * tile); };
  for (size_t j = 0; j < n && j < S; ++j) {
    const size_t t = t0 + j;
    mbar_expect_tx(&mbar[j], len_of(t));
    tma_load(sm + j * tile, src + t * tile, len_of(t), &mbar[j]);
  }
  for (size_t i = 0; i < n; ++i) {
    const int s = i % S;
    const size_t t = t0 + i;
    mbar_wait(&mbar[s], (uint32_t)((i / S) & 1));
    tma_store(dst + t * tile, sm + s * tile, len_of(t));
    const size_t j = i + S;
    if (j < n) {
      tma_wait_read<0>();   // smem of stage s consumed by the store
      const size_t tj = t0 + j;
      mbar_expect_tx(&mbar[s], len_of(tj));
      tma_load(sm + s * tile, src + tj * tile, len_of(tj), &mbar[s]);
    }
  }
  tma_wait_all();
}



// Bidirectional mode ("bidir"): GPU0 -> GPU1 and GPU1 -> GPU0 at the same time, as in the
// steady state of a PP2 1F1B step (F_m+1 and B_m in flight together).  Each direction's
// mover runs `reps` back-to-back launches on its own stream; GB/s per direction.
static int bidir() {
  const size_t maxb = 256ull << 20;
  uint8_t* a[2];   // a[d]: source of direction d's data, lives on GPU d
  uint8_t* b[2];   // b[d]: destination of direction d, lives on GPU 1-d
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMalloc(&a[d], maxb)); CK(cudaMemset(a[d], 1 + d, maxb));
    CK(cudaMalloc(&b[1 - d], maxb)); CK(cudaMemset(b[1 - d], 0, maxb));   // on GPU d
  }
  const int tile = 32 << 10, S = 6;
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaFuncSetAttribute(tma_copy<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * tile));
  }
  // mover kinds: 0 = SM load on the receiver, 1 = SM store on the sender, 2 = CE, 3 = TMA load
  auto launch = [&](int kind, int d, int g, size_t bytes, cudaStream_t* sts) {
    const int rx = 1 - d;          // receiving GPU of direction d
    const size_t nv = bytes / 32;
    uint8_t* out = b[d];       // allocated on GPU rx
    if (kind == 0) {
      CK(cudaSetDevice(rx));
      simt_copy<8, true><<<g, 512, 0, sts[rx]>>>((V32*)out, (const V32*)a[d], nv);
    } else if (kind == 1) {
      CK(cudaSetDevice(d));
      simt_copy<8, false><<<g, 512, 0, sts[d]>>>((V32*)out, (const V32*)a[d], nv);
    } else if (kind == 2) {
      CK(cudaSetDevice(d));
      CK(cudaMemcpyPeerAsync(out, rx, a[d], d, bytes, sts[d]));
    } else {
      CK(cudaSetDevice(rx));
      tma_copy<S><<<g, 32, S * tile, sts[rx]>>>(out, a[d], bytes, tile);
    }
  };
  const char* names[] = {"load", "store", "ce", "tma_load"};
  // the stream a direction's work runs on: receiver's for pulls, sender's for pushes / CE
  auto stream_dev = [&](int kind, int d) { return (kind == 0 || kind == 3) ? 1 - d : d; };
  for (size_t bytes : {32ull << 20, 256ull << 20}) {
    const int reps = bytes <= (32u << 20) ? 40 : 8;
    for (int k0 : {0, 1, 2, 3})
      for (int k1 : {0, 1, 2, 3}) {
        if (k1 < k0) continue;
        for (int g : {64, 96, 148}) {
          if (k0 == 2 && k1 == 2 && g != 64) continue;
          const int kinds[2] = {k0, k1};
          // both directions on different devices' streams: if they collide on one device
          // (e.g. load for d=0 runs on GPU1, store for d=1 runs on GPU1) use two streams
          cudaStream_t sts2[2][2];
          for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaStreamCreateWithFlags(&sts2[d][0], cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&sts2[d][1], cudaStreamNonBlocking));
          }
          cudaStream_t use[2][2];   // use[d] = stream array indexed by device for direction d
          for (int d = 0; d < 2; ++d) { use[d][0] = sts2[0][d]; use[d][1] = sts2[1][d]; }
          cudaEvent_t e0[2], e1[2];
          for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(stream_dev(kinds[d], d)));
            CK(cudaEventCreate(&e0[d])); CK(cudaEventCreate(&e1[d]));
          }
          for (int d = 0; d < 2; ++d) launch(kinds[d], d, g, bytes, use[d]);
          for (int dev = 0; dev < 2; ++dev) { CK(cudaSetDevice(dev)); CK(cudaDeviceSynchronize()); }
          for (int d = 0; d < 2; ++d) {
            const int sd = stream_dev(kinds[d], d);
            CK(cudaSetDevice(sd)); CK(cudaEventRecord(e0[d], use[d][sd]));
          }
          for (int r = 0; r < reps; ++r)
            for (int d = 0; d < 2; ++d) launch(kinds[d], d, g, bytes, use[d]);
          for (int d = 0; d < 2; ++d) {
            const int sd = stream_dev(kinds[d], d);
            CK(cudaSetDevice(sd)); CK(cudaEventRecord(e1[d], use[d][sd]));
          }
          double gb[2];
          for (int d = 0; d < 2; ++d) {
            CK(cudaEventSynchronize(e1[d]));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
            gb[d] = (double)bytes * reps / (ms * 1e-3) / 1e9;
          }
          CK(cudaGetLastError());
          printf("{\"bidir\": \"%s+%s\", \"bytes\": %zu, \"grid\": %d, \"gbps_d0\": %.1f, "
                 "\"gbps_d1\": %.1f}\n", names[k0], names[k1], bytes, g, gb[0], gb[1]);
          fflush(stdout);
          for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            cudaStreamDestroy(sts2[d][0]); cudaStreamDestroy(sts2[d][1]);
            cudaEventDestroy(e0[d]); cudaEventDestroy(e1[d]);
          }
        }
      }
  }
  return 0;
}

// Local HBM copy mode ("hbm", one GPU): the virtual-stage hand-off copy, SIMT vs TMA bulk.
static int hbm() {
  CK(cudaSetDevice(0));
  const size_t maxb = 256ull << 20;
  uint8_t *a, *b;
  CK(cudaMalloc(&a, maxb)); CK(cudaMemset(a, 1, maxb));
  CK(cudaMalloc(&b, maxb)); CK(cudaMemset(b, 0, maxb));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  const int S = 6;
  for (int tile : {16 << 10, 32 << 10})
    CK(cudaFuncSetAttribute(tma_copy<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * tile));
  for (size_t bytes : {32ull << 20, 256ull << 20}) {
    const int reps = bytes <= (32u << 20) ? 50 : 10;
    auto run = [&](const char* name, int grid, auto launch) {
      cudaEvent_t e0, e1;
      CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
      launch();
      CK(cudaStreamSynchronize(st));
      CK(cudaEventRecord(e0, st));
      for (int r = 0; r < reps; ++r) launch();
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double us = ms * 1e3 / reps;
      printf("{\"hbm\": \"%s\", \"bytes\": %zu, \"grid\": %d, \"us\": %.2f, \"rw_gbps\": %.1f}\n",
             name, bytes, grid, us, 2.0 * bytes / (us * 1e-6) / 1e9);
      fflush(stdout);
      cudaEventDestroy(e0); cudaEventDestroy(e1);
    };
    const size_t nv = bytes / 32;
    for (int g : {148, 296, 592}) {
      run("simt_u4", g, [&] { simt_copy<4, false><<<g, 512, 0, st>>>((V32*)b, (const V32*)a, nv); });
      run("simt_u8", g, [&] { simt_copy<8, false><<<g, 512, 0, st>>>((V32*)b, (const V32*)a, nv); });
      run("tma_32K", g, [&] { tma_copy<S><<<g, 32, S * (32 << 10), st>>>(b, a, bytes, 32 << 10); });
      run("tma_16K", g, [&] { tma_copy<S><<<g, 32, S * (16 << 10), st>>>(b, a, bytes, 16 << 10); });
    }
    run("memcpy_d2d", 0, [&] { CK(cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice, st)); });
  }
  return 0;
}

// PCIe mode ("pcie", one GPU): the e2e roofline.  Pinned host <-> device copies of 32 MiB
// messages (the C2 boundary), 16 back to back per direction, H2D alone, D2H alone, and both
// at once on two streams (the e2e step moves 512 MiB each way per step).
static int pcie() {
  CK(cudaSetDevice(0));
  const size_t msg = 32ull << 20;
  const int n = 16;
  uint8_t *hin, *hout, *din, *dout;
  CK(cudaMallocHost(&hin, msg * n)); memset(hin, 1, msg * n);
  CK(cudaMallocHost(&hout, msg * n)); memset(hout, 0, msg * n);
  CK(cudaMalloc(&din, msg * n));
  CK(cudaMalloc(&dout, msg * n)); CK(cudaMemset(dout, 2, msg * n));
  cudaStream_t sh, sd;
  CK(cudaStreamCreateWithFlags(&sh, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking));
  cudaEvent_t e0, e1, e2;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1)); CK(cudaEventCreate(&e2));
  for (int mode = 0; mode < 3; ++mode)
    for (int rep = 0; rep < 4; ++rep) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0, sh));
      CK(cudaStreamWaitEvent(sd, e0, 0));
      for (int i = 0; i < n; ++i) {
        if (mode != 1) CK(cudaMemcpyAsync(din + i * msg, hin + i * msg, msg, cudaMemcpyHostToDevice, sh));
        if (mode != 0) CK(cudaMemcpyAsync(hout + i * msg, dout + i * msg, msg, cudaMemcpyDeviceToHost, sd));
      }
      CK(cudaEventRecord(e1, sh));
      CK(cudaEventRecord(e2, sd));
      CK(cudaDeviceSynchronize());
      float a = 0, b = 0;
      CK(cudaEventElapsedTime(&a, e0, e1));
      CK(cudaEventElapsedTime(&b, e0, e2));
      const float ms = mode == 0 ? a : mode == 1 ? b : std::max(a, b);
      const double gb = (double)msg * n / 1e9;
      printf("{\"pcie\": \"%s\", \"rep\": %d, \"bytes_per_dir\": %zu, \"ms\": %.3f, "
             "\"h2d_gbps\": %.1f, \"d2h_gbps\": %.1f}\n",
             mode == 0 ? "h2d" : mode == 1 ? "d2h" : "both", rep, msg * n, ms,
             mode != 1 ? gb / (a * 1e-3) : 0.0, mode != 0 ? gb / (b * 1e-3) : 0.0);
      fflush(stdout);
    }
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "hbm") return hbm();
  if (argc > 1 && std::string(argv[1]) == "pcie") return pcie();
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("{\"error\": \"needs 2 GPUs\"}\n"); return 0; }
  CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0));
  if (argc > 1 && std::string(argv[1]) == "bidir") return bidir();
  const size_t sizes[] = {32ull << 20, 256ull << 20, 1ull << 30};
  const size_t maxb = 1ull << 30;
  uint8_t *a0, *b1;
  CK(cudaSetDevice(0)); CK(cudaMalloc(&a0, maxb)); CK(cudaMemset(a0, 1, maxb));
  CK(cudaSetDevice(1)); CK(cudaMalloc(&b1, maxb)); CK(cudaMemset(b1, 0, maxb));
  cudaStream_t s0, s1;
  CK(cudaSetDevice(0)); CK(cudaStreamCreate(&s0));
  CK(cudaSetDevice(1)); CK(cudaStreamCreate(&s1));
  const int tile = 32 << 10, S = 6;
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaFuncSetAttribute(tma_copy<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * tile));
  }
  const int grids[] = {16, 32, 64, 96, 128, 148, 296};
  for (size_t bytes : sizes) {
    const int reps = bytes <= (32u << 20) ? 50 : 10;
    auto run = [&](const char* name, int dev, cudaStream_t st, int grid, auto launch) {
      CK(cudaSetDevice(dev));
      cudaEvent_t e0, e1;
      CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
      launch();
      CK(cudaStreamSynchronize(st));
      CK(cudaEventRecord(e0, st));
      for (int r = 0; r < reps; ++r) launch();
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double us = ms * 1e3 / reps;
      printf("{\"mover\": \"%s\", \"bytes\": %zu, \"grid\": %d, \"us\": %.2f, \"gbps\": %.1f}\n", name,
             bytes, grid, us, bytes / (us * 1e-6) / 1e9);
      fflush(stdout);
      cudaEventDestroy(e0); cudaEventDestroy(e1);
    };
    const size_t nv = bytes / 32;
    uint64_t* flags1;
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&flags1, 1 << 16));
    for (int g : grids) {
      for (size_t ch : {256ull << 10, 1ull << 20}) {
        const size_t cv = ch / 32;
        char n1[64], n2[64];
        snprintf(n1, 64, "flag_allfence_c%zuK", ch >> 10);
        snprintf(n2, 64, "flag_fence1_c%zuK", ch >> 10);
        run(n1, 0, s0, g, [&] { simt_store_flagged<4, true><<<g, 512, 0, s0>>>((V32*)b1, (const V32*)a0, nv, cv, flags1, 1); });
        run(n2, 0, s0, g, [&] { simt_store_flagged<4, false><<<g, 512, 0, s0>>>((V32*)b1, (const V32*)a0, nv, cv, flags1, 1); });
      }
      run("simt_store_u4", 0, s0, g, [&] { simt_copy<4, false><<<g, 512, 0, s0>>>((V32*)b1, (const V32*)a0, nv); });
      run("simt_store_u8", 0, s0, g, [&] { simt_copy<8, false><<<g, 512, 0, s0>>>((V32*)b1, (const V32*)a0, nv); });
      run("simt_load_u4", 1, s1, g, [&] { simt_copy<4, true><<<g, 512, 0, s1>>>((V32*)b1, (const V32*)a0, nv); });
      run("simt_load_u8", 1, s1, g, [&] { simt_copy<8, true><<<g, 512, 0, s1>>>((V32*)b1, (const V32*)a0, nv); });
      run("tma_store", 0, s0, g, [&] { tma_copy<S><<<g, 32, S * tile, s0>>>(b1, a0, bytes, tile); });
      run("tma_load", 1, s1, g, [&] { tma_copy<S><<<g, 32, S * tile, s1>>>(b1, a0, bytes, tile); });
    }
    run("ce_memcpy_peer", 0, s0, 0, [&] { CK(cudaMemcpyPeerAsync(b1, 1, a0, 0, bytes, s0)); });
  }
  return 0;
}
