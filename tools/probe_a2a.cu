// Probe: all-to-all push bandwidth (every GPU writes `bytes` to each of its N-1 peers at
// once, the reduce-scatter traffic pattern) for copy engines vs SM stores.
//   ce1   : N-1 cudaMemcpyAsync on one stream per GPU (the TWOSHOT_CE push)
//   ceN   : one stream per peer
//   sm<c> : one kernel per GPU, c CTAs, CTA b writes to peer (b % (N-1)), 8 x 16 B per thread in flight
// Reported: per-GPU out bandwidth = (N-1)*bytes / max-over-GPUs time.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/probe_a2a tools/probe_a2a.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                                \
  do {                                                                                       \
    cudaError_t e = (x);                                                                     \
    if (e != cudaSuccess) {                                                                  \
      fprintf(stderr, "%s: %s (%s:%d)\n", #x, cudaGetErrorString(e), __FILE__, __LINE__);   \
      exit(1);                                                                               \
    }                                                                                        \
  } while (0)

constexpr int kMax = 8;
struct Dsts {
  int4* p[kMax];
  int n;
};

__global__ void k_push(const int4* __restrict__ src, Dsts d, uint64_t n16) {
  const int peer = blockIdx.x % d.n;
  const int per = gridDim.x / d.n, b = blockIdx.x / d.n;
  int4* dst = d.p[peer];
  const uint64_t st = (uint64_t)per * blockDim.x;
  uint64_t i = b * (uint64_t)blockDim.x + threadIdx.x;
  for (; i + 7 * st < n16; i += 8 * st) {
    int4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + i + u * st);
#pragma unroll
    for (int u = 0; u < 8; ++u) __stcg(dst + i + u * st, v[u]);
  }
  for (; i < n16; i += st) __stcg(dst + i, __ldcg(src + i));
}

int main() {
  int N = 0;
  CK(cudaGetDeviceCount(&N));
  if (N < 2) return 0;
  if (N > kMax) N = kMax;
  const uint64_t sizes[] = {8ull << 20, 32ull << 20, 64ull << 20};
  void* src[kMax];
  void* rx[kMax];  // rx[d]: (N) slots of max bytes
  const uint64_t maxb = 64ull << 20;
  cudaStream_t st[kMax][kMax];
  cudaEvent_t e0[kMax], e1[kMax];
  for (int d = 0; d < N; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMalloc(&src[d], maxb));
    CK(cudaMemset(src[d], d + 1, maxb));
    CK(cudaMalloc(&rx[d], maxb * N));
    for (int p = 0; p < N; ++p)
      if (p != d) CK(cudaDeviceEnablePeerAccess(p, 0));
    for (int k = 0; k < N; ++k) CK(cudaStreamCreateWithFlags(&st[d][k], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  const char* modes[] = {"ce1", "ceN", "sm16", "sm32", "sm48", "sm64", "sm148", "sm296"};
  const int ctas[] = {0, 0, 16, 32, 48, 64, 148, 296};
  for (uint64_t bytes : sizes) {
    for (int m = 0; m < 8; ++m) {
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        for (int d = 0; d < N; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaDeviceSynchronize());
        }
        for (int d = 0; d < N; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventRecord(e0[d], st[d][0]));
          for (int k = 1; k < N; ++k) CK(cudaStreamWaitEvent(st[d][k], e0[d], 0));
          if (m < 2) {
            for (int k = 1; k < N; ++k) {
              int p = (d + k) % N;
              cudaStream_t s = m == 0 ? st[d][0] : st[d][k];
              CK(cudaMemcpyAsync((uint8_t*)rx[p] + d * maxb, src[d], bytes, cudaMemcpyDeviceToDevice, s));
            }
            if (m == 1)
              for (int k = 1; k < N; ++k) {
                cudaEvent_t ev;
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                CK(cudaEventRecord(ev, st[d][k]));
                CK(cudaStreamWaitEvent(st[d][0], ev, 0));
                CK(cudaEventDestroy(ev));
              }
          } else {
            Dsts ds{};
            for (int k = 1; k < N; ++k) ds.p[ds.n++] = (int4*)((uint8_t*)rx[(d + k) % N] + d * maxb);
            int g = ctas[m] / ds.n * ds.n;
            k_push<<<g, 512, 0, st[d][0]>>>((const int4*)src[d], ds, bytes / 16);
            CK(cudaGetLastError());
          }
          CK(cudaEventRecord(e1[d], st[d][0]));
        }
        float worst = 0;
        for (int d = 0; d < N; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventSynchronize(e1[d]));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
          if (ms > worst) worst = ms;
        }
        if (rep && worst < best) best = worst;
      }
      double out = (double)(N - 1) * bytes / (best / 1e3) / 1e9;
      printf("{\"n_gpus\": %d, \"mode\": \"%s\", \"bytes_per_peer\": %llu, \"ms\": %.4f, \"out_GBps_per_gpu\": %.1f}\n", N,
             modes[m], (unsigned long long)bytes, best, out);
      fflush(stdout);
    }
  }
  return 0;
}
