// Probe: NVLink bandwidth one GPU can move to a peer as a function of the number of
// CTAs, for four mechanisms (no flags / fences, pure data movement):
//   0 sm-push  : ld.global.v4 local -> st.global.v4 peer (8 x 16 B in flight per thread)
//   1 tma-push : cp.async.bulk local -> smem ring -> cp.async.bulk peer (one thread per CTA)
//   2 sm-pull  : ld.global.v4 peer -> st.global.v4 local
//   3 tma-pull : cp.async.bulk peer -> smem ring -> cp.async.bulk local
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/probe_push tools/probe_push.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      fprintf(stderr, "%s: %s (%s:%d)\n", #x, cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

constexpr int kStage = 32768;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_sm(const int4* __restrict__ src, int4* __restrict__ dst, uint64_t n) {
  const uint64_t st = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; i + 7 * st < n; i += 8 * st) {
    int4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + i + u * st);
#pragma unroll
    for (int u = 0; u < 8; ++u) __stcg(dst + i + u * st, v[u]);
  }
  for (; i < n; i += st) __stcg(dst + i, __ldcg(src + i));
}

template <int S>
__global__ void k_tma(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint64_t bytes) {
  extern __shared__ __align__(128) uint8_t ring[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + S * kStage);
  if (threadIdx.x != 0) return;
  for (int k = 0; k < S; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[k])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint64_t tiles = bytes / kStage;
  uint32_t phase[S] = {};
  int slot = 0;
  uint64_t issued = 0;
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++issued) {
    if (issued >= (uint64_t)S) {  // the stage's previous store must have read smem
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(S - 1) : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[slot])), "r"(kStage) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(ring + slot * kStage)),
                 "l"(src + t * kStage), "r"(kStage), "r"(sa(&bars[slot]))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
            sa(&bars[slot])),
        "r"(phase[slot])
        : "memory");
    phase[slot] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + t * kStage),
                 "r"(sa(ring + slot * kStage)), "r"(kStage)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    slot = (slot + 1) % S;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// tma variant with loads issued S-1 tiles ahead (loads and stores both in flight)
template <int S>
__global__ void k_tma2(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint64_t bytes) {
  extern __shared__ __align__(128) uint8_t ring[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + S * kStage);
  if (threadIdx.x != 0) return;
  for (int k = 0; k < S; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[k])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint64_t tiles = bytes / kStage;
  const uint64_t mine = tiles > blockIdx.x ? (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto tile = [&](uint64_t j) { return blockIdx.x + j * gridDim.x; };
  auto load = [&](uint64_t j) {
    int s = (int)(j % S);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[s])), "r"(kStage) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(ring + s * kStage)),
                 "l"(src + tile(j) * kStage), "r"(kStage), "r"(sa(&bars[s]))
                 : "memory");
  };
  const uint64_t pre = mine < (uint64_t)(S - 1) ? mine : (uint64_t)(S - 1);
  for (uint64_t j = 0; j < pre; ++j) load(j);
  for (uint64_t j = 0; j < mine; ++j) {
    int s = (int)(j % S);
    uint32_t ph = (uint32_t)((j / S) & 1);
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
            sa(&bars[s])),
        "r"(ph)
        : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + tile(j) * kStage),
                 "r"(sa(ring + s * kStage)), "r"(kStage)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (j + S - 1 < mine) {
      // stage (j+S-1)%S was last used by the store of tile j-1: wait until it was read
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      load(j + S - 1);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const uint64_t bytes = 256ull << 20;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("{\"error\": \"needs 2 GPUs\"}\n");
    return 0;
  }
  void *a0, *a1, *b0, *b1;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&a1, bytes));
  CK(cudaMalloc(&b1, bytes));
  CK(cudaMemset(a1, 1, bytes));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaSetDevice(0));
  CK(cudaMalloc(&a0, bytes));
  CK(cudaMalloc(&b0, bytes));
  CK(cudaMemset(a0, 2, bytes));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  constexpr int S = 6;
  const int smem = S * kStage + S * 8;
  CK(cudaFuncSetAttribute(k_tma<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_tma2<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const char* names[] = {"sm-push", "tma-push", "tma2-push", "sm-pull", "tma-pull", "tma2-pull", "memcpy-push"};
  int ctas[] = {4, 8, 16, 32, 64, 148, 296};
  for (int mode = 0; mode < 7; ++mode) {
    for (int c : ctas) {
      if (mode == 6 && c != 4) continue;
      const void* src = (mode >= 3 && mode <= 5) ? a1 : a0;  // pull: read the peer
      void* dst = (mode >= 3 && mode <= 5) ? b0 : b1;        // push: write the peer
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        CK(cudaEventRecord(e0));
        switch (mode) {
          case 0:
          case 3: k_sm<<<c, 512>>>((const int4*)src, (int4*)dst, bytes / 16); break;
          case 1:
          case 4: k_tma<S><<<c, 32, smem>>>((const uint8_t*)src, (uint8_t*)dst, bytes); break;
          case 2:
          case 5: k_tma2<S><<<c, 32, smem>>>((const uint8_t*)src, (uint8_t*)dst, bytes); break;
          case 6: CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice)); break;
        }
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep && ms < best) best = ms;
      }
      printf("{\"mode\": \"%s\", \"ctas\": %d, \"ms\": %.4f, \"GBps\": %.1f, \"GBps_per_cta\": %.2f}\n", names[mode], c,
             best, bytes / (best / 1e3) / 1e9, bytes / (best / 1e3) / 1e9 / c);
      fflush(stdout);
    }
  }
  return 0;
}
