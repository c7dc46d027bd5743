// Probe for a 128-byte-line protocol over NVLink (design input for the 1–16 MB gap,
// DESIGN.md §8): a warp writes 128-byte lines into a peer with one 16-byte volatile store per
// lane, the line's last 8 bytes carrying the flag; the reader polls only the flag word and
// then checks the other 120 bytes.  If lines were ever observed torn (flag new, payload old)
// the protocol would be unsafe on this fabric.  Counts torn lines over many lines/iterations.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/probe_ll128 tools/probe_ll128.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      fprintf(stderr, "%s: %s (%s:%d)\n", #x, cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

__device__ __forceinline__ uint64_t val(uint32_t it, uint64_t line, int word) {
  uint64_t z = ((uint64_t)it << 40) ^ (line << 4) ^ (uint64_t)word;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  return z ^ (z >> 27);
}

// lanes 8q..8q+7 write line (base + q): lane 8q+k stores words 2k, 2k+1; word 15 = flag
__global__ void k_write(uint64_t* dst, uint64_t lines, uint32_t it) {
  const int lane = threadIdx.x & 31, q = lane >> 3, k = lane & 7;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t l0 = warp * 4; l0 < lines; l0 += nwarps * 4) {
    const uint64_t line = l0 + q;
    if (line >= lines) continue;
    uint64_t a = val(it, line, 2 * k), b = (k == 7) ? (uint64_t)it : val(it, line, 2 * k + 1);
    uint64_t* p = dst + line * 16 + 2 * k;
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
  }
}

__global__ void k_read(const uint64_t* src, uint64_t lines, uint32_t it, unsigned long long* torn,
                       unsigned long long* checked, unsigned long long* timeouts) {
  const int lane = threadIdx.x & 31, q = lane >> 3, k = lane & 7;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t l0 = warp * 4; l0 < lines; l0 += nwarps * 4) {
    const uint64_t line = l0 + q;
    const bool have = line < lines;
    uint64_t a = 0, b = 0;
    long long t0 = clock64();
    bool ok = false;
    while (true) {
      if (have)
        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(src + line * 16 + 2 * k)
                     : "memory");
      // the line is ready when lane 8q+7 sees the flag; broadcast within the 8-lane group
      const unsigned flag_ok = __ballot_sync(0xffffffffu, have && k == 7 && b == (uint64_t)it);
      ok = (flag_ok >> (q * 8 + 7)) & 1u;
      const unsigned all = __ballot_sync(0xffffffffu, !have || ok);
      if (all == 0xffffffffu) break;
      if (clock64() - t0 > 400000000ll) {  // ~0.2 s: give up on this launch
        if (lane == 0) atomicAdd(timeouts, 1ull);
        return;
      }
    }
    if (have && ok) {
      const bool good = a == val(it, line, 2 * k) && (k == 7 || b == val(it, line, 2 * k + 1));
      if (!good) atomicAdd(torn, 1ull);
      if (k == 0) atomicAdd(checked, 1ull);
    }
  }
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) return 0;
  const uint64_t lines = 1 << 20;  // 128 MB per iteration
  const int iters = 24;
  uint64_t* buf;  // on GPU 1, written by GPU 0
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&buf, lines * 128 * iters));
  CK(cudaMemset(buf, 0, lines * 128 * iters));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  unsigned long long *torn, *checked, *timeouts;
  CK(cudaMallocManaged(&torn, 8));
  CK(cudaMallocManaged(&checked, 8));
  CK(cudaMallocManaged(&timeouts, 8));
  *torn = *checked = *timeouts = 0;
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  cudaStream_t s0, s1;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaSetDevice(1));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  for (int it = 1; it <= iters; ++it) {
    uint64_t* region = buf + (uint64_t)(it - 1) * lines * 16;
    CK(cudaSetDevice(1));
    k_read<<<148, 256, 0, s1>>>(region, lines, (uint32_t)it, torn, checked, timeouts);  // reader first: polls
    CK(cudaSetDevice(0));
    k_write<<<148 * 2, 256, 0, s0>>>(region, lines, (uint32_t)it);
    CK(cudaStreamSynchronize(s0));
    CK(cudaSetDevice(1));
    CK(cudaStreamSynchronize(s1));
  }
  printf("{\"probe\": \"ll128 over NVLink\", \"lines_checked\": %llu, \"torn\": %llu, \"timeouts\": %llu, "
         "\"bytes_per_line\": 128}\n",
         *checked, *torn, *timeouts);
  return 0;
}
