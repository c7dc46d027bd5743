// pgx — B200-native per-layer gradient exchange (arXiv 1706.00095 hot path).
// Shared device/host helpers: error plumbing, system-scope release/acquire
// flag operations for one-sided notify-writes over NVLink, vector memory ops.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/pgx.h"

namespace pgx {

// ---------------------------------------------------------------- host errors
void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);

#define PGX_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t e__ = (call);                                                       \
    if (e__ != cudaSuccess)                                                         \
      return ::pgx::fail(PGX_E_CUDA, "%s failed: %s (%s:%d)", #call,                \
                         cudaGetErrorString(e__), __FILE__, __LINE__);              \
  } while (0)

#define PGX_LAUNCH_CHECK()                                                          \
  do {                                                                              \
    cudaError_t e__ = cudaGetLastError();                                           \
    if (e__ != cudaSuccess)                                                         \
      return ::pgx::fail(PGX_E_CUDA, "kernel launch failed: %s (%s:%d)",            \
                         cudaGetErrorString(e__), __FILE__, __LINE__);              \
  } while (0)

// ------------------------------------------------------- device memory model
// A notify-write is: payload stores (weak, any thread) -> CTA barrier ->
// one thread: fence.acq_rel.sys + relaxed store / red of the flag.  The bar.sync
// orders the CTA's payload stores before the fence (causality order is
// transitive through the barrier); the .sys fence makes them visible to every
// agent (the peer GPU) before the flag.  The consumer does ld.acquire.sys on the
// flag, then bar.sync, then reads the payload with L1-bypassing loads.

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// 128-bit loads that bypass L1 (.cg): receive slots are written by peers during
// the kernel's lifetime, so a stale L1 line must never serve them.
__device__ __forceinline__ float4 ld_cg_f4(const float4* p) { return __ldcg(p); }
__device__ __forceinline__ double2 ld_cg_d2(const double2* p) { return __ldcg(p); }
// Streaming 128-bit loads of data that is read exactly once (own gradients).
__device__ __forceinline__ float4 ld_cs_f4(const float4* p) { return __ldcs(p); }

// Wait until *flag >= want (epoch semantics).  Bounded: past the deadline the
// kernel records PGX_E_TIMEOUT in the status word and gives up the wait, so a
// dead peer can never wedge the GPU.  Returns false on timeout.
struct Status {
  uint32_t* word;          // host-mapped (zero-copy) status: 0 = ok
  uint64_t timeout_ns;     // 0 -> no timeout
};

__device__ __forceinline__ bool wait_geq(const uint32_t* flag, uint32_t want, Status st) {
  uint32_t v = ld_acquire_sys(flag);
  if ((int32_t)(v - want) >= 0) return true;
  uint64_t t0 = globaltimer_ns();
  uint32_t spins = 0;
  while (true) {
    v = ld_acquire_sys(flag);
    if ((int32_t)(v - want) >= 0) return true;
    if (++spins > 64) __nanosleep(spins > 4096 ? 1000 : 64);
    if ((spins & 255) == 0) {
      if (st.word && *(volatile uint32_t*)st.word) return false;  // someone else failed
      if (st.timeout_ns && globaltimer_ns() - t0 > st.timeout_ns) {
        if (st.word) atomicCAS(st.word, 0u, (uint32_t)PGX_E_TIMEOUT);
        return false;
      }
    }
  }
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace pgx
