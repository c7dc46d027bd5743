// Device-driven per-layer gradient exchange (the fast path).
//
// Reference behaviour (pipelined.py:43-218, runtime.py:185-251): as each layer's
// gradient is emitted by backward, the rank one-sidedly writes it to its
// reduction parent with a notification; parents fold child contributions in
// ascending child order, the master applies the update and the new weights flow
// back down the same tree; no barrier anywhere.  Here the writes are NVLink peer
// stores issued by this GPU's SMs, notifications are u32 flags raised with a
// system-scope release, and the waits are device-side acquire spins, so the host
// never polls.
//
//   TREE         the paper's schedule: chunk-pipelined binomial reduce to rank 0,
//                fused update on rank 0, chunk-pipelined broadcast down the edges.
//   TWOSHOT      every rank pushes shard j of its gradient into owner j's receive
//                slot; owner j folds the N contributions in the SAME binomial order
//                (tree_sum<N>), applies the fused update, and stores the updated
//                shard straight into every peer's weight buffer.
//   TWOSHOT_CE   the same schedule with the shards moved by copy engines
//                (cudaMemcpyAsync + k_signal); the SM kernel only folds + updates.
//   TWOSHOT_CEP  copy-engine reduce-scatter, SM owner kernel (fold + update +
//                all-gather stores) on a capped grid.
//   ONESHOT      small layers: everyone pushes everything once, every rank folds
//                and updates its own copy; ONESHOT_LL does it fence-free with
//                {value, epoch} words.
//   NVLS         multicast objects: switch-side reduce (multimem.ld_reduce) and
//                broadcast (multimem.st); fp32 tolerance parity.
//
// All but NVLS give bit-identical weights to the reference fold order; modes
// ref64 / ref32 / fast32 / sum32 (update off) select the per-element update.  Work is split
// into chunks (the notification unit, runtime.py:209-222) claimed through a
// per-layer atomic queue: every non-waiting push chunk is claimed before any
// waiting chunk, so a launch makes progress with any number of resident CTAs.
#include <cuda.h>
#include <cuda_runtime.h>
#include <string.h>
#include <unistd.h>

#include <vector>

#include "pgx_common.cuh"
#include "pgx_tree.cuh"

namespace pgx {
int world_rank(pgx_world* w);
int world_size(pgx_world* w);
int world_device(pgx_world* w);
Status world_status(pgx_world* w);
bool world_seg(pgx_world* w, int rank, uint32_t id, void** data, uint32_t** flags, uint64_t* size);
}  // namespace pgx

using namespace pgx;

namespace {

constexpr int kThreads = 512;
constexpr uint64_t kAlignElems = 64;  // 256 B for f32 — layer/shard bases

template <class T>
struct VecT;
template <>
struct VecT<float> {
  using V = float4;
  static constexpr int W = 4;
};
template <>
struct VecT<double> {
  using V = double2;
  static constexpr int W = 2;
};

struct Pieces {
  const void* p[PGX_MAX_PIECES];
  uint64_t end[PGX_MAX_PIECES];  // cumulative element ends
  int n;
};

struct XArgs {
  Pieces g;                            // this rank's layer gradient
  void* model[PGX_MAX_RANKS];          // every rank's flat model buffer (element ptr to layer base)
  uint32_t* mflags[PGX_MAX_RANKS];     // every rank's model-segment flags
  void* rx[PGX_MAX_RANKS];             // every rank's receive area for this layer
  uint32_t* rxflags[PGX_MAX_RANKS];    // every rank's rx flags for this layer
  float* v;                            // momentum (local, layer base)
  uint32_t* queue;                     // [claim, done]
  uint64_t S, sl, CH;                  // layer elems, shard elems, chunk elems
  uint32_t C;                          // chunks per shard (twoshot) / per layer (tree)
  uint32_t dflag;                      // tree: index of this layer's first down flag in mflags
  uint32_t layer, epoch;
  int rank, world, parity, K;          // K: rx slots per parity
  uint32_t push_items, items;
  uint32_t item_begin, item_end;       // claimed range (phase selection)
  uint64_t olo, ohi;                   // TWOSHOT_CE owner sub-range (ohi == 0: the whole shard)
  uint64_t CHo;                        // TWOSHOT_L128: lines per owner item
  uint32_t Co;                         // TWOSHOT_L128: owner items
  int single_buffer;                   // rx parity fixed at 0 (TWOSHOT_CEP: host-addressed copies)
  int bulk_lean;                       // TWOSHOT_BULK: the lean footprint (PGX_XF_BULK_LEAN)
  unsigned long long* trace;           // debug: per-item globaltimer stamps (pgx_xchg_set_trace) or null
  const uint32_t* iter;                // device iteration counter (graph mode) or null
  double lr;
  float scale, mu, wd;
  int mode;
  Status st;
};

template <class T>
__device__ __forceinline__ T grad_elem(const Pieces& P, uint64_t e) {
  int k = 0;
  while (k < P.n - 1 && e >= P.end[k]) ++k;
  uint64_t base = k ? P.end[k - 1] : 0;
  return static_cast<const T*>(P.p[k])[e - base];
}

// Load W consecutive gradient elements starting at logical element e (cnt valid).
template <class T>
__device__ __forceinline__ void grad_vec(const Pieces& P, uint64_t e, int cnt, T* out) {
  constexpr int W = VecT<T>::W;
  int k = 0;
  while (k < P.n - 1 && e >= P.end[k]) ++k;
  uint64_t base = k ? P.end[k - 1] : 0;
  const T* src = static_cast<const T*>(P.p[k]) + (e - base);
  if (cnt == W && e + W <= P.end[k] && (reinterpret_cast<uintptr_t>(src) % sizeof(typename VecT<T>::V)) == 0) {
    typename VecT<T>::V v = __ldcs(reinterpret_cast<const typename VecT<T>::V*>(src));
    memcpy(out, &v, sizeof(v));
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) out[i] = i < cnt ? grad_elem<T>(P, e + i) : T(0);
  }
}

// The gradient of [lo, hi) when it lies in ONE piece at a 16-byte aligned address (the
// common case: only the slab holding the [W][b] boundary straddles pieces), else null.
// Owner loops resolve it once per slab instead of searching the piece table (dynamically
// indexed kernel parameters: LDC + short-scoreboard waits) for every vector.
template <class T>
__device__ __forceinline__ const T* slab_grad(const Pieces& P, uint64_t lo, uint64_t hi) {
  uint64_t pb = 0;
  for (int k = 0; k < P.n; ++k) {
    const uint64_t pe = P.end[k];
    if (lo >= pb && hi <= pe) {
      const T* g = static_cast<const T*>(P.p[k]) + (lo - pb);
      return (reinterpret_cast<uintptr_t>(g) & 15) ? nullptr : g;
    }
    pb = pe;
  }
  return nullptr;
}

// W gradient elements at logical element e: from the resolved slab pointer (gs = element
// lo) when there is one, else through the piece table.
template <class T>
__device__ __forceinline__ void grad_vec_slab(const T* gs, const Pieces& P, uint64_t lo, uint64_t e, int cnt, T* out) {
  constexpr int W = VecT<T>::W;
  if (gs) {
    const T* src = gs + (e - lo);
    if (cnt == W) {
      typename VecT<T>::V v = __ldcs(reinterpret_cast<const typename VecT<T>::V*>(src));
      memcpy(out, &v, sizeof(v));
    } else {
#pragma unroll
      for (int i = 0; i < W; ++i) out[i] = i < cnt ? src[i] : T(0);
    }
  } else {
    grad_vec<T>(P, e, cnt, out);
  }
}

template <class T>
__device__ __forceinline__ void ld_vec(const T* p, int cnt, T* out) {
  constexpr int W = VecT<T>::W;
  if (cnt == W) {
    typename VecT<T>::V v = __ldcg(reinterpret_cast<const typename VecT<T>::V*>(p));
    memcpy(out, &v, sizeof(v));
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) out[i] = i < cnt ? __ldcg(p + i) : T(0);
  }
}

template <class T>
__device__ __forceinline__ void st_vec(T* p, int cnt, const T* in) {
  constexpr int W = VecT<T>::W;
  if (cnt == W) {
    typename VecT<T>::V v;
    memcpy(&v, in, sizeof(v));
    *reinterpret_cast<typename VecT<T>::V*>(p) = v;
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i)
      if (i < cnt) p[i] = in[i];
  }
}

// Fused update of one element (pgx_mode), identical to pgx_ops.cu / the oracle.
template <class T>
__device__ __forceinline__ T apply_update(T w, T g, float& v, const XArgs& a) {
  if constexpr (sizeof(T) == 8) {
    return __dsub_rn(w, __dmul_rn(a.lr, g));
  } else {
    if (a.mode == PGX_MODE_REF32) return __double2float_rn(__dsub_rn((double)w, __dmul_rn(a.lr, (double)g)));
    if (a.mode == PGX_MODE_SUM32) return __fmul_rn(a.scale, g);
    float gg = __fadd_rn(__fmul_rn(a.scale, g), __fmul_rn(a.wd, w));
    float vv = __fadd_rn(__fmul_rn(a.mu, v), __fmul_rn((float)a.lr, gg));
    v = vv;
    return __fsub_rn(w, vv);
  }
}

template <class T>
__device__ __forceinline__ void update_vec(T* w, const T* g, float* v, int cnt, const XArgs& a) {
  constexpr int W = VecT<T>::W;
  if constexpr (sizeof(T) == 4) {
    if (a.mode == PGX_MODE_FAST32) {
      float vv[W];
      ld_vec<float>(v, cnt, vv);
#pragma unroll
      for (int k = 0; k < W; ++k) w[k] = apply_update<T>(w[k], g[k], vv[k], a);
      st_vec<float>(v, cnt, vv);
      return;
    }
  }
  float dummy = 0.f;
#pragma unroll
  for (int k = 0; k < W; ++k) w[k] = apply_update<T>(w[k], g[k], dummy, a);
}

// Owner work on U vectors per thread: all loads first (U*(N+2) 16-byte requests in
// flight), then tree-order fold, fused update, local + peer stores.
// kRemote: store the updated vector into every peer's weights (register path);
// tile != nullptr: also stage it in shared memory for TMA bulk stores.
template <int N, class T, int U, bool kRemote = true>
__device__ __forceinline__ void owner_vectors(const XArgs& a, const T* rxb, uint64_t lo, uint64_t hi,
                                              uint64_t q0, uint64_t nvec, T* tile = nullptr, const T* gs = nullptr) {
  constexpr int W = VecT<T>::W;
  const int me = a.rank;
  const bool fast = sizeof(T) == 4 && a.mode == PGX_MODE_FAST32;
  T vals[U][N][W];
  T w[U][W];
  float vv[U][W];
  int cnt[U];
  if (gs != nullptr && lo + (q0 + (uint64_t)(U - 1) * blockDim.x + 1) * W <= hi) {
    // every vector of this call is whole: straight-line code, all U*(N+2) loads in flight
    // before the first use (the per-vector count / piece checks serialised them)
    using V = typename VecT<T>::V;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t q = q0 + (uint64_t)u * blockDim.x, e = lo + q * W;
      cnt[u] = W;
#pragma unroll
      for (int s = 0; s < N; ++s) {
        const T* src = (s == me) ? gs + (e - lo) : rxb + (uint64_t)s * a.sl + q * W;
        const V x = __ldcg(reinterpret_cast<const V*>(src));
        memcpy(vals[u][s], &x, sizeof(x));
      }
      if (a.mode != PGX_MODE_SUM32) {
        const V x = __ldcg(reinterpret_cast<const V*>(static_cast<const T*>(a.model[me]) + e));
        memcpy(w[u], &x, sizeof(x));
      } else {
#pragma unroll
        for (int k = 0; k < W; ++k) w[u][k] = T(0);
      }
      if constexpr (sizeof(T) == 4) {
        if (fast) {
          const float4 x = __ldcg(reinterpret_cast<const float4*>(a.v + e));
          memcpy(vv[u], &x, sizeof(x));
        }
      }
    }
  } else
#pragma unroll
  for (int u = 0; u < U; ++u) {
    uint64_t q = q0 + (uint64_t)u * blockDim.x;
    uint64_t e = lo + q * W;
    cnt[u] = q < nvec ? (int)min((uint64_t)W, hi - e) : 0;
    if (cnt[u] > 0) {
#pragma unroll
      for (int s = 0; s < N; ++s) {
        if (s == me)
          grad_vec_slab<T>(gs, a.g, lo, e, cnt[u], vals[u][s]);
        else
          ld_vec<T>(rxb + (uint64_t)s * a.sl + q * W, cnt[u], vals[u][s]);
      }
      if (a.mode != PGX_MODE_SUM32) {  // update off: the weights are not an input
        ld_vec<T>(static_cast<const T*>(a.model[me]) + e, cnt[u], w[u]);
      } else {
#pragma unroll
        for (int k = 0; k < W; ++k) w[u][k] = T(0);
      }
      if (fast) ld_vec<float>(a.v + e, cnt[u], vv[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (cnt[u] <= 0) continue;
    uint64_t e = lo + (q0 + (uint64_t)u * blockDim.x) * W;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      T col[N];
#pragma unroll
      for (int s = 0; s < N; ++s) col[s] = vals[u][s][k];
      T g;
      if constexpr (sizeof(T) == 8)
        g = tree_sum<N>(col, AddF64{});
      else
        g = tree_sum<N>(col, AddF32{});
      w[u][k] = apply_update<T>(w[u][k], g, vv[u][k], a);
    }
    st_vec<T>(static_cast<T*>(a.model[me]) + e, cnt[u], w[u]);
    if (fast) st_vec<float>(a.v + e, cnt[u], vv[u]);
    if (tile) st_vec<T>(tile + (e - lo), cnt[u], w[u]);
    if constexpr (kRemote) {
#pragma unroll
      for (int s = 0; s < N; ++s)
        if (s != me) st_vec<T>(static_cast<T*>(a.model[s]) + e, cnt[u], w[u]);
    }
  }
}

// One thread raises a flag / counter on a peer after the CTA's payload stores.
__device__ __forceinline__ void cta_release_flag(uint32_t* flag, uint32_t value) {
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_sys();
    st_release_sys(flag, value);
  }
}

// Claim the next work item; the last CTA out resets the queue for the next launch.
__device__ __forceinline__ uint32_t claim(uint32_t* q, uint32_t* smem) {
  __syncthreads();
  if (threadIdx.x == 0) *smem = atomicAdd(q, 1u);
  __syncthreads();
  return *smem;
}
__device__ __forceinline__ void retire(uint32_t* q) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    uint32_t done = atomicAdd(q + 1, 1u);
    if (done == gridDim.x - 1) {
      q[0] = 0;
      q[1] = 0;
      __threadfence();
    }
  }
}

// Thread i < n waits on flags[i*stride] >= want; then the CTA proceeds.
__device__ __forceinline__ void cta_wait_flags(uint32_t* const* flags, int n, uint32_t want, const Status& st) {
  if (threadIdx.x < (unsigned)n) wait_geq(flags[threadIdx.x], want, st);
  __syncthreads();
}

// ============================================================== TMA helpers
// Bulk copies through the Tensor Memory Accelerator: global -> shared (mbarrier
// complete_tx) and shared -> (peer) global (bulk group).  One thread drives them, so a
// chunk's remote writes are full-line bulk stores issued without the SM's LSU pipe.
constexpr int kTmaStage = 16384;  // bytes per smem stage
constexpr int kTmaStages = 4;     // 64 KB = one default chunk in flight per CTA

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Copy [src, src+bytes) -> dst by TMA, 16-byte granular; returns the bytes NOT copied
// (a <16-byte tail or misaligned range is left to the caller).  Caller: one thread.
__device__ __forceinline__ uint64_t tma_copy(uint8_t* dst, const uint8_t* src, uint64_t bytes, uint8_t* stages,
                                             uint64_t* bars, uint32_t& phase) {
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) return bytes;
  uint64_t body = bytes & ~uint64_t(15), off = 0;
  while (off < body) {
    int used = 0;
    for (; used < kTmaStages && off + (uint64_t)used * kTmaStage < body; ++used) {
      uint64_t o = off + (uint64_t)used * kTmaStage;
      uint32_t n = (uint32_t)min((uint64_t)kTmaStage, body - o);
      mbar_expect_tx(&bars[used], n);
      tma_load(stages + used * kTmaStage, src + o, n, &bars[used]);
    }
    for (int k = 0; k < used; ++k) {
      uint64_t o = off + (uint64_t)k * kTmaStage;
      uint32_t n = (uint32_t)min((uint64_t)kTmaStage, body - o);
      mbar_wait(&bars[k], phase);
      tma_store(dst + o, stages + k * kTmaStage, n);
      tma_commit();
    }
    phase ^= 1u;
    off += (uint64_t)used * kTmaStage;
    tma_wait_all();  // stores finished (also frees the stages for the next round)
  }
  return bytes - body;
}

// ============================================================== TWOSHOT
// kTma (N > 1): push chunks and all-gather tiles move as TMA bulk copies through a
// 64 KB shared-memory buffer (dynamic smem), driven by thread 0.
template <int N, class T, bool kTma>
__global__ void __launch_bounds__(kThreads, (N <= 4 && !kTma) ? 2 : 1) k_twoshot(XArgs a) {
  constexpr int W = VecT<T>::W;
  const uint32_t epoch = a.iter ? *a.iter + 1 : a.epoch;
  const int parity = a.single_buffer ? 0 : (a.iter ? (int)(*a.iter & 1) : a.parity);
  extern __shared__ __align__(128) uint8_t tma_buf[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(tma_buf + kTmaStages * kTmaStage);
  uint32_t tma_phase = 0;
  if constexpr (kTma) {
    if (threadIdx.x == 0) {
      for (int k = 0; k < kTmaStages; ++k) mbar_init(&bars[k], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
  }

  __shared__ uint32_t s_item;
  __shared__ uint32_t* s_flags[PGX_MAX_RANKS];
  const int me = a.rank;
  while (true) {
    uint32_t it = claim(a.queue, &s_item) + a.item_begin;
    if (it >= a.item_end) break;
    if (N > 1 && it < a.push_items) {
      // ---- reduce-scatter push: chunk c of owner j's shard -> j's rx[parity][me]
      constexpr int NP = N > 1 ? N - 1 : 1;
      uint32_t c = it / NP;
      int j = it % NP;
      j += (j >= me);
      uint64_t lo = j * a.sl + (uint64_t)c * a.CH;
      uint64_t hi = min(min(lo + a.CH, (uint64_t)(j + 1) * a.sl), a.S);
      if (lo < hi && kTma) {
        T* dst = static_cast<T*>(a.rx[j]) + ((uint64_t)(parity * a.K + me) * a.sl + (lo - j * a.sl));
        if (threadIdx.x == 0) {
          uint64_t pb = 0;
          for (int k = 0; k < a.g.n; ++k) {  // the chunk may straddle gradient pieces (dW | db)
            uint64_t pe = a.g.end[k], ol = max(lo, pb), oh = min(hi, pe);
            if (ol < oh) {
              const uint8_t* src = static_cast<const uint8_t*>(a.g.p[k]) + (ol - pb) * sizeof(T);
              uint8_t* d = reinterpret_cast<uint8_t*>(dst + (ol - lo));
              uint64_t bytes = (oh - ol) * sizeof(T);
              uint64_t rest = tma_copy(d, src, bytes, tma_buf, bars, tma_phase);
              for (uint64_t b = bytes - rest; b < bytes; ++b) d[b] = src[b];  // ragged tail / misaligned
            }
            pb = pe;
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");  // async-proxy writes before the flag
          fence_acq_rel_sys();
          st_release_sys(a.rxflags[j] + (uint64_t)me * a.C + c, epoch);
        }
        __syncthreads();
      } else if (lo < hi) {
        T* dst = static_cast<T*>(a.rx[j]) + ((uint64_t)(parity * a.K + me) * a.sl + (lo - j * a.sl));
        uint64_t nvec = (hi - lo + W - 1) / W;
        constexpr int UP = 4;
        const T* gs = slab_grad<T>(a.g, lo, hi);
        for (uint64_t q0 = threadIdx.x; q0 < nvec; q0 += (uint64_t)UP * blockDim.x) {
          T buf[UP][W];
          int cnt[UP];
#pragma unroll
          for (int u = 0; u < UP; ++u) {
            uint64_t q = q0 + (uint64_t)u * blockDim.x;
            uint64_t e = lo + q * W;
            cnt[u] = q < nvec ? (int)min((uint64_t)W, hi - e) : 0;
            if (cnt[u] > 0) grad_vec_slab<T>(gs, a.g, lo, e, cnt[u], buf[u]);
          }
#pragma unroll
          for (int u = 0; u < UP; ++u)
            if (cnt[u] > 0) st_vec<T>(dst + (q0 + (uint64_t)u * blockDim.x) * W, cnt[u], buf[u]);
        }
        cta_release_flag(a.rxflags[j] + (uint64_t)me * a.C + c, epoch);
      }
    } else {
      // ---- owner: fold N contributions in tree order, update, all-gather store
      uint32_t c = it - a.push_items;
      uint64_t lo = me * a.sl + (uint64_t)c * a.CH;
      uint64_t hi = min(min(lo + a.CH, (uint64_t)(me + 1) * a.sl), a.S);
      if (lo >= hi) continue;
      if (threadIdx.x < N - 1) {
        int s = threadIdx.x + (threadIdx.x >= (unsigned)me);
        s_flags[threadIdx.x] = a.rxflags[me] + (uint64_t)s * a.C + c;
      }
      __syncthreads();
      cta_wait_flags(s_flags, N - 1, epoch, a.st);
      const T* rxb = static_cast<const T*>(a.rx[me]) + (uint64_t)parity * a.K * a.sl + (lo - me * a.sl);
      uint64_t nvec = (hi - lo + W - 1) / W;
      constexpr int U = N <= 2 ? 2 : 1;  // 2 CTAs/SM (64 regs) without spills
      const T* gs = slab_grad<T>(a.g, lo, hi);
      if constexpr (kTma) {
        T* tile = reinterpret_cast<T*>(tma_buf);
        for (uint64_t q0 = threadIdx.x; q0 < nvec; q0 += (uint64_t)U * blockDim.x)
          owner_vectors<N, T, U, false>(a, rxb, lo, hi, q0, nvec, tile, gs);
        __syncthreads();
        if (threadIdx.x == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
          const uint64_t bytes = (hi - lo) * sizeof(T), body = bytes & ~uint64_t(15);
          for (int d = 1; d < N; ++d) {
            uint8_t* dst = reinterpret_cast<uint8_t*>(static_cast<T*>(a.model[(me + d) % N]) + lo);
            for (uint64_t o = 0; o < body; o += kTmaStage) tma_store(dst + o, tma_buf + o, (uint32_t)min((uint64_t)kTmaStage, body - o));
            tma_commit();
          }
          tma_wait_all();
          for (int d = 1; d < N; ++d) {  // ragged tail of the layer
            uint8_t* dst = reinterpret_cast<uint8_t*>(static_cast<T*>(a.model[(me + d) % N]) + lo);
            for (uint64_t b = body; b < bytes; ++b) dst[b] = tma_buf[b];
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
          fence_acq_rel_sys();
          for (int d = 1; d < N; ++d) red_release_sys_add(a.mflags[(me + d) % N] + a.layer, 1u);
        }
        __syncthreads();  // the tile is reused by the next item
      } else {
        for (uint64_t q0 = threadIdx.x; q0 < nvec; q0 += (uint64_t)U * blockDim.x)
          owner_vectors<N, T, U>(a, rxb, lo, hi, q0, nvec, nullptr, gs);
        __syncthreads();
        if (threadIdx.x < N - 1) {
          int s = threadIdx.x + (threadIdx.x >= (unsigned)me);
          fence_acq_rel_sys();
          red_release_sys_add(a.mflags[s] + a.layer, 1u);
        }
      }
    }
  }
  retire(a.queue);
}

// Debug timeline (pgx_xchg_set_trace): item `it` -> [claim, mid, end, smid, 4 kernel-specific
// accumulators], thread 0 only.
__device__ __forceinline__ void trace_stamp(const XArgs& a, uint32_t it, int slot) {
  if (a.trace && threadIdx.x == 0) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    a.trace[(uint64_t)it * 8 + slot] = globaltimer_ns();
    a.trace[(uint64_t)it * 8 + 3] = sm;
  }
}

// ============================================================== TWOSHOT_BULK
// The two-shot schedule with every NVLink byte moved by the Tensor Memory Accelerator on
// a capped grid (the large-layer variant): per CTA one thread streams a slab through a
// shared-memory ring — cp.async.bulk global->smem (mbarrier complete_tx), smem->peer
// global (bulk group), loads issued S-1 tiles ahead and ring slots recycled as soon as
// the store has READ them (wait_group.read), so the bytes in flight on NVLink are not
// bounded by the ring.  One system fence + release flag per slab (~1 MB), not per 64 KB
// chunk (the per-chunk fence capped the register two-shot at ~7.5 GB/s per CTA).  Owner
// slabs fold the N contributions in tree order (tree_sum<N>) tile by tile into the ring
// and the elected thread bulk-stores each updated tile into every peer's weights.  16-24
// CTAs saturate NVLink (tools/probe_push.cu: 689 GB/s push from 16 CTAs), so the layer
// leaves the other SMs to the backward kernels it overlaps with.
constexpr int kBulkStage = 32768;  // bytes per push ring slot
// Two footprints: FULL owns an SM (512 threads, 224 KB ring: 3 loads + 4 stores in flight per
// CTA); LEAN (256 threads, 64 KB ring: 1 load + 1 store in flight) leaves room on the SM for
// the backward's CTAs, so the exchange is not starved of whole SMs while they run.
template <bool LEAN>
struct BulkGeo {
  static constexpr int kThreads = LEAN ? 256 : 512;
  static constexpr int kStages = LEAN ? 2 : 7;
  static constexpr int kAhead = LEAN ? 1 : 3;
  static constexpr int kRing = kStages * kBulkStage;
  static constexpr size_t kSmem = (size_t)kRing + kStages * sizeof(uint64_t);
};
constexpr int kBulkCtas = 24;      // default grid of a bulk layer

__device__ __forceinline__ void tma_wait_read_1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void tma_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(K) : "memory"); }

struct BulkSeg {
  const uint8_t* src;
  uint8_t* dst;
  uint64_t bytes;  // multiple of 16, both ends 16-byte aligned
};

// Tile j of the concatenated segments.
__device__ __forceinline__ uint32_t bulk_tile(const BulkSeg* s, int n, uint32_t j, const uint8_t** src, uint8_t** dst) {
  for (int k = 0; k < n; ++k) {
    const uint32_t t = (uint32_t)((s[k].bytes + kBulkStage - 1) / kBulkStage);
    if (j < t) {
      const uint64_t o = (uint64_t)j * kBulkStage;
      *src = s[k].src + o;
      *dst = s[k].dst + o;
      return (uint32_t)min((uint64_t)kBulkStage, s[k].bytes - o);
    }
    j -= t;
  }
  return 0;
}

// One thread: copy the segments through the ring, L loads and up to S - L stores in
// flight.  `gload` counts every load this CTA ever issued: load g uses slot g % S at
// mbarrier phase (g / S) & 1.  Returns with stores possibly in flight (caller: wait_group 0).
template <int S, int L>
__device__ __forceinline__ void bulk_stream(const BulkSeg* segs, int nseg, uint8_t* ring, uint64_t* bars,
                                            uint32_t& gload) {
  uint32_t n = 0;
  for (int k = 0; k < nseg; ++k) n += (uint32_t)((segs[k].bytes + kBulkStage - 1) / kBulkStage);
  auto load = [&](uint32_t j) {
    const int s = (int)((gload + j) % S);
    const uint8_t* src;
    uint8_t* dst;
    const uint32_t b = bulk_tile(segs, nseg, j, &src, &dst);
    mbar_expect_tx(&bars[s], b);
    tma_load(ring + (size_t)s * kBulkStage, src, b, &bars[s]);
  };
  const uint32_t pre = min(n, (uint32_t)L);
  for (uint32_t j = 0; j < pre; ++j) load(j);
  for (uint32_t j = 0; j < n; ++j) {
    const uint32_t g = gload + j;
    const int s = (int)(g % S);
    mbar_wait(&bars[s], (g / S) & 1u);
    const uint8_t* src;
    uint8_t* dst;
    const uint32_t b = bulk_tile(segs, nseg, j, &src, &dst);
    tma_store(dst, ring + (size_t)s * kBulkStage, b);
    tma_commit();
    if (j + L < n) {
      tma_wait_read<S - L>();  // slot (j+L)%S was read by the store of tile j+L-S
      load(j + L);
    }
  }
  gload += n;
}

// The fused update with the mode fixed at compile time (same per-element expressions as
// apply_update): the bulk kernel runs on few SMs, so its fold is issue-bound and every
// instruction per element counts.
template <int MODE, class T>
__device__ __forceinline__ T bulk_update(T w, T g, float& v, double lr, float scale, float mu, float wd) {
  if constexpr (MODE == PGX_MODE_REF64) {
    return __dsub_rn(w, __dmul_rn(lr, g));
  } else if constexpr (MODE == PGX_MODE_REF32) {
    return __double2float_rn(__dsub_rn((double)w, __dmul_rn(lr, (double)g)));
  } else if constexpr (MODE == PGX_MODE_SUM32) {
    return __fmul_rn(scale, g);
  } else {
    const float gg = __fadd_rn(__fmul_rn(scale, g), __fmul_rn(wd, w));
    const float vv = __fadd_rn(__fmul_rn(mu, v), __fmul_rn((float)lr, gg));
    v = vv;
    return __fsub_rn(w, vv);
  }
}

// Owner fold fed by TMA loads.  The LSU path (one 16-byte load per thread and stream)
// keeps ~48 KB in flight per SM and was lg_throttle-bound at ~39 GB/s per SM (ncu r5z:
// the 24-CTA owner phase of fc6 ran 395 us); bulk loads keep whole tiles of all N + 2
// input streams (N partials, w, v) in flight per CTA with no LSU slots at all.
// Warp-specialised: thread 0 of warp 0 is the producer — it issues the N + 2
// cp.async.bulk loads of a tile onto the stage's `full` mbarrier, waits on the stage's
// `done` mbarrier, bulk-stores the updated w tile into the local and every peer's
// weights and the v tile into the local momentum, and reloads a stage once
// wait_group.read says its stores have read it.  Warps 1.. are the consumers: wait
// `full`, fold their vectors from shared memory in tree order, apply the fused update,
// write w / v back IN PLACE and arrive on `done` (one arrival per warp).  No CTA-wide
// barrier per tile, so the consumers never wait for the producer's store bookkeeping
// (the first cut's per-tile __syncthreads left 0.55 eligible warps per scheduler, r6c).
template <int N, bool LEAN>
struct OwnerGeo {
  static constexpr int kTile = LEAN ? (N <= 4 ? 4096 : 2048) : (N <= 4 ? 8192 : 4096);  // bytes per stream
  static constexpr int kStage = (N + 2) * kTile;
  static constexpr int kStages0 = BulkGeo<LEAN>::kRing / kStage;
  static constexpr int kStages = kStages0 > 8 ? 8 : kStages0;
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Folds [lo, lo + body) of the owner slab (body: the 16-byte-granular prefix) through the
// TMA pipeline; returns the first element NOT done (lo when the slab is not eligible).
// `ouse` counts the tiles this CTA ever consumed (mbarrier phases), identical in all threads.
// obars[0..7] = full, obars[8..15] = done (count: consumer warps).
// kGather = false (TWOSHOT_CE: the copy engines all-gather): local stores only.
template <int N, class T, int MODE, bool LEAN, bool kGather = true>
__device__ __forceinline__ uint64_t owner_tma(const XArgs& a, const T* rx0, const T* gs, uint64_t lo, uint64_t hi,
                                              uint8_t* ring, uint64_t* obars, uint32_t& ouse) {
  using OG = OwnerGeo<N, LEAN>;
  constexpr int SO = OG::kStages;
  constexpr int TB = OG::kTile;
  constexpr int TE = TB / (int)sizeof(T);
  constexpr bool fast = MODE == PGX_MODE_FAST32;
  constexpr bool upd = MODE != PGX_MODE_SUM32;
  if constexpr (SO < 2) {
    return lo;
  } else {
    const int me = a.rank;
    T* wme = static_cast<T*>(a.model[me]);
    if (gs == nullptr) return lo;
    uintptr_t al = reinterpret_cast<uintptr_t>(wme + lo);
    if (fast) al |= reinterpret_cast<uintptr_t>(a.v + lo);
    for (int s = 0; s < N; ++s)
      if (s != me) al |= reinterpret_cast<uintptr_t>(rx0 + (uint64_t)s * a.sl + lo);
    if constexpr (kGather)
      for (int d = 1; d < N; ++d) al |= reinterpret_cast<uintptr_t>(static_cast<T*>(a.model[(me + d) % N]) + lo);
    if (al & 15) return lo;
    const uint64_t body = (((hi - lo) * sizeof(T)) & ~uint64_t(15)) / sizeof(T);
    const uint32_t nt = (uint32_t)((body + TE - 1) / TE);
    if (nt == 0) return lo;
    uint64_t* full = obars;
    uint64_t* done = obars + 8;
    auto tile_bytes = [&](uint32_t t) { return (uint32_t)(min((uint64_t)TE, lo + body - (lo + (uint64_t)t * TE)) * sizeof(T)); };
    if (threadIdx.x == 0) {
      // ---- producer
      constexpr uint32_t nstream = N + (upd ? 1 : 0) + (fast ? 1 : 0);
      auto issue = [&](uint32_t i) {  // tile i of the slab -> stage (ouse + i) % SO
        const uint64_t e0 = lo + (uint64_t)i * TE;
        const uint32_t nb = tile_bytes(i);
        const uint32_t st = (ouse + i) % SO;
        uint8_t* stage = ring + (size_t)st * OG::kStage;
        mbar_expect_tx(&full[st], nb * nstream);
#pragma unroll
        for (int s = 0; s < N; ++s)
          tma_load(stage + s * TB, (s == me) ? gs + (e0 - lo) : rx0 + (uint64_t)s * a.sl + e0, nb, &full[st]);
        if constexpr (upd) tma_load(stage + N * TB, wme + e0, nb, &full[st]);
        if constexpr (fast) tma_load(stage + (N + 1) * TB, a.v + e0, nb, &full[st]);
      };
      asm volatile("fence.proxy.async.global;" ::: "memory");  // acquired rx data -> async-proxy reads
      for (uint32_t i = 0; i < min(nt, (uint32_t)SO); ++i) issue(i);
      for (uint32_t t = 0; t < nt; ++t) {
        const uint32_t g = ouse + t, st = g % SO;
        const uint64_t e0 = lo + (uint64_t)t * TE;
        const uint32_t nb = tile_bytes(t);
        uint8_t* stage = ring + (size_t)st * OG::kStage;
        mbar_wait(&done[st], (g / SO) & 1u);  // the consumers wrote the tile's w / v
        tma_store(wme + e0, stage + N * TB, nb);
        if constexpr (kGather)
          for (int d = 1; d < N; ++d) tma_store(static_cast<T*>(a.model[(me + d) % N]) + e0, stage + N * TB, nb);
        if constexpr (fast) tma_store(a.v + e0, stage + (N + 1) * TB, nb);
        tma_commit();
        if (t >= 1 && t - 1 + SO < nt) {
          tma_wait_read<1>();  // the stores of tile t - 1 have read its stage
          issue(t - 1 + SO);
        }
      }
      tma_wait_read<0>();  // the ring is free for the next slab / the LSU tail
    } else if (threadIdx.x >= 32) {
      // ---- consumers
      using V = typename VecT<T>::V;
      constexpr int W = VecT<T>::W;
      const double lr = a.lr;
      const float scale = a.scale, mu = a.mu, wd = a.wd;
      const uint32_t ct = threadIdx.x - 32, nct = blockDim.x - 32;
      for (uint32_t t = 0; t < nt; ++t) {
        const uint32_t g = ouse + t, st = g % SO;
        const uint32_t nb = tile_bytes(t);
        uint8_t* stage = ring + (size_t)st * OG::kStage;
        mbar_wait(&full[st], (g / SO) & 1u);
        for (uint32_t q = ct; q < nb / 16; q += nct) {
          T vals[N][W], w[W];
          float vv[W];
#pragma unroll
          for (int s = 0; s < N; ++s) {
            const V x = *reinterpret_cast<const V*>(stage + s * TB + q * 16);
            memcpy(vals[s], &x, sizeof(x));
          }
          if constexpr (upd) {
            const V x = *reinterpret_cast<const V*>(stage + N * TB + q * 16);
            memcpy(w, &x, sizeof(x));
          }
          if constexpr (fast) {
            const float4 x = *reinterpret_cast<const float4*>(stage + (N + 1) * TB + q * 16);
            memcpy(vv, &x, sizeof(x));
          }
#pragma unroll
          for (int k = 0; k < W; ++k) {
            T col[N];
#pragma unroll
            for (int s = 0; s < N; ++s) col[s] = vals[s][k];
            T gsum;
            if constexpr (sizeof(T) == 8)
              gsum = tree_sum<N>(col, AddF64{});
            else
              gsum = tree_sum<N>(col, AddF32{});
            w[k] = bulk_update<MODE, T>(upd ? w[k] : T(0), gsum, vv[k], lr, scale, mu, wd);
          }
          V xo;
          memcpy(&xo, w, sizeof(xo));
          *reinterpret_cast<V*>(stage + N * TB + q * 16) = xo;  // w slot holds the output (also when upd is off)
          if constexpr (fast) {
            float4 xv;
            memcpy(&xv, vv, sizeof(xv));
            *reinterpret_cast<float4*>(stage + (N + 1) * TB + q * 16) = xv;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> async proxy
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&done[st]);
      }
    }
    ouse += nt;
    __syncthreads();
    return lo + body;
  }
}

// wait until at most k bulk groups are still reading their shared-memory sources
__device__ __forceinline__ void tma_wait_read_n(int k) {
  switch (k) {
    case 0: tma_wait_read<0>(); break;
    case 1: tma_wait_read<1>(); break;
    case 2: tma_wait_read<2>(); break;
    case 3: tma_wait_read<3>(); break;
    case 4: tma_wait_read<4>(); break;
    case 5: tma_wait_read<5>(); break;
    case 6: tma_wait_read<6>(); break;
    default: tma_wait_read<7>(); break;
  }
}

template <int N, class T, int MODE, bool LEAN>
__global__ void __launch_bounds__(BulkGeo<LEAN>::kThreads, 1) k_twoshot_bulk(XArgs a) {
  using G = BulkGeo<LEAN>;
  constexpr int W = VecT<T>::W;
  constexpr int S = G::kStages;
  const uint32_t epoch = a.iter ? *a.iter + 1 : a.epoch;
  const int parity = a.single_buffer ? 0 : (a.iter ? (int)(*a.iter & 1) : a.parity);
  extern __shared__ __align__(128) uint8_t ring[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + G::kRing);  // push ring mbarriers
  __shared__ uint32_t s_item;
  __shared__ uint32_t* s_flags[PGX_MAX_RANKS];
  __shared__ uint64_t obars[16];  // owner-tile mbarriers (owner_tma): full[8], done[8]
  if (threadIdx.x == 0) {
    for (int k = 0; k < S; ++k) mbar_init(&bars[k], 1);
    for (int k = 0; k < 8; ++k) mbar_init(&obars[k], 1);
    for (int k = 8; k < 16; ++k) mbar_init(&obars[k], blockDim.x / 32 - 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t gload = 0;  // thread 0's push load counter (mbarrier phases)
  uint32_t ouse = 0;   // owner tiles consumed (owner_tma phases)
  const int me = a.rank;
  constexpr bool fast = MODE == PGX_MODE_FAST32;
  constexpr bool upd = MODE != PGX_MODE_SUM32;
  const double lr = a.lr;
  const float scale = a.scale, mu = a.mu, wd = a.wd;
  while (true) {
    const uint32_t it = claim(a.queue, &s_item) + a.item_begin;
    if (it >= a.item_end) break;
    if (threadIdx.x == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // ring: generic <-> async
    trace_stamp(a, it, 0);
    if (N > 1 && it < a.push_items) {
      // ---- reduce-scatter: slab c of owner j's shard -> j's rx[parity][me]
      constexpr int NP = N > 1 ? N - 1 : 1;
      const uint32_t c = it / NP;
      const int j = (me + 1 + (int)(it % NP)) % N;  // rotated: ranks start on different owners
      const uint64_t lo = j * a.sl + (uint64_t)c * a.CH;
      const uint64_t hi = min(min(lo + a.CH, (uint64_t)(j + 1) * a.sl), a.S);
      if (lo >= hi) continue;
      T* dst = static_cast<T*>(a.rx[j]) + ((uint64_t)(parity * a.K + me) * a.sl + (lo - j * a.sl));
      BulkSeg segs[PGX_MAX_PIECES];
      int nseg = 0;
      uint64_t pb = 0;
      for (int k = 0; k < a.g.n; ++k) {  // the slab may straddle gradient pieces (dW | db)
        const uint64_t pe = a.g.end[k], ol = max(lo, pb), oh = min(hi, pe);
        if (ol < oh) {
          const T* src = static_cast<const T*>(a.g.p[k]) + (ol - pb);
          T* d = dst + (ol - lo);
          uint64_t head = 0, body = 0;
          const uintptr_t sa = reinterpret_cast<uintptr_t>(src), da = reinterpret_cast<uintptr_t>(d);
          if ((sa & 15) == (da & 15)) {  // co-aligned: scalar head, bulk body, scalar tail
            head = min(oh - ol, (uint64_t)(((16 - (sa & 15)) & 15) / sizeof(T)));
            body = ((oh - ol - head) * sizeof(T)) & ~uint64_t(15);
          }
          if (body) segs[nseg++] = {reinterpret_cast<const uint8_t*>(src + head), reinterpret_cast<uint8_t*>(d + head), body};
          const uint64_t tail0 = head + body / sizeof(T);
          for (uint64_t e = threadIdx.x; e < head; e += blockDim.x) d[e] = src[e];
          for (uint64_t e = tail0 + threadIdx.x; e < oh - ol; e += blockDim.x) d[e] = src[e];
        }
        pb = pe;
      }
      if (threadIdx.x == 0 && nseg) bulk_stream<S, G::kAhead>(segs, nseg, ring, bars, gload);
      trace_stamp(a, it, 1);
      __syncthreads();
      if (threadIdx.x == 0) {
        tma_wait_all();                                      // the slab's bulk writes are done
        asm volatile("fence.proxy.async.global;" ::: "memory");
        fence_acq_rel_sys();
        st_release_sys(a.rxflags[j] + (uint64_t)me * a.C + c, epoch);
      }
      trace_stamp(a, it, 2);
    } else {
      // ---- owner slab: fold the N contributions in tree order + fused update with the LSU
      // (local HBM streams, U vectors per thread, every load of a round in flight at once),
      // the updated weights staged in a shared-memory ring and all-gathered into every
      // peer's weights by TMA bulk stores (several rounds of stores in flight).
      const uint32_t c = it - a.push_items;
      const uint64_t lo = me * a.sl + (uint64_t)c * a.CH;
      const uint64_t hi = min(min(lo + a.CH, (uint64_t)(me + 1) * a.sl), a.S);
      if (lo >= hi) continue;
      if (threadIdx.x < N - 1) {
        const int s = threadIdx.x + (threadIdx.x >= (unsigned)me);
        s_flags[threadIdx.x] = a.rxflags[me] + (uint64_t)s * a.C + c;
      }
      __syncthreads();
      cta_wait_flags(s_flags, N - 1, epoch, a.st);
      trace_stamp(a, it, 1);
      const T* rx0 = static_cast<const T*>(a.rx[me]) + (uint64_t)parity * a.K * a.sl - (uint64_t)me * a.sl;
      T* wme = static_cast<T*>(a.model[me]);
      const T* gs = slab_grad<T>(a.g, lo, hi);
      const uint64_t lo_lsu = owner_tma<N, T, MODE, LEAN>(a, rx0, gs, lo, hi, ring, obars, ouse);
      constexpr int U = N <= 4 ? 4 : 2;                         // vectors per thread per round
      const uint64_t RE = (uint64_t)blockDim.x * U * W;         // elements per round
      const int K = (int)(G::kRing / (RE * sizeof(T)));         // output ring slots
      unsigned long long t_ld = 0, t_ring = 0, t_st = 0, t_x = 0;
      const bool tr = a.trace && threadIdx.x == 0;
      uint32_t r = 0;
      for (uint64_t t0 = lo_lsu; t0 < hi; t0 += RE, ++r) {  // the ragged (< 16 B) end, or an ineligible slab
        const uint64_t t1 = min(t0 + RE, hi);
        T* slot = reinterpret_cast<T*>(ring + (size_t)(r % K) * RE * sizeof(T));
        if (tr) t_x = globaltimer_ns();
        T vals[U][N][W], w[U][W];
        float vv[U][W];
        int cnt[U];
        if (gs != nullptr && t1 - t0 == RE) {
          // full round (every slab but a ragged last one): straight-line code, all U*(N+2)
          // 16-byte loads issued before the first use — no per-vector count checks or
          // piece lookups between them (those branches serialised the loads, ncu r5t/r5y)
          using V = typename VecT<T>::V;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint64_t e = t0 + ((uint64_t)u * blockDim.x + threadIdx.x) * W;
            cnt[u] = W;
#pragma unroll
            for (int s = 0; s < N; ++s) {
              const T* src = (s == me) ? gs + (e - lo) : rx0 + (uint64_t)s * a.sl + e;
              const V x = __ldcg(reinterpret_cast<const V*>(src));
              memcpy(vals[u][s], &x, sizeof(x));
            }
            if constexpr (upd) {
              const V x = __ldcg(reinterpret_cast<const V*>(wme + e));
              memcpy(w[u], &x, sizeof(x));
            }
            if constexpr (fast) {
              const float4 x = __ldcg(reinterpret_cast<const float4*>(a.v + e));
              memcpy(vv[u], &x, sizeof(x));
            }
          }
        } else {
#pragma unroll
          for (int u = 0; u < U; ++u) {  // every load of the round first
            const uint64_t e = t0 + ((uint64_t)u * blockDim.x + threadIdx.x) * W;
            cnt[u] = e < t1 ? (int)min((uint64_t)W, t1 - e) : 0;
            if (cnt[u] > 0) {
#pragma unroll
              for (int s = 0; s < N; ++s) {
                if (s == me)
                  grad_vec_slab<T>(gs, a.g, lo, e, cnt[u], vals[u][s]);
                else
                  ld_vec<T>(rx0 + (uint64_t)s * a.sl + e, cnt[u], vals[u][s]);
              }
              if constexpr (upd) ld_vec<T>(wme + e, cnt[u], w[u]);
              if constexpr (fast) ld_vec<float>(a.v + e, cnt[u], vv[u]);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (cnt[u] <= 0) continue;
          const uint64_t q = (uint64_t)u * blockDim.x + threadIdx.x;
#pragma unroll
          for (int k = 0; k < W; ++k) {
            T col[N];
#pragma unroll
            for (int s = 0; s < N; ++s) col[s] = vals[u][s][k];
            T gsum;
            if constexpr (sizeof(T) == 8)
              gsum = tree_sum<N>(col, AddF64{});
            else
              gsum = tree_sum<N>(col, AddF32{});
            w[u][k] = bulk_update<MODE, T>(upd ? w[u][k] : T(0), gsum, vv[u][k], lr, scale, mu, wd);
          }
          st_vec<T>(wme + t0 + q * W, cnt[u], w[u]);
          if constexpr (fast) st_vec<float>(a.v + t0 + q * W, cnt[u], vv[u]);
          if (N > 1) st_vec<T>(slot + q * W, cnt[u], w[u]);  // all-gather source
        }
        if (tr) t_ld += globaltimer_ns() - t_x;
        if (N > 1) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> async proxy
          __syncthreads();
          if (threadIdx.x == 0) {
            if (tr) t_x = globaltimer_ns();
            const uint64_t bytes = (t1 - t0) * sizeof(T), body = bytes & ~uint64_t(15);
            if (body)
              for (int d = 1; d < N; ++d) tma_store(static_cast<T*>(a.model[(me + d) % N]) + t0, slot, (uint32_t)body);
            tma_commit();  // one group per round (possibly empty)
            for (int d = 1; d < N; ++d) {  // ragged end of the layer (< 16 bytes)
              uint8_t* dst = reinterpret_cast<uint8_t*>(static_cast<T*>(a.model[(me + d) % N]) + t0);
              for (uint64_t b = body; b < bytes; ++b) dst[b] = reinterpret_cast<const uint8_t*>(slot)[b];
            }
            if (tr) t_st += globaltimer_ns() - t_x, t_x = globaltimer_ns();
            // the next round writes slot (r+1)%K, last read by round r+1-K's stores
            tma_wait_read_n(K - 1);
            if (tr) t_ring += globaltimer_ns() - t_x;
          }
          __syncthreads();
        }
      }
      if (N > 1 && threadIdx.x == 0) {
        tma_wait_all();
        asm volatile("fence.proxy.async.global;" ::: "memory");
        fence_acq_rel_sys();
        for (int d = 1; d < N; ++d) red_release_sys_add(a.mflags[(me + d) % N] + a.layer, 1u);
      }
      if (tr) {
        a.trace[(uint64_t)it * 8 + 4] = t_ld;    // loads + fold + update + local stores
        a.trace[(uint64_t)it * 8 + 5] = t_st;    // issuing the all-gather stores
        a.trace[(uint64_t)it * 8 + 6] = t_ring;  // waiting for an output slot
        a.trace[(uint64_t)it * 8 + 7] = r;       // rounds
      }
      trace_stamp(a, it, 2);
    }
  }
  if (threadIdx.x == 0) tma_wait_all();
  retire(a.queue);
}

// ============================================================== ONESHOT
// Small layers are latency-bound: every rank pushes its whole gradient to every peer
// (one NVLink traversal), then folds all N contributions in the same binomial order
// and applies the update to its own copy.  No all-gather, no second hop; bit-identical
// to the other variants because every rank evaluates the same expression.
template <int N, class T>
__global__ void __launch_bounds__(kThreads, (sizeof(T) == 4 && N >= 3 && N <= 4) ? 1 : 2) k_oneshot(XArgs a) {
  constexpr int W = VecT<T>::W;
  const uint32_t epoch = a.iter ? *a.iter + 1 : a.epoch;
  const int parity = a.iter ? (int)(*a.iter & 1) : a.parity;
  __shared__ uint32_t s_item;
  __shared__ uint32_t* s_flags[PGX_MAX_RANKS];
  const int me = a.rank;
  while (true) {
    uint32_t it = claim(a.queue, &s_item) + a.item_begin;
    if (it >= a.item_end) break;
    trace_stamp(a, it, 0);
    if (N > 1 && it < a.push_items) {
      constexpr int NP = N > 1 ? N - 1 : 1;
      uint32_t c = it / NP;
      int j = it % NP;
      j += (j >= me);
      uint64_t lo = (uint64_t)c * a.CH, hi = min(lo + a.CH, a.S);
      T* dst = static_cast<T*>(a.rx[j]) + ((uint64_t)(parity * a.K + me) * a.sl + lo);
      uint64_t nvec = (hi - lo + W - 1) / W;
      const T* gs = slab_grad<T>(a.g, lo, hi);
      for (uint64_t q = threadIdx.x; q < nvec; q += blockDim.x) {
        uint64_t e = lo + q * W;
        int cnt = (int)min((uint64_t)W, hi - e);
        T buf[W];
        grad_vec_slab<T>(gs, a.g, lo, e, cnt, buf);
        st_vec<T>(dst + q * W, cnt, buf);
      }
      trace_stamp(a, it, 1);
      cta_release_flag(a.rxflags[j] + (uint64_t)me * a.C + c, epoch);
      trace_stamp(a, it, 2);
    } else {
      uint32_t c = it - a.push_items;
      uint64_t lo = (uint64_t)c * a.CH, hi = min(lo + a.CH, a.S);
      if (threadIdx.x < N - 1) {
        int s = threadIdx.x + (threadIdx.x >= (unsigned)me);
        s_flags[threadIdx.x] = a.rxflags[me] + (uint64_t)s * a.C + c;
      }
      __syncthreads();
      cta_wait_flags(s_flags, N - 1, epoch, a.st);
      trace_stamp(a, it, 1);
      const T* rxb = static_cast<const T*>(a.rx[me]) + (uint64_t)parity * a.K * a.sl + lo;
      uint64_t nvec = (hi - lo + W - 1) / W;
      // fp32 and N <= 4: two vectors per thread in flight (the fold is load-latency bound;
      // profiles/r4i: 8 us of a 1 MB exchange at N=4 with one)
      constexpr int UO = (sizeof(T) == 4 && N <= 4) ? 2 : 1;
      const T* gs = slab_grad<T>(a.g, lo, hi);
      for (uint64_t q0 = threadIdx.x; q0 < nvec; q0 += (uint64_t)UO * blockDim.x)
        owner_vectors<N, T, UO, false>(a, rxb, lo, hi, q0, nvec, nullptr, gs);
      __syncthreads();
      trace_stamp(a, it, 2);
    }
  }
  retire(a.queue);
}

// ============================================================== ONESHOT_LL
// Latency path for small fp32 layers, fence-free: every element travels as one 8-byte
// word {value bits, epoch} (LL: the flag rides in the same single-copy-atomic word), four
// words per 16-byte volatile store.  Every rank writes its whole gradient into each peer's
// slot [parity][me]; every rank polls its own slots word by word until the epoch matches,
// folds the N contributions in the binomial order and updates its own copy (as ONESHOT, so
// bit-identical).  No bar.sync / fence / flag round trip between a store and its use: one
// NVLink traversal.  Items: C push chunks, then C fold chunks (claimed in order, so every
// push is claimed before any poll: no deadlock at any residency).  Costs 2x the bytes.
__device__ __forceinline__ void st_ll4(uint64_t* p, const float* v, int cnt, uint32_t ep) {
  if (cnt == 4) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(__float_as_uint(v[0])), "r"(ep),
                 "r"(__float_as_uint(v[1])), "r"(ep)
                 : "memory");
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p + 2), "r"(__float_as_uint(v[2])), "r"(ep),
                 "r"(__float_as_uint(v[3])), "r"(ep)
                 : "memory");
  } else {
    for (int i = 0; i < cnt; ++i)
      asm volatile("st.volatile.global.v2.u32 [%0], {%1, %2};" ::"l"(p + i), "r"(__float_as_uint(v[i])), "r"(ep)
                   : "memory");
  }
}

// Poll cnt words until every epoch field equals ep; bounded like wait_geq.
__device__ __forceinline__ bool ld_ll4(const uint64_t* p, float* v, int cnt, uint32_t ep, const Status& st) {
  uint64_t t0 = 0;
  for (uint32_t spins = 0;; ++spins) {
    uint32_t d[4], f[4];
    if (cnt == 4) {
      asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(d[0]), "=r"(f[0]), "=r"(d[1]), "=r"(f[1])
                   : "l"(p)
                   : "memory");
      asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(d[2]), "=r"(f[2]), "=r"(d[3]), "=r"(f[3])
                   : "l"(p + 2)
                   : "memory");
    } else {
      for (int i = 0; i < 4; ++i) {
        if (i < cnt)
          asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(d[i]), "=r"(f[i]) : "l"(p + i) : "memory");
        else
          d[i] = 0, f[i] = ep;
      }
    }
    if (f[0] == ep && f[1] == ep && f[2] == ep && f[3] == ep) {
      for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(d[i]);
      return true;
    }
    if (spins > 1024) __nanosleep(spins > 65536 ? 1000 : 32);
    if ((spins & 1023) == 1023) {
      if (!t0) t0 = globaltimer_ns();
      if (st.word && *(volatile uint32_t*)st.word) return false;
      if (st.timeout_ns && globaltimer_ns() - t0 > st.timeout_ns) {
        if (st.word) atomicCAS(st.word, 0u, (uint32_t)PGX_E_TIMEOUT);
        return false;
      }
    }
  }
}

template <int N>
__global__ void __launch_bounds__(kThreads, N <= 4 ? 2 : 1) k_oneshot_ll(XArgs a) {
  const uint32_t epoch = a.iter ? *a.iter + 1 : a.epoch;
  const int parity = a.iter ? (int)(*a.iter & 1) : a.parity;
  __shared__ uint32_t s_item;
  const int me = a.rank;
  auto slot = [&](int r, int s) {  // rank r's slot [parity][s]: one u64 word per element
    return reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(a.rx[r]) + (uint64_t)(parity * N + s) * a.sl * 4);
  };
  while (true) {
    uint32_t it = claim(a.queue, &s_item) + a.item_begin;
    if (it >= a.item_end) break;
    const bool push = it < a.push_items;
    const uint32_t c = push ? it : it - a.push_items;
    const uint64_t lo = (uint64_t)c * a.CH, hi = min(lo + a.CH, a.S);
    const uint64_t nq = (hi - lo + 3) / 4;
    if (push) {
      if (N == 1) continue;
      for (uint64_t q = threadIdx.x; q < nq; q += blockDim.x) {
        const uint64_t e = lo + q * 4;
        const int cnt = (int)min((uint64_t)4, hi - e);
        float g[4];
        grad_vec<float>(a.g, e, cnt, g);
#pragma unroll
        for (int d = 1; d < N; ++d) {
          const int j = (me + d) % N;
          st_ll4(slot(j, me) + e, g, cnt, epoch);
        }
      }
    } else {
      const bool fast = a.mode == PGX_MODE_FAST32;
      for (uint64_t q = threadIdx.x; q < nq; q += blockDim.x) {
        const uint64_t e = lo + q * 4;
        const int cnt = (int)min((uint64_t)4, hi - e);
        float vals[N][4];
        bool ok = true;
#pragma unroll
        for (int s = 0; s < N; ++s) {
          if (s == me)
            grad_vec<float>(a.g, e, cnt, vals[s]);
          else
            ok &= ld_ll4(slot(me, s) + e, vals[s], cnt, epoch, a.st);
        }
        if (!ok) break;  // timed out: the host raises TransportError
        float w[4] = {0.f, 0.f, 0.f, 0.f}, vv[4] = {0.f, 0.f, 0.f, 0.f};
        float* wp = static_cast<float*>(a.model[me]) + e;
        if (a.mode != PGX_MODE_SUM32) ld_vec<float>(wp, cnt, w);
        if (fast) ld_vec<float>(a.v + e, cnt, vv);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float col[N];
#pragma unroll
          for (int s = 0; s < N; ++s) col[s] = vals[s][k];
          w[k] = apply_update<float>(w[k], tree_sum<N>(col, AddF32{}), vv[k], a);
        }
        st_vec<float>(wp, cnt, w);
        if (fast) st_vec<float>(a.v + e, cnt, vv);
      }
    }
  }
  retire(a.queue);
}

// ============================================================== ONESHOT_L128
// ONESHOT over 128-byte lines: 30 fp32 values + an 8-byte {epoch, epoch} flag per line,
// written by 8 lanes of a warp with one 16-byte volatile store each (one line = one
// NVLink write, profiles/r4l: 25 M lines, none observed torn); the receiver polls the flag
// word of each line (lane 7), then uses the line.  No fence, 128/120 bytes on the wire
// (LL: 2x).  Items: C push chunks of lines, then C fold chunks (push-first claims).
constexpr int kL128Vals = 30;

template <int N>
__global__ void __launch_bounds__(kThreads, N <= 4 ? 2 : 1) k_oneshot_l128(XArgs a) {
  const uint32_t epoch = a.iter ? *a.iter + 1 : a.epoch;
  const int parity = a.iter ? (int)(*a.iter & 1) : a.parity;
  __shared__ uint32_t s_item;
  const int me = a.rank;
  const int lane = threadIdx.x & 31, q = lane >> 3, k = lane & 7;
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint64_t lines = (a.S + kL128Vals - 1) / kL128Vals;
  auto slot = [&](int r, int s) {  // rank r's slot [parity][s]: `lines` 128-byte lines
    return static_cast<uint8_t*>(a.rx[r]) + (uint64_t)(parity * N + s) * a.sl * 4;
  };
  const int nv = k < 7 ? 4 : 2;  // values carried by this lane
  while (true) {
    uint32_t it = claim(a.queue, &s_item) + a.item_begin;
    if (it >= a.item_end) break;
    const bool push = it < a.push_items;
    const uint32_t c = push ? it : it - a.push_items;
    const uint64_t l_lo = (uint64_t)c * a.CH, l_hi = min(l_lo + a.CH, lines);  // CH = lines per chunk
    bool failed = false;
    for (uint64_t l0 = l_lo + (uint64_t)warp * 4; l0 < l_hi && !failed; l0 += (uint64_t)nwarps * 4) {
      const uint64_t line = l0 + q;
      const bool have = line < l_hi;
      const uint64_t e0 = line * kL128Vals + 4 * k;
      if (push) {
        if (N == 1) break;
        uint32_t w4[4] = {0u, 0u, epoch, epoch};
        if (have)
          for (int i = 0; i < nv; ++i)
            if (e0 + i < a.S) w4[i] = __float_as_uint(grad_elem<float>(a.g, e0 + i));
        __syncwarp();  // the 8 lanes of a line store together: one 128-byte write
        if (have) {
#pragma unroll
          for (int d = 1; d < N; ++d) {
            uint8_t* p = slot((me + d) % N, me) + line * 128 + 16 * k;
            asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(w4[0]), "r"(w4[1]),
                         "r"(w4[2]), "r"(w4[3])
                         : "memory");
          }
        }
      } else {
        float vals[N][4];
#pragma unroll
        for (int s = 0; s < N; ++s) {
          if (s == me) {
            for (int i = 0; i < 4; ++i)
              vals[s][i] = (have && i < nv && e0 + i < a.S) ? grad_elem<float>(a.g, e0 + i) : 0.f;
            continue;
          }
          const uint8_t* p = slot(me, s) + line * 128 + 16 * k;
          uint64_t t0 = 0;
          for (uint32_t spins = 0;; ++spins) {
            uint32_t x0 = 0, x1 = 0, x2 = 0, x3 = 0;
            if (have)
              asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                           : "l"(p)
                           : "memory");
            const unsigned ok = __ballot_sync(0xffffffffu, k == 7 && have && x2 == epoch && x3 == epoch);
            const bool mine_ok = !have || ((ok >> (q * 8 + 7)) & 1u);
            vals[s][0] = __uint_as_float(x0);
            vals[s][1] = __uint_as_float(x1);
            vals[s][2] = __uint_as_float(x2);
            vals[s][3] = __uint_as_float(x3);
            if (__all_sync(0xffffffffu, mine_ok)) break;
            if (spins > 1024) __nanosleep(32);
            if ((spins & 1023) == 1023) {  // warp-uniform give-up decision (lane 0 decides)
              int stop = 0;
              if (lane == 0) {
                if (!t0) t0 = globaltimer_ns();
                stop = (a.st.word && *(volatile uint32_t*)a.st.word) ||
                       (a.st.timeout_ns && globaltimer_ns() - t0 > a.st.timeout_ns);
                if (stop && a.st.word) atomicCAS(a.st.word, 0u, (uint32_t)PGX_E_TIMEOUT);
              }
              if (__shfl_sync(0xffffffffu, stop, 0)) {
                failed = true;
                break;
              }
            }
          }
          if (failed) break;
        }
        if (failed || !have) continue;
        const bool fast = a.mode == PGX_MODE_FAST32;
        float* wp = static_cast<float*>(a.model[me]);
        for (int i = 0; i < nv; ++i) {
          const uint64_t e = e0 + i;
          if (e >= a.S) break;
          float col[N];
#pragma unroll
          for (int s = 0; s < N; ++s) col[s] = vals[s][i];
          float v = fast ? a.v[e] : 0.f;
          const float w = a.mode == PGX_MODE_SUM32 ? 0.f : wp[e];
          wp[e] = apply_update<float>(w, tree_sum<N>(col, AddF32{}), v, a);
          if (fast) a.v[e] = v;
        }
      }
    }
  }
  retire(a.queue);
}

// ============================================================== TWOSHOT_L128
// TWOSHOT over 128-byte lines (the ONESHOT_L128 line format: 30 fp32 values + an 8-byte
// {epoch, epoch} flag, one 16-byte volatile store per lane of an 8-lane group), for the
// 1-16 MB range where a system fence + flag per chunk costs more than the bytes:
//   push items    : line chunks of every peer's shard -> the owner's slot [parity][me]
//   owner items   : poll the N-1 slots of my shard's lines, fold in tree order with my own
//                   gradient, fused update into my weights (+ momentum), and the updated
//                   line -> every peer's gather area [parity][line]
//   install items : poll the gather area for another owner's lines -> my weights
// Items are claimed push < owner < install, so a CTA only waits on items already claimed
// by running CTAs (no deadlock at any residency).  No fence or flag round trip anywhere;
// (N-1)/N of the layer crosses NVLink twice at 128/120 bytes per value byte.
// Host-stepped launches: PHASE_PUSH, PHASE_OWNER, PHASE_DOWN (= install) in that order.

// 2 or 4 consecutive gradient values at logical element e (e even): two 8-byte loads when
// they sit in one piece at an 8-byte aligned address, else element by element.
__device__ __forceinline__ void l128_grad(const Pieces& P, uint64_t e, int cnt, int nv, uint32_t* w4) {
  int k = 0;
  while (k < P.n - 1 && e >= P.end[k]) ++k;
  const uint64_t base = k ? P.end[k - 1] : 0;
  const float* src = static_cast<const float*>(P.p[k]) + (e - base);
  if (cnt == nv && e + nv <= P.end[k] && (reinterpret_cast<uintptr_t>(src) & 7) == 0) {
    const float2 x = __ldcs(reinterpret_cast<const float2*>(src));
    w4[0] = __float_as_uint(x.x);
    w4[1] = __float_as_uint(x.y);
    if (nv == 4) {
      const float2 y = __ldcs(reinterpret_cast<const float2*>(src + 2));
      w4[2] = __float_as_uint(y.x);
      w4[3] = __float_as_uint(y.y);
    }
  } else {
    for (int i = 0; i < nv; ++i) w4[i] = i < cnt ? __float_as_uint(grad_elem<float>(P, e + i)) : 0u;
  }
}

// 2 or 4 fp32 values at p (8-byte aligned) / back.
__device__ __forceinline__ void l128_ld(const float* p, int cnt, int nv, float* out) {
  if (cnt == nv) {
    const float2 x = __ldcg(reinterpret_cast<const float2*>(p));
    out[0] = x.x;
    out[1] = x.y;
    if (nv == 4) {
      const float2 y = __ldcg(reinterpret_cast<const float2*>(p + 2));
      out[2] = y.x;
      out[3] = y.y;
    }
  } else {
    for (int i = 0; i < 4; ++i) out[i] = i < cnt ? __ldcg(p + i) : 0.f;
  }
}
__device__ __forceinline__ void l128_st(float* p, int cnt, int nv, const float* in) {
  if (cnt == nv) {
    *reinterpret_cast<float2*>(p) = make_float2(in[0], in[1]);
    if (nv == 4) *reinterpret_cast<float2*>(p + 2) = make_float2(in[2], in[3]);
  } else {
    for (int i = 0; i < cnt; ++i) p[i] = in[i];
  }
}

__device__ __forceinline__ void l128_put(uint8_t* p, const uint32_t* w4) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(w4[0]), "r"(w4[1]), "r"(w4[2]),
               "r"(w4[3])
               : "memory");
}

// Warp-collective: every 8-lane group polls its line (lane k's 16 bytes at p) until the
// group's lane 7 sees {epoch, epoch}; returns false (warp-uniform) on timeout / abort.
__device__ __forceinline__ bool l128_wait(const uint8_t* p, bool have, uint32_t epoch, int lane, uint32_t* x,
                                          const Status& st) {
  const int q = lane >> 3, k = lane & 7;
  uint64_t t0 = 0;
  for (uint32_t spins = 0;; ++spins) {
    x[0] = x[1] = x[2] = x[3] = 0;
    if (have)
      asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3])
                   : "l"(p)
                   : "memory");
    const unsigned ok = __ballot_sync(0xffffffffu, k == 7 && have && x[2] == epoch && x[3] == epoch);
    const bool mine_ok = !have || ((ok >> (q * 8 + 7)) & 1u);
    if (__all_sync(0xffffffffu, mine_ok)) return true;
    if (spins > 1024) __nanosleep(32);
    if ((spins & 1023) == 1023) {  // warp-uniform give-up decision (lane 0 decides)
      int stop = 0;
      if (lane == 0) {
        if (!t0) t0 = globaltimer_ns();
        stop = (st.word && *(volatile uint32_t*)st.word) || (st.timeout_ns && globaltimer_ns() - t0 > st.timeout_ns);
        if (stop && st.word) atomicCAS(st.word, 0u, (uint32_t)PGX_E_TIMEOUT);
      }
      if (__shfl_sync(0xffffffffu, stop, 0)) return false;
    }
  }
}

template <int N>
__global__ void __launch_bounds__(kThreads, N <= 4 ? 2 : 1) k_twoshot_l128(XArgs a) {
  const uint32_t epoch = a.iter ? *a.iter + 1 : a.epoch;
  const int parity = a.iter ? (int)(*a.iter & 1) : a.parity;
  __shared__ uint32_t s_item;
  const int me = a.rank;
  const int lane = threadIdx.x & 31, q = lane >> 3, k = lane & 7;
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint64_t lines = (a.S + kL128Vals - 1) / kL128Vals;
  const uint64_t Ls = (lines + N - 1) / N;                  // lines per owner shard
  const uint64_t agl = (lines * 32 + kAlignElems - 1) / kAlignElems * kAlignElems;
  uint8_t* const rx_me = static_cast<uint8_t*>(a.rx[me]);
  auto slot = [&](int r, int s) {  // rank r's reduce-scatter slot [parity][s] (Ls lines)
    return static_cast<uint8_t*>(a.rx[r]) + ((uint64_t)parity * (N * a.sl + agl) + (uint64_t)s * a.sl) * 4;
  };
  auto gather = [&](int r) {  // rank r's gather area [parity] (every line of the layer)
    return static_cast<uint8_t*>(a.rx[r]) + ((uint64_t)parity * (N * a.sl + agl) + (uint64_t)N * a.sl) * 4;
  };
  const int nv = k < 7 ? 4 : 2;  // values carried by this lane
  constexpr int NP = N > 1 ? N - 1 : 1;
  const uint32_t owner_end = a.push_items + a.Co;
  float* const wbase = static_cast<float*>(a.model[me]);
  const bool fast = a.mode == PGX_MODE_FAST32;
  while (true) {
    const uint32_t it = claim(a.queue, &s_item) + a.item_begin;
    if (it >= a.item_end) break;
    int kind, j;  // 0 push (to owner j), 1 owner (j = me), 2 install (from owner j)
    uint32_t c;
    if (it < a.push_items) {
      kind = 0;
      c = it / NP;
      j = (me + 1 + (int)(it % NP)) % N;
    } else if (it < owner_end) {  // owner items: CHo lines each (the heavier work, finer grain)
      kind = 1;
      c = it - a.push_items;
      j = me;
    } else {
      kind = 2;
      const uint32_t i2 = it - owner_end;
      c = i2 / NP;
      j = (me + 1 + (int)(i2 % NP)) % N;
    }
    const uint64_t s_lo = (uint64_t)j * Ls, s_hi = min(s_lo + Ls, lines);
    const uint64_t ch = kind == 1 ? a.CHo : a.CH;
    const uint64_t l_lo = s_lo + (uint64_t)c * ch, l_hi = min(l_lo + ch, s_hi);
    bool failed = false;
    for (uint64_t l0 = l_lo + (uint64_t)warp * 4; l0 < l_hi && !failed; l0 += (uint64_t)nwarps * 4) {
      const uint64_t line = l0 + q;
      const bool have = line < l_hi;
      const uint64_t e0 = line * kL128Vals + 4 * k;
      const int cnt = have && e0 < a.S ? (int)min((uint64_t)nv, a.S - e0) : 0;
      if (kind == 0) {
        uint32_t w4[4] = {0u, 0u, epoch, epoch};
        if (cnt) l128_grad(a.g, e0, cnt, nv, w4);
        __syncwarp();  // the 8 lanes of a line store together: one 128-byte write
        if (have) l128_put(slot(j, me) + (line - s_lo) * 128 + 16 * k, w4);
      } else if (kind == 1) {
        float vals[N][4];
#pragma unroll
        for (int s = 0; s < N; ++s) {
          uint32_t x[4];
          if (s == me) {
            x[0] = x[1] = x[2] = x[3] = 0u;
            if (cnt) l128_grad(a.g, e0, cnt, nv, x);
          } else if (!l128_wait(slot(me, s) + (line - s_lo) * 128 + 16 * k, have, epoch, lane, x, a.st)) {
            failed = true;
            break;
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) vals[s][i] = __uint_as_float(x[i]);
        }
        if (failed) break;
        float w[4] = {0.f, 0.f, 0.f, 0.f}, v[4] = {0.f, 0.f, 0.f, 0.f};
        if (cnt) {
          if (a.mode != PGX_MODE_SUM32) l128_ld(wbase + e0, cnt, nv, w);
          if (fast) l128_ld(a.v + e0, cnt, nv, v);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float col[N];
#pragma unroll
            for (int s = 0; s < N; ++s) col[s] = vals[s][i];
            w[i] = apply_update<float>(w[i], tree_sum<N>(col, AddF32{}), v[i], a);
          }
          l128_st(wbase + e0, cnt, nv, w);
          if (fast) l128_st(a.v + e0, cnt, nv, v);
        }
        uint32_t w4[4] = {__float_as_uint(w[0]), __float_as_uint(w[1]), epoch, epoch};
        if (nv == 4) {
          w4[2] = __float_as_uint(w[2]);
          w4[3] = __float_as_uint(w[3]);
        }
        __syncwarp();
        if (have) {
#pragma unroll
          for (int d = 1; d < N; ++d) l128_put(gather((me + d) % N) + line * 128 + 16 * k, w4);
        }
      } else {
        uint32_t x[4];
        if (!l128_wait(rx_me + ((uint64_t)parity * (N * a.sl + agl) + (uint64_t)N * a.sl) * 4 + line * 128 + 16 * k,
                       have, epoch, lane, x, a.st)) {
          failed = true;
          break;
        }
        if (!cnt) continue;
        float w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = __uint_as_float(x[i]);
        l128_st(wbase + e0, cnt, nv, w);
      }
    }
  }
  retire(a.queue);
}

// ============================================================== TREE (paper)
// Up: chunk c: acc = own + child_0 + child_1 + ... (children ascending, each the
// child's subtree sum), then to the parent's rx slot, or on rank 0 the update
// and the first hop of the broadcast.
template <class T>
__global__ void __launch_bounds__(kThreads) k_tree_up(XArgs a) {
  constexpr int W = VecT<T>::W;
  const uint32_t epoch = a.iter ? *a.iter + 1 : a.epoch;
  const int parity = a.iter ? (int)(*a.iter & 1) : a.parity;

  __shared__ uint32_t s_item;
  __shared__ uint32_t* s_flags[PGX_MAX_RANKS];
  const int me = a.rank;
  const int nc = tree_num_children(me, a.world);
  const int parent = tree_parent(me);
  const int myslot = me ? tree_slot_in_parent(me) : 0;
  while (true) {
    uint32_t c = claim(a.queue, &s_item) + a.item_begin;
    if (c >= a.item_end) break;
    uint64_t lo = (uint64_t)c * a.CH, hi = min(lo + a.CH, a.S);
    if (threadIdx.x < (unsigned)nc) s_flags[threadIdx.x] = a.rxflags[me] + (uint64_t)threadIdx.x * a.C + c;
    __syncthreads();
    cta_wait_flags(s_flags, nc, epoch, a.st);
    const T* rxb = static_cast<const T*>(a.rx[me]) + (uint64_t)parity * a.K * a.sl;
    uint64_t nvec = (hi - lo + W - 1) / W;
    const T* gs = slab_grad<T>(a.g, lo, hi);
    for (uint64_t q = threadIdx.x; q < nvec; q += blockDim.x) {
      uint64_t e = lo + q * W;
      int cnt = (int)min((uint64_t)W, hi - e);
      T acc[W];
      grad_vec_slab<T>(gs, a.g, lo, e, cnt, acc);
      for (int s = 0; s < nc; ++s) {
        T x[W];
        ld_vec<T>(rxb + (uint64_t)s * a.sl + e, cnt, x);
#pragma unroll
        for (int k = 0; k < W; ++k) {
          if constexpr (sizeof(T) == 8)
            acc[k] = __dadd_rn(acc[k], x[k]);
          else
            acc[k] = __fadd_rn(acc[k], x[k]);
        }
      }
      if (me == 0) {
        T* wp = static_cast<T*>(a.model[0]) + e;
        T w[W];
        ld_vec<T>(wp, cnt, w);
        update_vec<T>(w, acc, a.v ? a.v + e : nullptr, cnt, a);
        st_vec<T>(wp, cnt, w);
        for (int s = 0; s < nc; ++s) st_vec<T>(static_cast<T*>(a.model[tree_child(0, s)]) + e, cnt, w);
      } else {
        T* dst = static_cast<T*>(a.rx[parent]) + ((uint64_t)(parity * a.K + myslot) * a.sl + e);
        st_vec<T>(dst, cnt, acc);
      }
    }
    __syncthreads();
    if (me == 0) {
      if (threadIdx.x < (unsigned)nc) {
        int child = tree_child(0, threadIdx.x);
        fence_acq_rel_sys();
        st_release_sys(a.mflags[child] + a.dflag + c, epoch);
        red_release_sys_add(a.mflags[child] + a.layer, 1u);
      }
    } else if (threadIdx.x == 0) {
      fence_acq_rel_sys();
      st_release_sys(a.rxflags[parent] + (uint64_t)myslot * a.C + c, epoch);
    }
  }
  retire(a.queue);
}

// Down (inner ranks): forward each arrived model chunk to the broadcast children.
template <class T>
__global__ void __launch_bounds__(kThreads) k_tree_down(XArgs a) {
  constexpr int W = VecT<T>::W;
  const uint32_t epoch = a.iter ? *a.iter + 1 : a.epoch;
  __shared__ uint32_t s_item;
  __shared__ uint32_t* s_flags[1];
  const int me = a.rank;
  const int nc = tree_num_children(me, a.world);
  while (true) {
    uint32_t c = claim(a.queue, &s_item) + a.item_begin;
    if (c >= a.item_end) break;
    uint64_t lo = (uint64_t)c * a.CH, hi = min(lo + a.CH, a.S);
    if (threadIdx.x == 0) s_flags[0] = a.mflags[me] + a.dflag + c;
    __syncthreads();
    cta_wait_flags(s_flags, 1, epoch, a.st);
    uint64_t nvec = (hi - lo + W - 1) / W;
    const T* src = static_cast<const T*>(a.model[me]);
    for (uint64_t q = threadIdx.x; q < nvec; q += blockDim.x) {
      uint64_t e = lo + q * W;
      int cnt = (int)min((uint64_t)W, hi - e);
      T w[W];
      ld_vec<T>(src + e, cnt, w);
      for (int s = 0; s < nc; ++s) st_vec<T>(static_cast<T*>(a.model[tree_child(me, s)]) + e, cnt, w);
    }
    __syncthreads();
    if (threadIdx.x < (unsigned)nc) {
      int child = tree_child(me, threadIdx.x);
      fence_acq_rel_sys();
      st_release_sys(a.mflags[child] + a.dflag + c, epoch);
      red_release_sys_add(a.mflags[child] + a.layer, 1u);
    }
  }
  retire(a.queue);
}

// ============================================================== NVLS
// NVLink SHARP: the switch reduces and multicasts.  Every rank publishes its layer
// gradient into its slice of a multicast object; the owner of shard j reads the SUM of
// all ranks' slices with one multimem.ld_reduce per vector (the reduction happens in the
// NVSwitch), applies the fused update, and writes the new weights to every GPU with one
// multimem.st.  Per GPU ~S bytes leave over NVLink instead of 2(N-1)/N*S.  The switch's
// summation order is not the binomial order, so this variant is tolerance-only (fast32).
struct NvArgs {
  Pieces g;
  float* uc_model;            // layer base, local mapping
  float* uc_grad;             // layer base, local mapping
  uint64_t mc_model, mc_grad; // layer base, multicast mapping
  uint32_t* uc_ready;         // this layer's ready[owner][chunk] counters (local view)
  uint64_t mc_ready, mc_arrive;
  float* v;
  uint32_t* queue;
  uint64_t S, sl, CH;
  uint32_t C;                 // chunks per shard
  uint32_t pub_items, items, epoch;
  const uint32_t* iter;
  int rank, world;
  double lr;
  float scale, mu, wd;
  Status st;
};

__device__ __forceinline__ float4 mm_ld_reduce4(uint64_t addr) {
  float4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(addr)
               : "memory");
  return r;
}
__device__ __forceinline__ float mm_ld_reduce1(uint64_t addr) {
  float r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(r) : "l"(addr) : "memory");
  return r;
}
__device__ __forceinline__ void mm_st4(uint64_t addr, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mm_st1(uint64_t addr, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void mm_red_release_add(uint64_t addr, uint32_t v) {
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ float fast32_update(float w, float g, float& v, const NvArgs& a) {
  float gg = __fadd_rn(__fmul_rn(a.scale, g), __fmul_rn(a.wd, w));
  float vv = __fadd_rn(__fmul_rn(a.mu, v), __fmul_rn((float)a.lr, gg));
  v = vv;
  return __fsub_rn(w, vv);
}

// Items: publish (chunk c of owner j's shard, c-major so early chunks of every shard go
// first) -> ready[j][c] += 1 on every GPU (multimem.red); owner chunk c of my shard waits
// ready[me][c] >= N*epoch, so publish and reduction pipeline chunk by chunk.
#ifndef NVLS_U
#define NVLS_U 2  // multimem.ld_reduce in flight per thread (r1v: 4 -> 882 us, r1w: 8 -> 965 us @ 256 MB, N=4)
#endif
#ifndef NVLS_MINB
#define NVLS_MINB 2
#endif
__global__ void __launch_bounds__(kThreads, NVLS_MINB) k_nvls(NvArgs a) {
  __shared__ uint32_t s_item;
  const uint32_t epoch = a.iter ? *a.iter + 1 : a.epoch;
  const int me = a.rank, N = a.world;
  while (true) {
    uint32_t it = claim(a.queue, &s_item);
    if (it >= a.items) break;
    if (it < a.pub_items) {
      // ---- publish chunk c of owner j's shard into my slice of the multicast object
      uint32_t c = it / (uint32_t)N;
      int j = it % N;
      uint64_t lo = j * a.sl + (uint64_t)c * a.CH;
      uint64_t hi = min(min(lo + a.CH, (uint64_t)(j + 1) * a.sl), a.S);
      if (lo >= hi) continue;
      constexpr int UP = 4;
      for (uint64_t e0 = lo + threadIdx.x * 4; e0 < hi; e0 += (uint64_t)UP * blockDim.x * 4) {
        float buf[UP][4];
        int cnt[UP];
#pragma unroll
        for (int u = 0; u < UP; ++u) {
          uint64_t e = e0 + (uint64_t)u * blockDim.x * 4;
          cnt[u] = e < hi ? (int)min((uint64_t)4, hi - e) : 0;
          if (cnt[u] > 0) grad_vec<float>(a.g, e, cnt[u], buf[u]);
        }
#pragma unroll
        for (int u = 0; u < UP; ++u)
          if (cnt[u] > 0) st_vec<float>(a.uc_grad + e0 + (uint64_t)u * blockDim.x * 4, cnt[u], buf[u]);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        fence_acq_rel_sys();
        mm_red_release_add(a.mc_ready + ((uint64_t)j * a.C + c) * 4, 1u);
      }
    } else {
      // ---- owner chunk: switch-reduced gradient, fused update, multicast store of the weights
      uint32_t c = it - a.pub_items;
      uint64_t lo = me * a.sl + (uint64_t)c * a.CH;
      uint64_t hi = min(min(lo + a.CH, (uint64_t)(me + 1) * a.sl), a.S);
      if (lo >= hi) continue;
      if (threadIdx.x == 0) wait_geq(a.uc_ready + (uint64_t)me * a.C + c, epoch * (uint32_t)N, a.st);
      __syncthreads();
      constexpr int U = NVLS_U;
      uint64_t body = lo + (hi - lo) / 4 * 4;
      for (uint64_t e0 = lo + threadIdx.x * 4; e0 < body; e0 += (uint64_t)U * blockDim.x * 4) {
        float4 g[U], w[U], v[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          uint64_t e = e0 + (uint64_t)u * blockDim.x * 4;
          ok[u] = e < body;
          if (ok[u]) g[u] = mm_ld_reduce4(a.mc_grad + e * 4);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          uint64_t e = e0 + (uint64_t)u * blockDim.x * 4;
          if (ok[u]) {
            w[u] = __ldcg(reinterpret_cast<const float4*>(a.uc_model + e));
            v[u] = *reinterpret_cast<const float4*>(a.v + e);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (!ok[u]) continue;
          uint64_t e = e0 + (uint64_t)u * blockDim.x * 4;
          w[u].x = fast32_update(w[u].x, g[u].x, v[u].x, a);
          w[u].y = fast32_update(w[u].y, g[u].y, v[u].y, a);
          w[u].z = fast32_update(w[u].z, g[u].z, v[u].z, a);
          w[u].w = fast32_update(w[u].w, g[u].w, v[u].w, a);
          *reinterpret_cast<float4*>(a.v + e) = v[u];
          mm_st4(a.mc_model + e * 4, w[u]);
        }
      }
      for (uint64_t k = body + threadIdx.x; k < hi; k += blockDim.x) {  // ragged end of the layer
        float g = mm_ld_reduce1(a.mc_grad + k * 4);
        float w = __ldcg(a.uc_model + k), v = a.v[k];
        w = fast32_update(w, g, v, a);
        a.v[k] = v;
        mm_st1(a.mc_model + k * 4, w);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        fence_acq_rel_sys();
        mm_red_release_add(a.mc_arrive, 1u);
      }
    }
  }
  retire(a.queue);
}

// Gate: the stream proceeds once `want` chunk arrivals were counted.
// want = *iter * per_epoch (graph mode: gate for the iteration before the current one)
__global__ void k_gate(const uint32_t* counter, uint32_t want, const uint32_t* iter, uint32_t add, uint32_t per_epoch,
                       Status st) {
  if (threadIdx.x == 0) wait_geq(counter, iter ? (*iter + add) * per_epoch : want, st);
}

// Copy-engine two-shot (TWOSHOT_CE): the gradient shards and the updated shards
// travel as peer DMA copies (the GPU's copy engines are the RDMA engine of a
// GPI-2 write_notify: one-sided and without compute resources); each transfer is
// followed by a fenced stream write of the notification.  SMs only run the local
// fold + update below and these bounded flag waits.
struct FlagSet {
  const uint32_t* f[PGX_MAX_RANKS];
  int n;
};
__global__ void k_wait_flags(FlagSet fs, uint32_t want, const uint32_t* iter, uint32_t add, Status st) {
  if (threadIdx.x < (unsigned)fs.n) wait_geq(fs.f[threadIdx.x], iter ? *iter + add : want, st);
}

// Raise peers' flags after this stream's preceding copies completed (stream order):
// system fence, then release stores of the epoch.
struct FlagOut {
  uint32_t* f[PGX_MAX_RANKS];
  int n;
};
__global__ void k_signal(FlagOut fo, uint32_t value, const uint32_t* iter) {
  if (threadIdx.x < (unsigned)fo.n) {
    fence_acq_rel_sys();
    st_release_sys(fo.f[threadIdx.x], iter ? *iter + 1 : value);
  }
}

// Raise every chunk flag of each peer's slot (after this stream's copies, stream order).
struct FlagRanges {
  uint32_t* f[PGX_MAX_RANKS];
  uint32_t n[PGX_MAX_RANKS];
  int k;
};
__global__ void k_signal_range(FlagRanges fr, uint32_t value, const uint32_t* iter) {
  const uint32_t v = iter ? *iter + 1 : value;
  if (threadIdx.x == 0) fence_acq_rel_sys();
  __syncthreads();
  for (int q = 0; q < fr.k; ++q)
    for (uint32_t c = threadIdx.x; c < fr.n[q]; c += blockDim.x) st_release_sys(fr.f[q] + c, v);
}

__global__ void k_tick(uint32_t* iter) { *iter += 1; }

// Whole-model gate: every (flag, multiplier) entry of every layer in one launch;
// entry i waits until *flag >= it * mult, it = the awaited iteration + 1.
struct GateEntry {
  const uint32_t* flag;
  uint32_t mult;
};
__global__ void k_gate_all(const GateEntry* __restrict__ ents, int n, uint32_t it_host, const uint32_t* iter,
                           uint32_t add, Status st) {
  const uint32_t it = iter ? *iter + add : it_host;
  for (int i = threadIdx.x; i < n; i += blockDim.x) wait_geq(ents[i].flag, it * ents[i].mult, st);
}

template <int N, class T>
__global__ void __launch_bounds__(kThreads) k_owner_local(XArgs a) {
  constexpr int W = VecT<T>::W;
  constexpr int U = N <= 4 ? 2 : 1;
  const int me = a.rank;
  const uint64_t base = min((uint64_t)me * a.sl, a.S);
  uint64_t lo = base, hi = min((uint64_t)(me + 1) * a.sl, a.S);
  if (a.ohi) {
    lo = a.olo;
    hi = a.ohi;
  }
  if (lo >= hi) return;
  // receive slots are indexed from the shard start; owner_vectors indexes them by q
  const T* rxb = static_cast<const T*>(a.rx[me]) + (uint64_t)a.parity * a.K * a.sl + (lo - base);
  const uint64_t nvec = (hi - lo + W - 1) / W, span = (uint64_t)U * blockDim.x;
  const T* gs = slab_grad<T>(a.g, lo, hi);
  for (uint64_t blk = blockIdx.x; blk * span < nvec; blk += gridDim.x)
    owner_vectors<N, T, U, false>(a, rxb, lo, hi, blk * span + threadIdx.x, nvec, nullptr, gs);
}

constexpr int kCepCtas = 48;  // TWOSHOT_CEP owner grid default
constexpr int kCeTmaCtas = 32;  // TWOSHOT_CE + PGX_XF_CE_TMA_OWNER owner grid default
constexpr int kLeanThreads = 128;  // PGX_XF_LEAN_CAPPED: threads per CTA of capped LL / L128 layers
constexpr uint64_t kAutoChunkMax = 65536;  // elements
constexpr uint64_t kN1Chunk = 4096;        // elements per item of a one-rank (update-only) launch

// TWOSHOT_CE owner fold on a capped grid (PGX_XF_CE_TMA_OWNER): the part [olo, ohi) split
// into one contiguous 16-byte-aligned slab per CTA, each folded through owner_tma (TMA
// loads of the N partials + w + v into the ring, fold + update from shared memory, bulk
// stores of w / v).  On the full grid the fold of k_owner_local saturates HBM with every SM
// waiting on it; a TMA-fed CTA moves ~1.5x more bytes per SM (ncu r6a), so a few dozen
// CTAs do the same fold in far fewer SM-cycles while the copy engines move the shards.
template <int N, class T, int MODE>
__global__ void __launch_bounds__(BulkGeo<false>::kThreads, 1) k_owner_tma(XArgs a) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ uint64_t obars[16];
  if (threadIdx.x == 0) {
    for (int k = 0; k < 8; ++k) mbar_init(&obars[k], 1);
    for (int k = 8; k < 16; ++k) mbar_init(&obars[k], blockDim.x / 32 - 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int me = a.rank;
  const uint64_t base = min((uint64_t)me * a.sl, a.S);
  uint64_t lo = base, hi = min((uint64_t)(me + 1) * a.sl, a.S);
  if (a.ohi) {
    lo = a.olo;
    hi = a.ohi;
  }
  if (lo >= hi) return;
  const uint64_t per = ((hi - lo + gridDim.x - 1) / gridDim.x + 3) / 4 * 4;
  const uint64_t slo = lo + (uint64_t)blockIdx.x * per, shi = min(hi, slo + per);
  if (slo >= shi) return;
  const T* rx0 = static_cast<const T*>(a.rx[me]) + (uint64_t)a.parity * a.K * a.sl - base;
  const T* gs = slab_grad<T>(a.g, slo, shi);
  uint32_t ouse = 0;
  const uint64_t done = owner_tma<N, T, MODE, false, false>(a, rx0, gs, slo, shi, ring, obars, ouse);
  if (threadIdx.x == 0) tma_wait_all();  // w / v stores complete before the kernel ends
  // the ragged end (< 16 bytes) or an ineligible slab: element by element, same arithmetic
  constexpr bool fast = MODE == PGX_MODE_FAST32;
  constexpr bool upd = MODE != PGX_MODE_SUM32;
  T* wme = static_cast<T*>(a.model[me]);
  for (uint64_t e = done + threadIdx.x; e < shi; e += blockDim.x) {
    T col[N];
#pragma unroll
    for (int s = 0; s < N; ++s) col[s] = (s == me) ? grad_elem<T>(a.g, e) : __ldcg(rx0 + (uint64_t)s * a.sl + e);
    T gsum;
    if constexpr (sizeof(T) == 8)
      gsum = tree_sum<N>(col, AddF64{});
    else
      gsum = tree_sum<N>(col, AddF32{});
    float vv = fast ? a.v[e] : 0.f;
    wme[e] = bulk_update<MODE, T>(upd ? wme[e] : T(0), gsum, vv, a.lr, a.scale, a.mu, a.wd);
    if (fast) a.v[e] = vv;
  }
}

struct LayerPlan {
  uint64_t S = 0;
  int variant = 0;
  uint64_t sl = 0;       // shard elems (twoshot) or S (tree)
  uint32_t C = 0;        // chunks per shard / per layer
  uint64_t CH = 0;       // chunk elems (notification granularity) of this layer
  int K = 0;             // rx slots per parity
  uint64_t model_off = 0, rx_off = 0;
  uint64_t rxflag_off = 0;
  uint32_t dflag = 0;    // tree down flags index (in mflags)
  uint32_t push_items = 0, items = 0, down_items = 0;
  uint32_t expected = 0; // remote chunk arrivals per epoch
  uint64_t CHo = 0;      // TWOSHOT_L128: lines per owner item (finer than the push items)
  uint32_t Co = 0;       // TWOSHOT_L128: owner items
  int grid = 0, down_grid = 0;
  uint64_t nvlink_bytes = 0, hbm_bytes = 0;
  bool lean = false;     // LL / L128 layer with a CTA cap under PGX_XF_LEAN_CAPPED: 128-thread CTAs
};

}  // namespace

// An event plus where it was last recorded: eagerly (cap = 0) or inside the stream
// capture with id `cap`.  Waits only bind to records of the same capture (or eager
// records from eager streams) — a captured graph may not depend on uncaptured work.
struct XEvent {
  cudaEvent_t e = nullptr;
  unsigned long long cap = 0;
  cudaStream_t rec = nullptr;
  bool valid = false;
};

static unsigned long long capture_id(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  if (cudaStreamGetCaptureInfo(s, &st, &id) != cudaSuccess) return 0;
  return st == cudaStreamCaptureStatusActive ? id : 0;
}
static cudaError_t xrecord(XEvent& ev, cudaStream_t s) {
  ev.cap = capture_id(s);
  ev.rec = s;
  ev.valid = true;
  return cudaEventRecord(ev.e, s);
}
// Wait when both sides are eager, when both belong to the same capture, or to fork an
// eager stream into a live capture (the event was recorded by a stream still capturing).
static cudaError_t xwait(cudaStream_t s, const XEvent& ev) {
  if (!ev.valid) return cudaSuccess;
  const unsigned long long c = capture_id(s);
  bool wait = ev.cap == 0 ? c == 0 : (c == ev.cap || (c == 0 && capture_id(ev.rec) == ev.cap));
  return wait ? cudaStreamWaitEvent(s, ev.e, 0) : cudaSuccess;
}

struct pgx_xchg {
  pgx_world* w = nullptr;
  pgx_xchg_config cfg{};
  int rank = 0, world = 1, dev = 0, esz = 4;
  std::vector<LayerPlan> L;
  uint32_t seg_model = 0, seg_rx = 0;
  void* model = nullptr;
  uint32_t* mflags = nullptr;
  void* rx = nullptr;
  uint32_t* rxflags = nullptr;
  float* v = nullptr;
  uint32_t* queues = nullptr;  // 4 per layer
  void* peer_model[PGX_MAX_RANKS] = {};
  uint32_t* peer_mflags[PGX_MAX_RANKS] = {};
  void* peer_rx[PGX_MAX_RANKS] = {};
  uint32_t* peer_rxflags[PGX_MAX_RANKS] = {};
  bool connected = false;
  uint64_t launches = 0;
  cudaStream_t down = nullptr;
  cudaStream_t ce_rs = nullptr, ce_own = nullptr;  // TWOSHOT_CE: push copies / owner side
  cudaStream_t ce_ag = nullptr, ce_rs2 = nullptr;  // TWOSHOT_CE: all-gather copies / 2nd push stream
  int ce_parts = 4, ce_rs_streams = 1;             // owner pipelining depth, push streams (measured, r1l)
  bool ce_rs_parts = false;                        // push signals per owner part (signals on ce_rs2)
  bool tma = false;  // TWOSHOT: push / all-gather as TMA bulk copies (PGX_TMA=1; slower fused at N=4, profiles/r1r)
  bool bulk_ce_rs = false;  // TWOSHOT_BULK: reduce-scatter by the copy engines (PGX_XF_BULK_CE_RS)
  bool ce_tma_owner = false;  // TWOSHOT_CE: owner fold by k_owner_tma on a capped grid (PGX_XF_CE_TMA_OWNER)
  bool oneshot_small_chunks = false;  // PGX_ONESHOT_SMALL_CHUNKS=1: measured slower (profiles/r3v)
  bool auto_chunk_tree = false, auto_chunk_nvls = true;  // size-scaled chunks: NVLS yes, tree no (its pipeline
                                                        // fill grows with the chunk; profiles/r3r)
  bool own_streams = true;                         // false once the caller supplied them
  std::vector<XEvent> done;
  std::vector<XEvent> ready;                       // gradient ready on the launch stream
  std::vector<XEvent> rs_done, down_done;          // side-stream completion (joins for graph capture)
  std::vector<XEvent> rs2_done;
  std::vector<std::vector<XEvent>> part_ev;        // TWOSHOT_CE owner parts ready for their all-gather
  std::vector<std::vector<XEvent>> rs_part_ev;     // TWOSHOT_CE push parts copied (per-part signals)
  uint32_t* iter_dev = nullptr;                    // device iteration counter (graph mode)
  unsigned long long* trace = nullptr;             // debug timeline buffer (pgx_xchg_set_trace)
  bool device_iter = false;
  uint32_t ownerflag_base = 0;                     // mflags index of [layer][owner] arrival flags
  GateEntry* gate_table = nullptr;                 // device: every layer's arrival flags
  int gate_entries = 0;
  struct Nvls {                                    // NVLS: one multicast object [model | grad | flags]
    bool on = false;
    size_t size = 0;
    CUmemGenericAllocationHandle mc = 0, mem = 0;
    CUdeviceptr uc = 0, mcp = 0;                   // unicast (local) and multicast mappings
    uint64_t grad_off = 0, flag_off = 0;           // bytes
    std::vector<uint64_t> fl;                      // per layer: [arrive | ready[N][C]] offset in the flags
  } nv;
};

namespace {

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

int sm_count(int dev) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

XArgs base_args(pgx_xchg* x, int l, uint32_t iteration) {
  const LayerPlan& P = x->L[l];
  XArgs a;
  memset(&a, 0, sizeof(a));
  for (int r = 0; r < x->world; ++r) {
    a.model[r] = static_cast<uint8_t*>(x->peer_model[r]) + P.model_off * x->esz;
    a.mflags[r] = x->peer_mflags[r];
    a.rx[r] = static_cast<uint8_t*>(x->peer_rx[r]) + P.rx_off * x->esz;
    a.rxflags[r] = x->peer_rxflags[r] + P.rxflag_off;
  }
  a.v = x->v ? x->v + P.model_off : nullptr;
  a.S = P.S;
  a.sl = P.sl;
  a.CH = P.CH;
  a.C = P.C;
  a.K = P.K;
  a.dflag = P.dflag;
  a.layer = l;
  a.epoch = iteration + 1;  // notification value = iteration + 1 (runtime.py:205)
  a.rank = x->rank;
  a.world = x->world;
  a.parity = iteration & 1;
  a.push_items = P.push_items;
  a.items = P.items;
  a.CHo = P.CHo;
  a.Co = P.Co;
  a.lr = x->cfg.lr;
  a.scale = x->cfg.scale;
  a.mu = x->cfg.momentum;
  a.wd = x->cfg.weight_decay;
  a.mode = x->cfg.mode;
  a.st = world_status(x->w);
  a.iter = x->device_iter ? x->iter_dev : nullptr;
  a.trace = x->trace;
  a.bulk_lean = (x->cfg.flags & PGX_XF_BULK_LEAN) != 0;
  return a;
}

// Grid = min(requested, resident CTAs): CTAs beyond what fits only spin up to
// find the queue empty.
constexpr size_t kTmaSmem = (size_t)kTmaStages * kTmaStage + kTmaStages * sizeof(uint64_t);

template <int N, class T, bool kTma>
int resident_grid(int want, int dev) {
  static int cap[PGX_MAX_RANKS] = {};  // per instantiation and device
  if (!cap[dev]) {
    if (kTma) cudaFuncSetAttribute(k_twoshot<N, T, kTma>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_twoshot<N, T, kTma>, kThreads, kTma ? kTmaSmem : 0);
    cap[dev] = std::max(1, per_sm) * sm_count(dev);
  }
  return std::max(1, std::min(want, cap[dev]));
}

template <class T>
void launch_twoshot(int N, bool tma, int want, int dev, cudaStream_t s, const XArgs& a) {
  switch (N) {
#define PGX_CASE(n)                                                                 \
  case n:                                                                           \
    if (n > 1 && tma) {                                                             \
      int g = resident_grid<n, T, true>(want, dev);                                 \
      k_twoshot<n, T, true><<<g, kThreads, kTmaSmem, s>>>(a);                       \
    } else {                                                                        \
      int g = resident_grid<n, T, false>(want, dev);                                \
      k_twoshot<n, T, false><<<g, kThreads, 0, s>>>(a);                             \
    }                                                                               \
    break;
    PGX_CASE(1) PGX_CASE(2) PGX_CASE(3) PGX_CASE(4) PGX_CASE(5) PGX_CASE(6) PGX_CASE(7) PGX_CASE(8)
#undef PGX_CASE
  }
}

template <int N, class T, int MODE, bool LEAN>
void launch_bulk_nml(int grid, int dev, cudaStream_t s, const XArgs& a) {
  using G = BulkGeo<LEAN>;
  static bool attr[64] = {};  // per device
  if (!attr[dev & 63]) {
    cudaFuncSetAttribute(k_twoshot_bulk<N, T, MODE, LEAN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::kSmem);
    attr[dev & 63] = true;
  }
  k_twoshot_bulk<N, T, MODE, LEAN><<<grid, G::kThreads, G::kSmem, s>>>(a);
}

template <int N, class T, int MODE>
void launch_bulk_nm(int grid, int dev, cudaStream_t s, const XArgs& a) {
  if (a.bulk_lean)
    launch_bulk_nml<N, T, MODE, true>(grid, dev, s, a);
  else
    launch_bulk_nml<N, T, MODE, false>(grid, dev, s, a);
}

template <int N>
void launch_bulk_n(int grid, int dev, cudaStream_t s, const XArgs& a) {
  switch (a.mode) {
    case PGX_MODE_REF64: launch_bulk_nm<N, double, PGX_MODE_REF64>(grid, dev, s, a); break;
    case PGX_MODE_REF32: launch_bulk_nm<N, float, PGX_MODE_REF32>(grid, dev, s, a); break;
    case PGX_MODE_SUM32: launch_bulk_nm<N, float, PGX_MODE_SUM32>(grid, dev, s, a); break;
    default: launch_bulk_nm<N, float, PGX_MODE_FAST32>(grid, dev, s, a); break;
  }
}

void launch_twoshot_bulk(int N, int grid, int dev, cudaStream_t s, const XArgs& a) {
  switch (N) {
#define PGX_CASE(n) \
  case n: launch_bulk_n<n>(grid, dev, s, a); break;
    PGX_CASE(1) PGX_CASE(2) PGX_CASE(3) PGX_CASE(4) PGX_CASE(5) PGX_CASE(6) PGX_CASE(7) PGX_CASE(8)
#undef PGX_CASE
  }
}

template <int N, class T>
int oneshot_grid(int want, int dev) {
  static int cap[PGX_MAX_RANKS] = {};
  if (!cap[dev]) {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_oneshot<N, T>, kThreads, 0);
    cap[dev] = std::max(1, per_sm) * sm_count(dev);
  }
  return std::max(1, std::min(want, cap[dev]));
}

template <class T>
void launch_oneshot(int N, int want, int dev, cudaStream_t s, const XArgs& a) {
  switch (N) {
#define PGX_CASE(n)                                                        \
  case n:                                                                  \
    k_oneshot<n, T><<<oneshot_grid<n, T>(want, dev), kThreads, 0, s>>>(a); \
    break;
    PGX_CASE(1) PGX_CASE(2) PGX_CASE(3) PGX_CASE(4) PGX_CASE(5) PGX_CASE(6) PGX_CASE(7) PGX_CASE(8)
#undef PGX_CASE
  }
}

template <int N>
int oneshot_ll_grid(int want, int dev) {
  static int cap[PGX_MAX_RANKS] = {};
  if (!cap[dev]) {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_oneshot_ll<N>, kThreads, 0);
    cap[dev] = std::max(1, per_sm) * sm_count(dev);
  }
  return std::max(1, std::min(want, cap[dev]));
}

template <int N>
int oneshot_l128_grid(int want, int dev) {
  static int cap[PGX_MAX_RANKS] = {};
  if (!cap[dev]) {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_oneshot_l128<N>, kThreads, 0);
    cap[dev] = std::max(1, per_sm) * sm_count(dev);
  }
  return std::max(1, std::min(want, cap[dev]));
}

void launch_oneshot_l128(int N, int want, int dev, cudaStream_t s, const XArgs& a) {
  switch (N) {
#define PGX_CASE(n)                                                                \
  case n:                                                                          \
    k_oneshot_l128<n><<<oneshot_l128_grid<n>(want, dev), kThreads, 0, s>>>(a);   \
    break;
    PGX_CASE(1) PGX_CASE(2) PGX_CASE(3) PGX_CASE(4) PGX_CASE(5) PGX_CASE(6) PGX_CASE(7) PGX_CASE(8)
#undef PGX_CASE
  }
}

template <int N>
int twoshot_l128_grid(int want, int dev) {
  static int cap[PGX_MAX_RANKS] = {};
  if (!cap[dev]) {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_twoshot_l128<N>, kThreads, 0);
    cap[dev] = std::max(1, per_sm) * sm_count(dev);
  }
  return std::max(1, std::min(want, cap[dev]));
}

void launch_twoshot_l128(int N, int want, int dev, cudaStream_t s, const XArgs& a, int threads = kThreads) {
  switch (N) {
#define PGX_CASE(n)                                                                \
  case n:                                                                          \
    k_twoshot_l128<n><<<twoshot_l128_grid<n>(want, dev), threads, 0, s>>>(a);     \
    break;
    PGX_CASE(1) PGX_CASE(2) PGX_CASE(3) PGX_CASE(4) PGX_CASE(5) PGX_CASE(6) PGX_CASE(7) PGX_CASE(8)
#undef PGX_CASE
  }
}

void launch_oneshot_ll(int N, int want, int dev, cudaStream_t s, const XArgs& a, int threads = kThreads) {
  switch (N) {
#define PGX_CASE(n)                                                            \
  case n:                                                                      \
    k_oneshot_ll<n><<<oneshot_ll_grid<n>(want, dev), threads, 0, s>>>(a);   \
    break;
    PGX_CASE(1) PGX_CASE(2) PGX_CASE(3) PGX_CASE(4) PGX_CASE(5) PGX_CASE(6) PGX_CASE(7) PGX_CASE(8)
#undef PGX_CASE
  }
}

template <int N, class T, int MODE>
void launch_owner_tma_nm(int grid, int dev, cudaStream_t s, const XArgs& a) {
  using G = BulkGeo<false>;
  static bool attr[64] = {};  // per device
  if (!attr[dev & 63]) {
    cudaFuncSetAttribute(k_owner_tma<N, T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::kSmem);
    attr[dev & 63] = true;
  }
  k_owner_tma<N, T, MODE><<<grid, G::kThreads, G::kSmem, s>>>(a);
}

template <int N>
void launch_owner_tma_n(int mode, int grid, int dev, cudaStream_t s, const XArgs& a) {
  switch (mode) {
    case PGX_MODE_REF64: launch_owner_tma_nm<N, double, PGX_MODE_REF64>(grid, dev, s, a); break;
    case PGX_MODE_REF32: launch_owner_tma_nm<N, float, PGX_MODE_REF32>(grid, dev, s, a); break;
    case PGX_MODE_SUM32: launch_owner_tma_nm<N, float, PGX_MODE_SUM32>(grid, dev, s, a); break;
    default: launch_owner_tma_nm<N, float, PGX_MODE_FAST32>(grid, dev, s, a); break;
  }
}

void launch_owner_tma(int N, int mode, int grid, int dev, cudaStream_t s, const XArgs& a) {
  switch (N) {
#define PGX_CASE(n) \
  case n: launch_owner_tma_n<n>(mode, grid, dev, s, a); break;
    PGX_CASE(1) PGX_CASE(2) PGX_CASE(3) PGX_CASE(4) PGX_CASE(5) PGX_CASE(6) PGX_CASE(7) PGX_CASE(8)
#undef PGX_CASE
  }
}

template <class T>
void launch_owner_local(int N, int grid, cudaStream_t s, const XArgs& a) {
  switch (N) {
#define PGX_CASE(n) \
  case n: k_owner_local<n, T><<<grid, kThreads, 0, s>>>(a); break;
    PGX_CASE(1) PGX_CASE(2) PGX_CASE(3) PGX_CASE(4) PGX_CASE(5) PGX_CASE(6) PGX_CASE(7) PGX_CASE(8)
#undef PGX_CASE
  }
}

}  // namespace


// ---------------------------------------------------------------- NVLS setup
// Driver entry points through the runtime (libpgx.so does not link libcuda).
template <class F>
static F drv(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}
#define PGX_DRV(fn) static auto p_##fn = drv<decltype(&fn)>(#fn)
#define PGX_CU(call)                                                                      \
  do {                                                                                    \
    CUresult r__ = (call);                                                                \
    if (r__ != CUDA_SUCCESS) return fail(PGX_E_CUDA, "%s failed (CUresult %d)", #call, (int)r__); \
  } while (0)

static bool nvls_layers(const pgx_xchg* x) {
  for (auto& P : x->L)
    if (P.variant == PGX_VARIANT_NVLS) return true;
  return false;
}

static size_t nvls_size(pgx_xchg* x, size_t gran) {
  uint64_t model_bytes = 0;
  for (auto& P : x->L) model_bytes = std::max<uint64_t>(model_bytes, (P.model_off + P.S) * 4);
  model_bytes = (model_bytes + 255) / 256 * 256;
  x->nv.grad_off = model_bytes;
  x->nv.flag_off = 2 * model_bytes;
  x->nv.fl.clear();
  uint64_t f = 0;
  for (auto& P : x->L) {  // [arrive counter (128 B) | ready[N][C] u32]
    x->nv.fl.push_back(f);
    f += 128 + ((uint64_t)x->world * P.C * 4 + 127) / 128 * 128;
  }
  size_t total = 2 * model_bytes + f;
  return (total + gran - 1) / gran * gran;
}

static int nvls_granularity(pgx_xchg* x, size_t* gran) {
  PGX_DRV(cuMulticastGetGranularity);
  PGX_DRV(cuMemGetAllocationGranularity);
  if (!p_cuMulticastGetGranularity || !p_cuMemGetAllocationGranularity)
    return fail(PGX_E_CUDA, "multicast driver entry points unavailable");
  CUmulticastObjectProp mp{};
  mp.numDevices = x->world;
  mp.size = 1 << 21;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g1 = 0, g2 = 0;
  PGX_CU(p_cuMulticastGetGranularity(&g1, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = x->dev;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  PGX_CU(p_cuMemGetAllocationGranularity(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  *gran = std::max(g1, g2);
  return PGX_OK;
}

extern "C" int pgx_xchg_nvls_export(pgx_xchg* x, int* fd_out) {
  *fd_out = -1;
  if (!nvls_layers(x)) return fail(PGX_E_CONFIG, "no NVLS layers in this exchange");
  if (x->cfg.mode != PGX_MODE_FAST32) return fail(PGX_E_CONFIG, "NVLS reduces in the switch: fast32 only");
  size_t gran = 0;
  int rc = nvls_granularity(x, &gran);
  if (rc) return rc;
  x->nv.size = nvls_size(x, gran);
  if (x->rank != 0) return PGX_OK;
  PGX_DRV(cuMulticastCreate);
  PGX_DRV(cuMemExportToShareableHandle);
  if (!p_cuMulticastCreate || !p_cuMemExportToShareableHandle) return fail(PGX_E_CUDA, "multicast entry points");
  CUmulticastObjectProp mp{};
  mp.numDevices = x->world;
  mp.size = x->nv.size;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  PGX_CU(p_cuMulticastCreate(&x->nv.mc, &mp));
  int fd = -1;
  PGX_CU(p_cuMemExportToShareableHandle(&fd, x->nv.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  *fd_out = fd;
  return PGX_OK;
}

extern "C" int pgx_xchg_nvls_import(pgx_xchg* x, int fd) {
  PGX_DRV(cuMemImportFromShareableHandle);
  PGX_DRV(cuMulticastAddDevice);
  PGX_DRV(cuDeviceGet);
  if (!p_cuMemImportFromShareableHandle || !p_cuMulticastAddDevice || !p_cuDeviceGet)
    return fail(PGX_E_CUDA, "multicast entry points");
  if (x->rank != 0) {
    if (fd < 0) return fail(PGX_E_CONFIG, "no multicast handle received");
    PGX_CU(p_cuMemImportFromShareableHandle(&x->nv.mc, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
    close(fd);
  }
  CUdevice d;
  PGX_CU(p_cuDeviceGet(&d, x->dev));
  PGX_CU(p_cuMulticastAddDevice(x->nv.mc, d));
  return PGX_OK;
}

// After EVERY rank added its device: bind local memory, map unicast + multicast views,
// move the weights into the multicast-backed buffer (the model the framework aliases).
extern "C" int pgx_xchg_nvls_bind(pgx_xchg* x) {
  PGX_DRV(cuMemCreate);
  PGX_DRV(cuMulticastBindMem);
  PGX_DRV(cuMemAddressReserve);
  PGX_DRV(cuMemMap);
  PGX_DRV(cuMemSetAccess);
  if (!p_cuMemCreate || !p_cuMulticastBindMem || !p_cuMemAddressReserve || !p_cuMemMap || !p_cuMemSetAccess)
    return fail(PGX_E_CUDA, "multicast entry points");
  int prev;
  cudaGetDevice(&prev);
  cudaSetDevice(x->dev);
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = x->dev;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // multicast binding needs a shareable type
  PGX_CU(p_cuMemCreate(&x->nv.mem, x->nv.size, &ap, 0));
  {
    CUresult r = p_cuMulticastBindMem(x->nv.mc, 0, x->nv.mem, 0, x->nv.size, 0);
    if (r != CUDA_SUCCESS)
      return fail(PGX_E_CUDA, "cuMulticastBindMem failed (CUresult %d, size %zu)", (int)r, x->nv.size);
  }
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = x->dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  PGX_CU(p_cuMemAddressReserve(&x->nv.uc, x->nv.size, 0, 0, 0));
  PGX_CU(p_cuMemMap(x->nv.uc, x->nv.size, 0, x->nv.mem, 0));
  PGX_CU(p_cuMemSetAccess(x->nv.uc, x->nv.size, &acc, 1));
  PGX_CU(p_cuMemAddressReserve(&x->nv.mcp, x->nv.size, 0, 0, 0));
  PGX_CU(p_cuMemMap(x->nv.mcp, x->nv.size, 0, x->nv.mc, 0));
  PGX_CU(p_cuMemSetAccess(x->nv.mcp, x->nv.size, &acc, 1));
  PGX_CUDA(cudaMemset((void*)x->nv.uc, 0, x->nv.size));
  uint64_t model_bytes = x->nv.grad_off;
  PGX_CUDA(cudaMemcpy((void*)x->nv.uc, x->model, model_bytes, cudaMemcpyDeviceToDevice));
  x->model = (void*)x->nv.uc;
  x->nv.on = true;
  // gate table: arrival counters live in the multicast-backed flags now
  std::vector<GateEntry> ents;
  for (size_t l = 0; l < x->L.size(); ++l)
    ents.push_back({reinterpret_cast<uint32_t*>(x->nv.uc + x->nv.flag_off + x->nv.fl[l]), x->L[l].expected});
  PGX_CUDA(cudaMemcpy(x->gate_table, ents.data(), ents.size() * sizeof(GateEntry), cudaMemcpyHostToDevice));
  x->gate_entries = (int)ents.size();
  PGX_CUDA(cudaDeviceSynchronize());
  cudaSetDevice(prev);
  return PGX_OK;
}

static void nvls_release(pgx_xchg* x) {
  if (!x->nv.mc) return;
  PGX_DRV(cuMemUnmap);
  PGX_DRV(cuMemAddressFree);
  PGX_DRV(cuMemRelease);
  PGX_DRV(cuMulticastUnbind);
  PGX_DRV(cuDeviceGet);
  if (x->nv.mcp && p_cuMemUnmap) p_cuMemUnmap(x->nv.mcp, x->nv.size);
  if (x->nv.uc && p_cuMemUnmap) p_cuMemUnmap(x->nv.uc, x->nv.size);
  if (x->nv.mcp && p_cuMemAddressFree) p_cuMemAddressFree(x->nv.mcp, x->nv.size);
  if (x->nv.uc && p_cuMemAddressFree) p_cuMemAddressFree(x->nv.uc, x->nv.size);
  CUdevice d;
  if (x->nv.mem && p_cuMulticastUnbind && p_cuDeviceGet && p_cuDeviceGet(&d, x->dev) == CUDA_SUCCESS)
    p_cuMulticastUnbind(x->nv.mc, d, 0, x->nv.size);
  if (x->nv.mem && p_cuMemRelease) p_cuMemRelease(x->nv.mem);
  if (p_cuMemRelease) p_cuMemRelease(x->nv.mc);
  x->nv = pgx_xchg::Nvls{};
}

static int launch_nvls(pgx_xchg* x, int l, const LayerPlan& P, const XArgs& a, cudaStream_t s) {
  if (!x->nv.on) return fail(PGX_E_CONFIG, "NVLS exchange not bound (pgx_xchg_nvls_bind)");
  NvArgs n;
  memset(&n, 0, sizeof(n));
  n.g = a.g;
  n.uc_model = reinterpret_cast<float*>(x->nv.uc) + P.model_off;
  n.uc_grad = reinterpret_cast<float*>(x->nv.uc + x->nv.grad_off) + P.model_off;
  n.mc_model = x->nv.mcp + P.model_off * 4;
  n.mc_grad = x->nv.mcp + x->nv.grad_off + P.model_off * 4;
  n.uc_ready = reinterpret_cast<uint32_t*>(x->nv.uc + x->nv.flag_off + x->nv.fl[l] + 128);
  n.mc_ready = x->nv.mcp + x->nv.flag_off + x->nv.fl[l] + 128;
  n.mc_arrive = x->nv.mcp + x->nv.flag_off + x->nv.fl[l];
  n.C = P.C;
  n.v = a.v;
  n.queue = a.queue;
  n.S = P.S;
  n.sl = P.sl;
  n.CH = P.CH;
  n.pub_items = P.push_items;
  n.items = P.items;
  n.epoch = a.epoch;
  n.iter = a.iter;
  n.rank = x->rank;
  n.world = x->world;
  n.lr = a.lr;
  n.scale = a.scale;
  n.mu = a.mu;
  n.wd = a.wd;
  n.st = a.st;
  ++x->launches;
  k_nvls<<<P.grid, kThreads, 0, s>>>(n);
  return PGX_OK;
}

// TWOSHOT_CE: owner j's shard split into its pipelined parts (the same split on the
// pushing and the owning side); returns the part count and part p's [lo, hi).
static int ce_split(const pgx_xchg* x, const LayerPlan& P, int j, int p, uint64_t* plo, uint64_t* phi) {
  const uint64_t lo = std::min(P.S, (uint64_t)j * P.sl), hi = std::min(P.S, (uint64_t)(j + 1) * P.sl);
  int parts = x->world > 1 ? x->ce_parts : 1;
  const uint64_t min_part = 1u << 18;  // elements: do not split small shards
  while (parts > 1 && (hi - lo) / parts < min_part) --parts;
  parts = std::min<int>(parts, (int)P.C);
  if (parts < 1) parts = 1;
  if (plo) {
    *plo = lo + ((hi - lo) * p / parts) / 4 * 4;
    *phi = p + 1 == parts ? hi : lo + ((hi - lo) * (p + 1) / parts) / 4 * 4;
  }
  return parts;
}

// TWOSHOT_CE launch: reduce-scatter and all-gather as peer DMA copies, each batch
// followed (in stream order) by k_signal raising the peers' notifications with a
// system-scope release; owner fold/update as a local kernel.
static int launch_twoshot_ce(pgx_xchg* x, int l, const LayerPlan& P, XArgs& a, cudaStream_t s, int phases) {
  const int N = x->world, me = x->rank;
  const int esz = x->esz;
  a.parity = 0;  // single-buffered: a sender rewrites a slot only after it gated on this owner's previous
                 // all-gather, which the owner sends after reading the slot (per-layer forward gate)
  cudaError_t e = xrecord(x->ready[l], s);
  if (e != cudaSuccess) return fail(PGX_E_CUDA, "event: %s", cudaGetErrorString(e));
  const bool rs_parts = x->ce_rs_parts && N > 1;
  if ((phases & PGX_PHASE_PUSH) && rs_parts) {
    // part-major push: all peers' part p, then an event; the signals for part p run on
    // ce_rs2 behind that event, so the copy queue never drains waiting for a kernel and
    // each owner starts folding part p while part p+1 is still in flight
    xwait(x->ce_rs, x->ready[l]);
    xwait(x->ce_rs2, x->ready[l]);
    int np[PGX_MAX_RANKS] = {}, pmax = 0;
    for (int j = 0; j < N; ++j) pmax = std::max(pmax, np[j] = ce_split(x, P, j, 0, nullptr, nullptr));
    for (int p = 0; p < pmax; ++p) {
      FlagOut fo{};
      for (int d = 1; d < N; ++d) {
        int j = (me + d) % N;
        if (p >= np[j]) continue;
        uint64_t lo, hi, jlo = std::min(P.S, (uint64_t)j * P.sl);
        ce_split(x, P, j, p, &lo, &hi);
        uint8_t* dst = static_cast<uint8_t*>(a.rx[j]) + ((uint64_t)(a.parity * a.K + me) * P.sl + (lo - jlo)) * esz;
        uint64_t pb = 0;
        for (int k = 0; k < a.g.n && lo < hi; ++k) {
          uint64_t pe = a.g.end[k];
          uint64_t ol = std::max(lo, pb), oh = std::min(hi, pe);
          if (ol < oh) {
            e = cudaMemcpyAsync(dst + (ol - lo) * esz, static_cast<const uint8_t*>(a.g.p[k]) + (ol - pb) * esz,
                                (oh - ol) * esz, cudaMemcpyDeviceToDevice, x->ce_rs);
            if (e != cudaSuccess) return fail(PGX_E_CUDA, "peer copy: %s", cudaGetErrorString(e));
          }
          pb = pe;
        }
        fo.f[fo.n++] = a.rxflags[j] + (uint64_t)me * P.C + p;
      }
      if (!fo.n) continue;
      xrecord(x->rs_part_ev[l][p], x->ce_rs);
      xwait(x->ce_rs2, x->rs_part_ev[l][p]);
      k_signal<<<1, 32, 0, x->ce_rs2>>>(fo, a.epoch, a.iter);
      ++x->launches;
    }
    xrecord(x->rs_done[l], x->ce_rs);
    xrecord(x->rs2_done[l], x->ce_rs2);
  } else if (phases & PGX_PHASE_PUSH) {
    // peers alternate between one or two copy streams; each stream signals its own peers
    const int ns = (x->ce_rs_streams > 1 && N > 2) ? 2 : 1;
    cudaStream_t rs[2] = {x->ce_rs, x->ce_rs2};
    FlagOut fo[2] = {};
    for (int q = 0; q < ns; ++q) xwait(rs[q], x->ready[l]);
    for (int d = 1; d < N; ++d) {
      int j = (me + d) % N;
      cudaStream_t cs = rs[(d - 1) % ns];
      uint64_t lo = std::min(P.S, (uint64_t)j * P.sl), hi = std::min(P.S, (uint64_t)(j + 1) * P.sl);
      uint8_t* dst = static_cast<uint8_t*>(a.rx[j]) + ((uint64_t)(a.parity * a.K + me) * P.sl) * esz;
      uint64_t pb = 0;
      for (int k = 0; k < a.g.n && lo < hi; ++k) {
        uint64_t pe = a.g.end[k];
        uint64_t ol = std::max(lo, pb), oh = std::min(hi, pe);
        if (ol < oh) {
          e = cudaMemcpyAsync(dst + (ol - lo) * esz, static_cast<const uint8_t*>(a.g.p[k]) + (ol - pb) * esz,
                              (oh - ol) * esz, cudaMemcpyDeviceToDevice, cs);
          if (e != cudaSuccess) return fail(PGX_E_CUDA, "peer copy: %s", cudaGetErrorString(e));
        }
        pb = pe;
      }
      FlagOut& f = fo[(d - 1) % ns];
      f.f[f.n++] = a.rxflags[j] + (uint64_t)me * P.C;
    }
    for (int q = 0; q < ns; ++q) {
      if (fo[q].n) {
        k_signal<<<1, 32, 0, rs[q]>>>(fo[q], a.epoch, a.iter);
        ++x->launches;
      }
      xrecord(q == 0 ? x->rs_done[l] : x->rs2_done[l], rs[q]);
    }
  }
  if (phases & PGX_PHASE_OWNER) {
    xwait(x->ce_own, x->ready[l]);
    const uint64_t lo = std::min(P.S, (uint64_t)me * P.sl), hi = std::min(P.S, (uint64_t)(me + 1) * P.sl);
    // owner fold/update in parts; each part's all-gather copies start as soon as it is done
    const int parts = ce_split(x, P, me, 0, nullptr, nullptr);
    for (int p = 0; p < parts; ++p) {
      if (p == 0 || rs_parts) {  // whole-shard signal, or this part's signal from every peer
        FlagSet fs{};
        for (int sidx = 0; sidx < N; ++sidx)
          if (sidx != me) fs.f[fs.n++] = a.rxflags[me] + (uint64_t)sidx * P.C + (rs_parts ? p : 0);
        if (fs.n) {
          k_wait_flags<<<1, 32, 0, x->ce_own>>>(fs, a.epoch, a.iter, 1u, a.st);
          ++x->launches;
        }
      }
      uint64_t plo, phi;
      ce_split(x, P, me, p, &plo, &phi);
      a.olo = plo;
      a.ohi = phi;
      int grid = std::max(1, std::min(P.grid, (int)(((phi - plo) / VecT<float>::W + kThreads - 1) / kThreads)));
      if (phi > plo && x->ce_tma_owner) {
        launch_owner_tma(N, x->cfg.mode, std::max(1, std::min(P.grid, (int)((phi - plo + 8191) / 8192))), x->dev,
                         x->ce_own, a);
        ++x->launches;
      } else if (phi > plo) {
        if (esz == 8)
          launch_owner_local<double>(N, grid, x->ce_own, a);
        else
          launch_owner_local<float>(N, grid, x->ce_own, a);
        ++x->launches;
      }
      if (N == 1) continue;
      xrecord(x->part_ev[l][p], x->ce_own);
      xwait(x->ce_ag, x->part_ev[l][p]);
      for (int d = 1; d < N && phi > plo; ++d) {
        int t = (me + d) % N;
        e = cudaMemcpyAsync(static_cast<uint8_t*>(a.model[t]) + plo * esz, static_cast<uint8_t*>(a.model[me]) + plo * esz,
                            (phi - plo) * esz, cudaMemcpyDeviceToDevice, x->ce_ag);
        if (e != cudaSuccess) return fail(PGX_E_CUDA, "peer copy: %s", cudaGetErrorString(e));
      }
    }
    cudaStream_t tail = N > 1 ? x->ce_ag : x->ce_own;
    if (N == 1 || lo >= hi) xwait(x->ce_ag, x->ready[l]);  // keep ce_ag joined even with nothing to copy
    FlagOut fo{};
    for (int d = 1; d < N; ++d)
      fo.f[fo.n++] = a.mflags[(me + d) % N] + x->ownerflag_base + (uint64_t)l * N + me;
    if (fo.n) {
      k_signal<<<1, 32, 0, tail>>>(fo, a.epoch, a.iter);
      ++x->launches;
    }
    e = xrecord(x->done[l], tail);
    if (e != cudaSuccess) return fail(PGX_E_CUDA, "event: %s", cudaGetErrorString(e));
  }
  return PGX_OK;
}

// TWOSHOT_CEP launch: the reduce-scatter as copy-engine peer copies (one per peer, the
// sizes where the copy engines run at full rate), then one k_signal_range raising every
// chunk flag of the shard; the owner side is the SM two-shot kernel's owner items
// (tree-order fold + fused update + all-gather peer stores + arrival counters) on its
// own stream behind a one-CTA wait, so its CTAs do not spin while the copies fly.
static int launch_twoshot_cep(pgx_xchg* x, int l, const LayerPlan& P, XArgs& a, cudaStream_t s, int phases) {
  const int N = x->world, me = x->rank, esz = x->esz;
  a.single_buffer = 1;  // host-addressed copies: parity 0 (safe: senders gate on the previous all-gather)
  a.parity = 0;
  cudaError_t e = xrecord(x->ready[l], s);
  if (e != cudaSuccess) return fail(PGX_E_CUDA, "event: %s", cudaGetErrorString(e));
  auto shard = [&](int j, uint64_t& lo, uint64_t& hi) {
    lo = std::min(P.S, (uint64_t)j * P.sl);
    hi = std::min(P.S, (uint64_t)(j + 1) * P.sl);
  };
  if (phases & PGX_PHASE_PUSH) {
    xwait(x->ce_rs, x->ready[l]);
    FlagRanges fr{};
    for (int d = 1; d < N; ++d) {
      int j = (me + d) % N;
      uint64_t lo, hi;
      shard(j, lo, hi);
      if (lo >= hi) continue;
      uint8_t* dst = static_cast<uint8_t*>(a.rx[j]) + ((uint64_t)me * P.sl) * esz;
      uint64_t pb = 0;
      for (int k = 0; k < a.g.n; ++k) {
        uint64_t pe = a.g.end[k];
        uint64_t ol = std::max(lo, pb), oh = std::min(hi, pe);
        if (ol < oh) {
          e = cudaMemcpyAsync(dst + (ol - lo) * esz, static_cast<const uint8_t*>(a.g.p[k]) + (ol - pb) * esz,
                              (oh - ol) * esz, cudaMemcpyDeviceToDevice, x->ce_rs);
          if (e != cudaSuccess) return fail(PGX_E_CUDA, "peer copy: %s", cudaGetErrorString(e));
        }
        pb = pe;
      }
      fr.f[fr.k] = a.rxflags[j] + (uint64_t)me * P.C;
      fr.n[fr.k++] = (uint32_t)((hi - lo + P.CH - 1) / P.CH);
    }
    if (fr.k) {
      k_signal_range<<<1, 256, 0, x->ce_rs>>>(fr, a.epoch, a.iter);
      ++x->launches;
    }
    xrecord(x->rs_done[l], x->ce_rs);
  }
  if (phases & PGX_PHASE_OWNER) {
    xwait(x->ce_own, x->ready[l]);
    uint64_t lo, hi;
    shard(me, lo, hi);
    const uint32_t mine = lo < hi ? (uint32_t)((hi - lo + P.CH - 1) / P.CH) : 0;
    if (mine && N > 1) {  // every peer raises all of a shard's flags at once: wait on the last one
      FlagSet fs{};
      for (int sidx = 0; sidx < N; ++sidx)
        if (sidx != me) fs.f[fs.n++] = a.rxflags[me] + (uint64_t)sidx * P.C + (mine - 1);
      k_wait_flags<<<1, 32, 0, x->ce_own>>>(fs, a.epoch, a.iter, 1u, a.st);
      ++x->launches;
    }
    a.item_begin = P.push_items;
    a.item_end = P.items;
    if (mine) {
      int grid = (int)std::min<uint32_t>(mine, (uint32_t)P.grid);
      ++x->launches;
      if (esz == 8)
        launch_twoshot<double>(N, false, grid, x->dev, x->ce_own, a);
      else
        launch_twoshot<float>(N, false, grid, x->dev, x->ce_own, a);
    }
    e = cudaGetLastError();
    if (e == cudaSuccess) e = xrecord(x->done[l], x->ce_own);
    if (e != cudaSuccess) return fail(PGX_E_CUDA, "exchange launch failed: %s", cudaGetErrorString(e));
  }
  return PGX_OK;
}

// TWOSHOT_BULK with PGX_XF_BULK_CE_RS: the reduce-scatter moves by the copy engines (zero
// SM time) in part-major copies — part p of every peer's shard, then one k_signal_range on a
// second stream raising exactly the chunk flags that part covers — so the owner kernel
// (k_twoshot_bulk owner slabs: tree-order fold + fused update + TMA bulk all-gather, capped
// grid) folds part p while part p+1 is still on the wire.  Receive slots are single-buffered
// like the other host-addressed variants (a sender rewrites a slot only after gating on this
// owner's previous all-gather, which follows the owner's reads of the slot).
constexpr uint32_t kCebParts = 4;

static int launch_bulk_ce_rs(pgx_xchg* x, int l, const LayerPlan& P, XArgs& a, int phases) {
  const int N = x->world, me = x->rank, esz = x->esz;
  a.single_buffer = 1;
  a.parity = 0;
  cudaError_t e = cudaSuccess;
  const uint32_t cp = (P.C + kCebParts - 1) / kCebParts;  // chunks per part
  auto shard = [&](int j, uint64_t& lo, uint64_t& hi) {
    lo = std::min(P.S, (uint64_t)j * P.sl);
    hi = std::min(P.S, (uint64_t)(j + 1) * P.sl);
  };
  if (phases & PGX_PHASE_PUSH) {
    xwait(x->ce_rs, x->ready[l]);
    xwait(x->ce_rs2, x->ready[l]);
    for (uint32_t p = 0; (uint64_t)p * cp < P.C; ++p) {
      FlagRanges fr{};
      for (int d = 1; d < N; ++d) {
        const int j = (me + d) % N;
        uint64_t jlo, jhi;
        shard(j, jlo, jhi);
        const uint64_t lo = std::min(jhi, jlo + (uint64_t)p * cp * P.CH);
        const uint64_t hi = std::min(jhi, jlo + (uint64_t)(p + 1) * cp * P.CH);
        if (lo >= hi) continue;
        uint8_t* dst = static_cast<uint8_t*>(a.rx[j]) + ((uint64_t)me * P.sl + (lo - jlo)) * esz;
        uint64_t pb = 0;
        for (int k = 0; k < a.g.n; ++k) {
          const uint64_t pe = a.g.end[k], ol = std::max(lo, pb), oh = std::min(hi, pe);
          if (ol < oh) {
            e = cudaMemcpyAsync(dst + (ol - lo) * esz, static_cast<const uint8_t*>(a.g.p[k]) + (ol - pb) * esz,
                                (oh - ol) * esz, cudaMemcpyDeviceToDevice, x->ce_rs);
            if (e != cudaSuccess) return fail(PGX_E_CUDA, "peer copy: %s", cudaGetErrorString(e));
          }
          pb = pe;
        }
        fr.f[fr.k] = a.rxflags[j] + (uint64_t)me * P.C + (uint64_t)p * cp;
        fr.n[fr.k++] = (uint32_t)((hi - lo + P.CH - 1) / P.CH);
      }
      if (!fr.k) continue;
      xrecord(x->rs_part_ev[l][p], x->ce_rs);
      xwait(x->ce_rs2, x->rs_part_ev[l][p]);
      k_signal_range<<<1, 256, 0, x->ce_rs2>>>(fr, a.epoch, a.iter);
      ++x->launches;
    }
    xrecord(x->rs_done[l], x->ce_rs);
    xrecord(x->rs2_done[l], x->ce_rs2);
  }
  if (phases & PGX_PHASE_OWNER) {
    xwait(x->ce_own, x->ready[l]);
    uint64_t lo, hi;
    shard(me, lo, hi);
    const uint32_t mine = lo < hi ? (uint32_t)((hi - lo + P.CH - 1) / P.CH) : 0;
    if (mine && N > 1) {  // the owner CTAs start once the first part has arrived from every peer
      FlagSet fs{};
      for (int sidx = 0; sidx < N; ++sidx)
        if (sidx != me) fs.f[fs.n++] = a.rxflags[me] + (uint64_t)sidx * P.C + (std::min(cp, mine) - 1);
      k_wait_flags<<<1, 32, 0, x->ce_own>>>(fs, a.epoch, a.iter, 1u, a.st);
      ++x->launches;
    }
    a.item_begin = P.push_items;
    a.item_end = P.items;
    if (mine) {
      ++x->launches;
      launch_twoshot_bulk(N, (int)std::min<uint32_t>(mine, (uint32_t)P.grid), x->dev, x->ce_own, a);
    }
    e = cudaGetLastError();
    if (e == cudaSuccess) e = xrecord(x->done[l], x->ce_own);
    if (e != cudaSuccess) return fail(PGX_E_CUDA, "exchange launch failed: %s", cudaGetErrorString(e));
  }
  return PGX_OK;
}

extern "C" {

int pgx_xchg_create(pgx_world* w, const pgx_xchg_config* cfg, pgx_xchg** out) {
  if (!cfg || cfg->num_layers < 1) return fail(PGX_E_CONFIG, "exchange needs at least one layer");
  if (cfg->chunk_elems < 4 || cfg->chunk_elems % 4) return fail(PGX_E_CONFIG, "chunk_elems must be a positive multiple of 4");
  if (cfg->mode < 0 || cfg->mode > 3) return fail(PGX_E_CONFIG, "unknown mode %d", cfg->mode);
  if (!(cfg->lr > 0)) return fail(PGX_E_CONFIG, "epsilon must be > 0, got %g", cfg->lr);
  if (cfg->ce_parts < 0 || cfg->ce_parts > 8) return fail(PGX_E_CONFIG, "ce_parts must be 0 (default) or 1..8");
  if (cfg->ce_rs_streams < 0 || cfg->ce_rs_streams > 2)
    return fail(PGX_E_CONFIG, "ce_rs_streams must be 0 (default), 1 or 2");
  for (int l = 0; l < cfg->num_layers; ++l) {
    if (cfg->variant && (cfg->variant[l] == PGX_VARIANT_ONESHOT_L128 || cfg->variant[l] == PGX_VARIANT_TWOSHOT_L128)) {
      // fence-free 128-byte lines rest on a probed (not promised) property of sm_100 NVLink
      // writes: only on explicit request, only on that architecture
      if (!(cfg->flags & PGX_XF_ALLOW_L128))
        return fail(PGX_E_CONFIG, "layer %d: the 128-byte-line variants need the PGX_XF_ALLOW_L128 opt-in flag", l);
      int dev = 0, major = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
      if (major != 10) return fail(PGX_E_CONFIG, "the 128-byte-line variants were validated on sm_100 only (device is sm_%d x)", major);
    }
  }
  pgx_xchg* x = new pgx_xchg();
  x->w = w;
  x->cfg = *cfg;
  x->rank = world_rank(w);
  x->world = world_size(w);
  x->dev = world_device(w);
  x->esz = cfg->mode == PGX_MODE_REF64 ? 8 : 4;
  // former environment knobs, now part of the config (ABI 3); 0 = the measured defaults
  x->auto_chunk_tree = (cfg->flags & PGX_XF_AUTO_CHUNK_TREE) != 0;
  x->auto_chunk_nvls = (cfg->flags & PGX_XF_NO_AUTO_CHUNK_NVLS) == 0;
  x->oneshot_small_chunks = (cfg->flags & PGX_XF_ONESHOT_SMALL_CHUNKS) != 0;
  x->tma = (cfg->flags & PGX_XF_TMA) != 0;
  x->bulk_ce_rs = (cfg->flags & PGX_XF_BULK_CE_RS) != 0;
  x->ce_tma_owner = (cfg->flags & PGX_XF_CE_TMA_OWNER) != 0;
  x->ce_rs_parts = (cfg->flags & PGX_XF_CE_RS_PARTS) != 0;
  if (cfg->ce_parts) x->ce_parts = cfg->ce_parts;
  if (cfg->ce_rs_streams) x->ce_rs_streams = cfg->ce_rs_streams;
  x->seg_model = cfg->seg_base;
  x->seg_rx = cfg->seg_base + 1;
  const int N = x->world;
  int kmax = 0;
  for (int r = 0; r < N; ++r) kmax = std::max(kmax, tree_num_children(r, N));
  int sms = sm_count(x->dev);
  const int cap_all = cfg->max_ctas > 0 ? cfg->max_ctas : 2 * sms;
  uint64_t moff = 0, rxoff = 0, rxfoff = 0;
  uint32_t dflag = cfg->num_layers;
  x->L.resize(cfg->num_layers);
  for (int l = 0; l < cfg->num_layers; ++l) {
    LayerPlan& P = x->L[l];
    P.S = cfg->layer_elems[l];
    if (P.S < 1) {
      delete x;
      return fail(PGX_E_CONFIG, "layer %d has no elements", l);
    }
    P.variant = cfg->variant ? cfg->variant[l] : PGX_VARIANT_TWOSHOT;
    const bool ch_given = cfg->layer_chunk_elems && cfg->layer_chunk_elems[l];
    uint64_t CH = ch_given ? cfg->layer_chunk_elems[l] : cfg->chunk_elems;
    if (!ch_given && N > 1 && P.variant != PGX_VARIANT_TWOSHOT_CE && P.variant != PGX_VARIANT_ONESHOT &&
        P.variant != PGX_VARIANT_TWOSHOT_BULK &&
        P.variant != PGX_VARIANT_ONESHOT_LL && P.variant != PGX_VARIANT_ONESHOT_L128 && P.variant != PGX_VARIANT_TWOSHOT_L128 &&
        !(P.variant == PGX_VARIANT_TREE && !x->auto_chunk_tree) && !(P.variant == PGX_VARIANT_NVLS && !x->auto_chunk_nvls)) {
      // big shards: chunks of up to 64 K elements (~128 per shard) amortise the system fence
      // that ends every chunk; chunk_elems stays the minimum (profiles/r3e, r3n)
      const uint64_t shard = P.variant == PGX_VARIANT_TREE ? P.S : (P.S + N - 1) / N;
      const uint64_t target = shard / 128;
      uint64_t c = CH;
      while (c * 2 <= target && c * 2 <= kAutoChunkMax) c *= 2;
      // small shards (<= 1 MB): half-size chunks double the parallel pushes (4 MB layer at
      // N=4: 40 vs 46 us, profiles/r3x)
      if (P.variant == PGX_VARIANT_TWOSHOT && shard <= (1u << 18) && c >= 8192 && c == CH) c /= 2;
      CH = c;
    }
    if (!ch_given && N == 1 && P.variant == PGX_VARIANT_TWOSHOT && CH > kN1Chunk) {
      // one rank: the launch is the fused update alone, a pure HBM stream; 4 K-element items
      // keep the last wave short (fc6 alone: 0.938 of the HBM peak with 16 K, 0.987 with 4 K;
      // 2 K items pay more in claims than they save, profiles/r6f_prof_update.jsonl)
      CH = kN1Chunk;
    }
    if (CH < 4 || CH % 4) {
      delete x;
      return fail(PGX_E_CONFIG, "layer %d: chunk_elems must be a positive multiple of 4", l);
    }
    if (!ch_given && P.variant == PGX_VARIANT_TWOSHOT_BULK) {
      // slabs (one fence + flag each) of 64 K .. 256 K elements, >= ~one owner slab per CTA
      const uint64_t shard = (P.S + N - 1) / N;
      const int g = (cfg->layer_max_ctas && cfg->layer_max_ctas[l] > 0) ? cfg->layer_max_ctas[l]
                    : cfg->max_ctas > 0 ? cfg->max_ctas : kBulkCtas;
      uint64_t c = (shard + g - 1) / g;
      c = std::max<uint64_t>(65536, std::min<uint64_t>(262144, c));
      CH = align_up(c, 8192);  // whole ring tiles (32 KB of fp32)
    }
    P.CH = CH;
    // per-layer CTA cap (large layers: fewer CTAs with bigger chunks leave SMs to the backward)
    const bool lcapped = cfg->layer_max_ctas && cfg->layer_max_ctas[l] > 0;
    int cap = lcapped ? cfg->layer_max_ctas[l] : cap_all;
    bool capped = lcapped || cfg->max_ctas > 0;
    P.lean = (cfg->flags & PGX_XF_LEAN_CAPPED) && lcapped &&
             (P.variant == PGX_VARIANT_ONESHOT_LL || P.variant == PGX_VARIANT_TWOSHOT_L128);
    if (P.variant == PGX_VARIANT_TWOSHOT_CEP && !capped) {  // 48 CTAs saturate NVLink (profiles/r3h)
      cap = std::min(cap, kCepCtas);
      capped = true;
    }
    if (P.variant == PGX_VARIANT_TWOSHOT_CE && x->ce_tma_owner && !capped) {
      cap = kCeTmaCtas;
      capped = true;
    }
    if (P.variant == PGX_VARIANT_TWOSHOT_BULK && !capped) {  // 16-24 TMA CTAs saturate NVLink (r3d)
      cap = kBulkCtas;
      capped = true;
    }
    P.model_off = moff;
    moff = align_up(moff + P.S, kAlignElems);
    if (P.variant == PGX_VARIANT_NVLS && (cfg->mode != PGX_MODE_FAST32 || N < 2)) {
      delete x;
      return fail(PGX_E_CONFIG, "NVLS layers need fast32 and at least 2 ranks");
    }
    if (P.variant == PGX_VARIANT_TWOSHOT || P.variant == PGX_VARIANT_TWOSHOT_CE || P.variant == PGX_VARIANT_NVLS ||
        P.variant == PGX_VARIANT_TWOSHOT_CEP || P.variant == PGX_VARIANT_TWOSHOT_BULK) {
      P.sl = align_up((P.S + N - 1) / N, 4);
      P.C = (uint32_t)((P.sl + CH - 1) / CH);
      P.K = N;
      P.rx_off = rxoff;
      rxoff = align_up(rxoff + 2 * (uint64_t)N * P.sl, kAlignElems);
      P.rxflag_off = rxfoff;
      rxfoff += (uint64_t)N * P.C;
      uint64_t my_lo = std::min(P.S, (uint64_t)x->rank * P.sl), my_hi = std::min(P.S, (uint64_t)(x->rank + 1) * P.sl);
      uint32_t my_chunks = (uint32_t)((my_hi - my_lo + CH - 1) / CH);
      P.push_items = (uint32_t)(N - 1) * P.C;
      P.items = P.push_items + P.C;
      uint32_t remote = 0;
      for (int j = 0; j < N; ++j) {
        if (j == x->rank) continue;
        uint64_t lo = std::min(P.S, (uint64_t)j * P.sl), hi = std::min(P.S, (uint64_t)(j + 1) * P.sl);
        remote += (uint32_t)((hi - lo + CH - 1) / CH);
      }
      P.expected = remote;
      if (P.variant == PGX_VARIANT_NVLS) {  // publish (owner, chunk) items, then own chunks
        P.push_items = (uint32_t)N * P.C;
        P.items = P.push_items + P.C;
        P.expected = remote + my_chunks;  // every owner's chunks arrive by multicast, own ones included
      }
      P.grid = (int)std::min<uint64_t>(P.items, capped ? cap : (N == 1 ? 4 * sms : cap));
      uint64_t own = my_hi - my_lo;
      P.nvlink_bytes = (N > 1) ? 2ull * (P.S - own) * x->esz : 0;  // RS out + AG out
      // owner fold: N partial reads + w (+v) read/write; pushes read the rest of the gradient
      P.hbm_bytes = ((uint64_t)N + 2 + (cfg->mode == PGX_MODE_FAST32 ? 2 : cfg->mode == PGX_MODE_SUM32 ? -1 : 0)) * own * x->esz +
                    (P.S - own) * x->esz;

    } else if (P.variant == PGX_VARIANT_ONESHOT_L128) {
      if (x->esz != 4) {
        delete x;
        return fail(PGX_E_CONFIG, "layer %d: ONESHOT_L128 carries fp32 values (not ref64)", l);
      }
      const uint64_t lines = (P.S + kL128Vals - 1) / kL128Vals;
      P.sl = align_up(lines * 32, kAlignElems);  // slot: `lines` 128-byte lines (in 4-byte units)
      // chunk = lines per item: ~one item per SM per phase, at least 32 lines (4 per warp)
      CH = std::max<uint64_t>(32, (lines + sms - 1) / sms);
      if (ch_given) CH = std::max<uint64_t>(1, cfg->layer_chunk_elems[l] / kL128Vals);
      P.CH = CH;
      P.C = (uint32_t)((lines + CH - 1) / CH);
      P.K = N;
      P.rx_off = rxoff;
      rxoff = align_up(rxoff + 2 * (uint64_t)N * P.sl, kAlignElems);
      P.rxflag_off = rxfoff;  // no flags: the epoch rides in every line
      P.push_items = P.C;
      P.items = 2 * P.C;
      P.expected = 0;
      P.grid = (int)std::min<uint64_t>(P.items, cap);
      P.nvlink_bytes = (uint64_t)(N - 1) * lines * 128;
      P.hbm_bytes = ((uint64_t)N + 2 + (cfg->mode == PGX_MODE_FAST32 ? 2 : cfg->mode == PGX_MODE_SUM32 ? -1 : 0)) * P.S * x->esz +
                    (uint64_t)(N - 1) * lines * 128;
    } else if (P.variant == PGX_VARIANT_TWOSHOT_L128) {
      if (x->esz != 4) {
        delete x;
        return fail(PGX_E_CONFIG, "layer %d: TWOSHOT_L128 carries fp32 values (not ref64)", l);
      }
      const uint64_t lines = (P.S + kL128Vals - 1) / kL128Vals;
      const uint64_t Ls = (lines + N - 1) / N;
      P.sl = align_up(Ls * 32, kAlignElems);            // reduce-scatter slot: Ls lines (4-byte units)
      const uint64_t agl = align_up(lines * 32, kAlignElems);  // gather area: every line
      // chunk = lines per item: ~one push item per SM, at least 64 lines (4 per warp)
      CH = std::max<uint64_t>(64, ((uint64_t)std::max(N - 1, 1) * Ls + sms - 1) / sms);
      if (ch_given) CH = std::max<uint64_t>(1, cfg->layer_chunk_elems[l] / kL128Vals);
      P.CH = CH;
      P.C = (uint32_t)((Ls + CH - 1) / CH);  // chunks per shard (ragged last shard: empty items)
      // owner items fold N-1 polled lines and store N-1 copies per line: (N-1)x finer than
      // the push items so the owner phase spreads over as many CTAs as the push phase
      P.CHo = std::max<uint64_t>(64, align_up((CH + std::max(N - 1, 1) - 1) / std::max(N - 1, 1), 4));
      if (P.CHo > CH) P.CHo = CH;
      P.Co = (uint32_t)((Ls + P.CHo - 1) / P.CHo);
      P.K = N;
      P.rx_off = rxoff;
      rxoff = align_up(rxoff + 2 * ((uint64_t)N * P.sl + agl), kAlignElems);
      P.rxflag_off = rxfoff;  // no flags: the epoch rides in every line
      P.push_items = (uint32_t)(N - 1) * P.C;
      P.down_items = (uint32_t)(N - 1) * P.C;  // install items (PGX_PHASE_DOWN)
      P.items = P.push_items + P.Co + P.down_items;
      P.expected = 0;  // this rank's own install items complete the layer
      P.grid = (int)std::min<uint64_t>(P.items, cap);
      const uint64_t my_lines = std::min(lines, (uint64_t)(x->rank + 1) * Ls) - std::min(lines, (uint64_t)x->rank * Ls);
      // out: my gradient's lines of the other shards + my updated lines to every peer
      P.nvlink_bytes = N > 1 ? ((lines - my_lines) + (uint64_t)(N - 1) * my_lines) * 128 : 0;
      const uint64_t own = std::min<uint64_t>(P.S, (uint64_t)(x->rank + 1) * Ls * kL128Vals) -
                           std::min<uint64_t>(P.S, (uint64_t)x->rank * Ls * kL128Vals);
      const uint64_t wv = cfg->mode == PGX_MODE_FAST32 ? 4 : cfg->mode == PGX_MODE_SUM32 ? 1 : 2;  // w (+v) traffic
      // push reads + owner (own gradient, w/v) + rx lines written by peers and read back +
      // gather lines written by owners and read back + install stores into the weights
      P.hbm_bytes = 2 * (P.S - own) * x->esz + (1 + wv) * own * x->esz +
                    2 * ((uint64_t)(N - 1) * my_lines + (lines - my_lines)) * 128;
    } else if (P.variant == PGX_VARIANT_ONESHOT_LL) {
      if (x->esz != 4) {
        delete x;
        return fail(PGX_E_CONFIG, "layer %d: ONESHOT_LL carries fp32 values (not ref64)", l);
      }
      P.sl = align_up(2 * P.S, kAlignElems);  // slot: one 8-byte {value, epoch} word per element
      if (!ch_given) {  // latency path: spread even small layers over ~one CTA per SM per phase
        const uint64_t want = align_up((P.S + sms - 1) / sms, 4);
        CH = std::min<uint64_t>(CH, std::max<uint64_t>(256, want));
        P.CH = CH;
      }
      P.C = (uint32_t)((P.S + CH - 1) / CH);
      P.K = N;
      P.rx_off = rxoff;
      rxoff = align_up(rxoff + 2 * (uint64_t)N * P.sl, kAlignElems);
      P.rxflag_off = rxfoff;  // no flags: the epoch rides in every word
      P.push_items = P.C;
      P.items = 2 * P.C;
      P.expected = 0;  // each rank updates its own copy
      P.grid = (int)std::min<uint64_t>(P.items, cap);
      P.nvlink_bytes = 2ull * (N - 1) * P.S * x->esz;
      P.hbm_bytes = ((uint64_t)N + 2 + (cfg->mode == PGX_MODE_FAST32 ? 2 : cfg->mode == PGX_MODE_SUM32 ? -1 : 0)) * P.S * x->esz +
                    (uint64_t)(N - 1) * P.S * x->esz;
    } else if (P.variant == PGX_VARIANT_ONESHOT) {
      P.sl = align_up(P.S, kAlignElems);  // slot stride: every peer's whole gradient
      if (!ch_given && x->oneshot_small_chunks) {  // latency: more, smaller chunks in parallel
        const uint64_t want = align_up((P.S + sms - 1) / sms, 4);
        CH = std::min<uint64_t>(CH, std::max<uint64_t>(1024, want));
        P.CH = CH;
      }
      P.C = (uint32_t)((P.S + CH - 1) / CH);
      P.K = N;
      P.rx_off = rxoff;
      rxoff = align_up(rxoff + 2 * (uint64_t)N * P.sl, kAlignElems);
      P.rxflag_off = rxfoff;
      rxfoff += (uint64_t)N * P.C;
      P.push_items = (uint32_t)(N - 1) * P.C;
      P.items = P.push_items + P.C;
      P.expected = 0;  // each rank updates its own copy
      P.grid = (int)std::min<uint64_t>(P.items, cap);
      P.nvlink_bytes = (uint64_t)(N - 1) * P.S * x->esz;
      P.hbm_bytes = ((uint64_t)N + 2 + (cfg->mode == PGX_MODE_FAST32 ? 2 : cfg->mode == PGX_MODE_SUM32 ? -1 : 0)) * P.S * x->esz +
                    (uint64_t)(N - 1) * P.S * x->esz;
    } else if (P.variant == PGX_VARIANT_TREE) {
      P.sl = align_up(P.S, kAlignElems);  // slot stride keeps every slot 16B-aligned
      P.C = (uint32_t)((P.S + CH - 1) / CH);
      P.K = std::max(kmax, 1);
      P.rx_off = rxoff;
      rxoff = align_up(rxoff + 2 * (uint64_t)P.K * P.sl, kAlignElems);
      P.rxflag_off = rxfoff;
      rxfoff += (uint64_t)P.K * P.C;
      P.dflag = dflag;
      dflag += P.C;
      P.push_items = 0;
      P.items = P.C;
      int nc = tree_num_children(x->rank, N);
      P.down_items = (x->rank != 0 && nc > 0) ? P.C : 0;
      P.expected = x->rank == 0 ? 0 : P.C;
      P.grid = (int)std::min<uint64_t>(P.items, cap);
      P.down_grid = (int)std::min<uint64_t>(P.down_items, cap);
      uint64_t out_up = x->rank ? P.S : 0;
      P.nvlink_bytes = (out_up + (uint64_t)nc * P.S) * x->esz;
      P.hbm_bytes = ((uint64_t)nc + 1 + (x->rank == 0 ? 2 + (cfg->mode == PGX_MODE_FAST32 ? 2 : cfg->mode == PGX_MODE_SUM32 ? -1 : 0) : 0)) * P.S * x->esz;
    } else {
      delete x;
      return fail(PGX_E_CONFIG, "layer %d: unknown variant %d", l, P.variant);
    }
  }
  int rc;
  // model segment: flat weights + [arrival counters | tree down flags]
  x->ownerflag_base = dflag;
  dflag += (uint32_t)cfg->num_layers * N;  // TWOSHOT_CE per-(layer, owner) arrival flags
  rc = pgx_segment_create(w, x->seg_model, std::max<uint64_t>(moff, 1) * x->esz, dflag, &x->model, &x->mflags);
  if (rc) { delete x; return rc; }
  rc = pgx_segment_create(w, x->seg_rx, std::max<uint64_t>(rxoff, 1) * x->esz, (uint32_t)std::max<uint64_t>(rxfoff, 1),
                          &x->rx, &x->rxflags);
  if (rc) { delete x; return rc; }
  {
    int prev;
    cudaGetDevice(&prev);
    cudaSetDevice(x->dev);
    cudaError_t e = cudaSuccess;
    if (cfg->mode == PGX_MODE_FAST32) {
      e = cudaMalloc(&x->v, std::max<uint64_t>(moff, 1) * sizeof(float));
      if (e == cudaSuccess) e = cudaMemset(x->v, 0, std::max<uint64_t>(moff, 1) * sizeof(float));
    }
    if (e == cudaSuccess) e = cudaMalloc(&x->queues, (size_t)cfg->num_layers * 4 * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(x->queues, 0, (size_t)cfg->num_layers * 4 * sizeof(uint32_t));
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&x->down, cudaStreamNonBlocking, hi_prio);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&x->ce_rs, cudaStreamNonBlocking, hi_prio);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&x->ce_own, cudaStreamNonBlocking, hi_prio);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&x->ce_ag, cudaStreamNonBlocking, hi_prio);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&x->ce_rs2, cudaStreamNonBlocking, hi_prio);
    x->done.resize(cfg->num_layers);
    x->ready.resize(cfg->num_layers);
    x->rs_done.resize(cfg->num_layers);
    x->rs2_done.resize(cfg->num_layers);
    x->down_done.resize(cfg->num_layers);
    x->part_ev.resize(cfg->num_layers, std::vector<XEvent>(8));
    x->rs_part_ev.resize(cfg->num_layers, std::vector<XEvent>(8));
    for (int l = 0; l < cfg->num_layers && e == cudaSuccess; ++l) {
      e = cudaEventCreateWithFlags(&x->done[l].e, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x->ready[l].e, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x->rs_done[l].e, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x->down_done[l].e, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x->rs2_done[l].e, cudaEventDisableTiming);
      for (int p = 0; p < 8 && e == cudaSuccess; ++p) {
        e = cudaEventCreateWithFlags(&x->part_ev[l][p].e, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x->rs_part_ev[l][p].e, cudaEventDisableTiming);
      }
    }
    if (e == cudaSuccess) e = cudaMalloc(&x->iter_dev, sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(x->iter_dev, 0xFF, sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
      delete x;
      return fail(PGX_E_CUDA, "exchange allocation failed: %s", cudaGetErrorString(e));
    }
  }
  {  // whole-model gate table (all arrival flags live in this rank's own model segment)
    std::vector<GateEntry> ents;
    for (int l = 0; l < cfg->num_layers; ++l) {
      const LayerPlan& P = x->L[l];
      if (P.variant == PGX_VARIANT_TWOSHOT_CE) {
        for (int j = 0; j < N; ++j)
          if (j != x->rank) ents.push_back({x->mflags + x->ownerflag_base + (uint64_t)l * N + j, 1u});
      } else if (P.expected) {
        ents.push_back({x->mflags + l, P.expected});
      }
    }
    x->gate_entries = (int)ents.size();
    int prev;
    cudaGetDevice(&prev);
    cudaSetDevice(x->dev);
    cudaError_t e = cudaMalloc(&x->gate_table, std::max<size_t>(1, ents.size()) * sizeof(GateEntry));
    if (e == cudaSuccess && !ents.empty())
      e = cudaMemcpy(x->gate_table, ents.data(), ents.size() * sizeof(GateEntry), cudaMemcpyHostToDevice);
    cudaSetDevice(prev);
    if (e != cudaSuccess) return fail(PGX_E_CUDA, "gate table: %s", cudaGetErrorString(e));
  }
  *out = x;
  return PGX_OK;
}

int pgx_xchg_destroy(pgx_xchg* x) {
  if (!x) return PGX_OK;
  int prev;
  cudaGetDevice(&prev);
  cudaSetDevice(x->dev);
  cudaDeviceSynchronize();
  if (x->v) cudaFree(x->v);
  if (x->queues) cudaFree(x->queues);
  for (auto& e : x->done) cudaEventDestroy(e.e);
  for (auto& e : x->ready) cudaEventDestroy(e.e);
  for (auto& e : x->rs_done) cudaEventDestroy(e.e);
  for (auto& e : x->down_done) cudaEventDestroy(e.e);
  for (auto& e : x->rs2_done) cudaEventDestroy(e.e);
  for (auto& v : x->part_ev)
    for (auto& e : v) cudaEventDestroy(e.e);
  for (auto& v : x->rs_part_ev)
    for (auto& e : v) cudaEventDestroy(e.e);
  if (x->iter_dev) cudaFree(x->iter_dev);
  if (x->gate_table) cudaFree(x->gate_table);
  nvls_release(x);
  if (x->own_streams) {
    if (x->down) cudaStreamDestroy(x->down);
    if (x->ce_rs) cudaStreamDestroy(x->ce_rs);
    if (x->ce_own) cudaStreamDestroy(x->ce_own);
    if (x->ce_ag) cudaStreamDestroy(x->ce_ag);
    if (x->ce_rs2) cudaStreamDestroy(x->ce_rs2);
  }
  cudaSetDevice(prev);
  delete x;  // segments belong to the world
  return PGX_OK;
}

int pgx_xchg_model(pgx_xchg* x, void** model, uint64_t* offsets) {
  if (model) *model = x->model;
  if (offsets)
    for (size_t l = 0; l < x->L.size(); ++l) offsets[l] = x->L[l].model_off;
  return PGX_OK;
}

int pgx_xchg_connect(pgx_xchg* x) {
  for (int r = 0; r < x->world; ++r) {
    uint64_t sz;
    if (!world_seg(x->w, r, x->seg_model, &x->peer_model[r], &x->peer_mflags[r], &sz))
      return fail(PGX_E_ROUTING, "rank %d's model segment %u is not attached", r, x->seg_model);
    if (!world_seg(x->w, r, x->seg_rx, &x->peer_rx[r], &x->peer_rxflags[r], &sz))
      return fail(PGX_E_ROUTING, "rank %d's receive segment %u is not attached", r, x->seg_rx);
  }
  x->connected = true;
  return PGX_OK;
}

int pgx_xchg_layer(pgx_xchg* x, int l, uint32_t iteration, const void* const* pieces, const uint64_t* piece_elems,
                   int npieces, int phases, void* stream) {
  if (!x->connected) return fail(PGX_E_CONFIG, "exchange not connected");
  if (l < 0 || l >= (int)x->L.size()) return fail(PGX_E_RANGE, "layer %d outside 0..%d", l, (int)x->L.size() - 1);
  if (npieces < 1 || npieces > PGX_MAX_PIECES) return fail(PGX_E_SHAPE, "1..%d gradient pieces, got %d", PGX_MAX_PIECES, npieces);
  const LayerPlan& P = x->L[l];
  XArgs a = base_args(x, l, iteration);
  uint64_t tot = 0;
  for (int k = 0; k < npieces; ++k) {
    a.g.p[k] = pieces[k];
    tot += piece_elems[k];
    a.g.end[k] = tot;
  }
  a.g.n = npieces;
  if (tot != P.S)
    return fail(PGX_E_SHAPE, "layer %d gradient has %llu elements, layer needs %llu", l, (unsigned long long)tot,
                (unsigned long long)P.S);
  a.queue = x->queues + 4 * l;
  cudaStream_t s = (cudaStream_t)stream;
  int prev;
  cudaGetDevice(&prev);
  if (prev != x->dev) cudaSetDevice(x->dev);
  if (P.variant == PGX_VARIANT_ONESHOT_LL || P.variant == PGX_VARIANT_ONESHOT_L128) {
    xrecord(x->ready[l], s);
    a.item_begin = (phases & PGX_PHASE_PUSH) ? 0 : P.push_items;
    a.item_end = (phases & PGX_PHASE_OWNER) ? P.items : P.push_items;
    if (a.item_end > a.item_begin) {
      ++x->launches;
      const int want = (int)std::min<uint32_t>(a.item_end - a.item_begin, (uint32_t)P.grid);
      if (P.variant == PGX_VARIANT_ONESHOT_LL)
        launch_oneshot_ll(x->world, want, x->dev, s, a, P.lean ? kLeanThreads : kThreads);
      else
        launch_oneshot_l128(x->world, want, x->dev, s, a);
    }
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = xrecord(x->done[l], s);
    if (prev != x->dev) cudaSetDevice(prev);
    if (e != cudaSuccess) return fail(PGX_E_CUDA, "exchange launch failed: %s", cudaGetErrorString(e));
    return PGX_OK;
  }
  if (P.variant == PGX_VARIANT_TWOSHOT_L128) {
    // items: [0, push) reduce-scatter, [push, push + C) owner, [push + C, items) install
    xrecord(x->ready[l], s);
    const uint32_t own_end = P.push_items + P.Co;
    a.item_begin = (phases & PGX_PHASE_PUSH) ? 0 : (phases & PGX_PHASE_OWNER) ? P.push_items : own_end;
    a.item_end = (phases & PGX_PHASE_DOWN) ? P.items : (phases & PGX_PHASE_OWNER) ? own_end : P.push_items;
    if (a.item_end > a.item_begin) {
      ++x->launches;
      const int want = (int)std::min<uint32_t>(a.item_end - a.item_begin, (uint32_t)P.grid);
      launch_twoshot_l128(x->world, want, x->dev, s, a, P.lean ? kLeanThreads : kThreads);
    }
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = xrecord(x->done[l], s);
    if (prev != x->dev) cudaSetDevice(prev);
    if (e != cudaSuccess) return fail(PGX_E_CUDA, "exchange launch failed: %s", cudaGetErrorString(e));
    return PGX_OK;
  }
  if (P.variant == PGX_VARIANT_ONESHOT) {
    xrecord(x->ready[l], s);
    a.item_begin = (phases & PGX_PHASE_PUSH) ? 0 : P.push_items;
    a.item_end = (phases & PGX_PHASE_OWNER) ? P.items : P.push_items;
    if (a.item_end > a.item_begin) {
      ++x->launches;
      int grid = (int)std::min<uint32_t>(a.item_end - a.item_begin, (uint32_t)P.grid);
      if (x->esz == 8)
        launch_oneshot<double>(x->world, grid, x->dev, s, a);
      else
        launch_oneshot<float>(x->world, grid, x->dev, s, a);
    }
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = xrecord(x->done[l], s);
    if (prev != x->dev) cudaSetDevice(prev);
    if (e != cudaSuccess) return fail(PGX_E_CUDA, "exchange launch failed: %s", cudaGetErrorString(e));
    return PGX_OK;
  }
  if (P.variant == PGX_VARIANT_NVLS) {
    xrecord(x->ready[l], s);
    int rc = launch_nvls(x, l, P, a, s);
    if (rc == PGX_OK) xrecord(x->done[l], s);
    if (prev != x->dev) cudaSetDevice(prev);
    return rc;
  }
  if (P.variant == PGX_VARIANT_TWOSHOT_CEP) {
    int rc = launch_twoshot_cep(x, l, P, a, s, phases);
    if (prev != x->dev) cudaSetDevice(prev);
    return rc;
  }
  if (P.variant == PGX_VARIANT_TWOSHOT_CE) {
    int rc = launch_twoshot_ce(x, l, P, a, s, phases);
    if (prev != x->dev) cudaSetDevice(prev);
    return rc;
  }
  xrecord(x->ready[l], s);
  if (P.variant == PGX_VARIANT_TWOSHOT_BULK && x->bulk_ce_rs && x->world > 1) {
    const int rc = launch_bulk_ce_rs(x, l, P, a, phases);
    if (prev != x->dev) cudaSetDevice(prev);
    return rc;
  }
  if (P.variant == PGX_VARIANT_TWOSHOT_BULK) {
    a.item_begin = (phases & PGX_PHASE_PUSH) ? 0 : P.push_items;
    a.item_end = (phases & PGX_PHASE_OWNER) ? P.items : P.push_items;
    uint32_t n = a.item_end > a.item_begin ? a.item_end - a.item_begin : 0;
    if (n) {
      ++x->launches;
      int grid = (int)std::min<uint32_t>(n, (uint32_t)P.grid);
      launch_twoshot_bulk(x->world, grid, x->dev, s, a);
    }
  } else if (P.variant == PGX_VARIANT_TWOSHOT) {
    a.item_begin = (phases & PGX_PHASE_PUSH) ? 0 : P.push_items;
    a.item_end = (phases & PGX_PHASE_OWNER) ? P.items : P.push_items;
    uint32_t n = a.item_end > a.item_begin ? a.item_end - a.item_begin : 0;
    if (n) {
      ++x->launches;
      int grid = (int)std::min<uint32_t>(n, (uint32_t)P.grid);
      if (x->esz == 8)
        launch_twoshot<double>(x->world, x->tma, grid, x->dev, s, a);
      else
        launch_twoshot<float>(x->world, x->tma, grid, x->dev, s, a);
    }
  } else {
    if (phases & PGX_PHASE_PUSH) {
      ++x->launches;
      a.item_begin = 0;
      a.item_end = P.items;
      if (x->esz == 8)
        k_tree_up<double><<<P.grid, kThreads, 0, s>>>(a);
      else
        k_tree_up<float><<<P.grid, kThreads, 0, s>>>(a);
    }
    if (P.down_items && (phases & PGX_PHASE_DOWN)) {
      XArgs d = a;
      d.items = P.down_items;
      d.item_begin = 0;
      d.item_end = P.down_items;
      d.queue = a.queue + 2;
      // the down pass waits on the round trip: its own stream, so later layers'
      // up passes are not queued behind it (host-stepped callers pass PUSH and
      // DOWN separately and get the down pass on `stream`)
      cudaStream_t ds = (phases & PGX_PHASE_PUSH) ? x->down : s;
      ++x->launches;
      if (ds == x->down) xwait(x->down, x->ready[l]);
      if (x->esz == 8)
        k_tree_down<double><<<P.down_grid, kThreads, 0, ds>>>(d);
      else
        k_tree_down<float><<<P.down_grid, kThreads, 0, ds>>>(d);
      xrecord(x->down_done[l], ds);
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = xrecord(x->done[l], s);
  if (prev != x->dev) cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(PGX_E_CUDA, "exchange launch failed: %s", cudaGetErrorString(e));
  return PGX_OK;
}

int pgx_xchg_gate(pgx_xchg* x, int l, uint32_t iteration, void* stream) {
  if (l < 0 || l >= (int)x->L.size()) return fail(PGX_E_RANGE, "layer %d outside 0..%d", l, (int)x->L.size() - 1);
  const LayerPlan& P = x->L[l];
  cudaStream_t s = (cudaStream_t)stream;
  int prev;
  cudaGetDevice(&prev);
  if (prev != x->dev) cudaSetDevice(x->dev);
  cudaError_t e = xwait(s, x->done[l]);
  if (e == cudaSuccess) e = xwait(s, x->rs_done[l]);
  if (e == cudaSuccess) e = xwait(s, x->rs2_done[l]);
  if (e == cudaSuccess) e = xwait(s, x->down_done[l]);
  const uint32_t* it = x->device_iter ? x->iter_dev : nullptr;
  if (e == cudaSuccess && P.variant == PGX_VARIANT_TWOSHOT_CE) {
    FlagSet fs{};
    for (int j = 0; j < x->world; ++j)
      if (j != x->rank) fs.f[fs.n++] = x->mflags + x->ownerflag_base + (uint64_t)l * x->world + j;
    if (fs.n) {
      ++x->launches;
      k_wait_flags<<<1, 32, 0, s>>>(fs, iteration + 1, it, iteration + 1, world_status(x->w));
      e = cudaGetLastError();
    }
  } else if (e == cudaSuccess && P.expected) {
    ++x->launches;
    const uint32_t* counter = x->mflags + l;
    if (P.variant == PGX_VARIANT_NVLS)
      counter = reinterpret_cast<const uint32_t*>(x->nv.uc + x->nv.flag_off + x->nv.fl[l]);
    k_gate<<<1, 32, 0, s>>>(counter, (iteration + 1) * P.expected, it, iteration + 1, P.expected,
                            world_status(x->w));
    e = cudaGetLastError();
  }
  if (prev != x->dev) cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(PGX_E_CUDA, "gate failed: %s", cudaGetErrorString(e));
  return PGX_OK;
}

int pgx_xchg_device_iteration(pgx_xchg* x, int enable, uint32_t current) {
  int prev;
  cudaGetDevice(&prev);
  cudaSetDevice(x->dev);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(x->iter_dev, &current, sizeof(uint32_t), cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(PGX_E_CUDA, "device iteration: %s", cudaGetErrorString(e));
  x->device_iter = enable != 0;
  return PGX_OK;
}

int pgx_xchg_tick(pgx_xchg* x, void* stream) {
  if (!x->device_iter) return fail(PGX_E_CONFIG, "tick needs device-iteration mode");
  int prev;
  cudaGetDevice(&prev);
  if (prev != x->dev) cudaSetDevice(x->dev);
  k_tick<<<1, 1, 0, (cudaStream_t)stream>>>(x->iter_dev);
  ++x->launches;
  cudaError_t e = cudaGetLastError();
  if (prev != x->dev) cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(PGX_E_CUDA, "tick: %s", cudaGetErrorString(e));
  return PGX_OK;
}

int pgx_xchg_set_streams(pgx_xchg* x, void* const* streams, int n) {
  if (n != PGX_XCHG_STREAMS) return fail(PGX_E_CONFIG, "%d streams required, got %d", PGX_XCHG_STREAMS, n);
  for (int i = 0; i < n; ++i)
    if (!streams[i]) return fail(PGX_E_CONFIG, "stream %d is null", i);
  int prev;
  cudaGetDevice(&prev);
  cudaSetDevice(x->dev);
  cudaDeviceSynchronize();
  if (x->own_streams) {
    cudaStreamDestroy(x->down);
    cudaStreamDestroy(x->ce_rs);
    cudaStreamDestroy(x->ce_own);
    cudaStreamDestroy(x->ce_ag);
    cudaStreamDestroy(x->ce_rs2);
  }
  cudaSetDevice(prev);
  x->down = (cudaStream_t)streams[0];
  x->ce_rs = (cudaStream_t)streams[1];
  x->ce_own = (cudaStream_t)streams[2];
  x->ce_ag = (cudaStream_t)streams[3];
  x->ce_rs2 = (cudaStream_t)streams[4];
  x->own_streams = false;
  return PGX_OK;
}

int pgx_xchg_stream(pgx_xchg* x, int which, void** out) {
  cudaStream_t st[PGX_XCHG_STREAMS] = {x->down, x->ce_rs, x->ce_own, x->ce_ag, x->ce_rs2};
  if (which < 0 || which >= PGX_XCHG_STREAMS)
    return fail(PGX_E_RANGE, "stream index %d outside 0..%d", which, PGX_XCHG_STREAMS - 1);
  *out = st[which];
  return PGX_OK;
}

int pgx_xchg_join(pgx_xchg* x, int l, void* stream) {
  if (l < 0 || l >= (int)x->L.size()) return fail(PGX_E_RANGE, "layer %d outside 0..%d", l, (int)x->L.size() - 1);
  PGX_CUDA(xwait((cudaStream_t)stream, x->done[l]));
  PGX_CUDA(xwait((cudaStream_t)stream, x->rs_done[l]));
  PGX_CUDA(xwait((cudaStream_t)stream, x->rs2_done[l]));
  PGX_CUDA(xwait((cudaStream_t)stream, x->down_done[l]));
  return PGX_OK;
}

int pgx_xchg_launch_count(pgx_xchg* x, uint64_t* n) {
  *n = x->launches;
  return PGX_OK;
}

int pgx_xchg_gate_all(pgx_xchg* x, uint32_t iteration, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int prev;
  cudaGetDevice(&prev);
  if (prev != x->dev) cudaSetDevice(x->dev);
  cudaError_t e = cudaSuccess;
  for (size_t l = 0; l < x->L.size() && e == cudaSuccess; ++l) {
    e = xwait(s, x->done[l]);
    if (e == cudaSuccess) e = xwait(s, x->rs_done[l]);
    if (e == cudaSuccess) e = xwait(s, x->rs2_done[l]);
    if (e == cudaSuccess) e = xwait(s, x->down_done[l]);
  }
  if (e == cudaSuccess && x->gate_entries) {
    ++x->launches;
    k_gate_all<<<1, 256, 0, s>>>(x->gate_table, x->gate_entries, iteration + 1,
                                  x->device_iter ? x->iter_dev : nullptr, iteration + 1, world_status(x->w));
    e = cudaGetLastError();
  }
  if (prev != x->dev) cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(PGX_E_CUDA, "gate_all failed: %s", cudaGetErrorString(e));
  return PGX_OK;
}

int pgx_xchg_layer_bytes(pgx_xchg* x, int l, uint64_t* nvl, uint64_t* hbm) {
  if (l < 0 || l >= (int)x->L.size()) return fail(PGX_E_RANGE, "layer %d outside 0..%d", l, (int)x->L.size() - 1);
  if (nvl) *nvl = x->L[l].nvlink_bytes;
  if (hbm) *hbm = x->L[l].hbm_bytes;
  return PGX_OK;
}

int pgx_xchg_layer_parts(pgx_xchg* x, int l, int* parts) {
  if (l < 0 || l >= (int)x->L.size()) return fail(PGX_E_RANGE, "layer %d outside 0..%d", l, (int)x->L.size() - 1);
  *parts = x->L[l].variant == PGX_VARIANT_TWOSHOT_CE ? ce_split(x, x->L[l], x->rank, 0, nullptr, nullptr) : 1;
  return PGX_OK;
}

int pgx_xchg_set_trace(pgx_xchg* x, void* device_buffer) {
  x->trace = static_cast<unsigned long long*>(device_buffer);
  return PGX_OK;
}

int pgx_graph_instantiate_prio(void* graph, void** exec_out) {
  if (!graph || !exec_out) return fail(PGX_E_CONFIG, "graph and exec_out must be non-null");
  cudaGraphExec_t ex = nullptr;
  cudaError_t e = cudaGraphInstantiateWithFlags(&ex, static_cast<cudaGraph_t>(graph), cudaGraphInstantiateFlagUseNodePriority);
  if (e != cudaSuccess) return fail(PGX_E_CUDA, "cudaGraphInstantiateWithFlags: %s", cudaGetErrorString(e));
  *exec_out = ex;
  return PGX_OK;
}

int pgx_graph_launch(void* exec, void* stream) {
  cudaError_t e = cudaGraphLaunch(static_cast<cudaGraphExec_t>(exec), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(PGX_E_CUDA, "cudaGraphLaunch: %s", cudaGetErrorString(e));
  return PGX_OK;
}

int pgx_graph_exec_destroy(void* exec) {
  cudaError_t e = cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(exec));
  if (e != cudaSuccess) return fail(PGX_E_CUDA, "cudaGraphExecDestroy: %s", cudaGetErrorString(e));
  return PGX_OK;
}

int pgx_xchg_layer_plan(pgx_xchg* x, int l, uint64_t* chunk_elems, int* ctas) {
  if (l < 0 || l >= (int)x->L.size()) return fail(PGX_E_RANGE, "layer %d outside 0..%d", l, (int)x->L.size() - 1);
  if (chunk_elems) *chunk_elems = x->L[l].CH;
  if (ctas) *ctas = x->L[l].grid;
  return PGX_OK;
}

}  // extern "C"
