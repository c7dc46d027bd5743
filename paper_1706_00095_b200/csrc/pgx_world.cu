// World, segments, one-sided notify-writes, notifications, tickets, barrier.
//
// Replaces the reference's transport layer (transport/base.py:129-225,
// transport/inproc.py:62-149) for ranks that are GPUs of one NVSwitch box:
// a Segment is one cudaMalloc'ed block [data | pad | u32 notification flags],
// IPC-exported so every peer maps it and writes into it with ordinary device
// stores over NVLink.  A notification is a u32 flag raised with a system-scope
// release after the payload; polling reads the flags, reset consumes them.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#include <map>
#include <mutex>
#include <string>

#include "pgx_common.cuh"

namespace pgx {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

}  // namespace pgx

using namespace pgx;

struct SegRec {
  void* data = nullptr;
  uint32_t* flags = nullptr;
  uint64_t size = 0;
  uint32_t count = 0;
  bool owned = false;   // allocated by this world
  bool ipc = false;     // opened via cudaIpcOpenMemHandle
  void* base = nullptr; // allocation base (owned or ipc-opened)
};

struct pgx_world {
  int rank = 0, world = 1, device = 0;
  std::map<uint32_t, SegRec> segs[PGX_MAX_RANKS];
  uint32_t* status_host = nullptr;  // host-mapped
  uint32_t* status_dev = nullptr;
  uint64_t timeout_ns = 30ull * 1000000000ull;  // finalize_timeout_s default, config.py:33
  uint32_t barrier_epoch = 0;
  cudaStream_t aux = nullptr;       // private stream for synchronous host ops
  uint32_t* pinned = nullptr;       // small pinned scratch
  std::mutex mu;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

inline uint64_t flags_offset(uint64_t size) { return (size + 255) & ~uint64_t(255); }

SegRec* find_seg(pgx_world* w, int rank, uint32_t id) {
  if (rank < 0 || rank >= w->world) return nullptr;
  auto it = w->segs[rank].find(id);
  return it == w->segs[rank].end() ? nullptr : &it->second;
}

// ------------------------------------------------------------------ kernels
// Byte-exact copy of one chunk by one CTA: 16-byte vector body when source and
// destination share alignment, scalar head/tail otherwise.
__device__ __forceinline__ void cta_copy(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                         uint64_t n) {
  const uint32_t tid = threadIdx.x, nt = blockDim.x;
  const uintptr_t sa = reinterpret_cast<uintptr_t>(src) & 15, da = reinterpret_cast<uintptr_t>(dst) & 15;
  if (sa == da && n >= 32) {
    uint64_t head = (16 - sa) & 15;
    if (tid < head) dst[tid] = src[tid];
    const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
    uint4* d4 = reinterpret_cast<uint4*>(dst + head);
    uint64_t nv = (n - head) >> 4;
    uint64_t i = tid;
    // 4 independent 16-byte loads in flight per thread before the stores
    for (; i + 3 * nt < nv; i += 4 * nt) {
      uint4 a = __ldcg(s4 + i), b = __ldcg(s4 + i + nt), c = __ldcg(s4 + i + 2 * nt),
            d = __ldcg(s4 + i + 3 * nt);
      d4[i] = a;
      d4[i + nt] = b;
      d4[i + 2 * nt] = c;
      d4[i + 3 * nt] = d;
    }
    for (; i < nv; i += nt) d4[i] = __ldcg(s4 + i);
    uint64_t done = head + (nv << 4);
    for (uint64_t j = done + tid; j < n; j += nt) dst[j] = src[j];
  } else {
    for (uint64_t j = tid; j < n; j += nt) dst[j] = src[j];
  }
}

// Chunk j of a transfer raises id chunk_notification_id(base, j, n)
// (engine/layout.py:130-139): the final chunk carries base, earlier base+1+j.
__global__ void k_put_chunked(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                              uint64_t total, uint64_t chunk, uint32_t nchunks,
                              uint32_t* __restrict__ flags, uint32_t base_id, uint32_t value) {
  for (uint32_t j = blockIdx.x; j < nchunks; j += gridDim.x) {
    uint64_t off = (uint64_t)j * chunk;
    uint64_t n = total - off < chunk ? total - off : chunk;
    cta_copy(src + off, dst + off, n);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t nid = (j == nchunks - 1) ? base_id : base_id + 1 + j;
      fence_acq_rel_sys();
      st_release_sys(flags + nid, value);
    }
  }
}

__global__ void k_reset_flag(uint32_t* flags, uint32_t nid, uint32_t* out) {
  *out = atomicExch(flags + nid, 0u);
}

// Device flag barrier: rank r raises ctrl[r] = epoch on every peer, then waits
// until its own ctrl[j] >= epoch for all j.
struct BarrierArgs {
  uint32_t* peer_ctrl[PGX_MAX_RANKS];
};
__global__ void k_barrier(BarrierArgs a, uint32_t* own_ctrl, int rank, int world, uint32_t epoch,
                          Status st) {
  int j = threadIdx.x;
  if (j < world && j != rank) {
    fence_acq_rel_sys();
    st_release_sys(a.peer_ctrl[j] + rank, epoch);
  }
  __syncwarp();
  if (j < world && j != rank) wait_geq(own_ctrl + j, epoch, st);
}

}  // namespace

extern "C" {

int pgx_abi_version(void) { return PGX_ABI_VERSION; }
const char* pgx_last_error(void) { return pgx::g_err; }

int pgx_world_create(int rank, int world_size, int device, pgx_world** out) {
  if (world_size < 1 || world_size > PGX_MAX_RANKS)
    return fail(PGX_E_CONFIG, "world size must be in 1..%d, got %d", PGX_MAX_RANKS, world_size);
  if (rank < 0 || rank >= world_size)
    return fail(PGX_E_CONFIG, "rank %d outside world of size %d", rank, world_size);
  int ndev = 0;
  PGX_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(PGX_E_CONFIG, "device %d outside 0..%d", device, ndev - 1);
  DeviceGuard g(device);
  pgx_world* w = new pgx_world();
  w->rank = rank;
  w->world = world_size;
  w->device = device;
  cudaError_t e = cudaHostAlloc(&w->status_host, 4096, cudaHostAllocMapped);
  if (e != cudaSuccess) {
    delete w;
    return fail(PGX_E_CUDA, "cudaHostAlloc: %s", cudaGetErrorString(e));
  }
  memset(w->status_host, 0, 4096);
  w->pinned = w->status_host + 64;
  PGX_CUDA(cudaHostGetDevicePointer(&w->status_dev, w->status_host, 0));
  PGX_CUDA(cudaStreamCreateWithFlags(&w->aux, cudaStreamNonBlocking));
  *out = w;
  // The control segment (transport/base.py:21) backs the device barrier.
  void* d;
  uint32_t* f;
  int rc = pgx_segment_create(w, PGX_CONTROL_SEGMENT, 256, PGX_MAX_RANKS, &d, &f);
  return rc;
}

int pgx_world_destroy(pgx_world* w) {
  if (!w) return PGX_OK;
  DeviceGuard g(w->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < w->world; ++r)
    for (auto& kv : w->segs[r]) {
      if (kv.second.ipc) cudaIpcCloseMemHandle(kv.second.base);
      if (kv.second.owned) cudaFree(kv.second.base);
    }
  if (w->aux) cudaStreamDestroy(w->aux);
  if (w->status_host) cudaFreeHost(w->status_host);
  delete w;
  return PGX_OK;
}

int pgx_enable_peer_access(int device, int peer) {
  DeviceGuard g(device);
  int can = 0;
  PGX_CUDA(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) return fail(PGX_E_ROUTING, "device %d cannot access device %d", device, peer);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return PGX_OK;
  }
  if (e != cudaSuccess) return fail(PGX_E_CUDA, "cudaDeviceEnablePeerAccess: %s", cudaGetErrorString(e));
  return PGX_OK;
}

int pgx_world_status(pgx_world* w, uint32_t* s) {
  *s = *(volatile uint32_t*)w->status_host;
  return PGX_OK;
}
int pgx_world_clear_status(pgx_world* w) {
  *(volatile uint32_t*)w->status_host = 0;
  return PGX_OK;
}
int pgx_world_set_timeout(pgx_world* w, double seconds) {
  if (!(seconds >= 0)) return fail(PGX_E_CONFIG, "timeout must be >= 0");
  w->timeout_ns = (uint64_t)(seconds * 1e9);
  return PGX_OK;
}

int pgx_segment_create(pgx_world* w, uint32_t id, uint64_t size, uint32_t count, void** data,
                       uint32_t** flags) {
  if (id >= 65536) return fail(PGX_E_CONFIG, "segment id %u outside u16 range", id);
  if (size < 1) return fail(PGX_E_CONFIG, "segment size must be >= 1, got %llu", (unsigned long long)size);
  if (count < 1) return fail(PGX_E_CONFIG, "notification count must be >= 1, got %u", count);
  std::lock_guard<std::mutex> lk(w->mu);
  if (w->segs[w->rank].count(id))
    return fail(PGX_E_CONFIG, "segment %u already exists on rank %d", id, w->rank);
  DeviceGuard g(w->device);
  uint64_t fo = flags_offset(size);
  uint64_t bytes = fo + (uint64_t)count * 4;
  void* base = nullptr;
  PGX_CUDA(cudaMalloc(&base, bytes));
  PGX_CUDA(cudaMemset(base, 0, bytes));
  PGX_CUDA(cudaDeviceSynchronize());
  SegRec s;
  s.base = s.data = base;
  s.flags = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(base) + fo);
  s.size = size;
  s.count = count;
  s.owned = true;
  w->segs[w->rank][id] = s;
  if (data) *data = s.data;
  if (flags) *flags = s.flags;
  return PGX_OK;
}

int pgx_segment_info(pgx_world* w, int rank, uint32_t id, void** data, uint32_t** flags,
                     uint64_t* size, uint32_t* count) {
  if (rank < 0 || rank >= w->world)
    return fail(PGX_E_ROUTING, "rank %d outside world of size %d", rank, w->world);
  SegRec* s = find_seg(w, rank, id);
  if (!s) {
    if (rank == w->rank) return fail(PGX_E_CONFIG, "segment %u does not exist on rank %d", id, rank);
    return fail(PGX_E_ROUTING, "rank %d has no segment %u attached", rank, id);
  }
  if (data) *data = s->data;
  if (flags) *flags = s->flags;
  if (size) *size = s->size;
  if (count) *count = s->count;
  return PGX_OK;
}

int pgx_segment_export(pgx_world* w, uint32_t id, void* handle) {
  SegRec* s = find_seg(w, w->rank, id);
  if (!s) return fail(PGX_E_CONFIG, "segment %u does not exist on rank %d", id, w->rank);
  DeviceGuard g(w->device);
  cudaIpcMemHandle_t h;
  PGX_CUDA(cudaIpcGetMemHandle(&h, s->base));
  static_assert(sizeof(h) == PGX_IPC_HANDLE_BYTES, "ipc handle size");
  memcpy(handle, &h, sizeof(h));
  return PGX_OK;
}

int pgx_segment_attach_ipc(pgx_world* w, int peer, uint32_t id, const void* handle, uint64_t size,
                           uint32_t count) {
  if (peer < 0 || peer >= w->world || peer == w->rank)
    return fail(PGX_E_ROUTING, "cannot attach rank %d's segment on rank %d", peer, w->rank);
  std::lock_guard<std::mutex> lk(w->mu);
  if (w->segs[peer].count(id)) return fail(PGX_E_CONFIG, "segment %u of rank %d already attached", id, peer);
  DeviceGuard g(w->device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  PGX_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  SegRec s;
  s.base = s.data = base;
  s.flags = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(base) + flags_offset(size));
  s.size = size;
  s.count = count;
  s.ipc = true;
  w->segs[peer][id] = s;
  return PGX_OK;
}

int pgx_segment_attach_local(pgx_world* w, int peer, uint32_t id, void* data, uint32_t* flags,
                             uint64_t size, uint32_t count) {
  if (peer < 0 || peer >= w->world || peer == w->rank)
    return fail(PGX_E_ROUTING, "cannot attach rank %d's segment on rank %d", peer, w->rank);
  std::lock_guard<std::mutex> lk(w->mu);
  if (w->segs[peer].count(id)) return fail(PGX_E_CONFIG, "segment %u of rank %d already attached", id, peer);
  SegRec s;
  s.base = s.data = data;
  s.flags = flags;
  s.size = size;
  s.count = count;
  w->segs[peer][id] = s;
  return PGX_OK;
}

int pgx_write_notify_chunked(pgx_world* w, uint32_t lseg, uint64_t loff, int rank, uint32_t rseg,
                             uint64_t roff, uint64_t size, uint64_t chunk, uint32_t base_id,
                             uint32_t value, void* stream) {
  // _validate_request (transport/base.py:217-225)
  if (value == 0) return fail(PGX_E_PROTOCOL, "notification value 0 is reserved; use values >= 1");
  SegRec* src = find_seg(w, w->rank, lseg);
  if (!src) return fail(PGX_E_CONFIG, "segment %u does not exist on rank %d", lseg, w->rank);
  if (loff + size > src->size || loff > src->size)
    return fail(PGX_E_RANGE, "range [%llu, %llu) outside segment %u of size %llu", (unsigned long long)loff,
                (unsigned long long)(loff + size), lseg, (unsigned long long)src->size);
  if (rank < 0 || rank >= w->world) return fail(PGX_E_ROUTING, "rank %d outside world of size %d", rank, w->world);
  SegRec* dst = find_seg(w, rank, rseg);
  if (!dst) return fail(PGX_E_ROUTING, "rank %d has no segment %u", rank, rseg);
  if (roff + size > dst->size || roff > dst->size)
    return fail(PGX_E_RANGE, "range [%llu, %llu) outside segment %u of size %llu", (unsigned long long)roff,
                (unsigned long long)(roff + size), rseg, (unsigned long long)dst->size);
  if (chunk == 0) return fail(PGX_E_CONFIG, "chunk_bytes must be positive");
  uint64_t n = size == 0 ? 1 : (size + chunk - 1) / chunk;
  uint32_t last_id = n == 1 ? base_id : base_id + (uint32_t)n - 1;
  if (base_id >= dst->count || last_id >= dst->count)
    return fail(PGX_E_RANGE, "notification id %u outside 0..%u", last_id > base_id ? last_id : base_id,
                dst->count - 1);
  DeviceGuard g(w->device);
  int grid = (int)(n < 1024 ? n : 1024);
  k_put_chunked<<<grid, 256, 0, (cudaStream_t)stream>>>(
      static_cast<const uint8_t*>(src->data) + loff, static_cast<uint8_t*>(dst->data) + roff, size,
      size == 0 ? 1 : chunk, (uint32_t)n, dst->flags, base_id, value);
  PGX_LAUNCH_CHECK();
  return PGX_OK;
}

int pgx_write_notify(pgx_world* w, uint32_t lseg, uint64_t loff, int rank, uint32_t rseg, uint64_t roff,
                     uint64_t size, uint32_t nid, uint32_t value, void* stream) {
  uint64_t chunk = size > 0 ? size : 1;
  return pgx_write_notify_chunked(w, lseg, loff, rank, rseg, roff, size, chunk, nid, value, stream);
}

int pgx_notify_poll(pgx_world* w, uint32_t id, uint32_t first, uint32_t count, uint32_t* ids,
                    uint32_t* vals, uint32_t cap, uint32_t* n_out) {
  SegRec* s = find_seg(w, w->rank, id);
  if (!s) return fail(PGX_E_CONFIG, "segment %u does not exist on rank %d", id, w->rank);
  if ((uint64_t)first + count > s->count)
    return fail(PGX_E_RANGE, "poll range [%u, %llu) outside 0..%u", first, (unsigned long long)first + count,
                s->count - 1);
  *n_out = 0;
  if (count == 0) return PGX_OK;
  DeviceGuard g(w->device);
  // Host snapshot of the flag words (one D2H copy), then a sparse scan.
  static thread_local uint32_t* buf = nullptr;
  static thread_local uint32_t buf_cap = 0;
  if (buf_cap < count) {
    if (buf) cudaFreeHost(buf);
    buf_cap = count < 4096 ? 4096 : count;
    PGX_CUDA(cudaMallocHost(&buf, (size_t)buf_cap * 4));
  }
  PGX_CUDA(cudaMemcpyAsync(buf, s->flags + first, (size_t)count * 4, cudaMemcpyDeviceToHost, w->aux));
  PGX_CUDA(cudaStreamSynchronize(w->aux));
  uint32_t n = 0;
  for (uint32_t i = 0; i < count; ++i) {
    if (buf[i]) {
      if (n < cap) {
        ids[n] = first + i;
        vals[n] = buf[i];
      }
      ++n;
    }
  }
  *n_out = n;
  if (n > cap) return fail(PGX_E_RANGE, "poll found %u notifications, capacity %u", n, cap);
  return PGX_OK;
}

int pgx_notify_reset(pgx_world* w, uint32_t id, uint32_t nid, uint32_t* old) {
  SegRec* s = find_seg(w, w->rank, id);
  if (!s) return fail(PGX_E_CONFIG, "segment %u does not exist on rank %d", id, w->rank);
  if (nid >= s->count) return fail(PGX_E_RANGE, "notification id %u outside 0..%u", nid, s->count - 1);
  DeviceGuard g(w->device);
  uint32_t* out_dev;
  PGX_CUDA(cudaHostGetDevicePointer(&out_dev, w->pinned, 0));
  k_reset_flag<<<1, 1, 0, w->aux>>>(s->flags, nid, out_dev);
  PGX_LAUNCH_CHECK();
  PGX_CUDA(cudaStreamSynchronize(w->aux));
  *old = *(volatile uint32_t*)w->pinned;
  return PGX_OK;
}

int pgx_ticket_record(void* stream, void** out) {
  cudaEvent_t ev;
  PGX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  PGX_CUDA(cudaEventRecord(ev, (cudaStream_t)stream));
  *out = ev;
  return PGX_OK;
}

int pgx_ticket_query(void* t) {
  cudaError_t e = cudaEventQuery((cudaEvent_t)t);
  if (e == cudaSuccess) return 1;
  if (e == cudaErrorNotReady) return 0;
  return -fail(PGX_E_CUDA, "ticket failed: %s", cudaGetErrorString(e));
}

int pgx_ticket_wait(void* t, double timeout_s) {
  struct timespec t0, now;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  while (true) {
    cudaError_t e = cudaEventQuery((cudaEvent_t)t);
    if (e == cudaSuccess) return PGX_OK;
    if (e != cudaErrorNotReady) return fail(PGX_E_TRANSPORT, "write failed: %s", cudaGetErrorString(e));
    clock_gettime(CLOCK_MONOTONIC, &now);
    double dt = (now.tv_sec - t0.tv_sec) + 1e-9 * (now.tv_nsec - t0.tv_nsec);
    if (timeout_s >= 0 && dt > timeout_s)
      return fail(PGX_E_TIMEOUT, "write did not complete within %g s", timeout_s);
    usleep(5);
  }
}

int pgx_ticket_release(void* t) {
  PGX_CUDA(cudaEventDestroy((cudaEvent_t)t));
  return PGX_OK;
}

static int launch_barrier(pgx_world* w, void* stream, double timeout_s);

int pgx_barrier(pgx_world* w, void* stream, double timeout_s) {
  if (w->world == 1) return PGX_OK;
  int rc = launch_barrier(w, stream, timeout_s);
  if (rc) return rc;
  PGX_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  if (*(volatile uint32_t*)w->status_host)
    return fail(PGX_E_TIMEOUT, "barrier did not complete within %g s", timeout_s);
  return PGX_OK;
}

int pgx_barrier_async(pgx_world* w, void* stream, double timeout_s) {
  if (w->world == 1) return PGX_OK;
  return launch_barrier(w, stream, timeout_s);
}

static int launch_barrier(pgx_world* w, void* stream, double timeout_s) {
  BarrierArgs a;
  for (int j = 0; j < w->world; ++j) {
    SegRec* s = find_seg(w, j, PGX_CONTROL_SEGMENT);
    if (!s) return fail(PGX_E_ROUTING, "rank %d's control segment is not attached", j);
    a.peer_ctrl[j] = s->flags;
  }
  uint32_t epoch = ++w->barrier_epoch;
  Status st{w->status_dev, (uint64_t)(timeout_s * 1e9)};
  DeviceGuard g(w->device);
  k_barrier<<<1, 32, 0, (cudaStream_t)stream>>>(a, a.peer_ctrl[w->rank], w->rank, w->world, epoch, st);
  PGX_LAUNCH_CHECK();
  return PGX_OK;
}

}  // extern "C"

// Accessors used by the other translation units.
namespace pgx {
int world_rank(pgx_world* w) { return w->rank; }
int world_size(pgx_world* w) { return w->world; }
int world_device(pgx_world* w) { return w->device; }
Status world_status(pgx_world* w) { return Status{w->status_dev, w->timeout_ns}; }
uint32_t* world_status_host(pgx_world* w) { return w->status_host; }
bool world_seg(pgx_world* w, int rank, uint32_t id, void** data, uint32_t** flags, uint64_t* size) {
  SegRec* s = find_seg(w, rank, id);
  if (!s) return false;
  *data = s->data;
  *flags = s->flags;
  if (size) *size = s->size;
  return true;
}
}  // namespace pgx
