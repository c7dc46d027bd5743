// PSGD1 model checkpoints (engine/checkpoint.py:1-71) built and read on the device.
//
// Image (little-endian): "PSGD1", then per layer l: u32 l, u64 count, count x f64.
// Layer l's header starts at off[l] = 5 + sum_{i<l} (12 + 8 n_i), so every value
// sits at an odd byte offset: the pack kernel assembles each ALIGNED 16-byte output
// pair from the three values it straddles (funnel shifts) and writes it with one
// 128-bit store, so a launch is a single coalesced HBM stream (read n*esz, write
// 8n bytes); only pairs touching a header or the magic are built byte by byte.
// Unpack is the mirror: each value is read from its two aligned image words.
// fp32 layers are promoted exactly to f64 on the way out (the reference
// serializes np.asarray(values, "<f8")) and rounded to nearest on the way in.
// Header validation (pgx_ckpt_parse) is host code over the file bytes, with the
// reference's FormatError messages.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "pgx_common.cuh"

using namespace pgx;

namespace {

constexpr int kMaxLayers = PGX_CKPT_MAX_LAYERS;
constexpr int kThreads = 256;

struct CkptTable {                // kernel parameter (< 32 KB): up to kMaxLayers layers
  const void* p[kMaxLayers];      // layer data: source (pack) or destination (unpack)
  uint64_t off[kMaxLayers + 1];   // byte offset of layer l's header; off[L] = image bytes
  uint64_t cum[kMaxLayers + 1];   // cumulative element counts
  int L;
  int esz;
};

// The same table in device memory, for checkpoints of more layers (the PSGD1 format has no
// layer limit, checkpoint.py:29-39); the kernels are templates over the two.
struct CkptDevTable {
  const void* const* p;
  const uint64_t* off;
  const uint64_t* cum;
  int L;
  int esz;
};

__device__ __forceinline__ int find_layer(const uint64_t* a, int L, uint64_t x) {
  // largest l in [0, L) with a[l] <= x (a ascending, a[0] <= x)
  int lo = 0, hi = L - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (a[mid] <= x)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

template <class Tab>
__device__ __forceinline__ uint64_t value_bits(const Tab& t, int l, uint64_t k) {
  if (t.esz == 8) return (uint64_t)__double_as_longlong(static_cast<const double*>(t.p[l])[k]);
  return (uint64_t)__double_as_longlong((double)static_cast<const float*>(t.p[l])[k]);
}

template <class Tab>
__device__ uint8_t image_byte(const Tab& t, uint64_t pos) {
  if (pos < 5) return (uint8_t)("PSGD1"[pos]);
  int l = find_layer(t.off, t.L, pos);
  uint64_t r = pos - t.off[l];
  if (r < 4) return (uint8_t)((uint32_t)l >> (8 * r));
  if (r < 12) return (uint8_t)((t.cum[l + 1] - t.cum[l]) >> (8 * (r - 4)));
  r -= 12;
  return (uint8_t)(value_bits(t, l, r >> 3) >> (8 * (r & 7)));
}

// One thread = one aligned 16-byte output pair (one 128-bit store).
template <class Tab>
__global__ void __launch_bounds__(kThreads) k_ckpt_pack(const __grid_constant__ Tab t, uint4* __restrict__ img,
                                                        uint64_t pairs) {
  const uint64_t bytes = t.off[t.L];
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < pairs; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p0 = q * 16;
    uint64_t w0 = 0, w1 = 0;
    bool done = false;
    if (t.L > 0 && p0 >= t.off[0]) {
      const int l = find_layer(t.off, t.L, p0);
      const uint64_t d = t.off[l] + 12;  // first value byte of layer l
      if (p0 >= d && p0 + 16 <= t.off[l + 1]) {
        const uint64_t rel = p0 - d, k = rel >> 3;
        const int m = (int)(rel & 7);  // the same for every word of the layer
        const uint64_t a = value_bits(t, l, k), b = value_bits(t, l, k + 1);
        if (m) {
          const uint64_t c = value_bits(t, l, k + 2);
          w0 = (a >> (8 * m)) | (b << (64 - 8 * m));
          w1 = (b >> (8 * m)) | (c << (64 - 8 * m));
        } else {
          w0 = a;
          w1 = b;
        }
        done = true;
      }
    }
    if (!done) {  // touches the magic, a header, a layer edge or the padding
      for (int b = 0; b < 8; ++b) {
        if (p0 + b < bytes) w0 |= (uint64_t)image_byte(t, p0 + b) << (8 * b);
        if (p0 + 8 + b < bytes) w1 |= (uint64_t)image_byte(t, p0 + 8 + b) << (8 * b);
      }
    }
    img[q] = make_uint4((uint32_t)w0, (uint32_t)(w0 >> 32), (uint32_t)w1, (uint32_t)(w1 >> 32));
  }
}

template <class Tab>
__global__ void __launch_bounds__(kThreads) k_ckpt_unpack(const __grid_constant__ Tab t,
                                                          const uint64_t* __restrict__ img) {
  const uint64_t total = t.cum[t.L];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const int l = find_layer(t.cum, t.L, i);  // the largest such l skips empty layers
    const uint64_t k = i - t.cum[l];
    const uint64_t pos = t.off[l] + 12 + 8 * k;
    const int m = (int)(pos & 7);
    uint64_t bits = img[pos >> 3] >> (8 * m);
    if (m) bits |= img[(pos >> 3) + 1] << (64 - 8 * m);
    const double v = __longlong_as_double((long long)bits);
    if (t.esz == 8)
      static_cast<double*>(const_cast<void*>(t.p[l]))[k] = v;
    else
      static_cast<float*>(const_cast<void*>(t.p[l]))[k] = __double2float_rn(v);
  }
}

// Host copy of a table of any size: per-layer pointers, header offsets, cumulative counts.
struct HostTable {
  std::vector<const void*> p;
  std::vector<uint64_t> off, cum;
};

int build_host_table(HostTable& h, const void* const* layers, const uint64_t* counts, int L, int esz) {
  if (L < 0) return fail(PGX_E_CONFIG, "negative checkpoint layer count %d", L);
  if (esz != 4 && esz != 8) return fail(PGX_E_CONFIG, "element size %d is not 4 or 8", esz);
  h.p.assign(std::max(L, 1), nullptr);
  h.off.assign(L + 1, 5);
  h.cum.assign(L + 1, 0);
  for (int l = 0; l < L; ++l) {
    if (counts[l] && !layers[l]) return fail(PGX_E_INPUT, "layer %d has no data pointer", l);
    h.p[l] = layers[l];
    h.off[l + 1] = h.off[l] + 12 + 8 * counts[l];
    h.cum[l + 1] = h.cum[l] + counts[l];
  }
  return PGX_OK;
}

// Stream-ordered device copy of a large table: [p | off | cum] in one allocation, freed
// behind the launch on the same stream.
int upload_table(const HostTable& h, int L, int esz, cudaStream_t s, CkptDevTable* out, void** mem) {
  const size_t np = h.p.size() * sizeof(void*), no = h.off.size() * sizeof(uint64_t);
  std::vector<uint8_t> buf(np + 2 * no);
  memcpy(buf.data(), h.p.data(), np);
  memcpy(buf.data() + np, h.off.data(), no);
  memcpy(buf.data() + np + no, h.cum.data(), no);
  cudaError_t e = cudaMallocAsync(mem, buf.size(), s);
  // pageable source: the copy is staged before cudaMemcpyAsync returns, so `buf` may go
  if (e == cudaSuccess) e = cudaMemcpyAsync(*mem, buf.data(), buf.size(), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return fail(PGX_E_CUDA, "checkpoint table upload: %s", cudaGetErrorString(e));
  uint8_t* d = static_cast<uint8_t*>(*mem);
  *out = {reinterpret_cast<const void* const*>(d), reinterpret_cast<const uint64_t*>(d + np),
          reinterpret_cast<const uint64_t*>(d + np + no), L, esz};
  return PGX_OK;
}

int build_table(CkptTable& t, const void* const* layers, const uint64_t* counts, int L, int esz) {
  if (L < 0 || L > kMaxLayers) return fail(PGX_E_CONFIG, "checkpoint layer count %d outside 0..%d", L, kMaxLayers);
  if (esz != 4 && esz != 8) return fail(PGX_E_CONFIG, "element size %d is not 4 or 8", esz);
  t.L = L;
  t.esz = esz;
  t.off[0] = 5;
  t.cum[0] = 0;
  for (int l = 0; l < L; ++l) {
    if (counts[l] && !layers[l]) return fail(PGX_E_INPUT, "layer %d has no data pointer", l);
    t.p[l] = layers[l];
    t.off[l + 1] = t.off[l] + 12 + 8 * counts[l];
    t.cum[l + 1] = t.cum[l] + counts[l];
  }
  return PGX_OK;
}

int grid_for(uint64_t items) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t want = (items + kThreads - 1) / kThreads, cap = (uint64_t)sms * 8;
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

// Python's repr() of a bytes object (the reference formats the bad magic with !r).
std::string py_bytes_repr(const uint8_t* b, size_t n) {
  bool sq = false, dq = false;
  for (size_t i = 0; i < n; ++i) {
    sq |= b[i] == '\'';
    dq |= b[i] == '"';
  }
  const char quote = (sq && !dq) ? '"' : '\'';
  std::string s = "b";
  s += quote;
  char tmp[8];
  for (size_t i = 0; i < n; ++i) {
    uint8_t c = b[i];
    if (c == (uint8_t)quote || c == '\\') {
      s += '\\';
      s += (char)c;
    } else if (c == '\t') {
      s += "\\t";
    } else if (c == '\n') {
      s += "\\n";
    } else if (c == '\r') {
      s += "\\r";
    } else if (c < 0x20 || c >= 0x7f) {
      snprintf(tmp, sizeof(tmp), "\\x%02x", c);
      s += tmp;
    } else {
      s += (char)c;
    }
  }
  s += quote;
  return s;
}

}  // namespace

extern "C" {

int pgx_ckpt_image_bytes(const uint64_t* counts, int num_layers, uint64_t* bytes_out) {
  if (num_layers < 0) return fail(PGX_E_CONFIG, "negative layer count");
  uint64_t b = 5;
  for (int l = 0; l < num_layers; ++l) b += 12 + 8 * counts[l];
  *bytes_out = b;
  return PGX_OK;
}

int pgx_ckpt_parse(const void* blob, uint64_t bytes, uint64_t* counts_out, int capacity, int* num_layers_out) {
  const uint8_t* b = static_cast<const uint8_t*>(blob);
  static const uint8_t magic[5] = {'P', 'S', 'G', 'D', '1'};
  if (bytes < 5 || memcmp(b, magic, 5) != 0)
    return fail(PGX_E_FORMAT, "bad checkpoint magic %s", py_bytes_repr(b, bytes < 5 ? bytes : 5).c_str());
  uint64_t pos = 5;
  int n = 0;
  while (pos < bytes) {
    if (bytes - pos < 12) return fail(PGX_E_FORMAT, "truncated checkpoint: partial layer header");
    uint32_t index;
    uint64_t count;
    memcpy(&index, b + pos, 4);  // little-endian host (x86-64 / aarch64)
    memcpy(&count, b + pos + 4, 8);
    pos += 12;
    if (index != (uint32_t)n) return fail(PGX_E_FORMAT, "layer %d recorded with index %u", n, index);
    if (count > (bytes - pos) / 8) return fail(PGX_E_FORMAT, "truncated checkpoint: layer %u shorter than declared", index);
    if (counts_out && n < capacity) counts_out[n] = count;
    ++n;
    pos += count * 8;
  }
  if (n == 0) return fail(PGX_E_FORMAT, "checkpoint holds no layers");
  *num_layers_out = n;
  if (counts_out && n > capacity) return fail(PGX_E_RANGE, "checkpoint holds %d layers, capacity %d", n, capacity);
  return PGX_OK;
}

int pgx_ckpt_pack(const void* const* layers, const uint64_t* counts, int num_layers, int elem_size, void* image,
                  uint64_t capacity, void* stream) {
  HostTable h;
  int rc = build_host_table(h, layers, counts, num_layers, elem_size);
  if (rc) return rc;
  const uint64_t bytes = h.off[num_layers], pairs = (bytes + 15) / 16;
  if (capacity < pairs * 16) return fail(PGX_E_RANGE, "image buffer %llu bytes < %llu", (unsigned long long)capacity,
                                         (unsigned long long)(pairs * 16));
  if (reinterpret_cast<uintptr_t>(image) & 15) return fail(PGX_E_INPUT, "image buffer is not 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  if (num_layers <= kMaxLayers) {  // the table travels as the kernel parameter
    std::unique_ptr<CkptTable> tp(new CkptTable());  // 12 KB; the launch copies it
    rc = build_table(*tp, layers, counts, num_layers, elem_size);
    if (rc) return rc;
    k_ckpt_pack<CkptTable><<<grid_for(pairs), kThreads, 0, s>>>(*tp, static_cast<uint4*>(image), pairs);
    PGX_LAUNCH_CHECK();
    return PGX_OK;
  }
  CkptDevTable d;
  void* mem = nullptr;
  rc = upload_table(h, num_layers, elem_size, s, &d, &mem);
  if (rc) return rc;
  k_ckpt_pack<CkptDevTable><<<grid_for(pairs), kThreads, 0, s>>>(d, static_cast<uint4*>(image), pairs);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(mem, s);
  if (e != cudaSuccess) return fail(PGX_E_CUDA, "kernel launch: %s", cudaGetErrorString(e));
  return PGX_OK;
}

int pgx_ckpt_unpack(const void* image, uint64_t capacity, const uint64_t* counts, int num_layers, int elem_size,
                    void* const* layers, void* stream) {
  HostTable h;
  int rc = build_host_table(h, const_cast<const void* const*>(layers), counts, num_layers, elem_size);
  if (rc) return rc;
  const uint64_t need = (h.off[num_layers] + 7) / 8 * 8 + 8;  // the last value reads one word past its own
  if (capacity < need) return fail(PGX_E_RANGE, "image buffer %llu bytes < %llu", (unsigned long long)capacity,
                                   (unsigned long long)need);
  if (reinterpret_cast<uintptr_t>(image) & 7) return fail(PGX_E_INPUT, "image buffer is not 8-byte aligned");
  if (h.cum[num_layers] == 0) return PGX_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t total = h.cum[num_layers];
  if (num_layers <= kMaxLayers) {
    std::unique_ptr<CkptTable> tp(new CkptTable());
    rc = build_table(*tp, const_cast<const void* const*>(layers), counts, num_layers, elem_size);
    if (rc) return rc;
    k_ckpt_unpack<CkptTable><<<grid_for(total), kThreads, 0, s>>>(*tp, static_cast<const uint64_t*>(image));
    PGX_LAUNCH_CHECK();
    return PGX_OK;
  }
  CkptDevTable d;
  void* mem = nullptr;
  rc = upload_table(h, num_layers, elem_size, s, &d, &mem);
  if (rc) return rc;
  k_ckpt_unpack<CkptDevTable><<<grid_for(total), kThreads, 0, s>>>(d, static_cast<const uint64_t*>(image));
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(mem, s);
  if (e != cudaSuccess) return fail(PGX_E_CUDA, "kernel launch: %s", cudaGetErrorString(e));
  return PGX_OK;
}

}  // extern "C"
