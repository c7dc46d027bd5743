// Element-wise arithmetic of the exchange path, bit-exact with the reference.
//
//   buffer_axpy    buffers.py:69-74      y := y + (alpha*x)          two roundings
//   master_update  engine/sgd.py:27-33   out = w - eps*g  in float64  two roundings
//   tree_reduce    engine/sgd.py:53-69   binomial fold, children ascending
//   fold+update    pipelined.py:158-188 + :103-108 fused on the master
//   seeded_fill    buffers.py:54-66      splitmix64 -> [-scale, scale]
//
// FMA contraction would change the last bit of `w - eps*g` and `y + a*x`, so
// every operation uses an explicit round-to-nearest intrinsic.  All kernels
// are HBM-bound streams: 128-bit vector accesses, grid sized to 4 CTAs/SM.
#include <cuda_runtime.h>

#include "pgx_common.cuh"
#include "pgx_tree.cuh"

using namespace pgx;

namespace {

constexpr int kThreads = 256;

int grid_for(uint64_t nvec) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  uint64_t want = (nvec + kThreads - 1) / kThreads;
  uint64_t cap = (uint64_t)sms * 8;
  if (want > cap) want = cap;
  return (int)(want < 1 ? 1 : want);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ------------------------------------------------------------------- scalars
__device__ __forceinline__ float axpy1(float a, float x, float y) { return __fadd_rn(y, __fmul_rn(a, x)); }
__device__ __forceinline__ double axpy1(double a, double x, double y) { return __dadd_rn(y, __dmul_rn(a, x)); }
__device__ __forceinline__ double upd64(double w, double g, double eps) { return __dsub_rn(w, __dmul_rn(eps, g)); }
__device__ __forceinline__ float upd32(float w, float g, double eps) {
  return __double2float_rn(__dsub_rn((double)w, __dmul_rn(eps, (double)g)));
}

// ------------------------------------------------------------------- axpy
template <class T, class V>
__global__ void k_axpy(T a, const T* __restrict__ x, T* __restrict__ y, uint64_t n, bool vec) {
  constexpr int W = sizeof(V) / sizeof(T);
  uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, st = (uint64_t)gridDim.x * blockDim.x;
  uint64_t nv = vec ? n / W : 0;
  const V* xv = reinterpret_cast<const V*>(x);
  V* yv = reinterpret_cast<V*>(y);
  for (uint64_t i = i0; i < nv; i += st) {
    V xx = xv[i], yy = yv[i];
    T* xs = reinterpret_cast<T*>(&xx);
    T* ys = reinterpret_cast<T*>(&yy);
#pragma unroll
    for (int k = 0; k < W; ++k) ys[k] = axpy1(a, xs[k], ys[k]);
    yv[i] = yy;
  }
  for (uint64_t i = nv * W + i0; i < n; i += st) y[i] = axpy1(a, x[i], y[i]);
}

// ------------------------------------------------------------------- update
template <class TI, class TO>
__global__ void k_update(const TI* __restrict__ w, const TI* __restrict__ g, double eps, TO* __restrict__ out,
                         uint64_t n) {
  uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, st = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = i0; i < n; i += st) {
    if constexpr (sizeof(TI) == 8)
      out[i] = upd64(w[i], g[i], eps);
    else
      out[i] = upd32(w[i], g[i], eps);
  }
}

// ------------------------------------------------------------------- tree fold (+ update)
struct Parts {
  const void* p[PGX_MAX_RANKS];
};

template <int S, class T>
__device__ __forceinline__ T tree_at(const Parts& P, uint64_t i) {
  T v[S];
#pragma unroll
  for (int r = 0; r < S; ++r) v[r] = __ldcs(static_cast<const T*>(P.p[r]) + i);
  if constexpr (sizeof(T) == 8)
    return tree_sum<S>(v, AddF64{});
  else
    return tree_sum<S>(v, AddF32{});
}

// mode: -1 = fold only (out), else pgx_mode applied in place on w (+v)
template <int S, class T>
__global__ void k_fold(Parts P, T* __restrict__ out, uint64_t n, int mode, double eps, float scale, float mu,
                       float wd, float* __restrict__ v) {
  uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, st = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = i0; i < n; i += st) {
    T g = tree_at<S, T>(P, i);
    if (mode < 0) {
      out[i] = g;
    } else if constexpr (sizeof(T) == 8) {
      out[i] = upd64(out[i], g, eps);
    } else {
      float w = out[i];
      if (mode == PGX_MODE_REF32) {
        out[i] = upd32(w, g, eps);
      } else {  // FAST32: g*scale + wd*w ; v = mu*v + lr*g ; w -= v  (oracle fast32_update)
        float gg = __fadd_rn(__fmul_rn(scale, g), __fmul_rn(wd, w));
        float vv = __fadd_rn(__fmul_rn(mu, v[i]), __fmul_rn((float)eps, gg));
        v[i] = vv;
        out[i] = __fsub_rn(w, vv);
      }
    }
  }
}

template <class T>
int launch_fold(const void* const* parts, int world, T* out, uint64_t n, int mode, double eps, float scale,
                float mu, float wd, float* v, cudaStream_t s) {
  if (world < 1 || world > PGX_MAX_RANKS) return fail(PGX_E_CONFIG, "world %d outside 1..%d", world, PGX_MAX_RANKS);
  Parts P{};
  for (int r = 0; r < world; ++r) P.p[r] = parts[r];
  int grid = grid_for(n);
  switch (world) {
#define PGX_CASE(S) \
  case S: k_fold<S, T><<<grid, kThreads, 0, s>>>(P, out, n, mode, eps, scale, mu, wd, v); break;
    PGX_CASE(1) PGX_CASE(2) PGX_CASE(3) PGX_CASE(4) PGX_CASE(5) PGX_CASE(6) PGX_CASE(7) PGX_CASE(8)
#undef PGX_CASE
  }
  PGX_LAUNCH_CHECK();
  return PGX_OK;
}

// ------------------------------------------------------------------- seeded fill
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
template <class T>
__global__ void k_fill(uint64_t seed, double scale, T* out, uint64_t n) {
  uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, st = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = i0; i < n; i += st) {
    uint64_t z = mix64(seed + (i + 1) * 0x9E3779B97F4A7C15ull);
    double u = __dmul_rn((double)(z >> 11), 0x1.0p-53);
    double x = __dmul_rn(scale, __dsub_rn(__dmul_rn(2.0, u), 1.0));
    out[i] = (T)x;
  }
}

}  // namespace

extern "C" {

int pgx_axpy_f64(double a, const double* x, double* y, uint64_t n, void* s) {
  if (!n) return PGX_OK;
  bool vec = aligned16(x) && aligned16(y);
  k_axpy<double, double2><<<grid_for(vec ? n / 2 : n), kThreads, 0, (cudaStream_t)s>>>(a, x, y, n, vec);
  PGX_LAUNCH_CHECK();
  return PGX_OK;
}

int pgx_axpy_f32(float a, const float* x, float* y, uint64_t n, void* s) {
  if (!n) return PGX_OK;
  bool vec = aligned16(x) && aligned16(y);
  k_axpy<float, float4><<<grid_for(vec ? n / 4 : n), kThreads, 0, (cudaStream_t)s>>>(a, x, y, n, vec);
  PGX_LAUNCH_CHECK();
  return PGX_OK;
}

int pgx_master_update_f64(const double* w, const double* g, double eps, double* out, uint64_t n, void* s) {
  if (!n) return PGX_OK;
  k_update<double, double><<<grid_for(n), kThreads, 0, (cudaStream_t)s>>>(w, g, eps, out, n);
  PGX_LAUNCH_CHECK();
  return PGX_OK;
}

int pgx_master_update_f32(const float* w, const float* g, double eps, float* out, uint64_t n, void* s) {
  if (!n) return PGX_OK;
  k_update<float, float><<<grid_for(n), kThreads, 0, (cudaStream_t)s>>>(w, g, eps, out, n);
  PGX_LAUNCH_CHECK();
  return PGX_OK;
}

int pgx_tree_reduce_f64(const double* const* parts, int world, double* out, uint64_t n, void* s) {
  if (!n) return PGX_OK;
  return launch_fold<double>(reinterpret_cast<const void* const*>(parts), world, out, n, -1, 0, 0, 0, 0, nullptr,
                             (cudaStream_t)s);
}

int pgx_tree_reduce_f32(const float* const* parts, int world, float* out, uint64_t n, void* s) {
  if (!n) return PGX_OK;
  return launch_fold<float>(reinterpret_cast<const void* const*>(parts), world, out, n, -1, 0, 0, 0, 0, nullptr,
                            (cudaStream_t)s);
}

int pgx_fold_update(int mode, const void* const* parts, int world, void* w, float* v, uint64_t n, double eps,
                    float scale, float mu, float wd, void* s) {
  if (!n) return PGX_OK;
  if (mode == PGX_MODE_REF64)
    return launch_fold<double>(parts, world, static_cast<double*>(w), n, mode, eps, scale, mu, wd, v,
                               (cudaStream_t)s);
  if (mode == PGX_MODE_REF32 || mode == PGX_MODE_FAST32) {
    if (mode == PGX_MODE_FAST32 && !v) return fail(PGX_E_CONFIG, "FAST32 needs a momentum buffer");
    return launch_fold<float>(parts, world, static_cast<float*>(w), n, mode, eps, scale, mu, wd, v,
                              (cudaStream_t)s);
  }
  return fail(PGX_E_CONFIG, "unknown mode %d", mode);
}

int pgx_seeded_fill_f64(uint64_t seed, double scale, double* out, uint64_t n, void* s) {
  if (!n) return fail(PGX_E_SHAPE, "buffer length must be positive, got 0");
  k_fill<double><<<grid_for(n), kThreads, 0, (cudaStream_t)s>>>(seed, scale, out, n);
  PGX_LAUNCH_CHECK();
  return PGX_OK;
}

int pgx_seeded_fill_f32(uint64_t seed, double scale, float* out, uint64_t n, void* s) {
  if (!n) return fail(PGX_E_SHAPE, "buffer length must be positive, got 0");
  k_fill<float><<<grid_for(n), kThreads, 0, (cudaStream_t)s>>>(seed, scale, out, n);
  PGX_LAUNCH_CHECK();
  return PGX_OK;
}

}  // extern "C"
