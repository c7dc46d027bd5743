// Binomial-tree fold order as a compile-time expression.
//
// The reference fixes the float summation order of the gradient reduction by
// the reduction tree: parent(r) = r & (r-1), children ascending
// (topology.py:34-45), folded as tree_reduce does (engine/sgd.py:53-69) and
// as the pipelined engine does (pipelined.py:158-177).  Closed form, verified
// against tree_reduce for s = 1..16:
//
//   sum(r) = g_r;  for j = 1, 2, 4, ... while (r == 0 || j < lowbit(r)) && r + j < s:
//                     sum(r) = sum(r) + sum(r + j)
//
// Sub<S, R>::eval evaluates sum(R) for a world of S ranks over a register
// array, fully unrolled, so a single thread reproduces the whole distributed
// fold bit for bit.
#pragma once

namespace pgx {

template <int S, int R, int J>
struct TreeKids;

template <int S, int R>
struct TreeSub {
  template <class T, class Add>
  __device__ __forceinline__ static T eval(const T* v, Add add) {
    T acc = v[R];
    return TreeKids<S, R, 1>::eval(acc, v, add);
  }
};

template <int S, int R, int J>
struct TreeKids {
  static constexpr bool kOk = (R == 0 || J < (R & -R)) && (R + J < S);
  template <class T, class Add>
  __device__ __forceinline__ static T eval(T acc, const T* v, Add add) {
    if constexpr (kOk) {
      acc = add(acc, TreeSub<S, R + J>::eval(v, add));
      return TreeKids<S, R, 2 * J>::eval(acc, v, add);
    } else {
      return acc;
    }
  }
};

template <int S, class T, class Add>
__device__ __forceinline__ T tree_sum(const T* v, Add add) {
  return TreeSub<S, 0>::eval(v, add);
}

struct AddF32 {
  __device__ __forceinline__ float operator()(float a, float b) const { return __fadd_rn(a, b); }
};
struct AddF64 {
  __device__ __forceinline__ double operator()(double a, double b) const { return __dadd_rn(a, b); }
};

// Host-side mirror used for launch planning.
__host__ __device__ inline int tree_parent(int r) { return r & (r - 1); }
__host__ __device__ inline int tree_num_children(int r, int s) {
  int n = 0;
  long low = r ? (long)(r & -r) : (1L << 30);
  for (long j = 1; j < low && r + j < s; j <<= 1) ++n;
  return n;
}
__host__ __device__ inline int tree_child(int r, int slot) { return r + (1 << slot); }
__host__ __device__ inline int tree_slot_in_parent(int r) {  // index of r in children(parent(r))
  int p = tree_parent(r);
  int d = r - p;
  int slot = 0;
  while ((1 << slot) != d) ++slot;
  return slot;
}

}  // namespace pgx
