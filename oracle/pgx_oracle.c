/*
 * pgx_oracle.c — CPU restatement of the reference's exchange data plane.
 * TEST / BASELINE INFRASTRUCTURE ONLY: loaded by tests/ (as a checker) and by
 * bench.py's cpu_baseline and --impl reference legs (as the timed CPU port).
 * The product path (paper_1706_00095_b200/) never links or calls it.
 *
 * Follows /root/reference/pkg/src/pipesgd:
 *   buffer_axpy      buffers.py:69-74     y := y + (1.0*x)   (fp32 stays fp32)
 *   master_update    engine/sgd.py:27-33  w - eps*g in float64
 *   tree order       topology.py:34-45 + pipelined.py:158-177 (children ascending)
 *   send / install   runtime.py:185-251, pipelined.py:190-203 (memcpy into the
 *                    receiver's slot = what write_notify does, inproc.py:93-99)
 * fast32 (momentum / weight decay / 1/N) restates Caffe SGDSolver and is
 * "parity unpinned" (no reference counterpart).
 * Compiled with -ffp-contract=off so no FMA changes a rounding.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { MODE_REF64 = 0, MODE_REF32 = 1, MODE_FAST32 = 2, MODE_SUM32 = 3 };

static int lowbit(int r) { return r & -r; }

/* ---------------------------------------------------------------- scalars */
void oracle_tree_fold_f32(const float* const* parts, int world, float* out, size_t n) {
  /* acc[r] = g_r ; for r = s-1..0: acc[r] += acc[c] for children c ascending */
  float* acc = (float*)malloc(sizeof(float) * (size_t)world);
  for (size_t i = 0; i < n; ++i) {
    for (int r = 0; r < world; ++r) acc[r] = parts[r][i];
    for (int r = world - 1; r >= 0; --r) {
      int low = r ? lowbit(r) : (1 << 30);
      for (int j = 1; j < low && r + j < world; j <<= 1) acc[r] = acc[r] + acc[r + j];
    }
    out[i] = acc[0];
  }
  free(acc);
}

void oracle_tree_fold_f64(const double* const* parts, int world, double* out, size_t n) {
  double* acc = (double*)malloc(sizeof(double) * (size_t)world);
  for (size_t i = 0; i < n; ++i) {
    for (int r = 0; r < world; ++r) acc[r] = parts[r][i];
    for (int r = world - 1; r >= 0; --r) {
      int low = r ? lowbit(r) : (1 << 30);
      for (int j = 1; j < low && r + j < world; j <<= 1) acc[r] = acc[r] + acc[r + j];
    }
    out[i] = acc[0];
  }
  free(acc);
}

void oracle_update_ref64(double* w, const double* g, double eps, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    double t = eps * g[i];
    w[i] = w[i] - t;
  }
}

void oracle_update_ref32(float* w, const float* g, double eps, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    double t = eps * (double)g[i];
    w[i] = (float)((double)w[i] - t);
  }
}

void oracle_update_fast32(float* w, float* v, const float* g, float scale, float lr, float mu, float wd,
                          size_t n) {
  for (size_t i = 0; i < n; ++i) {
    float a = scale * g[i];
    float b = wd * w[i];
    float gg = a + b;
    float m = mu * v[i];
    float l = lr * gg;
    float vv = m + l;
    v[i] = vv;
    w[i] = w[i] - vv;
  }
}

/* -------------------------------------------------- data-plane port (bench) */
/* One iteration of the reference's pipelined exchange for `world` ranks, all in
 * this process, fp32 storage: for every layer (backward order) each rank's
 * gradient travels up the binomial tree (memcpy into the parent's receive slot,
 * then an in-order fold), rank 0 applies the update, and the new weights travel
 * down (memcpy into each child's receive slot, then install).  Threads split
 * every layer into contiguous element ranges; each thread runs the whole
 * sequence on its range (the reference's per-element arithmetic is
 * range-independent). */
typedef struct {
  int world, nlayers, mode;
  const uint64_t* elems;
  float*** grad;  /* [rank][layer] */
  float*** w;     /* [rank][layer] */
  float** v;      /* [layer] rank 0 momentum */
  float*** rx;    /* [rank][layer] receive slot (one per rank is enough per turn) */
  double lr;
  float scale, mu, wd;
  int tid, nthreads;
} Job;


/* For r = world-1 down to 0, every child r+c (c = 1, 2, 4, .. < lowbit(r)) is a
 * higher rank whose subtree sum is already final: copy it into r's slot (the
 * write_notify) and fold in ascending child order (pipelined.py:166-177). */
static void* run_job_ordered(void* p) {
  Job* j = (Job*)p;
  for (int l = j->nlayers - 1; l >= 0; --l) {
    size_t n = j->elems[l];
    size_t lo = n * (size_t)j->tid / (size_t)j->nthreads, hi = n * (size_t)(j->tid + 1) / (size_t)j->nthreads;
    size_t m = hi - lo;
    if (!m) continue;
    for (int r = j->world - 1; r >= 0; --r) {
      int low = r ? lowbit(r) : (1 << 30);
      for (int c = 1; c < low && r + c < j->world; c <<= 1) {
        /* child r+c's subtree sum is final (higher ranks done); write it into r's slot, fold */
        memcpy(j->rx[r][l] + lo, j->grad[r + c][l] + lo, m * sizeof(float));
        float* y = j->grad[r][l] + lo;
        const float* x = j->rx[r][l] + lo;
        for (size_t i = 0; i < m; ++i) y[i] = y[i] + x[i];
      }
    }
    if (j->mode == MODE_FAST32) {
      oracle_update_fast32(j->w[0][l] + lo, j->v[l] + lo, j->grad[0][l] + lo, j->scale, (float)j->lr, j->mu, j->wd, m);
    } else if (j->mode == MODE_SUM32) {  /* update off: the averaged tree-order sum */
      float* w0 = j->w[0][l] + lo;
      const float* g = j->grad[0][l] + lo;
      for (size_t i = 0; i < m; ++i) w0[i] = j->scale * g[i];
    } else {
      oracle_update_ref32(j->w[0][l] + lo, j->grad[0][l] + lo, j->lr, m);
    }
    for (int r = 1; r < j->world; ++r) {
      int parent = r & (r - 1);
      memcpy(j->rx[r][l] + lo, j->w[parent][l] + lo, m * sizeof(float));
      memcpy(j->w[r][l] + lo, j->rx[r][l] + lo, m * sizeof(float));
    }
  }
  return NULL;
}

/* grads are consumed (folded in place), like the reference's grad views. */
int oracle_exchange_iteration(int world, int nlayers, const uint64_t* elems, float*** grad, float*** w, float** v,
                              float*** rx, int mode, double lr, float scale, float mu, float wd, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  Job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    Job jb = {world, nlayers, mode, elems, grad, w, v, rx, lr, scale, mu, wd, t, nthreads};
    jobs[t] = jb;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, run_job_ordered, &jobs[t]);
  run_job_ordered(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  return 0;
}
