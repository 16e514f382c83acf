// kstep.cu -- the replay producer: the k-step training
// targets of a batch of trajectory-optimisation solutions
// (ilqr.kstep_targets, ilqr.py:358-407, no critic hook -- the form the trainer
// calls, trainer.py:200-201) appended to the device replay ring with FIFO
// eviction (ReplayBuffer.push_many, buffer.py:108-130) in one launch.
//
// Input: R solutions concatenated row-wise, solution r owning rows
// [off[r], off[r+1]) = its T_r + 1 states (X), per-step costs, V_bar, V_bar_x,
// and controls (U, T_r rows + one ignored padding row).  One thread per output
// row k of solution r:
//   j      = k + min(K, T_r - k)
//   v_bar  = V_bar[k]                    if j == T_r   (ilqr.py:386-389)
//          = sum(step_costs[k:j])        otherwise     (NumPy pairwise order)
//   row    = ([X[k], t0+k], U[k] or 0 at k = T_r, v_bar, V_bar_x[k], [X[j], t0+j])
// Row i of the concatenation lands in ring slot (cursor + i - first) % capacity,
// rows before `first` being the ones FIFO eviction drops (buffer.py:118-121).
// Every value is the float64 input or a float64 sum of inputs, cast once to the
// ring's precision: bit-exact with the reference in fp64, and with the rounded
// reference in fp32.
#include <type_traits>

#include "common.cuh"

namespace cacto {

// numpy/core/src/umath/loops_utils.h pairwise_sum (blocks of 8 accumulators
// up to 128 terms, halving recursion above), plus the reduction's +0.0 identity
__device__ __noinline__ double np_pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise(a, n2), np_pairwise(a + n2, n - n2));
}

template <typename T>
struct KstepArgs {
  const int64_t* off;  // [R + 1]
  const int32_t* t0;   // [R]
  const double *X, *U, *sc, *vb, *vbx;
  int64_t R, first, rows, capacity, cursor;
  int n, m, K;
  T *xa, *u, *v, *vx, *xk;
  int32_t* bad;  // set when a v_bar is not finite (TOSample, buffer.py:33-35)
};

template <typename T>
__global__ void kstep_push_kernel(const KstepArgs<T> a) {
  for (int64_t i = a.first + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = a.R;  // solution r: off[r] <= i < off[r+1]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(a.off + mid) <= i) lo = mid;
      else hi = mid;
    }
    const int64_t base = __ldg(a.off + lo);
    const int64_t T_r = __ldg(a.off + lo + 1) - base - 1;
    const int64_t k = i - base;
    const int64_t j = k + min((int64_t)a.K, T_r - k);
    const double v = (j == T_r) ? a.vb[i] : __dadd_rn(np_pairwise(a.sc + i, j - k), 0.0);
    if (!isfinite(v)) atomicOr(a.bad, 1);
    const int t0 = __ldg(a.t0 + lo);
    const int64_t s = (a.cursor + (i - a.first)) % a.capacity;
    const int n = a.n, m = a.m;
    for (int c = 0; c < n; ++c) {
      a.xa[s * (n + 1) + c] = (T)a.X[i * n + c];
      a.xk[s * (n + 1) + c] = (T)a.X[(base + j) * n + c];
      a.vx[s * n + c] = (T)a.vbx[i * n + c];
    }
    a.xa[s * (n + 1) + n] = (T)(double)(t0 + k);
    a.xk[s * (n + 1) + n] = (T)(double)(t0 + j);
    for (int c = 0; c < m; ++c) a.u[s * m + c] = k < T_r ? (T)a.U[i * m + c] : (T)0;
    a.v[s] = (T)v;
  }
}

}  // namespace cacto

using namespace cacto;

extern "C" int cacto_kstep_push(const cacto_solutions_t* s, int32_t K, int32_t ring_dtype, void* ring_xa,
                                void* ring_u, void* ring_v_bar, void* ring_v_bar_x, void* ring_xa_plus_k,
                                int64_t capacity, int64_t cursor, int64_t first, int32_t* bad, void* stream) {
  if (K < 1) return set_error(CACTO_EVALUE, "K must be >= 1");
  if (!s || s->count < 0 || s->rows < 0 || s->n < 1 || s->m < 1 || capacity < 1 || first < 0 ||
      s->rows - first > capacity || cursor < 0 || cursor >= capacity)
    return set_error(CACTO_EVALUE, "kstep_push: bad sizes");
  if (s->rows <= first || s->count == 0) return CACTO_OK;
  if (!bad) return set_error(CACTO_EVALUE, "kstep_push: `bad` flag pointer required");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t todo = s->rows - first;
  const unsigned grid = (unsigned)((todo + 127) / 128 < 4096 ? (todo + 127) / 128 : 4096);
  auto fill = [&](auto* tag) {
    using T = std::remove_pointer_t<decltype(tag)>;
    KstepArgs<T> a;
    a.off = s->offsets; a.t0 = s->t0;
    a.X = s->X; a.U = s->U; a.sc = s->step_costs; a.vb = s->v_bar; a.vbx = s->v_bar_x;
    a.R = s->count; a.first = first; a.rows = s->rows; a.capacity = capacity; a.cursor = cursor;
    a.n = s->n; a.m = s->m; a.K = K;
    a.xa = (T*)ring_xa; a.u = (T*)ring_u; a.v = (T*)ring_v_bar; a.vx = (T*)ring_v_bar_x; a.xk = (T*)ring_xa_plus_k;
    a.bad = bad;
    kstep_push_kernel<T><<<grid, 128, 0, st>>>(a);
  };
  if (ring_dtype == CACTO_F32) fill((float*)nullptr);
  else if (ring_dtype == CACTO_F64) fill((double*)nullptr);
  else return set_error(CACTO_EVALUE, "kstep_push: dtype");
  return check_launch("kstep_push_kernel");
}
