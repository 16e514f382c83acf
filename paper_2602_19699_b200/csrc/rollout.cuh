// rollout.cuh -- K1 rollout arguments and NumPy's pairwise-sum emulation,
// shared by the SIMT rollout (rollout.cu) and the tensor-core rollout
// (rollout_tc.cu).
#pragma once
#include "common.cuh"
#include "systems.cuh"

namespace cacto {

template <typename T>
struct RolloutArgs {
  SysDev<T> sys;
  CostDev<T> cost;
  NetConst<T> nc;
  int has_cost;
  int nh, out, act, head;
  const T* params;
  const double* x0;
  const int32_t* t0;
  int t0_scalar;
  int64_t N;
  int t_hor;      // >= 0 fixed horizon; CACTO_FULL_HORIZON (-1) -> per-start t_max - t0
  int t_stride;   // row stride of the per-step outputs
  int u_tmajor;   // U layout: 0 [N][t_stride][m], 1 [t_hor][m][N] (CACTO_ROLLOUT_U_TIME_MAJOR),
                  // 2 [t_hor][N][m] (CACTO_ROLLOUT_U_STEP_MAJOR)
  CACTO_D int64_t u_at(int64_t gi, int k, int j, int m) const {
    if (u_tmajor == 2) return ((int64_t)k * N + gi) * m + j;
    return u_tmajor ? ((int64_t)k * m + j) * N + gi : (gi * t_stride + k) * m + j;
  }
  T* U;
  T* X;
  T* SC;
  T* C;
  // fused BIC scoring (tensor-core path, trainer.py:150-151 + gap modes): forward
  // passes of up to two scalar nets on [x0, t0] before the rollout, scores
  // written when the cost-to-go is known
  int n_pre;             // 0..2
  int pre_kind[2];       // 0: std net (sigma head), 1: critic (linear head)
  const T* pre_params[2];
  NetConst<T> pre_nc[2];
  int score_mode;        // CACTO_SCORE_*
  T* scores;
  int cta_rows;          // tensor-core rollout: starts per CTA (set by its launcher)
};

// NumPy pairwise summation (numpy/_core/src/umath/loops_utils.h.src) for
// n <= 128 terms, fed one term at a time.  Longer sums chain 128-blocks.
template <typename T>
struct PairwiseSum {
  T r[8];
  T res;
  int n;  // total terms
  CACTO_D void init(int n_) {
    n = n_;
    res = T(0);
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = T(0);
  }
  CACTO_D static T combine(const T (&r)[8]) {
    return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  }
  CACTO_D void add(int i, T v) {
    if (n < 8) {
      res += v;
      return;
    }
    if (n > 128) {  // chained blocks of 128 (not bit-exact beyond 128 terms)
      int blk = i >> 7, off = i & 127;
      int len = min(128, n - (blk << 7));
      if (off == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = T(0);
      }
      sub(off, len, v, blk > 0);
      return;
    }
    sub(i, n, v, false);
  }
  CACTO_D void sub(int i, int len, T v, bool chain) {
    int body = len - (len % 8);
    if (len < 8) {
      res += v;
      return;
    }
    if (i < body) {
      int j = i & 7;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q == j) r[q] = (i < 8) ? v : r[q] + v;
      if (i == body - 1 && body == len) res = chain ? res + combine(r) : combine(r);
    } else {
      if (i == body) res = chain ? res + combine(r) : combine(r);
      res += v;
    }
  }
};

// The same summation with the 8 partial sums in shared memory (one 9-float
// stride per thread, bank-conflict free): the tensor-core rollout keeps its
// registers for the epilogue, and a dynamically indexed r[i & 7] is one LDS/STS
// instead of an 8-way select chain.
template <typename T>
struct PairwiseSumS {
  T* r;
  T res;
  int n;
  CACTO_D void init(int n_, T* r_) {
    n = n_;
    r = r_;
    res = T(0);
  }
  CACTO_D T combine() const {
    return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  }
  CACTO_D void add(int i, T v) {
    if (n < 8) {
      res += v;
      return;
    }
    if (n > 128) {  // chained blocks of 128, as PairwiseSum
      const int blk = i >> 7, off = i & 127;
      sub(off, min(128, n - (blk << 7)), v, blk > 0);
      return;
    }
    sub(i, n, v, false);
  }
  CACTO_D void sub(int i, int len, T v, bool chain) {
    const int body = len - (len % 8);
    if (len < 8) {
      res += v;
      return;
    }
    if (i < body) {
      const int j = i & 7;
      r[j] = (i < 8) ? v : r[j] + v;
      if (i == body - 1 && body == len) res = chain ? res + combine() : combine();
    } else {
      if (i == body) res = chain ? res + combine() : combine();
      res += v;
    }
  }
};

}  // namespace cacto
