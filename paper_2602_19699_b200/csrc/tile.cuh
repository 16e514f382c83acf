// tile.cuh -- shared-memory tile engine for the fused small-MLP kernels.
//
// A CTA of 256 threads owns a tile of S samples.  Activations live in shared
// memory "unit-major": tile[r][s] (row r = unit / feature, s = sample), with an
// XOR swizzle on 4-element chunks so that both the GEMM inner loops (a warp
// reads 4 distinct sample-chunks of one row) and the epilogue stores (a warp
// writes 8 rows x 4 chunks) are bank-conflict free.  Weights are staged once
// per CTA in shared memory in the reference row-major layout W[out][in]
// (nets.py:116), swizzled the same way; ONE copy serves the forward GEMMs
// (z = a W^T, reading 4 consecutive k of a row) and the backward GEMMs
// (s = g W, reading TN consecutive in-units of a row).
//
// Register micro-tile: each thread owns TM=4 samples x TN units (TN = HP/TX).
#pragma once

#include "common.cuh"

namespace cacto {

// swizzled index of element (r, c) in a row-major [*][C] array (C % 4 == 0,
// C/4 a power of two)
template <int C>
CACTO_HD int swz(int r, int c) {
  constexpr int NCH = C / 4;
  constexpr int KM = (NCH >= 8 ? 8 : NCH) - 1;
  return r * C + ((((c >> 2) ^ ((r >> 2) & KM))) << 2) + (c & 3);
}

// runtime-C variant (C in {8, 16, 32, 64, 128})
CACTO_HD int swz_rt(int C, int r, int c) {
  int nch = C >> 2;
  int km = (nch >= 8 ? 8 : nch) - 1;
  return r * C + ((((c >> 2) ^ ((r >> 2) & km))) << 2) + (c & 3);
}

template <typename T, int S, int HP>
struct Tile {
  static constexpr int TM = 4;
  static constexpr int TY = S / TM;
  static constexpr int TX = kThreads / TY;
  static constexpr int TN = HP / TX;
  static_assert(TY * TX == kThreads, "tile/thread mismatch");
  static_assert(TN >= 1 && TN * TX == HP, "hidden width must split over TX");
  static constexpr int LX = TX < 8 ? TX : 8;
  static constexpr int LY = 32 / LX;
  static constexpr int WX = TX / LX;
  static constexpr int ELEMS = HP * S;  // elements of one [HP][S] tile

  int tx, ty;

  CACTO_D Tile() {
    int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    tx = (warp % WX) * LX + (lane % LX);
    ty = (warp / WX) * LY + (lane / LX);
  }

  CACTO_D static int at(int r, int s) { return swz<S>(r, s); }

  // acc[j][i] = sum_k A[k][s_i] * W[n_j][k]   (W swizzled, row length K)
  template <int K>
  CACTO_D void gemm_fwd(const T* __restrict__ W, const T* __restrict__ A, T (&acc)[TN][TM]) const {
#pragma unroll
    for (int j = 0; j < TN; ++j)
#pragma unroll
      for (int i = 0; i < TM; ++i) acc[j][i] = T(0);
#pragma unroll 2
    for (int kc = 0; kc < K / 4; ++kc) {
      T a[4][TM];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        V4<T> v = ld4(A + swz<S>(4 * kc + kk, ty * TM));
#pragma unroll
        for (int i = 0; i < TM; ++i) a[kk][i] = v.v[i];
      }
      T w[TN][4];
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        V4<T> v = ld4(W + swz<K>(tx * TN + j, 4 * kc));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) w[j][kk] = v.v[kk];
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int i = 0; i < TM; ++i) acc[j][i] = fma(a[kk][i], w[j][kk], acc[j][i]);
    }
  }

  // acc[j][i] = sum_{o<K} A[o][s_i] * W[o][n_j]   (W [K][HP] swizzled; K runtime)
  CACTO_D void gemm_bwd(const T* __restrict__ W, const T* __restrict__ A, int K, T (&acc)[TN][TM]) const {
#pragma unroll
    for (int j = 0; j < TN; ++j)
#pragma unroll
      for (int i = 0; i < TM; ++i) acc[j][i] = T(0);
#pragma unroll 4
    for (int o = 0; o < K; ++o) {
      V4<T> a = ld4(A + swz<S>(o, ty * TM));
      T w[TN];
      if constexpr (TN % 4 == 0) {
#pragma unroll
        for (int q = 0; q < TN / 4; ++q) {
          V4<T> v = ld4(W + swz<HP>(o, tx * TN + 4 * q));
#pragma unroll
          for (int e = 0; e < 4; ++e) w[4 * q + e] = v.v[e];
        }
      } else {
#pragma unroll
        for (int j = 0; j < TN; ++j) w[j] = W[swz<HP>(o, tx * TN + j)];
      }
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int i = 0; i < TM; ++i) acc[j][i] = fma(a.v[i], w[j], acc[j][i]);
    }
  }

  // out[n_j][s_i] = f(acc[j][i], n_j, s_i) for the thread's micro-tile
  template <typename F>
  CACTO_D void store(T* __restrict__ out, const T (&acc)[TN][TM], F f) const {
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int r = tx * TN + j;
      V4<T> v;
#pragma unroll
      for (int i = 0; i < TM; ++i) v.v[i] = f(acc[j][i], r, ty * TM + i);
      st4(out + swz<S>(r, ty * TM), v);
    }
  }

  // narrow output: for every (s, j<nout): f(s, j, sum_{k<K} A[k][s] * w(j, k))
  // 4 lanes split K and combine with shuffles (K % 4 == 0).
  template <int K, typename WF, typename F>
  CACTO_D static void narrow(const T* __restrict__ A, int nout, WF w, F f) {
    const int total = S * nout * 4;
    for (int base = 0; base < total; base += kThreads) {
      int idx = base + threadIdx.x;
      bool live = idx < total;
      int q = idx & 3, p = idx >> 2;
      int s = p % S, j = p / S;
      T sum = T(0);
      if (live) {
#pragma unroll 4
        for (int k = q * (K / 4); k < (q + 1) * (K / 4); ++k) sum = fma(A[swz<S>(k, s)], w(j, k), sum);
      }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      if (live && q == 0) f(s, j, sum);
    }
  }

  // elementwise over a logical [R][S] region: f(r, s, index)
  template <typename F>
  CACTO_D static void each(int R, F f) {
    for (int p = threadIdx.x; p < R * S; p += kThreads) {
      int r = p / S, s = p % S;
      f(r, s, swz<S>(r, s));
    }
  }
};

// load a padded row-major [rows][cols] global matrix into swizzled shared memory
template <typename T>
CACTO_D void stage_matrix(T* __restrict__ dst, const T* __restrict__ src, int rows, int cols) {
  int nch = rows * cols / 4;
  for (int q = threadIdx.x; q < nch; q += kThreads) {
    int r = (q * 4) / cols, c = (q * 4) % cols;
    st4(dst + swz_rt(cols, r, c), ld4(src + (int64_t)q * 4));
  }
}
template <typename T>
CACTO_D void stage_vector(T* __restrict__ dst, const T* __restrict__ src, int n) {
  for (int q = threadIdx.x; q < n; q += kThreads) dst[q] = src[q];
}

}  // namespace cacto
