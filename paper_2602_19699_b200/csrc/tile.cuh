// tile.cuh -- shared-memory tile engine for the fused small-MLP kernels.
//
// A CTA of 256 threads owns a tile of S samples.  Activations live in shared
// memory "unit-major": tile[r][s] (row r = unit / feature, s = sample).  Weights
// are staged once per CTA in the reference row-major layout W[out][in]
// (nets.py:116); ONE copy serves the forward GEMMs (z = a W^T: a thread reads 4
// consecutive k of its unit rows) and the backward GEMMs (s = g W: a thread
// reads its TN consecutive in-units of one row).
//
// Register micro-tile: each thread owns TM = 4 samples x TN = HP/TX units,
// units contiguous (rows tx*TN .. tx*TN+TN-1).  Every [rows][C] array is XOR
// swizzled on 16-byte chunks with the key (row >> KS) & 7, KS = log2(TN): the
// 8 threads of a warp that read 8 different unit rows at the same logical
// chunk then hit 8 different bank groups (conflict-free), and epilogue stores
// (8 rows x 4 sample chunks per warp) take the minimum 4 wavefronts.  All
// addressing is hoisted: per 4-k chunk a thread does one XOR for its weight
// rows and one for its sample chunk.
#pragma once

#include "common.cuh"

namespace cacto {

constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v / 2); }

// swizzled index of element (r, c) in a row-major [*][C] array; C % 4 == 0 and
// C/4 a power of two; KS = key shift
template <int C, int KS>
CACTO_HD int swz(int r, int c) {
  constexpr int NCH = C / 4;
  constexpr int KM = (NCH >= 8 ? 8 : NCH) - 1;
  return r * C + ((((c >> 2) ^ ((r >> KS) & KM))) << 2) + (c & 3);
}

// stride of the first layer's weight rows in shared memory: at least 32 columns
// so that the XOR key has 8 chunk positions (rows are only IP = 8..32 wide)
template <int IP>
constexpr int w0_stride() { return IP < 32 ? 32 : IP; }

template <typename T, int S, int HP, int TM_ = 4>
struct Tile {
  static constexpr int TM = TM_;  // samples per thread: 4 or 8 (1 or 2 16-byte chunks)
  static constexpr int TC = TM / 4;
  static constexpr int TY = S / TM;
  static constexpr int TX = kThreads / TY;
  static constexpr int TN = HP / TX;
  static constexpr int KS = ilog2(TN);
  static_assert(TY * TX == kThreads, "tile/thread mismatch");
  static_assert(TM == 4 || TM == 8, "TM must be 4 or 8");
  static_assert(TN >= 1 && TN * TX == HP && (1 << KS) == TN, "hidden width must split over TX");
  static constexpr int LX = TX < 8 ? TX : 8;
  static constexpr int LY = 32 / LX;
  static constexpr int WX = TX / LX;
  static constexpr int KMS = (S / 4 >= 8 ? 8 : S / 4) - 1;  // key mask of activation tiles

  int tx, ty;

  CACTO_D Tile() {
    int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    tx = (warp % WX) * LX + (lane % LX);
    ty = (warp / WX) * LY + (lane / LX);
  }

  // activation tile [rows][S]
  CACTO_HD static int at(int r, int s) { return swz<S, KS>(r, s); }
  // weight matrix with row stride C
  template <int C>
  CACTO_HD static int wat(int r, int c) { return swz<C, KS>(r, c); }

  // acc[j][i] = sum_{k<K} A[k][s_i] * W[n_j][k]   (W rows of stride WC, swizzled)
  template <int K, int WC>
  CACTO_D void gemm_fwd(const T* __restrict__ W, const T* __restrict__ A, T (&acc)[TN][TM]) const {
    constexpr int KMW = (WC / 4 >= 8 ? 8 : WC / 4) - 1;
    constexpr uint32_t ES = sizeof(T);
#pragma unroll
    for (int j = 0; j < TN; ++j)
#pragma unroll
      for (int i = 0; i < TM; ++i) acc[j][i] = T(0);
    const uint32_t wrow = saddr(W) + (uint32_t)(tx * TN * WC) * ES;
    const uint32_t abase = saddr(A);
    const int wkey = tx & KMW;  // (tx*TN + j) >> KS == tx for every j < TN
#pragma unroll 4
    for (int kc = 0; kc < K / 4; ++kc) {
      T a[4][TM];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int r = 4 * kc + kk;
        const int key = (r >> KS) & KMS;  // uniform over the warp
#pragma unroll
        for (int h = 0; h < TC; ++h) {
          V4<T> v = lds4(abase + (uint32_t)(r * S + (((ty * TC + h) ^ key) << 2)) * ES, (T*)nullptr);
#pragma unroll
          for (int e = 0; e < 4; ++e) a[kk][4 * h + e] = v.v[e];
        }
      }
      const uint32_t wc = wrow + (uint32_t)((kc ^ wkey) << 2) * ES;
      T w[TN][4];
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        V4<T> v = lds4(wc + j * WC * ES, (T*)nullptr);
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

  // acc[j][i] = sum_{o<K} A[o][s_i] * W[o][n_j]   (W [K][HP], stride HP; K runtime)
  CACTO_D void gemm_bwd(const T* __restrict__ W, const T* __restrict__ A, int K, T (&acc)[TN][TM]) const {
    constexpr int KMW = (HP / 4 >= 8 ? 8 : HP / 4) - 1;
    constexpr uint32_t ES = sizeof(T);
#pragma unroll
    for (int j = 0; j < TN; ++j)
#pragma unroll
      for (int i = 0; i < TM; ++i) acc[j][i] = T(0);
    const uint32_t abase = saddr(A), wbase = saddr(W);
#pragma unroll 4
    for (int o = 0; o < K; ++o) {
      T a[TM];
#pragma unroll
      for (int h = 0; h < TC; ++h) {
        V4<T> v = lds4(abase + (uint32_t)(o * S + (((ty * TC + h) ^ ((o >> KS) & KMS)) << 2)) * ES, (T*)nullptr);
#pragma unroll
        for (int e = 0; e < 4; ++e) a[4 * h + e] = v.v[e];
      }
      const int wk = (o >> KS) & KMW;
      const uint32_t wr = wbase + (uint32_t)(o * HP) * ES;
      T w[TN];
      if constexpr (TN % 4 == 0) {
#pragma unroll
        for (int q = 0; q < TN / 4; ++q) {
          V4<T> v = lds4(wr + (uint32_t)((((tx * TN) / 4 + q) ^ wk) << 2) * ES, (T*)nullptr);
#pragma unroll
          for (int e = 0; e < 4; ++e) w[4 * q + e] = v.v[e];
        }
      } else {
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          const int n = tx * TN + j;
          w[j] = lds1(wr + (uint32_t)((((n >> 2) ^ wk) << 2) + (n & 3)) * ES, (T*)nullptr);
        }
      }
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int i = 0; i < TM; ++i) acc[j][i] = fma(a[i], w[j], acc[j][i]);
    }
  }

  // out[n_j][s_i] = f(acc[j][i], n_j, s_i) for the thread's micro-tile
  template <typename F>
  CACTO_D void store(T* __restrict__ out, const T (&acc)[TN][TM], F f) const {
    constexpr uint32_t ES = sizeof(T);
    const uint32_t ob = saddr(out) + (uint32_t)(tx * TN * S) * ES;
    const int key = tx & KMS;  // row key of every row tx*TN + j
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int r = tx * TN + j;
#pragma unroll
      for (int h = 0; h < TC; ++h) {
        V4<T> v;
#pragma unroll
        for (int e = 0; e < 4; ++e) v.v[e] = f(acc[j][4 * h + e], r, ty * TM + 4 * h + e);
        sts4(ob + (uint32_t)(j * S + (((ty * TC + h) ^ key) << 2)) * ES, v);
      }
    }
  }

  // narrow output (nout <= 8 columns): f(s, j, sum_{k<K} A[k][s] * W[j][k]),
  // W rows of stride WC (swizzled with KS).  Work item = (sample, K-quarter);
  // the 4 quarter lanes of a sample are adjacent and combine with shuffles.
  // Per 4 rows: 4 scalar A loads (one row key per 4-row group when TN >= 4),
  // one 16-byte W load per output, 4*nout FMAs.
  template <int K, int WC, typename F>
  CACTO_D static void narrow_rows(const T* __restrict__ A, const T* __restrict__ W, int nout, F f) {
    static_assert(K % 16 == 0 || K == 8, "K must split into 4-row groups per quarter");
    constexpr int Q = (K >= 16) ? 4 : 2;
    constexpr int KQ = K / Q;
    constexpr int KMW = (WC / 4 >= 8 ? 8 : WC / 4) - 1;
    constexpr uint32_t ES = sizeof(T);
    const uint32_t abase = saddr(A), wbase = saddr(W);
    for (int item = threadIdx.x; item < S * Q; item += kThreads) {
      const int s = item / Q, q = item % Q;
      const int sc = s >> 2, s3 = s & 3;
      T acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = T(0);
      const uint32_t ab = abase + (uint32_t)(q * KQ * S + s3) * ES;
#pragma unroll
      for (int kk = 0; kk < KQ; kk += 4) {
        const int k0 = q * KQ + kk;
        T a[4];
        if constexpr (KS >= 2) {
          const uint32_t off = (uint32_t)((sc ^ ((k0 >> KS) & KMS)) << 2) * ES;
#pragma unroll
          for (int r = 0; r < 4; ++r) a[r] = lds1(ab + (uint32_t)((kk + r) * S) * ES + off, (T*)nullptr);
        } else {
#pragma unroll
          for (int r = 0; r < 4; ++r)
            a[r] = lds1(ab + (uint32_t)((kk + r) * S + ((sc ^ (((k0 + r) >> KS) & KMS)) << 2)) * ES, (T*)nullptr);
        }
        const int kc = k0 >> 2;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j < nout) {
            V4<T> w = lds4(wbase + (uint32_t)(j * WC + ((kc ^ ((j >> KS) & KMW)) << 2)) * ES, (T*)nullptr);
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[j] = fma(a[r], w.v[r], acc[j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < nout) {
          T v = acc[j];
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          if constexpr (Q == 4) v += __shfl_xor_sync(0xffffffffu, v, 2);
          if (q == 0) f(s, j, v);
        }
      }
    }
  }

  // transposed narrow (nout <= NMAX columns): f(s, c, sum_{k<K} A[k][s] * W[k][c]),
  // W [K][WC] rows swizzled with KS -- the input-gradient s_0 = g_0 W_0.
  template <int K, int WC, int NMAX, typename F>
  CACTO_D static void narrow_cols(const T* __restrict__ A, const T* __restrict__ W, int nout, F f) {
    static_assert(NMAX % 4 == 0 && NMAX <= WC, "column block");
    static_assert(K % 16 == 0, "K must split into 4 quarters of 4-row groups");
    constexpr int Q = 4, KQ = K / Q;
    constexpr int KMW = (WC / 4 >= 8 ? 8 : WC / 4) - 1;
    constexpr uint32_t ES = sizeof(T);
    const uint32_t abase = saddr(A), wbase = saddr(W);
    for (int item = threadIdx.x; item < S * Q; item += kThreads) {
      const int s = item / Q, q = item % Q;
      const int sc = s >> 2, s3 = s & 3;
      T acc[NMAX];
#pragma unroll
      for (int c = 0; c < NMAX; ++c) acc[c] = T(0);
      const uint32_t ab = abase + (uint32_t)(q * KQ * S + s3) * ES;
#pragma unroll 4
      for (int kk = 0; kk < KQ; ++kk) {
        const int k = q * KQ + kk;
        const T a = lds1(ab + (uint32_t)(kk * S + ((sc ^ ((k >> KS) & KMS)) << 2)) * ES, (T*)nullptr);
        const int wk = (k >> KS) & KMW;
#pragma unroll
        for (int cc = 0; cc < NMAX / 4; ++cc) {
          if (4 * cc < nout) {
            V4<T> w = lds4(wbase + (uint32_t)(k * WC + ((cc ^ wk) << 2)) * ES, (T*)nullptr);
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[4 * cc + e] = fma(a, w.v[e], acc[4 * cc + e]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NMAX; ++c) {
        if (c < nout) {
          T v = acc[c];
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          if (q == 0) f(s, c, v);
        }
      }
    }
  }

  // elementwise over a logical [R][S] region: f(r, s, index)
  template <typename F>
  CACTO_D static void each(int R, F f) {
    for (int p = threadIdx.x; p < R * S; p += kThreads) {
      int r = p / S, s = p % S;
      f(r, s, at(r, s));
    }
  }
};

// runtime swizzle (staging): row length C in {8..128}, key shift KS
CACTO_HD int swz_rt(int C, int KS, int r, int c) {
  int nch = C >> 2;
  int km = (nch >= 8 ? 8 : nch) - 1;
  return r * C + ((((c >> 2) ^ ((r >> KS) & km))) << 2) + (c & 3);
}

// load a padded row-major [rows][cols] global matrix into shared memory rows of
// stride `stride` (>= cols), swizzled with key shift KS
template <typename T>
CACTO_D void stage_matrix(T* __restrict__ dst, const T* __restrict__ src, int rows, int cols, int stride, int KS) {
  int cq = cols / 4, nch = rows * cq;
  for (int q = threadIdx.x; q < nch; q += kThreads) {
    int r = q / cq, c = (q % cq) * 4;
    st4(dst + swz_rt(stride, KS, r, c), ld4(src + (int64_t)r * cols + c));
  }
}
template <typename T>
CACTO_D void stage_vector(T* __restrict__ dst, const T* __restrict__ src, int n) {
  for (int q = threadIdx.x; q < n; q += kThreads) dst[q] = src[q];
}

}  // namespace cacto
