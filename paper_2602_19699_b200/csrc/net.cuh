// net.cuh -- a whole (padded) MLP staged in shared memory, with the tile-level
// forward pass (nets.py:132-141) and the input-gradient sweep (nets.py:176-206,
// 258-266) used by the forward / score / loss kernels.
#pragma once

#include "tile.cuh"

namespace cacto {

template <typename T, int HP, int IP>
struct NetSm {
  T* W[CACTO_MAX_LAYERS];  // swizzled [rows][cols]
  T* b[CACTO_MAX_LAYERS];
  int L, nh, in, out;

  // elements needed for a network with nh hidden layers and `out` outputs
  static CACTO_HD size_t elems(int nh, int out) {
    if (nh == 0) return (size_t)4 * ((out + 3) / 4) * IP + 4 * ((out + 3) / 4);
    return (size_t)HP * IP + HP + (size_t)(nh - 1) * (HP * HP + HP) + (size_t)4 * ((out + 3) / 4) * HP +
           4 * ((out + 3) / 4);
  }

  // carve from `base`; returns the end pointer
  CACTO_D T* carve(T* base, int nh_, int in_, int out_) {
    nh = nh_;
    L = nh_ + 1;
    in = in_;
    out = out_;
    int out4 = 4 * ((out_ + 3) / 4);
    T* p = base;
    for (int i = 0; i < L; ++i) {
      int rows = (i == L - 1) ? out4 : HP;
      int cols = (i == 0) ? IP : HP;
      W[i] = p;
      p += rows * cols;
      b[i] = p;
      p += (i == L - 1) ? out4 : HP;
    }
    return p;
  }

  // copy the padded global parameters (include/cacto_b200.h layout)
  CACTO_D void stage(const T* __restrict__ g) const {
    for (int i = 0; i < L; ++i) {
      int rows = (i == L - 1) ? out : HP;
      int cols = (i == 0) ? IP : HP;
      stage_matrix(W[i], g, rows, cols);
      g += rows * cols;
      stage_vector(b[i], g, rows);
      g += rows;
    }
  }
};

// Fill the input tile A0[c][s] = normalised xa[row(s)][c] (zeros beyond `in`
// and for rows past the batch).  `row(s)` returns -1 for padding samples.
template <typename T, int S, typename RowF, typename ValF>
CACTO_D void load_input_tile(T* A0, int IP, int in, const NetConst<T>& nc, RowF row, ValF val) {
  for (int p = threadIdx.x; p < IP * S; p += kThreads) {
    int c = p / S, s = p % S;
    int64_t r = row(s);
    T v = T(0);
    if (r >= 0 && c < in) {
      v = val(r, c);
      if (nc.has_norm) v = (v - nc.in_center[c]) / nc.in_half[c];
    }
    A0[swz_rt(S, c, s)] = v;
  }
}

// Forward through the hidden layers.  Z[i] receives the pre-activations z_i
// when Z != nullptr (training), and the final hidden activation tile is
// returned (written into one of the two ping-pong buffers P0/P1).
// Ends with a __syncthreads.
template <typename T, int S, int HP, int IP>
CACTO_D const T* forward_hidden(const Tile<T, S, HP>& tl, const NetSm<T, HP, IP>& net, int act, const T* A0,
                                T* P0, T* P1, T* const* Z) {
  using TL = Tile<T, S, HP>;
  T acc[TL::TN][TL::TM];
  const T* cur = A0;
  T* bufs[2] = {P0, P1};
  for (int i = 0; i < net.nh; ++i) {
    if (i == 0)
      tl.template gemm_fwd<IP>(net.W[0], cur, acc);
    else
      tl.template gemm_fwd<HP>(net.W[i], cur, acc);
    const T* bi = net.b[i];
    if (Z) tl.store(Z[i], acc, [&](T v, int r, int) { return v + bi[r]; });
    T* dst = bufs[i & 1];
    tl.store(dst, acc, [&](T v, int r, int) { return act_value(act, v + bi[r]); });
    __syncthreads();
    cur = dst;
  }
  return cur;
}

// Raw network outputs o[s][j] (pre-head) for the tile: f(s, j, o).
template <typename T, int S, int HP, int IP, typename F>
CACTO_D void forward_output(const NetSm<T, HP, IP>& net, const T* last, F f) {
  using TL = Tile<T, S, HP>;
  const int Lm = net.L - 1;
  const T* W = net.W[Lm];
  const T* b = net.b[Lm];
  if (net.nh == 0)
    TL::template narrow<IP>(last, net.out, [&](int j, int k) { return W[swz<IP>(j, k)]; },
                            [&](int s, int j, T v) { f(s, j, v + b[j]); });
  else
    TL::template narrow<HP>(last, net.out, [&](int j, int k) { return W[swz<HP>(j, k)]; },
                            [&](int s, int j, T v) { f(s, j, v + b[j]); });
}

// Input-gradient sweep for output row j (nets.py:186-188 / 201-203):
//   s_L = W_L[j]; g_i = act'(z_i) * s_{i+1}; s_i = g_i W_i
// G[i] receives g_i (i = 0..nh-1) when non-null (critic loss keeps them),
// otherwise the ping-pong buffers P0/P1 are used.  The gradient w.r.t. the
// normalised input is delivered as f(s, c, value) for c < in (not divided by
// in_half).  Requires Z (pre-activations).  Ends with a __syncthreads.
template <typename T, int S, int HP, int IP, typename F>
CACTO_D void input_grad_sweep(const Tile<T, S, HP>& tl, const NetSm<T, HP, IP>& net, int act, int j,
                              T* const* Z, T* const* G, T* P0, T* P1, F f) {
  using TL = Tile<T, S, HP>;
  const int nh = net.nh;
  if (nh == 0) {
    const T* W = net.W[0];
    for (int p = threadIdx.x; p < S * net.in; p += kThreads) {
      int s = p % S, c = p / S;
      f(s, c, W[swz<IP>(j, c)]);
    }
    __syncthreads();
    return;
  }
  T acc[TL::TN][TL::TM];
  const T* WL = net.W[nh];
  // g_{nh-1} = act'(z_{nh-1}) * W_L[j]
  T* gbuf = G ? G[nh - 1] : P0;
  {
    const T* z = Z[nh - 1];
    TL::each(HP, [&](int r, int, int idx) { gbuf[idx] = act_d1(act, z[idx]) * WL[swz<HP>(j, r)]; });
  }
  __syncthreads();
  for (int i = nh - 1; i >= 1; --i) {
    // s_i = g_i W_i  ([S][HP] = [S][HP] x [HP][HP]); g_{i-1} = act'(z_{i-1}) * s_i
    tl.gemm_bwd(net.W[i], gbuf, HP, acc);
    T* nb = G ? G[i - 1] : (gbuf == P0 ? P1 : P0);
    const T* z = Z[i - 1];
    tl.store(nb, acc, [&](T v, int r, int s) { return act_d1(act, z[TL::at(r, s)]) * v; });
    __syncthreads();
    gbuf = nb;
  }
  // s_0 = g_0 W_0  ([S][in], narrow over the input width)
  const T* W0 = net.W[0];
  TL::template narrow<HP>(gbuf, net.in, [&](int c, int k) { return W0[swz<IP>(k, c)]; },
                          [&](int s, int c, T v) { f(s, c, v); });
  __syncthreads();
}

}  // namespace cacto
