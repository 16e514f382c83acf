// net.cuh -- a whole (padded) MLP staged in shared memory, with the tile-level
// forward pass (nets.py:132-141) and the input-gradient sweep (nets.py:176-206,
// 258-266) used by the forward / score / loss kernels.
#pragma once

#include "tile.cuh"

namespace cacto {

// Shared-memory image of one network for kernels whose tiles use key shift KS.
// Layer 0 rows have stride W0S (>= 32), hidden / output rows stride HP.
template <typename T, int HP, int IP, int KS>
struct NetSmem {
  using elem_t = T;
  static constexpr int kHP = HP, kIP = IP, kKS = KS;
  static constexpr int W0S = w0_stride<IP>();
  T* base;  // layer pointers are closed-form offsets (no per-layer pointer arrays:
            // dynamically indexed arrays would live on the local-memory stack)
  int L, nh, in, out;

  static CACTO_HD int out4(int out) { return 4 * ((out + 3) / 4); }

  // elements needed for a network with nh hidden layers and `out` outputs
  static CACTO_HD size_t elems(int nh, int out) {
    if (nh == 0) return (size_t)out4(out) * W0S + out4(out);
    return (size_t)HP * W0S + HP + (size_t)(nh - 1) * (HP * HP + HP) + (size_t)out4(out) * HP + out4(out);
  }

  CACTO_HD static int stride(int i) { return i == 0 ? W0S : HP; }

  // start of layer i's weights / biases
  CACTO_D T* W(int i) const {
    if (i == 0) return base;
    return base + (HP * W0S + HP) + (i - 1) * (HP * HP + HP);
  }
  CACTO_D T* b(int i) const {
    const int rows = (i == L - 1) ? out4(out) : HP;
    return W(i) + rows * stride(i);
  }

  // carve from `p`; returns the end pointer
  CACTO_D T* carve(T* p, int nh_, int in_, int out_) {
    nh = nh_;
    L = nh_ + 1;
    in = in_;
    out = out_;
    base = p;
    return p + elems(nh_, out_);
  }

  // copy the padded global parameters (include/cacto_b200.h layout)
  CACTO_D void stage(const T* __restrict__ g) const {
    for (int i = 0; i < L; ++i) {
      int rows = (i == L - 1) ? out : HP;
      int cols = (i == 0) ? IP : HP;
      stage_matrix(W(i), g, rows, cols, stride(i), KS);
      g += rows * cols;
      stage_vector(b(i), g, rows);
      g += rows;
    }
  }

  // element (r, c) of layer i's weight matrix (explicit shared load)
  CACTO_D T w(int i, int r, int c) const {
    const int e = i == 0 ? swz<W0S, KS>(r, c) : swz<HP, KS>(r, c);
    return lds1(saddr(W(i)) + (uint32_t)e * (uint32_t)sizeof(T), (T*)nullptr);
  }
};

template <typename T, int HP, int IP>
CACTO_HD size_t net_elems(int nh, int out) { return NetSmem<T, HP, IP, 0>::elems(nh, out); }

// Fill the input tile A0[c][s] = normalised xa[row(s)][c] (zeros beyond `in`
// and for rows past the batch).  `row(s)` returns -1 for padding samples.
template <typename TL, typename T, typename RowF, typename ValF>
CACTO_D void load_input_tile(T* A0, int IP, int in, const NetConst<T>& nc, RowF row, ValF val) {
  constexpr int S = TL::TY * TL::TM;
  for (int p = threadIdx.x; p < IP * S; p += kThreads) {
    int c = p / S, s = p % S;
    int64_t r = row(s);
    T v = T(0);
    if (r >= 0 && c < in) {
      v = val(r, c);
      if (nc.has_norm) v = (v - nc.in_center[c]) / nc.in_half[c];
    }
    A0[TL::at(c, s)] = v;
  }
}

// Forward through the hidden layers.  Tile i of Zb (consecutive [HP][S] tiles)
// receives the pre-activations z_i when Zb != nullptr (training); the final
// hidden activation tile is
// returned (written into one of the two ping-pong buffers P0/P1).
// Ends with a __syncthreads.
template <typename TL, typename NS, typename T = typename NS::elem_t>
CACTO_D const T* forward_hidden(const TL& tl, const NS& net, int act, const T* A0, T* P0, T* P1, T* Zb) {
  constexpr int HP = NS::kHP, IP = NS::kIP;
  static_assert(NS::kKS == TL::KS, "network staged with a different swizzle");
  T acc[TL::TN][TL::TM];
  const T* cur = A0;
  for (int i = 0; i < net.nh; ++i) {
    if (i == 0)
      tl.template gemm_fwd<IP, NS::W0S>(net.W(0), cur, acc);
    else
      tl.template gemm_fwd<HP, HP>(net.W(i), cur, acc);
    const T* bi = net.b(i);
    if (Zb) tl.store(Zb + i * (HP * (TL::TY * TL::TM)), acc, [&](T v, int r, int) { return v + bi[r]; });
    T* dst = (i & 1) ? P1 : P0;
    tl.store(dst, acc, [&](T v, int r, int) { return act_fast(act, v + bi[r]); });
    __syncthreads();
    cur = dst;
  }
  return cur;
}

// Raw network outputs o[s][j] (pre-head) for the tile: f(s, j, o).
template <typename TL, typename NS, typename F, typename T = typename NS::elem_t>
CACTO_D void forward_output(const NS& net, const T* last, F f) {
  constexpr int HP = NS::kHP, IP = NS::kIP;
  const int Lm = net.L - 1;
  const T* b = net.b(Lm);
  if (net.nh == 0)
    TL::template narrow_rows<IP, NS::W0S>(last, net.W(0), net.out, [&](int s, int j, T v) { f(s, j, v + b[j]); });
  else
    TL::template narrow_rows<HP, HP>(last, net.W(Lm), net.out, [&](int s, int j, T v) { f(s, j, v + b[j]); });
}

// Input-gradient sweep for output row j (nets.py:186-188 / 201-203):
//   s_L = W_L[j]; g_i = act'(z_i) * s_{i+1}; s_i = g_i W_i
// Tile i of Gb receives g_i (i = 0..nh-1) when Gb != nullptr (critic loss keeps
// them), otherwise the ping-pong buffers P0/P1 are used.  Zb holds z_i.  The gradient w.r.t. the
// normalised input is delivered as f(s, c, value) for c < in (not divided by
// in_half).  Requires Z (pre-activations).  Ends with a __syncthreads.
template <typename TL, typename NS, typename F, typename T = typename NS::elem_t>
CACTO_D void input_grad_sweep(const TL& tl, const NS& net, int act, int j, const T* Zb, T* Gb, T* P0, T* P1, F f) {
  constexpr int S = TL::TY * TL::TM;
  constexpr int HP = NS::kHP;
  constexpr int TS = HP * S;  // elements per tile
  const int nh = net.nh;
  if (nh == 0) {
    for (int p = threadIdx.x; p < S * net.in; p += kThreads) {
      int s = p % S, c = p / S;
      f(s, c, net.w(0, j, c));
    }
    __syncthreads();
    return;
  }
  T acc[TL::TN][TL::TM];
  // g_{nh-1} = act'(z_{nh-1}) * W_L[j]
  T* gbuf = Gb ? Gb + (nh - 1) * TS : P0;
  {
    const T* z = Zb + (nh - 1) * TS;
    TL::each(HP, [&](int r, int, int idx) { gbuf[idx] = act_d1(act, z[idx]) * net.w(nh, j, r); });
  }
  __syncthreads();
  for (int i = nh - 1; i >= 1; --i) {
    // s_i = g_i W_i  ([S][HP] = [S][HP] x [HP][HP]); g_{i-1} = act'(z_{i-1}) * s_i
    tl.gemm_bwd(net.W(i), gbuf, HP, acc);
    T* nb = Gb ? Gb + (i - 1) * TS : (gbuf == P0 ? P1 : P0);
    const T* z = Zb + (i - 1) * TS;
    tl.store(nb, acc, [&](T v, int r, int s) { return act_d1(act, z[TL::at(r, s)]) * v; });
    __syncthreads();
    gbuf = nb;
  }
  // s_0 = g_0 W_0  ([S][in], narrow over the input width)
  TL::template narrow_cols<HP, NS::W0S, NS::kIP>(gbuf, net.W(0), net.in, [&](int s, int c, T v) { f(s, c, v); });
  __syncthreads();
}

}  // namespace cacto
