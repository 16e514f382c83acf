// train.cu -- K5-K7: fused per-tile losses with exact parameter gradients.
//
//  critic  nets.critic_loss (nets.py:233-290): forward (z kept), input-gradient
//          sweep (g_i kept), gradient-path cotangent with the ELU/tanh second
//          derivative injected as zeta_i, value-path backprop -- all on one
//          S-sample tile in shared memory; the bootstrap target V_tgt(x_{+k})
//          is a separate batched forward (nets.py:249), as in the reference.
//  actor   nets.actor_loss (nets.py:293-334): (1) actor forward + dynamics /
//          stage-cost epilogue -> x', l; (2) critic value + state gradient at
//          (x', t+1); (3) actor forward + dq/du = l_u + f_u^T dV/dx' + backprop.
//  std     nets.std_critic_loss (nets.py:337-353): critic forward -> error,
//          then the std forward + NLL backprop.
//
// Parameter gradients are accumulated by each CTA into its own slot of the
// workspace ([grid][P+1], last entry = loss partial); cacto_reduce_* folds the
// slots in a fixed order, so results are deterministic run to run.
#include "net.cuh"
#include "systems.cuh"

#ifndef CACTO_CRITIC_FUSED_TARGET
#define CACTO_CRITIC_FUSED_TARGET 1  // bootstrap target forward inside critic_kernel
#endif

namespace cacto {

template <typename T>
struct BatchDev {
  const int64_t* idx;
  const int64_t* cycle;
  int64_t idx_stride;
  const T *xa, *u, *v_bar, *v_bar_x, *xa_plus_k;
  int64_t rows;
  int n, m, t_max;
  CACTO_D int64_t row(int64_t b) const {
    if (!idx) return b;
    return cycle ? idx[(*cycle) * idx_stride + b] : idx[b];
  }
};

template <typename T>
BatchDev<T> batch_dev(const cacto_batch_t& b) {
  BatchDev<T> d;
  d.idx = b.idx;
  d.cycle = b.cycle;
  d.idx_stride = b.idx_stride;
  d.xa = (const T*)b.xa;
  d.u = (const T*)b.u;
  d.v_bar = (const T*)b.v_bar;
  d.v_bar_x = (const T*)b.v_bar_x;
  d.xa_plus_k = (const T*)b.xa_plus_k;
  d.rows = b.rows;
  d.n = b.n;
  d.m = b.m;
  d.t_max = b.t_max;
  return d;
}

// ---- gradient-slot accumulation helpers (slot is this CTA's private region) -----
// g[r][c] += sum_s A[r][s] * B[c][s]  (R, C multiples of 4; A, B swizzled tiles)
template <typename TL, typename T>
CACTO_D void outer_acc4(T* __restrict__ g, int R, int C, const T* __restrict__ A, const T* __restrict__ B) {
  constexpr int S = TL::TY * TL::TM;
  const int cb = C / 4, nblk = (R / 4) * cb;
  for (int blk = threadIdx.x; blk < nblk; blk += kThreads) {
    int r0 = (blk / cb) * 4, c0 = (blk % cb) * 4;
    T acc[4][4] = {};
#pragma unroll 2
    for (int sc = 0; sc < S / 4; ++sc) {
      V4<T> a[4], b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        a[j] = ld4(A + TL::at(r0 + j, 4 * sc));
        b[j] = ld4(B + TL::at(c0 + j, 4 * sc));
      }
#pragma unroll
      for (int jr = 0; jr < 4; ++jr)
#pragma unroll
        for (int jc = 0; jc < 4; ++jc)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[jr][jc] = fma(a[jr].v[e], b[jc].v[e], acc[jr][jc]);
    }
#pragma unroll
    for (int jr = 0; jr < 4; ++jr)
#pragma unroll
      for (int jc = 0; jc < 4; ++jc) g[(int64_t)(r0 + jr) * C + c0 + jc] += acc[jr][jc];
  }
}
// same with 1-row blocks (any R)
template <typename TL, typename T>
CACTO_D void outer_acc1(T* __restrict__ g, int R, int C, const T* __restrict__ A, const T* __restrict__ B) {
  constexpr int S = TL::TY * TL::TM;
  const int cb = C / 4, nblk = R * cb;
  for (int blk = threadIdx.x; blk < nblk; blk += kThreads) {
    int r0 = blk / cb, c0 = (blk % cb) * 4;
    T acc[4] = {};
    for (int sc = 0; sc < S / 4; ++sc) {
      V4<T> a = ld4(A + TL::at(r0, 4 * sc));
#pragma unroll
      for (int jc = 0; jc < 4; ++jc) {
        V4<T> b = ld4(B + TL::at(c0 + jc, 4 * sc));
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[jc] = fma(a.v[e], b.v[e], acc[jc]);
      }
    }
#pragma unroll
    for (int jc = 0; jc < 4; ++jc) g[(int64_t)r0 * C + c0 + jc] += acc[jc];
  }
}
// g[r] += sum_s A[r][s]
template <typename TL, typename T>
CACTO_D void rowsum_acc(T* __restrict__ g, int R, const T* __restrict__ A) {
  constexpr int S = TL::TY * TL::TM;
  for (int r = threadIdx.x; r < R; r += kThreads) {
    T acc = T(0);
    for (int sc = 0; sc < S / 4; ++sc) {
      V4<T> a = ld4(A + TL::at(r, 4 * sc));
      acc += (a.v[0] + a.v[1]) + (a.v[2] + a.v[3]);
    }
    g[r] += acc;
  }
}

// block sum of one value per thread -> thread 0 adds it to *dst
template <typename T>
CACTO_D void block_add(T v, T* dst) {
  __shared__ T red[kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    T s = T(0);
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
    *dst += s;
  }
  __syncthreads();
}

template <typename T>
CACTO_D void zero_slot(T* slot, int64_t count) {
  for (int64_t i = threadIdx.x; i < count; i += kThreads) slot[i] = T(0);
  __syncthreads();
}

struct Offs {
  int64_t w[CACTO_MAX_LAYERS], b[CACTO_MAX_LAYERS];
  int cols[CACTO_MAX_LAYERS];
  int64_t total;
};
inline Offs offs_of(const cacto_mlp_t& m) {
  LayerOffsets lo = layer_offsets(shape_of(m));
  Offs o;
  for (int i = 0; i < CACTO_MAX_LAYERS; ++i) {
    o.w[i] = lo.w[i];
    o.b[i] = lo.b[i];
    o.cols[i] = lo.cols[i];
  }
  o.total = lo.total;
  return o;
}

// =====================================================================================
// Critic Sobolev loss
// =====================================================================================
template <typename T>
struct CriticArgs {
  NetConst<T> nc;
  int nh, in, act;
  const T* params;
  Offs off;
  BatchDev<T> b;
  T inv_denom;
  T k_s;
  const T* v_next;  // [rows] target value at x_{+k} (bootstrap) or null
  const T* tparams; // target net (the critic's shape) evaluated in-kernel at x_{+k}, or null
  NetConst<T> nc_t; // its input normalisation
  T* ws;            // [grid][P+1]
  int smem_slot;    // accumulate the CTA's gradient slot in shared memory, store it once
};

template <typename T, int HP, int IP, int S>
__global__ void __launch_bounds__(kThreads, 1) critic_kernel(const CriticArgs<T> a) {
  using TL = Tile<T, S, HP>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  NetSmem<T, HP, IP, TL::KS> net;
  T* p = net.carve(sm, a.nh, a.in, 1);
  T* A0 = p;
  p += IP * S;
  T* U0 = p;
  p += IP * S;
  constexpr int TS = HP * S;  // elements per [HP][S] tile
  T* const Zb = p;            // z_i tiles (consecutive)
  p += (size_t)a.nh * TS;
  T* const Gb = p;            // g_i -> zeta_i -> zbar_i tiles
  p += (size_t)a.nh * TS;
  T* P = p;
  p += HP * S;
  T* Q = p;
  p += HP * S;
  T* EV = p;  // [S] target y, then e_v, then delta
  p += S;
  T* EG = p;  // [n][S] gradient errors
  p += (size_t)CACTO_MAX_IN * S;
  // bootstrap target forward in the same kernel (the critic's shape, its own staged
  // copy): one launch per critic update instead of rows_forward_kernel + critic_kernel
  NetSmem<T, HP, IP, TL::KS> tnet;
  T* VT = nullptr;  // [S] target values of the tile
  if (a.tparams) {
    p = tnet.carve(p, a.nh, a.in, 1);
    VT = p;
    p += S;
    tnet.stage(a.tparams);
  }

  net.stage(a.params);
  const int64_t P_total = a.off.total;
  T* const gslot = a.ws + (int64_t)blockIdx.x * (P_total + 1);
  // the CTA's gradient slot: in shared memory when it fits (one coalesced store at
  // the end instead of read-modify-writes through L2 per tile), else in the workspace
  T* slot = a.smem_slot ? p : gslot;
  zero_slot(slot, P_total + 1);

  const TL tl;
  const int n = a.b.n, nh = a.nh, L1 = nh;  // index of the output layer
  const int KL = nh > 0 ? HP : IP;          // input width of the output layer
  const int64_t ntiles = (a.b.rows + S - 1) / S;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * S;
    if (a.tparams) {  // V_target(x_{+k}) of the tile (nets.py:247-251), as rows_forward_kernel
      __syncthreads();
      load_input_tile<TL>(A0, IP, a.in, a.nc_t,
                            [&](int s) { return base + s < a.b.rows ? a.b.row(base + s) : (int64_t)-1; },
                            [&](int64_t r, int c) { return a.b.xa_plus_k[r * a.in + c]; });
      __syncthreads();
      const T* lastt = forward_hidden(tl, tnet, a.act, A0, P, Q, (T*)nullptr);
      forward_output<TL>(tnet, lastt, [&](int s, int, T o) { VT[s] = o; });
      __syncthreads();
    }
    load_input_tile<TL>(A0, IP, a.in, a.nc,
                          [&](int s) { return base + s < a.b.rows ? a.b.row(base + s) : (int64_t)-1; },
                          [&](int64_t r, int c) { return a.b.xa[r * a.in + c]; });
    for (int s = threadIdx.x; s < S; s += kThreads) {
      T y = T(0);
      if (base + s < a.b.rows) {
        int64_t r = a.b.row(base + s);
        y = a.b.v_bar[r];
        if (a.v_next || a.tparams) {  // nets.py:247-251
          bool gate = a.b.xa_plus_k[r * (n + 1) + n] < (T)a.b.t_max;
          y = y + (gate ? (a.tparams ? VT[s] : a.v_next[base + s]) : T(0));
        }
      }
      EV[s] = y;
    }
    __syncthreads();
    const T* last = forward_hidden(tl, net, a.act, A0, P, Q, Zb);
    forward_output<TL>(net, last, [&](int s, int, T o) {
      EV[s] = (base + s < a.b.rows) ? EV[s] - o : T(0);  // e_v = y - V
    });
    __syncthreads();
    // input-gradient sweep -> e_g = v_bar_x - dV/dx[:n]  (nets.py:258-270)
    input_grad_sweep(tl, net, a.act, 0, Zb, Gb, P, Q, [&](int s, int c, T v) {
      if (c < n) {
        T e = T(0);
        if (base + s < a.b.rows) e = a.b.v_bar_x[a.b.row(base + s) * n + c] - v / a.nc.in_half[c];
        EG[c * S + s] = e;
      }
    });
    // loss partial: (e_v^2 + k_s |e_g|^2) / B  (nets.py:271)
    {
      T term = T(0);
      for (int s = threadIdx.x; s < S; s += kThreads) {
        T eg2 = T(0);
        for (int c = 0; c < n; ++c) eg2 += EG[c * S + s] * EG[c * S + s];
        term += (EV[s] * EV[s] + a.k_s * eg2) * a.inv_denom;
      }
      block_add(term, slot + P_total);
    }
    // gradient-path cotangent u_0 (nets.py:276-277)
    {
      const T coef = T(-2) * a.k_s * a.inv_denom;
      for (int q = threadIdx.x; q < IP * S; q += kThreads) {
        int c = q / S, s = q % S;
        U0[TL::at(c, s)] = c < n ? coef * EG[c * S + s] / a.nc.in_half[c] : T(0);
      }
    }
    __syncthreads();
    // gradient path (nets.py:279-284)
    const T* u = U0;
    T* rb = Q;
    T accm[TL::TN][TL::TM];
    for (int i = 0; i < nh; ++i) {
      if (i == 0)
        tl.template gemm_fwd<IP, decltype(net)::W0S>(net.W(0), u, accm);
      else
        tl.template gemm_fwd<HP, HP>(net.W(i), u, accm);
      tl.store(rb, accm, [](T v, int, int) { return v; });
      outer_acc4<TL>(slot + a.off.w[i], HP, i == 0 ? IP : HP, (Gb + (i) * TS), u);  // (d1 * s)^T u
      __syncthreads();
      {
        const T* z = (Zb + (i) * TS);
        T* g = (Gb + (i) * TS);
        TL::each(HP, [&](int, int, int q) {
          T zz = z[q], r = rb[q];
          g[q] = act_h(a.act, zz) * g[q] * r;  // zeta_i = act''(z) s rbar
          rb[q] = act_d1(a.act, zz) * r;       // u_{i+1} = act'(z) rbar
        });
      }
      __syncthreads();
      u = rb;
      rb = (rb == Q) ? P : Q;
    }
    rowsum_acc<TL>(slot + a.off.w[L1], KL, u);  // grads[2*last] += u.sum(0)
    // value path (nets.py:287-289, 215-230)
    for (int s = threadIdx.x; s < S; s += kThreads) EV[s] = T(-2) * a.inv_denom * EV[s];  // delta
    __syncthreads();
    {
      const T* aL = A0;
      if (nh > 0) {
        T* dst = (u == P) ? Q : P;  // a buffer not holding u
        const T* z = (Zb + (nh - 1) * TS);
        TL::each(HP, [&](int, int, int q) { dst[q] = act_value(a.act, z[q]); });
        __syncthreads();
        aL = dst;
      }
      // gW_L[0][k] += sum_s delta_s a_L[k][s] ; gb_L += sum_s delta_s
      for (int k = threadIdx.x; k < KL; k += kThreads) {
        T acc = T(0);
        for (int s = 0; s < S; ++s) acc = fma(EV[s], aL[TL::at(k, s)], acc);
        slot[a.off.w[L1] + k] += acc;
      }
      if (threadIdx.x == 0) {
        T acc = T(0);
        for (int s = 0; s < S; ++s) acc += EV[s];
        slot[a.off.b[L1]] += acc;
      }
      __syncthreads();
    }
    if (nh > 0) {
      T* AB = P;  // abar
      T* AS = Q;  // a_i scratch
      TL::each(HP, [&](int r, int s, int q) { AB[q] = EV[s] * net.w(L1, 0, r); });
      __syncthreads();
      for (int i = nh - 1; i >= 0; --i) {
        {
          const T* z = (Zb + (i) * TS);
          T* g = (Gb + (i) * TS);
          TL::each(HP, [&](int, int, int q) { g[q] = act_d1(a.act, z[q]) * AB[q] + g[q]; });  // zbar_i
        }
        if (i > 0) {
          const T* z = (Zb + (i - 1) * TS);
          TL::each(HP, [&](int, int, int q) { AS[q] = act_value(a.act, z[q]); });
        }
        __syncthreads();
        rowsum_acc<TL>(slot + a.off.b[i], HP, (Gb + (i) * TS));
        outer_acc4<TL>(slot + a.off.w[i], HP, i == 0 ? IP : HP, (Gb + (i) * TS), i == 0 ? A0 : AS);
        if (i > 0) {
          tl.gemm_bwd(net.W(i), (Gb + (i) * TS), HP, accm);
          __syncthreads();  // AS / AB reads of this layer are complete
          tl.store(AB, accm, [](T v, int, int) { return v; });
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
  if (a.smem_slot)
    for (int64_t i = threadIdx.x; i <= P_total; i += kThreads) gslot[i] = slot[i];
}

// =====================================================================================
// Generic value-path loss: forward (z kept), per-sample output cotangent from a
// functor, backprop (nets.py:215-230).  Used by the std and actor losses.
// =====================================================================================
template <typename T>
struct VpArgs {
  NetConst<T> nc;
  int nh, in, out, act, head;
  const T* params;
  Offs off;
  BatchDev<T> b;
  const int64_t* live_rows;  // device count (actor) or null -> inv_denom
  int count_live;            // actor: count the live rows in-kernel (live_rows == null)
  T inv_denom;
  // std loss
  const T* err;               // [rows] v_bar - V(xa)
  const int64_t* err_cycle;   // optional: err += (*err_cycle) * err_stride (precomputed errors)
  int64_t err_stride;
  // actor loss
  SysDev<T> sys;
  CostDev<T> cost;
  const T* xn;      // [rows][n+1] next augmented state (prep kernel)
  const T* lstage;  // [rows] stage cost
  const T* vn;      // [rows] critic value at xn
  const T* gn;      // [rows][n+1] critic state gradient at xn
  T* ws;
  int smem_slot;    // accumulate the CTA's gradient slot in shared memory, store it once
};

enum { VP_STD = 0, VP_ACTOR = 1 };

template <typename T, int HP, int IP, int S, int KIND, int SYS>
__global__ void __launch_bounds__(kThreads, 1) vp_kernel(const VpArgs<T> a) {
  using TL = Tile<T, S, HP>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  NetSmem<T, HP, IP, TL::KS> net;
  T* p = net.carve(sm, a.nh, a.in, a.out);
  T* A0 = p;
  p += IP * S;
  constexpr int TS = HP * S;
  T* const Zb = p;  // z_i tiles (consecutive), overwritten by zbar_i in the backward pass
  p += (size_t)a.nh * TS;
  T* P = p;
  p += HP * S;
  T* Q = p;
  p += HP * S;
  T* OUT = p;  // [out][S] raw outputs
  p += CACTO_MAX_OUT * S;
  T* DEL = p;  // [out4][S] swizzled tile of output cotangents
  p += 4 * ((CACTO_MAX_OUT + 3) / 4) * S;

  net.stage(a.params);
  const int64_t P_total = a.off.total;
  T* const gslot = a.ws + (int64_t)blockIdx.x * (P_total + 1);
  T* slot = a.smem_slot ? p : gslot;  // as critic_kernel
  zero_slot(slot, P_total + 1);
  T inv_denom = a.live_rows ? T(1) / (T)(*a.live_rows) : a.inv_denom;
  if (a.count_live) {  // rows with t < t_max (nets.py:310-312), counted by every CTA
    __shared__ unsigned int live_acc;
    if (threadIdx.x == 0) live_acc = 0;
    __syncthreads();
    unsigned int c = 0;
    for (int64_t b = threadIdx.x; b < a.b.rows; b += kThreads)
      c += a.b.xa[a.b.row(b) * (a.b.n + 1) + a.b.n] < (T)a.b.t_max ? 1u : 0u;
    atomicAdd(&live_acc, c);
    __syncthreads();
    inv_denom = T(1) / (T)live_acc;
  }

  const TL tl;
  const int nh = a.nh, L1 = nh, out = a.out, n = a.b.n;
  const int KL = nh > 0 ? HP : IP;
  const int64_t ntiles = (a.b.rows + S - 1) / S;
  T accm[TL::TN][TL::TM];
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * S;
    load_input_tile<TL>(A0, IP, a.in, a.nc,
                          [&](int s) { return base + s < a.b.rows ? a.b.row(base + s) : (int64_t)-1; },
                          [&](int64_t r, int c) { return a.b.xa[r * a.in + c]; });
    __syncthreads();
    const T* last = forward_hidden(tl, net, a.act, A0, P, Q, Zb);
    forward_output<TL>(net, last, [&](int s, int j, T o) { OUT[j * S + s] = o; });
    __syncthreads();
    // per-sample output cotangent + loss term
    T term = T(0);
    for (int s = threadIdx.x; s < S; s += kThreads) {
      T d[CACTO_MAX_OUT];
#pragma unroll
      for (int j = 0; j < CACTO_MAX_OUT; ++j) d[j] = T(0);
      bool valid = base + s < a.b.rows;
      if (valid) {
        int64_t r = a.b.row(base + s);
        if constexpr (KIND == VP_STD) {
          // nets.py:343-352
          T o = OUT[s];
          T sigma = head_value(a.head, a.nc, 0, o);
          T e = a.err[(a.err_cycle ? (*a.err_cycle) * a.err_stride : 0) + base + s];
          term = (m_log(sigma) + T(0.5) * e * e / (sigma * sigma)) * inv_denom;
          T dl = (T(1) / sigma - e * e / (sigma * sigma * sigma)) * inv_denom;
          d[0] = dl * sigmoid(o);
        } else {
          constexpr int nn = SysDims<SYS>::n, mm = SysDims<SYS>::m;
          const T* xa = a.b.xa + r * (nn + 1);
          if (xa[nn] < (T)a.sys.t_max) {  // nets.py:308-312
            T x[nn], u[mm], g[nn], ft[mm];
#pragma unroll
            for (int c = 0; c < nn; ++c) x[c] = xa[c];
#pragma unroll
            for (int j = 0; j < mm; ++j) u[j] = head_value(a.head, a.nc, j, OUT[j * S + s]);
#pragma unroll
            for (int c = 0; c < nn; ++c) g[c] = a.gn[(base + s) * (nn + 1) + c];
            fu_t_g<SYS>(a.sys, x, u, g, ft);
            term = (a.lstage[base + s] + a.vn[base + s]) * inv_denom;  // nets.py:328
#pragma unroll
            for (int j = 0; j < mm; ++j) {
              T dq = T(2) * a.cost.w_u * u[j] + ft[j];  // nets.py:329, l_u costs.py:162
              d[j] = (dq * inv_denom) * head_chain(a.head, a.nc, j, OUT[j * S + s]);
            }
          }
        }
      }
      for (int j = 0; j < out; ++j) DEL[TL::at(j, s)] = d[j];
    }
    block_add(term, slot + P_total);  // (contains __syncthreads)
    // output layer: gW_L += DEL^T a_L ; gb_L += rowsum(DEL)
    const T* aL = A0;
    if (nh > 0) {
      const T* z = (Zb + (nh - 1) * TS);
      TL::each(HP, [&](int, int, int q) { P[q] = act_value(a.act, z[q]); });
      __syncthreads();
      aL = P;
    }
    outer_acc1<TL>(slot + a.off.w[L1], out, KL, DEL, aL);
    rowsum_acc<TL>(slot + a.off.b[L1], out, DEL);
    if (nh > 0) {
      // abar = DEL W_L
      tl.gemm_bwd(net.W(L1), DEL, out, accm);
      __syncthreads();
      tl.store(Q, accm, [](T v, int, int) { return v; });
      __syncthreads();
      for (int i = nh - 1; i >= 0; --i) {
        T* zb = (Zb + (i) * TS);
        if (i > 0) {
          const T* zp = (Zb + (i - 1) * TS);
          TL::each(HP, [&](int, int, int q) {
            zb[q] = act_d1(a.act, zb[q]) * Q[q];  // zbar_i (overwrites z_i)
            P[q] = act_value(a.act, zp[q]);       // a_i
          });
        } else {
          TL::each(HP, [&](int, int, int q) { zb[q] = act_d1(a.act, zb[q]) * Q[q]; });
        }
        __syncthreads();
        rowsum_acc<TL>(slot + a.off.b[i], HP, zb);
        outer_acc4<TL>(slot + a.off.w[i], HP, i == 0 ? IP : HP, zb, i == 0 ? A0 : P);
        if (i > 0) {
          tl.gemm_bwd(net.W(i), zb, HP, accm);
          __syncthreads();
          tl.store(Q, accm, [](T v, int, int) { return v; });
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
  if (a.smem_slot)
    for (int64_t i = threadIdx.x; i <= P_total; i += kThreads) gslot[i] = slot[i];
}

// ---- actor prep: actor forward + stage cost + dynamics -> x' (nets.py:319-325) -----
template <typename T>
struct PrepArgs {
  NetConst<T> nc;
  int nh, in, out, act, head;
  const T* params;
  BatchDev<T> b;
  SysDev<T> sys;
  CostDev<T> cost;
  T* xn;      // [rows][n+1]
  T* lstage;  // [rows]
};

template <typename T, int HP, int IP, int S, int SYS>
__global__ void __launch_bounds__(kThreads) actor_prep_kernel(const PrepArgs<T> a) {
  using TL = Tile<T, S, HP>;
  constexpr int nn = SysDims<SYS>::n, mm = SysDims<SYS>::m;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  NetSmem<T, HP, IP, TL::KS> net;
  T* p = net.carve(sm, a.nh, a.in, a.out);
  T* A0 = p;
  T* P0 = A0 + IP * S;
  T* P1 = P0 + HP * S;
  T* OUT = P1 + HP * S;
  net.stage(a.params);
  const TL tl;
  const int64_t ntiles = (a.b.rows + S - 1) / S;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * S;
    __syncthreads();
    load_input_tile<TL>(A0, IP, a.in, a.nc,
                          [&](int s) { return base + s < a.b.rows ? a.b.row(base + s) : (int64_t)-1; },
                          [&](int64_t r, int c) { return a.b.xa[r * a.in + c]; });
    __syncthreads();
    const T* last = forward_hidden(tl, net, a.act, A0, P0, P1, (T*)nullptr);
    forward_output<TL>(net, last, [&](int s, int j, T o) { OUT[j * S + s] = o; });
    __syncthreads();
    for (int s = threadIdx.x; s < S; s += kThreads) {
      if (base + s >= a.b.rows) continue;
      const T* xa = a.b.xa + a.b.row(base + s) * (nn + 1);
      T x[nn], u[mm], xn[nn];
#pragma unroll
      for (int c = 0; c < nn; ++c) x[c] = xa[c];
#pragma unroll
      for (int j = 0; j < mm; ++j) u[j] = head_value(a.head, a.nc, j, OUT[j * S + s]);
      a.lstage[base + s] = cost_and_step<SYS>(a.sys, a.cost, true, x, u, xn);
      T* o = a.xn + (base + s) * (nn + 1);
#pragma unroll
      for (int c = 0; c < nn; ++c) o[c] = xn[c];
      o[nn] = xa[nn] + T(1);
    }
  }
}

__global__ void count_live_kernel(const int64_t* idx, const int64_t* cycle, int64_t stride, const void* xa, int dtype,
                                  int64_t rows, int n, int t_max, int64_t* out) {
  __shared__ unsigned long long acc;
  if (threadIdx.x == 0) acc = 0;
  __syncthreads();
  if (idx && cycle) idx += (*cycle) * stride;
  unsigned long long c = 0;
  for (int64_t b = threadIdx.x; b < rows; b += blockDim.x) {
    int64_t r = idx ? idx[b] : b;
    double t = dtype == CACTO_F32 ? (double)((const float*)xa)[r * (n + 1) + n] : ((const double*)xa)[r * (n + 1) + n];
    c += t < (double)t_max ? 1ull : 0ull;
  }
  atomicAdd(&acc, c);
  __syncthreads();
  if (threadIdx.x == 0) *out = (int64_t)acc;
}

}  // namespace cacto

// ======================================================================================
// launchers / C ABI
// ======================================================================================
using namespace cacto;

int validate_mlp(const cacto_mlp_t* m, const char* who);  // abi.cu
namespace cacto {  // wide.cu (padded hidden width > 64: layer-wise tcgen05 path)
bool is_wide(const cacto_mlp_t* m);
size_t wide_workspace_bytes(const cacto_mlp_t* m, int64_t rows);
int wide_critic_loss(const cacto_mlp_t* cm, const cacto_mlp_t* tm, const cacto_batch_t* bt, double k_s, int boot,
                     void* ws, size_t ws_bytes, cudaStream_t st);
int wide_std_loss(const cacto_mlp_t* sm, const cacto_mlp_t* cm, const cacto_batch_t* bt, void* ws, size_t ws_bytes,
                  cudaStream_t st);
int wide_actor_loss(const cacto_mlp_t* am, const cacto_mlp_t* cm, const cacto_system_t* sys, const cacto_cost_t* cost,
                    const cacto_batch_t* bt, const int64_t* live, void* ws, size_t ws_bytes, cudaStream_t st);
// critic_tc.cu (3 x 64 critic on the tensor cores, large batches)
bool critic_tc_eligible(const cacto_mlp_t* c, const cacto_mlp_t* tgt, int64_t rows);
size_t critic_tc_workspace_bytes(const cacto_mlp_t* c, int64_t rows);
int critic_tc_loss(const cacto_mlp_t* c, const cacto_mlp_t* tgt, const cacto_batch_t* bt, double k_s, void* ws,
                   size_t ws_bytes, cudaStream_t st);
}  // namespace cacto
int cacto_forward_rows(const cacto_mlp_t* mlp, const cacto_batch_t* rows_of, int which, void* out,
                       void* stream);  // forward.cu helper (gathered rows)

// the gradient slot goes to shared memory when the kernel's tiles + slot fit the
// per-CTA limit (CACTO_SMEM_SLOT=0 keeps it in the workspace: A/B measurements)
static int smem_slot_fits(const void* kern, size_t bytes) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("CACTO_SMEM_SLOT");
    env = e ? atoi(e) : 1;
  }
  int dev = 0, maxb = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxb, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  (void)kern;
  return env != 0 && bytes + 1024 <= (size_t)maxb;
}

static int loss_grid(int64_t rows, int S) {
  int64_t tiles = (rows + S - 1) / S;
  int64_t cap = num_sms();
  return (int)(tiles < 1 ? 1 : (tiles < cap ? tiles : cap));
}


extern "C" size_t cacto_loss_workspace_bytes(const cacto_mlp_t* net, int64_t rows) {
  if (!net) return 0;
  if (is_wide(net)) return wide_workspace_bytes(net, rows);
  size_t es = net->dtype == CACTO_F32 ? 4 : 8;
  LayerOffsets lo = layer_offsets(shape_of(*net));
  size_t slots = (size_t)num_sms() * (size_t)(lo.total + 1) * es;
  size_t scratch = (size_t)(rows > 0 ? rows : 1) * (2 * CACTO_MAX_IN + 4) * es;  // prep / target / err arrays
  size_t bytes = ((slots + 255) & ~(size_t)255) + scratch + 256;
  if (net->head == CACTO_HEAD_LINEAR && critic_tc_eligible(net, nullptr, rows)) {
    const size_t tcb = critic_tc_workspace_bytes(net, rows);  // tensor-core critic (critic_tc.cu)
    if (tcb > bytes) bytes = tcb;
  }
  return bytes;
}

static void* scratch_of(const cacto_mlp_t* net, void* ws) {
  size_t es = net->dtype == CACTO_F32 ? 4 : 8;
  LayerOffsets lo = layer_offsets(shape_of(*net));
  size_t slots = (size_t)num_sms() * (size_t)(lo.total + 1) * es;
  return (char*)ws + ((slots + 255) & ~(size_t)255);
}

// samples per CTA tile: 64 (fp32) once the batch gives every SM a tile, else 32 --
// small minibatches (the M-cycle loop's B = 128) then spread over twice the CTAs
// and each CTA's serial layer chain is half as long
static bool small_batch(int64_t rows) { return rows < (int64_t)64 * num_sms(); }
static bool tiny_batch(int64_t rows) { return rows <= (int64_t)16 * num_sms(); }

template <typename T, int HP, int IP, int S>
static int launch_critic_s(const CriticArgs<T>& a, int64_t rows, int* grid_out, cudaStream_t st) {
  size_t el = net_elems<T, HP, IP>(a.nh, 1) + 2 * (size_t)IP * S + (2 * (size_t)a.nh + 2) * HP * S + S +
              (size_t)CACTO_MAX_IN * S;
  if (a.tparams) el += net_elems<T, HP, IP>(a.nh, 1) + S;  // the staged target net + its tile values
  size_t bytes = el * sizeof(T);
  auto kern = critic_kernel<T, HP, IP, S>;
  CriticArgs<T> b = a;
  const size_t slot_bytes = ((size_t)a.off.total + 1 + 3) / 4 * 4 * sizeof(T);
  b.smem_slot = smem_slot_fits((const void*)kern, bytes + slot_bytes);
  if (b.smem_slot) bytes += slot_bytes;
  if (!ensure_smem((const void*)kern, bytes))
    return set_error(CACTO_EUNSUPPORTED, "critic_loss: %zu B shared memory not available", bytes);
  int grid = loss_grid(rows, S);
  kern<<<grid, kThreads, bytes, st>>>(b);
  *grid_out = grid;
  return check_launch("critic_kernel");
}

template <typename T, int HP, int IP>
static int launch_critic(const CriticArgs<T>& a, int64_t rows, int* grid_out, cudaStream_t st) {
  if constexpr (sizeof(T) == 4) {
    if (!small_batch(rows)) return launch_critic_s<T, HP, IP, 64>(a, rows, grid_out, st);
    if constexpr (HP == 64) {
      if (tiny_batch(rows)) return launch_critic_s<T, HP, IP, 16>(a, rows, grid_out, st);
    }
  }
  return launch_critic_s<T, HP, IP, 32>(a, rows, grid_out, st);
}

template <typename T>
static int critic_entry(const cacto_mlp_t* c, const cacto_mlp_t* tgt, const cacto_batch_t* b, double k_s,
                        int boot, void* ws, int32_t* n_partials, cudaStream_t st) {
  NetShape sh = shape_of(*c);
  CriticArgs<T> a{};
  a.nc = net_const<T>(*c);
  a.nh = sh.nh; a.in = sh.in; a.act = sh.act;
  a.params = (const T*)c->params;
  a.off = offs_of(*c);
  a.b = batch_dev<T>(*b);
  a.inv_denom = T(1) / (T)(b->denom > 0 ? b->denom : b->rows);
  a.k_s = (T)k_s;
  a.ws = (T*)ws;
  if (boot && tgt) {
    const NetShape tsh = shape_of(*tgt);
    if (CACTO_CRITIC_FUSED_TARGET && tsh.hp == sh.hp && tsh.ip == sh.ip && tsh.nh == sh.nh && tsh.in == sh.in &&
        tsh.act == sh.act && tsh.head == CACTO_HEAD_LINEAR && tgt->dtype == c->dtype) {
      a.tparams = (const T*)tgt->params;
      a.nc_t = net_const<T>(*tgt);
    } else {
      T* vnext = (T*)scratch_of(c, ws);
      int rc = cacto_forward_rows(tgt, b, /*xa_plus_k*/ 1, vnext, st);
      if (rc) return rc;
      a.v_next = vnext;
    }
  }
  int grid = 0;
  auto launch = [&]() {
    if (sh.hp == 32 && sh.ip == 8) return launch_critic<T, 32, 8>(a, b->rows, &grid, st);
    if (sh.hp == 32 && sh.ip == 16) return launch_critic<T, 32, 16>(a, b->rows, &grid, st);
    if (sh.hp == 64 && sh.ip == 8) return launch_critic<T, 64, 8>(a, b->rows, &grid, st);
    if (sh.hp == 64 && sh.ip == 16) return launch_critic<T, 64, 16>(a, b->rows, &grid, st);
    return set_error(CACTO_EUNSUPPORTED, "critic_loss: hidden %d / input %d not built", sh.hp, sh.in);
  };
  int rc = launch();
  if (rc == CACTO_EUNSUPPORTED && a.tparams) {
    // the staged target does not fit beside the tile (fp64, wide tiles): the separate
    // target forward, then the plain kernel (nothing was launched above)
    a.tparams = nullptr;
    T* vnext = (T*)scratch_of(c, ws);
    rc = cacto_forward_rows(tgt, b, /*xa_plus_k*/ 1, vnext, st);
    if (rc) return rc;
    a.v_next = vnext;
    rc = launch();
  }
  *n_partials = grid;
  return rc;
}

extern "C" int cacto_critic_loss(const cacto_mlp_t* critic, const cacto_mlp_t* target, const cacto_batch_t* batch,
                                 double k_s, int32_t bootstrap, void* workspace, size_t workspace_bytes,
                                 int32_t* n_partials, void* stream) {
  int rc = validate_mlp(critic, "critic_loss");
  if (rc) return rc;
  if (!batch || batch->rows <= 0) return set_error(CACTO_EVALUE, "empty batch");
  if (critic->sizes[critic->n_layers] != 1) return set_error(CACTO_EVALUE, "critic_loss: critic must be scalar");
  if (critic->sizes[0] != batch->n + 1) return set_error(CACTO_EVALUE, "critic_loss: input dim mismatch");
  if (bootstrap && target) {
    rc = validate_mlp(target, "critic_loss(target)");
    if (rc) return rc;
  }
  if (workspace_bytes < cacto_loss_workspace_bytes(critic, batch->rows))
    return set_error(CACTO_EVALUE, "critic_loss: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  if (critic_tc_eligible(critic, bootstrap ? target : nullptr, batch->rows)) {
    *n_partials = 1;
    return critic_tc_loss(critic, bootstrap ? target : nullptr, batch, k_s, workspace, workspace_bytes, st);
  }
  if (is_wide(critic)) {
    *n_partials = 1;
    return wide_critic_loss(critic, bootstrap ? target : nullptr, batch, k_s, bootstrap, workspace, workspace_bytes,
                            st);
  }
  if (critic->dtype == CACTO_F32)
    return critic_entry<float>(critic, target, batch, k_s, bootstrap, workspace, n_partials, st);
  return critic_entry<double>(critic, target, batch, k_s, bootstrap, workspace, n_partials, st);
}

template <typename T, int HP, int IP, int KIND, int SYS, int S>
static int launch_vp_s(const VpArgs<T>& a, int64_t rows, int* grid_out, cudaStream_t st) {
  size_t el = net_elems<T, HP, IP>(a.nh, a.out) + (size_t)IP * S + ((size_t)a.nh + 2) * HP * S +
              (size_t)CACTO_MAX_OUT * S + 4 * ((CACTO_MAX_OUT + 3) / 4) * S;
  size_t bytes = el * sizeof(T);
  auto kern = vp_kernel<T, HP, IP, S, KIND, SYS>;
  VpArgs<T> b = a;
  const size_t slot_bytes = ((size_t)a.off.total + 1 + 3) / 4 * 4 * sizeof(T);
  b.smem_slot = smem_slot_fits((const void*)kern, bytes + slot_bytes);
  if (b.smem_slot) bytes += slot_bytes;
  if (!ensure_smem((const void*)kern, bytes))
    return set_error(CACTO_EUNSUPPORTED, "loss: %zu B shared memory not available", bytes);
  int grid = loss_grid(rows, S);
  kern<<<grid, kThreads, bytes, st>>>(b);
  *grid_out = grid;
  return check_launch("vp_kernel");
}

template <typename T, int HP, int IP, int KIND, int SYS>
static int launch_vp(const VpArgs<T>& a, int64_t rows, int* grid_out, cudaStream_t st) {
  if constexpr (sizeof(T) == 4) {
    if (!small_batch(rows)) return launch_vp_s<T, HP, IP, KIND, SYS, 64>(a, rows, grid_out, st);
    if constexpr (HP == 64) {
      if (tiny_batch(rows)) return launch_vp_s<T, HP, IP, KIND, SYS, 16>(a, rows, grid_out, st);
    }
  }
  return launch_vp_s<T, HP, IP, KIND, SYS, 32>(a, rows, grid_out, st);
}

#define CACTO_VP_DISPATCH(T, KIND, SYS, hp, ip, a, rows, grid, st)                   \
  do {                                                                               \
    if (hp == 32 && ip == 8) return launch_vp<T, 32, 8, KIND, SYS>(a, rows, grid, st);   \
    if (hp == 32 && ip == 16) return launch_vp<T, 32, 16, KIND, SYS>(a, rows, grid, st); \
    if (hp == 64 && ip == 8) return launch_vp<T, 64, 8, KIND, SYS>(a, rows, grid, st);   \
    if (hp == 64 && ip == 16) return launch_vp<T, 64, 16, KIND, SYS>(a, rows, grid, st); \
  } while (0)

template <typename T>
static int std_entry(const cacto_mlp_t* sn, const cacto_mlp_t* cn, const cacto_batch_t* b, void* ws,
                     int32_t* n_partials, cudaStream_t st) {
  // err = v_bar - V(xa)  (nets.py:343)
  T* err = (T*)scratch_of(sn, ws);
  int rc = cacto_forward_rows(cn, b, /*err*/ 2, err, st);
  if (rc) return rc;
  NetShape sh = shape_of(*sn);
  VpArgs<T> a{};
  a.nc = net_const<T>(*sn);
  a.nh = sh.nh; a.in = sh.in; a.out = sh.out; a.act = sh.act; a.head = sh.head;
  a.params = (const T*)sn->params;
  a.off = offs_of(*sn);
  a.b = batch_dev<T>(*b);
  a.inv_denom = T(1) / (T)(b->denom > 0 ? b->denom : b->rows);
  a.err = err;
  a.ws = (T*)ws;
  CACTO_VP_DISPATCH(T, VP_STD, 0, sh.hp, sh.ip, a, b->rows, n_partials, st);
  return set_error(CACTO_EUNSUPPORTED, "std_loss: hidden %d / input %d not built", sh.hp, sh.in);
}

// the std loss from precomputed errors e = v_bar - V(xa) (cacto_value_errors): the
// update loop's std phase runs with the final critic, so every cycle's errors come
// from ONE batched critic forward instead of one per cycle
template <typename T>
static int std_err_entry(const cacto_mlp_t* sn, const void* err, const cacto_batch_t* b, void* ws,
                         int32_t* n_partials, cudaStream_t st) {
  NetShape sh = shape_of(*sn);
  VpArgs<T> a{};
  a.nc = net_const<T>(*sn);
  a.nh = sh.nh; a.in = sh.in; a.out = sh.out; a.act = sh.act; a.head = sh.head;
  a.params = (const T*)sn->params;
  a.off = offs_of(*sn);
  a.b = batch_dev<T>(*b);
  a.inv_denom = T(1) / (T)(b->denom > 0 ? b->denom : b->rows);
  a.err = (const T*)err;
  a.err_cycle = b->cycle;
  a.err_stride = b->idx_stride;
  a.ws = (T*)ws;
  CACTO_VP_DISPATCH(T, VP_STD, 0, sh.hp, sh.ip, a, b->rows, n_partials, st);
  return set_error(CACTO_EUNSUPPORTED, "std_loss: hidden %d / input %d not built", sh.hp, sh.in);
}

extern "C" int cacto_value_errors(const cacto_mlp_t* critic, const cacto_batch_t* batch, void* err, void* stream) {
  int rc = validate_mlp(critic, "value_errors");
  if (rc) return rc;
  if (!batch || !err) return set_error(CACTO_EVALUE, "value_errors: null argument");
  return cacto_forward_rows(critic, batch, /*err*/ 2, err, stream);
}

extern "C" int cacto_std_loss_err(const cacto_mlp_t* std_net, const void* err, const cacto_batch_t* batch,
                                  void* workspace, size_t workspace_bytes, int32_t* n_partials, void* stream) {
  int rc = validate_mlp(std_net, "std_loss");
  if (rc) return rc;
  if (!batch || batch->rows <= 0 || !err) return set_error(CACTO_EVALUE, "empty batch");
  if (std_net->sizes[std_net->n_layers] != 1 || std_net->head != CACTO_HEAD_STD)
    return set_error(CACTO_EVALUE, "std_loss: std net must have a scalar std head");
  if (workspace_bytes < cacto_loss_workspace_bytes(std_net, batch->rows))
    return set_error(CACTO_EVALUE, "std_loss: workspace too small");
  if (is_wide(std_net)) return set_error(CACTO_EUNSUPPORTED, "std_loss_err: wide networks use cacto_std_loss");
  cudaStream_t st = (cudaStream_t)stream;
  if (std_net->dtype == CACTO_F32) return std_err_entry<float>(std_net, err, batch, workspace, n_partials, st);
  return std_err_entry<double>(std_net, err, batch, workspace, n_partials, st);
}

extern "C" int cacto_std_loss(const cacto_mlp_t* std_net, const cacto_mlp_t* critic, const cacto_batch_t* batch,
                              void* workspace, size_t workspace_bytes, int32_t* n_partials, void* stream) {
  int rc = validate_mlp(std_net, "std_loss");
  if (rc) return rc;
  rc = validate_mlp(critic, "std_loss(critic)");
  if (rc) return rc;
  if (!batch || batch->rows <= 0) return set_error(CACTO_EVALUE, "empty batch");
  if (std_net->sizes[std_net->n_layers] != 1 || std_net->head != CACTO_HEAD_STD)
    return set_error(CACTO_EVALUE, "std_loss: std net must have a scalar std head");
  if (workspace_bytes < cacto_loss_workspace_bytes(std_net, batch->rows))
    return set_error(CACTO_EVALUE, "std_loss: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  if (is_wide(std_net)) {
    *n_partials = 1;
    return wide_std_loss(std_net, critic, batch, workspace, workspace_bytes, st);
  }
  if (std_net->dtype == CACTO_F32) return std_entry<float>(std_net, critic, batch, workspace, n_partials, st);
  return std_entry<double>(std_net, critic, batch, workspace, n_partials, st);
}

template <typename T, int HP, int IP, int SYS, int S>
static int launch_prep_s(const PrepArgs<T>& a, cudaStream_t st) {
  size_t el = net_elems<T, HP, IP>(a.nh, a.out) + (size_t)IP * S + 2 * (size_t)HP * S + (size_t)CACTO_MAX_OUT * S;
  size_t bytes = el * sizeof(T);
  auto kern = actor_prep_kernel<T, HP, IP, S, SYS>;
  if (!ensure_smem((const void*)kern, bytes))
    return set_error(CACTO_EUNSUPPORTED, "actor_prep: %zu B shared memory not available", bytes);
  int64_t tiles = (a.b.rows + S - 1) / S;
  int grid = (int)(tiles < 2 * num_sms() ? tiles : 2 * num_sms());
  kern<<<grid, kThreads, bytes, st>>>(a);
  return check_launch("actor_prep_kernel");
}

template <typename T, int HP, int IP, int SYS>
static int launch_prep(const PrepArgs<T>& a, cudaStream_t st) {
  if (!small_batch(a.b.rows)) return launch_prep_s<T, HP, IP, SYS, 64>(a, st);
  if constexpr (HP == 64) {
    if (tiny_batch(a.b.rows)) return launch_prep_s<T, HP, IP, SYS, 16>(a, st);
  }
  return launch_prep_s<T, HP, IP, SYS, 32>(a, st);
}

template <typename T, int SYS>
static int actor_sys(const cacto_mlp_t* an, const cacto_mlp_t* cn, const cacto_system_t* sys,
                     const cacto_cost_t* cost, const cacto_batch_t* b, const int64_t* live, void* ws,
                     int32_t* n_partials, cudaStream_t st) {
  constexpr int nn = SysDims<SYS>::n;
  NetShape sh = shape_of(*an);
  T* scratch = (T*)scratch_of(an, ws);
  int64_t R = b->rows;
  T* xn = scratch;                    // [R][n+1]
  T* gn = xn + R * (nn + 1);          // [R][n+1]
  T* vn = gn + R * (nn + 1);          // [R]
  T* ls = vn + R;                     // [R]
  PrepArgs<T> pa{};
  pa.nc = net_const<T>(*an);
  pa.nh = sh.nh; pa.in = sh.in; pa.out = sh.out; pa.act = sh.act; pa.head = sh.head;
  pa.params = (const T*)an->params;
  pa.b = batch_dev<T>(*b);
  pa.sys = sys_dev<T>(*sys);
  pa.cost = cost_dev<T>(*cost);
  pa.xn = xn;
  pa.lstage = ls;
  int rc = CACTO_EUNSUPPORTED;
  if (sh.hp == 32 && sh.ip == 8) rc = launch_prep<T, 32, 8, SYS>(pa, st);
  else if (sh.hp == 32 && sh.ip == 16) rc = launch_prep<T, 32, 16, SYS>(pa, st);
  else if (sh.hp == 64 && sh.ip == 8) rc = launch_prep<T, 64, 8, SYS>(pa, st);
  else if (sh.hp == 64 && sh.ip == 16) rc = launch_prep<T, 64, 16, SYS>(pa, st);
  else return set_error(CACTO_EUNSUPPORTED, "actor_loss: hidden %d / input %d not built", sh.hp, sh.in);
  if (rc) return rc;
  // value and state gradient of the (updated) critic at (x', t+1)  (nets.py:326)
  rc = cacto_mlp_jacobian(cn, xn, R, vn, gn, st);
  if (rc) return rc;
  VpArgs<T> a{};
  a.nc = pa.nc;
  a.nh = sh.nh; a.in = sh.in; a.out = sh.out; a.act = sh.act; a.head = sh.head;
  a.params = pa.params;
  a.off = offs_of(*an);
  a.b = pa.b;
  a.live_rows = live;
  a.count_live = live == nullptr;
  a.sys = pa.sys;
  a.cost = pa.cost;
  a.xn = xn;
  a.lstage = ls;
  a.vn = vn;
  a.gn = gn;
  a.ws = (T*)ws;
  CACTO_VP_DISPATCH(T, VP_ACTOR, SYS, sh.hp, sh.ip, a, R, n_partials, st);
  return set_error(CACTO_EUNSUPPORTED, "actor_loss: hidden %d / input %d not built", sh.hp, sh.in);
}

template <typename T>
static int actor_entry(const cacto_mlp_t* an, const cacto_mlp_t* cn, const cacto_system_t* sys,
                       const cacto_cost_t* cost, const cacto_batch_t* b, const int64_t* live, void* ws,
                       int32_t* np, cudaStream_t st) {
  switch (sys->kind) {
    case CACTO_SYS_TOY1D: return actor_sys<T, CACTO_SYS_TOY1D>(an, cn, sys, cost, b, live, ws, np, st);
    case CACTO_SYS_POINTMASS: return actor_sys<T, CACTO_SYS_POINTMASS>(an, cn, sys, cost, b, live, ws, np, st);
    case CACTO_SYS_DUBINS: return actor_sys<T, CACTO_SYS_DUBINS>(an, cn, sys, cost, b, live, ws, np, st);
    case CACTO_SYS_MANIPULATOR3: return actor_sys<T, CACTO_SYS_MANIPULATOR3>(an, cn, sys, cost, b, live, ws, np, st);
    case CACTO_SYS_ALIENGO_LIPM: return actor_sys<T, CACTO_SYS_ALIENGO_LIPM>(an, cn, sys, cost, b, live, ws, np, st);
    default: return set_error(CACTO_EUNSUPPORTED, "actor_loss: unknown system %d", sys->kind);
  }
}

extern "C" int cacto_actor_loss(const cacto_mlp_t* actor, const cacto_mlp_t* critic, const cacto_system_t* sys,
                                const cacto_cost_t* cost, const cacto_batch_t* batch, const int64_t* live_rows,
                                void* workspace, size_t workspace_bytes, int32_t* n_partials, void* stream) {
  int rc = validate_mlp(actor, "actor_loss");
  if (rc) return rc;
  rc = validate_mlp(critic, "actor_loss(critic)");
  if (rc) return rc;
  if (!sys || !cost || !batch) return set_error(CACTO_EVALUE, "actor_loss: null argument");
  if (batch->rows <= 0) return set_error(CACTO_EVALUE, "empty batch");
  if (actor->sizes[0] != sys->n + 1 || actor->sizes[actor->n_layers] != sys->m || critic->sizes[0] != sys->n + 1)
    return set_error(CACTO_EVALUE, "actor_loss: dims do not match the system");
  if (critic->dtype != actor->dtype) return set_error(CACTO_EVALUE, "actor_loss: dtype mismatch");
  if (workspace_bytes < cacto_loss_workspace_bytes(actor, batch->rows))
    return set_error(CACTO_EVALUE, "actor_loss: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  if (is_wide(actor)) {
    *n_partials = 1;
    return wide_actor_loss(actor, critic, sys, cost, batch, live_rows, workspace, workspace_bytes, st);
  }
  if (actor->dtype == CACTO_F32)
    return actor_entry<float>(actor, critic, sys, cost, batch, live_rows, workspace, n_partials, st);
  return actor_entry<double>(actor, critic, sys, cost, batch, live_rows, workspace, n_partials, st);
}

extern "C" int cacto_count_live(const cacto_batch_t* batch, int64_t* live_rows, void* stream) {
  if (!batch || !live_rows) return set_error(CACTO_EVALUE, "count_live: null argument");
  count_live_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(batch->idx, batch->cycle, batch->idx_stride, batch->xa,
                                                         batch->dtype, batch->rows, batch->n, batch->t_max, live_rows);
  return check_launch("count_live_kernel");
}
