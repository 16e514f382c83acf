// rollout.cu -- K1: fused closed-loop actor rollout (nets.actor_rollout,
// nets.py:403-423) for a batch of starts.
//
// One CTA owns S starts for the whole horizon.  Per time step:
//   input tile  a0[c][s] = (x_s[c] - center[c]) / half[c], time row t0_s + k
//   hidden      a_{i+1} = act(a_i W_i^T + b_i)        (register-tiled GEMM, smem weights)
//   head        u_s = out_scale * tanh(a W_L^T + b_L)  (4-lane split + shuffles)
//   dynamics    x_s <- f(x_s, u_s), stage cost l(x_s, u_s) accumulated in the
//               thread that owns start s, in NumPy's pairwise-sum order, so
//               cost == Trajectory.cost (ilqr.py:76-78) term for term.
#include <stdlib.h>

#include <algorithm>

#include "net.cuh"
#include "rollout.cuh"
#include "systems.cuh"

namespace cacto {

// S starts per CTA; TM = 8 (8x8 micro-tiles, 1 CTA / SM) for the 256-start
// tile, TM = 4 otherwise
template <typename T, int SYS, int HP, int S>
__global__ void __launch_bounds__(kThreads, ((sizeof(T) == 4 && S <= 128) ? 2 : 1))
rollout_kernel(const RolloutArgs<T> a) {
  using TL = Tile<T, S, HP, (S >= 256 ? 8 : 4)>;
  constexpr int n = SysDims<SYS>::n;
  constexpr int m = SysDims<SYS>::m;
  constexpr int IP = (n + 1) <= 8 ? 8 : ((n + 1) <= 16 ? 16 : 32);
  using NS = NetSmem<T, HP, IP, TL::KS>;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  NS net;
  T* A0 = net.carve(sm, a.nh, n + 1, m);  // [IP][S] input tile
  T* BA = A0 + IP * S;                     // [HP][S]
  T* BB = BA + HP * S;                     // [HP][S]
  T* US = BB + HP * S;                     // [m][S] raw head outputs
  net.stage(a.params);
  // zero the padded input rows once
  for (int p = threadIdx.x; p < IP * S; p += kThreads) A0[p] = T(0);

  // ---- per-start registers (thread s < S owns start s of this tile) ------------
  static_assert(S <= kThreads, "one thread per start");
  const int s_own = threadIdx.x;
  const int64_t gi = (int64_t)blockIdx.x * S + s_own;
  const bool owner = s_own < S && gi < a.N;
  T x[n];
  int t0 = 0, T_i = 0;
  PairwiseSum<T> acc;
  if (owner) {
#pragma unroll
    for (int c = 0; c < n; ++c) x[c] = (T)a.x0[gi * n + c];
    t0 = a.t0 ? a.t0[gi] : a.t0_scalar;
    T_i = a.t_hor >= 0 ? a.t_hor : (a.sys.t_max - t0);
    acc.init(T_i + 1);
    if (a.X) {
#pragma unroll
      for (int c = 0; c < n; ++c) a.X[gi * (int64_t)(a.t_stride + 1) * n + c] = x[c];
    }
  } else {
#pragma unroll
    for (int c = 0; c < n; ++c) x[c] = T(0);
  }
  // block-wide horizon (max over owned starts)
  __shared__ int s_kmax;
  if (threadIdx.x == 0) s_kmax = 0;
  __syncthreads();
  if (owner) atomicMax(&s_kmax, T_i);
  __syncthreads();
  const int kmax = s_kmax;

  const TL tl;
  for (int k = 0; k < kmax; ++k) {
    // ---- normalised network input [x, t0 + k] (nets.py:416, 126-129) ----------
    if (owner) {
#pragma unroll
      for (int c = 0; c < n; ++c) A0[TL::at(c, s_own)] = (x[c] - a.nc.in_center[c]) / a.nc.in_half[c];
      A0[TL::at(n, s_own)] = ((T)(t0 + k) - a.nc.in_center[n]) / a.nc.in_half[n];
    } else if (s_own < S) {
#pragma unroll
      for (int c = 0; c <= n; ++c) A0[TL::at(c, s_own)] = T(0);
    }
    __syncthreads();
    const T* last = forward_hidden(tl, net, a.act, A0, BA, BB, (T*)nullptr);
    forward_output<TL>(net, last, [&](int s, int j, T v) { US[j * S + s] = v; });
    __syncthreads();
    // ---- head, running cost, dynamics (thread per start) -----------------------
    if (owner && k < T_i) {
      T u[m];
#pragma unroll
      for (int j = 0; j < m; ++j) u[j] = head_value(a.head, a.nc, j, US[j * S + s_own]);
      if (a.U) {
#pragma unroll
        for (int j = 0; j < m; ++j) a.U[a.u_at(gi, k, j, m)] = u[j];
      }
      T xn[n];
      const T sc = cost_and_step<SYS>(a.sys, a.cost, a.has_cost, x, u, xn);
      acc.add(k, sc);
      if (a.SC) a.SC[gi * (int64_t)(a.t_stride + 1) + k] = sc;
#pragma unroll
      for (int c = 0; c < n; ++c) x[c] = xn[c];
      if (a.X) {
#pragma unroll
        for (int c = 0; c < n; ++c) a.X[(gi * (int64_t)(a.t_stride + 1) + k + 1) * n + c] = x[c];
      }
    }
    // the next iteration's first barrier orders A0 writes after these US reads
  }
  if (owner) {
    T term = a.has_cost ? terminal_cost<SYS>(a.sys, a.cost, x) : T(0);
    acc.add(T_i, term);
    if (a.SC) a.SC[gi * (int64_t)(a.t_stride + 1) + T_i] = term;
    if (a.C) a.C[gi] = acc.res;
  }
}

template <typename T, int SYS, int HP, int S>
static int launch_rollout_s(const RolloutArgs<T>& a, cudaStream_t st) {
  constexpr int n = SysDims<SYS>::n, m = SysDims<SYS>::m;
  constexpr int IP = (n + 1) <= 8 ? 8 : ((n + 1) <= 16 ? 16 : 32);
  using NS = NetSmem<T, HP, IP, Tile<T, S, HP, (S >= 256 ? 8 : 4)>::KS>;
  size_t elems = NS::elems(a.nh, m) + (size_t)IP * S + 2 * (size_t)HP * S + (size_t)m * S;
  size_t bytes = elems * sizeof(T);
  auto kern = rollout_kernel<T, SYS, HP, S>;
  if (!ensure_smem((const void*)kern, bytes))
    return set_error(CACTO_ECUDA, "rollout: %zu B of shared memory not available", bytes);
  int64_t blocks = (a.N + S - 1) / S;
  kern<<<(unsigned)blocks, kThreads, bytes, st>>>(a);
  return check_launch("rollout_kernel");
}

// Tile size: 128 starts per CTA (2 CTAs / SM) when the batch fills the GPU,
// 32-start tiles for small batches (e.g. the kept warm-start re-rollout) so
// that the CTAs still cover every SM.
static int tile_override() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CACTO_ROLLOUT_TILE");  // 128 / 256 (experiments)
    v = e ? atoi(e) : 0;
  }
  return v;
}

// rollout_tc.cu: the tensor-core rollout (fp32, n + 1 <= 16, 1..3 hidden layers)
template <int SYS, int HP>
int launch_rollout_tc(const RolloutArgs<float>& a, cudaStream_t st);
bool rollout_tc_enabled();

template <typename T, int SYS, int HP>
static int launch_rollout(const RolloutArgs<T>& a, cudaStream_t st) {
  if constexpr (sizeof(T) == 4) {
    if (rollout_tc_enabled() && a.nh >= 1 && a.nh <= 3 && SysDims<SYS>::n + 1 <= 16 && SysDims<SYS>::m <= 8)
      return launch_rollout_tc<SYS, HP>(a, st);
    // 128-start tiles (2 CTAs / SM, 4x8 micro-tiles) measured faster than 256-start
    // tiles (1 CTA / SM, 8x8) on B200: 4.13 vs 4.57 ms (profiles/README.md)
    const int ov = tile_override();
    if (ov == 256 && a.N >= (int64_t)256 * num_sms() && HP == 64) return launch_rollout_s<T, SYS, HP, 256>(a, st);
    if (a.N >= (int64_t)128 * num_sms()) return launch_rollout_s<T, SYS, HP, 128>(a, st);
    return launch_rollout_s<T, SYS, HP, 32>(a, st);
  } else {
    if (a.N >= (int64_t)64 * num_sms()) return launch_rollout_s<T, SYS, HP, 64>(a, st);
    return launch_rollout_s<T, SYS, HP, 32>(a, st);
  }
}

template <typename T>
static int dispatch_rollout(const RolloutArgs<T>& a, int kind, int hp, cudaStream_t st) {
#define CACTO_ROLL_CASE(SYSK)                                              \
  case SYSK:                                                               \
    if (hp == 32) return launch_rollout<T, SYSK, 32>(a, st);               \
    if (hp == 64) return launch_rollout<T, SYSK, 64>(a, st);               \
    break;
  switch (kind) {
    CACTO_ROLL_CASE(CACTO_SYS_TOY1D)
    CACTO_ROLL_CASE(CACTO_SYS_POINTMASS)
    CACTO_ROLL_CASE(CACTO_SYS_DUBINS)
    CACTO_ROLL_CASE(CACTO_SYS_MANIPULATOR3)
    CACTO_ROLL_CASE(CACTO_SYS_ALIENGO_LIPM)
    default:
      break;
  }
#undef CACTO_ROLL_CASE
  return set_error(CACTO_EUNSUPPORTED, "rollout: system kind %d with hidden width %d not built", kind, hp);
}

}  // namespace cacto

using namespace cacto;

static int system_dims_ok(const cacto_system_t* s) {
  static const int dims[5][2] = {{1, 1}, {4, 2}, {5, 2}, {6, 3}, {15, 6}};
  if (s->kind < 0 || s->kind > 4) return 0;
  return s->n == dims[s->kind][0] && s->m == dims[s->kind][1];
}

extern "C" int cacto_rollout(const cacto_system_t* sys, const cacto_cost_t* cost, const cacto_mlp_t* actor,
                             const double* x0, const int32_t* t0, int32_t t0_scalar, int64_t N, int32_t t_hor,
                             void* U, void* X, void* step_costs, void* cost_to_go, void* stream) {
  return cacto_rollout_ex(sys, cost, actor, x0, t0, t0_scalar, N, t_hor, 0, U, X, step_costs, cost_to_go, stream);
}

namespace cacto {
// a block takes 8 kept columns: their indices loaded once, then every thread copies
// rows r = tid, tid + blockDim, ... of all 8 (8 independent scattered loads in flight
// per thread, coalesced stores along r); 32-bit row arithmetic
template <typename T>
__global__ void __launch_bounds__(128) take_columns_kernel(const T* __restrict__ src, int64_t R, int64_t N,
                                                           const int64_t* __restrict__ idx, int64_t K, T* dst) {
  const int64_t i0 = (int64_t)blockIdx.x * 8;
  int64_t col[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) col[u] = i0 + u < K ? idx[i0 + u] : -1;
  const int r_n = (int)R;
  for (int r = threadIdx.x; r < r_n; r += blockDim.x) {
    const T* row = src + (int64_t)r * N;
    T v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = col[u] >= 0 ? __ldg(row + col[u]) : T(0);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (col[u] >= 0) dst[(i0 + u) * R + r] = v[u];
  }
}
// dst[i, :] = src[idx[i], :] for rows of R elements: one warp per row, 16-byte
// vectors when the rows allow (the kept warm starts of a start-major U)
template <typename T>
__global__ void take_rows_kernel(const T* __restrict__ src, int64_t R, const int64_t* __restrict__ idx, int64_t K,
                                 T* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = (R * (int64_t)sizeof(T)) % 16 == 0 && ((uintptr_t)src % 16) == 0 && ((uintptr_t)dst % 16) == 0;
  for (int64_t i = w0; i < K; i += nw) {
    const int64_t r = idx[i];
    if (vec) {
      const int64_t nv = R * (int64_t)sizeof(T) / 16;
      const float4* s4 = reinterpret_cast<const float4*>(src + r * R);
      float4* d4 = reinterpret_cast<float4*>(dst + i * R);
      for (int64_t v = lane; v < nv; v += 32) d4[v] = __ldg(s4 + v);
    } else {
      for (int64_t e = lane; e < R; e += 32) dst[i * R + e] = src[r * R + e];
    }
  }
}
// dst[k, t, :] = src[t, idx[k], :] for a step-major U [T][N][M]: one warp per kept
// start, lanes over its T steps (M contiguous values each: one sector per step instead
// of one per (step, control) of the time-major column take), coalesced stores along
// the kept start's [T][M] row
template <typename T_>
__global__ void take_steps_kernel(const T_* __restrict__ src, int64_t T, int64_t N, int M,
                                  const int64_t* __restrict__ idx, int64_t K, T_* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < K; i += nw) {
    const int64_t col = idx[i];
    T_* d = dst + i * T * M;
    for (int64_t t = lane; t < T; t += 32) {
      const T_* s = src + (t * N + col) * M;
      for (int j = 0; j < M; ++j) d[t * M + j] = __ldg(s + j);
    }
  }
}
}  // namespace cacto

extern "C" int cacto_take_steps(int32_t dtype, const void* src, int64_t T, int64_t N, int32_t M, const int64_t* idx,
                                int64_t K, void* dst, void* stream) {
  if (T < 0 || N < 0 || M <= 0 || K < 0 || (T * K > 0 && (!src || !idx || !dst)))
    return set_error(CACTO_EVALUE, "take_steps: bad arguments");
  if (T * K == 0) return CACTO_OK;
  const unsigned grid = (unsigned)std::min<int64_t>((K + 7) / 8, 32 * (int64_t)num_sms());
  if (dtype == CACTO_F32)
    take_steps_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>((const float*)src, T, N, M, idx, K, (float*)dst);
  else
    take_steps_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>((const double*)src, T, N, M, idx, K,
                                                                       (double*)dst);
  return check_launch("take_steps_kernel");
}

extern "C" int cacto_take_rows(int32_t dtype, const void* src, int64_t R, const int64_t* idx, int64_t K, void* dst,
                               void* stream) {
  if (R < 0 || K < 0 || (R * K > 0 && (!src || !idx || !dst))) return set_error(CACTO_EVALUE, "take_rows: bad arguments");
  if (R * K == 0) return CACTO_OK;
  unsigned grid = (unsigned)std::min<int64_t>((K + 7) / 8, 16 * (int64_t)num_sms());
  if (dtype == CACTO_F32)
    take_rows_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>((const float*)src, R, idx, K, (float*)dst);
  else
    take_rows_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>((const double*)src, R, idx, K, (double*)dst);
  return check_launch("take_rows_kernel");
}

extern "C" int cacto_take_columns(int32_t dtype, const void* src, int64_t R, int64_t N, const int64_t* idx, int64_t K,
                                  void* dst, void* stream) {
  if (R < 0 || N < 0 || K < 0 || (R * K > 0 && (!src || !idx || !dst)))
    return set_error(CACTO_EVALUE, "take_columns: bad arguments");
  if (R * K == 0) return CACTO_OK;
  if (R > 0x7fffffff || (K + 7) / 8 > 0x7fffffff) return set_error(CACTO_EVALUE, "take_columns: too large");
  const unsigned grid = (unsigned)((K + 7) / 8);
  if (dtype == CACTO_F32)
    take_columns_kernel<float><<<grid, 128, 0, (cudaStream_t)stream>>>((const float*)src, R, N, idx, K, (float*)dst);
  else
    take_columns_kernel<double><<<grid, 128, 0, (cudaStream_t)stream>>>((const double*)src, R, N, idx, K,
                                                                         (double*)dst);
  return check_launch("take_columns_kernel");
}

extern "C" int cacto_rollout_ex(const cacto_system_t* sys, const cacto_cost_t* cost, const cacto_mlp_t* actor,
                                const double* x0, const int32_t* t0, int32_t t0_scalar, int64_t N, int32_t t_hor,
                                int32_t flags, void* U, void* X, void* step_costs, void* cost_to_go, void* stream) {
  if ((flags & ~(CACTO_ROLLOUT_U_TIME_MAJOR | CACTO_ROLLOUT_U_STEP_MAJOR)) ||
      (flags & CACTO_ROLLOUT_U_TIME_MAJOR && flags & CACTO_ROLLOUT_U_STEP_MAJOR))
    return set_error(CACTO_EVALUE, "rollout: unknown flags %d", flags);
  if (!sys || !actor || !x0) return set_error(CACTO_EVALUE, "rollout: null argument");
  if (!system_dims_ok(sys)) return set_error(CACTO_EUNSUPPORTED, "rollout: unknown system kind %d / dims", sys->kind);
  if (N < 0) return set_error(CACTO_EVALUE, "rollout: N < 0");
  if (actor->sizes[0] != sys->n + 1 || actor->sizes[actor->n_layers] != sys->m)
    return set_error(CACTO_EVALUE, "rollout: actor dims [%d -> %d] do not match system (n=%d, m=%d)",
                     actor->sizes[0], actor->sizes[actor->n_layers], sys->n, sys->m);
  if (t_hor < CACTO_FULL_HORIZON) return set_error(CACTO_EVALUE, "rollout: negative horizon %d", t_hor);
  if (!t0 && (t_hor > sys->t_max - t0_scalar || t0_scalar > sys->t_max))
    return set_error(CACTO_EVALUE, "rollout of %d steps exceeds horizon from t=%d", t_hor, t0_scalar);
  if (N == 0) return CACTO_OK;
  int stride = t_hor >= 0 ? t_hor : sys->t_max;
  cudaStream_t st = (cudaStream_t)stream;
  NetShape sh = shape_of(*actor);
  if (actor->dtype == CACTO_F32) {
    RolloutArgs<float> a{};
    a.sys = sys_dev<float>(*sys);
    if (cost) a.cost = cost_dev<float>(*cost);
    a.nc = net_const<float>(*actor);
    a.has_cost = cost != nullptr;
    a.nh = sh.nh; a.out = sh.out; a.act = sh.act; a.head = sh.head;
    a.params = (const float*)actor->params;
    a.x0 = x0; a.t0 = t0; a.t0_scalar = t0_scalar; a.N = N; a.t_hor = t_hor; a.t_stride = stride;
    a.u_tmajor = (flags & CACTO_ROLLOUT_U_TIME_MAJOR) ? 1 : ((flags & CACTO_ROLLOUT_U_STEP_MAJOR) ? 2 : 0);
    a.U = (float*)U; a.X = (float*)X; a.SC = (float*)step_costs; a.C = (float*)cost_to_go;
    return dispatch_rollout(a, sys->kind, sh.hp, st);
  }
  RolloutArgs<double> a{};
  a.sys = sys_dev<double>(*sys);
  if (cost) a.cost = cost_dev<double>(*cost);
  a.nc = net_const<double>(*actor);
  a.has_cost = cost != nullptr;
  a.nh = sh.nh; a.out = sh.out; a.act = sh.act; a.head = sh.head;
  a.params = (const double*)actor->params;
  a.x0 = x0; a.t0 = t0; a.t0_scalar = t0_scalar; a.N = N; a.t_hor = t_hor; a.t_stride = stride;
  a.u_tmajor = (flags & CACTO_ROLLOUT_U_TIME_MAJOR) ? 1 : ((flags & CACTO_ROLLOUT_U_STEP_MAJOR) ? 2 : 0);
  a.U = (double*)U; a.X = (double*)X; a.SC = (double*)step_costs; a.C = (double*)cost_to_go;
  return dispatch_rollout(a, sys->kind, sh.hp, st);
}

// ---- K1 + K2 in one launch: rollout with the BIC scores of the same starts -------
int validate_mlp(const cacto_mlp_t* m, const char* who);  // abi.cu

static bool same_body(const cacto_mlp_t* a, const cacto_mlp_t* b) {
  return b->dtype == a->dtype && b->hp == a->hp && b->n_layers == a->n_layers && b->activation == a->activation &&
         b->sizes[0] == a->sizes[0];
}

extern "C" int cacto_rollout_score(const cacto_system_t* sys, const cacto_cost_t* cost, const cacto_mlp_t* actor,
                                   int32_t mode, const cacto_mlp_t* std_net, const cacto_mlp_t* critic,
                                   const double* x0, int32_t t0_scalar, int64_t N, int32_t t_hor, int32_t flags,
                                   void* U, void* cost_to_go, void* scores, void* stream) {
  if (mode < 0 || mode > 2) return set_error(CACTO_EVALUE, "rollout_score: unknown mode %d", mode);
  if (!scores) return set_error(CACTO_EVALUE, "rollout_score: null scores");
  if ((flags & ~(CACTO_ROLLOUT_U_TIME_MAJOR | CACTO_ROLLOUT_U_STEP_MAJOR)) ||
      (flags & CACTO_ROLLOUT_U_TIME_MAJOR && flags & CACTO_ROLLOUT_U_STEP_MAJOR))
    return set_error(CACTO_EVALUE, "rollout_score: unknown flags %d", flags);
  if (!sys || !actor || !x0) return set_error(CACTO_EVALUE, "rollout_score: null argument");
  if (!system_dims_ok(sys)) return set_error(CACTO_EUNSUPPORTED, "rollout_score: unknown system kind %d", sys->kind);
  const bool need_std = mode != CACTO_SCORE_GAP, need_crit = mode != CACTO_SCORE_STD;
  int rc = validate_mlp(actor, "rollout_score(actor)");
  if (rc) return rc;
  if (need_std && (rc = validate_mlp(std_net, "rollout_score(std)"))) return rc;
  if (need_crit && (rc = validate_mlp(critic, "rollout_score(critic)"))) return rc;
  if (need_crit && !cost) return set_error(CACTO_EVALUE, "rollout_score: gap modes need the cost field");
  if (actor->sizes[0] != sys->n + 1 || actor->sizes[actor->n_layers] != sys->m)
    return set_error(CACTO_EVALUE, "rollout_score: actor dims do not match the system");
  if (need_std && (std_net->sizes[std_net->n_layers] != 1 || std_net->head != CACTO_HEAD_STD))
    return set_error(CACTO_EVALUE, "rollout_score: std net must be scalar with a std head");
  if (need_crit && critic->sizes[critic->n_layers] != 1)
    return set_error(CACTO_EVALUE, "rollout_score: critic must be scalar");
  if (t_hor < 0 || t_hor > sys->t_max - t0_scalar)
    return set_error(CACTO_EVALUE, "rollout of %d steps exceeds horizon from t=%d", t_hor, t0_scalar);
  // fused only on the tensor-core path with nets of the actor's shape
  NetShape sh = shape_of(*actor);
  const bool tc_ok = actor->dtype == CACTO_F32 && rollout_tc_enabled() && sh.nh >= 1 && sh.nh <= 3 &&
                     (sh.hp == 32 || sh.hp == 64) && sys->n + 1 <= 16 && sys->m <= 8 &&
                     (!need_std || same_body(actor, std_net)) && (!need_crit || same_body(actor, critic));
  if (!tc_ok) return set_error(CACTO_EUNSUPPORTED, "rollout_score: fused scoring needs the fp32 tensor-core path");
  if (N == 0) return CACTO_OK;
  RolloutArgs<float> a{};
  a.sys = sys_dev<float>(*sys);
  if (cost) a.cost = cost_dev<float>(*cost);
  a.nc = net_const<float>(*actor);
  a.has_cost = cost != nullptr;
  a.nh = sh.nh; a.out = sh.out; a.act = sh.act; a.head = sh.head;
  a.params = (const float*)actor->params;
  a.x0 = x0; a.t0 = nullptr; a.t0_scalar = t0_scalar; a.N = N; a.t_hor = t_hor;
  a.t_stride = t_hor;
  a.u_tmajor = (flags & CACTO_ROLLOUT_U_TIME_MAJOR) ? 1 : ((flags & CACTO_ROLLOUT_U_STEP_MAJOR) ? 2 : 0);
  a.U = (float*)U; a.C = (float*)cost_to_go;
  if (need_std) {
    a.pre_kind[a.n_pre] = 0;
    a.pre_params[a.n_pre] = (const float*)std_net->params;
    a.pre_nc[a.n_pre] = net_const<float>(*std_net);
    ++a.n_pre;
  }
  if (need_crit) {
    a.pre_kind[a.n_pre] = 1;
    a.pre_params[a.n_pre] = (const float*)critic->params;
    a.pre_nc[a.n_pre] = net_const<float>(*critic);
    ++a.n_pre;
  }
  a.score_mode = mode;
  a.scores = (float*)scores;
  cudaStream_t st = (cudaStream_t)stream;
#define CACTO_RS_CASE(SYSK)                                                    \
  case SYSK:                                                                   \
    return sh.hp == 32 ? launch_rollout_tc<SYSK, 32>(a, st) : launch_rollout_tc<SYSK, 64>(a, st);
  switch (sys->kind) {
    CACTO_RS_CASE(CACTO_SYS_TOY1D)
    CACTO_RS_CASE(CACTO_SYS_POINTMASS)
    CACTO_RS_CASE(CACTO_SYS_DUBINS)
    CACTO_RS_CASE(CACTO_SYS_MANIPULATOR3)
    CACTO_RS_CASE(CACTO_SYS_ALIENGO_LIPM)
    default:
      break;
  }
#undef CACTO_RS_CASE
  return set_error(CACTO_EUNSUPPORTED, "rollout_score: system kind %d", sys->kind);
}
