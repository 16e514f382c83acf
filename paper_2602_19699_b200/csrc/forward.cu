// forward.cu -- batched network forward (nets.mlp_forward, nets.py:165-173),
// per-sample input Jacobian (nets.mlp_input_gradient / value_and_state_grad,
// nets.py:176-206) and the fused BIC score (trainer.py:150-151 std mode;
// north_star gap mode |V(x0) - J(x0)|).
#include <type_traits>

#include "net.cuh"

namespace cacto {

template <typename T>
constexpr int fwd_S() { return sizeof(T) == 4 ? 64 : 32; }  // samples per tile (large batches)

// samples per tile for a batch of `rows`: fp32 uses 64 once every SM gets a tile,
// else 32 (16 for tiny batches at hidden 64) so small minibatches spread over
// more CTAs; fp64 always 32
template <typename T, int HP, typename F>
static int with_tile(int64_t rows, F f) {
  if constexpr (sizeof(T) == 4) {
    if (rows >= (int64_t)64 * num_sms()) return f(std::integral_constant<int, 64>());
    if constexpr (HP == 64) {
      if (rows <= (int64_t)16 * num_sms()) return f(std::integral_constant<int, 16>());
    }
  }
  return f(std::integral_constant<int, 32>());
}

template <typename T>
struct FwdArgs {
  NetConst<T> nc;
  int nh, in, out, act, head;
  const T* params;
  const T* xa;
  int64_t B;
  T* out_y;    // [B][out] head values
  T* out_jac;  // [B][out][in] (jacobian kernel)
};

template <typename T, int HP, int IP, int S>
__global__ void __launch_bounds__(kThreads) mlp_forward_kernel(const FwdArgs<T> a) {
  using TL = Tile<T, S, HP>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  NetSmem<T, HP, IP, TL::KS> net;
  T* p = net.carve(sm, a.nh, a.in, a.out);
  T* A0 = p;
  T* P0 = A0 + IP * S;
  T* P1 = P0 + HP * S;
  net.stage(a.params);
  const TL tl;
  const int64_t ntiles = (a.B + S - 1) / S;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * S;
    __syncthreads();
    load_input_tile<TL>(A0, IP, a.in, a.nc, [&](int s) { return base + s < a.B ? base + s : (int64_t)-1; },
                          [&](int64_t r, int c) { return a.xa[r * a.in + c]; });
    __syncthreads();
    const T* last = forward_hidden(tl, net, a.act, A0, P0, P1, (T*)nullptr);
    forward_output<TL>(net, last, [&](int s, int j, T o) {
      if (base + s < a.B) a.out_y[(base + s) * a.out + j] = head_value(a.head, a.nc, j, o);
    });
  }
}

template <typename T, int HP, int IP, int S>
__global__ void __launch_bounds__(kThreads) mlp_jacobian_kernel(const FwdArgs<T> a) {
  using TL = Tile<T, S, HP>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  NetSmem<T, HP, IP, TL::KS> net;
  T* p = net.carve(sm, a.nh, a.in, a.out);
  T* A0 = p;
  T* P0 = A0 + IP * S;
  T* P1 = P0 + HP * S;
  T* Zb = P1 + HP * S;  // nh x [HP][S]
  T* OUT = Zb + (size_t)(a.nh > 0 ? a.nh : 1) * HP * S;  // [out][S] raw outputs
  net.stage(a.params);
  const TL tl;
  const int64_t ntiles = (a.B + S - 1) / S;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * S;
    __syncthreads();
    load_input_tile<TL>(A0, IP, a.in, a.nc, [&](int s) { return base + s < a.B ? base + s : (int64_t)-1; },
                          [&](int64_t r, int c) { return a.xa[r * a.in + c]; });
    __syncthreads();
    const T* last = forward_hidden(tl, net, a.act, A0, P0, P1, Zb);
    forward_output<TL>(net, last, [&](int s, int j, T o) {
      OUT[j * S + s] = o;
      if (base + s < a.B) a.out_y[(base + s) * a.out + j] = head_value(a.head, a.nc, j, o);
    });
    __syncthreads();
    for (int j = 0; j < a.out; ++j) {
      input_grad_sweep(tl, net, a.act, j, Zb, (T*)nullptr, P0, P1, [&](int s, int c, T v) {
        if (base + s < a.B) {
          T chain = head_chain(a.head, a.nc, j, OUT[j * S + s]);
          a.out_jac[((base + s) * a.out + j) * a.in + c] = v * chain / a.nc.in_half[c];
        }
      });
    }
  }
}

// ---- BIC scores ---------------------------------------------------------------
template <typename T>
struct ScoreArgs {
  int mode;
  NetConst<T> nc_std, nc_crit;
  int nh_std, nh_crit, in, act_std, act_crit, head_std;
  const T* p_std;
  const T* p_crit;
  const T* xa;
  const T* rollout_cost;
  int64_t N;
  T* scores;
};

template <typename T, int HP, int IP>
__global__ void __launch_bounds__(kThreads) score_kernel(const ScoreArgs<T> a) {
  constexpr int S = fwd_S<T>();
  using TL = Tile<T, S, HP>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const bool need_std = a.mode != CACTO_SCORE_GAP;
  const bool need_crit = a.mode != CACTO_SCORE_STD;
  NetSmem<T, HP, IP, TL::KS> nstd, ncrit;
  T* p = sm;
  if (need_std) p = nstd.carve(p, a.nh_std, a.in, 1);
  if (need_crit) p = ncrit.carve(p, a.nh_crit, a.in, 1);
  T* A0 = p;
  T* P0 = A0 + IP * S;
  T* P1 = P0 + HP * S;
  T* SIG = P1 + HP * S;  // [S]
  if (need_std) nstd.stage(a.p_std);
  if (need_crit) ncrit.stage(a.p_crit);
  const TL tl;
  const int64_t ntiles = (a.N + S - 1) / S;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * S;
    __syncthreads();
    if (need_std) {
      load_input_tile<TL>(A0, IP, a.in, a.nc_std,
                            [&](int s) { return base + s < a.N ? base + s : (int64_t)-1; },
                            [&](int64_t r, int c) { return a.xa[r * a.in + c]; });
      __syncthreads();
      const T* last = forward_hidden(tl, nstd, a.act_std, A0, P0, P1, (T*)nullptr);
      forward_output<TL>(nstd, last, [&](int s, int, T o) {
        T sig = head_value(a.head_std, a.nc_std, 0, o);
        SIG[s] = sig;
        if (a.mode == CACTO_SCORE_STD && base + s < a.N) a.scores[base + s] = sig;
      });
      __syncthreads();
    }
    if (need_crit) {
      load_input_tile<TL>(A0, IP, a.in, a.nc_crit,
                            [&](int s) { return base + s < a.N ? base + s : (int64_t)-1; },
                            [&](int64_t r, int c) { return a.xa[r * a.in + c]; });
      __syncthreads();
      const T* last = forward_hidden(tl, ncrit, a.act_crit, A0, P0, P1, (T*)nullptr);
      forward_output<TL>(ncrit, last, [&](int s, int, T v) {
        if (base + s < a.N) {
          T gap = fabs(v - a.rollout_cost[base + s]);
          a.scores[base + s] = a.mode == CACTO_SCORE_GAP ? gap : SIG[s] * gap;
        }
      });
    }
  }
}

template <typename T, int HP, int IP, typename K>
static int launch_tiles(K kern, size_t smem_elems, int64_t rows, cudaStream_t st, const char* name,
                        const void* args_ptr, int S = fwd_S<T>()) {
  size_t bytes = smem_elems * sizeof(T);
  if (!ensure_smem((const void*)kern, bytes))
    return set_error(CACTO_ECUDA, "%s: %zu B of shared memory not available", name, bytes);
  int64_t tiles = (rows + S - 1) / S;
  int64_t grid = tiles < 4 * num_sms() ? tiles : 4 * num_sms();
  if (grid < 1) grid = 1;
  (void)args_ptr;
  return (int)grid;  // caller launches (kernel args differ)
}

template <typename T, int HP, int IP>
static int run_forward(const FwdArgs<T>& a, bool jac, cudaStream_t st) {
  return with_tile<T, HP>(a.B, [&](auto s_) {
    constexpr int S = decltype(s_)::value;
    size_t net_el = net_elems<T, HP, IP>(a.nh, a.out);
    size_t el = net_el + (size_t)IP * S + 2 * (size_t)HP * S;
    if (jac) el += (size_t)(a.nh > 0 ? a.nh : 1) * HP * S + (size_t)a.out * S;
    int grid;
    if (jac) {
      auto kern = mlp_jacobian_kernel<T, HP, IP, S>;
      grid = launch_tiles<T, HP, IP>(kern, el, a.B, st, "mlp_jacobian", &a, S);
      if (grid < 0) return grid;
      kern<<<grid, kThreads, el * sizeof(T), st>>>(a);
      return check_launch("mlp_jacobian_kernel");
    }
    auto kern = mlp_forward_kernel<T, HP, IP, S>;
    grid = launch_tiles<T, HP, IP>(kern, el, a.B, st, "mlp_forward", &a, S);
    if (grid < 0) return grid;
    kern<<<grid, kThreads, el * sizeof(T), st>>>(a);
    return check_launch("mlp_forward_kernel");
  });
}

template <typename T, int HP, int IP>
static int run_score(const ScoreArgs<T>& a, cudaStream_t st) {
  constexpr int S = fwd_S<T>();
  size_t el = (size_t)IP * S + 2 * (size_t)HP * S + S;
  if (a.mode != CACTO_SCORE_GAP) el += net_elems<T, HP, IP>(a.nh_std, 1);
  if (a.mode != CACTO_SCORE_STD) el += net_elems<T, HP, IP>(a.nh_crit, 1);
  auto kern = score_kernel<T, HP, IP>;
  int grid = launch_tiles<T, HP, IP>(kern, el, a.N, st, "score", &a);
  if (grid < 0) return grid;
  kern<<<grid, kThreads, el * sizeof(T), st>>>(a);
  return check_launch("score_kernel");
}

// dispatch on (hp, ip)
#define CACTO_HP_IP_DISPATCH(FN, T, hp_, ip, ...)                             \
  do {                                                                        \
    const int hp = (hp_) == 0 ? 32 : (hp_);                                   \
    if (hp == 32 && ip == 8) return FN<T, 32, 8>(__VA_ARGS__);                \
    if (hp == 32 && ip == 16) return FN<T, 32, 16>(__VA_ARGS__);              \
    if (hp == 32 && ip == 32) return FN<T, 32, 32>(__VA_ARGS__);              \
    if (hp == 64 && ip == 8) return FN<T, 64, 8>(__VA_ARGS__);                \
    if (hp == 64 && ip == 16) return FN<T, 64, 16>(__VA_ARGS__);              \
    if (hp == 64 && ip == 32) return FN<T, 64, 32>(__VA_ARGS__);              \
  } while (0)

template <typename T>
static int forward_entry(const cacto_mlp_t* m, const void* xa, int64_t B, void* y, void* jac, cudaStream_t st) {
  NetShape sh = shape_of(*m);
  FwdArgs<T> a{};
  a.nc = net_const<T>(*m);
  a.nh = sh.nh; a.in = sh.in; a.out = sh.out; a.act = sh.act; a.head = sh.head;
  a.params = (const T*)m->params;
  a.xa = (const T*)xa;
  a.B = B;
  a.out_y = (T*)y;
  a.out_jac = (T*)jac;
  CACTO_HP_IP_DISPATCH(run_forward, T, sh.hp, sh.ip, a, jac != nullptr, st);
  return set_error(CACTO_EUNSUPPORTED, "forward: hidden width %d / input %d not built", sh.hp, sh.in);
}

}  // namespace cacto

using namespace cacto;

int validate_mlp(const cacto_mlp_t* m, const char* who);  // abi.cu
namespace cacto {  // wide.cu (padded hidden width > 64)
bool is_wide(const cacto_mlp_t* m);
int wide_mlp_entry(const cacto_mlp_t* m, const void* xa, int64_t B, void* value, void* jac, cudaStream_t st);
int wide_score(int mode, const cacto_mlp_t* sn, const cacto_mlp_t* cn, const float* xa, const float* rc, int64_t N,
               float* scores, cudaStream_t st);
int wide_forward_rows(const cacto_mlp_t* m, const cacto_batch_t* bt, int which, float* out, cudaStream_t st);
}  // namespace cacto

extern "C" int cacto_mlp_forward(const cacto_mlp_t* mlp, const void* xa, int64_t B, void* out, void* stream) {
  int rc = validate_mlp(mlp, "mlp_forward");
  if (rc) return rc;
  if (B < 0 || (B > 0 && (!xa || !out))) return set_error(CACTO_EVALUE, "mlp_forward: bad batch");
  if (B == 0) return CACTO_OK;
  if (is_wide(mlp)) return wide_mlp_entry(mlp, xa, B, out, nullptr, (cudaStream_t)stream);
  if (mlp->dtype == CACTO_F32) return forward_entry<float>(mlp, xa, B, out, nullptr, (cudaStream_t)stream);
  return forward_entry<double>(mlp, xa, B, out, nullptr, (cudaStream_t)stream);
}

extern "C" int cacto_mlp_jacobian(const cacto_mlp_t* mlp, const void* xa, int64_t B, void* value, void* jac,
                                  void* stream) {
  int rc = validate_mlp(mlp, "mlp_jacobian");
  if (rc) return rc;
  if (B < 0 || (B > 0 && (!xa || !value || !jac))) return set_error(CACTO_EVALUE, "mlp_jacobian: bad batch");
  if (B == 0) return CACTO_OK;
  if (is_wide(mlp)) return wide_mlp_entry(mlp, xa, B, value, jac, (cudaStream_t)stream);
  if (mlp->dtype == CACTO_F32) return forward_entry<float>(mlp, xa, B, value, jac, (cudaStream_t)stream);
  return forward_entry<double>(mlp, xa, B, value, jac, (cudaStream_t)stream);
}

template <typename T>
static int score_entry(int mode, const cacto_mlp_t* sn, const cacto_mlp_t* cn, const void* xa, const void* rc,
                       int64_t N, void* scores, cudaStream_t st) {
  ScoreArgs<T> a{};
  a.mode = mode;
  const cacto_mlp_t* any = sn ? sn : cn;
  NetShape sh = shape_of(*any);
  if (sn) {
    NetShape s1 = shape_of(*sn);
    a.nc_std = net_const<T>(*sn);
    a.nh_std = s1.nh; a.act_std = s1.act; a.head_std = s1.head;
    a.p_std = (const T*)sn->params;
  }
  if (cn) {
    NetShape s2 = shape_of(*cn);
    a.nc_crit = net_const<T>(*cn);
    a.nh_crit = s2.nh; a.act_crit = s2.act;
    a.p_crit = (const T*)cn->params;
  }
  a.in = sh.in;
  a.xa = (const T*)xa;
  a.rollout_cost = (const T*)rc;
  a.N = N;
  a.scores = (T*)scores;
  CACTO_HP_IP_DISPATCH(run_score, T, sh.hp, sh.ip, a, st);
  return set_error(CACTO_EUNSUPPORTED, "score: hidden width %d / input %d not built", sh.hp, sh.in);
}

extern "C" int cacto_score(int32_t mode, const cacto_mlp_t* std_net, const cacto_mlp_t* critic, const void* xa,
                           const void* rollout_cost, int64_t N, void* scores, void* stream) {
  if (mode < 0 || mode > 2) return set_error(CACTO_EVALUE, "score: unknown mode %d", mode);
  bool need_std = mode != CACTO_SCORE_GAP, need_crit = mode != CACTO_SCORE_STD;
  if (need_std) {
    int rc = validate_mlp(std_net, "score(std)");
    if (rc) return rc;
    if (std_net->sizes[std_net->n_layers] != 1) return set_error(CACTO_EVALUE, "score: std net must be scalar");
  }
  if (need_crit) {
    int rc = validate_mlp(critic, "score(critic)");
    if (rc) return rc;
    if (critic->sizes[critic->n_layers] != 1) return set_error(CACTO_EVALUE, "score: critic must be scalar");
    if (!rollout_cost) return set_error(CACTO_EVALUE, "score: gap modes need rollout costs");
  }
  if (need_std && need_crit &&
      (std_net->dtype != critic->dtype || std_net->hp != critic->hp || std_net->sizes[0] != critic->sizes[0]))
    return set_error(CACTO_EVALUE, "score: std and critic nets must share dtype / widths");
  if (N < 0) return set_error(CACTO_EVALUE, "score: N < 0");
  if (N == 0) return CACTO_OK;
  if (is_wide(need_std ? std_net : critic))
    return wide_score(mode, need_std ? std_net : nullptr, need_crit ? critic : nullptr, (const float*)xa,
                      (const float*)rollout_cost, N, (float*)scores, (cudaStream_t)stream);
  int dtype = need_std ? std_net->dtype : critic->dtype;
  if (dtype == CACTO_F32)
    return score_entry<float>(mode, need_std ? std_net : nullptr, need_crit ? critic : nullptr, xa, rollout_cost, N,
                              scores, (cudaStream_t)stream);
  return score_entry<double>(mode, need_std ? std_net : nullptr, need_crit ? critic : nullptr, xa, rollout_cost, N,
                             scores, (cudaStream_t)stream);
}

// ---- forward over (gathered) replay rows: target value at x_{+k} (which=1,
// nets.py:249) or the critic error v_bar - V(xa) (which=2, nets.py:343) -------
namespace cacto {

template <typename T>
struct RowsArgs {
  NetConst<T> nc;
  int nh, in, act, head, which;
  const T* params;
  const int64_t* idx;
  const int64_t* cycle;
  int64_t stride;
  const T* x;      // xa or xa_plus_k column
  const T* v_bar;
  int64_t rows;
  T* out;
};

template <typename T, int HP, int IP, int S>
__global__ void __launch_bounds__(kThreads) rows_forward_kernel(const RowsArgs<T> a) {
  using TL = Tile<T, S, HP>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  NetSmem<T, HP, IP, TL::KS> net;
  T* p = net.carve(sm, a.nh, a.in, 1);
  T* A0 = p;
  T* P0 = A0 + IP * S;
  T* P1 = P0 + HP * S;
  net.stage(a.params);
  const TL tl;
  const int64_t* idx = (a.idx && a.cycle) ? a.idx + (*a.cycle) * a.stride : a.idx;
  const int64_t ntiles = (a.rows + S - 1) / S;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * S;
    __syncthreads();
    load_input_tile<TL>(A0, IP, a.in, a.nc,
                          [&](int s) { return base + s < a.rows ? (idx ? idx[base + s] : base + s) : (int64_t)-1; },
                          [&](int64_t r, int c) { return a.x[r * a.in + c]; });
    __syncthreads();
    const T* last = forward_hidden(tl, net, a.act, A0, P0, P1, (T*)nullptr);
    forward_output<TL>(net, last, [&](int s, int, T o) {
      int64_t b = base + s;
      if (b >= a.rows) return;
      if (a.which == 1) {
        a.out[b] = head_value(a.head, a.nc, 0, o);
      } else {
        int64_t r = idx ? idx[b] : b;
        a.out[b] = a.v_bar[r] - head_value(a.head, a.nc, 0, o);
      }
    });
  }
}

template <typename T, int HP, int IP>
static int run_rows(const RowsArgs<T>& a, cudaStream_t st) {
  return with_tile<T, HP>(a.rows, [&](auto s_) {
    constexpr int S = decltype(s_)::value;
    size_t el = net_elems<T, HP, IP>(a.nh, 1) + (size_t)IP * S + 2 * (size_t)HP * S;
    auto kern = rows_forward_kernel<T, HP, IP, S>;
    int grid = launch_tiles<T, HP, IP>(kern, el, a.rows, st, "rows_forward", &a, S);
    if (grid < 0) return grid;
    kern<<<grid, kThreads, el * sizeof(T), st>>>(a);
    return check_launch("rows_forward_kernel");
  });
}

template <typename T>
static int rows_entry(const cacto_mlp_t* m, const cacto_batch_t* b, int which, void* out, cudaStream_t st) {
  NetShape sh = shape_of(*m);
  RowsArgs<T> a{};
  a.nc = net_const<T>(*m);
  a.nh = sh.nh; a.in = sh.in; a.act = sh.act; a.head = sh.head; a.which = which;
  a.params = (const T*)m->params;
  a.idx = b->idx;
  a.cycle = b->cycle;
  a.stride = b->idx_stride;
  a.x = (const T*)(which == 1 ? b->xa_plus_k : b->xa);
  a.v_bar = (const T*)b->v_bar;
  a.rows = b->rows;
  a.out = (T*)out;
  CACTO_HP_IP_DISPATCH(run_rows, T, sh.hp, sh.ip, a, st);
  return set_error(CACTO_EUNSUPPORTED, "rows_forward: hidden width %d / input %d not built", sh.hp, sh.in);
}

}  // namespace cacto

int cacto_forward_rows(const cacto_mlp_t* mlp, const cacto_batch_t* b, int which, void* out, void* stream) {
  int rc = validate_mlp(mlp, "forward_rows");
  if (rc) return rc;
  if (mlp->sizes[mlp->n_layers] != 1) return set_error(CACTO_EVALUE, "forward_rows: scalar network required");
  if (mlp->sizes[0] != b->n + 1) return set_error(CACTO_EVALUE, "forward_rows: input dim mismatch");
  if (b->rows == 0) return CACTO_OK;
  if (is_wide(mlp)) return wide_forward_rows(mlp, b, which, (float*)out, (cudaStream_t)stream);
  if (mlp->dtype == CACTO_F32) return rows_entry<float>(mlp, b, which, out, (cudaStream_t)stream);
  return rows_entry<double>(mlp, b, which, out, (cudaStream_t)stream);
}
