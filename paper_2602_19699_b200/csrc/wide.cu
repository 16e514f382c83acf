// wide.cu -- wide networks (padded hidden width > 64, fp32): the layer-wise
// form of the MLP forward (nets.py:132-141), input-gradient sweep
// (nets.py:176-206), Sobolev critic loss (nets.py:233-290), std loss
// (nets.py:337-353) and actor loss (nets.py:293-334), built from the tcgen05
// 3xTF32 GEMM (gemm_tc.cu) plus fused elementwise / column-reduction kernels.
// Activations live in HBM as [B][H] row-major matrices; every dense-layer GEMM
// (z = a W^T, s = g W, gW += g^T a) is one gemm_tf32 call with K-major or
// MN-major operands.  Gradients are written in the padded parameter layout into
// workspace slot 0 (n_partials = 1), with the loss at index P, so the existing
// fold / Adam kernels apply unchanged.  Deterministic: no atomics.
#include <cstdlib>

#include "net.cuh"
#include "systems.cuh"

int cacto_forward_rows(const cacto_mlp_t* mlp, const cacto_batch_t* rows_of, int which, void* out,
                       void* stream);  // forward.cu (narrow nets, gathered rows)

namespace cacto {

int wide_jac_store(const float* S0, int ip, const float* O, int opad, const float* bL, NetConst<float> nc, int head,
                   int j, int out, int in, int64_t B, float* jac, cudaStream_t st);
int wide_add_bias_col0(float* O, int opad, const float* b, int64_t B, cudaStream_t st);
int wide_jacobian_ws(const cacto_mlp_t* mlp, const float* xa, int64_t B, float* value, float* jac, void* ws,
                     size_t ws_bytes, cudaStream_t st);

int gemm_tf32(int M, int N, int K, const float* A, int64_t sam, int64_t sak, const float* B, int64_t sbn, int64_t sbk,
              float* D, int64_t ldd, int accumulate, float alpha, int passes, void* ws, size_t ws_bytes,
              cudaStream_t st);
size_t gemm_workspace_bytes(int M, int N, int K);

namespace wide {

constexpr int kPasses = 3;  // 3xTF32: fp32-faithful
constexpr int kRedRows = 64;  // column-sum partial count

static unsigned grid1d(int64_t n) {
  int64_t b = (n + 255) / 256;
  int64_t cap = 16 * (int64_t)num_sms();
  return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

// ---- bump allocator over the caller's workspace ------------------------------------
struct Arena {
  char* p;
  size_t left;
  bool ok = true;
  float* f(size_t n) {
    size_t b = ((n * 4) + 255) & ~(size_t)255;
    if (b > left) {
      ok = false;
      return nullptr;
    }
    float* r = (float*)p;
    p += b;
    left -= b;
    return r;
  }
};

struct WNet {
  NetShape sh;
  LayerOffsets lo;
  NetConst<float> nc;
  const float* P;
  int H;   // padded hidden width
  int ip;  // padded input width
  const float* W(int i) const { return P + lo.w[i]; }
  const float* b(int i) const { return P + lo.b[i]; }
  int cols(int i) const { return lo.cols[i]; }
};

static WNet wnet(const cacto_mlp_t* m) {
  WNet w;
  w.sh = shape_of(*m);
  w.lo = layer_offsets(w.sh);
  w.nc = net_const<float>(*m);
  w.P = (const float*)m->params;
  w.H = w.sh.hp;
  w.ip = w.sh.ip;
  return w;
}

// ---- elementwise / reduction kernels ------------------------------------------------
struct RowSrc {  // rows of a batch column (optionally gathered) or of a plain array
  const float* x;
  int64_t stride;
  const int64_t* idx;
  const int64_t* cycle;
  int64_t idx_stride;
  CACTO_D int64_t row(int64_t b) const {
    if (!idx) return b;
    return cycle ? idx[(*cycle) * idx_stride + b] : idx[b];
  }
};

__global__ void input_kernel(float* X, int64_t B, int ip, int in, RowSrc src, NetConst<float> nc) {
  const int64_t total = B * ip;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / ip;
    const int c = (int)(e - b * ip);
    float v = 0.f;
    if (c < in) {
      v = src.x[src.row(b) * src.stride + c];
      if (nc.has_norm) v = (v - nc.in_center[c]) / nc.in_half[c];
    }
    X[e] = v;
  }
}

// ---- [B][H] elementwise passes, 4 columns per thread (H % 4 == 0, 16-byte rows) ----
CACTO_D int col_of4(int64_t e4, int H4) {  // first column of float4 e4 (32-bit modulo when it fits)
  return 4 * (int)(e4 < 0x7fffffff ? (uint32_t)e4 % (uint32_t)H4 : e4 % H4);
}
#define CACTO_FOR4(e4, n4) \
  for (int64_t e4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e4 < (n4); e4 += (int64_t)gridDim.x * blockDim.x)

__global__ void bias_act_kernel(float* Z, const float* __restrict__ bias, float* A, int act, int64_t B, int H) {
  float4* Z4 = reinterpret_cast<float4*>(Z);
  float4* A4 = reinterpret_cast<float4*>(A);
  CACTO_FOR4(e, B * (H / 4)) {
    const int c = col_of4(e, H / 4);
    float4 z = Z4[e];
    z.x += bias[c];
    z.y += bias[c + 1];
    z.z += bias[c + 2];
    z.w += bias[c + 3];
    Z4[e] = z;
    A4[e] = make_float4(act_value(act, z.x), act_value(act, z.y), act_value(act, z.z), act_value(act, z.w));
  }
}

// G = act'(Z) * (S or broadcast row w)
__global__ void d1_mul_kernel(float* G, const float* __restrict__ Z, const float* S, const float* w, int act,
                              int64_t B, int H) {
  const float4* Z4 = reinterpret_cast<const float4*>(Z);
  CACTO_FOR4(e, B * (H / 4)) {
    float4 s;
    if (S) {
      s = reinterpret_cast<const float4*>(S)[e];
    } else {
      const int c = col_of4(e, H / 4);
      s = make_float4(w[c], w[c + 1], w[c + 2], w[c + 3]);
    }
    const float4 z = Z4[e];
    reinterpret_cast<float4*>(G)[e] =
        make_float4(act_d1(act, z.x) * s.x, act_d1(act, z.y) * s.y, act_d1(act, z.z) * s.z, act_d1(act, z.w) * s.w);
  }
}

// zeta = act''(z) s rbar = h(z) g rbar  -> G ;  u_{i+1} = act'(z) rbar -> R   (nets.py:282-283)
__global__ void zeta_u_kernel(const float* __restrict__ Z, float* G, float* R, int act, int64_t n) {
  float4* G4 = reinterpret_cast<float4*>(G);
  float4* R4 = reinterpret_cast<float4*>(R);
  CACTO_FOR4(e, n / 4) {
    const float4 z = reinterpret_cast<const float4*>(Z)[e], r = R4[e], g = G4[e];
    G4[e] = make_float4(act_h(act, z.x) * g.x * r.x, act_h(act, z.y) * g.y * r.y, act_h(act, z.z) * g.z * r.z,
                        act_h(act, z.w) * g.w * r.w);
    R4[e] = make_float4(act_d1(act, z.x) * r.x, act_d1(act, z.y) * r.y, act_d1(act, z.z) * r.z,
                        act_d1(act, z.w) * r.w);
  }
}

// zbar = act'(z) abar (+ zeta)   (nets.py:225-227)
__global__ void zbar_kernel(const float* __restrict__ Z, const float* __restrict__ ABAR, float* G, int has_zeta,
                            int act, int64_t n) {
  float4* G4 = reinterpret_cast<float4*>(G);
  CACTO_FOR4(e, n / 4) {
    const float4 z = reinterpret_cast<const float4*>(Z)[e], ab = reinterpret_cast<const float4*>(ABAR)[e];
    float4 v = make_float4(act_d1(act, z.x) * ab.x, act_d1(act, z.y) * ab.y, act_d1(act, z.z) * ab.z,
                           act_d1(act, z.w) * ab.w);
    if (has_zeta) {
      const float4 g = G4[e];
      v = make_float4(v.x + g.x, v.y + g.y, v.z + g.z, v.w + g.w);
    }
    G4[e] = v;
  }
}

// top hidden layer of the value-path backprop: abar = delta W_L (small K = out)
// and zbar = act'(z) abar (+ zeta) in one pass, 4 columns per thread
// (nets.py:221-227; replaces an outer-product pass + zbar_kernel)
__global__ void outer_zbar_kernel(float* G, const float* __restrict__ Z, const float* __restrict__ DEL, int ldd,
                                  int nout, const float* __restrict__ W, int has_zeta, int act, int H, int64_t B) {
  const int H4 = H >> 2;
  const int64_t total = B * H4;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / H4;
    const int h = (int)(e - b * H4) * 4;
    float s[4] = {0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < nout; ++j) {
      const float d = DEL[b * ldd + j];
      const float4 w = *reinterpret_cast<const float4*>(W + (int64_t)j * H + h);
      s[0] = fmaf(d, w.x, s[0]);
      s[1] = fmaf(d, w.y, s[1]);
      s[2] = fmaf(d, w.z, s[2]);
      s[3] = fmaf(d, w.w, s[3]);
    }
    const int64_t o = b * H + h;
    const float4 z = *reinterpret_cast<const float4*>(Z + o);
    float4 r = make_float4(act_d1(act, z.x) * s[0], act_d1(act, z.y) * s[1], act_d1(act, z.z) * s[2],
                           act_d1(act, z.w) * s[3]);
    if (has_zeta) {
      const float4 g = *reinterpret_cast<const float4*>(G + o);
      r.x += g.x;
      r.y += g.y;
      r.z += g.z;
      r.w += g.w;
    }
    *reinterpret_cast<float4*>(G + o) = r;
  }
}

// column sums, stage 1: part[r][c] = sum over row chunk r of w_b * X[b][c]
__global__ void colsum_partial_kernel(const float* __restrict__ X, int64_t ldx, const float* __restrict__ wrow,
                                      int64_t ldw, int64_t B, int W, float* part) {
  __shared__ float red[8][33];
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int rl = threadIdx.x >> 5;  // 0..7
  const int64_t chunk = (B + gridDim.y - 1) / gridDim.y;
  const int64_t b0 = blockIdx.y * chunk, b1 = min(B, b0 + chunk);
  float s = 0.f;
  if (c < W)
    for (int64_t b = b0 + rl; b < b1; b += 8) {
      const float x = X[b * ldx + c];
      s += wrow ? wrow[b * ldw] * x : x;
    }
  red[rl][threadIdx.x & 31] = s;
  __syncthreads();
  if (rl == 0 && c < W) {
    float t = 0.f;
    for (int q = 0; q < 8; ++q) t += red[q][threadIdx.x & 31];
    part[(int64_t)blockIdx.y * W + c] = t;
  }
}
// stage 2: out[c] (+)= sum_r part[r][c]
__global__ void colsum_final_kernel(const float* __restrict__ part, int R, int W, float* out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < W; c += gridDim.x * blockDim.x) {
    float t = 0.f;
    for (int r = 0; r < R; ++r) t += part[(int64_t)r * W + c];
    out[c] += t;
  }
}

// sum of per-block loss partials -> *dst (one thread, fixed order)
__global__ void fold_loss_kernel(const float* __restrict__ part, int n, float* dst) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    float s = 0.f;
    for (int i = 0; i < n; ++i) s += part[i];
    *dst += s;
  }
}

template <typename F>
CACTO_D void block_sum_to(float v, float* dst, F) {
  __shared__ float red[8];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    *dst = s;
  }
}

// critic errors (nets.py:247-277): y, e_v, e_g, loss partial, U0, delta
struct CriticErrArgs {
  int64_t B;
  int n, ip;
  RowSrc vbar, vbarx, xk;  // v_bar [*], v_bar_x [*][n], xa_plus_k [*][n+1]
  const float* vnext;      // [B] or null
  int t_max;
  const float* O;          // [B][4] critic raw output (col 0)
  float bL;
  const float* S0;         // [B][ip] d V / d normalised input
  NetConst<float> nc;
  float k_s, inv_denom;
  float* U0;               // [B][ip]
  float* DEL;              // [B][4] (col 0)
  float* lossp;            // [gridDim.x]
};
__global__ void critic_err_kernel(CriticErrArgs a) {
  float term = 0.f;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < a.B; b += (int64_t)gridDim.x * blockDim.x) {
    float y = a.vbar.x[a.vbar.row(b)];
    if (a.vnext) {
      const bool gate = a.xk.x[a.xk.row(b) * a.xk.stride + a.n] < (float)a.t_max;
      y = y + (gate ? a.vnext[b] : 0.f);
    }
    const float ev = y - (a.O[b * 4] + a.bL);
    float eg2 = 0.f;
    const int64_t vr = a.vbarx.row(b);
    for (int c = 0; c < a.ip; ++c) {
      float u = 0.f;
      if (c < a.n) {
        const float eg = a.vbarx.x[vr * a.vbarx.stride + c] - a.S0[b * a.ip + c] / a.nc.in_half[c];
        eg2 += eg * eg;
        u = -2.f * a.k_s * a.inv_denom * eg / a.nc.in_half[c];
      }
      a.U0[b * a.ip + c] = u;
    }
    term += (ev * ev + a.k_s * eg2) * a.inv_denom;
    a.DEL[b * 4] = -2.f * a.inv_denom * ev;
    a.DEL[b * 4 + 1] = 0.f;
    a.DEL[b * 4 + 2] = 0.f;
    a.DEL[b * 4 + 3] = 0.f;
  }
  block_sum_to(term, a.lossp + blockIdx.x, 0);
}

// std loss (nets.py:343-352): delta = dl/dsigma * sigmoid(o)
__global__ void std_delta_kernel(int64_t B, const float* __restrict__ err, const float* __restrict__ O, float bL,
                                 NetConst<float> nc, int head, float inv_denom, float* DEL, float* lossp) {
  float term = 0.f;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) {
    const float o = O[b * 4] + bL;
    const float sigma = head_value(head, nc, 0, o);
    const float e = err[b];
    term += (logf(sigma) + 0.5f * e * e / (sigma * sigma)) * inv_denom;
    const float dl = (1.f / sigma - e * e / (sigma * sigma * sigma)) * inv_denom;
    DEL[b * 4] = dl * sigmoid(o);
    DEL[b * 4 + 1] = DEL[b * 4 + 2] = DEL[b * 4 + 3] = 0.f;
  }
  block_sum_to(term, lossp + blockIdx.x, 0);
}

// err = v_bar - V(xa)  (O raw critic output)
__global__ void value_err_kernel(int64_t B, RowSrc vbar, const float* __restrict__ O, float bL, float* err) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x)
    err[b] = vbar.x[vbar.row(b)] - (O[b * 4] + bL);
}

// head outputs of a forward (value [B][out]): y = head(o + b)
__global__ void head_kernel(int64_t B, int out, const float* __restrict__ O, int ldo, const float* __restrict__ bL,
                            NetConst<float> nc, int head, float* Y) {
  const int64_t total = B * out;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / out;
    const int j = (int)(e - b * out);
    Y[e] = head_value(head, nc, j, O[b * ldo + j] + bL[j]);
  }
}

// actor prep (nets.py:319-325): u = head(o), l(x, u), x' = f(x, u), t+1
template <int SYS>
__global__ void actor_prep_rows_kernel(int64_t B, RowSrc xa, const float* __restrict__ O, int ldo,
                                       const float* __restrict__ bL, NetConst<float> nc, int head, SysDev<float> sys,
                                       CostDev<float> cost, float* XN, float* LS) {
  constexpr int nn = SysDims<SYS>::n, mm = SysDims<SYS>::m;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) {
    const float* x0 = xa.x + xa.row(b) * xa.stride;
    float x[nn], u[mm], xn[nn];
#pragma unroll
    for (int c = 0; c < nn; ++c) x[c] = x0[c];
#pragma unroll
    for (int j = 0; j < mm; ++j) u[j] = head_value(head, nc, j, O[b * ldo + j] + bL[j]);
    LS[b] = cost_and_step<SYS>(sys, cost, true, x, u, xn);
#pragma unroll
    for (int c = 0; c < nn; ++c) XN[b * (nn + 1) + c] = xn[c];
    XN[b * (nn + 1) + nn] = x0[nn] + 1.f;
  }
}

// actor output cotangent (nets.py:328-333)
template <int SYS>
__global__ void actor_delta_kernel(int64_t B, RowSrc xa, const float* __restrict__ O, int ldo,
                                   const float* __restrict__ bL, NetConst<float> nc, int head, SysDev<float> sys,
                                   CostDev<float> cost, const float* __restrict__ GN, const float* __restrict__ VN,
                                   const float* __restrict__ LS, const int64_t* live, float* DEL, int ldd,
                                   float* lossp) {
  constexpr int nn = SysDims<SYS>::n, mm = SysDims<SYS>::m;
  const float inv = 1.f / (float)(*live);
  float term = 0.f;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) {
    const float* x0 = xa.x + xa.row(b) * xa.stride;
    float d[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (x0[nn] < (float)sys.t_max) {
      float x[nn], u[mm], g[nn], ft[mm];
#pragma unroll
      for (int c = 0; c < nn; ++c) x[c] = x0[c];
#pragma unroll
      for (int j = 0; j < mm; ++j) u[j] = head_value(head, nc, j, O[b * ldo + j] + bL[j]);
#pragma unroll
      for (int c = 0; c < nn; ++c) g[c] = GN[b * (nn + 1) + c];
      fu_t_g<SYS>(sys, x, u, g, ft);
      term += (LS[b] + VN[b]) * inv;
#pragma unroll
      for (int j = 0; j < mm; ++j)
        d[j] = ((2.f * cost.w_u * u[j] + ft[j]) * inv) * head_chain(head, nc, j, O[b * ldo + j] + bL[j]);
    }
    for (int j = 0; j < ldd; ++j) DEL[b * ldd + j] = j < 8 ? d[j] : 0.f;
  }
  block_sum_to(term, lossp + blockIdx.x, 0);
}

// ---- layer-wise building blocks ------------------------------------------------------
struct Ctx {
  cudaStream_t st;
  void* gws;  // split-K workspace
  size_t gws_bytes;
  float* colpart;  // [kRedRows][max width]
};

static int gemm(const Ctx& c, int M, int N, int K, const float* A, int64_t sam, int64_t sak, const float* B,
                int64_t sbn, int64_t sbk, float* D, int64_t ldd, int acc) {
  return gemm_tf32(M, N, K, A, sam, sak, B, sbn, sbk, D, ldd, acc, 1.f, kPasses, c.gws, c.gws_bytes, c.st);
}

static int colsum(const Ctx& c, const float* X, int64_t ldx, const float* w, int64_t ldw, int64_t B, int W,
                  float* out) {
  dim3 g1((W + 31) / 32, kRedRows);
  colsum_partial_kernel<<<g1, 256, 0, c.st>>>(X, ldx, w, ldw, B, W, c.colpart);
  colsum_final_kernel<<<(W + 255) / 256, 256, 0, c.st>>>(c.colpart, kRedRows, W, out);
  return check_launch("colsum");
}

struct Acts {  // per-layer device buffers of one network evaluation
  float* X0;       // [B][ip]
  float* Z;        // nh x [B][H]
  float* A;        // nh x [B][H]   (a_{i+1})
  float* G;        // nh x [B][H]   (g_i / zeta_i / zbar_i)
  float* O;        // [B][opad]
  int opad;
};

static Acts alloc_acts(Arena& ar, const WNet& w, int64_t B, bool grads) {
  Acts a{};
  const int nh = w.sh.nh;
  a.opad = w.sh.out <= 4 ? 4 : 8;
  a.X0 = ar.f((size_t)B * w.ip);
  a.Z = ar.f((size_t)nh * B * w.H);
  a.A = ar.f((size_t)nh * B * w.H);
  a.G = grads ? ar.f((size_t)nh * B * w.H) : nullptr;
  a.O = ar.f((size_t)B * a.opad);
  return a;
}

// forward: X0 filled; fills Z_i, A_{i+1}, O (raw, bias not added)
static int forward(const Ctx& c, const WNet& w, const Acts& a, int64_t B) {
  const int nh = w.sh.nh, H = w.H;
  const float* cur = a.X0;
  int width = w.ip;
  for (int i = 0; i < nh; ++i) {
    float* Z = a.Z + (size_t)i * B * H;
    float* A = a.A + (size_t)i * B * H;
    int rc = gemm(c, (int)B, H, w.cols(i), cur, width, 1, w.W(i), w.cols(i), 1, Z, H, 0);
    if (rc) return rc;
    bias_act_kernel<<<grid1d(B * H / 4), 256, 0, c.st>>>(Z, w.b(i), A, w.sh.act, B, H);
    cur = A;
    width = H;
  }
  return gemm(c, (int)B, w.sh.out, w.cols(nh), cur, width, 1, w.W(nh), w.cols(nh), 1, a.O, a.opad, 0);
}

// input-gradient sweep of output j: G_i = g_i, S0 [B][ip] = g_0 W_0 (w.r.t. normalised input)
static int sweep(const Ctx& c, const WNet& w, const Acts& a, int64_t B, int j, float* S, float* S0) {
  const int nh = w.sh.nh, H = w.H;
  const int64_t TS = B * H;
  d1_mul_kernel<<<grid1d(TS / 4), 256, 0, c.st>>>(a.G + (nh - 1) * TS, a.Z + (nh - 1) * TS, nullptr,
                                              w.W(nh) + (int64_t)j * H, w.sh.act, B, H);
  for (int i = nh - 1; i >= 1; --i) {
    int rc = gemm(c, (int)B, H, H, a.G + i * TS, H, 1, w.W(i), 1, H, S, H, 0);
    if (rc) return rc;
    d1_mul_kernel<<<grid1d(TS / 4), 256, 0, c.st>>>(a.G + (i - 1) * TS, a.Z + (i - 1) * TS, S, nullptr, w.sh.act, B, H);
  }
  return gemm(c, (int)B, w.ip, H, a.G, H, 1, w.W(0), 1, w.ip, S0, w.ip, 0);
}

// value-path backprop with output cotangent DEL [B][ldd] and optional zeta in G
// (critic); accumulates into the padded gradient buffer `grad`
static int backprop(const Ctx& c, const WNet& w, const Acts& a, int64_t B, const float* DEL, int ldd, bool has_zeta,
                    float* ABAR, float* grad) {
  const int nh = w.sh.nh, H = w.H, out = w.sh.out;
  const int64_t TS = B * H;
  const float* aL = nh > 0 ? a.A + (nh - 1) * TS : a.X0;
  const int wL = w.cols(nh);
  // gW_L += DEL^T a_L ; gb_L += colsum(DEL)
  int rc = gemm(c, out, wL, (int)B, DEL, 1, ldd, aL, 1, wL, grad + w.lo.w[nh], wL, 1);
  if (rc) return rc;
  rc = colsum(c, DEL, ldd, nullptr, 0, B, out, grad + w.lo.b[nh]);
  if (rc) return rc;
  if (nh == 0) return CACTO_OK;
  for (int i = nh - 1; i >= 0; --i) {
    float* G = a.G + i * TS;
    if (i == nh - 1)
      outer_zbar_kernel<<<grid1d(TS / 4), 256, 0, c.st>>>(G, a.Z + i * TS, DEL, ldd, out, w.W(nh), has_zeta ? 1 : 0,
                                                          w.sh.act, H, B);
    else
      zbar_kernel<<<grid1d(TS / 4), 256, 0, c.st>>>(a.Z + i * TS, ABAR, G, has_zeta ? 1 : 0, w.sh.act, TS);
    rc = colsum(c, G, H, nullptr, 0, B, H, grad + w.lo.b[i]);
    if (rc) return rc;
    const float* ai = i == 0 ? a.X0 : a.A + (i - 1) * TS;
    const int wi = w.cols(i);
    rc = gemm(c, H, wi, (int)B, G, 1, H, ai, 1, wi, grad + w.lo.w[i], wi, 1);
    if (rc) return rc;
    if (i > 0) {
      rc = gemm(c, (int)B, H, H, G, H, 1, w.W(i), 1, H, ABAR, H, 0);
      if (rc) return rc;
    }
  }
  return check_launch("wide backprop");
}

static void fill_input(const Ctx& c, const WNet& w, float* X0, int64_t B, RowSrc src) {
  input_kernel<<<grid1d(B * w.ip), 256, 0, c.st>>>(X0, B, w.ip, w.sh.in, src, w.nc);
}

static RowSrc batch_src(const cacto_batch_t* b, const void* col, int64_t stride) {
  RowSrc s;
  s.x = (const float*)col;
  s.stride = stride;
  s.idx = b->idx;
  s.cycle = b->cycle;
  s.idx_stride = b->idx_stride;
  return s;
}

}  // namespace wide

// ======================================================================================
// entry points used by the C ABI (dispatch when hp > 64)
// ======================================================================================
using namespace wide;

// CACTO_WIDE_MIN=<w> moves the layer-wise path's threshold down (measurement aid:
// fp32 nets with hp >= w take it; default: hp > 64 only)
static int wide_min() {
  static int v = [] {
    const char* e = getenv("CACTO_WIDE_MIN");
    return e ? atoi(e) : 65;
  }();
  return v;
}
bool is_wide(const cacto_mlp_t* m) {
  return m && m->n_layers > 1 && (m->hp > 64 || (m->dtype == CACTO_F32 && m->hp >= wide_min()));
}

// one network's loss / Jacobian workspace: gradient slot, per-layer Z / A / G,
// two [B][H] scratch matrices, the [B][ip] input / sweep / cotangent tiles, the
// per-row vectors, column-sum and loss partials and the split-K partials
size_t wide_workspace_bytes(const cacto_mlp_t* m, int64_t rows) {
  if (!is_wide(m)) return 0;
  NetShape sh = shape_of(*m);
  const size_t B = (size_t)(rows > 0 ? rows : 1);
  const size_t H = (size_t)sh.hp, nh = (size_t)sh.nh;
  LayerOffsets lo = layer_offsets(sh);
  size_t f = (size_t)(lo.total + 1);
  f += 3 * B * sh.ip + 3 * nh * B * H + 2 * B * H;  // X0 S0 U0 | Z A G | R0 R1 (S, ABAR)
  f += 8 * B + 8 * B + 2 * 32 * B + 4 * B;           // O, DEL, XN / GN, per-row vectors
  f += (size_t)kRedRows * (H > 32 ? H : 32) + 1024 + 64 * 32;  // partials + arena alignment slack
  size_t g = gemm_workspace_bytes((int)H, (int)H, (int)B);
  size_t g2 = gemm_workspace_bytes((int)H, 32, (int)B);
  return f * 4 + (g > g2 ? g : g2) + 256;
}

static Ctx make_ctx(Arena& ar, int H, int64_t B, cudaStream_t st) {
  Ctx c;
  c.st = st;
  size_t g = gemm_workspace_bytes(H, H, (int)B), g2 = gemm_workspace_bytes(H, 32, (int)B);
  size_t gb = g > g2 ? g : g2;
  c.gws = gb ? (void*)ar.f(gb / 4 + 1) : nullptr;
  c.gws_bytes = gb;
  c.colpart = ar.f((size_t)kRedRows * (H > 32 ? H : 32));
  return c;
}

// value [B][out] (head applied) and optionally jac [B][out][in] w.r.t. the raw input
int wide_forward(const cacto_mlp_t* m, const float* xa, int64_t B, float* y, float* jac, void* ws, size_t ws_bytes,
                 cudaStream_t st) {
  WNet w = wnet(m);
  Arena ar{(char*)ws, ws_bytes};
  Ctx c = make_ctx(ar, w.H, B, st);
  Acts a = alloc_acts(ar, w, B, jac != nullptr);
  float* S = jac ? ar.f((size_t)B * w.H) : nullptr;
  float* S0 = jac ? ar.f((size_t)B * w.ip) : nullptr;
  if (!ar.ok) return set_error(CACTO_EVALUE, "wide forward: workspace too small");
  RowSrc src{xa, w.sh.in, nullptr, nullptr, 0};
  fill_input(c, w, a.X0, B, src);
  int rc = forward(c, w, a, B);
  if (rc) return rc;
  head_kernel<<<grid1d(B * w.sh.out), 256, 0, st>>>(B, w.sh.out, a.O, a.opad, w.b(w.sh.nh), w.nc, w.sh.head, y);
  if (!jac) return check_launch("wide forward");
  for (int j = 0; j < w.sh.out; ++j) {
    rc = sweep(c, w, a, B, j, S, S0);
    if (rc) return rc;
    // jac[b][j][c] = S0[b][c] * head_chain(o_j) / in_half[c]
    rc = wide_jac_store(S0, w.ip, a.O, a.opad, w.b(w.sh.nh), w.nc, w.sh.head, j, w.sh.out, w.sh.in, B, jac, st);
    if (rc) return rc;
  }
  return check_launch("wide jacobian");
}

__global__ void jac_store_kernel(const float* __restrict__ S0, int ip, const float* __restrict__ O, int opad,
                                 const float* __restrict__ bL, NetConst<float> nc, int head, int j, int out, int in,
                                 int64_t B, float* jac) {
  const int64_t total = B * in;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / in;
    const int cc = (int)(e - b * in);
    const float chain = head_chain(head, nc, j, O[b * opad + j] + bL[j]);
    jac[(b * out + j) * in + cc] = S0[b * ip + cc] * chain / nc.in_half[cc];
  }
}

int wide_jac_store(const float* S0, int ip, const float* O, int opad, const float* bL, NetConst<float> nc, int head,
                   int j, int out, int in, int64_t B, float* jac, cudaStream_t st) {
  jac_store_kernel<<<grid1d(B * in), 256, 0, st>>>(S0, ip, O, opad, bL, nc, head, j, out, in, B, jac);
  return check_launch("jac_store");
}

// Sobolev critic loss; gradient + loss into slot 0 of `ws` (n_partials = 1)
int wide_critic_loss(const cacto_mlp_t* cm, const cacto_mlp_t* tm, const cacto_batch_t* bt, double k_s, int boot,
                     void* ws, size_t ws_bytes, cudaStream_t st) {
  WNet w = wnet(cm);
  const int64_t B = bt->rows;
  const int n = bt->n, H = w.H;
  Arena ar{(char*)ws, ws_bytes};
  float* slot = ar.f((size_t)w.lo.total + 1);
  Ctx c = make_ctx(ar, H, B, st);
  Acts a = alloc_acts(ar, w, B, true);
  float* R0 = ar.f((size_t)B * H);
  float* R1 = ar.f((size_t)B * H);
  float* S0 = ar.f((size_t)B * w.ip);
  float* U0 = ar.f((size_t)B * w.ip);
  float* DEL = ar.f((size_t)B * 4);
  float* vnext = boot && tm ? ar.f((size_t)B) : nullptr;
  float* lossp = ar.f(1024);
  if (!ar.ok) return set_error(CACTO_EVALUE, "wide critic: workspace too small");
  cudaMemsetAsync(slot, 0, ((size_t)w.lo.total + 1) * 4, st);
  const float inv_denom = 1.f / (float)(bt->denom > 0 ? bt->denom : B);
  int rc;
  // bootstrap target V_tgt(x_{+k}) (nets.py:249)
  if (vnext) {
    if (is_wide(tm)) {
      WNet wt = wnet(tm);
      Acts at = a;  // the critic buffers are free until its own forward
      fill_input(c, wt, at.X0, B, batch_src(bt, bt->xa_plus_k, n + 1));
      rc = forward(c, wt, at, B);
      if (rc) return rc;
      head_kernel<<<grid1d(B), 256, 0, st>>>(B, 1, at.O, at.opad, wt.b(wt.sh.nh), wt.nc, wt.sh.head, vnext);
    } else {
      rc = ::cacto_forward_rows(tm, bt, 1, vnext, st);
      if (rc) return rc;
    }
  }
  fill_input(c, w, a.X0, B, batch_src(bt, bt->xa, n + 1));
  rc = forward(c, w, a, B);
  if (rc) return rc;
  rc = sweep(c, w, a, B, 0, R0, S0);
  if (rc) return rc;
  CriticErrArgs e{};
  e.B = B;
  e.n = n;
  e.ip = w.ip;
  e.vbar = batch_src(bt, bt->v_bar, 1);
  e.vbarx = batch_src(bt, bt->v_bar_x, n);
  e.xk = batch_src(bt, bt->xa_plus_k, n + 1);
  e.vnext = vnext;
  e.t_max = bt->t_max;
  e.O = a.O;
  e.S0 = S0;
  e.nc = w.nc;
  e.k_s = (float)k_s;
  e.inv_denom = inv_denom;
  e.U0 = U0;
  e.DEL = DEL;
  e.lossp = lossp;
  unsigned eg = grid1d(B) > 1024 ? 1024 : grid1d(B);
  // the output bias is added on device (O += b_L) before the error kernel
  rc = wide_add_bias_col0(a.O, a.opad, w.b(w.sh.nh), B, st);
  if (rc) return rc;
  e.bL = 0.f;
  critic_err_kernel<<<eg, 256, 0, st>>>(e);
  fold_loss_kernel<<<1, 32, 0, st>>>(lossp, (int)eg, slot + w.lo.total);
  // gradient path (nets.py:279-284)
  const int nh = w.sh.nh;
  const int64_t TS = B * H;
  const float* U = U0;
  int uw = w.ip;
  float* Rcur = R0;
  float* Rnext = R1;
  for (int i = 0; i < nh; ++i) {
    rc = gemm(c, (int)B, H, w.cols(i), U, uw, 1, w.W(i), w.cols(i), 1, Rcur, H, 0);  // rbar = u W^T
    if (rc) return rc;
    rc = gemm(c, H, w.cols(i), (int)B, a.G + i * TS, 1, H, U, 1, uw, slot + w.lo.w[i], w.cols(i), 1);  // g^T u
    if (rc) return rc;
    zeta_u_kernel<<<grid1d(TS / 4), 256, 0, st>>>(a.Z + i * TS, a.G + i * TS, Rcur, w.sh.act, TS);
    U = Rcur;
    uw = H;
    float* t = Rcur;
    Rcur = Rnext;
    Rnext = t;
  }
  rc = colsum(c, U, uw, nullptr, 0, B, uw, slot + w.lo.w[nh]);  // grads[2*last] += u.sum(0)
  if (rc) return rc;
  // value path with the injected zeta terms (nets.py:287-289)
  rc = backprop(c, w, a, B, DEL, 4, true, Rcur, slot);
  if (rc) return rc;
  return check_launch("wide critic loss");
}

__global__ void add_bias_col0_kernel(float* O, int opad, const float* __restrict__ b, int64_t B) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x)
    O[i * opad] += b[0];
}
int wide_add_bias_col0(float* O, int opad, const float* b, int64_t B, cudaStream_t st) {
  add_bias_col0_kernel<<<grid1d(B), 256, 0, st>>>(O, opad, b, B);
  return check_launch("add_bias_col0");
}

// std loss (nets.py:337-353); critic may be narrow or wide
int wide_std_loss(const cacto_mlp_t* sm, const cacto_mlp_t* cm, const cacto_batch_t* bt, void* ws, size_t ws_bytes,
                  cudaStream_t st) {
  WNet w = wnet(sm);
  const int64_t B = bt->rows;
  const int n = bt->n, H = w.H;
  Arena ar{(char*)ws, ws_bytes};
  float* slot = ar.f((size_t)w.lo.total + 1);
  Ctx c = make_ctx(ar, H, B, st);
  Acts a = alloc_acts(ar, w, B, true);
  float* ABAR = ar.f((size_t)B * H);
  float* err = ar.f((size_t)B);
  float* DEL = ar.f((size_t)B * 4);
  float* lossp = ar.f(1024);
  if (!ar.ok) return set_error(CACTO_EVALUE, "wide std: workspace too small");
  cudaMemsetAsync(slot, 0, ((size_t)w.lo.total + 1) * 4, st);
  int rc;
  if (is_wide(cm)) {  // critic forward in the std buffers (free until the std forward)
    WNet wc = wnet(cm);
    fill_input(c, wc, a.X0, B, batch_src(bt, bt->xa, n + 1));
    rc = forward(c, wc, a, B);
    if (rc) return rc;
    rc = wide_add_bias_col0(a.O, a.opad, wc.b(wc.sh.nh), B, st);
    if (rc) return rc;
    value_err_kernel<<<grid1d(B), 256, 0, st>>>(B, batch_src(bt, bt->v_bar, 1), a.O, 0.f, err);
  } else {
    rc = ::cacto_forward_rows(cm, bt, 2, err, st);
    if (rc) return rc;
  }
  fill_input(c, w, a.X0, B, batch_src(bt, bt->xa, n + 1));
  rc = forward(c, w, a, B);
  if (rc) return rc;
  rc = wide_add_bias_col0(a.O, a.opad, w.b(w.sh.nh), B, st);
  if (rc) return rc;
  unsigned eg = grid1d(B) > 1024 ? 1024 : grid1d(B);
  std_delta_kernel<<<eg, 256, 0, st>>>(B, err, a.O, 0.f, w.nc, w.sh.head,
                                       1.f / (float)(bt->denom > 0 ? bt->denom : B), DEL, lossp);
  fold_loss_kernel<<<1, 32, 0, st>>>(lossp, (int)eg, slot + w.lo.total);
  return backprop(c, w, a, B, DEL, 4, false, ABAR, slot);
}

// actor loss (nets.py:293-334) for a wide actor (critic narrow or wide)

template <int SYS>
static int wide_actor_sys(const cacto_mlp_t* am, const cacto_mlp_t* cm, const cacto_system_t* sys,
                          const cacto_cost_t* cost, const cacto_batch_t* bt, const int64_t* live, void* ws,
                          size_t ws_bytes, cudaStream_t st) {
  constexpr int nn = SysDims<SYS>::n;
  WNet w = wnet(am);
  const int64_t B = bt->rows;
  const int H = w.H;
  Arena ar{(char*)ws, ws_bytes};
  float* slot = ar.f((size_t)w.lo.total + 1);
  Ctx c = make_ctx(ar, H, B, st);
  Acts a = alloc_acts(ar, w, B, true);
  float* ABAR = ar.f((size_t)B * H);
  float* XN = ar.f((size_t)B * (nn + 1));
  float* LS = ar.f((size_t)B);
  float* VN = ar.f((size_t)B);
  float* GN = ar.f((size_t)B * (nn + 1));
  float* DEL = ar.f((size_t)B * 8);
  float* lossp = ar.f(1024);
  int64_t* live_own = live ? nullptr : reinterpret_cast<int64_t*>(ar.f(2));  // live == null: count here
  size_t cws = ar.left;  // the rest for the critic Jacobian
  void* cwsp = ar.p;
  if (!ar.ok) return set_error(CACTO_EVALUE, "wide actor: workspace too small");
  cudaMemsetAsync(slot, 0, ((size_t)w.lo.total + 1) * 4, st);
  if (live_own) {
    int rc0 = cacto_count_live(bt, live_own, st);
    if (rc0) return rc0;
    live = live_own;
  }
  RowSrc xs = batch_src(bt, bt->xa, nn + 1);
  fill_input(c, w, a.X0, B, xs);
  int rc = forward(c, w, a, B);
  if (rc) return rc;
  SysDev<float> sd = sys_dev<float>(*sys);
  CostDev<float> cd = cost_dev<float>(*cost);
  actor_prep_rows_kernel<SYS><<<grid1d(B), 256, 0, st>>>(B, xs, a.O, a.opad, w.b(w.sh.nh), w.nc, w.sh.head, sd, cd,
                                                         XN, LS);
  rc = wide_jacobian_ws(cm, XN, B, VN, GN, cwsp, cws, st);
  if (rc) return rc;
  unsigned eg = grid1d(B) > 1024 ? 1024 : grid1d(B);
  actor_delta_kernel<SYS><<<eg, 256, 0, st>>>(B, xs, a.O, a.opad, w.b(w.sh.nh), w.nc, w.sh.head, sd, cd, GN, VN, LS,
                                              live, DEL, 8, lossp);
  fold_loss_kernel<<<1, 32, 0, st>>>(lossp, (int)eg, slot + w.lo.total);
  return backprop(c, w, a, B, DEL, 8, false, ABAR, slot);
}

int wide_actor_loss(const cacto_mlp_t* am, const cacto_mlp_t* cm, const cacto_system_t* sys, const cacto_cost_t* cost,
                    const cacto_batch_t* bt, const int64_t* live, void* ws, size_t ws_bytes, cudaStream_t st) {
  switch (sys->kind) {
    case CACTO_SYS_TOY1D: return wide_actor_sys<CACTO_SYS_TOY1D>(am, cm, sys, cost, bt, live, ws, ws_bytes, st);
    case CACTO_SYS_POINTMASS: return wide_actor_sys<CACTO_SYS_POINTMASS>(am, cm, sys, cost, bt, live, ws, ws_bytes, st);
    case CACTO_SYS_DUBINS: return wide_actor_sys<CACTO_SYS_DUBINS>(am, cm, sys, cost, bt, live, ws, ws_bytes, st);
    case CACTO_SYS_MANIPULATOR3:
      return wide_actor_sys<CACTO_SYS_MANIPULATOR3>(am, cm, sys, cost, bt, live, ws, ws_bytes, st);
    case CACTO_SYS_ALIENGO_LIPM:
      return wide_actor_sys<CACTO_SYS_ALIENGO_LIPM>(am, cm, sys, cost, bt, live, ws, ws_bytes, st);
    default: return set_error(CACTO_EUNSUPPORTED, "wide actor: unknown system");
  }
}

int wide_mlp_entry(const cacto_mlp_t* m, const void* xa, int64_t B, void* value, void* jac, cudaStream_t st);

// value + state gradient of the critic at x' for the actor loss: in the caller's
// workspace when it is large enough, else through the library scratch
int wide_jacobian_ws(const cacto_mlp_t* mlp, const float* xa, int64_t B, float* value, float* jac, void* ws,
                     size_t ws_bytes, cudaStream_t st) {
  if (!is_wide(mlp)) return cacto_mlp_jacobian(mlp, xa, B, value, jac, st);
  if (ws_bytes >= wide_workspace_bytes(mlp, B)) return wide_forward(mlp, xa, B, value, jac, ws, ws_bytes, st);
  return wide_mlp_entry(mlp, xa, B, value, jac, st);
}

// library-owned scratch for the workspace-free entry points (forward / jacobian /
// score) on wide nets; grown outside any capture, one per device
static void* scratch(size_t bytes, cudaStream_t st) {
  static void* buf[64] = {};
  static size_t cap[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (cap[dev] < bytes) {
    cudaStreamSynchronize(st);
    if (buf[dev]) cudaFree(buf[dev]);
    buf[dev] = nullptr;
    cap[dev] = 0;
    if (cudaMalloc(&buf[dev], bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    cap[dev] = bytes;
  }
  return buf[dev];
}

int wide_mlp_entry(const cacto_mlp_t* m, const void* xa, int64_t B, void* value, void* jac, cudaStream_t st) {
  if (m->dtype != CACTO_F32) return set_error(CACTO_EUNSUPPORTED, "hidden width %d > 64 needs fp32", m->hp);
  size_t bytes = wide_workspace_bytes(m, B);
  void* ws = scratch(bytes, st);
  if (!ws) return set_error(CACTO_ECUDA, "wide net: cannot allocate %zu B scratch", bytes);
  return wide_forward(m, (const float*)xa, B, (float*)value, (float*)jac, ws, bytes, st);
}

__global__ void score_combine_kernel(int mode, int64_t N, const float* __restrict__ sig, const float* __restrict__ v,
                                     const float* __restrict__ rc, float* scores) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    if (mode == CACTO_SCORE_STD) {
      scores[i] = sig[i];
    } else {
      const float gap = fabsf(v[i] - rc[i]);
      scores[i] = mode == CACTO_SCORE_GAP ? gap : sig[i] * gap;
    }
  }
}

// BIC scores with wide nets (trainer.py:150-151 + the gap modes): two layer-wise
// forwards and one combine pass
int wide_score(int mode, const cacto_mlp_t* sn, const cacto_mlp_t* cn, const float* xa, const float* rc, int64_t N,
               float* scores, cudaStream_t st) {
  const cacto_mlp_t* any = sn ? sn : cn;
  if (any->dtype != CACTO_F32) return set_error(CACTO_EUNSUPPORTED, "hidden width %d > 64 needs fp32", any->hp);
  size_t wb = std::max(wide_workspace_bytes(sn, N), wide_workspace_bytes(cn, N));
  size_t vec = (((size_t)N * 4 + 255) & ~(size_t)255);
  char* ws = (char*)scratch(wb + 2 * vec, st);
  if (!ws) return set_error(CACTO_ECUDA, "score: cannot allocate scratch");
  float* sig = (float*)(ws + wb);
  float* v = (float*)(ws + wb + vec);
  int r;
  if (sn) {
    r = wide_forward(sn, xa, N, sig, nullptr, ws, wb, st);
    if (r) return r;
  }
  if (cn) {
    r = wide_forward(cn, xa, N, v, nullptr, ws, wb, st);
    if (r) return r;
  }
  score_combine_kernel<<<grid1d(N), 256, 0, st>>>(mode, N, sig, v, rc, scores);
  return check_launch("score_combine");
}

// forward over gathered batch rows for a wide net (the wide form of
// cacto_forward_rows): which 1 -> V(xa_plus_k), 2 -> v_bar - V(xa)
int wide_forward_rows(const cacto_mlp_t* m, const cacto_batch_t* bt, int which, float* out, cudaStream_t st) {
  if (m->dtype != CACTO_F32) return set_error(CACTO_EUNSUPPORTED, "hidden width %d > 64 needs fp32", m->hp);
  const int64_t B = bt->rows;
  size_t bytes = wide_workspace_bytes(m, B);
  void* ws = scratch(bytes, st);
  if (!ws) return set_error(CACTO_ECUDA, "wide net: cannot allocate %zu B scratch", bytes);
  WNet w = wnet(m);
  Arena ar{(char*)ws, bytes};
  Ctx c = make_ctx(ar, w.H, B, st);
  Acts a = alloc_acts(ar, w, B, false);
  if (!ar.ok) return set_error(CACTO_EVALUE, "wide rows: scratch too small");
  fill_input(c, w, a.X0, B, batch_src(bt, which == 1 ? bt->xa_plus_k : bt->xa, bt->n + 1));
  int rc = forward(c, w, a, B);
  if (rc) return rc;
  if (which == 1) {
    head_kernel<<<grid1d(B), 256, 0, st>>>(B, 1, a.O, a.opad, w.b(w.sh.nh), w.nc, w.sh.head, out);
  } else {
    rc = wide_add_bias_col0(a.O, a.opad, w.b(w.sh.nh), B, st);
    if (rc) return rc;
    value_err_kernel<<<grid1d(B), 256, 0, st>>>(B, batch_src(bt, bt->v_bar, 1), a.O, 0.f, out);
  }
  return check_launch("wide forward rows");
}

}  // namespace cacto
