// common.cuh -- shared device helpers for the CACTO-BIC sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "cacto_b200.h"

#define CACTO_HD __host__ __device__ __forceinline__
#define CACTO_D __device__ __forceinline__

namespace cacto {

constexpr int kThreads = 256;  // every tile kernel runs 8 warps

// ---- status / error plumbing (abi.cu) -------------------------------------
int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);

// ---- math wrappers (float / double overloads) -----------------------------
CACTO_D float m_exp(float x) { return expf(x); }
CACTO_D double m_exp(double x) { return exp(x); }
CACTO_D float m_expm1(float x) { return expm1f(x); }
CACTO_D double m_expm1(double x) { return expm1(x); }
CACTO_D float m_log1p(float x) { return log1pf(x); }
CACTO_D double m_log1p(double x) { return log1p(x); }
CACTO_D float m_log(float x) { return logf(x); }
CACTO_D double m_log(double x) { return log(x); }
CACTO_D float m_tanh(float x) { return tanhf(x); }
CACTO_D double m_tanh(double x) { return tanh(x); }
CACTO_D float m_sqrt(float x) { return sqrtf(x); }
CACTO_D double m_sqrt(double x) { return sqrt(x); }
CACTO_D float m_cosh(float x) { return coshf(x); }
CACTO_D double m_cosh(double x) { return cosh(x); }
CACTO_D float m_sinh(float x) { return sinhf(x); }
CACTO_D double m_sinh(double x) { return sinh(x); }
CACTO_D void m_sincos(float x, float* s, float* c) { sincosf(x, s, c); }
CACTO_D void m_sincos(double x, double* s, double* c) { sincos(x, s, c); }
CACTO_D float m_cospi(float x) { return cospif(x); }
CACTO_D double m_cospi(double x) { return cospi(x); }

// np.logaddexp(0, z) (npy_logaddexp: equal args -> x + log 2; NaN propagates)
template <typename T>
CACTO_D T softplus(T z) {
  if (z == T(0)) return T(0.69314718055994530942);
  if (z > T(0)) return z + m_log1p(m_exp(-z));
  if (z <= T(0)) return m_log1p(m_exp(z));
  return z;  // NaN
}
// fp32 cost-field terms on the SFU (the rollout epilogue's per-start work):
// np.logaddexp(0, z) = max(z, 0) + log1p(exp(-|z|)) with ex2 / lg2.approx
// (absolute error ~2e-7, vs the cost's O(10^2-10^3) per-step scale; log1p of a
// small argument by its series), exp(x) = ex2(x log2 e).  NaN propagates,
// +-inf give inf / 0 like NumPy.  fp64 keeps the libm forms (bit-level parity).
CACTO_D float sfu_ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
CACTO_D float sfu_lg2(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
CACTO_D float cost_exp(float x) { return sfu_ex2(x * 1.4426950408889634f); }
CACTO_D double cost_exp(double x) { return exp(x); }
CACTO_D float cost_softplus(float z) {
  const float e = sfu_ex2(-fabsf(z) * 1.4426950408889634f);
  const float l = e < 1e-3f ? e * fmaf(-0.5f, e, 1.f) : sfu_lg2(1.f + e) * 0.6931471805599453f;
  return fmaxf(z, 0.f) + l;
}
template <typename T>
CACTO_D T softplus(T z);
CACTO_D double cost_softplus(double z) { return softplus(z); }

// exp(z - logaddexp(0, z)) (nets.py:59-60, costs.py:26-29)
template <typename T>
CACTO_D T sigmoid(T z) { return m_exp(z - softplus(z)); }

// activation value / first derivative / the factor h with d2 = h * d1
// (ELU: h = [z <= 0]; tanh: h = -2 tanh z), nets.py:27-52
template <typename T>
CACTO_D T act_value(int act, T z) {
  if (act == CACTO_ACT_ELU) return z > T(0) ? z : m_expm1(z);
  return m_tanh(z);
}
// forward-pass activation: fp32 ELU uses the SFU exponential (__expf(z) - 1,
// abs. error ~1e-7, inside the fp32 tolerance); fp64 keeps expm1 exactly
CACTO_D float act_fast(int act, float z) {
  if (act == CACTO_ACT_ELU) return z > 0.0f ? z : __expf(z) - 1.0f;
  return tanhf(z);
}
CACTO_D double act_fast(int act, double z) { return act_value(act, z); }
template <typename T>
CACTO_D T act_d1(int act, T z) {
  if (act == CACTO_ACT_ELU) return z > T(0) ? T(1) : m_exp(z);
  T t = m_tanh(z);
  return T(1) - t * t;
}
template <typename T>
CACTO_D T act_h(int act, T z) {
  if (act == CACTO_ACT_ELU) return z > T(0) ? T(0) : T(1);
  return T(-2) * m_tanh(z);
}

// ---- 4-wide vector access (16B for float, 2x16B for double) ---------------
template <typename T> struct V4 { T v[4]; };

CACTO_D V4<float> ld4(const float* p) {
  float4 a = *reinterpret_cast<const float4*>(p);
  return {{a.x, a.y, a.z, a.w}};
}
CACTO_D V4<double> ld4(const double* p) {
  double2 a = *reinterpret_cast<const double2*>(p);
  double2 b = *reinterpret_cast<const double2*>(p + 2);
  return {{a.x, a.y, b.x, b.y}};
}
CACTO_D void st4(float* p, const V4<float>& v) {
  *reinterpret_cast<float4*>(p) = make_float4(v.v[0], v.v[1], v.v[2], v.v[3]);
}
CACTO_D void st4(double* p, const V4<double>& v) {
  *reinterpret_cast<double2*>(p) = make_double2(v.v[0], v.v[1]);
  *reinterpret_cast<double2*>(p + 2) = make_double2(v.v[2], v.v[3]);
}

// ---- explicit shared-memory access (32-bit shared-window addresses) ---------
// The tile loops address shared memory through 32-bit offsets so that every
// access is an LDS/STS even when pointers pass through helper structs.
CACTO_D uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
CACTO_D V4<float> lds4(uint32_t a, float*) {
  V4<float> r;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
               : "r"(a));
  return r;
}
CACTO_D V4<double> lds4(uint32_t a, double*) {
  V4<double> r;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "r"(a));
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.v[2]), "=d"(r.v[3]) : "r"(a + 16));
  return r;
}
CACTO_D float lds1(uint32_t a, float*) {
  float r;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(a));
  return r;
}
CACTO_D double lds1(uint32_t a, double*) {
  double r;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(a));
  return r;
}
CACTO_D void sts4(uint32_t a, const V4<float>& v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.v[0]), "f"(v.v[1]), "f"(v.v[2]),
               "f"(v.v[3])
               : "memory");
}
CACTO_D void sts4(uint32_t a, const V4<double>& v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.v[0]), "d"(v.v[1]) : "memory");
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a + 16), "d"(v.v[2]), "d"(v.v[3]) : "memory");
}

// ---- padded parameter layout (see include/cacto_b200.h) --------------------
CACTO_HD int padded_in(int in) { return in <= 8 ? 8 : (in <= 16 ? 16 : 32); }

struct NetShape {
  int L;        // affine layers
  int nh;       // hidden layers = L - 1
  int in, ip;   // true / padded input width
  int out;      // output width
  int hp;       // padded hidden width
  int act, head;
};

CACTO_HD NetShape shape_of(const cacto_mlp_t& m) {
  NetShape s;
  s.L = m.n_layers;
  s.nh = m.n_layers - 1;
  s.in = m.sizes[0];
  s.ip = padded_in(m.sizes[0]);
  s.out = m.sizes[m.n_layers];
  s.hp = m.n_layers > 1 ? m.hp : 32;  // single affine layer: no hidden width
  s.act = m.activation;
  s.head = m.head;
  return s;
}

// offsets (elements) of W_i and b_i in the padded buffer
struct LayerOffsets {
  int64_t w[CACTO_MAX_LAYERS];
  int64_t b[CACTO_MAX_LAYERS];
  int rows[CACTO_MAX_LAYERS];  // padded out width of layer i
  int cols[CACTO_MAX_LAYERS];  // padded in width of layer i
  int64_t total;
};

CACTO_HD LayerOffsets layer_offsets(const NetShape& s) {
  LayerOffsets o;
  int64_t off = 0;
  for (int i = 0; i < s.L; ++i) {
    int cols = (i == 0) ? s.ip : s.hp;
    int rows = (i == s.L - 1) ? s.out : s.hp;
    o.rows[i] = rows;
    o.cols[i] = cols;
    o.w[i] = off;
    off += (int64_t)rows * cols;
    o.b[i] = off;
    off += rows;
  }
  o.total = off;
  return o;
}

// ---- small device-side copies of descriptor constants ----------------------
template <typename T>
struct NetConst {
  T in_center[CACTO_MAX_IN];
  T in_inv_half[CACTO_MAX_IN];  // unused; normalisation divides like the reference
  T in_half[CACTO_MAX_IN];
  T out_scale[CACTO_MAX_OUT];
  T sigma_min;
  int has_norm;
};

template <typename T>
NetConst<T> net_const(const cacto_mlp_t& m) {
  NetConst<T> c;
  for (int i = 0; i < CACTO_MAX_IN; ++i) {
    bool v = m.has_norm && i < m.sizes[0];
    c.in_center[i] = v ? (T)m.in_center[i] : T(0);
    c.in_half[i] = v ? (T)m.in_half[i] : T(1);
    c.in_inv_half[i] = T(1) / c.in_half[i];
  }
  for (int i = 0; i < CACTO_MAX_OUT; ++i) c.out_scale[i] = (T)m.out_scale[i];
  c.sigma_min = (T)m.sigma_min;
  c.has_norm = m.has_norm;
  return c;
}

// head value / chain (nets.py:144-162)
template <typename T>
CACTO_D T head_value(int head, const NetConst<T>& c, int j, T o) {
  if (head == CACTO_HEAD_TANH) return c.out_scale[j] * m_tanh(o);
  if (head == CACTO_HEAD_STD) return c.sigma_min + softplus(o);
  return o;
}
template <typename T>
CACTO_D T head_chain(int head, const NetConst<T>& c, int j, T o) {
  if (head == CACTO_HEAD_TANH) {
    T t = m_tanh(o);
    return c.out_scale[j] * (T(1) - t * t);
  }
  if (head == CACTO_HEAD_STD) return sigmoid(o);
  return T(1);
}

// set the dynamic shared-memory opt-in of a kernel once (idempotent, so no
// runtime attribute call happens inside a CUDA-graph capture after warm-up)
bool ensure_smem(const void* kernel, size_t bytes);

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace cacto
