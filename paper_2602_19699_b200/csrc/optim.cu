// optim.cu -- K8: fold the per-CTA gradient slots, Adam with bias correction
// (nets.adam_step, nets.py:375-392) and Polyak averaging (nets.polyak,
// nets.py:395-398), optionally fused into one pass over the parameters.
//
// Arithmetic follows the reference expression order with explicitly rounded
// multiplies/adds (no FMA contraction), so the float64 update is bit-identical
// to NumPy's for identical gradients.
#include "common.cuh"

namespace cacto {

CACTO_D float r_mul(float a, float b) { return __fmul_rn(a, b); }
CACTO_D double r_mul(double a, double b) { return __dmul_rn(a, b); }
CACTO_D float r_add(float a, float b) { return __fadd_rn(a, b); }
CACTO_D double r_add(double a, double b) { return __dadd_rn(a, b); }
CACTO_D float r_sub(float a, float b) { return __fsub_rn(a, b); }
CACTO_D double r_sub(double a, double b) { return __dsub_rn(a, b); }
CACTO_D float r_div(float a, float b) { return __fdiv_rn(a, b); }
CACTO_D double r_div(double a, double b) { return __ddiv_rn(a, b); }
CACTO_D float r_sqrt(float a) { return __fsqrt_rn(a); }
CACTO_D double r_sqrt(double a) { return __dsqrt_rn(a); }

template <typename T>
struct AdamK {
  T lr, b1, b2, eps, one_m_b1, one_m_b2, bc1, bc2;
};

template <typename T>
AdamK<T> adam_consts(int64_t step, double lr, double b1, double b2, double eps) {
  // t = step + 1; bc = 1 - beta**t in double precision like Python floats
  double t = (double)(step + 1);
  AdamK<T> k;
  k.lr = (T)lr;
  k.b1 = (T)b1;
  k.b2 = (T)b2;
  k.eps = (T)eps;
  k.one_m_b1 = (T)(1.0 - b1);
  k.one_m_b2 = (T)(1.0 - b2);
  k.bc1 = (T)(1.0 - pow(b1, t));
  k.bc2 = (T)(1.0 - pow(b2, t));
  return k;
}

template <typename T>
CACTO_D void adam_one(const AdamK<T>& k, T g, T& p, T& m, T& v) {
  m = r_add(r_mul(k.b1, m), r_mul(k.one_m_b1, g));
  v = r_add(r_mul(k.b2, v), r_mul(k.one_m_b2, r_mul(g, g)));
  T num = r_mul(k.lr, r_div(m, k.bc1));
  T den = r_add(r_sqrt(r_div(v, k.bc2)), k.eps);
  p = r_sub(p, r_div(num, den));
}

template <typename T>
__global__ void adam_kernel(T* p, T* m, T* v, const T* __restrict__ g, int64_t P, AdamK<T> k) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    T pp = p[i], mm = m[i], vv = v[i];
    adam_one(k, g[i], pp, mm, vv);
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
  }
}

template <typename T>
__global__ void polyak_kernel(T* tgt, const T* __restrict__ on, int64_t P, T one_m_tau, T tau) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x)
    tgt[i] = r_add(r_mul(one_m_tau, tgt[i]), r_mul(tau, on[i]));
}

// sum of the n_partials slots ([n][P+1]) in slot order
template <typename T>
CACTO_D T fold(const T* __restrict__ ws, int n, int64_t stride, int64_t i) {
  T s = T(0);
  for (int g = 0; g < n; ++g) s += ws[(int64_t)g * stride + i];
  return s;
}

template <typename T>
__global__ void reduce_kernel(const T* __restrict__ ws, int n, int64_t P, T* grad, T* loss) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= P; i += (int64_t)gridDim.x * blockDim.x) {
    T s = fold(ws, n, P + 1, i);
    if (i < P) {
      if (grad) grad[i] = s;
    } else if (loss) {
      *loss = s;
    }
  }
}

template <typename T>
__global__ void reduce_adam_kernel(const T* __restrict__ ws, int n, int64_t P, T* p, T* m, T* v, AdamK<T> k, T* tgt,
                                   T one_m_tau, T tau, T* grad_out, T* loss_out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= P; i += (int64_t)gridDim.x * blockDim.x) {
    T g = fold(ws, n, P + 1, i);
    if (i == P) {
      if (loss_out) *loss_out = g;
      continue;
    }
    if (grad_out) grad_out[i] = g;
    T pp = p[i], mm = m[i], vv = v[i];
    adam_one(k, g, pp, mm, vv);
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
    if (tgt) tgt[i] = r_add(r_mul(one_m_tau, tgt[i]), r_mul(tau, pp));  // trainer.py:219-220
  }
}

template <typename T>
__global__ void reduce_adam_graph_kernel(const T* __restrict__ ws, int n, int64_t P, T* p, T* m, T* v,
                                         const int64_t* counter, const int64_t* step_base, const double* bc1,
                                         const double* bc2, T lr, T b1, T b2, T eps, T one_m_b1, T one_m_b2, T* tgt,
                                         T one_m_tau, T tau, T* loss_base, T* ring = nullptr, int64_t ring_n = 1,
                                         int64_t ring_ld = 0) {
  const int64_t c = *counter;
  // optional: the updated parameters also into ring slot c % ring_n (the ring_copy of
  // the pipelined M-cycle loop, engine.py, fused into the update: one launch less)
  T* rslot = ring ? ring + (c % ring_n) * ring_ld : nullptr;
  const int64_t t = *step_base + c + 1;
  AdamK<T> k;
  k.lr = lr;
  k.b1 = b1;
  k.b2 = b2;
  k.eps = eps;
  k.one_m_b1 = one_m_b1;
  k.one_m_b2 = one_m_b2;
  k.bc1 = (T)bc1[t];
  k.bc2 = (T)bc2[t];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= P; i += (int64_t)gridDim.x * blockDim.x) {
    T g = fold(ws, n, P + 1, i);
    if (i == P) {
      if (loss_base) loss_base[c] = g;
      continue;
    }
    T pp = p[i], mm = m[i], vv = v[i];
    adam_one(k, g, pp, mm, vv);
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
    if (tgt) tgt[i] = r_add(r_mul(one_m_tau, tgt[i]), r_mul(tau, pp));
    if (rslot) rslot[i] = pp;
  }
}

__global__ void counter_tick_kernel(int64_t* c) { *c += 1; }

// ring slot (*counter % ring) of a [ring][P] buffer <-> a [P] vector
template <typename T>
__global__ void ring_copy_kernel(T* ring, const int64_t* counter, int64_t ring_n, int64_t ld, int64_t P, T* vec,
                                 int save) {
  T* slot = ring + (*counter % ring_n) * ld;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    if (save)
      slot[i] = vec[i];
    else
      vec[i] = slot[i];
  }
}

static unsigned grid_of(int64_t P) {
  int64_t b = (P + 255) / 256;
  int64_t cap = 8 * (int64_t)num_sms();
  if (b > cap) b = cap;
  return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace cacto

using namespace cacto;

extern "C" int cacto_adam_step(int32_t dtype, void* params, void* m, void* v, const void* grad, int64_t P,
                               int64_t step, double lr, double beta1, double beta2, double eps, void* stream) {
  if (P < 0 || (P > 0 && (!params || !m || !v || !grad))) return set_error(CACTO_EVALUE, "adam: bad arguments");
  if (P == 0) return CACTO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CACTO_F32)
    adam_kernel<float><<<grid_of(P), 256, 0, st>>>((float*)params, (float*)m, (float*)v, (const float*)grad, P,
                                                   adam_consts<float>(step, lr, beta1, beta2, eps));
  else
    adam_kernel<double><<<grid_of(P), 256, 0, st>>>((double*)params, (double*)m, (double*)v, (const double*)grad, P,
                                                    adam_consts<double>(step, lr, beta1, beta2, eps));
  return check_launch("adam_kernel");
}

extern "C" int cacto_polyak(int32_t dtype, void* target, const void* online, int64_t P, double tau, void* stream) {
  if (P < 0 || (P > 0 && (!target || !online))) return set_error(CACTO_EVALUE, "polyak: bad arguments");
  if (P == 0) return CACTO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CACTO_F32)
    polyak_kernel<float><<<grid_of(P), 256, 0, st>>>((float*)target, (const float*)online, P, (float)(1.0 - tau),
                                                     (float)tau);
  else
    polyak_kernel<double><<<grid_of(P), 256, 0, st>>>((double*)target, (const double*)online, P, 1.0 - tau, tau);
  return check_launch("polyak_kernel");
}

extern "C" int cacto_reduce_grads(int32_t dtype, const void* workspace, int32_t n_partials, int64_t P, void* grad,
                                  void* loss, void* stream) {
  if (!workspace || n_partials < 1 || P < 0) return set_error(CACTO_EVALUE, "reduce_grads: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CACTO_F32)
    reduce_kernel<float><<<grid_of(P + 1), 256, 0, st>>>((const float*)workspace, n_partials, P, (float*)grad,
                                                         (float*)loss);
  else
    reduce_kernel<double><<<grid_of(P + 1), 256, 0, st>>>((const double*)workspace, n_partials, P, (double*)grad,
                                                          (double*)loss);
  return check_launch("reduce_kernel");
}

extern "C" int cacto_reduce_adam(int32_t dtype, const void* workspace, int32_t n_partials, int64_t P, void* params,
                                 void* m, void* v, int64_t step, double lr, double beta1, double beta2, double eps,
                                 void* target, double tau, void* grad_out, void* loss_out, void* stream) {
  if (!workspace || n_partials < 1 || P < 0 || !params || !m || !v)
    return set_error(CACTO_EVALUE, "reduce_adam: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CACTO_F32)
    reduce_adam_kernel<float><<<grid_of(P + 1), 256, 0, st>>>(
        (const float*)workspace, n_partials, P, (float*)params, (float*)m, (float*)v,
        adam_consts<float>(step, lr, beta1, beta2, eps), (float*)target, (float)(1.0 - tau), (float)tau,
        (float*)grad_out, (float*)loss_out);
  else
    reduce_adam_kernel<double><<<grid_of(P + 1), 256, 0, st>>>(
        (const double*)workspace, n_partials, P, (double*)params, (double*)m, (double*)v,
        adam_consts<double>(step, lr, beta1, beta2, eps), (double*)target, 1.0 - tau, tau, (double*)grad_out,
        (double*)loss_out);
  return check_launch("reduce_adam_kernel");
}

extern "C" int cacto_reduce_adam_graph(int32_t dtype, const void* workspace, int32_t n_partials, int64_t P,
                                       void* params, void* m, void* v, const int64_t* counter, const int64_t* step_base,
                                       const double* bc1, const double* bc2, double lr, double beta1, double beta2,
                                       double eps, void* target, double tau, void* loss_base, void* stream) {
  if (!workspace || n_partials < 1 || P < 0 || !params || !m || !v || !counter || !step_base || !bc1 || !bc2)
    return set_error(CACTO_EVALUE, "reduce_adam_graph: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CACTO_F32)
    reduce_adam_graph_kernel<float><<<grid_of(P + 1), 256, 0, st>>>(
        (const float*)workspace, n_partials, P, (float*)params, (float*)m, (float*)v, counter, step_base, bc1, bc2,
        (float)lr, (float)beta1, (float)beta2, (float)eps, (float)(1.0 - beta1), (float)(1.0 - beta2),
        (float*)target, (float)(1.0 - tau), (float)tau, (float*)loss_base);
  else
    reduce_adam_graph_kernel<double><<<grid_of(P + 1), 256, 0, st>>>(
        (const double*)workspace, n_partials, P, (double*)params, (double*)m, (double*)v, counter, step_base, bc1,
        bc2, lr, beta1, beta2, eps, 1.0 - beta1, 1.0 - beta2, (double*)target, 1.0 - tau, tau, (double*)loss_base);
  return check_launch("reduce_adam_graph_kernel");
}

extern "C" int cacto_reduce_adam_graph_ring(int32_t dtype, const void* workspace, int32_t n_partials, int64_t P,
                                            void* params, void* m, void* v, const int64_t* counter,
                                            const int64_t* step_base, const double* bc1, const double* bc2, double lr,
                                            double beta1, double beta2, double eps, void* target, double tau,
                                            void* loss_base, void* ring, int64_t ring_n, int64_t ring_ld,
                                            void* stream) {
  if (!workspace || n_partials < 1 || P < 0 || !params || !m || !v || !counter || !step_base || !bc1 || !bc2 ||
      !ring || ring_n < 1 || ring_ld < P)
    return set_error(CACTO_EVALUE, "reduce_adam_graph_ring: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CACTO_F32)
    reduce_adam_graph_kernel<float><<<grid_of(P + 1), 256, 0, st>>>(
        (const float*)workspace, n_partials, P, (float*)params, (float*)m, (float*)v, counter, step_base, bc1, bc2,
        (float)lr, (float)beta1, (float)beta2, (float)eps, (float)(1.0 - beta1), (float)(1.0 - beta2),
        (float*)target, (float)(1.0 - tau), (float)tau, (float*)loss_base, (float*)ring, ring_n, ring_ld);
  else
    reduce_adam_graph_kernel<double><<<grid_of(P + 1), 256, 0, st>>>(
        (const double*)workspace, n_partials, P, (double*)params, (double*)m, (double*)v, counter, step_base, bc1,
        bc2, lr, beta1, beta2, eps, 1.0 - beta1, 1.0 - beta2, (double*)target, 1.0 - tau, tau, (double*)loss_base,
        (double*)ring, ring_n, ring_ld);
  return check_launch("reduce_adam_graph_kernel");
}

extern "C" int cacto_ring_copy(int32_t dtype, void* ring, const int64_t* counter, int64_t ring_n, int64_t ld,
                               int64_t P, void* vec, int32_t save, void* stream) {
  if (!ring || !counter || !vec || ring_n < 1 || P < 0 || ld < P)
    return set_error(CACTO_EVALUE, "ring_copy: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CACTO_F32)
    ring_copy_kernel<float><<<grid_of(P), 256, 0, st>>>((float*)ring, counter, ring_n, ld, P, (float*)vec, save);
  else
    ring_copy_kernel<double><<<grid_of(P), 256, 0, st>>>((double*)ring, counter, ring_n, ld, P, (double*)vec, save);
  return check_launch("ring_copy_kernel");
}

__global__ void counter_span_kernel(int64_t* base, int64_t* span, int k) {
  const int64_t b = *base;
  for (int i = threadIdx.x; i < k; i += blockDim.x) span[i] = b + i;
  __syncthreads();
  if (threadIdx.x == 0) *base = b + k;
}

extern "C" int cacto_counter_span(int64_t* base, int64_t* span, int32_t k, void* stream) {
  if (!base || !span || k < 1) return set_error(CACTO_EVALUE, "counter_span: bad arguments");
  counter_span_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(base, span, k);
  return check_launch("counter_span_kernel");
}

extern "C" int cacto_counter_tick(int64_t* counter, void* stream) {
  if (!counter) return set_error(CACTO_EVALUE, "counter_tick: null counter");
  counter_tick_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(counter);
  return check_launch("counter_tick_kernel");
}
