// gather.cu -- K4: replay-ring gather (ReplayBuffer.sample_minibatch,
// buffer.py:132-138) and FIFO append (push_many, buffer.py:108-130), plus K9:
// device replay of NumPy's PCG64 Generator.uniform start sampling
// (envs/__init__.py:119-121), bit-exact.
//
// Gather: one warp per sampled row-block; every column is copied with
// coalesced loads (consecutive lanes read consecutive elements of the
// concatenated row fields) -- the columns are tiny (3n+m+3 values per row),
// so the kernel treats the 5 columns as one logical row of W values.
#include "common.cuh"

namespace cacto {

template <typename T>
struct Cols {
  const T* src[5];
  T* dst[5];
  int width[5];
};

// One warp per group of 32 sampled rows: the warp loads the 32 indices once
// (one coalesced 256 B read), then copies each column's contiguous
// [32 x width] output block with consecutive lanes on consecutive elements; the
// source row of element e is broadcast from lane e / width by a shuffle, so all
// index arithmetic is 32-bit and there is no per-element 64-bit division.
template <typename T>
__global__ void __launch_bounds__(256) gather_kernel(Cols<T> c, const int64_t* __restrict__ idx,
                                                     const int64_t* cycle, int64_t stride, int64_t B) {
  if (cycle) idx += (*cycle) * stride;
  const int lane = threadIdx.x & 31;
  const int64_t groups = (B + 31) >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < groups; g += nwarps) {
    const int64_t b0 = g << 5;
    const int nb = B - b0 < 32 ? (int)(B - b0) : 32;
    const int64_t my_row = lane < nb ? __ldg(idx + b0 + lane) : 0;
#pragma unroll
    for (int col = 0; col < 5; ++col) {
      const int w = c.width[col];
      const int tot = nb * w;
      const int span = ((32 * w) + 31) & ~31;  // uniform trip count: every lane joins the shuffles
      const T* __restrict__ src = c.src[col];
      T* __restrict__ dst = c.dst[col] + b0 * w;
      for (int e = lane; e < span; e += 32) {
        const int r = e / w;
        const int64_t row = __shfl_sync(0xffffffffu, my_row, r & 31);
        if (e < tot) dst[e] = __ldg(src + row * w + (e - r * w));
      }
    }
  }
}

// FIFO append: row r lands in slot (cursor + r) % capacity, so within one column
// element e of the source goes to (cursor * w + e) mod (capacity * w) -- both
// sides contiguous, the modulo a single conditional subtract (cursor < capacity,
// rows <= capacity).
template <typename T>
__global__ void ring_push_kernel(Cols<T> c, int64_t rows, int64_t capacity, int64_t cursor) {
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
#pragma unroll
  for (int col = 0; col < 5; ++col) {
    const int64_t w = c.width[col];
    const int64_t total = rows * w, cap_w = capacity * w, base = cursor * w;
    const T* __restrict__ src = c.src[col];
    T* __restrict__ dst = c.dst[col];
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += step) {
      int64_t o = base + e;
      if (o >= cap_w) o -= cap_w;
      dst[o] = src[e];
    }
  }
}

// ---- PCG64 (numpy/random/src/pcg64): 128-bit LCG, advance then XSL-RR ------
struct U128 {
  unsigned long long hi, lo;
};
CACTO_D U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
  return r;
}
CACTO_D U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}
// state after `delta` LCG steps (Brown's jump-ahead)
CACTO_D U128 pcg_advance(U128 state, U128 inc, unsigned long long delta) {
  U128 mult = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};
  U128 acc_mult = {0, 1}, acc_plus = {0, 0};
  U128 cur_mult = mult, cur_plus = inc;
  while (delta) {
    if (delta & 1ull) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, U128{0, 1}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  return add128(mul128(acc_mult, state), acc_plus);
}
CACTO_D unsigned long long pcg_output(U128 s) {
  unsigned long long x = s.hi ^ s.lo;
  unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__global__ void sample_states_kernel(U128 state, U128 inc, int64_t first_row, int64_t N, int n,
                                     const double* __restrict__ lo, const double* __restrict__ hi, double* x) {
  U128 mult = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    // draw d of the stream uses the state advanced d+1 times
    U128 s = pcg_advance(state, inc, (unsigned long long)((first_row + i) * n));
    for (int j = 0; j < n; ++j) {
      s = add128(mul128(s, mult), inc);
      double u = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
      // separate multiply and add (no FMA contraction) to match NumPy bit for bit
      x[i * n + j] = __dadd_rn(__dmul_rn(u, __dsub_rn(hi[j], lo[j])), lo[j]);
    }
  }
}

template <typename T>
static Cols<T> batch_cols(const cacto_batch_t* b) {
  Cols<T> c{};
  c.src[0] = (const T*)b->xa;
  c.src[1] = (const T*)b->u;
  c.src[2] = (const T*)b->v_bar;
  c.src[3] = (const T*)b->v_bar_x;
  c.src[4] = (const T*)b->xa_plus_k;
  c.width[0] = b->n + 1;
  c.width[1] = b->m;
  c.width[2] = 1;
  c.width[3] = b->n;
  c.width[4] = b->n + 1;
  return c;
}

static unsigned grid_for(int64_t work) {
  int64_t b = (work + 255) / 256;
  int64_t cap = 16 * (int64_t)num_sms();
  if (b > cap) b = cap;
  return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace cacto

using namespace cacto;

extern "C" int cacto_gather(const cacto_batch_t* ring, void* xa, void* u, void* v_bar, void* v_bar_x,
                            void* xa_plus_k, void* stream) {
  if (!ring || !ring->idx) return set_error(CACTO_EVALUE, "gather: ring with indices required");
  if (ring->rows < 0) return set_error(CACTO_EVALUE, "gather: negative rows");
  if (ring->rows == 0) return CACTO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (ring->dtype == CACTO_F32) {
    Cols<float> c = batch_cols<float>(ring);
    c.dst[0] = (float*)xa; c.dst[1] = (float*)u; c.dst[2] = (float*)v_bar; c.dst[3] = (float*)v_bar_x;
    c.dst[4] = (float*)xa_plus_k;
    gather_kernel<float><<<grid_for(ring->rows * 8), 256, 0, st>>>(c, ring->idx, ring->cycle, ring->idx_stride,
                                                                    ring->rows);
  } else {
    Cols<double> c = batch_cols<double>(ring);
    c.dst[0] = (double*)xa; c.dst[1] = (double*)u; c.dst[2] = (double*)v_bar; c.dst[3] = (double*)v_bar_x;
    c.dst[4] = (double*)xa_plus_k;
    gather_kernel<double><<<grid_for(ring->rows * 8), 256, 0, st>>>(c, ring->idx, ring->cycle, ring->idx_stride,
                                                                     ring->rows);
  }
  return check_launch("gather_kernel");
}

extern "C" int cacto_ring_push(const cacto_batch_t* src, void* ring_xa, void* ring_u, void* ring_v_bar,
                               void* ring_v_bar_x, void* ring_xa_plus_k, int64_t capacity, int64_t cursor,
                               void* stream) {
  if (!src || capacity < 1 || src->rows > capacity || src->rows < 0 || cursor < 0 || cursor >= capacity)
    return set_error(CACTO_EVALUE, "ring_push: bad sizes");
  if (src->rows == 0) return CACTO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t W = 3 * src->n + src->m + 3;
  if (src->dtype == CACTO_F32) {
    Cols<float> c = batch_cols<float>(src);
    c.dst[0] = (float*)ring_xa; c.dst[1] = (float*)ring_u; c.dst[2] = (float*)ring_v_bar;
    c.dst[3] = (float*)ring_v_bar_x; c.dst[4] = (float*)ring_xa_plus_k;
    ring_push_kernel<float><<<grid_for(src->rows * W), 256, 0, st>>>(c, src->rows, capacity, cursor);
  } else {
    Cols<double> c = batch_cols<double>(src);
    c.dst[0] = (double*)ring_xa; c.dst[1] = (double*)ring_u; c.dst[2] = (double*)ring_v_bar;
    c.dst[3] = (double*)ring_v_bar_x; c.dst[4] = (double*)ring_xa_plus_k;
    ring_push_kernel<double><<<grid_for(src->rows * W), 256, 0, st>>>(c, src->rows, capacity, cursor);
  }
  return check_launch("ring_push_kernel");
}

extern "C" int cacto_sample_states(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                                   int64_t first_row, int64_t N, int32_t n, const double* lo, const double* hi,
                                   double* x, void* stream) {
  if (N < 0 || n < 1) return set_error(CACTO_EVALUE, "sample_states: bad sizes");
  if (N == 0) return CACTO_OK;
  U128 s = {state_hi, state_lo}, inc = {inc_hi, inc_lo};
  sample_states_kernel<<<grid_for(N), 256, 0, (cudaStream_t)stream>>>(s, inc, first_row, N, n, lo, hi, x);
  return check_launch("sample_states_kernel");
}
