// select.cu -- K3: stable descending top-k, exactly
//   order = np.argsort(-scores, kind="stable")[:keep]        (trainer.py:152)
// i.e. larger score first, equal scores by ascending index, NaN last and
// -0.0 == +0.0.  Scores map to order-preserving unsigned keys (ascending key =
// descending score); (key, index) pairs are unique, so any exact selection +
// sort of the pairs reproduces the stable argsort.
//
//  1. radix select (cooperative kernel, 8-bit digits, MSB first): threshold key
//     K* with #(key < K*) < keep <= #(key <= K*), warp-privatised histograms
//  2. ordered compaction: all keys < K*, plus the lowest-index keep-#(<K*)
//     keys == K* (ballot/popc prefix in index order across the grid)
//  3. sort the keep survivors: bitonic sort of 2048-pair chunks in shared
//     memory, then merge passes (merge-path lower_bound)
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace cacto {

struct Pair {
  unsigned long long key;
  long long idx;
};

CACTO_D bool pair_less(const Pair& a, const Pair& b) {
  return a.key < b.key || (a.key == b.key && a.idx < b.idx);
}

// fp32 scores with N < 2^32: (32-bit key, 32-bit index) packed in one 64-bit
// word whose unsigned order is the pair order -- half the bytes per sort step
// and a single compare.  fp64 (64-bit keys) and shard merges keep `Pair`.
typedef unsigned long long Packed;
CACTO_D bool elem_less(Packed a, Packed b) { return a < b; }
CACTO_D bool elem_less(const Pair& a, const Pair& b) { return pair_less(a, b); }
CACTO_D void make_elem(Packed& e, unsigned long long k, long long i) { e = (k << 32) | (unsigned long long)(unsigned int)i; }
CACTO_D void make_elem(Pair& e, unsigned long long k, long long i) { e = Pair{k, i}; }
CACTO_D void make_pad(Packed& e) { e = ~0ull; }
CACTO_D void make_pad(Pair& e) { e = Pair{~0ull, 0x7fffffffffffffffll}; }
CACTO_D unsigned long long elem_key(Packed e) { return e >> 32; }
CACTO_D unsigned long long elem_key(const Pair& e) { return e.key; }
CACTO_D long long elem_idx(Packed e) { return (long long)(e & 0xffffffffull); }
CACTO_D long long elem_idx(const Pair& e) { return e.idx; }
CACTO_D Packed shfl_elem(Packed v, int j) { return __shfl_xor_sync(0xffffffffu, v, j); }
CACTO_D Pair shfl_elem(const Pair& v, int j) {
  return Pair{__shfl_xor_sync(0xffffffffu, v.key, j), __shfl_xor_sync(0xffffffffu, v.idx, j)};
}

// keys: NaN -> (max - 1), the max key is reserved for padding rows of merged runs
CACTO_D unsigned long long score_key(float s) {
  if (s != s) return 0xFFFFFFFEull;  // NaN last
  if (s == 0.0f) s = 0.0f;           // -0.0 -> +0.0
  unsigned int b = __float_as_uint(s);
  unsigned int u = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return (unsigned long long)(~u);
}
CACTO_D unsigned long long score_key(double s) {
  if (s != s) return 0xFFFFFFFFFFFFFFFEull;
  if (s == 0.0) s = 0.0;
  unsigned long long b = (unsigned long long)__double_as_longlong(s);
  unsigned long long u = (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
  return ~u;
}
CACTO_D float key_score(unsigned long long k, float*) {
  if (k >= 0xFFFFFFFEull) return __uint_as_float(0x7fc00000u);
  unsigned int u = ~(unsigned int)k;
  unsigned int b = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
  return __uint_as_float(b);
}
CACTO_D double key_score(unsigned long long k, double*) {
  if (k >= 0xFFFFFFFFFFFFFFFEull) return __longlong_as_double(0x7ff8000000000000ll);
  unsigned long long u = ~k;
  unsigned long long b = (u & 0x8000000000000000ull) ? (u & 0x7FFFFFFFFFFFFFFFull) : ~u;
  return __longlong_as_double((long long)b);
}

constexpr int kSelThreads = 256;
constexpr int kSortChunk = 2048;
constexpr int kMaxSelBlocks = 1024;
constexpr int kSelBatch = 4;  // candidates per thread per histogram sweep

struct SelState {
  unsigned int hist[8][256];
  unsigned long long n_lt;
  unsigned int block_eq[kMaxSelBlocks];
};

template <typename T, int KB, typename E>
__global__ void __launch_bounds__(kSelThreads) radix_select_kernel(const T* __restrict__ scores, int64_t N,
                                                                   int64_t keep, SelState* st, E* __restrict__ sel) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned int wh[kSelThreads / 32][256];
  __shared__ unsigned long long s_prefix;
  __shared__ long long s_need;
  __shared__ unsigned int s_warp[kSelThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = gridDim.x;
  const int64_t chunk = (N + G - 1) / G;
  const int64_t c0 = blockIdx.x * chunk;
  const int64_t c1 = c0 + chunk < N ? c0 + chunk : N;

  unsigned long long prefix = 0;
  long long need = keep;
  constexpr int PASSES = KB / 8;
  for (int p = 0; p < PASSES; ++p) {
    const int shift = KB - 8 * (p + 1);
    for (int q = tid; q < (kSelThreads / 32) * 256; q += kSelThreads) (&wh[0][0])[q] = 0;
    __syncthreads();
    // kSelBatch independent loads in flight per thread before the histogram updates
    for (int64_t i0 = c0 + tid; i0 < c1; i0 += kSelBatch * kSelThreads) {
      T v[kSelBatch];
#pragma unroll
      for (int u = 0; u < kSelBatch; ++u) {
        const int64_t i = i0 + u * kSelThreads;
        v[u] = i < c1 ? scores[i] : T(0);
      }
#pragma unroll
      for (int u = 0; u < kSelBatch; ++u) {
        const unsigned long long k = score_key(v[u]);
        const bool match = (i0 + u * kSelThreads < c1) &&
                           ((p == 0) || ((k >> (shift + 8)) == (prefix >> (shift + 8))));
        if (match) {
          unsigned int d = (unsigned int)((k >> shift) & 255ull);
          // warp-aggregated increment: lanes with the same digit combine
          unsigned int peers = __match_any_sync(__activemask(), d);
          int leader = __ffs(peers) - 1;
          if (lane == leader) atomicAdd(&wh[warp][d], (unsigned int)__popc(peers));
        }
      }
    }
    __syncthreads();
    for (int d = tid; d < 256; d += kSelThreads) {
      unsigned int c = 0;
#pragma unroll
      for (int w = 0; w < kSelThreads / 32; ++w) c += wh[w][d];
      if (c) atomicAdd(&st->hist[p][d], c);
    }
    grid.sync();
    {
      // threshold digit: block-wide inclusive scan of the 256 bins (one bin per
      // thread), the first digit whose running count reaches `need`
      static_assert(kSelThreads == 256, "one histogram bin per thread");
      const unsigned int h = __ldcg(&st->hist[p][tid]);
      unsigned int x = h;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_warp[warp] = x;
      __syncthreads();
      long long incl = x;
      for (int w = 0; w < warp; ++w) incl += s_warp[w];
      const long long excl = incl - h;
      if (incl >= need && excl < need) {
        s_need = need - excl;
        s_prefix = prefix | ((unsigned long long)tid << shift);
      } else if (tid == 255 && incl < need) {  // unreachable for consistent counts
        s_need = need - incl;
        s_prefix = prefix | (255ull << shift);
      }
    }
    __syncthreads();
    prefix = s_prefix;
    need = s_need;
  }
  // prefix == K*, need == number of K*-equal pairs to take (lowest indices)
  const unsigned long long kstar = prefix;
  const long long need_eq = need;
  const long long n_lt_total = keep - need_eq;

  // ordered count of equal keys in this block's chunk
  unsigned int my_eq = 0;
  for (int64_t b0 = c0; b0 < c1; b0 += kSelBatch * kSelThreads) {
    T v[kSelBatch];
#pragma unroll
    for (int u = 0; u < kSelBatch; ++u) {
      const int64_t i = b0 + u * kSelThreads + tid;
      v[u] = i < c1 ? scores[i] : T(0);
    }
#pragma unroll
    for (int u = 0; u < kSelBatch; ++u) {
      const bool eq = b0 + u * kSelThreads + tid < c1 && score_key(v[u]) == kstar;
      unsigned int b = __ballot_sync(0xffffffffu, eq);
      if (lane == 0) my_eq += __popc(b);
    }
  }
  if (lane == 0) s_warp[warp] = my_eq;
  __syncthreads();
  if (tid == 0) {
    unsigned int tot = 0;
    for (int w = 0; w < kSelThreads / 32; ++w) tot += s_warp[w];
    st->block_eq[blockIdx.x] = tot;
  }
  grid.sync();
  __shared__ long long s_off;
  {
    long long off = 0;
    for (int b = tid; b < (int)blockIdx.x; b += kSelThreads) off += __ldcg(&st->block_eq[b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) off += __shfl_xor_sync(0xffffffffu, off, o);
    if (tid == 0) s_off = 0;
    __syncthreads();
    if (lane == 0 && off) atomicAdd((unsigned long long*)&s_off, (unsigned long long)off);
    __syncthreads();
  }
  long long running = s_off;
  for (int64_t b0 = c0; b0 < c1; b0 += kSelBatch * kSelThreads) {  // block-uniform trip count
    unsigned long long kk[kSelBatch];
#pragma unroll
    for (int u = 0; u < kSelBatch; ++u) {
      const int64_t i = b0 + u * kSelThreads + tid;
      kk[u] = i < c1 ? score_key(scores[i]) : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < kSelBatch; ++u) {
      const int64_t i = b0 + u * kSelThreads + tid;
      const unsigned long long k = kk[u];
      const bool lt = i < c1 && k < kstar;
      const bool eq = i < c1 && k == kstar;
      // keys < K*: any slot order (sorted afterwards); one atomic per warp
      const unsigned int lb = __ballot_sync(0xffffffffu, lt);
      if (lb) {
        unsigned long long wbase = 0;
        if (lane == 0) wbase = atomicAdd(&st->n_lt, (unsigned long long)__popc(lb));
        wbase = __shfl_sync(0xffffffffu, wbase, 0);
        if (lt) make_elem(sel[wbase + __popc(lb & ((1u << lane) - 1u))], k, (long long)i);
      }
      // keys == K*: the lowest-index need_eq of them, in index order
      const unsigned int b = __ballot_sync(0xffffffffu, eq);
      if (lane == 0) s_warp[warp] = __popc(b);
      __syncthreads();
      long long woff = running;
      for (int w = 0; w < warp; ++w) woff += s_warp[w];
      unsigned int tot = 0;
      for (int w = 0; w < kSelThreads / 32; ++w) tot += s_warp[w];
      if (eq) {
        long long r = woff + __popc(b & ((1u << lane) - 1u));
        if (r < need_eq) make_elem(sel[n_lt_total + r], k, (long long)i);
      }
      running += tot;
      __syncthreads();
    }
  }
}

// bitonic sort of kSortChunk-pair chunks (pads with +inf pairs), register
// resident: warp w owns positions [64w, 64w + 64), lane l holds 64w + l and
// 64w + 32 + l.  Exchanges at distance j = 32 stay inside a thread, j < 32 are
// warp shuffles; only the 15 rounds with j >= 64 go through shared memory
// (two barriers each) -- 30 barriers instead of one per round (66).
constexpr int kSortThreads = kSortChunk / 2;

// element at position i keeps min(a, b) if it is the lower of the pair in an
// ascending run, or the upper one in a descending run
template <typename E>
CACTO_D E bitonic_keep(const E& a, const E& b, int i, int j, int k) {
  const bool take_min = ((i & k) == 0) == ((i & j) == 0);
  return (elem_less(b, a) == take_min) ? b : a;
}

// ascending bitonic sort of S = 64..kSortChunk elements held two per thread
// (S / 2 threads), `sh` is S elements of scratch
template <typename E>
CACTO_D void bitonic_sort_regs(E& v0, E& v1, E* sh, int p0, int p1, int S) {
  for (int k = 2; k <= S; k <<= 1) {
    int j = k >> 1;
    for (; j >= 64; j >>= 1) {
      sh[p0] = v0;
      sh[p1] = v1;
      __syncthreads();
      const E b0 = sh[p0 ^ j], b1 = sh[p1 ^ j];
      __syncthreads();
      v0 = bitonic_keep(v0, b0, p0, j, k);
      v1 = bitonic_keep(v1, b1, p1, j, k);
    }
    if (j == 32) {
      const bool up = (p0 & k) == 0;
      if (elem_less(v1, v0) == up) {
        const E t = v0;
        v0 = v1;
        v1 = t;
      }
      j = 16;
    }
    for (; j > 0; j >>= 1) {
      const E b0 = shfl_elem(v0, j), b1 = shfl_elem(v1, j);
      v0 = bitonic_keep(v0, b0, p0, j, k);
      v1 = bitonic_keep(v1, b1, p1, j, k);
    }
  }
}

template <typename E>
__global__ void __launch_bounds__(kSortThreads) chunk_sort_kernel(E* data, int64_t M) {
  __shared__ E sh[kSortChunk];
  const int64_t base = (int64_t)blockIdx.x * kSortChunk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p0 = warp * 64 + lane, p1 = p0 + 32;
  E pad;
  make_pad(pad);
  E v0 = (base + p0 < M) ? data[base + p0] : pad;
  E v1 = (base + p1 < M) ? data[base + p1] : pad;
  bitonic_sort_regs(v0, v1, sh, p0, p1, kSortChunk);
  if (base + p0 < M) data[base + p0] = v0;
  if (base + p1 < M) data[base + p1] = v1;
}

// N <= kSortChunk candidates (e.g. the 750-start CPU-reference config): the whole
// select in one CTA -- keys, one bitonic sort of all N pairs, emit the first keep
template <typename T, typename E>
__global__ void __launch_bounds__(kSortThreads) small_select_kernel(const T* __restrict__ scores, int N, int keep,
                                                                     int64_t base_index, int64_t* order,
                                                                     T* top_scores, int S) {
  __shared__ E sh[kSortChunk];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p0 = warp * 64 + lane, p1 = p0 + 32;
  E v0, v1;
  make_pad(v0);
  make_pad(v1);
  if (p0 < N) make_elem(v0, score_key(scores[p0]), p0);
  if (p1 < N) make_elem(v1, score_key(scores[p1]), p1);
  bitonic_sort_regs(v0, v1, sh, p0, p1, S);
  if (p0 < keep) {
    order[p0] = elem_idx(v0) + base_index;
    if (top_scores) top_scores[p0] = key_score(elem_key(v0), (T*)nullptr);
  }
  if (p1 < keep) {
    order[p1] = elem_idx(v1) + base_index;
    if (top_scores) top_scores[p1] = key_score(elem_key(v1), (T*)nullptr);
  }
}

// merge adjacent sorted runs of width w into runs of width 2w
template <typename E>
__global__ void merge_pass_kernel(const E* __restrict__ in, E* __restrict__ out, int64_t M, int64_t w) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t run = i / w;
    int64_t pair_start = (run / 2) * 2 * w;
    bool left = (run % 2) == 0;
    int64_t my_start = run * w;
    int64_t o_start = left ? my_start + w : pair_start;
    int64_t o_end = left ? my_start + 2 * w : my_start;
    if (o_start > M) o_start = M;
    if (o_end > M) o_end = M;
    const E e = in[i];
    // stable merge: a left-run element goes before equal right-run elements, so it
    // counts the partner elements < e and a right-run element those <= e (equal
    // elements, e.g. the padding pairs of several shards, land in distinct slots)
    int64_t lo = o_start, hi = o_end;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      const E p = in[mid];
      if (left ? elem_less(p, e) : !elem_less(e, p))
        lo = mid + 1;
      else
        hi = mid;
    }
    out[pair_start + (i - my_start) + (lo - o_start)] = e;
  }
}

template <typename T, typename E>
__global__ void emit_kernel(const E* __restrict__ sel, int64_t keep, int64_t base_index, int64_t* order,
                            T* top_scores) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < keep; i += (int64_t)gridDim.x * blockDim.x) {
    const E p = sel[i];
    order[i] = elem_idx(p) + base_index;
    if (top_scores) top_scores[i] = key_score(elem_key(p), (T*)nullptr);
  }
}

template <typename T>
__global__ void runs_to_pairs_kernel(const T* __restrict__ s, const int64_t* __restrict__ idx, int64_t M, Pair* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = Pair{idx[i] < 0 ? ~0ull : score_key(s[i]), (long long)idx[i]};  // idx < 0: padding
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// sorts `M` pairs in a (ping-pong with b); returns the buffer holding the result
template <typename E>
static E* sort_pairs(E* a, E* b, int64_t M, int64_t first_width, cudaStream_t st) {
  int64_t w = first_width;
  if (w <= 0) {
    int64_t chunks = (M + kSortChunk - 1) / kSortChunk;
    if (chunks > 0) chunk_sort_kernel<E><<<(unsigned)chunks, kSortThreads, 0, st>>>(a, M);
    w = kSortChunk;
  }
  E* src = a;
  E* dst = b;
  while (w < M) {
    int64_t blocks = (M + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    merge_pass_kernel<E><<<(unsigned)blocks, 256, 0, st>>>(src, dst, M, w);
    E* t = src;
    src = dst;
    dst = t;
    w *= 2;
  }
  return src;
}

}  // namespace cacto

using namespace cacto;

extern "C" size_t cacto_select_workspace_bytes(int32_t dtype, int64_t N, int64_t keep) {
  (void)dtype;
  (void)N;
  int64_t k = keep > 0 ? keep : 1;
  return align256(sizeof(SelState)) + 2 * align256((size_t)k * sizeof(Pair));
}

template <typename T, typename E>
static int select_run(const T* scores, int64_t N, int64_t keep, int64_t base_index, int64_t* order, T* top,
                      void* ws, cudaStream_t st) {
  if (N <= kSortChunk) {
    int S = 64;
    while (S < N) S <<= 1;
    small_select_kernel<T, E><<<1, S / 2, 0, st>>>(scores, (int)N, (int)keep, base_index, order, top, S);
    return check_launch("small_select_kernel");
  }
  SelState* state = (SelState*)ws;
  E* a = (E*)((char*)ws + align256(sizeof(SelState)));
  E* b = (E*)((char*)a + align256((size_t)keep * sizeof(E)));
  if (cudaMemsetAsync(state, 0, sizeof(SelState), st) != cudaSuccess)
    return set_error(CACTO_ECUDA, "select: memset failed");
  constexpr int KB = sizeof(T) == 4 ? 32 : 64;
  auto kern = radix_select_kernel<T, KB, E>;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kSelThreads, 0);
  if (occ < 1) occ = 1;
  // one load batch per thread when the grid allows (65,536 candidates -> 64 CTAs):
  // each pass is then one round of L2 latency, not eight
  int64_t want = (N + kSelThreads * kSelBatch - 1) / (kSelThreads * kSelBatch);
  int64_t cap = (int64_t)occ * num_sms();
  if (cap > kMaxSelBlocks) cap = kMaxSelBlocks;
  int G = (int)(want < 1 ? 1 : (want > cap ? cap : want));
  void* args[] = {(void*)&scores, (void*)&N, (void*)&keep, (void*)&state, (void*)&a};
  if (cudaLaunchCooperativeKernel((void*)kern, G, kSelThreads, args, 0, st) != cudaSuccess)
    return check_launch("radix_select_kernel (cooperative)");
  E* res = sort_pairs<E>(a, b, keep, 0, st);
  int64_t eb = (keep + 255) / 256;
  emit_kernel<T, E><<<(unsigned)(eb > 4096 ? 4096 : eb), 256, 0, st>>>(res, keep, base_index, order, top);
  return check_launch("select emit");
}

template <typename T>
static int select_entry(const T* scores, int64_t N, int64_t keep, int64_t base_index, int64_t* order, T* top,
                        void* ws, cudaStream_t st) {
  if (sizeof(T) == 4 && N <= 0xFFFFFFFFll)
    return select_run<T, Packed>(scores, N, keep, base_index, order, top, ws, st);
  return select_run<T, Pair>(scores, N, keep, base_index, order, top, ws, st);
}

extern "C" int cacto_select_topk(int32_t dtype, const void* scores, int64_t N, int64_t keep, int64_t base_index,
                                 int64_t* order, void* top_scores, void* workspace, size_t workspace_bytes,
                                 void* stream) {
  if (keep > N) return set_error(CACTO_EVALUE, "keep=%lld exceeds %lld candidates", (long long)keep, (long long)N);
  if (keep < 0 || N < 0) return set_error(CACTO_EVALUE, "select: negative sizes");
  if (keep == 0) return CACTO_OK;
  if (!scores || !order || !workspace) return set_error(CACTO_EVALUE, "select: null buffer");
  if (N > 0xFFFFFFFFll) return set_error(CACTO_EVALUE, "select: N too large");
  if (workspace_bytes < cacto_select_workspace_bytes(dtype, N, keep))
    return set_error(CACTO_EVALUE, "select: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CACTO_F32)
    return select_entry<float>((const float*)scores, N, keep, base_index, order, (float*)top_scores, workspace, st);
  return select_entry<double>((const double*)scores, N, keep, base_index, order, (double*)top_scores, workspace, st);
}

extern "C" int cacto_select_merge(int32_t dtype, const void* run_scores, const int64_t* run_index, int32_t R,
                                  int64_t keep, int64_t* order, void* top_scores, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  if (R < 1 || keep < 0) return set_error(CACTO_EVALUE, "select_merge: bad sizes");
  if (keep == 0) return CACTO_OK;
  int64_t M = (int64_t)R * keep;
  size_t need = 2 * align256((size_t)M * sizeof(Pair));
  if (workspace_bytes < need) return set_error(CACTO_EVALUE, "select_merge: workspace too small (%zu)", need);
  cudaStream_t st = (cudaStream_t)stream;
  Pair* a = (Pair*)workspace;
  Pair* b = (Pair*)((char*)workspace + align256((size_t)M * sizeof(Pair)));
  int64_t blocks = (M + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (dtype == CACTO_F32)
    runs_to_pairs_kernel<float><<<(unsigned)blocks, 256, 0, st>>>((const float*)run_scores, run_index, M, a);
  else
    runs_to_pairs_kernel<double><<<(unsigned)blocks, 256, 0, st>>>((const double*)run_scores, run_index, M, a);
  Pair* res = sort_pairs(a, b, M, keep, st);
  int64_t eb = (keep + 255) / 256;
  if (dtype == CACTO_F32)
    emit_kernel<float, Pair><<<(unsigned)(eb > 4096 ? 4096 : eb), 256, 0, st>>>(res, keep, 0, order, (float*)top_scores);
  else
    emit_kernel<double, Pair><<<(unsigned)(eb > 4096 ? 4096 : eb), 256, 0, st>>>(res, keep, 0, order, (double*)top_scores);
  return check_launch("select_merge");
}

// ---------------------------------------------------------------------------------
// Distributed stable top-k over contiguous shards (trainer.py:152
// over the union of every rank's candidates).  The host sequences the phases and
// runs the collectives between them (python: parallel.distributed_select):
//   begin                         zero the state
//   for each 8-bit digit (MSB first):
//     pass   -> local 256-bin histogram of the digit among keys matching the prefix
//     [all-reduce SUM of the histogram, 2 KB]
//     digit  -> the digit where the global cumulative count reaches the still-needed
//               k; prefix, k and this rank's count of keys < prefix updated
//   counts -> (lt_local, eq_local) of the final threshold key K*
//   [all-gather of (lt, eq), 16 B per rank]     host: take_r, offset_r (rank order =
//               global index order, so ties at K* go to the lowest ranks first)
//   compact -> every local key <= K* as (key, global index) elements
//   [sort]  -> the rank's winners: the first lt_r + take_r sorted elements, written
//               into its [offset_r, offset_r + c_r) segment of a zeroed keep-row buffer
//               and their LOCAL indices (the rank's own kept rows, for the warm starts)
//   [all-reduce SUM of the keep-row buffer: disjoint segments -> concatenation]
//   finish  -> sort of the keep elements -> global order + scores on every rank
// Only the threshold histograms, the counts and the keep winners cross ranks.
// ---------------------------------------------------------------------------------
namespace cacto {

struct DSelState {
  unsigned long long prefix, mask;
  long long need;       // global count still needed among keys matching the prefix
  long long lt_local;   // this rank's keys < prefix (decided digits)
  long long eq_local;   // this rank's keys == K* (after the last pass)
};

template <typename T>
__global__ void __launch_bounds__(256) dsel_hist_kernel(const T* __restrict__ scores, int64_t N, int shift,
                                                        const DSelState* __restrict__ st, long long* hist) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const unsigned long long prefix = st->prefix, mask = st->mask;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = score_key(scores[i]);
    if ((k & mask) == prefix) atomicAdd(&h[(k >> shift) & 255u], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd((unsigned long long*)&hist[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}

// one CTA of 256 threads: inclusive scan of the global histogram, pick the digit
__global__ void __launch_bounds__(256) dsel_digit_kernel(const long long* __restrict__ hist_local,
                                                         const long long* __restrict__ hist_global, int shift,
                                                         int last, DSelState* st, long long* counts) {
  __shared__ long long sg[256], sl[256];
  const int t = threadIdx.x;
  sg[t] = hist_global[t];
  sl[t] = hist_local[t];
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {  // Hillis-Steele inclusive scans
    long long a = t >= o ? sg[t - o] : 0, b = t >= o ? sl[t - o] : 0;
    __syncthreads();
    sg[t] += a;
    sl[t] += b;
    __syncthreads();
  }
  const long long need = st->need;
  const long long before = t ? sg[t - 1] : 0;
  if (before < need && need <= sg[t]) {  // exactly one digit qualifies
    st->need = need - before;
    st->prefix |= (unsigned long long)t << shift;
    st->mask |= 255ull << shift;
    st->lt_local += t ? sl[t - 1] : 0;
    const long long eq = sl[t] - (t ? sl[t - 1] : 0);
    if (last) {
      st->eq_local = eq;
      counts[0] = st->lt_local;
      counts[1] = eq;
      counts[2] = st->need;  // keys == K* to take, over all ranks
    }
  }
}

template <typename T, typename E>
__global__ void dsel_compact_kernel(const T* __restrict__ scores, int64_t N, int64_t base,
                                    const DSelState* __restrict__ st, E* out, unsigned long long* cursor) {
  const unsigned long long K = st->prefix;
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < N; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    unsigned long long k = ~0ull;
    if (i < N) k = score_key(scores[i]);
    const bool take = i < N && k <= K;
    const unsigned int ball = __ballot_sync(0xffffffffu, take);
    unsigned long long w = 0;
    if (lane == 0 && ball) w = atomicAdd(cursor, (unsigned long long)__popc(ball));
    w = __shfl_sync(0xffffffffu, w, 0);
    if (take) {
      E e;
      make_elem(e, k, base + i);
      out[w + __popc(ball & ((1u << lane) - 1u))] = e;
    }
  }
}

// first c sorted elements -> global segment [off, off + c) and local indices
template <typename E>
__global__ void dsel_emit_local_kernel(const E* __restrict__ sorted, int64_t c, int64_t base, int64_t off,
                                       E* global, int64_t* local_sel) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c; i += (int64_t)gridDim.x * blockDim.x) {
    const E e = sorted[i];
    global[off + i] = e;
    if (local_sel) local_sel[i] = elem_idx(e) - base;
  }
}

static size_t dsel_elem_bytes(int32_t dtype) { return dtype == CACTO_F32 ? sizeof(Packed) : sizeof(Pair); }

}  // namespace cacto

extern "C" size_t cacto_dselect_workspace_bytes(int32_t dtype, int64_t N_local, int64_t keep) {
  const size_t eb = dsel_elem_bytes(dtype);
  const int64_t M = (N_local > keep ? N_local : keep) + 1;
  // state | cursor | 8 x 256 local hist | 2 x M elements (sort ping-pong)
  return align256(sizeof(DSelState)) + align256(sizeof(unsigned long long)) + align256(8 * 256 * sizeof(long long)) +
         2 * align256((size_t)M * eb);
}

struct DselWs {
  DSelState* st;
  unsigned long long* cursor;
  long long* hist;
  char* a;
  char* b;
};

static DselWs dsel_ws(void* ws, int32_t dtype, int64_t N_local, int64_t keep) {
  DselWs w;
  char* p = (char*)ws;
  w.st = (DSelState*)p;
  p += align256(sizeof(DSelState));
  w.cursor = (unsigned long long*)p;
  p += align256(sizeof(unsigned long long));
  w.hist = (long long*)p;
  p += align256(8 * 256 * sizeof(long long));
  const int64_t M = (N_local > keep ? N_local : keep) + 1;
  w.a = p;
  w.b = p + align256((size_t)M * dsel_elem_bytes(dtype));
  return w;
}

extern "C" int cacto_dselect_begin(int32_t dtype, int64_t N_local, int64_t keep, int64_t keep_global, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  if (keep < 0 || keep_global < 0 || N_local < 0 || !workspace)
    return set_error(CACTO_EVALUE, "dselect: bad arguments");
  if (workspace_bytes < cacto_dselect_workspace_bytes(dtype, N_local, keep))
    return set_error(CACTO_EVALUE, "dselect: workspace too small");
  DselWs w = dsel_ws(workspace, dtype, N_local, keep);
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(workspace, 0, (char*)w.a - (char*)workspace, st) != cudaSuccess)
    return set_error(CACTO_ECUDA, "dselect: memset failed");
  DSelState s0{0ull, 0ull, (long long)keep_global, 0ll, 0ll};
  if (cudaMemcpyAsync(w.st, &s0, sizeof(s0), cudaMemcpyHostToDevice, st) != cudaSuccess)
    return set_error(CACTO_ECUDA, "dselect: state upload failed");
  return CACTO_OK;
}

extern "C" int cacto_dselect_pass(int32_t dtype, const void* scores, int64_t N_local, int64_t keep, int32_t pass,
                                  void* workspace, int64_t* hist_out, void* stream) {
  const int KB = dtype == CACTO_F32 ? 32 : 64;
  if (pass < 0 || pass >= KB / 8 || !hist_out) return set_error(CACTO_EVALUE, "dselect: bad pass %d", pass);
  DselWs w = dsel_ws(workspace, dtype, N_local, keep);
  cudaStream_t st = (cudaStream_t)stream;
  long long* h = w.hist + pass * 256;
  if (N_local > 0) {
    int64_t blocks = (N_local + 255) / 256;
    int64_t cap = 4 * (int64_t)num_sms();
    if (blocks > cap) blocks = cap;
    const int shift = KB - 8 * (pass + 1);
    if (dtype == CACTO_F32)
      dsel_hist_kernel<float><<<(unsigned)blocks, 256, 0, st>>>((const float*)scores, N_local, shift, w.st, h);
    else
      dsel_hist_kernel<double><<<(unsigned)blocks, 256, 0, st>>>((const double*)scores, N_local, shift, w.st, h);
  }
  if (cudaMemcpyAsync(hist_out, h, 256 * sizeof(long long), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return set_error(CACTO_ECUDA, "dselect: hist copy failed");
  return check_launch("dsel_hist_kernel");
}

extern "C" int cacto_dselect_digit(int32_t dtype, int64_t N_local, int64_t keep, int32_t pass,
                                   const int64_t* hist_global, void* workspace, int64_t* counts, void* stream) {
  const int KB = dtype == CACTO_F32 ? 32 : 64;
  if (pass < 0 || pass >= KB / 8 || !hist_global || !counts) return set_error(CACTO_EVALUE, "dselect: bad digit");
  DselWs w = dsel_ws(workspace, dtype, N_local, keep);
  dsel_digit_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(w.hist + pass * 256, (const long long*)hist_global,
                                                          KB - 8 * (pass + 1), pass == KB / 8 - 1, w.st,
                                                          (long long*)counts);
  return check_launch("dsel_digit_kernel");
}

template <typename T, typename E>
static int dsel_local(const T* scores, int64_t N, int64_t keep, int64_t base, int64_t n_cand, int64_t c, int64_t off,
                      DselWs w, void* global, int64_t* local_sel, cudaStream_t st) {
  if (n_cand > 0) {
    int64_t blocks = (N + 255) / 256;
    int64_t cap = 4 * (int64_t)num_sms();
    if (blocks > cap) blocks = cap;
    dsel_compact_kernel<T, E><<<(unsigned)blocks, 256, 0, st>>>(scores, N, base, w.st, (E*)w.a, w.cursor);
  }
  E* res = n_cand > 0 ? sort_pairs<E>((E*)w.a, (E*)w.b, n_cand, 0, st) : (E*)w.a;
  if (c > 0) {
    int64_t eb = (c + 255) / 256;
    dsel_emit_local_kernel<E><<<(unsigned)(eb > 4096 ? 4096 : eb), 256, 0, st>>>(res, c, base, off, (E*)global,
                                                                                local_sel);
  }
  return check_launch("dselect_local");
}

extern "C" int cacto_dselect_local(int32_t dtype, const void* scores, int64_t N_local, int64_t keep,
                                   int64_t base_index, int64_t n_candidates, int64_t n_take, int64_t offset,
                                   void* workspace, void* global_elems, int64_t* local_sel, void* stream) {
  if (n_candidates < n_take || n_take < 0 || n_candidates > N_local || n_take > keep)
    return set_error(CACTO_EVALUE, "dselect_local: bad counts");
  if (dtype == CACTO_F32 && base_index + N_local > 0xFFFFFFFFll)
    return set_error(CACTO_EVALUE, "dselect_local: global index exceeds 32 bits");
  DselWs w = dsel_ws(workspace, dtype, N_local, keep);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CACTO_F32)
    return dsel_local<float, Packed>((const float*)scores, N_local, keep, base_index, n_candidates, n_take, offset, w,
                                     global_elems, local_sel, st);
  return dsel_local<double, Pair>((const double*)scores, N_local, keep, base_index, n_candidates, n_take, offset, w,
                                  global_elems, local_sel, st);
}

extern "C" int cacto_dselect_finish(int32_t dtype, void* global_elems, int64_t keep_global, int64_t* order,
                                    void* top_scores, void* scratch, size_t scratch_bytes, void* stream) {
  if (keep_global <= 0) return CACTO_OK;
  const size_t eb = dsel_elem_bytes(dtype);
  if (!global_elems || !order || !scratch || scratch_bytes < (size_t)keep_global * eb)
    return set_error(CACTO_EVALUE, "dselect_finish: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t blocks = (keep_global + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (dtype == CACTO_F32) {
    Packed* res = sort_pairs<Packed>((Packed*)global_elems, (Packed*)scratch, keep_global, 0, st);
    emit_kernel<float, Packed><<<(unsigned)blocks, 256, 0, st>>>(res, keep_global, 0, order, (float*)top_scores);
  } else {
    Pair* res = sort_pairs<Pair>((Pair*)global_elems, (Pair*)scratch, keep_global, 0, st);
    emit_kernel<double, Pair><<<(unsigned)blocks, 256, 0, st>>>(res, keep_global, 0, order, (double*)top_scores);
  }
  return check_launch("dselect_finish");
}
