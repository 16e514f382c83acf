// gemm_tc.cu -- tcgen05 tensor-core GEMM for the wide training layers
// (H = 128..512, north_star: "tensor-core tcgen05 GEMMs only for the wide
// batched layers").
//
//   D[m][n] (+)= alpha * sum_k A(m, k) * B(n, k)       fp32 in / fp32 out
//
// A(m,k) = A[m*sam + k*sak], B(n,k) = B[n*sbn + k*sbk]; each operand is either
// K-major (sak == 1) or MN-major (sam == 1), so the three GEMMs of a dense layer
// (z = a W^T, s = g W, gW = g^T a) are plain calls with no transposes.
//
// fp32 accuracy from TF32 tensor cores ("3xTF32"): the tensor core reads a raw
// fp32 operand as its TF32 truncation hi = trunc(x); split warps compute
// lo = x - hi in shared memory and the MMA issues hi*hi + hi*lo + lo*hi.
//
// Persistent pipeline (one CTA per SM walks the 128 x BN output tiles, n fastest;
// 3 shared-memory stages form one ring across all of a CTA's tiles):
//   warp 0      TMA producer: cp.async.bulk.tensor 2D loads straight into the
//               canonical UMMA layouts (K-major: 128B swizzle; MN-major: 128B
//               swizzle with 32-byte atoms, the tf32 MN-major layout), one
//               mbarrier per stage
//   warp 1      one lane issues tcgen05.mma.cta_group::1.kind::tf32 (M = 128,
//               N = BN, K = 8 per instruction), commits each stage to its "empty"
//               mbarrier and each finished tile to acc_full[buf]
//   warps 2-5   split workers (lo tiles, layout-agnostic smem->smem)
//   warps 6-9   epilogue: tcgen05.ld 32x32b -> registers -> global, from the
//               other half of a double-buffered TMEM accumulator (2 x BN columns),
//               so a tile's epilogue overlaps the next tile's MMAs
// Split-K (tile index carries the split) writes per-split partials (deterministic reduce after).
#include <cuda.h>

#include <algorithm>

#include "tc.cuh"

namespace cacto {

namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per 128-byte swizzle row
constexpr int kThreadsTC = 320;  // TMA, MMA, 4 split warps, 4 epilogue warps

struct GemmArgs {
  int M, N, K;
  int a_kmajor, b_kmajor;
  int passes;
  float* D;
  int64_t ldd;
  int accumulate;
  float alpha;
  int kb_per_split;
  int mtiles, ntiles, splits;
  int64_t split_stride;  // elements between per-split partial outputs (0: no split)
};

// descriptors of the k-step `kk` (8 tf32) of an operand tile
//  K-major : SW128 atoms of 8 rows x 128 B; a k-step is 32 B inside the row
//  MN-major: SW128_BASE32B atoms of 4 k-rows x 128 B (32 MN elements, SBO = 512 B),
//            MN blocks of 32 at LBO = 4 KB (one TMA box each); a k-step = 8 rows
CACTO_D uint64_t op_desc(uint32_t tile, int kmajor, int kk) {
  if (kmajor) return make_desc(tile + kk * 32, 16, 1024, 2);
  return make_desc(tile + kk * 1024, 4096, 512, 1);
}

template <int BN, int kStages>
__global__ void __launch_bounds__(kThreadsTC, 1)
    gemm_tf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const GemmArgs g) {
  constexpr uint32_t A_BYTES = BM * BK * 4, B_BYTES = BN * BK * 4;
  constexpr uint32_t STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // raw A, raw B, lo A, lo B
  constexpr uint32_t ACC_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  constexpr uint32_t TMEM_COLS = 2 * ACC_COLS;  // double-buffered accumulator
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t tma_bar[kStages], split_bar[kStages], empty_bar[kStages];
  __shared__ __align__(8) uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb_all = (g.K + BK - 1) / BK;
  const bool three = g.passes == 3;
  const int ntiles = g.mtiles * g.ntiles * g.splits;
  // tile t -> (split, m tile, n tile), n fastest: the n tiles of one A row strip
  // run on neighbouring CTAs at the same time, so A is read from HBM once
  auto tile_of = [&](int t, int& m0, int& n0, int& kb0, int& nkb) {
    const int nt = t % g.ntiles;
    const int r = t / g.ntiles;
    const int mt = r % g.mtiles;
    const int z = r / g.mtiles;
    m0 = mt * BM;
    n0 = nt * BN;
    kb0 = z * g.kb_per_split;
    nkb = max(0, min(nkb_all, kb0 + g.kb_per_split) - kb0);
    return z;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&tma_bar[s], 1);
      mbar_init(&split_bar[s], 128);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_base_sh)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  if (warp == 0) {
    // ---- TMA producer: one stage ring across all of this CTA's tiles -------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int m0, n0, kb0, nkb;
        tile_of(t, m0, n0, kb0, nkb);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          mbar_wait(&empty_bar[s], ph ^ 1);
          unsigned char* st = base + s * STAGE_BYTES;
          const int k0 = (kb0 + i) * BK;
          mbar_expect_tx(&tma_bar[s], A_BYTES + B_BYTES);
          if (g.a_kmajor) {
            tma_load_2d(st, &tmA, &tma_bar[s], k0, m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 32; ++j) tma_load_2d(st + j * 4096, &tmA, &tma_bar[s], m0 + 32 * j, k0);
          }
          if (g.b_kmajor) {
            tma_load_2d(st + A_BYTES, &tmB, &tma_bar[s], k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 32; ++j)
              tma_load_2d(st + A_BYTES + j * 4096, &tmB, &tma_bar[s], n0 + 32 * j, k0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: accumulator buffer (local tile & 1) ------------------------------
    const uint32_t idesc = idesc_tf32(BN, !g.a_kmajor, !g.b_kmajor);
    int it = 0, lt = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      int m0, n0, kb0, nkb;
      tile_of(t, m0, n0, kb0, nkb);
      if (nkb == 0) continue;
      const int buf = lt & 1;
      const uint32_t tmem_d = tmem_base + buf * ACC_COLS;
      mbar_wait(&acc_empty[buf], ((lt >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % kStages;
        const uint32_t ph = (it / kStages) & 1;
        mbar_wait(three ? &split_bar[s] : &tma_bar[s], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t st = saddr(base + s * STAGE_BYTES);
          const uint32_t a_raw = st, b_raw = st + A_BYTES, a_lo = st + A_BYTES + B_BYTES, b_lo = a_lo + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint32_t acc0 = (i > 0 || kk > 0) ? 1u : 0u;
            mma_tf32(tmem_d, op_desc(a_raw, g.a_kmajor, kk), op_desc(b_raw, g.b_kmajor, kk), idesc, acc0);
            if (three) {
              mma_tf32(tmem_d, op_desc(a_raw, g.a_kmajor, kk), op_desc(b_lo, g.b_kmajor, kk), idesc, 1u);
              mma_tf32(tmem_d, op_desc(a_lo, g.a_kmajor, kk), op_desc(b_raw, g.b_kmajor, kk), idesc, 1u);
            }
          }
          tc_commit(&empty_bar[s]);
          if (i == nkb - 1) tc_commit(&acc_full[buf]);
        }
        __syncwarp();
      }
    }
  } else if (warp <= 5) {
    // ---- split workers: lo = x - trunc_tf32(x) (layout-agnostic) -----------------
    const int t0 = threadIdx.x - 64;  // 0..127
    if (three) {
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int m0, n0, kb0, nkb;
        tile_of(t, m0, n0, kb0, nkb);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          mbar_wait(&tma_bar[s], ph);
          unsigned char* st = base + s * STAGE_BYTES;
          const float4* src = reinterpret_cast<const float4*>(st);
          float4* dst = reinterpret_cast<float4*>(st + A_BYTES + B_BYTES);
          constexpr int NV = (A_BYTES + B_BYTES) / 16;
#pragma unroll 4
          for (int q = t0; q < NV; q += 128) {
            float4 x = src[q];
            float4 lo;
            lo.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
            lo.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
            lo.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
            lo.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
            dst[q] = lo;
          }
          fence_async_smem();
          mbar_arrive(&split_bar[s]);
        }
      }
    }
  } else {
    // ---- epilogue warps 6..9: TMEM -> registers -> global, overlapping the next tile's MMAs
    const int lane_grp = warp & 3;  // tcgen05.ld lane quarter of this warp
    int lt = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      int m0, n0, kb0, nkb;
      const int z = tile_of(t, m0, n0, kb0, nkb);
      const int buf = lt & 1;
      const uint32_t tmem_d = tmem_base + buf * ACC_COLS;
      const int row = m0 + lane_grp * 32 + lane;
      float* dbase = g.D + (int64_t)z * g.split_stride;
      if (nkb > 0) {
        mbar_wait(&acc_full[buf], (lt >> 1) & 1);
        tc_fence_after();
      }
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t v[16];
        if (nkb > 0) {
          const uint32_t taddr = tmem_d + ((uint32_t)(lane_grp * 32) << 16) + (uint32_t)c0;
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
              "%13, %14, %15}, [%16];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                "=r"(v[15])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] = 0u;
        }
        if (c0 + 16 >= BN && nkb > 0) {
          // whole accumulator is in registers: hand the buffer back to the MMA warp
          tc_fence_before();
          mbar_arrive(&acc_empty[buf]);
        }
        if (row < g.M) {
          float* d = dbase + (int64_t)row * g.ldd + n0 + c0;
          if (n0 + c0 + 16 <= g.N && !g.accumulate && ((((uintptr_t)d) & 15) == 0)) {
#pragma unroll
            for (int q = 0; q < 16; q += 4)
              *reinterpret_cast<float4*>(d + q) =
                  make_float4(g.alpha * __uint_as_float(v[q]), g.alpha * __uint_as_float(v[q + 1]),
                              g.alpha * __uint_as_float(v[q + 2]), g.alpha * __uint_as_float(v[q + 3]));
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              if (n0 + c0 + q < g.N) {
                float val = g.alpha * __uint_as_float(v[q]);
                d[q] = g.accumulate ? d[q] + val : val;
              }
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
}

// ---- host: tensor maps ------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// operand with element (r, k) at X[r*sr + k*sk], rows x K; box_rows for K-major
static int make_map(CUtensorMap* map, const float* X, int rows, int K, int64_t sr, int64_t sk, int box_rows,
                    int* kmajor) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return set_error(CACTO_ECUDA, "gemm: cuTensorMapEncodeTiled unavailable");
  if (((uintptr_t)X) & 15) return set_error(CACTO_EVALUE, "gemm: operand not 16-byte aligned");
  cuuint64_t dims[2], strides[1];
  cuuint32_t box[2], estr[2] = {1, 1};
  if (sk == 1) {
    *kmajor = 1;
    dims[0] = (cuuint64_t)K;
    dims[1] = (cuuint64_t)rows;
    strides[0] = (cuuint64_t)sr * 4;
    box[0] = BK;
    box[1] = (cuuint32_t)box_rows;
  } else if (sr == 1) {
    *kmajor = 0;
    dims[0] = (cuuint64_t)rows;
    dims[1] = (cuuint64_t)K;
    strides[0] = (cuuint64_t)sk * 4;
    box[0] = 32;
    box[1] = BK;
  } else {
    return set_error(CACTO_EVALUE, "gemm: operands must be K-major or MN-major");
  }
  if (strides[0] % 16) return set_error(CACTO_EVALUE, "gemm: operand row stride must be a multiple of 16 bytes");
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)X, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   *kmajor ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(CACTO_ECUDA, "gemm: tensor map encode failed (%d)", (int)r);
  return CACTO_OK;
}

// shared-memory stages: 3 at BN <= 128 (64 KB each), 2 at BN = 256 (96 KB each)
// narrow tiles (BN <= 64) run two CTAs per SM with two stages each (2 x 97 KB
// smem, 2 x 128 TMEM columns): two independent TMA -> split -> MMA chains per SM.
// (BN = 96 does not fit twice: 2 x (113 KB + 1 KB reserved) > 228 KB)
inline bool pair_ctas(int bn) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("CACTO_GEMM_PAIR");
    env = e ? atoi(e) : 1;
  }
  return env != 0 && bn <= 64;
}
inline int cta_slots(int bn) { return (pair_ctas(bn) ? 2 : 1) * num_sms(); }

template <int BN, int kStages>
static int launch_gemm_k(const CUtensorMap& ma, const CUtensorMap& mb, GemmArgs g, int splits, int slots,
                         cudaStream_t st) {
  constexpr uint32_t STAGE_BYTES = 2 * BM * BK * 4 + 2 * BN * BK * 4;
  const size_t smem = kStages * STAGE_BYTES + 1024;
  auto kern = gemm_tf32_kernel<BN, kStages>;
  if (!ensure_smem((const void*)kern, smem)) return set_error(CACTO_ECUDA, "gemm: %zu B smem unavailable", smem);
  g.mtiles = (g.M + BM - 1) / BM;
  g.ntiles = (g.N + BN - 1) / BN;
  g.splits = splits;
  // persistent: one CTA per slot walks the tiles (double-buffered TMEM accumulator)
  const int64_t tiles = (int64_t)g.mtiles * g.ntiles * splits;
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, slots);
  kern<<<grid, kThreadsTC, smem, st>>>(ma, mb, g);
  return check_launch("gemm_tf32_kernel");
}
template <int BN>
static int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, GemmArgs g, int splits, cudaStream_t st) {
  if constexpr (BN <= 64) {
    if (pair_ctas(BN)) return launch_gemm_k<BN, 2>(ma, mb, g, splits, cta_slots(BN), st);
  }
  return launch_gemm_k<BN, BN >= 256 ? 2 : 3>(ma, mb, g, splits, num_sms(), st);
}

__global__ void splitk_reduce_kernel(const float* __restrict__ part, int splits, int64_t split_stride, int M, int N,
                                     int64_t ldp, float* D, int64_t ldd, int accumulate) {
  const int64_t total = (int64_t)M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / N, n = e - m * N;
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += part[z * split_stride + m * ldp + n];
    float* d = D + m * ldd + n;
    *d = accumulate ? *d + s : s;
  }
}

// many splits (small output, long K): one warp per output element, lanes over
// the splits, a fixed shuffle tree -- deterministic
__global__ void splitk_reduce_warp_kernel(const float* __restrict__ part, int splits, int64_t split_stride, int M,
                                          int N, float* D, int64_t ldd, int accumulate) {
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)M * N;
  for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < total;
       e += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    float s = 0.f;
    for (int z = lane; z < splits; z += 32) s += part[z * split_stride + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const int64_t m = e / N, n = e - m * N;
      float* d = D + m * ldd + n;
      *d = accumulate ? *d + s : s;
    }
  }
}

}  // namespace tc

// output tile width for an N-column GEMM
// (256 only for N >= 512: at N = 256 the halved tile count quantises badly on 148 SMs)
// (96 for 65..96 columns, e.g. the critic's 65-column [W|b] reductions: 25 % fewer MMA columns than 128)
static int tile_bn(int N) {
  return N <= 64 ? 64 : (N <= 96 ? 96 : (N >= 512 && N % 256 == 0 ? 256 : 128));
}

// split-K when the tile grid cannot fill the GPU and K is long (weight gradients):
// as many splits as fill the SMs (not only powers of two), >= 8 k-blocks each,
// never an empty split
static int choose_splits(int tiles, int nkb, int slots) {
  if (tiles * 2 > slots) return 1;
  int splits = std::max(1, std::min(slots / tiles, nkb / 8));
  if (splits > 1) {
    const int per = (nkb + splits - 1) / splits;
    splits = (nkb + per - 1) / per;
  }
  return splits;
}

// workspace bytes a gemm of this shape may need for split-K partials
size_t gemm_workspace_bytes(int M, int N, int K) {
  const int bn = tile_bn(N);
  const int tiles = ((M + tc::BM - 1) / tc::BM) * ((N + bn - 1) / bn);
  const int nkb = (K + tc::BK - 1) / tc::BK;
  const int splits = choose_splits(tiles, nkb, tc::cta_slots(bn));
  return splits > 1 ? (size_t)splits * M * N * 4 : 0;
}

// partials_only: always write the per-split partial products [splits][M][N] into
// ws (splits reported in *splits_out) and skip the split-K reduction -- for callers
// that fuse the reduction into their own consumer (critic_tc's gradient scatter)
static int gemm_tf32_impl(int M, int N, int K, const float* A, int64_t sam, int64_t sak, const float* B, int64_t sbn,
                          int64_t sbk, float* D, int64_t ldd, int accumulate, float alpha, int passes, void* ws,
                          size_t ws_bytes, cudaStream_t st, bool partials_only, int* splits_out) {
  if (M <= 0 || N <= 0) return CACTO_OK;
  const int bn = tile_bn(N);
  CUtensorMap ma, mb;
  tc::GemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.passes = passes;
  int rc = tc::make_map(&ma, A, M, K, sam, sak, tc::BM, &g.a_kmajor);
  if (rc) return rc;
  rc = tc::make_map(&mb, B, N, K, sbn, sbk, bn, &g.b_kmajor);
  if (rc) return rc;
  // split-K when the tile grid cannot fill the GPU and K is long (weight gradients)
  const int tiles = ((M + tc::BM - 1) / tc::BM) * ((N + bn - 1) / bn);
  const int nkb = (K + tc::BK - 1) / tc::BK;
  int splits = choose_splits(tiles, nkb, tc::cta_slots(bn));
  if (splits > 1 && (!ws || ws_bytes < (size_t)splits * M * N * 4)) splits = 1;
  if (partials_only && (!ws || ws_bytes < (size_t)M * N * 4))
    return set_error(CACTO_EVALUE, "gemm: partials workspace too small");
  g.kb_per_split = (nkb + splits - 1) / splits;
  if (g.kb_per_split > 0) splits = (nkb + g.kb_per_split - 1) / g.kb_per_split;  // no empty split
  g.alpha = alpha;
  if (splits_out) *splits_out = splits;
  if (splits > 1 || partials_only) {
    g.D = (float*)ws;
    g.ldd = N;
    g.accumulate = 0;
    g.split_stride = (int64_t)M * N;
  } else {
    g.D = D;
    g.ldd = ldd;
    g.accumulate = accumulate;
    g.split_stride = 0;
  }
  rc = bn == 64    ? tc::launch_gemm<64>(ma, mb, g, splits, st)
       : bn == 96  ? tc::launch_gemm<96>(ma, mb, g, splits, st)
       : bn == 128 ? tc::launch_gemm<128>(ma, mb, g, splits, st)
                   : tc::launch_gemm<256>(ma, mb, g, splits, st);
  if (rc || splits == 1 || partials_only) return rc;
  int64_t total = (int64_t)M * N;
  unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 8 * num_sms());
  if (splits >= 16 && total < 65536) {  // few outputs: lanes over splits; else coalesced per element
    const int64_t warps = total;
    unsigned g2 = (unsigned)std::min<int64_t>((warps * 32 + 255) / 256, 16 * num_sms());
    tc::splitk_reduce_warp_kernel<<<g2, 256, 0, st>>>((const float*)ws, splits, (int64_t)M * N, M, N, D, ldd,
                                                      accumulate);
    return check_launch("splitk_reduce_warp_kernel");
  }
  tc::splitk_reduce_kernel<<<grid, 256, 0, st>>>((const float*)ws, splits, (int64_t)M * N, M, N, N, D, ldd, accumulate);
  return check_launch("splitk_reduce_kernel");
}

int gemm_tf32(int M, int N, int K, const float* A, int64_t sam, int64_t sak, const float* B, int64_t sbn, int64_t sbk,
              float* D, int64_t ldd, int accumulate, float alpha, int passes, void* ws, size_t ws_bytes,
              cudaStream_t st) {
  return gemm_tf32_impl(M, N, K, A, sam, sak, B, sbn, sbk, D, ldd, accumulate, alpha, passes, ws, ws_bytes, st,
                        false, nullptr);
}

int gemm_tf32_partials(int M, int N, int K, const float* A, int64_t sam, int64_t sak, const float* B, int64_t sbn,
                       int64_t sbk, float alpha, int passes, void* ws, size_t ws_bytes, int* splits_out,
                       cudaStream_t st) {
  return gemm_tf32_impl(M, N, K, A, sam, sak, B, sbn, sbk, nullptr, 0, 0, alpha, passes, ws, ws_bytes, st, true,
                        splits_out);
}


}  // namespace cacto

using namespace cacto;

extern "C" size_t cacto_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K) { return gemm_workspace_bytes(M, N, K); }

extern "C" int cacto_gemm_tf32(int32_t M, int32_t N, int32_t K, const float* A, int64_t sam, int64_t sak,
                               const float* B, int64_t sbn, int64_t sbk, float* D, int64_t ldd, int32_t accumulate,
                               float alpha, int32_t passes, void* workspace, size_t workspace_bytes, void* stream) {
  if (!A || !B || !D || M < 0 || N < 0 || K < 0) return set_error(CACTO_EVALUE, "gemm: bad arguments");
  if (passes != 1 && passes != 3) return set_error(CACTO_EVALUE, "gemm: passes must be 1 or 3");
  return gemm_tf32(M, N, K, A, sam, sak, B, sbn, sbk, D, ldd, accumulate, alpha, passes, workspace, workspace_bytes,
                   (cudaStream_t)stream);
}
