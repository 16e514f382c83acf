// gemm_tc.cu -- tcgen05 tensor-core GEMM for the wide training layers
// (H = 128..512, north_star: "tensor-core tcgen05 GEMMs only for the wide
// batched layers").
//
//   D[m][n] (+)= sum_k A(m, k) * B(n, k)       fp32 in / fp32 out
//
// A(m,k) = A[m*sam + k*sak], B(n,k) = B[n*sbn + k*sbk]: any of the three GEMMs of a
// dense layer (z = a W^T, s = g W, gW = g^T a) is one call with the right strides.
// fp32 accuracy with TF32 tensor cores: every operand is split x = hi + lo
// (hi = tf32(x), lo = tf32(x - hi)) and D accumulates hi*hi + hi*lo + lo*hi
// ("3xTF32"; relative error ~1e-6, vs ~1e-3 for a single TF32 pass).
//
// CTA = one 128 x BN output tile (UMMA M = 128, cta_group::1, N = BN <= 256).
//   warps 0-3  producers: global fp32 -> split -> canonical K-major SWIZZLE_128B
//              smem tiles (32 fp32 = 128 B per row, chunk ^= row % 8), 2 stages;
//              then the epilogue: tcgen05.ld 32x32b -> registers -> global
//   warp 4     one elected lane issues tcgen05.mma.kind::tf32 (4 K-steps of 8 per
//              128-byte row, x3 products) and commits to the stage's mbarrier
// The accumulator lives in TMEM (128 lanes x BN fp32 columns).
#include "common.cuh"

namespace cacto {

namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per 128-byte row
constexpr int kProducers = 128;
constexpr int kThreadsTC = 160;

CACTO_D void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
CACTO_D void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}
CACTO_D void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}
CACTO_D void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
CACTO_D void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
CACTO_D void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
CACTO_D void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(bar))
               : "memory");
}
CACTO_D uint32_t tf32_round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// SWIZZLE_128B K-major smem descriptor (version 1 = Blackwell): start address,
// SBO = 1024 B between 8-row groups, LBO unused for swizzled K-major.
CACTO_D uint64_t make_desc(uint32_t saddr_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr_bytes >> 4) & 0x3FFF);
  d |= (uint64_t)(1) << 16;                 // LBO (ignored)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;  // SBO
  d |= (uint64_t)1 << 46;                   // version
  d |= (uint64_t)2 << 61;                   // SWIZZLE_128B
  return d;
}

// instruction descriptor: D f32, A/B tf32, K-major both, M = 128, N = BN
template <int BN>
constexpr uint32_t idesc_tf32() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

CACTO_D void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}

// byte offset of element (row, k) of a [rows][32] fp32 tile in the SW128 layout
CACTO_D uint32_t sw128(int row, int k) {
  return (uint32_t)(row * 128 + ((((k >> 2) ^ (row & 7))) << 4) + ((k & 3) << 2));
}

struct GemmArgs {
  int M, N, K;
  const float* A;
  int64_t sam, sak;
  const float* B;
  int64_t sbn, sbk;
  float* D;
  int64_t ldd;
  int accumulate;  // D += product (else D = product)
  float alpha;
};

// producers: fill stage buffers for k-block kb (hi and lo parts of A and B tiles)
template <int BN>
CACTO_D void produce(const GemmArgs& g, int m0, int n0, int kb, unsigned char* sA_hi, unsigned char* sA_lo,
                     unsigned char* sB_hi, unsigned char* sB_lo) {
  const int t = threadIdx.x;  // 0..127
  const int k0 = kb * BK;
  // A tile [BM][BK]
  if (g.sak == 1) {
    for (int e = t * 4; e < BM * BK; e += kProducers * 4) {
      const int r = e / BK, c = e % BK;
      const int m = m0 + r, k = k0 + c;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m < g.M) {
        const float* p = g.A + (int64_t)m * g.sam + k;
        if (k + 3 < g.K && (((uintptr_t)p) & 15) == 0) {
          v = *reinterpret_cast<const float4*>(p);
        } else {
          v.x = k < g.K ? p[0] : 0.f;
          v.y = k + 1 < g.K ? p[1] : 0.f;
          v.z = k + 2 < g.K ? p[2] : 0.f;
          v.w = k + 3 < g.K ? p[3] : 0.f;
        }
      }
      const float x[4] = {v.x, v.y, v.z, v.w};
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        hi[q] = tf32_round(x[q]);
        lo[q] = tf32_round(x[q] - __uint_as_float(hi[q]));
      }
      const uint32_t off = sw128(r, c);
      *reinterpret_cast<uint4*>(sA_hi + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(sA_lo + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
  } else {  // M-contiguous: lanes walk m (coalesced), each thread one row, 32 k values
    for (int r = t; r < BM; r += kProducers) {
      const int m = m0 + r;
      for (int c = 0; c < BK; c += 4) {
        float x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = k0 + c + q;
          x[q] = (m < g.M && k < g.K) ? g.A[(int64_t)m * g.sam + (int64_t)k * g.sak] : 0.f;
        }
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          hi[q] = tf32_round(x[q]);
          lo[q] = tf32_round(x[q] - __uint_as_float(hi[q]));
        }
        const uint32_t off = sw128(r, c);
        *reinterpret_cast<uint4*>(sA_hi + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(sA_lo + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
    }
  }
  // B tile [BN][BK]
  if (g.sbk == 1) {
    for (int e = t * 4; e < BN * BK; e += kProducers * 4) {
      const int r = e / BK, c = e % BK;
      const int n = n0 + r, k = k0 + c;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (n < g.N) {
        const float* p = g.B + (int64_t)n * g.sbn + k;
        if (k + 3 < g.K && (((uintptr_t)p) & 15) == 0) {
          v = *reinterpret_cast<const float4*>(p);
        } else {
          v.x = k < g.K ? p[0] : 0.f;
          v.y = k + 1 < g.K ? p[1] : 0.f;
          v.z = k + 2 < g.K ? p[2] : 0.f;
          v.w = k + 3 < g.K ? p[3] : 0.f;
        }
      }
      const float x[4] = {v.x, v.y, v.z, v.w};
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        hi[q] = tf32_round(x[q]);
        lo[q] = tf32_round(x[q] - __uint_as_float(hi[q]));
      }
      const uint32_t off = sw128(r, c);
      *reinterpret_cast<uint4*>(sB_hi + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(sB_lo + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
  } else {
    for (int r = t; r < BN; r += kProducers) {
      const int n = n0 + r;
      for (int c = 0; c < BK; c += 4) {
        float x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = k0 + c + q;
          x[q] = (n < g.N && k < g.K) ? g.B[(int64_t)n * g.sbn + (int64_t)k * g.sbk] : 0.f;
        }
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          hi[q] = tf32_round(x[q]);
          lo[q] = tf32_round(x[q] - __uint_as_float(hi[q]));
        }
        const uint32_t off = sw128(r, c);
        *reinterpret_cast<uint4*>(sB_hi + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(sB_lo + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
    }
  }
}

template <int BN, int PASSES>
__global__ void __launch_bounds__(kThreadsTC, 1) gemm_tf32_kernel(const GemmArgs g) {
  constexpr int STAGES = 2;
  constexpr uint32_t A_BYTES = BM * BK * 4, B_BYTES = BN * BK * 4;
  constexpr uint32_t STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  constexpr uint32_t TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  // 1024-byte alignment of the swizzle atoms
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], done_bar;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int nkb = (g.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], kProducers);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
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
  const uint32_t tmem_d = tmem_base_sh;

  if (warp < 4) {
    // ---- producers -----------------------------------------------------------
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(&empty_bar[s], ph ^ 1);
      unsigned char* st = base + s * STAGE_BYTES;
      produce<BN>(g, m0, n0, kb, st, st + A_BYTES, st + 2 * A_BYTES, st + 2 * A_BYTES + B_BYTES);
      fence_async_smem();
      mbar_arrive(&full_bar[s]);
    }
    // ---- epilogue: TMEM -> registers -> global -----------------------------------
    mbar_wait(&done_bar, 0);
    tc_fence_after();
    const int row = m0 + warp * 32 + lane;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t v[16];
      const uint32_t taddr = tmem_d + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
          "%14, %15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < g.M) {
        float* d = g.D + (int64_t)row * g.ldd + n0 + c0;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          if (n0 + c0 + q < g.N) {
            float val = g.alpha * __uint_as_float(v[q]);
            d[q] = g.accumulate ? d[q] + val : val;
          }
        }
      }
    }
  } else if (warp == 4) {
    // ---- MMA issuer (one lane) --------------------------------------------------
    constexpr uint32_t idesc = idesc_tf32<BN>();
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(&full_bar[s], ph);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t st = saddr(base + s * STAGE_BYTES);
        const uint32_t a_hi = st, a_lo = st + A_BYTES, b_hi = st + 2 * A_BYTES, b_lo = b_hi + B_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {  // UMMA_K = 8 tf32 = 32 bytes
          const uint32_t ko = kk * 32;
          const uint32_t acc0 = (kb > 0 || kk > 0) ? 1u : 0u;
          mma_tf32(tmem_d, make_desc(a_hi + ko), make_desc(b_hi + ko), idesc, acc0);
          if (PASSES == 3) {
            mma_tf32(tmem_d, make_desc(a_hi + ko), make_desc(b_lo + ko), idesc, 1u);
            mma_tf32(tmem_d, make_desc(a_lo + ko), make_desc(b_hi + ko), idesc, 1u);
          }
        }
        tc_commit(&empty_bar[s]);
        if (kb == nkb - 1) tc_commit(&done_bar);
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(TMEM_COLS) : "memory");
  }
}

template <int BN, int PASSES>
static int launch_gemm(const GemmArgs& g, cudaStream_t st) {
  constexpr uint32_t STAGE_BYTES = 2 * BM * BK * 4 + 2 * BN * BK * 4;
  const size_t smem = 2 * STAGE_BYTES + 1024;
  auto kern = gemm_tf32_kernel<BN, PASSES>;
  if (!ensure_smem((const void*)kern, smem)) return set_error(CACTO_ECUDA, "gemm: %zu B smem unavailable", smem);
  dim3 grid((g.M + BM - 1) / BM, (g.N + BN - 1) / BN);
  kern<<<grid, kThreadsTC, smem, st>>>(g);
  return check_launch("gemm_tf32_kernel");
}

}  // namespace tc

int gemm_tf32(const tc::GemmArgs& g, int passes, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return CACTO_OK;
  // N tile: 128 (TMEM 128 columns) unless the problem is narrow
  if (passes == 3) {
    if (g.N <= 64) return tc::launch_gemm<64, 3>(g, st);
    return tc::launch_gemm<128, 3>(g, st);
  }
  if (g.N <= 64) return tc::launch_gemm<64, 1>(g, st);
  return tc::launch_gemm<128, 1>(g, st);
}

}  // namespace cacto

using namespace cacto;

extern "C" int cacto_gemm_tf32(int32_t M, int32_t N, int32_t K, const float* A, int64_t sam, int64_t sak,
                               const float* B, int64_t sbn, int64_t sbk, float* D, int64_t ldd, int32_t accumulate,
                               float alpha, int32_t passes, void* stream) {
  if (!A || !B || !D || M < 0 || N < 0 || K < 0) return set_error(CACTO_EVALUE, "gemm: bad arguments");
  if (passes != 1 && passes != 3) return set_error(CACTO_EVALUE, "gemm: passes must be 1 or 3");
  tc::GemmArgs g{M, N, K, A, sam, sak, B, sbn, sbk, D, ldd, accumulate, alpha};
  return gemm_tf32(g, passes, (cudaStream_t)stream);
}
