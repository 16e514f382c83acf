// critic_tc.cu -- the Sobolev critic loss (nets.critic_loss, nets.py:233-290) on
// the tensor cores for the 3 x 64 networks of the reference configs, fp32
// accurate through the 3xFP16 split of tcmlp.cuh.
//
// Two stages:
//  1. critic_tc_kernel -- per 128-sample tile (TMEM lane = sample), every
//     per-sample matrix product is a tcgen05 layer with A in TMEM: the target
//     forward at x_{+k} (4 layers), the critic forward at x (4, z_i kept in
//     TMEM), the input-gradient sweep s_i = g_i W_i (3, transposed weights), the
//     gradient-path r_i = W_i u_i (3) and the value-path abar_i = zbar_i W_i (2).
//     The epilogue warps (4 per TMEM lane quadrant, 16 columns each) apply the
//     activation / its derivatives (nets.py:27-52), form e_v, e_g, the loss and
//     the cotangents (nets.py:247-289), and stream the per-sample factors of the
//     weight gradients to HBM: [g_i ; zbar_i] and [u_i ; a_i] as 2B-row matrices.
//  2. the batch reductions -- gW_i = [g_i ; zbar_i]^T [u_i ; a_i] as one tcgen05
//     GEMM per layer over K = 2B (gemm_tc.cu, MN-major operands), bias and
//     output-row gradients (a matrix-vector product: out_row_grad_kernel on the
//     CUDA cores) as deterministic column sums.  One gradient slot
//     (n_partials = 1), so the fold / Adam kernels apply unchanged.
// TMEM (512 columns, one tile per CTA): D [64] | A_hi [32] | A_lo [32] |
// z_0..z_2 [3 x 64] | g_i -> zeta_i [3 x 64].
#include <algorithm>

#include "tcmlp.cuh"

namespace cacto {

int gemm_tf32(int M, int N, int K, const float* A, int64_t sam, int64_t sak, const float* B, int64_t sbn, int64_t sbk,
              float* D, int64_t ldd, int accumulate, float alpha, int passes, void* ws, size_t ws_bytes,
              cudaStream_t st);
size_t gemm_workspace_bytes(int M, int N, int K);
int gemm_tf32_partials(int M, int N, int K, const float* A, int64_t sam, int64_t sak, const float* B, int64_t sbn,
                       int64_t sbk, float alpha, int passes, void* ws, size_t ws_bytes, int* splits_out,
                       cudaStream_t st);

#if CACTO_CTC_TIMELINE
// clock64 timeline of CTA 10's second tile (profiles/critic_timeline.py):
// [critic-chain layer 0..11][0: MMA warp saw the hand-off, 1: MMAs + commit issued,
// 2: epilogue warp 0 saw the completion, 3: epilogue warp 0 handed the next layer off]
__device__ unsigned long long g_ctc_tl[12][4];
#define CTC_TL(I, E, T)                                                                 \
  do {                                                                                  \
    if (blockIdx.x == 10 && (T) == blockIdx.x + gridDim.x && lane == 0 && (I) < 12)     \
      g_ctc_tl[I][E] = clock64();                                                       \
  } while (0)
#else
#define CTC_TL(I, E, T) \
  do {                  \
  } while (0)
#endif

#ifndef CACTO_CTC_V8
#define CACTO_CTC_V8 1
#endif

#ifndef CACTO_CTC_SCATTER_COALESCED
#define CACTO_CTC_SCATTER_COALESCED 1
#endif

namespace ctc {

constexpr int HP = 64;
constexpr int TILE = 128;
constexpr int NEPI = 16;  // epilogue warps: 4 per lane quadrant x 16 columns
constexpr int MMA_WARP = NEPI;
constexpr int NTHR = NEPI * 32 + 32;
constexpr uint32_t TD = 0, TA_HI = 64, TA_LO = 96, TZ = 128, TG = 320;
// the target forward runs before any g_i exists: its D and A live in the G region
constexpr uint32_t TT_D = TG, TT_AHI = TG + 64, TT_ALO = TG + 96;
using PL = rtc::Plan<HP>;
constexpr uint32_t SLOT = PL::SLOT;             // 0 = critic, 1 = target (forward weights)
constexpr uint32_t W0T = rtc::NOUT * 128;       // W0^T [16][64] (N = padded input width)
constexpr uint32_t WHT = HP * 128;              // W_i^T [64][64]
constexpr uint32_t OFF_W0T = 2 * SLOT;          // hi, lo
constexpr uint32_t OFF_W1T = OFF_W0T + 2 * W0T;
constexpr uint32_t OFF_W2T = OFF_W1T + 2 * WHT;
constexpr uint32_t OFF_W3 = OFF_W2T + 2 * WHT;  // fp32 output row w_3 [64], unscaled
constexpr uint32_t IMG_BYTES = OFF_W3 + HP * 4;  // the staged weights (a multiple of 16 B)
constexpr uint32_t BYTES = IMG_BYTES + 1024;

struct CBatch {
  const int64_t* idx;
  const int64_t* cycle;
  int64_t idx_stride;
  const float *xa, *v_bar, *v_bar_x, *xa_plus_k;
  int64_t rows;
  int n, t_max;
  CACTO_D int64_t row(int64_t b) const {
    if (!idx) return b;
    return cycle ? idx[(*cycle) * idx_stride + b] : idx[b];
  }
};

struct Args {
  CBatch b;
  const float* critic;
  const float* target;  // null: no bootstrap
  NetConst<float> nc, nc_t;
  int ip;               // padded input width of W0 (8 or 16)
  float k_s, inv_denom;
  // per-sample factors of the weight gradients (rows = b.rows = B)
  float* GZ[3];  // [2B][64]: g_i rows, then zbar_i rows
  // [2B][W_i + 4]: u_i rows then a_i rows, plus a bias column (0 on u rows, 1 on
  // a rows) so one GEMM yields gW_i and gb_i; W_0 = 16, W_1 = W_2 = W_3 = 64
  float* UA[4];  // UA[3]: u_3 rows then a_3 rows (the output row w_3)
  float* V3;     // [2B]: 1 on u_3 rows, -2 e_v on a_3 rows (left factor of gW_3, gb_3)
  float* lossp;  // [gridDim.x]
  const unsigned char* img;  // pre-staged shared-memory image of the weights (or null)
};

// transposed copy: element (r = c, k = o) = W[o][c] * scale, K-major SW128 fp16
CACTO_D void stage_wt(unsigned char* hi, unsigned char* lo, const float* W, int out, int in, int stride, float scale,
                      int rrows, int tid, int nthr) {
  for (int e = tid; e < rrows * HP; e += nthr) {
    const int c = e / HP, o = e - c * HP;
    const float v = (c < in && o < out) ? W[(int64_t)o * stride + c] * scale : 0.f;
    const __half h = __float2half_rn(v);
    const uint32_t off = rtc::sw128h(c, o);
    *reinterpret_cast<__half*>(hi + off) = h;
    *reinterpret_cast<__half*>(lo + off) = __float2half_rn(v - __half2float(h));
  }
}

// one product layer: KSTEPS k-steps of 3 MMAs; `zero` starts a fresh accumulator
template <int KSTEPS>
// (one elected lane in a branch issues unpredicated MMAs: fewer instructions per
// MMA on the layer chain than elect-predicated ones, tcmlp.cuh issue_layer_commit)
CACTO_D void issue(uint32_t d, uint32_t ahi, uint32_t alo, uint64_t whi, uint64_t wlo, uint32_t idesc, bool zero) {
  if (tc::elect_one()) {
#pragma unroll
    for (int kk = 0; kk < KSTEPS; ++kk) {
      const uint64_t wo = (uint64_t)(kk * 2);
      const uint32_t ao = (uint32_t)(kk * 8);
      tc::mma_f16_ts(d, ahi + ao, whi + wo, idesc, (zero && kk == 0) ? 0u : 1u);
      tc::mma_f16_ts(d, ahi + ao, wlo + wo, idesc, 1u);
      tc::mma_f16_ts(d, alo + ao, whi + wo, idesc, 1u);
    }
  }
  __syncwarp();
}

// derivative factors of the activation at z (nets.py:27-52): d1 = act'(z),
// h with act''(z) = h * act'(z)
template <int ACT>
CACTO_D void d1h(float z, float& d1, float& h) {
  if constexpr (ACT == CACTO_ACT_ELU) {
    const float e = tc::ex2_ftz(fminf(z, 0.f) * rtc::LOG2E);
    d1 = z > 0.f ? 1.f : e;
    h = z > 0.f ? 0.f : 1.f;
  } else {
    const float t = tanhf(z);
    d1 = 1.f - t * t;
    h = -2.f * t;
  }
}

// 32-byte aligned destinations (the [g ; zbar] factor rows, 256 B apart): two 256-bit
// stores (STG.E.ENL2.256) instead of four 128-bit ones
using rtc::f2add;
using rtc::f2mul;
using rtc::f2pack;
using rtc::f2sub;
using rtc::f2unpack;

// the activation of 16 scaled accumulators D = S z (ELU: packed fp32x2, tcmlp.cuh elu2)
template <int ACT>
CACTO_D void act16(float (&v)[16]) {
  if constexpr (ACT == CACTO_ACT_ELU) {
#pragma unroll
    for (int c = 0; c < 16; c += 2) f2unpack(elu2(v[c], v[c + 1], ActTC<ACT>::S), v[c], v[c + 1]);
  } else {
#pragma unroll
    for (int c = 0; c < 16; ++c) v[c] = ActTC<ACT>::apply(v[c]);
  }
}
// act'(z) of 16 scaled pre-activations zs = S z.  ELU: S = 8 log2 e, so
// act' = e^min(z,0) = ex2(min(zs,0) / 8) -- 1 exactly for zs >= 0, no select -- with
// 2 min(zs,0) = zs - |zs| on packed FADD2 (one FMUL2 applies the 1/16)
template <int ACT>
CACTO_D void d1_16(const float (&zs)[16], float (&d1)[16]) {
  if constexpr (ACT == CACTO_ACT_ELU) {
#pragma unroll
    for (int c = 0; c < 16; c += 2) {
      const uint64_t z2 = f2pack(zs[c], zs[c + 1]), az = f2pack(fabsf(zs[c]), fabsf(zs[c + 1]));
      float m0, m1;
      f2unpack(f2mul(f2sub(z2, az), f2pack(1.f / 16.f, 1.f / 16.f)), m0, m1);
      d1[c] = tc::ex2_ftz(m0);
      d1[c + 1] = tc::ex2_ftz(m1);
    }
  } else {
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      float h;
      d1h<ACT>(zs[c] * (1.f / ActTC<ACT>::S), d1[c], h);
    }
  }
}
// act''(z) / act'(z) of one scaled pre-activation (ELU: 0 for z > 0, else 1)
template <int ACT>
CACTO_D float h_of(float zs) {
  if constexpr (ACT == CACTO_ACT_ELU) {
    return zs > 0.f ? 0.f : 1.f;
  } else {
    float d1, h;
    d1h<ACT>(zs * (1.f / ActTC<ACT>::S), d1, h);
    return h;
  }
}

CACTO_D void st16g_v8(float* dst, const float (&v)[16]) {
#if CACTO_CTC_V8
#pragma unroll
  for (int q = 0; q < 16; q += 8)
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + q), "f"(v[q]),
                 "f"(v[q + 1]), "f"(v[q + 2]), "f"(v[q + 3]), "f"(v[q + 4]), "f"(v[q + 5]), "f"(v[q + 6]),
                 "f"(v[q + 7])
                 : "memory");
#else
#pragma unroll
  for (int q = 0; q < 16; q += 4) *reinterpret_cast<float4*>(dst + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
#endif
}
CACTO_D void st16g(float* dst, const float (&v)[16]) {
#pragma unroll
  for (int q = 0; q < 16; q += 4) *reinterpret_cast<float4*>(dst + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
}

}  // namespace ctc

// the shared-memory image of one update's weights: critic + target forward slots
// (scaled hi/lo fp16, K-major SW128), the transposed critic layers and w_3; written
// by `tid` of `nthr` threads to `base` (shared memory, or the global image)
template <int ACT>
CACTO_D void critic_stage_all(unsigned char* base, const ctc::Args& a, int tid, int nthr) {
  using namespace ctc;
  using AF = ActTC<ACT>;
  constexpr float S = AF::S;
  const int ip = a.ip;
  const int d = a.b.n + 1;
  if (ip == 8) {
    stage_net<HP, 8, AF>(base, a.critic, 3, d, 1, tid, nthr);
    if (a.target) stage_net<HP, 8, AF>(base + SLOT, a.target, 3, d, 1, tid, nthr);
  } else {
    stage_net<HP, 16, AF>(base, a.critic, 3, d, 1, tid, nthr);
    if (a.target) stage_net<HP, 16, AF>(base + SLOT, a.target, 3, d, 1, tid, nthr);
  }
  const float* W0 = a.critic;
  const float* W1 = W0 + HP * ip + HP;
  const float* W2 = W1 + HP * HP + HP;
  const float* W3 = W2 + HP * HP + HP;
  stage_wt(base + OFF_W0T, base + OFF_W0T + W0T, W0, HP, d, ip, S, rtc::NOUT, tid, nthr);
  stage_wt(base + OFF_W1T, base + OFF_W1T + WHT, W1, HP, HP, HP, S, HP, tid, nthr);
  stage_wt(base + OFF_W2T, base + OFF_W2T + WHT, W2, HP, HP, HP, S, HP, tid, nthr);
  float* w3 = reinterpret_cast<float*>(base + OFF_W3);
  for (int c = tid; c < HP; c += nthr) w3[c] = W3[c];
}

template <int ACT>
__global__ void critic_tc_image_kernel(const ctc::Args a, unsigned char* img) {
  critic_stage_all<ACT>(img, a, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

template <int ACT>
__global__ void __launch_bounds__(ctc::NTHR, 1) critic_tc_kernel(const ctc::Args a) {
  using namespace ctc;
  using AF = ActTC<ACT>;
  constexpr float S = AF::S;            // forward / transposed hidden-layer weight scale
  constexpr float SO = rtc::WSCALE;     // output-layer weight scale
  // backward operands (g, u, zbar) enter the MMAs scaled by SB and the cotangents
  // are carried without the 1/B of the mean (applied in the reductions): both keep
  // the fp16 lo parts out of the subnormal range
  constexpr float SB = 16.f;
  constexpr float RS = 1.f / (S * SB);  // backward product -> value
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
  // two layer chains: "c" (critic forward, sweep, gradient and value paths) and
  // "t" (the target forward, interleaved with the critic forward)
  __shared__ __align__(8) uint64_t full_bar, done_bar, full_t, done_t;
  __shared__ uint32_t tmem_base_sh;
  __shared__ float red[NTHR / 32];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = a.b.n;
  const int d = n + 1;

  // ---- weights -> shared memory: one bulk copy of the image critic_tc_image_kernel
  //      built for this update (the per-CTA fp16 split + swizzle staging cost ~11 % of
  //      the kernel's stall samples), or stage it here -------------------------------
  if (a.img) {
    __shared__ __align__(8) uint64_t img_bar;
    if (threadIdx.x == 0) {
      tc::mbar_init(&img_bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      tc::mbar_expect_tx(&img_bar, IMG_BYTES);
      for (uint32_t o = 0; o < IMG_BYTES; o += 32768) {
        const uint32_t sz = IMG_BYTES - o < 32768 ? IMG_BYTES - o : 32768;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                saddr(base + o)),
            "l"(a.img + o), "r"(sz), "r"(saddr(&img_bar))
            : "memory");
      }
    }
    tc::mbar_wait(&img_bar, 0);
  } else {
    critic_stage_all<ACT>(base, a, threadIdx.x, NTHR);
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(&full_bar, NEPI);
    tc::mbar_init(&done_bar, 1);
    tc::mbar_init(&full_t, NEPI);
    tc::mbar_init(&done_t, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) tc::tmem_alloc(&tmem_base_sh, 512);
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t sbase = saddr(base);
  const int64_t B = a.b.rows;
  const int64_t ntiles = (B + TILE - 1) / TILE;
  const bool boot = a.target != nullptr;

  if (warp < NEPI) {
    // ---- epilogue ------------------------------------------------------------------
    const int q = warp & 3, part = warp >> 2;
    const int r = (q << 5) + lane;
    const int c0 = part * 16;  // my accumulator columns [c0, c0 + 16)
    const uint32_t lrow = tmem + ((uint32_t)(q * 32) << 16);
    const bool owner = part == 0;
    const float* w3 = reinterpret_cast<const float*>(base + OFF_W3);
    const uint32_t bias_c = sbase + PL::off_bias, bias_t = sbase + SLOT + PL::off_bias;
    uint32_t pd = 0, pdt = 0;
    float loss_acc = 0.f;
    int tl_w = 0, tl_h = 0;  // timeline counters (warp 0)
    int64_t tl_t = 0;
    (void)tl_w; (void)tl_h; (void)tl_t;
    auto handoff = [&]() {
      tc::tmem_wait_st();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full_bar);
#if CACTO_CTC_TIMELINE
      if (warp == 0) { CTC_TL(tl_h, 3, tl_t); ++tl_h; }
#endif
    };
    auto handoff_t = [&]() {
      tc::tmem_wait_st();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full_t);
    };
    auto wait_done_t = [&]() {
      tc::mbar_wait(&done_t, pdt);
      pdt ^= 1;
      tc::tc_fence_after();
    };
    auto wait_done = [&]() {
      tc::mbar_wait(&done_bar, pd);
#if CACTO_CTC_TIMELINE
      if (warp == 0) { CTC_TL(tl_w, 2, tl_t); ++tl_w; }
#endif
      pd ^= 1;
      tc::tc_fence_after();
    };
    auto ld16 = [&](uint32_t col, float (&v)[16]) { tc::tmem_ld16_wait(lrow + col, v); };
    auto st16 = [&](uint32_t col, const float (&v)[16]) { tc::tmem_st16(lrow + col, v); };
    // my 16 values -> next layer's A (hi/lo), columns [c0, c0 + 16) of the operand
    auto put_a = [&](const float (&v)[16]) {
      float hv[8], lv[8];
#pragma unroll
      for (int c = 0; c < 16; c += 2) {
        uint32_t h, l;
        rtc::split2(v[c], v[c + 1], h, l);
        hv[c / 2] = __uint_as_float(h);
        lv[c / 2] = __uint_as_float(l);
      }
      tc::tmem_st8(lrow + TA_HI + (uint32_t)(c0 / 2), hv);
      tc::tmem_st8(lrow + TA_LO + (uint32_t)(c0 / 2), lv);
    };
    auto put_at = [&](const float (&v)[16]) {  // the target chain's A (in the G region)
      float hv[8], lv[8];
#pragma unroll
      for (int c = 0; c < 16; c += 2) {
        uint32_t h, l;
        rtc::split2(v[c], v[c + 1], h, l);
        hv[c / 2] = __uint_as_float(h);
        lv[c / 2] = __uint_as_float(l);
      }
      tc::tmem_st8(lrow + TT_AHI + (uint32_t)(c0 / 2), hv);
      tc::tmem_st8(lrow + TT_ALO + (uint32_t)(c0 / 2), lv);
    };
    auto put_ab = [&](const float (&v)[16]) {  // backward operand, scaled by SB
      float w[16];
#pragma unroll
      for (int c = 0; c < 16; c += 2) f2unpack(f2mul(f2pack(v[c], v[c + 1]), f2pack(SB, SB)), w[c], w[c + 1]);
      put_a(w);
    };
    auto preload_bias = [&](uint32_t col, uint32_t bias_s, int layer) {
      float bv[16];
#pragma unroll
      for (int c = 0; c < 16; c += 4) {
        const V4<float> v = lds4(bias_s + (uint32_t)((layer * HP + c0 + c) * 4), (float*)nullptr);
        bv[c] = v.v[0]; bv[c + 1] = v.v[1]; bv[c + 2] = v.v[2]; bv[c + 3] = v.v[3];
      }
      st16(col + (uint32_t)c0, bv);  // my columns of the layer's accumulator
    };
    auto preload_out_bias = [&](uint32_t bias_s, uint32_t dcol = TD) {  // output layer: 16 columns (part 0)
      if (!owner) return;
      float bv[16];
#pragma unroll
      for (int c = 0; c < 16; c += 4) {
        const V4<float> v = lds4(bias_s + (uint32_t)((3 * HP + c) * 4), (float*)nullptr);
        bv[c] = v.v[0]; bv[c + 1] = v.v[1]; bv[c + 2] = v.v[2]; bv[c + 3] = v.v[3];
      }
      st16(dcol, bv);
    };
    // the owner's normalised input row (16 columns) -> A
    auto put_input = [&](const float (&v)[16]) {
      if (!owner) return;
      put_a(v);
    };
    auto put_input_t = [&](const float (&v)[16]) {
      if (!owner) return;
      put_at(v);
    };

    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      tl_w = tl_h = 0;
      tl_t = t;
      const int64_t gb = t * TILE + r;
      const bool valid = gb < B;
      const int64_t rr = valid ? a.b.row(gb) : 0;
      float y = 0.f;
      float xin[16];
      // the owner gathers every per-sample input of the tile up front (one round of
      // independent loads instead of dependent index -> row chains inside the layer
      // chain); fixed-trip loops keep the arrays in registers
      float xr[16], xkr[16], vxr[16], vbar = 0.f;
      bool gate = false;
#pragma unroll
      for (int c = 0; c < 16; ++c) xr[c] = xkr[c] = vxr[c] = 0.f;
      if (owner && valid) {
        const float* x = a.b.xa + rr * d;
        const float* xk = a.b.xa_plus_k + rr * d;
        const float* vx = a.b.v_bar_x + rr * n;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          if (c < d) {
            xr[c] = x[c];
            if (boot) xkr[c] = xk[c];
          }
          if (c < n) vxr[c] = vx[c];
        }
        vbar = a.b.v_bar[rr];
        gate = boot && xk[n] < (float)a.b.t_max;
      }
      // ---- target forward at x_{+k} (nets.py:247-251) and critic forward at x, as two
      //      interleaved layer chains (z_i of the critic kept in TMEM) -----------------
      if (boot) {
        if (owner) {
#pragma unroll
          for (int c = 0; c < 16; ++c)
            xin[c] = (valid && c < d) ? (xkr[c] - a.nc_t.in_center[c]) * a.nc_t.in_inv_half[c] : 0.f;
        }
        put_input_t(xin);
        preload_bias(TT_D, bias_t, 0);
        handoff_t();
      }
      if (owner) {
#pragma unroll
        for (int c = 0; c < 16; ++c) xin[c] = 0.f;
        if (valid) {
#pragma unroll
          for (int c = 0; c < 16; ++c) xin[c] = c < d ? (xr[c] - a.nc.in_center[c]) * a.nc.in_inv_half[c] : 0.f;
          y += vbar;
          st16g(a.UA[0] + (B + gb) * 20, xin);  // a_0 = normalised input
          *reinterpret_cast<float4*>(a.UA[0] + (B + gb) * 20 + 16) = make_float4(1.f, 0.f, 0.f, 0.f);
        }
      }
      put_input(xin);
      preload_bias(TZ, bias_c, 0);
      handoff();
      // L2 prefetch of this CTA's next tile's sample rows (issued while the first
      // layers' MMAs run): the gather at the next tile start then hits L2
      if (owner) {
        const int64_t gbn = (t + gridDim.x) * TILE + r;
        if (gbn < B) {
          const int64_t rn = a.b.row(gbn);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a.b.xa + rn * d));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a.b.v_bar_x + rn * n));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a.b.v_bar + rn));
          if (boot) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.b.xa_plus_k + rn * d));
        }
      }
      for (int l = 0; l < 3; ++l) {
        if (boot) {
          wait_done_t();
          float z[16];
          ld16(TT_D + c0, z);
          act16<ACT>(z);
          put_at(z);
          if (l < 2) preload_bias(TT_D, bias_t, l + 1);
          else preload_out_bias(bias_t, TT_D);
          handoff_t();
        }
        wait_done();
        float z[16];
        ld16(TZ + 64 * l + c0, z);
        float(&av)[16] = z;
        act16<ACT>(av);
        put_a(av);
        if (l < 2) preload_bias(TZ + 64 * (l + 1), bias_c, l + 1);
        else preload_out_bias(bias_c);
        handoff();
        // factor stores after the hand-off: the next layer's MMAs do not wait for them
        if (valid) {
          float* row = a.UA[l + 1] + (B + gb) * 68;
          st16g(row + c0, av);
          if (owner) *reinterpret_cast<float4*>(row + 64) = make_float4(1.f, 0.f, 0.f, 0.f);
        }
      }
      if (boot) {
        wait_done_t();
        if (owner) {
          float o[16];
          ld16(TT_D, o);
          if (valid) y += gate ? o[0] * (1.f / SO) : 0.f;
        }
      }
      // output: V, e_v, delta; then the sweep starts: g_2 = act'(z_2) w_3
      wait_done();
      float ev = 0.f, delta = 0.f;
      if (owner) {
        float o[16];
        ld16(TD, o);
        if (valid) {
          ev = y - o[0] * (1.f / SO);
          delta = -2.f * ev;  // x 1/denom in the reductions
          a.V3[gb] = 1.f;
          a.V3[B + gb] = delta;
        }
      }
      {
        float z[16], g[16];
        ld16(TZ + 128 + c0, z);
        float d1[16];
        d1_16<ACT>(z, d1);
#pragma unroll
        for (int c = 0; c < 16; ++c) g[c] = d1[c] * w3[c0 + c];
        st16(TG + 128 + c0, g);
        put_ab(g);
        handoff();  // S2: s_2 = g_2 W_2
        if (valid) st16g_v8(a.GZ[2] + gb * 64 + c0, g);
      }
      for (int l = 1; l >= 0; --l) {  // g_l = act'(z_l) s_{l+1}
        wait_done();
        float s[16], z[16], g[16];
        tc::tmem_ld16x2_wait(lrow + TD + c0, lrow + TZ + 64 * l + c0, s, z);
        float d1[16];
        d1_16<ACT>(z, d1);
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
          const uint64_t gp = f2mul(f2mul(f2pack(d1[c], d1[c + 1]), f2pack(s[c], s[c + 1])), f2pack(RS, RS));
          f2unpack(gp, g[c], g[c + 1]);
        }
        st16(TG + 64 * l + c0, g);
        put_ab(g);
        handoff();  // S1: s_1 = g_1 W_1 ; S0: s_0 = g_0 W_0 (N = 16)
        if (valid) st16g_v8(a.GZ[l] + gb * 64 + c0, g);
      }
      // errors, loss, u_0 (nets.py:268-277)
      wait_done();
      {
        float u0[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) u0[c] = 0.f;
        if (owner) {
          float s0[16];
          ld16(TD, s0);
          if (valid) {
            float eg2 = 0.f;
            const float coef = -2.f * a.k_s;  // x 1/denom in the reductions
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              if (c < n) {
                const float eg = vxr[c] - s0[c] * RS * a.nc.in_inv_half[c];
                eg2 += eg * eg;
                u0[c] = coef * eg * a.nc.in_inv_half[c];
              }
            }
            loss_acc += (ev * ev + a.k_s * eg2) * a.inv_denom;
            st16g(a.UA[0] + gb * 20, u0);
            *reinterpret_cast<float4*>(a.UA[0] + gb * 20 + 16) = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        if (owner) put_ab(u0);
        handoff();  // R0: r_0 = W_0 u_0
      }
      // gradient path (nets.py:279-284): zeta_l = h(z_l) g_l r_l, u_{l+1} = act'(z_l) r_l
      for (int l = 0; l < 3; ++l) {
        wait_done();
        float rv[16], z[16], g[16], u[16];
        tc::tmem_ld16x3_wait(lrow + TD + c0, lrow + TZ + 64 * l + c0, lrow + TG + 64 * l + c0, rv, z, g);
        float d1[16];
        d1_16<ACT>(z, d1);
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const float rr_ = rv[c] * RS;
          g[c] = h_of<ACT>(z[c]) * g[c] * rr_;  // zeta_l
          u[c] = d1[c] * rr_;
        }
        st16(TG + 64 * l + c0, g);
        if (l < 2) {
          put_ab(u);
          handoff();  // R1, R2
          if (valid) {
            float* row = a.UA[l + 1] + gb * 68;
            st16g(row + c0, u);
            if (owner) *reinterpret_cast<float4*>(row + 64) = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        } else {
          if (valid) {
            float* row = a.UA[3] + gb * 68;
            st16g(row + c0, u);
            if (owner) *reinterpret_cast<float4*>(row + 64) = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      }
      float zb[16];
      // value path (nets.py:287-289, 215-230): abar_3 = delta w_3,
      // zbar_2 = act'(z_2) abar_3 + zeta_2; delta lives in the quadrant's owner thread
      {
        __shared__ float del_sh[TILE];
        if (owner) del_sh[r] = delta;
        // epilogue warps only: a named barrier over the 16 epilogue warps
        asm volatile("bar.sync 1, %0;" ::"n"(NEPI * 32) : "memory");
        const float dlt = del_sh[r];
        float z[16], zeta[16];
        tc::tmem_ld16x2_wait(lrow + TZ + 128 + c0, lrow + TG + 128 + c0, z, zeta);
        float d1[16];
        d1_16<ACT>(z, d1);
#pragma unroll
        for (int c = 0; c < 16; ++c) zb[c] = d1[c] * (dlt * w3[c0 + c]) + zeta[c];
        // no second barrier before the next tile rewrites del_sh: that happens >= 10
        // layer hand-offs later, each needing all 16 epilogue warps (full_bar), so
        // every read above is done by then
      }
      put_ab(zb);
      handoff();  // B2: abar_2 = zbar_2 W_2
      if (valid) st16g_v8(a.GZ[2] + (B + gb) * 64 + c0, zb);
      for (int l = 1; l >= 0; --l) {
        wait_done();
        float ab[16], z[16], zeta[16];
        tc::tmem_ld16x3_wait(lrow + TD + c0, lrow + TZ + 64 * l + c0, lrow + TG + 64 * l + c0, ab, z, zeta);
        float d1[16];
        d1_16<ACT>(z, d1);
#pragma unroll
        for (int c = 0; c < 16; ++c) zb[c] = d1[c] * ab[c] * RS + zeta[c];
        if (l == 1) {
          put_ab(zb);
          handoff();  // B1: abar_1 = zbar_1 W_1
        }
        if (valid) st16g_v8(a.GZ[l] + (B + gb) * 64 + c0, zb);
      }
    }
    // loss partial of this CTA
    float v = loss_acc;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    asm volatile("bar.sync 1, %0;" ::"n"(NEPI * 32) : "memory");
    if (threadIdx.x == 0) {
      float s = 0.f;
      for (int w = 0; w < NEPI; ++w) s += red[w];
      a.lossp[blockIdx.x] = s;
    }
  } else {
    // ---- MMA issuer --------------------------------------------------------------------
    const uint32_t i64 = tc::idesc_f16(HP), i16 = tc::idesc_f16(rtc::NOUT);
    auto desc = [&](uint32_t off) { return tc::make_desc(sbase + off, 16, 1024, 2); };
    auto desc0 = [&](uint32_t off) { return tc::make_desc(sbase + off, rtc::W0_LBO, rtc::W0_SBO, 0); };
    const uint32_t ahi = tmem + TA_HI, alo = tmem + TA_LO;
    uint32_t pf = 0, pft = 0;
    auto fwd = [&](uint32_t so, int l, uint32_t dcol, uint32_t ah, uint32_t al) {
      if (l == 0) issue<1>(dcol, ah, al, desc0(so + PL::off_w0), desc0(so + PL::off_w0 + PL::W0), i64, false);
      else if (l < 3)
        issue<4>(dcol, ah, al, desc(so + PL::off_wh + (uint32_t)(2 * (l - 1)) * PL::WH),
                 desc(so + PL::off_wh + (uint32_t)(2 * (l - 1)) * PL::WH + PL::WH), i64, false);
      else issue<4>(dcol, ah, al, desc(so + PL::off_wo), desc(so + PL::off_wo + PL::WO), i16, false);
    };
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int l = 0; l < 4; ++l) {  // forwards: target layer l, then critic layer l
        if (boot) {
          tc::mbar_wait(&full_t, pft);
          pft ^= 1;
          tc::tc_fence_after();
          fwd(SLOT, l, tmem + TT_D, tmem + TT_AHI, tmem + TT_ALO);
          tc::tc_commit_elect(&done_t);
          __syncwarp();
        }
        tc::mbar_wait(&full_bar, pf);
        CTC_TL(l, 0, t);
        pf ^= 1;
        tc::tc_fence_after();
        fwd(0, l, l < 3 ? tmem + TZ + 64 * l : tmem + TD, ahi, alo);
        tc::tc_commit_elect(&done_bar);
        __syncwarp();
        CTC_TL(l, 1, t);
      }
      for (int k = 8; k < 16; ++k) {  // sweep, gradient path, value path
        tc::mbar_wait(&full_bar, pf);
        CTC_TL(k - 4, 0, t);
        pf ^= 1;
        tc::tc_fence_after();
        if (k == 8) {
          issue<4>(tmem + TD, ahi, alo, desc(OFF_W2T), desc(OFF_W2T + WHT), i64, true);  // s_2
        } else if (k == 9) {
          issue<4>(tmem + TD, ahi, alo, desc(OFF_W1T), desc(OFF_W1T + WHT), i64, true);  // s_1
        } else if (k == 10) {
          issue<4>(tmem + TD, ahi, alo, desc(OFF_W0T), desc(OFF_W0T + W0T), i16, true);  // s_0
        } else if (k == 11) {
          issue<1>(tmem + TD, ahi, alo, desc0(PL::off_w0), desc0(PL::off_w0 + PL::W0), i64, true);  // r_0
        } else if (k == 12 || k == 13) {
          const uint32_t wo = PL::off_wh + (uint32_t)(2 * (k - 12)) * PL::WH;
          issue<4>(tmem + TD, ahi, alo, desc(wo), desc(wo + PL::WH), i64, true);  // r_1, r_2
        } else if (k == 14) {
          issue<4>(tmem + TD, ahi, alo, desc(OFF_W2T), desc(OFF_W2T + WHT), i64, true);  // abar_2
        } else {
          issue<4>(tmem + TD, ahi, alo, desc(OFF_W1T), desc(OFF_W1T + WHT), i64, true);  // abar_1
        }
        tc::tc_commit_elect(&done_bar);
        __syncwarp();
        CTC_TL(k - 4, 1, t);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) tc::tmem_dealloc(tmem, 512);
}

// ======================================================================================
// host side
// ======================================================================================
namespace ctc {

struct Plan2 {  // workspace carve
  size_t off_gz[3], off_ua[4], off_v3, off_lossp, off_img, off_part[4], part_bytes[4], total;
};

static Plan2 plan2(int64_t B, int64_t P) {
  Plan2 p{};
  size_t o = ((size_t)(P + 1) * 4 + 255) & ~(size_t)255;  // gradient slot first
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 255) & ~(size_t)255;
    return r;
  };
  for (int l = 0; l < 3; ++l) p.off_gz[l] = take((size_t)2 * B * HP * 4);
  p.off_ua[0] = take((size_t)2 * B * 20 * 4);
  for (int l = 1; l < 4; ++l) p.off_ua[l] = take((size_t)2 * B * 68 * 4);
  p.off_v3 = take((size_t)2 * B * 4 + 16);
  p.off_lossp = take((size_t)4096 * 4);
  p.off_img = take(IMG_BYTES);
  // split-K partials of the four reduction GEMMs, each in its own region (the fused
  // reduce + scatter reads all four after the last GEMM)
  const int pm[4] = {HP, HP, HP, 1}, pn[4] = {17, 65, 65, 65};
  for (int l = 0; l < 4; ++l) {
    const size_t w = gemm_workspace_bytes(pm[l], pn[l], (int)(2 * B));
    size_t one = (size_t)pm[l] * pn[l] * 4;
    if (l == 3) one = (size_t)4 * 1024 * 65 * 4;  // out_row_grad_kernel: up to 4 x SMs partial rows
    else one = std::max(one, (size_t)2048 * HP * pn[l] * 4);  // wgrad_kernel: 2 partials per CTA
    p.part_bytes[l] = w > one ? w : one;
    p.off_part[l] = take(p.part_bytes[l]);
  }
  p.total = o + 256;
  return p;
}

// gradient entries of the four reduction outputs: W_0 [64][cols0], b_0, W_1, b_1, W_2, b_2, w_3 [64], b_3
constexpr int scatter_items(int cols0) { return HP * cols0 + HP + 2 * (HP * HP + HP) + HP + 1; }

// split-K reduction fused with the scatter: one warp per gradient entry, lanes
// over the splits and the fixed shuffle tree of tc::splitk_reduce_warp_kernel
// (same sums, same order), lane 0 adds into the gradient slot -- one launch
// instead of four reductions + a scatter
struct PartSet {
  const float* p[4];
  int splits[4];
  int64_t stride[4];
};
CACTO_D float split_sum(const PartSet& ps, int l, int64_t off, int lane) {
  float s = 0.f;
  for (int z = lane; z < ps.splits[l]; z += 32) s += ps.p[l][z * ps.stride[l] + off];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}
__global__ void reduce_scatter_grads_kernel(const PartSet ps, int cols0, float* slot, int64_t w0, int64_t b0,
                                            int64_t w1, int64_t b1, int64_t w2, int64_t b2, int64_t w3, int64_t b3) {
  const int lane = threadIdx.x & 31;
  int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // warp-uniform
  int l;
  int64_t off, dst;
  if (e < HP * cols0) {
    l = 0, off = (e / cols0) * 17 + (e % cols0), dst = w0 + e;
  } else if ((e -= HP * cols0) < HP) {
    l = 0, off = e * 17 + 16, dst = b0 + e;
  } else if ((e -= HP) < HP * HP) {
    l = 1, off = (e / HP) * 65 + (e % HP), dst = w1 + e;
  } else if ((e -= HP * HP) < HP) {
    l = 1, off = e * 65 + 64, dst = b1 + e;
  } else if ((e -= HP) < HP * HP) {
    l = 2, off = (e / HP) * 65 + (e % HP), dst = w2 + e;
  } else if ((e -= HP * HP) < HP) {
    l = 2, off = e * 65 + 64, dst = b2 + e;
  } else if ((e -= HP) < HP) {
    l = 3, off = e, dst = w3 + e;
  } else if ((e -= HP) == 0) {
    l = 3, off = 64, dst = b3;
  } else {
    return;
  }
  const float s = split_sum(ps, l, off, lane);
  if (lane == 0) slot[dst] += s;
}

// the same reduction with coalesced reads: layers 0..2 one THREAD per gradient entry,
// consecutive threads on consecutive (row, column) entries of the [rows][ncol] partials,
// each summing its entry's split partials in split order (a fixed order: deterministic;
// the warp-per-entry form read one 32-byte sector per partial and lane); the output
// row (65 entries over ~4 x SMs partials) keeps one warp per entry
__global__ void reduce_scatter_coalesced_kernel(const PartSet ps, int cols0, float* slot, int64_t w0, int64_t b0,
                                                int64_t w1, int64_t b1, int64_t w2, int64_t b2, int64_t w3,
                                                int64_t b3, int n_thr) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n_thr) {
    int l, nc;
    if (e < HP * 17) {
      l = 0, nc = 17;
    } else if ((e -= HP * 17) < HP * 65) {
      l = 1, nc = 65;
    } else {
      e -= HP * 65, l = 2, nc = 65;
    }
    const int o = e / nc, c = e - o * nc;
    int64_t dst;
    if (l == 0) {
      if (c == 16) dst = b0 + o;
      else if (c < cols0) dst = w0 + (int64_t)o * cols0 + c;
      else return;
    } else {
      dst = (c == 64 ? (l == 1 ? b1 : b2) + o : (l == 1 ? w1 : w2) + (int64_t)o * HP + c);
    }
    const float* p = ps.p[l] + e;
    const int64_t st = ps.stride[l];
    float s0 = 0.f, s1 = 0.f;  // even / odd splits, then one add: a fixed order
    int z = 0;
    for (; z + 1 < ps.splits[l]; z += 2) {
      s0 += p[z * st];
      s1 += p[(z + 1) * st];
    }
    if (z < ps.splits[l]) s0 += p[z * st];
    slot[dst] += s0 + s1;
    return;
  }
  // output row: warp per entry over the out_row partials
  const int we = (e - n_thr) >> 5, lane = threadIdx.x & 31;
  if (we > HP) return;
  const float sum = split_sum(ps, 3, we, lane);
  if (lane == 0) slot[we < HP ? w3 + we : b3] += sum;
}

// ---- weight gradients of layers 0..2 on the tensor cores, fp16 pairs -----------------
// gW_l[o][c] = alpha * sum_b G_l[b][o] * U_l[b][c] over the 2B rows b (g then zbar in G,
// u then a | bias column in U): the per-sample factors critic_tc_kernel streamed as fp32
// [2B][w] rows.  Per 64-sample k-block:
//   warp 16      TMA: the raw fp32 [64][64] G block and [64][w] U block -> a 3-stage ring
//   warps 0..15  read the raw block from shared memory, scale by SB, split each value into
//                fp16 hi + lo (as the per-sample MMAs do) and store them TRANSPOSED into
//                K-major SW128 tiles (row = o or c, 64 samples = 128 B), a 2-stage ring
//   warp 17      issues [G_hi ; G_lo] x U_hi and [G_hi ; G_lo] x U_lo (tcgen05 kind::f16,
//                M = 128: rows 0..63 take the hi parts of G, rows 64..127 the lo parts,
//                N = 32 / 80) into one TMEM accumulator: two MMAs per k-step and no padded
//                rows; the two row halves leave as two partials that the reduction sums
// Each factor is read from HBM once (the 3xTF32 GEMM it replaces split operands through
// shared memory at ~2.3 TB/s).  CTAs split K per layer; the partials go to
// reduce_scatter_grads_kernel (fixed order: deterministic).
constexpr int WG_KB = 64;
constexpr int WG_RAW = 3;    // raw fp32 stages
constexpr int WG_STAGES = 3; // converted fp16 stages
constexpr int WG_CONV = 16;
constexpr int WG_TMA_WARP = WG_CONV, WG_MMA_WARP = WG_CONV + 1;
constexpr int WG_THREADS = (WG_CONV + 2) * 32;
constexpr uint32_t WG_A = 128 * 128;  // [G_hi ; G_lo]: 128 rows x 64 samples (fp16)
constexpr uint32_t WG_B = 80 * 128;
constexpr uint32_t WG_STAGE = WG_A + 2 * WG_B;
constexpr uint32_t WG_RG = WG_KB * 64 * 4;   // raw G block
constexpr uint32_t WG_RU = WG_KB * 68 * 4;   // raw U block (widest row: 68 floats)
constexpr uint32_t WG_RSTAGE = WG_RG + WG_RU;
constexpr uint32_t WG_SMEM = WG_STAGES * WG_STAGE + WG_RAW * WG_RSTAGE + 1024;
constexpr float WG_SB = 16.f;

struct __align__(64) WgradArgs {
  CUtensorMap tg[3], tu[3];  // raw G / U blocks: boxes [64][64] and [64][uw]
  int uw[3], ncol[3], nmma[3];
  int cta0[4];
  int64_t chunk[3];
  int64_t K2;
  float* part[3];
  float alpha;
};

// 8 K-consecutive values of one row -> hi / lo fp16 16-byte chunks
CACTO_D void split8(const float (&v)[8], uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float a0, a1;  // the SB scaling on packed FMUL2
    rtc::f2unpack(rtc::f2mul(rtc::f2pack(v[2 * j], v[2 * j + 1]), rtc::f2pack(WG_SB, WG_SB)), a0, a1);
    rtc::split2(a0, a1, h[j], l[j]);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}
CACTO_D void sts128(uint32_t addr, const uint4& v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
CACTO_D float lds1f(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

__global__ void __launch_bounds__(WG_THREADS, 1) wgrad_kernel(const __grid_constant__ WgradArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t raw_full[WG_RAW], raw_empty[WG_RAW], full_bar[WG_STAGES], empty_bar[WG_STAGES],
      acc_bar;
  __shared__ uint32_t tmem_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int l = blockIdx.x >= a.cta0[2] ? 2 : (blockIdx.x >= a.cta0[1] ? 1 : 0);
  const int z = blockIdx.x - a.cta0[l];
  const int64_t k0 = (int64_t)z * a.chunk[l];
  const int64_t k1 = k0 + a.chunk[l] < a.K2 ? k0 + a.chunk[l] : a.K2;
  const int nkb = (int)((k1 - k0 + WG_KB - 1) / WG_KB);
  const int ncol = a.ncol[l], uw = a.uw[l];
  if (threadIdx.x == 0) {
    for (int s = 0; s < WG_RAW; ++s) {
      tc::mbar_init(&raw_full[s], 1);
      tc::mbar_init(&raw_empty[s], WG_CONV);
    }
    for (int s = 0; s < WG_STAGES; ++s) {
      tc::mbar_init(&full_bar[s], WG_CONV);
      tc::mbar_init(&empty_bar[s], 1);
    }
    tc::mbar_init(&acc_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == WG_MMA_WARP) tc::tmem_alloc(&tmem_sh, 128);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t sb = saddr(base);
  unsigned char* raw = base + WG_STAGES * WG_STAGE;

  if (warp == WG_TMA_WARP) {
    if (lane == 0) {
      const uint32_t ub = (uint32_t)(WG_KB * uw * 4);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % WG_RAW;
        if (kb >= WG_RAW) tc::mbar_wait(&raw_empty[s], ((kb / WG_RAW) - 1) & 1);
        tc::mbar_expect_tx(&raw_full[s], WG_RG + ub);
        const int row = (int)(k0 + (int64_t)kb * WG_KB);
        unsigned char* rs = raw + (uint32_t)s * WG_RSTAGE;
        tc::tma_load_2d(rs, &a.tg[l], &raw_full[s], 0, row);
        tc::tma_load_2d(rs + WG_RG, &a.tu[l], &raw_full[s], 0, row);
      }
    }
  } else if (warp < WG_CONV) {
    // warps 0..7 convert G, warps 8..15 U: warp w handles samples [8(w%8), +8) of every
    // k-block; lane L owns rows L, L+32 (and L+64 of U) -- 8 consecutive samples of a
    // row = one 16-byte chunk of the K-major tile
    const bool gw = warp < 8;
    const int sg = warp & 7;
    for (int kb = 0; kb < nkb; ++kb) {
      const int rs = kb % WG_RAW, s = kb % WG_STAGES;
      tc::mbar_wait(&raw_full[rs], (kb / WG_RAW) & 1);
      // k-blocks never straddle a chunk end (chunks are multiples of 64 samples) and rows
      // past K2 are TMA zero fill: no per-row masks
      float v[3][8];
      const float* rp = reinterpret_cast<const float*>(raw + (uint32_t)rs * WG_RSTAGE) + sg * 8 * 64;
      if (gw) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          v[0][j] = rp[j * 64 + lane];
          v[1][j] = rp[j * 64 + lane + 32];
        }
      } else {
        const float* up = reinterpret_cast<const float*>(raw + (uint32_t)rs * WG_RSTAGE + WG_RG) + sg * 8 * uw;
#pragma unroll
        for (int rr = 0; rr < 3; ++rr) {
          const int c = lane + 32 * rr;
          if (32 * rr < ncol) {  // warp-uniform
            const int cc = c < ncol ? c : 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) v[rr][j] = up[j * uw + cc];
          }
        }
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&raw_empty[rs]);
      if (kb >= WG_STAGES) tc::mbar_wait(&empty_bar[s], ((kb / WG_STAGES) - 1) & 1);
      const uint32_t st0 = sb + (uint32_t)s * WG_STAGE;
      uint4 hi, lo;
      if (gw) {
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int o = lane + 32 * rr, ol = o + 64;  // hi -> row o, lo -> row o + 64
          split8(v[rr], hi, lo);
          sts128(st0 + (uint32_t)o * 128 + (uint32_t)((sg ^ (o & 7)) << 4), hi);
          sts128(st0 + (uint32_t)ol * 128 + (uint32_t)((sg ^ (ol & 7)) << 4), lo);
        }
      } else {
#pragma unroll
        for (int rr = 0; rr < 3; ++rr) {
          const int c = lane + 32 * rr;
          if (32 * rr < ncol) {  // warp-uniform; lanes past ncol skip the store only
            split8(v[rr], hi, lo);
            const uint32_t off = (uint32_t)c * 128 + (uint32_t)((sg ^ (c & 7)) << 4);
            if (c < ncol) {
              sts128(st0 + WG_A + off, hi);
              sts128(st0 + WG_A + WG_B + off, lo);
            }
          }
        }
      }
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full_bar[s]);
    }
    if (warp < 4) {  // accumulator rows 0..63 (hi x U) -> partial 2z, rows 64..127 (lo x U) -> 2z + 1
      tc::mbar_wait(&acc_bar, 0);
      tc::tc_fence_after();
      const int row = warp * 32 + lane, orow = row & 63;
      float* dst = a.part[l] + ((int64_t)(2 * z + (row >> 6)) * HP + orow) * ncol;
      for (int c0 = 0; c0 < ncol; c0 += 16) {
        float v[16];
        tc::tmem_ld16_wait(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c0 + c < ncol) dst[c0 + c] = a.alpha * v[c];
      }
    }
  } else {
    // MMA issuer
    const uint32_t idesc = tc::idesc_f16(a.nmma[l]);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % WG_STAGES;
      tc::mbar_wait(&full_bar[s], (kb / WG_STAGES) & 1);
      tc::tc_fence_after();
      const uint32_t st0 = sb + (uint32_t)s * WG_STAGE;
      if (tc::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < WG_KB / 16; ++kk) {
          const uint64_t ad = tc::make_desc(st0 + kk * 32, 16, 1024, 2);
          const uint64_t bhi = tc::make_desc(st0 + WG_A + kk * 32, 16, 1024, 2);
          const uint64_t blo = tc::make_desc(st0 + WG_A + WG_B + kk * 32, 16, 1024, 2);
          tc::mma_f16_ss(tmem, ad, bhi, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          tc::mma_f16_ss(tmem, ad, blo, idesc, 1u);
        }
        tc::tc_commit(&empty_bar[s]);
      }
      __syncwarp();
    }
    tc::tc_commit_elect(&acc_bar);
    __syncwarp();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == WG_MMA_WARP) tc::tmem_dealloc(tmem, 128);
}

// 2D fp32 tensor map (no swizzle) over rows x cols with a row stride of `ld` floats
typedef CUresult (*WgEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static int wg_map(CUtensorMap* map, const float* X, int64_t rows, int cols, int ld, int box_rows) {
  static WgEncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return set_error(CACTO_ECUDA, "wgrad: cuTensorMapEncodeTiled unavailable");
    fn = (WgEncodeFn)p;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)cols, (cuuint32_t)box_rows}, estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)X, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(CACTO_ECUDA, "wgrad: tensor map encode failed (%d)", (int)r);
  return CACTO_OK;
}

// output-row gradient (w_3 and b_3): part[z][c] = alpha * sum_{b in chunk z} V3[b] * UA3[b][c],
// c < 65, over the 2B rows [u_3 ; a_3 | bias column] -- a matrix-vector product, so
// CUDA cores at HBM speed (one warp per row, lanes over columns; the 8 warps' sums
// folded in a fixed order: deterministic)
__global__ void __launch_bounds__(256) out_row_grad_kernel(const float* __restrict__ V3, const float* __restrict__ UA3,
                                                           int64_t K2, int64_t chunk, float alpha, float* part) {
  __shared__ float red[8][68];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b0 = (int64_t)blockIdx.x * chunk, b1 = b0 + chunk < K2 ? b0 + chunk : K2;
  // a half-warp per row (17 lanes x float4 = the 68-float row), two rows per warp
  // step and 4 steps in flight: 8 independent row loads per warp before the FMAs
  const int h = lane >> 4, c4 = lane & 15;  // row parity, float4 column (lanes 0..15 -> cols 0..63)
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float accb = 0.f;  // column 64 (bias), lane c4 == 0 of each half
  for (int64_t b = b0 + 2 * warp + h; b < b1; b += 4 * 16) {
    float v[4];
    float4 x[4];
    float xb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t r = b + u * 16;
      const bool ok = r < b1;
      v[u] = ok ? V3[r] : 0.f;
      x[u] = ok ? *reinterpret_cast<const float4*>(UA3 + r * 68 + 4 * c4) : make_float4(0.f, 0.f, 0.f, 0.f);
      xb[u] = (ok && c4 == 0) ? UA3[r * 68 + 64] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc.x = fmaf(v[u], x[u].x, acc.x);
      acc.y = fmaf(v[u], x[u].y, acc.y);
      acc.z = fmaf(v[u], x[u].z, acc.z);
      acc.w = fmaf(v[u], x[u].w, acc.w);
      accb = fmaf(v[u], xb[u], accb);
    }
  }
  // the two half-warps' row sums, then the 8 warps in a fixed order
  acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 16);
  acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 16);
  acc.z += __shfl_xor_sync(0xffffffffu, acc.z, 16);
  acc.w += __shfl_xor_sync(0xffffffffu, acc.w, 16);
  accb += __shfl_xor_sync(0xffffffffu, accb, 16);
  if (h == 0) {
    red[warp][4 * c4] = acc.x;
    red[warp][4 * c4 + 1] = acc.y;
    red[warp][4 * c4 + 2] = acc.z;
    red[warp][4 * c4 + 3] = acc.w;
    if (c4 == 0) red[warp][64] = accb;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 65; c += 256) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += red[w][c];
    part[(int64_t)blockIdx.x * 65 + c] = alpha * t;
  }
}

// loss partials of the per-tile CTAs -> one value; a fixed strided order per
// thread and a fixed shuffle / shared-memory tree (deterministic)
__global__ void loss_fold_kernel(const float* __restrict__ part, int n, float* dst) {
  __shared__ float ws[8];
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    *dst = t;
  }
}

}  // namespace ctc

static bool wgrad_enabled() {
  const char* e = getenv("CACTO_CRITIC_WGRAD");  // 0: the 3xTF32 GEMM reductions (A/B measurements)
  return !e || atoi(e) != 0;
}

bool critic_tc_enabled() {
  const char* e = getenv("CACTO_CRITIC_TC");  // 0: fused SIMT kernel (A/B measurements)
  return !e || atoi(e) != 0;
}

// eligible: fp32, 3 hidden layers of padded width 64, input n + 1 <= 16, target
// (if any) of the same shape; the batch large enough to fill the GPU with tiles
bool critic_tc_eligible(const cacto_mlp_t* c, const cacto_mlp_t* tgt, int64_t rows) {
  if (!critic_tc_enabled() || !c || c->dtype != CACTO_F32 || c->n_layers != 4 || c->hp != 64 || c->sizes[0] > 16 ||
      c->sizes[4] != 1)
    return false;
  if (tgt && (tgt->dtype != CACTO_F32 || tgt->n_layers != 4 || tgt->hp != 64 || tgt->sizes[0] != c->sizes[0] ||
              tgt->activation != c->activation))
    return false;
  const char* e = getenv("CACTO_CRITIC_TC_MIN");  // minimum batch (default: 32 tiles per SM-wave)
  const int64_t min_rows = e ? atoll(e) : (int64_t)8192;
  return rows >= min_rows;
}

size_t critic_tc_workspace_bytes(const cacto_mlp_t* c, int64_t rows) {
  NetShape sh = shape_of(*c);
  return ctc::plan2(rows > 0 ? rows : 1, layer_offsets(sh).total).total;
}

// a second stream (per device, created on first use outside stream capture) on
// which the output-row reduction and the loss fold run beside wgrad_kernel: they
// only need the per-sample factors, and wgrad leaves SM resources for their CTAs
// (fork / join by events, so the pair is captured into the update graph too)
struct AuxStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static AuxStream* aux_stream(cudaStream_t st) {
  static AuxStream aux[16];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
  AuxStream& x = aux[dev];
  if (!x.s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
    if (cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) != cudaSuccess) {
      x.s = nullptr;
      return nullptr;
    }
  }
  return &x;
}

extern "C" int cacto_debug_ctc_timeline(unsigned long long* host) {
#if CACTO_CTC_TIMELINE
  return cudaMemcpyFromSymbol(host, g_ctc_tl, sizeof(g_ctc_tl)) == cudaSuccess ? 0 : 1;
#else
  (void)host;
  return -1;
#endif
}

int critic_tc_loss(const cacto_mlp_t* c, const cacto_mlp_t* tgt, const cacto_batch_t* bt, double k_s, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  using namespace ctc;
  NetShape sh = shape_of(*c);
  LayerOffsets lo = layer_offsets(sh);
  const int64_t B = bt->rows;
  Plan2 p = plan2(B, lo.total);
  if (ws_bytes < p.total) return set_error(CACTO_EVALUE, "critic_loss(tc): workspace too small");
  char* w = (char*)ws;
  float* slot = (float*)w;
  cudaMemsetAsync(slot, 0, (size_t)(lo.total + 1) * 4, st);
  Args a{};
  a.b.idx = bt->idx;
  a.b.cycle = bt->cycle;
  a.b.idx_stride = bt->idx_stride;
  a.b.xa = (const float*)bt->xa;
  a.b.v_bar = (const float*)bt->v_bar;
  a.b.v_bar_x = (const float*)bt->v_bar_x;
  a.b.xa_plus_k = (const float*)bt->xa_plus_k;
  a.b.rows = B;
  a.b.n = bt->n;
  a.b.t_max = bt->t_max;
  a.critic = (const float*)c->params;
  a.target = tgt ? (const float*)tgt->params : nullptr;
  a.nc = net_const<float>(*c);
  a.nc_t = tgt ? net_const<float>(*tgt) : a.nc;
  a.ip = sh.ip;
  a.k_s = (float)k_s;
  a.inv_denom = 1.f / (float)(bt->denom > 0 ? bt->denom : B);
  for (int l = 0; l < 3; ++l) a.GZ[l] = (float*)(w + p.off_gz[l]);
  for (int l = 0; l < 4; ++l) a.UA[l] = (float*)(w + p.off_ua[l]);
  a.V3 = (float*)(w + p.off_v3);
  a.lossp = (float*)(w + p.off_lossp);
  const int64_t ntiles = (B + TILE - 1) / TILE;
  const int grid = (int)(ntiles < num_sms() ? ntiles : num_sms());
  a.img = (const unsigned char*)(w + p.off_img);
  if (c->activation == CACTO_ACT_ELU)
    critic_tc_image_kernel<CACTO_ACT_ELU><<<32, 256, 0, st>>>(a, (unsigned char*)(w + p.off_img));
  else
    critic_tc_image_kernel<CACTO_ACT_TANH><<<32, 256, 0, st>>>(a, (unsigned char*)(w + p.off_img));
  auto kern = c->activation == CACTO_ACT_ELU ? critic_tc_kernel<CACTO_ACT_ELU> : critic_tc_kernel<CACTO_ACT_TANH>;
  if (!ensure_smem((const void*)kern, BYTES))
    return set_error(CACTO_ECUDA, "critic_loss(tc): %u B of shared memory not available", BYTES);
  kern<<<grid, NTHR, BYTES, st>>>(a);
  int rc = check_launch("critic_tc_kernel");
  if (rc) return rc;
  // the output-row reduction + loss fold on the aux stream, beside the layer reductions
  // (measured: B = 8192 0.087 -> 0.081 ms; at B = 65,536 the two HBM-bound
  // reductions contend and the serial order is 1 % faster, so large batches keep it)
  AuxStream* aux = B <= 16384 ? aux_stream(st) : nullptr;
  cudaStream_t so = aux ? aux->s : st;
  if (aux) {
    cudaEventRecord(aux->fork, st);
    cudaStreamWaitEvent(so, aux->fork, 0);
  }
  const int64_t K2 = 2 * B;
  ctc::PartSet ps{};
  ps.p[3] = (const float*)(w + p.off_part[3]);
  ps.stride[3] = 65;
  {
    int S = 4 * num_sms();
    const int64_t maxS = (int64_t)(p.part_bytes[3] / (65 * 4));
    if (S > maxS) S = (int)maxS;
    const int64_t chunk = (K2 + S - 1) / S;
    S = (int)((K2 + chunk - 1) / chunk);
    ctc::out_row_grad_kernel<<<S, 256, 0, so>>>(a.V3, a.UA[3], K2, chunk, a.inv_denom, (float*)(w + p.off_part[3]));
    ps.splits[3] = S;
  }
  loss_fold_kernel<<<1, 256, 0, so>>>(a.lossp, grid, slot + lo.total);
  if (aux) cudaEventRecord(aux->join, so);
  // batch reductions: per layer ONE GEMM over K = 2B gives the weight gradient and,
  // from the bias column, the bias gradient; the output row w_3 and b_3 from a
  // 1-row GEMM with the [1 ; -2 e_v] factor.  Results (scaled by 1/denom) land in
  // small [rows][N] tiles that one kernel adds into the padded gradient slot.
  const int ncol[4] = {17, 65, 65, 65};
  const int wpad[4] = {20, 68, 68, 68};
  if (wgrad_enabled()) {
    // layers 0..2: wgrad_kernel, one wave of CTAs split by HBM bytes per layer
    ctc::WgradArgs g{};
    const double bytes[3] = {64.0 + 17.0, 64.0 + 65.0, 64.0 + 65.0};
    const int sms = num_sms();
    int c0 = 0;
    for (int l = 0; l < 3; ++l) {
      rc = ctc::wg_map(&g.tg[l], a.GZ[l], K2, HP, HP, ctc::WG_KB);
      if (!rc) rc = ctc::wg_map(&g.tu[l], a.UA[l], K2, wpad[l], wpad[l], ctc::WG_KB);
      if (rc) return rc;
      g.uw[l] = wpad[l];
      g.ncol[l] = ncol[l];
      g.nmma[l] = l == 0 ? 32 : 80;
      int S = (int)(sms * bytes[l] / (bytes[0] + bytes[1] + bytes[2]));
      if (S < 1) S = 1;
      int64_t chunk = (K2 + S - 1) / S;
      chunk = (chunk + ctc::WG_KB - 1) / ctc::WG_KB * ctc::WG_KB;
      S = (int)((K2 + chunk - 1) / chunk);
      g.chunk[l] = chunk;
      g.cta0[l] = c0;
      c0 += S;
      g.part[l] = (float*)(w + p.off_part[l]);
      ps.p[l] = g.part[l];
      ps.stride[l] = (int64_t)HP * ncol[l];
      ps.splits[l] = 2 * S;  // hi-row and lo-row partials of every CTA
    }
    g.cta0[3] = c0;
    g.K2 = K2;
    g.alpha = a.inv_denom / (ctc::WG_SB * ctc::WG_SB);
    if (!ensure_smem((const void*)ctc::wgrad_kernel, ctc::WG_SMEM))
      return set_error(CACTO_ECUDA, "critic_loss(tc): wgrad shared memory not available");
    ctc::wgrad_kernel<<<c0, ctc::WG_THREADS, ctc::WG_SMEM, st>>>(g);
    rc = check_launch("wgrad_kernel");
    if (rc) return rc;
  } else {
    for (int l = 0; l < 3; ++l) {
      ps.p[l] = (const float*)(w + p.off_part[l]);
      ps.stride[l] = (int64_t)HP * ncol[l];
      rc = gemm_tf32_partials(HP, ncol[l], (int)(2 * B), a.GZ[l], 1, HP, a.UA[l], 1, wpad[l], a.inv_denom, 3,
                              w + p.off_part[l], p.part_bytes[l], &ps.splits[l], st);
      if (rc) return rc;
    }
  }
  if (aux) cudaStreamWaitEvent(st, aux->join, 0);
  if (CACTO_CTC_SCATTER_COALESCED && wgrad_enabled()) {
    const int n_thr = ctc::HP * 17 + 2 * ctc::HP * 65;  // the wgrad partials' [rows][ncol] entries
    const int total = (n_thr + 31) / 32 * 32 + (ctc::HP + 1) * 32;
    ctc::reduce_scatter_coalesced_kernel<<<(total + 255) / 256, 256, 0, st>>>(
        ps, lo.cols[0], slot, lo.w[0], lo.b[0], lo.w[1], lo.b[1], lo.w[2], lo.b[2], lo.w[3], lo.b[3],
        (n_thr + 31) / 32 * 32);
  } else {
    const int items = ctc::scatter_items(lo.cols[0]);
    ctc::reduce_scatter_grads_kernel<<<(items * 32 + 255) / 256, 256, 0, st>>>(
        ps, lo.cols[0], slot, lo.w[0], lo.b[0], lo.w[1], lo.b[1], lo.w[2], lo.b[2], lo.w[3], lo.b[3]);
  }
  return check_launch("critic_tc reductions");
}

}  // namespace cacto
