// rollout_tc.cu -- K1 on the tensor cores: the fused closed-loop actor rollout
// (nets.actor_rollout, nets.py:403-423) with every policy layer issued as
// tcgen05.mma (kind::tf32, 3xTF32 for fp32 accuracy) into TMEM, and the
// activation / head / dynamics / running-cost work done by the thread that owns
// the start.
//
// CTA = NT tiles of 128 starts (TMEM lane = start) + one MMA warp.
//   TMEM per tile (2*HP columns): D [HP] accumulator | A_hi [HP] activations.
//   Shared memory: weights (hi and lo, K-major SW128) for the whole horizon, and
//   per tile the A_lo activations (K-major SW128).
//   Per layer and tile the MMA warp issues, for each k-step of 8,
//       D += A_hi(TMEM) W_hi + A_hi(TMEM) W_lo + A_lo(smem) W_hi
//   (3xTF32: x = hi + lo with hi = rna_tf32(x)) and commits to the tile's
//   mbarrier.  The tile's 4 epilogue warps (warp w -> TMEM lanes 32(w%4)..+31)
//   then tcgen05.ld the D row, add the bias, apply the activation, write hi back
//   to TMEM (tcgen05.st) and lo to shared memory, and arrive.  After the output
//   layer the owner thread applies the head, accumulates the stage cost in
//   NumPy's pairwise order, steps the dynamics and writes the next normalised
//   input row.
// The NT tiles are in flight together, so one tile's epilogue overlaps the other
// tiles' MMAs and hand-off latencies.  Nothing but the outputs touches HBM.
#include <stdlib.h>

#include "net.cuh"
#include "rollout.cuh"
#include "systems.cuh"
#include "tc.cuh"

namespace cacto {

namespace rtc {

constexpr int TILE = 128;
constexpr int NOUT = 16;  // output-layer MMA width (m <= 8 used)

CACTO_HD constexpr int kin_of(int n) { return ((n + 1) + 7) / 8 * 8; }  // input K (8 or 16)

// shared-memory plan (bytes, from a 1024-aligned base)
template <int HP, int NT>
struct Plan {
  static constexpr int KB = HP / 32;                // 32-wide K blocks of a hidden operand
  static constexpr uint32_t ALO = KB * TILE * 128;  // per tile: A_lo [128][HP] SW128
  static constexpr uint32_t W0 = HP * 128;          // [HP][32] one block
  static constexpr uint32_t WH = KB * HP * 128;     // [HP][HP]
  static constexpr uint32_t WO = KB * NOUT * 128;   // [16][HP]
  static constexpr uint32_t off_alo(int t) { return t * ALO; }
  static constexpr uint32_t off_w0 = NT * ALO;          // hi, lo
  static constexpr uint32_t off_wh = off_w0 + 2 * W0;   // (hi, lo) x (nh - 1), nh <= 3
  static constexpr uint32_t off_wo = off_wh + 2 * 2 * WH;
  static constexpr uint32_t off_bias = off_wo + 2 * WO;  // fp32 [3][HP] + [NOUT]
  static constexpr uint32_t bytes = off_bias + (3 * HP + NOUT) * 4 + 1024;
  static constexpr uint32_t TMEM_COLS = NT * 2 * HP <= 128 ? 128 : (NT * 2 * HP <= 256 ? 256 : 512);
  static_assert(NT * 2 * HP <= 512, "TMEM: 2*HP columns per tile");
};

// byte offset of element (r, c) in a K-major SW128 operand of `rows` rows
CACTO_HD uint32_t sw128(int rows, int r, int c) {
  const int kb = c >> 5, cc = c & 31;
  return (uint32_t)(kb * rows * 128 + r * 128 + ((((cc >> 2) ^ (r & 7))) << 4) + (cc & 3) * 4);
}

// stage a row-major [rows][cols] (stride) fp32 matrix as hi/lo K-major SW128
// operands of `rrows` x kcols (zero padded)
CACTO_D void stage_w(unsigned char* hi, unsigned char* lo, const float* src, int rows, int cols, int stride,
                     int rrows, int kcols, int tid, int nthr) {
  for (int e = tid; e < rrows * kcols; e += nthr) {
    const int r = e / kcols, c = e - r * kcols;
    const float v = (r < rows && c < cols) ? src[(int64_t)r * stride + c] : 0.f;
    const uint32_t o = sw128(rrows, r, c);
    const float vh = tc::tf32_rna(v);
    *reinterpret_cast<float*>(hi + o) = vh;
    *reinterpret_cast<float*>(lo + o) = v - vh;
  }
}

// one layer of one tile: KSTEPS k-steps of hi*hi + hi*lo + lo*hi; later k-steps'
// descriptors are the base descriptors plus constant start offsets (16-B units)
template <int KSTEPS, int WROWS>
CACTO_D void issue_layer(uint32_t dcol, uint32_t ahi_t, uint64_t alo, uint64_t whi, uint64_t wlo, uint32_t idesc) {
#pragma unroll
  for (int kk = 0; kk < KSTEPS; ++kk) {
    const uint64_t ao = (uint64_t)((((kk >> 2) * TILE * 128) + (kk & 3) * 32) >> 4);
    const uint64_t wo = (uint64_t)((((kk >> 2) * WROWS * 128) + (kk & 3) * 32) >> 4);
    tc::mma_tf32_ts_elect(dcol, ahi_t + (uint32_t)(kk * 8), whi + wo, idesc, kk > 0 ? 1u : 0u);
    tc::mma_tf32_ts_elect(dcol, ahi_t + (uint32_t)(kk * 8), wlo + wo, idesc, 1u);
    tc::mma_tf32_elect(dcol, alo + ao, whi + wo, idesc, 1u);
  }
}

}  // namespace rtc

// branch-free forward activation (ELU through the SFU exponential, like the SIMT
// path's act_fast); straight-line code lets the scheduler interleave columns
template <int ACT>
CACTO_D float act_tc(float z) {
  if constexpr (ACT == CACTO_ACT_ELU) {
    const float e = tc::ex2_ftz(fminf(z, 0.f) * 1.4426950408889634f) - 1.f;
    return z > 0.f ? z : e;
  }
  return tanhf(z);
}

template <int SYS, int HP, int NT, int SPLIT, int ACT>
__global__ void __launch_bounds__(NT * SPLIT * 128 + 32, 1) rollout_tc_kernel(const RolloutArgs<float> a) {
  using namespace rtc;
  using PL = Plan<HP, NT>;
  constexpr int n = SysDims<SYS>::n;
  constexpr int m = SysDims<SYS>::m;
  constexpr int KIN = kin_of(n);
  constexpr int IP = (n + 1) <= 8 ? 8 : ((n + 1) <= 16 ? 16 : 32);  // padded W0 row stride
  constexpr int WPT = 4 * SPLIT;       // epilogue warps per tile (SPLIT per TMEM lane quadrant)
  constexpr int COLS = HP / SPLIT;     // hidden columns per epilogue warp
  constexpr int CH = COLS < 32 ? COLS : 32;
  constexpr int NTHR = NT * WPT * 32 + 32;
  constexpr int MMA_WARP = NT * WPT;
  static_assert(COLS >= 16, "at least 16 columns per epilogue warp");
  static_assert(KIN <= 16 && m <= 8, "tensor-core rollout: n + 1 <= 16, m <= 8");

  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[NT], done_bar[NT];
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_kmax;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nh = a.nh;

  // ---- weights -> shared memory (hi/lo, SW128), biases (fp32) ----------------------
  {
    const float* P = a.params;
    const int64_t b0 = (int64_t)HP * IP;
    stage_w(base + PL::off_w0, base + PL::off_w0 + PL::W0, P, HP, n + 1, IP, HP, 32, threadIdx.x, NTHR);
    float* bias = reinterpret_cast<float*>(base + PL::off_bias);
    for (int c = threadIdx.x; c < HP; c += NTHR) bias[c] = P[b0 + c];
    int64_t off = b0 + HP;
    for (int i = 1; i < nh; ++i) {
      unsigned char* hi = base + PL::off_wh + (uint32_t)(2 * (i - 1)) * PL::WH;
      stage_w(hi, hi + PL::WH, P + off, HP, HP, HP, HP, HP, threadIdx.x, NTHR);
      for (int c = threadIdx.x; c < HP; c += NTHR) bias[i * HP + c] = P[off + (int64_t)HP * HP + c];
      off += (int64_t)HP * HP + HP;
    }
    stage_w(base + PL::off_wo, base + PL::off_wo + PL::WO, P + off, m, HP, HP, NOUT, HP, threadIdx.x, NTHR);
    for (int c = threadIdx.x; c < NOUT; c += NTHR) bias[3 * HP + c] = c < m ? P[off + (int64_t)m * HP + c] : 0.f;
  }
  if (threadIdx.x == 0) {
    for (int t = 0; t < NT; ++t) {
      tc::mbar_init(&full_bar[t], WPT);
      tc::mbar_init(&done_bar[t], 1);
    }
    s_kmax = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) tc::tmem_alloc(&tmem_base_sh, PL::TMEM_COLS);
  tc::fence_async_smem();  // staged weights -> async proxy
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t sbase = saddr(base);

  // ---- roles: epilogue warp w < MMA_WARP serves tile g = w / WPT, TMEM lanes
  //      32(w%4)..+31 = starts r of the tile, hidden columns [part*COLS, +COLS);
  //      the part-0 warp of a quadrant owns the starts' state -------------------------
  const bool epi = warp < MMA_WARP;
  const int g = warp / WPT;
  const int q = warp & 3;
  const int part = (warp % WPT) >> 2;
  const int r = (q << 5) + lane;
  const int64_t gi = ((int64_t)blockIdx.x * NT + g) * TILE + r;
  const bool owner = epi && part == 0 && gi < a.N;
  float x[n];
  int t0 = 0, T_i = 0;
  PairwiseSum<float> acc;
#pragma unroll
  for (int c = 0; c < n; ++c) x[c] = 0.f;
  if (owner) {
#pragma unroll
    for (int c = 0; c < n; ++c) x[c] = (float)a.x0[gi * n + c];
    t0 = a.t0 ? a.t0[gi] : a.t0_scalar;
    T_i = a.t_hor > 0 ? a.t_hor : (a.sys.t_max - t0);
    acc.init(T_i + 1);
    if (a.X) {
#pragma unroll
      for (int c = 0; c < n; ++c) a.X[gi * (int64_t)(a.t_stride + 1) * n + c] = x[c];
    }
    atomicMax(&s_kmax, T_i);
  }
  __syncthreads();
  const int kmax = s_kmax;

  if (epi) {
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(g * 2 * HP);
    const uint32_t t_d = lane_base, t_ahi = lane_base + HP;  // this thread's D / A_hi row
    const uint32_t alo = sbase + PL::off_alo(g);
    const uint32_t bias_s = sbase + PL::off_bias;
    uint32_t pd = 0;
    auto put_lo4 = [&](int c, float v0, float v1, float v2, float v3) {
      sts4(alo + sw128(TILE, r, c), V4<float>{{v0, v1, v2, v3}});
    };
    auto write_input = [&](int k) {
      if (part != 0) return;
      float v[KIN], hv[KIN];
#pragma unroll
      for (int c = 0; c < KIN; ++c) v[c] = 0.f;
      if (owner) {
#pragma unroll
        for (int c = 0; c < n; ++c) v[c] = (x[c] - a.nc.in_center[c]) / a.nc.in_half[c];
        v[n] = ((float)(t0 + k) - a.nc.in_center[n]) / a.nc.in_half[n];
      }
#pragma unroll
      for (int c = 0; c < KIN; ++c) hv[c] = tc::tf32_rna(v[c]);
      if constexpr (KIN == 8) tc::tmem_st8(t_ahi, hv);
      else tc::tmem_st16(t_ahi, hv);
#pragma unroll
      for (int c = 0; c < KIN; c += 4)
        put_lo4(c, v[c] - hv[c], v[c + 1] - hv[c + 1], v[c + 2] - hv[c + 2], v[c + 3] - hv[c + 3]);
    };
    auto handoff = [&]() {
      tc::tmem_wait_st();
      tc::tc_fence_before();
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full_bar[g]);
    };
    auto wait_done = [&]() {
      tc::mbar_wait_sleep(&done_bar[g], pd);
      pd ^= 1;
      tc::tc_fence_after();
    };
    if (kmax > 0) {
      write_input(0);
      handoff();
    }
    for (int k = 0; k < kmax; ++k) {
      for (int l = 0; l < nh; ++l) {  // hidden layers
        wait_done();
#pragma unroll
        for (int cc0 = 0; cc0 < COLS; cc0 += CH) {
          const int c0 = part * COLS + cc0;
          float z[CH], hv[CH];
          if constexpr (CH == 32) tc::tmem_ld32_wait(t_d + (uint32_t)c0, z);
          else tc::tmem_ld16_wait(t_d + (uint32_t)c0, z);
          const uint32_t bl = bias_s + (uint32_t)((l * HP + c0) * 4);
#pragma unroll
          for (int c = 0; c < CH; c += 4) {
            const V4<float> b4 = lds4(bl + c * 4, (float*)nullptr);
            float v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              v[j] = act_tc<ACT>(z[c + j] + b4.v[j]);
              hv[c + j] = tc::tf32_rna(v[j]);
            }
            put_lo4(c0 + c, v[0] - hv[c], v[1] - hv[c + 1], v[2] - hv[c + 2], v[3] - hv[c + 3]);
          }
          if constexpr (CH == 32) tc::tmem_st32(t_ahi + (uint32_t)c0, hv);
          else tc::tmem_st16(t_ahi + (uint32_t)c0, hv);
        }
        handoff();
      }
      // output layer -> head, cost, dynamics
      wait_done();
      float o[16];
      if (part == 0) tc::tmem_ld16_wait(t_d, o);
      if (owner && k < T_i) {
        const float* bias = reinterpret_cast<const float*>(base + PL::off_bias);
        float u[m];
#pragma unroll
        for (int j = 0; j < m; ++j) u[j] = head_value(a.head, a.nc, j, o[j] + bias[3 * HP + j]);
        if (a.U) {
#pragma unroll
          for (int j = 0; j < m; ++j) a.U[(gi * a.t_stride + k) * m + j] = u[j];
        }
        float sc = 0.f;
        if (a.has_cost) sc = stage_cost<SYS>(a.sys, a.cost, x, u);
        acc.add(k, sc);
        if (a.SC) a.SC[gi * (int64_t)(a.t_stride + 1) + k] = sc;
        float xn[n];
        step<SYS>(a.sys, x, u, xn);
#pragma unroll
        for (int c = 0; c < n; ++c) x[c] = xn[c];
        if (a.X) {
#pragma unroll
          for (int c = 0; c < n; ++c) a.X[(gi * (int64_t)(a.t_stride + 1) + k + 1) * n + c] = x[c];
        }
      }
      if (k + 1 < kmax) {
        write_input(k + 1);
        handoff();
      }
    }
    if (owner) {
      const float term = a.has_cost ? terminal_cost<SYS>(a.sys, a.cost, x) : 0.f;
      acc.add(T_i, term);
      if (a.SC) a.SC[gi * (int64_t)(a.t_stride + 1) + T_i] = term;
      if (a.C) a.C[gi] = acc.res;
    }
  } else {
    // ---- MMA issuer (whole warp converged; elect.sync picks the issuing lane) ----------
    const uint32_t idesc_h = tc::idesc_tf32(HP, 0, 0), idesc_o = tc::idesc_tf32(NOUT, 0, 0);
    auto desc = [&](uint32_t off) { return tc::make_desc(sbase + off, 16, 1024, 2); };
    const uint64_t w0h = desc(PL::off_w0), w0l = desc(PL::off_w0 + PL::W0);
    const uint64_t woh = desc(PL::off_wo), wol = desc(PL::off_wo + PL::WO);
    uint32_t pf[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) pf[t] = 0;
    for (int k = 0; k < kmax; ++k) {
      for (int l = 0; l <= nh; ++l) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          tc::mbar_wait_sleep(&full_bar[t], pf[t]);
          pf[t] ^= 1;
          tc::tc_fence_after();
          const uint32_t dcol = tmem + (uint32_t)(t * 2 * HP), ahi = dcol + HP;
          const uint64_t al = desc(PL::off_alo(t));
          if (l == 0) {
            issue_layer<KIN / 8, HP>(dcol, ahi, al, w0h, w0l, idesc_h);
          } else if (l < nh) {
            const uint32_t wo = PL::off_wh + (uint32_t)(2 * (l - 1)) * PL::WH;
            issue_layer<HP / 8, HP>(dcol, ahi, al, desc(wo), desc(wo + PL::WH), idesc_h);
          } else {
            issue_layer<HP / 8, NOUT>(dcol, ahi, al, woh, wol, idesc_o);
          }
          tc::tc_commit_elect(&done_bar[t]);
          __syncwarp();
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) tc::tmem_dealloc(tmem, PL::TMEM_COLS);
}

template <int SYS, int HP, int NT>
static int launch_rollout_tc_nt(const RolloutArgs<float>& a, cudaStream_t st) {
  using PL = rtc::Plan<HP, NT>;
  // 4 tiles: one epilogue warp per lane quadrant; fewer tiles: the columns are
  // split over more warps (shorter per-layer epilogue latency), 544 threads max
  constexpr int SPLIT = (NT == 4 || HP == 32) ? 1 : 4 / NT;
  auto kern = a.act == CACTO_ACT_ELU ? rollout_tc_kernel<SYS, HP, NT, SPLIT, CACTO_ACT_ELU>
                                     : rollout_tc_kernel<SYS, HP, NT, SPLIT, CACTO_ACT_TANH>;
  if (!ensure_smem((const void*)kern, PL::bytes))
    return set_error(CACTO_ECUDA, "rollout_tc: %u B of shared memory not available", PL::bytes);
  const int64_t per = (int64_t)NT * rtc::TILE;
  const int64_t blocks = (a.N + per - 1) / per;
  kern<<<(unsigned)blocks, NT * SPLIT * 128 + 32, PL::bytes, st>>>(a);
  return check_launch("rollout_tc_kernel");
}

static int tc_tiles_override() {
  const char* e = getenv("CACTO_ROLLOUT_TC_TILES");  // 1 / 2 / 4 (measurements)
  return e ? atoi(e) : 0;
}

// eligible: fp32, n + 1 <= 16, m <= 8, 1..3 hidden layers of width 32 or 64.
// Tiles per CTA: the most that still give (nearly) every SM a CTA -- more tiles
// in flight hide more latency, fewer CTAs than SMs leave SMs idle.
template <int SYS, int HP>
int launch_rollout_tc(const RolloutArgs<float>& a, cudaStream_t st) {
  int nt = tc_tiles_override();
  if (nt != 1 && nt != 2 && nt != 4) {
    const int64_t tiles = (a.N + rtc::TILE - 1) / rtc::TILE;
    const int64_t sms = num_sms();
    nt = tiles >= 4 * sms * 3 / 4 ? 4 : (tiles >= 2 * sms ? 2 : 1);
  }
  if (nt == 4) return launch_rollout_tc_nt<SYS, HP, 4>(a, st);
  if (nt == 2) return launch_rollout_tc_nt<SYS, HP, 2>(a, st);
  return launch_rollout_tc_nt<SYS, HP, 1>(a, st);
}

bool rollout_tc_enabled() {
  const char* e = getenv("CACTO_ROLLOUT_TC");  // 0: SIMT rollout (A/B measurements)
  return !e || atoi(e) != 0;
}

#define CACTO_RTC_INST(SYSK)                                                          \
  template int launch_rollout_tc<SYSK, 32>(const RolloutArgs<float>&, cudaStream_t); \
  template int launch_rollout_tc<SYSK, 64>(const RolloutArgs<float>&, cudaStream_t);
CACTO_RTC_INST(CACTO_SYS_TOY1D)
CACTO_RTC_INST(CACTO_SYS_POINTMASS)
CACTO_RTC_INST(CACTO_SYS_DUBINS)
CACTO_RTC_INST(CACTO_SYS_MANIPULATOR3)
CACTO_RTC_INST(CACTO_SYS_ALIENGO_LIPM)
#undef CACTO_RTC_INST

}  // namespace cacto
