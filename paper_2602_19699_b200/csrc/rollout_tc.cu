// rollout_tc.cu -- K1 on the tensor cores: the fused closed-loop actor rollout
// (nets.actor_rollout, nets.py:403-423) with every policy layer issued as
// tcgen05.mma and the activation / head / dynamics / running-cost work done by
// the thread that owns the start.
//
// Arithmetic: fp32 results from fp16 tensor-core products ("3xFP16"): every
// operand x = hi + lo with hi = fp16(x), lo = fp16(x - hi) (11 + 11 significant
// bits), and each layer issues hi*hi + hi*lo + lo*hi with fp32 accumulation --
// the precision of the 3xTF32 split at twice the MMA rate (kind::f16, K = 16 per
// instruction).  Weights are pre-scaled by powers of two (and log2 e for ELU) so
// their lo parts stay normal fp16 numbers.
//
// CTA = NT tiles of 128 starts (TMEM lane = start) + one MMA warp.
//   TMEM per tile (2*HP columns): D [HP] fp32 accumulator | A_hi [HP/2] | A_lo
//   [HP/2] (fp16 pairs).  Shared memory holds only the weights (hi/lo, K-major
//   SW128) and the scaled biases, for the whole horizon.
//   Per layer and tile the MMA warp issues, for each k-step of 16, the three
//   products with A read from TMEM, and commits to the tile's mbarrier.  The
//   tile's epilogue warps (warp w -> TMEM lanes 32(w%4)..+31) tcgen05.ld the D
//   row, apply the activation, tcgen05.st the split activations as the next
//   layer's A, pre-load D with the next layer's bias, and arrive.  After the
//   output layer the owner thread applies the head, accumulates the stage cost
//   in NumPy's pairwise order, steps the dynamics and writes the next input.
//
// ELU layers: the accumulator holds D = 8 log2(e) z, so
// ELU(z) = max(D,0)/(8 log2 e) + (ex2(min(D,0)/8) - 1): two FMNMX, one FMUL, one
// MUFU, one FADD, one FFMA per element, branch-free.
#include <cuda_fp16.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "net.cuh"
#include "rollout.cuh"
#include "systems.cuh"
#include "tc.cuh"
#include "tcmlp.cuh"

#ifndef CACTO_RTC_SELF
#define CACTO_RTC_SELF 1
#endif
#ifndef CACTO_RTC_SKIP_IDLE
#define CACTO_RTC_SKIP_IDLE 1
#endif
#ifndef CACTO_RTC_CORE_OUT
#define CACTO_RTC_CORE_OUT 1
#endif

namespace cacto {

#if CACTO_RTC_TIMELINE
// clock64 timeline of one CTA's tile leaders (profiles/k1_timeline.py): [tile][pass
// 20..27][layer 0..3][event: epilogue end, tile joined, issue end, MMA seen done]
__device__ unsigned long long g_rtc_tl[4][8][4][4];
#define RTC_TL(P, L, E)                                                                        \
  do {                                                                                         \
    if (blockIdx.x == 10 && lane == 0 && (P) >= 20 && (P) < 28 && (L) < 4)                    \
      g_rtc_tl[g][(P)-20][L][E] = clock64();                                                   \
  } while (0)
#else
#define RTC_TL(P, L, E) \
  do {                  \
  } while (0)
#endif

// threads of a CTA: NT tiles x 4 SPLIT epilogue warps (+ the MMA warp unless a
// leader warp of each tile issues its own MMAs)
template <int NT, int SPLIT>
constexpr int rtc_threads() { return NT * SPLIT * 128 + (CACTO_RTC_SELF ? 0 : 32); }

template <int SYS, int HP, int NT, int SPLIT, int ACT>
__global__ void __launch_bounds__(rtc_threads<NT, SPLIT>(), 1) rollout_tc_kernel(const RolloutArgs<float> a) {
  using namespace rtc;
  using PL = Plan<HP>;
  using TM = Tmem<HP, NT>;
  using AF = ActTC<ACT>;
  constexpr int n = SysDims<SYS>::n;
  constexpr int m = SysDims<SYS>::m;
  constexpr int IP = (n + 1) <= 8 ? 8 : ((n + 1) <= 16 ? 16 : 32);  // padded W0 row stride
  constexpr int WPT = 4 * SPLIT;    // epilogue warps per tile (SPLIT per TMEM lane quadrant)
  constexpr int COLS = HP / SPLIT;  // accumulator columns per epilogue warp
  constexpr int NTHR = rtc_threads<NT, SPLIT>();
  constexpr int MMA_WARP = NT * WPT;  // == the warp count when the tiles self-issue
  static_assert(n + 1 <= KIN && m <= 8 && HP <= 64, "tensor-core rollout: n + 1 <= 16, m <= 8, HP <= 64");
  static_assert(COLS == 16 || COLS == 32 || COLS == 64, "16, 32 or 64 columns per epilogue warp");
  // output layer on the CUDA cores (m <= 2, one warp per lane quadrant): the last
  // hidden epilogue accumulates o = W_out v + b from the fp32 activations it just
  // computed -- no output-layer MMAs, no hand-off / completion round trip, no TMEM
  // traffic for that layer (fp32 FMAs: more accurate than the 3xFP16 products)
  constexpr int MO = (CACTO_RTC_CORE_OUT && SPLIT == 1 && m <= 2) ? m : 0;
  constexpr uint32_t WF = (uint32_t)(MO * HP + 4) * 4;  // fp32 W_out [MO][HP] + b [MO] per net

  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[NT], done_bar[NT];
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_kmax;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nh = a.nh;
  const int n_pre = a.n_pre;

  // ---- networks -> shared-memory slots: 0 = actor, 1.. = the scoring nets --------
  stage_net<HP, IP, AF>(base, a.params, nh, n + 1, m, threadIdx.x, NTHR);
  for (int p = 0; p < n_pre; ++p)
    stage_net<HP, IP, AF>(base + (p + 1) * PL::SLOT, a.pre_params[p], nh, n + 1, 1, threadIdx.x, NTHR);
  // the bias MMAs' ones block, after the pairwise partial sums
  const uint32_t off_ones = (uint32_t)(1 + n_pre) * PL::SLOT + (uint32_t)NTHR * 9 * 4;
  if (CACTO_RTC_BIAS_MMA) stage_ones(base + off_ones, threadIdx.x, NTHR);
  const uint32_t off_wf = off_ones + ONES_BYTES;
  if constexpr (MO > 0) {
    // fp32 output layers (unscaled; rows past a net's outputs are zero)
    const int64_t wo_off = (int64_t)HP * IP + HP + (int64_t)(nh - 1) * (HP * HP + HP);
    for (int p = 0; p <= n_pre; ++p) {
      const float* P = p == 0 ? a.params : a.pre_params[p - 1];
      const int outs = p == 0 ? m : 1;
      float* dst = (float*)(base + off_wf + (uint32_t)p * WF);
      for (int e = threadIdx.x; e < MO * HP + MO; e += NTHR) {
        float v = 0.f;
        if (e < MO * HP) {
          const int j = e / HP;
          if (j < outs) v = P[wo_off + e];
        } else if (e - MO * HP < outs) {
          v = P[wo_off + (int64_t)outs * HP + (e - MO * HP)];
        }
        dst[e] = v;
      }
    }
  }
  if (threadIdx.x == 0) {
    for (int t = 0; t < NT; ++t) {
      tc::mbar_init(&full_bar[t], WPT);
      tc::mbar_init(&done_bar[t], 1);
    }
    s_kmax = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int alloc_warp = CACTO_RTC_SELF ? 0 : MMA_WARP;
  if (warp == alloc_warp) tc::tmem_alloc(&tmem_base_sh, TM::COLS);
  tc::fence_async_smem();  // staged weights -> async proxy
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t sbase = saddr(base);

  // ---- MMA issue of layer l of pass P for tile t (whole warp, converged) -----------
  const uint32_t idesc_h = tc::idesc_f16(HP), idesc_o = tc::idesc_f16(NOUT);
  const uint32_t off_ones_c = off_ones;
  auto issue = [&](int P, int l, int t) {
    auto desc = [&](uint32_t off) { return tc::make_desc(sbase + off, 16, 1024, 2); };
    auto desc0 = [&](uint32_t off) { return tc::make_desc(sbase + off, W0_LBO, W0_SBO, 0); };
    auto bdesc = [&](uint32_t off) { return tc::make_desc(sbase + off, BIAS_LBO, BIAS_SBO, 0); };
    const uint64_t ones = tc::make_desc(sbase + off_ones_c, ONES_LBO, ONES_SBO, 0);
    const uint32_t so = (uint32_t)(P < n_pre ? P + 1 : 0) * PL::SLOT;
    const uint32_t d = tmem + (uint32_t)(t * TM::PER_TILE), ahi = d + HP, alo = d + HP + HP / 2;
    const uint32_t bar = saddr(&done_bar[t]);
    if (l == 0) {
      issue_layer_commit<KIN / 16>(d, ahi, alo, desc0(so + PL::off_w0), desc0(so + PL::off_w0 + PL::W0), idesc_h, bar,
                                   ones, bdesc(so + PL::off_bmma));
    } else if (l < nh) {
      const uint32_t wo = so + PL::off_wh + (uint32_t)(2 * (l - 1)) * PL::WH;
      issue_layer_commit<HP / 16>(d, ahi, alo, desc(wo), desc(wo + PL::WH), idesc_h, bar, ones,
                                  bdesc(so + PL::off_bmma + (uint32_t)l * PL::BM_H));
    } else {
      issue_layer_commit<HP / 16>(d, ahi, alo, desc(so + PL::off_wo), desc(so + PL::off_wo + PL::WO), idesc_o, bar,
                                  ones, bdesc(so + PL::off_bmma_o));
    }
  };

  // ---- roles: epilogue warp w < MMA_WARP serves tile g = w / WPT, TMEM lanes
  //      32(w%4)..+31 = starts r of the tile, accumulator columns [part*COLS, +COLS);
  //      the part-0 warp of a quadrant owns the starts' state -------------------------
  const bool epi = warp < MMA_WARP;
  const int g = warp / WPT;
  const int q = warp & 3;
  const int part = (warp % WPT) >> 2;
  const int r = (q << 5) + lane;
  // the CTA's starts: cta_rows (a multiple of 32, <= NT * TILE) so that the grid
  // covers every SM; lanes past the CTA's range run the same code on zero inputs
  // and write nothing (skipping the math in whole idle warps measured slower: the
  // extra branch cost registers -> spills)
  const int64_t cta0 = (int64_t)blockIdx.x * a.cta_rows;
  const int lrow = g * TILE + r;
  const int64_t gi = cta0 + lrow;
  const bool owner = epi && part == 0 && lrow < a.cta_rows && gi < a.N;
  float x[n];
  int t0 = 0, T_i = 0;
  PairwiseSumS<float> acc;
  // per-thread pairwise partial sums live after the network slots
  float* acc_s = (float*)(base + (1 + n_pre) * PL::SLOT) + threadIdx.x * 9;
#pragma unroll
  for (int c = 0; c < n; ++c) x[c] = 0.f;
  if (owner) {
#pragma unroll
    for (int c = 0; c < n; ++c) x[c] = (float)a.x0[gi * n + c];
    t0 = a.t0 ? a.t0[gi] : a.t0_scalar;
    T_i = a.t_hor >= 0 ? a.t_hor : (a.sys.t_max - t0);
    acc.init(T_i + 1, acc_s);
    if (a.X) {
#pragma unroll
      for (int c = 0; c < n; ++c) a.X[gi * (int64_t)(a.t_stride + 1) * n + c] = x[c];
    }
    atomicMax(&s_kmax, T_i);
  }
  __syncthreads();
  const int kmax = s_kmax;
  // passes: the scoring nets' forwards on [x0, t0], then the kmax actor steps
  const int npass = n_pre + kmax;

  // warps whose 32 starts all lie past the CTA's range (the last tile of a
  // 448-row CTA has 2 of 4) skip the rollout: the tile's barriers count only its
  // active warps, so the idle ones free their issue slots (K1 is issue bound)
  const int tile_rows = min(TILE, max(0, a.cta_rows - g * TILE));
  const int act_q = (CACTO_RTC_SKIP_IDLE && CACTO_RTC_SELF) ? (tile_rows + 31) >> 5 : 4;  // active quadrants of tile g
  const int bar_n = act_q * SPLIT * 32;                                // threads on the tile's barriers
  if (epi && q < act_q) {
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(g * TM::PER_TILE);
    const uint32_t t_d = lane_base, t_ahi = lane_base + HP, t_alo = lane_base + HP + HP / 2;
    const int c_base = part * COLS;
    float sig = 0.f, val = 0.f;  // scoring nets' outputs
    uint32_t pd = 0;
    int tl_l = 0, tl_p = 0;  // layer / pass of the last issue (timeline)
    (void)tl_l; (void)tl_p;
    // D[my columns] <- scaled bias of layer l of the net in `slot` (l == nh: output)
    auto preload_bias = [&](int slot, int l) {
      if (CACTO_RTC_BIAS_MMA) return;  // the MMA warp's first MMA of the layer writes it
      const uint32_t bias_s = sbase + (uint32_t)slot * PL::SLOT + PL::off_bias;
      if (l == nh) {
        if (part != 0) return;
        float b[16];
#pragma unroll
        for (int c = 0; c < 16; c += 4) {
          const V4<float> v = lds4(bias_s + (uint32_t)((3 * HP + c) * 4), (float*)nullptr);
          b[c] = v.v[0]; b[c + 1] = v.v[1]; b[c + 2] = v.v[2]; b[c + 3] = v.v[3];
        }
        tc::tmem_st16(t_d, b);
        return;
      }
#pragma unroll
      for (int c0 = 0; c0 < COLS; c0 += 16) {
        float b[16];
#pragma unroll
        for (int c = 0; c < 16; c += 4) {
          const V4<float> v = lds4(bias_s + (uint32_t)((l * HP + c_base + c0 + c) * 4), (float*)nullptr);
          b[c] = v.v[0]; b[c + 1] = v.v[1]; b[c + 2] = v.v[2]; b[c + 3] = v.v[3];
        }
        tc::tmem_st16(t_d + (uint32_t)(c_base + c0), b);
      }
    };
    // normalised input row [x, t] of the net in `slot` (nets.py:126-129)
    auto write_input = [&](int slot, int t_abs) {
      if (part != 0) return;
      const NetConst<float>& nc = slot == 0 ? a.nc : a.pre_nc[slot - 1];
      float v[KIN];
#pragma unroll
      for (int c = 0; c < KIN; ++c) v[c] = 0.f;
      if (owner) {
#pragma unroll
        // fp32 path: multiply by the reciprocal half-width (<= 1.5 ulp from the
        // division, no FCHK / slow-path branch per input per step)
        for (int c = 0; c < n; ++c) v[c] = (x[c] - nc.in_center[c]) * nc.in_inv_half[c];
        v[n] = ((float)t_abs - nc.in_center[n]) * nc.in_inv_half[n];
      }
      float hv[KIN / 2], lv[KIN / 2];
#pragma unroll
      for (int c = 0; c < KIN; c += 2) {
        uint32_t h, l;
        split2(v[c], v[c + 1], h, l);
        hv[c / 2] = __uint_as_float(h);
        lv[c / 2] = __uint_as_float(l);
      }
      tc::tmem_st8(t_ahi, hv);
      tc::tmem_st8(t_alo, lv);
    };
    // the tile's leader warp (one per tile, on scheduler g % 4) polls its MMA
    // barrier and, self-issuing, issues its MMAs
    const bool leader = (warp % WPT) == (CACTO_RTC_SELF ? ((g & 3) < act_q ? (g & 3) : 0) : 0);
    auto handoff = [&](int P, int l) {
      tc::tmem_wait_st();
      tc::tc_fence_before();
#if CACTO_RTC_SELF
      // A of layer l is in TMEM once every warp of the tile has passed here: the
      // leader waits for the others in named barrier 1 + NT + g and issues
      if (leader) {
        RTC_TL(P, l, 0);
        asm volatile("bar.sync %0, %1;" ::"r"(1 + NT + g), "r"(bar_n) : "memory");
        RTC_TL(P, l, 1);
        tc::tc_fence_after();
        issue(P, l, g);
        RTC_TL(P, l, 2);
        tl_l = l; tl_p = P;
      } else {
        asm volatile("bar.arrive %0, %1;" ::"r"(1 + NT + g), "r"(bar_n) : "memory");
      }
#else
      (void)P; (void)l;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full_bar[g]);
#endif
    };
    auto wait_done = [&]() {
#ifndef CACTO_RTC_POLL_ALL
      // one warp of the tile polls the MMA barrier; the tile's other epilogue warps
      // block in a named barrier (no polling instructions on their schedulers):
      // manipulator3 K1 3.84 -> 3.78 ms (profiles/README.md)
      if (leader) {
        tc::mbar_wait_sleep(&done_bar[g], pd);
        RTC_TL(tl_p, tl_l, 3);
      }
      asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(bar_n) : "memory");
#elif defined(CACTO_RTC_PLAIN_WAIT)
      tc::mbar_wait(&done_bar[g], pd);
#else
      tc::mbar_wait_sleep(&done_bar[g], pd);
#endif
      pd ^= 1;
      tc::tc_fence_after();
    };
    auto start_pass = [&](int P) {
      const int slot = P < n_pre ? P + 1 : 0;
      write_input(slot, P < n_pre ? t0 : t0 + (P - n_pre));
      preload_bias(slot, 0);
      handoff(P, 0);
    };
    if (npass > 0) start_pass(0);
    for (int P = 0; P < npass; ++P) {
      const int slot = P < n_pre ? P + 1 : 0;
      float oc[MO > 0 ? MO : 1];  // output-layer values (CUDA-core path)
      for (int l = 0; l < nh; ++l) {  // hidden layers
        wait_done();
        if (MO > 0 && l == nh - 1) {
          const uint32_t wf = sbase + off_wf + (uint32_t)(P < n_pre ? P + 1 : 0) * WF;
          uint64_t acc[MO > 0 ? MO : 1];
#pragma unroll
          for (int j = 0; j < MO; ++j) acc[j] = 0ull;
          float za[16], zb[16];
          tc::tmem_ld16(t_d, za);
          tc::tmem_wait_ld_dep(za);
#pragma unroll
          for (int c0 = 0; c0 < COLS; c0 += 16) {
            if (c0 + 16 < COLS) tc::tmem_ld16(t_d + (uint32_t)(c0 + 16), zb);
#pragma unroll
            for (int c = 0; c < 16; c += 4) {
              uint64_t v01, v23;
              if constexpr (ACT == CACTO_ACT_ELU) {
                v01 = elu2(za[c], za[c + 1], AF::S);
                v23 = elu2(za[c + 2], za[c + 3], AF::S);
              } else {
                v01 = f2pack(AF::apply(za[c]), AF::apply(za[c + 1]));
                v23 = f2pack(AF::apply(za[c + 2]), AF::apply(za[c + 3]));
              }
#pragma unroll
              for (int j = 0; j < MO; ++j) {
                const V4<float> w = lds4(wf + (uint32_t)((j * HP + c0 + c) * 4), (float*)nullptr);
                acc[j] = f2fma(v01, f2pack(w.v[0], w.v[1]), acc[j]);
                acc[j] = f2fma(v23, f2pack(w.v[2], w.v[3]), acc[j]);
              }
            }
            if (c0 + 16 < COLS) {
              tc::tmem_wait_ld_dep(zb);
#pragma unroll
              for (int c = 0; c < 16; ++c) za[c] = zb[c];
            }
          }
#pragma unroll
          for (int j = 0; j < MO; ++j) {
            float e0, e1;
            f2unpack(acc[j], e0, e1);
            oc[j] = (e0 + e1) + lds1(wf + (uint32_t)((MO * HP + j) * 4), (float*)nullptr);
          }
          break;
        }
        // 16-column chunks, software pipelined: the next chunk's tcgen05.ld is in
        // flight while this chunk's activations are computed and stored (a single
        // warp's ld + wait costs ~160 cycles, profiles/probe_tmem.cu)
        float za[16], zb[16];
        tc::tmem_ld16(t_d + (uint32_t)c_base, za);
        tc::tmem_wait_ld_dep(za);
#pragma unroll
        for (int c0 = 0; c0 < COLS; c0 += 16) {
          if (c0 + 16 < COLS) tc::tmem_ld16(t_d + (uint32_t)(c_base + c0 + 16), zb);
          float hv[8], lv[8];
#pragma unroll
          for (int c = 0; c < 16; c += 2) {
            uint32_t h, lo;
            if constexpr (ACT == CACTO_ACT_ELU) elu_split2(za[c], za[c + 1], AF::S, h, lo);
            else split2(AF::apply(za[c]), AF::apply(za[c + 1]), h, lo);
            hv[c / 2] = __uint_as_float(h);
            lv[c / 2] = __uint_as_float(lo);
          }
          const uint32_t ac = (uint32_t)((c_base + c0) / 2);
          tc::tmem_st8(t_ahi + ac, hv);
          tc::tmem_st8(t_alo + ac, lv);
          if (c0 + 16 < COLS) {
            tc::tmem_wait_ld_dep(zb);
#pragma unroll
            for (int c = 0; c < 16; ++c) za[c] = zb[c];
          }
        }
        preload_bias(slot, l + 1);
        handoff(P, l + 1);
      }
      // output layer
      float o[16];
      if constexpr (MO > 0) {
#pragma unroll
        for (int j = 0; j < MO; ++j) o[j] = oc[j] * WSCALE;  // the MMA path's scaled D
      } else {
        wait_done();
        if (part == 0) tc::tmem_ld16_wait(t_d, o);
      }
      if (slot != 0) {
        // scoring net: sigma(x0) = sigma_min + softplus(o) or V(x0) = o
        const float ov = o[0] * (1.f / WSCALE);
        if (a.pre_kind[slot - 1] == 0) sig = head_value(CACTO_HEAD_STD, a.pre_nc[slot - 1], 0, ov);
        else val = ov;
      } else {
        const int k = P - n_pre;
        if (owner && k < T_i) {
          float u[m];
#pragma unroll
          for (int j = 0; j < m; ++j) u[j] = head_value(a.head, a.nc, j, o[j] * (1.f / WSCALE));
          if (a.U) {
#pragma unroll
            for (int j = 0; j < m; ++j) a.U[a.u_at(gi, k, j, m)] = u[j];
          }
          float xn[n];
          const float sc = cost_and_step<SYS>(a.sys, a.cost, a.has_cost, x, u, xn);
          acc.add(k, sc);
          if (a.SC) a.SC[gi * (int64_t)(a.t_stride + 1) + k] = sc;
#pragma unroll
          for (int c = 0; c < n; ++c) x[c] = xn[c];
          if (a.X) {
#pragma unroll
            for (int c = 0; c < n; ++c) a.X[(gi * (int64_t)(a.t_stride + 1) + k + 1) * n + c] = x[c];
          }
        }
      }
      if (P + 1 < npass) start_pass(P + 1);
    }
    if (owner) {
      const float term = a.has_cost ? terminal_cost<SYS>(a.sys, a.cost, x) : 0.f;
      acc.add(T_i, term);
      if (a.SC) a.SC[gi * (int64_t)(a.t_stride + 1) + T_i] = term;
      if (a.C) a.C[gi] = acc.res;
      if (a.scores) {
        const float gap = fabsf(val - acc.res);  // |V(x0) - J(x0)|
        a.scores[gi] = a.score_mode == CACTO_SCORE_STD ? sig : (a.score_mode == CACTO_SCORE_GAP ? gap : sig * gap);
      }
    }
  } else if (!CACTO_RTC_SELF) {
    // ---- MMA issuer (whole warp converged; elect.sync picks the issuing lane) ----------
    uint32_t pf[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) pf[t] = 0;
    for (int P = 0; P < npass; ++P) {
      const uint32_t so = (uint32_t)(P < n_pre ? P + 1 : 0) * PL::SLOT;
      for (int l = 0; l <= nh; ++l) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          tc::mbar_wait_sleep(&full_bar[t], pf[t]);
          pf[t] ^= 1;
          tc::tc_fence_after();
          issue(P, l, t);
          __syncwarp();
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == alloc_warp) tc::tmem_dealloc(tmem, TM::COLS);
}

template <int SYS, int HP, int NT>
static int launch_rollout_tc_nt(const RolloutArgs<float>& a, cudaStream_t st) {
  using PL = rtc::Plan<HP>;
  // 4 tiles: one epilogue warp per lane quadrant; fewer tiles: the columns are
  // split over more warps (shorter per-layer epilogue latency), 512 threads max
#ifndef CACTO_RTC_SPLIT4
#define CACTO_RTC_SPLIT4 1
#endif
  constexpr int SPLIT = NT == 4 ? CACTO_RTC_SPLIT4 : (NT == 2 ? (HP >= 32 ? 2 : 1) : (HP >= 64 ? 4 : HP / 16));
  auto kern = a.act == CACTO_ACT_ELU ? rollout_tc_kernel<SYS, HP, NT, SPLIT, CACTO_ACT_ELU>
                                     : rollout_tc_kernel<SYS, HP, NT, SPLIT, CACTO_ACT_TANH>;
  constexpr uint32_t ACC = (uint32_t)rtc_threads<NT, SPLIT>() * 9 * 4;  // pairwise partial sums
  constexpr uint32_t ONES = (CACTO_RTC_BIAS_MMA ? rtc::ONES_BYTES : 0) + 3 * (3 * HP + 4) * 4;  // + fp32 output layers
  const uint32_t bytes = (uint32_t)(1 + a.n_pre) * PL::SLOT + ACC + ONES + 1024;
  if (!ensure_smem((const void*)kern, 3 * PL::SLOT + ACC + ONES + 1024))
    return set_error(CACTO_ECUDA, "rollout_tc: %u B of shared memory not available", 3 * PL::SLOT + ACC + ONES + 1024);
  // starts per CTA: as even as 32-row granularity allows over whole waves of SMs
  // (65,536 starts: 147 CTAs of 448 instead of 128 CTAs of 512 leaving 20 SMs idle)
  const int64_t per = (int64_t)NT * rtc::TILE, sms = num_sms();
  const int64_t waves = std::max<int64_t>(1, (a.N + per * sms - 1) / (per * sms));
  int64_t rows = (a.N + waves * sms - 1) / (waves * sms);
  rows = std::min<int64_t>(per, (rows + 31) / 32 * 32);
  RolloutArgs<float> b = a;
  b.cta_rows = (int)rows;
  const int64_t blocks = (a.N + rows - 1) / rows;
  kern<<<(unsigned)blocks, rtc_threads<NT, SPLIT>(), bytes, st>>>(b);
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

extern "C" int cacto_debug_rtc_timeline(unsigned long long* host) {
#if CACTO_RTC_TIMELINE
  return cudaMemcpyFromSymbol(host, g_rtc_tl, sizeof(g_rtc_tl)) == cudaSuccess ? 0 : 1;
#else
  (void)host;
  return -1;
#endif
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
