// probe_f16.cu -- checks the tcgen05.mma kind::f16 data path this repo relies on:
// A (fp16, 128 x K) in TMEM, packed two K-consecutive halves per 32-bit column
// (low half = even k), B (fp16, N x K) K-major SW128 in shared memory, D fp32 in
// TMEM; compares D against a host fp64 product and times bursts of MMAs.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a
//        -I../paper_2602_19699_b200/csrc -I../include probe_f16.cu -o probe_f16 -lcuda
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "tc.cuh"

using namespace cacto;

int set_error(int, const char*, ...) { return -1; }
int check_launch(const char*) { return 0; }
bool ensure_smem(const void*, size_t) { return true; }

constexpr int M = 128, N = 64, K = 64;

CACTO_D void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// A [M][K] fp16 row-major, B [N][K] fp16 row-major -> D [M][N] fp32; cycles[0..1]
__global__ void kern(const __half* A, const __half* B, float* D, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // B -> SW128 K-major: row n = 128 bytes = 64 halves, 16-byte chunk j at (j ^ (n & 7))
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    const int n = e / K, k = e % K;
    const uint32_t off = n * 128 + ((((k * 2) >> 4) ^ (n & 7)) << 4) + ((k * 2) & 15);
    *reinterpret_cast<__half*>(base + off) = B[n * K + k];
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tc::tmem_alloc(&tbase, 256);
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tbase;
  // A -> TMEM columns [128, 128 + K/2): thread row r = 32*warp + lane
  {
    const int r = warp * 32 + lane;
    float v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      __half2 h = __halves2half2(A[r * K + 2 * c], A[r * K + 2 * c + 1]);
      v[c] = *reinterpret_cast<float*>(&h);
    }
    tc::tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + 128, v);
    tc::tmem_wait_st();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint64_t db = tc::make_desc(saddr(base), 16, 1024, 2);
    long long t0 = clock64();
#pragma unroll
    for (int kk = 0; kk < K / 16; ++kk)
      mma_f16_ts(tmem, tmem + 128 + (uint32_t)(kk * 8), db + (uint64_t)(kk * 2), idesc, kk > 0);
    tc::tc_commit_elect(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    // timing: 96 more dependent MMAs
#pragma unroll
    for (int i = 0; i < 96; ++i)
      mma_f16_ts(tmem + 64, tmem + 128 + (uint32_t)((i & 3) * 8), db + (uint64_t)((i & 3) * 2), idesc, i > 0);
    tc::tc_commit_elect(&bar);
    tc::mbar_wait(&bar, 1);
    long long t2 = clock64();
    if (lane == 0) {
      cycles[0] = t1 - t0;
      cycles[1] = t2 - t1;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  {
    const int r = warp * 32 + lane;
    float d[32];
    for (int c0 = 0; c0 < N; c0 += 32) {
      tc::tmem_ld32_wait(tmem + ((uint32_t)(warp * 32) << 16) + c0, d);
      for (int c = 0; c < 32; ++c) D[r * N + c0 + c] = d[c];
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

int main() {
  std::vector<__half> A(M * K), B(N * K);
  std::vector<double> Af(M * K), Bf(N * K);
  unsigned s = 1;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xFFFF) / 65536.0 - 0.5; };
  for (int i = 0; i < M * K; ++i) { A[i] = __float2half((float)rnd()); Af[i] = __half2float(A[i]); }
  for (int i = 0; i < N * K; ++i) { B[i] = __float2half((float)rnd()); Bf[i] = __half2float(B[i]); }
  __half *dA, *dB;
  float* dD;
  long long* dc;
  cudaMalloc(&dA, M * K * 2);
  cudaMalloc(&dB, N * K * 2);
  cudaMalloc(&dD, M * N * 4);
  cudaMalloc(&dc, 16);
  cudaMemcpy(dA, A.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), N * K * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  kern<<<1, 128, 64 * 1024>>>(dA, dB, dD, dc);
  std::vector<float> D(M * N);
  long long cyc[2];
  cudaError_t e = cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(cyc, dc, 16, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; }
  double maxerr = 0, maxref = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += Af[i * K + k] * Bf[j * K + k];
      maxerr = fmax(maxerr, fabs(ref - D[i * N + j]));
      maxref = fmax(maxref, fabs(ref));
    }
  printf("{\"probe\": \"kind::f16 A in TMEM (packed halves), B SW128 smem, M128 N64 K64\", \"max_abs_err\": %.3e, "
         "\"max_abs_ref\": %.3e, \"latency_4mma_cycles\": %lld, \"cycles_per_mma_burst96\": %.1f}\n",
         maxerr, maxref, cyc[0], cyc[1] / 96.0);
  return 0;
}
