// probe_tmem.cu -- TMEM -> register (tcgen05.ld 32x32b) and register -> TMEM
// (tcgen05.st) throughput on this B200, the data path of the rollout epilogue
// (rollout_tc.cu reads a 128 x 64 fp32 accumulator and writes 2 x 128 x 32 fp16
// pairs per layer and tile).  One CTA per SM, W warps (W/4 per sub-partition),
// each warp streaming loads of x32 columns from its lane quadrant with a wait
// after every G loads; reports bytes per SM per cycle.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a
//        -I../paper_2602_19699_b200/csrc -I../include probe_tmem.cu -o probe_tmem
#include <cstdio>

#include "tc.cuh"

using namespace cacto;

int set_error(int, const char*, ...) { return -1; }
int check_launch(const char*) { return 0; }
bool ensure_smem(const void*, size_t) { return true; }

template <int MODE>  // 0: ld x32 + wait each, 1: 2 x ld x32 then wait, 2: st x16 (pairs), 3: ld x32 + wait + FP work
__global__ void probe(int iters, long long* cycles, float* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t q = warp & 3;
  const uint32_t col = (uint32_t)((warp >> 2) * 64) & 511u;
  const uint32_t addr = tbase + (q * 32u << 16) + col;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if constexpr (MODE == 0 || MODE == 3) {
      float v[32];
      tc::tmem_ld32_wait(addr, v);
#pragma unroll
      for (int c = 0; c < 32; ++c) acc += v[c];
      if constexpr (MODE == 3) {
#pragma unroll
        for (int c = 0; c < 32; ++c) acc = fmaf(acc, 1.0001f, v[c] * 0.5f);
      }
    } else if constexpr (MODE == 1) {
      float v[32], w[32];
      tc::tmem_ld32_wait(addr, v);
      tc::tmem_ld32_wait(addr + 32, w);
#pragma unroll
      for (int c = 0; c < 32; ++c) acc += v[c] + w[c];
    } else {
      float v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] = acc + c;
      tc::tmem_st16(addr, v);
      tc::tmem_wait_st();
      acc += 1.f;
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

template <int MODE>
void run(int warps, const char* name) {
  const int sms = 148, iters = 4096;
  long long* cyc;
  float* sink;
  cudaMalloc(&cyc, sms * sizeof(long long));
  cudaMalloc(&sink, sms * 1024 * sizeof(float));
  probe<MODE><<<sms, warps * 32>>>(16, cyc, sink);
  probe<MODE><<<sms, warps * 32>>>(iters, cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += (double)h[i] / sms;
  const double bytes = (MODE == 2 ? 64.0 : (MODE == 1 ? 256.0 : 128.0)) * 32 * warps * iters;  // per SM
  printf("{\"mode\": \"%s\", \"warps\": %d, \"cycles\": %.0f, \"bytes_per_cycle_per_sm\": %.1f, "
         "\"cycles_per_op_per_warp\": %.1f, \"err\": \"%s\"}\n",
         name, warps, mean, bytes / mean, mean / iters, cudaGetErrorString(e));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 16, 32}) {
    run<0>(w, "ld32+wait");
    run<1>(w, "2x ld32, wait each");
    run<2>(w, "st16(f32)+wait");
    run<3>(w, "ld32+wait+64 FP ops");
  }
  return 0;
}
