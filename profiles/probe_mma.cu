// probe_mma.cu -- microbenchmark of tcgen05.mma.kind::tf32 issue/latency on
// one SM: cycles per MMA for chains into the same accumulator vs round-robin
// over independent accumulators, N = 16/64/128/256, A from SMEM or TMEM.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a
//        -I../paper_2602_19699_b200/csrc -I../include probe_mma.cu -o probe_mma -lcuda
#include <cstdio>

#include "tc.cuh"

using namespace cacto;

int set_error(int, const char*, ...) { return -1; }
int check_launch(const char*) { return 0; }
bool ensure_smem(const void*, size_t) { return true; }

template <int NM, int NACC, int BN, int ATMEM>
__global__ void probe_u(int reps, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.f;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::tmem_alloc(&tbase, 512);
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t sb = saddr(base);
  const uint64_t da = tc::make_desc(sb, 16, 1024, 2);
  const uint64_t db = tc::make_desc(sb + 32768, 16, 1024, 2);
  const uint32_t idesc = tc::idesc_tf32(BN, 0, 0);
  long long best = 1LL << 60, best_issue = 1LL << 60;
  uint32_t ph = 0;
  for (int rep = 0; rep < reps; ++rep) {
    __syncwarp();
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      const uint32_t d = tmem + (uint32_t)((i % NACC) * 64);
      if (ATMEM)
        tc::mma_tf32_ts_elect(d, tmem + 256 + (uint32_t)((i & 7) * 8), db + (uint64_t)((i & 3) * 2), idesc, i >= NACC);
      else
        tc::mma_tf32_elect(d, da + (uint64_t)((i & 3) * 2), db + (uint64_t)((i & 3) * 2), idesc, i >= NACC);
    }
    long long ti = clock64();
    tc::tc_commit_elect(&bar);
    tc::mbar_wait(&bar, ph);
    ph ^= 1;
    long long t1 = clock64();
    if (rep > 0 && t1 - t0 < best) best = t1 - t0;
    if (rep > 0 && ti - t0 < best_issue) best_issue = ti - t0;
  }
  if (threadIdx.x == 0) {
    out[0] = best;
    out[1] = best_issue;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tmem_dealloc(tmem, 512);
}

__global__ void probe(int n_mma, int n_acc, int bn, int a_tmem, int reps, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.f;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::tmem_alloc(&tbase, 512);
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t sb = saddr(base);
  const uint64_t da = tc::make_desc(sb, 16, 1024, 2);
  const uint64_t db = tc::make_desc(sb + 32768, 16, 1024, 2);
  const uint32_t idesc = tc::idesc_tf32(bn, 0, 0);
  const int acc_stride = 512 / (n_acc > 0 ? n_acc : 1) / 2;  // columns; A_tmem in the upper half
  long long best = 1LL << 60;
  uint32_t ph = 0;
  for (int rep = 0; rep < reps; ++rep) {
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int acc = i % n_acc;
      const uint32_t d = tmem + (uint32_t)(acc * acc_stride);
      const uint32_t acc_flag = (i >= n_acc) ? 1u : 0u;
      if (a_tmem)
        tc::mma_tf32_ts_elect(d, tmem + 256 + (uint32_t)((i & 7) * 8), db + (uint64_t)((i & 3) * 2), idesc, acc_flag);
      else
        tc::mma_tf32_elect(d, da + (uint64_t)((i & 3) * 2), db + (uint64_t)((i & 3) * 2), idesc, acc_flag);
    }
    tc::tc_commit_elect(&bar);
    tc::mbar_wait(&bar, ph);
    ph ^= 1;
    long long t1 = clock64();
    if (rep > 0 && t1 - t0 < best) best = t1 - t0;
  }
  if (threadIdx.x == 0) *out = best;
  tc::tc_fence_before();
  __syncthreads();
  tc::tmem_dealloc(tmem, 512);
}

template <int NM, int NACC, int BN, int ATMEM>
void run_u(long long* d, bool& first) {
  cudaFuncSetAttribute(probe_u<NM, NACC, BN, ATMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  probe_u<NM, NACC, BN, ATMEM><<<1, 32, 100 * 1024>>>(6, d);
  long long c[2] = {0, 0};
  cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
  printf("%s{\"unrolled\": 1, \"a_tmem\": %d, \"N\": %d, \"accumulators\": %d, \"mmas\": %d, \"cycles\": %lld, "
         "\"issue_cycles\": %lld, \"cycles_per_mma\": %.1f}",
         first ? "" : ",\n", ATMEM, BN, NACC, NM, c[0], c[1], (double)c[0] / NM);
  first = false;
}

int main() {
  long long* d;
  cudaMalloc(&d, 2 * sizeof(long long));
  bool first = true;
  printf("{\"probe\": \"tcgen05.mma kind::tf32 M=128 K=8, unrolled bursts\", \"rows\": [\n");
  run_u<24, 1, 16, 0>(d, first);
  run_u<24, 1, 64, 0>(d, first);
  run_u<24, 1, 128, 0>(d, first);
  run_u<24, 1, 256, 0>(d, first);
  run_u<96, 1, 64, 0>(d, first);
  run_u<96, 4, 64, 0>(d, first);
  run_u<96, 1, 256, 0>(d, first);
  run_u<24, 1, 64, 1>(d, first);
  run_u<96, 1, 64, 1>(d, first);
  run_u<96, 4, 64, 1>(d, first);
  run_u<96, 1, 256, 1>(d, first);
  printf("\n]}\n");
  return 0;
}
