// peak.cu -- FFMA / DFMA throughput microbenchmark: the measured roofline
// denominator for the CUDA-core (SIMT) kernels (MEASURED_PEAKS.json only
// carries HBM and bf16 tensor peaks).  16 independent FMA chains per thread,
// 8 CTAs x 256 threads per SM.
#include "common.cuh"

namespace cacto {

template <typename T>
__global__ void __launch_bounds__(256) fma_peak_kernel(T* out, int iters, T b, T c) {
  T a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = (T)(threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  }
  T s = T(0);
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == T(-1.2345)) out[blockIdx.x] = s;  // keeps the chains alive
}

}  // namespace cacto

using namespace cacto;

// FLOPs executed = 2 * 16 * 8 * iters * blocks * 256
extern "C" int cacto_fma_peak(int32_t dtype, int32_t blocks, int32_t iters, void* out, void* stream) {
  if (blocks < 1 || iters < 1 || !out) return set_error(CACTO_EVALUE, "fma_peak: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CACTO_F32)
    fma_peak_kernel<float><<<blocks, 256, 0, st>>>((float*)out, iters, 0.999999f, 1e-7f);
  else
    fma_peak_kernel<double><<<blocks, 256, 0, st>>>((double*)out, iters, 0.999999, 1e-7);
  return check_launch("fma_peak_kernel");
}
