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

namespace cacto {

// 3-register FFMA: every operand a per-thread register (the GEMM inner-loop form)
__global__ void __launch_bounds__(256) fma3_peak_kernel(float* out, int iters) {
  float a[16], b[16], c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    a[i] = (float)(threadIdx.x + i);
    b[i] = 0.999999f + 1e-9f * (float)(threadIdx.x * 16 + i);
    c[i] = 1e-7f * (float)(threadIdx.x + 3 * i);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b[i], c[i]);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == -1.2345f) out[blockIdx.x] = s;
}

// packed FFMA2 (fma.rn.f32x2): 2 FMAs per lane per instruction
__global__ void __launch_bounds__(256) ffma2_peak_kernel(float* out, int iters) {
  unsigned long long a[8], b[8], c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float2 x = make_float2((float)(threadIdx.x + i), (float)(threadIdx.x + 2 * i));
    float2 y = make_float2(0.999999f + 1e-9f * (float)(threadIdx.x + i), 0.999998f + 1e-9f * (float)i);
    float2 z = make_float2(1e-7f * (float)(threadIdx.x + i), 2e-7f * (float)i);
    a[i] = *reinterpret_cast<unsigned long long*>(&x);
    b[i] = *reinterpret_cast<unsigned long long*>(&y);
    c[i] = *reinterpret_cast<unsigned long long*>(&z);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(b[i]), "l"(c[i]));
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float2 x = *reinterpret_cast<float2*>(&a[i]);
    s += x.x + x.y;
  }
  if (s == -1.2345f) out[blockIdx.x] = s;
}

}  // namespace cacto

// mode 0: FFMA with constant operands, 1: 3-register FFMA, 2: packed FFMA2 (3-register);
// every mode executes 2*16*8*iters*blocks*256 FLOPs
extern "C" int cacto_fma_peak_mode(int32_t mode, int32_t blocks, int32_t iters, void* out, void* stream) {
  if (blocks < 1 || iters < 1 || !out) return set_error(CACTO_EVALUE, "fma_peak_mode: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (mode == 0)
    fma_peak_kernel<float><<<blocks, 256, 0, st>>>((float*)out, iters, 0.999999f, 1e-7f);
  else if (mode == 1)
    fma3_peak_kernel<<<blocks, 256, 0, st>>>((float*)out, iters);
  else
    ffma2_peak_kernel<<<blocks, 256, 0, st>>>((float*)out, iters);
  return check_launch("fma_peak_mode");
}
