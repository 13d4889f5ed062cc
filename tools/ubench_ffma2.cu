// Throughput of FFMA (3-register form) vs FFMA2 (packed f32x2) on one SM
// partition: 8 independent accumulator chains per thread, 1 warp per SMSP up
// to 8 warps per SMSP.  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/ub tools/ubench_ffma2.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ffma(float* out, float a, float b, int iters) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  float m = a + threadIdx.x * 1e-7f, c = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], m, c);
    m += 1e-9f;
    c -= 1e-9f;
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float a, float b, int iters) {
  unsigned long long x[4];
  for (int i = 0; i < 4; ++i) {
    float lo = threadIdx.x * 0.001f + 2 * i, hi = lo + 1;
    x[i] = ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
  }
  float mf = a + threadIdx.x * 1e-7f, cf = b;
  for (int it = 0; it < iters; ++it) {
    unsigned long long m = ((unsigned long long)__float_as_uint(mf) << 32) | __float_as_uint(mf + 1e-8f);
    unsigned long long c = ((unsigned long long)__float_as_uint(cf) << 32) | __float_as_uint(cf - 1e-8f);
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 4; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(m), "l"(c));
    mf += 1e-9f;
    cf -= 1e-9f;
  }
  float s = 0;
  for (int i = 0; i < 4; ++i) s += __uint_as_float((unsigned)x[i]) + __uint_as_float((unsigned)(x[i] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 1 << 24);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int wps = 1; wps <= 8; wps *= 2) {
    const int threads = 128 * wps;  // wps warps per SMSP, one CTA per SM
    for (int v = 0; v < 2; ++v) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (v == 0) k_ffma<<<148, threads>>>(out, 1.0001f, 0.5f, iters);
        else k_ffma2<<<148, threads>>>(out, 1.0001f, 0.5f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fmas = 148.0 * threads * iters * 16 * 8;
        if (rep) printf("%s warps/SMSP=%d: %.3f ms, %.1f TFMA/s, %.2f FMA/clk/SMSP @1.965GHz, instr/clk/SMSP=%.2f\n",
                        v ? "FFMA2" : "FFMA ", wps, ms, fmas / ms / 1e9, fmas / (ms * 1e-3) / 1.965e9 / 148 / 4 / 32,
                        fmas / (v ? 2 : 1) / (ms * 1e-3) / 1.965e9 / 148 / 4 / 32);
      }
    }
  }
  return 0;
}
