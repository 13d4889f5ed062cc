// Microbenchmark: dependent-chain latencies on B200 (cycles per op), one warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_latency tools/ubench_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void k_shfl(float* out, long long* cyc, float seed) {
  float v = seed + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) v = __shfl_sync(0xffffffffu, v, (threadIdx.x + 1) & 31);
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_shfl_xor(float* out, long long* cyc, float seed) {
  float v = seed + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1);
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_fadd(float* out, long long* cyc, float seed) {
  float v = seed + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) v = __fadd_rn(v, 1.0001f);
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_argmax(float* out, long long* cyc, float seed) {
  // v -> max(v + a, v + b) with index select: FADD, FSETP, FSEL chain
  float v = seed + threadIdx.x;
  int idx = 0;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    float a = __fadd_rn(v, 0.5f), b = __fadd_rn(v, 0.25f * (threadIdx.x & 3));
    bool p = b > a;
    v = p ? b : a;
    idx += p;
  }
  long long t1 = clock64();
  out[threadIdx.x] = v + idx;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_lds(float* out, long long* cyc, float seed) {
  __shared__ int buf[256];
  for (int i = threadIdx.x; i < 256; i += 32) buf[i] = (i * 7 + 1) & 255;
  __syncwarp();
  int v = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) v = buf[v];
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_mufu(float* out, long long* cyc, float seed) {
  float v = seed + threadIdx.x * 1e-3f;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    float r;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    v = r * 0.5f;
  }
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_vstep(float* out, long long* cyc, float seed) {
  // one K=4 Viterbi step chain: 4 shfl.idx -> 4 fadd -> fmax tree -> fadd
  const int g = threadIdx.x >> 2;
  float d = seed + threadIdx.x * 0.01f;
  const float a0 = 0.1f * threadIdx.x, a1 = 0.2f, a2 = 0.3f, a3 = -0.1f;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    float c0 = __fadd_rn(__shfl_sync(0xffffffffu, d, g * 4 + 0), a0);
    float c1 = __fadd_rn(__shfl_sync(0xffffffffu, d, g * 4 + 1), a1);
    float c2 = __fadd_rn(__shfl_sync(0xffffffffu, d, g * 4 + 2), a2);
    float c3 = __fadd_rn(__shfl_sync(0xffffffffu, d, g * 4 + 3), a3);
    d = __fadd_rn(fmaxf(fmaxf(c0, c1), fmaxf(c2, c3)), -0.5f);
  }
  long long t1 = clock64();
  out[threadIdx.x] = d;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_vstep_smem(float* out, long long* cyc, float seed) {
  // same chain with the exchange through shared memory (st, syncwarp, ld.v4)
  __shared__ __align__(16) float xb[32];
  const int g = threadIdx.x >> 2;
  float d = seed + threadIdx.x * 0.01f;
  const float a0 = 0.1f * threadIdx.x, a1 = 0.2f, a2 = 0.3f, a3 = -0.1f;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    xb[threadIdx.x] = d;
    __syncwarp();
    const float4 v = *reinterpret_cast<const float4*>(xb + 4 * g);
    __syncwarp();
    float c0 = __fadd_rn(v.x, a0), c1 = __fadd_rn(v.y, a1), c2 = __fadd_rn(v.z, a2), c3 = __fadd_rn(v.w, a3);
    d = __fadd_rn(fmaxf(fmaxf(c0, c1), fmaxf(c2, c3)), -0.5f);
  }
  long long t1 = clock64();
  out[threadIdx.x] = d;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(float));
  cudaMalloc(&cyc, sizeof(long long));
  struct {
    const char* name;
    void (*k)(float*, long long*, float);
  } ks[] = {{"shfl.idx", k_shfl}, {"shfl.bfly", k_shfl_xor}, {"fadd", k_fadd},
            {"fadd+fsetp+fsel (argmax2)", k_argmax}, {"lds chase", k_lds}, {"ex2+fmul", k_mufu},
            {"viterbi K=4 step (shfl)", k_vstep}, {"viterbi K=4 step (smem)", k_vstep_smem}};
  for (auto& k : ks) {
    for (int rep = 0; rep < 2; ++rep) k.k<<<1, 32>>>(out, cyc, 1.0f);
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("%-28s %.2f cycles per dependent step\n", k.name, (double)c / N);
  }
  return 0;
}
