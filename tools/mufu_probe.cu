// MUFU throughput probe on one B200: sin+cos (__sincosf), sin alone, ex2, rsqrt.
// Prints results per clock per SM (MUFU lane-ops / SM / clock).
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = (threadIdx.x + j) * 1e-3f;
  float acc = 0.f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) { float s, c; __sincosf(a[j], &s, &c); a[j] = s + c; }
      if (OP == 1) { a[j] = __sinf(a[j]); }
      if (OP == 2) { a[j] = exp2f(a[j]) * 0.5f; }
      if (OP == 3) { a[j] = rsqrtf(a[j] + 1.f); }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) acc += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sms * 8 * 1024 * 4);
  const char* names[4] = {"sincos (2 MUFU)", "sin", "ex2(+fmul)", "rsqrt(+fadd)"};
  const double mufu_per[4] = {2, 1, 1, 1};
  for (int op = 0; op < 4; ++op) {
    const int iters = 4096, blocks = sms * 8, threads = 256;
    cudaEvent_t s, e;
    cudaEventCreate(&s); cudaEventCreate(&e);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(s);
      if (op == 0) k<0><<<blocks, threads>>>(out, iters);
      if (op == 1) k<1><<<blocks, threads>>>(out, iters);
      if (op == 2) k<2><<<blocks, threads>>>(out, iters);
      if (op == 3) k<3><<<blocks, threads>>>(out, iters);
      cudaEventRecord(e);
      cudaEventSynchronize(e);
    }
    float ms; cudaEventElapsedTime(&ms, s, e);
    const double ops = (double)blocks * threads * iters * 8 * mufu_per[op];
    const double per_clk_sm = ops / (ms * 1e-3) / sms / (clk * 1e3);
    printf("%-18s %.3f ms  %.2f MUFU lane-ops/clk/SM (at %d MHz nominal)\n", names[op], ms, per_clk_sm, clk / 1000);
  }
  return 0;
}
