// L2-resident read+write bandwidth: a persistent grid sweeps a buffer of S MiB
// `reps` times (y = x + 1 in place, 16-byte accesses).  nvcc -arch=sm_100a -O3 tools/l2bw.cu -o tools/l2bw
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void sweep(float4* p, size_t n4, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = p[i];
      v.x += 1.f; v.y += 1.f; v.z += 1.f; v.w += 1.f;
      p[i] = v;
    }
}
__global__ void rd(const float4* p, size_t n4, int reps, float* out) {
  float acc = 0.f;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldcg(p + i);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 123.456f) *out = acc;
}
int main(int argc, char** argv) {
  const int reps = 50;
  for (int mb : {8, 16, 24, 32, 48, 64, 96, 128, 256, 1024}) {
    const size_t bytes = (size_t)mb << 20, n4 = bytes / 16;
    float4* p; float* o;
    cudaMalloc(&p, bytes); cudaMalloc(&o, 4);
    cudaMemset(p, 0, bytes);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int cta : {148 * 4, 148 * 8}) {
      sweep<<<cta, 256>>>(p, n4, 2);
      cudaEventRecord(a);
      sweep<<<cta, 256>>>(p, n4, reps);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double rw = 2.0 * bytes * reps / (ms * 1e-3) / 1e12;
      rd<<<cta, 256>>>(p, n4, 2, o);
      cudaEventRecord(a);
      rd<<<cta, 256>>>(p, n4, reps, o);
      cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("%4d MiB  %4d CTAs: read+write %.2f TB/s   read only %.2f TB/s\n", mb, cta, rw,
             1.0 * bytes * reps / (ms * 1e-3) / 1e12);
    }
    cudaFree(p); cudaFree(o);
  }
  return 0;
}
