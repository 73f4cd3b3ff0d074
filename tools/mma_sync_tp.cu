// Throughput probe for legacy mma.sync.m16n8k8 tf32 on sm_100a (HMMA path): 8 independent
// accumulators per warp, 4..32 warps per SM.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__global__ void k(float* out, int iters) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3, threadIdx.x * 5, threadIdx.x * 7};
  uint32_t b[8][2];
  float d[8][4] = {};
  for (int i = 0; i < 8; ++i) { b[i][0] = i + threadIdx.x; b[i][1] = i * 3; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) mma_tf32(d[i], a, b[i]);
  }
  float s = 0; for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += d[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 16 * 1024 * 4);
  int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    k<<<148 * 2, warps * 16>>>(o, 16);
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    cudaEventRecord(s);
    k<<<148 * 2, warps * 16>>>(o, iters);
    cudaEventRecord(e); cudaEventSynchronize(e);
    float ms; cudaEventElapsedTime(&ms, s, e);
    double mmas = 148.0 * 2 * (warps / 2) * iters * 8;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("warps/SM %d: %.3f ms, %.1f mma/clk/SM (at %d MHz), %.0f TFLOP/s\n", warps, ms,
           mmas / 148 / (ms * 1e-3 * clk * 1e3), clk / 1000, mmas * 2048 / (ms * 1e-3) / 1e12);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
