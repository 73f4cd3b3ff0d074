// Shared-memory bank behaviour of 8-byte accesses for the pair kernel's two
// exchange layouts (PL: lanes on index bits 2..6; P0: lanes on bits 0,1,7,8,9)
// under several padding functions.  Run under ncu with
//   --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__host__ __device__ constexpr uint32_t deposit(uint32_t v, uint32_t mask) {
  uint32_t out = 0; int src = 0;
  for (int b = 0; b < 32; ++b) if (mask & (1u << b)) { if (v & (1u << src)) out |= 1u << b; ++src; }
  return out;
}
template <int PAD> __device__ __forceinline__ uint32_t padf(uint32_t i) {
  if (PAD == 0) return i;
  if (PAD == 1) return i + (i >> 4) + 4 * (i >> 7);   // pad2 (current)
  if (PAD == 2) return i + (i >> 4);
  if (PAD == 3) return i + (i >> 3);
  if (PAD == 4) return i + 2 * (i >> 4);
  if (PAD == 5) return i + (i >> 5);
  return i + (i >> 4) + (i >> 7);
}
template <int PAD, int LAYOUT>
__global__ void k(float2* out, int iters) {
  __shared__ float2 s[1024 + 1024 / 8 + 64];
  const uint32_t lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 1024 + 128 + 64; i += blockDim.x) s[i] = make_float2(i, i);
  __syncthreads();
  constexpr uint32_t PL = 3u | (7u << 7), P0 = 0x7Cu, FULL = 1023u;
  constexpr uint32_t P = LAYOUT ? P0 : PL;
  const uint32_t tp = deposit(lane, FULL & ~P);
  float2 acc = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 32; ++kk) {
      const float2 v = s[padf<PAD>(tp) + padf<PAD>(deposit(kk, P))];
      acc.x += v.x; acc.y += v.y;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  float2* o; cudaMalloc(&o, 148 * 256 * 8);
#define RUN(P, L) k<P, L><<<148, 256>>>(o, 100);
  RUN(0, 0) RUN(0, 1) RUN(1, 0) RUN(1, 1) RUN(2, 0) RUN(2, 1) RUN(3, 0) RUN(3, 1) RUN(4, 0) RUN(4, 1)
  RUN(5, 0) RUN(5, 1) RUN(6, 0) RUN(6, 1)
  cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
