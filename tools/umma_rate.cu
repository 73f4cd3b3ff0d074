// tcgen05 kind::tf32 issue-rate probe: M=128, K=8 per instruction, N = 16..256,
// A from shared memory (ss) or tensor memory (ts), one issuing thread per CTA,
// one CTA per SM.  Prints MMAs per SM per clock and TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1702_08159_b200/csrc/umma.cuh"
using namespace mck;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k(int iters, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x;
  for (int i = t; i < (128 + 256) * 8; i += 128) reinterpret_cast<float*>(sm)[i] = 0.001f * (i & 7);
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (t < 32) umma::tmem_alloc<512>(&tslot);
  umma::fence_smem_to_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = tslot;
  if (t == 0) {
    constexpr uint32_t idesc = umma::idesc_tf32(128, N);
    const uint64_t ad = umma::smem_desc(sm, 128 * 16, 128);
    const uint64_t bd = umma::smem_desc(sm + 128 * 8 * 4, N * 16, 128);
    long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS) umma::mma_tf32_ts(tm, tm + 256, bd, idesc, 1u);
      else umma::mma_tf32(tm, ad, bd, idesc, 1u);
    }
    umma::commit(&bar);
    mbar_wait(&bar, 0);
    long long c1 = clock64();
    cyc[blockIdx.x] = c1 - c0;
  }
  umma::fence_before();
  __syncthreads();
  if (t < 32) umma::tmem_free<512>(tm);
}

template <int N, bool TS>
void run(int sms) {
  long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  const int iters = 20000;
  const size_t smem = (128 + 256) * 8 * 4;
  cudaFuncSetAttribute(k<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<N, TS><<<sms, 128, smem>>>(iters, cyc);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<N, TS><<<sms, 128, smem>>>(iters, cyc);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long h[256]; cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
  const double flop = 2.0 * 128 * N * 8 * iters * sms;
  printf("N=%3d %s: %.2f clk/MMA, %.1f TFLOP/s (%s)\n", N, TS ? "A=TMEM" : "A=SMEM", avg / iters,
         flop / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<16, false>(sms); run<16, true>(sms); run<32, true>(sms); run<64, true>(sms);
  run<128, true>(sms); run<256, true>(sms); run<256, false>(sms);
  return 0;
}
