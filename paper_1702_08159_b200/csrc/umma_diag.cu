// Self-test of the tcgen05 building blocks in umma.cuh: D (128 x 16, fp32) =
// A (128 x K, row-major) * B (16 x K, row-major)^T with kind::tf32, operands
// staged in shared memory in the interleaved K-major layout, accumulator in
// TMEM.  Exported as mck_diag_umma_tf32 so the GPU tests can pin descriptor
// encodings against torch before the fused kernels rely on them.
#include "mck_common.cuh"
#include "umma.cuh"

namespace mck {

constexpr int kDiagMaxK = 256;

__global__ void __launch_bounds__(128) k_umma_diag(const float* __restrict__ A,
                                                   const float* __restrict__ B, float* D, int K) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sa = reinterpret_cast<float*>(sm);                        // 128 x K
  float* sb = reinterpret_cast<float*>(sm + 128 * kDiagMaxK * 4);  // 16 x K
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x;
  for (int k = 0; k < K; ++k) {
    *reinterpret_cast<float*>(reinterpret_cast<char*>(sa) + umma::tile_off(t, k, 128)) = A[t * K + k];
    if (t < 16)
      *reinterpret_cast<float*>(reinterpret_cast<char*>(sb) + umma::tile_off(t, k, 16)) = B[t * K + k];
  }
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (t < 32) umma::tmem_alloc<32>(&tslot);
  umma::fence_smem_to_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = tslot;
  if (t == 0) {
    constexpr uint32_t idesc = umma::idesc_tf32(128, 16);
    for (int k0 = 0; k0 < K; k0 += 8) {
      const uint64_t ad = umma::smem_desc(reinterpret_cast<char*>(sa) + (k0 / 4) * 128 * 16, 128 * 16, 128);
      const uint64_t bd = umma::smem_desc(reinterpret_cast<char*>(sb) + (k0 / 4) * 16 * 16, 16 * 16, 128);
      umma::mma_tf32(tm, ad, bd, idesc, k0 > 0 ? 1u : 0u);
    }
    umma::commit(&bar);
  }
  mbar_wait(&bar, 0);
  umma::fence_after();
  float v[16];
  const int warp = t >> 5;
  umma::tmem_ld16(tm + ((uint32_t)(32 * warp) << 16), v);
#pragma unroll
  for (int j = 0; j < 16; ++j) D[t * 16 + j] = v[j];
  umma::fence_before();
  __syncthreads();
  if (t < 32) umma::tmem_free<32>(tm);
}

int umma_diag(const float* A, const float* B, float* D, int K, cudaStream_t st) {
  if (K < 8 || K > kDiagMaxK || K % 8) return fail_value("K must be a multiple of 8 in 8..256");
  const size_t smem = (size_t)(128 + 16) * kDiagMaxK * 4;
  MCK_TRY(check_cuda(cudaFuncSetAttribute(k_umma_diag, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem), "umma diag smem"));
  k_umma_diag<<<1, 128, smem, st>>>(A, B, D, K);
  return check_launch("k_umma_diag");
}

}  // namespace mck

extern "C" int mck_diag_umma_tf32(const float* A, const float* B, float* D, int32_t K, void* st) {
  return mck::umma_diag(A, B, D, K, reinterpret_cast<cudaStream_t>(st));
}
