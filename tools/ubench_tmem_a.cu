// Probe (not product): tcgen05.mma kind::tf32 with the A operand in TENSOR MEMORY (the "TS"
// form) — checks the layout assumed for a TMEM-resident left operand: M = 128 rows in the 128
// lanes, K along 32-bit columns, written by tcgen05.st (32x32b: each warp its lane quadrant).
// B is the K-major 64B-swizzled smem layout the LMME kernels use. C = A B on integer-valued
// operands (exact in TF32 and FP32) against the host product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2510_03426_b200/csrc \
//        -o tools/bin/ubench_tmem_a tools/ubench_tmem_a.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_ptx.cuh"

using namespace goom::tc;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}

__global__ void __launch_bounds__(128) probe(const float* A, const float* B, float* C, int mode) {
  __shared__ __align__(1024) uint8_t bsm[16 * 1024];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // B (K = 8 x N = 128) K-major: group n/8, row n%8, 16-byte chunk k/4, word k%4
  for (int e = tid; e < 8 * 128; e += 128) {
    const int k = e / 128, n = e % 128;
    const uint32_t off = (n >> 3) * 1024 + sw64_off(n & 7, k >> 2) + (k & 3) * 4;
    *reinterpret_cast<float*>(bsm + off) = B[k * 128 + n];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t acol = 128;  // A at columns 128..135, the accumulator at 0..127
  {
    uint32_t v[8];
    const int row = warp * 32 + lane;
    for (int k = 0; k < 8; ++k) v[k] = __float_as_uint(A[row * 8 + k]);
    tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + acol, v);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = tf32_idesc(128, 128);
    const uint64_t db = sw64_desc(smem_u32(bsm));
    if (mode == 0) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
          "r"(tmem + acol), "l"(db), "r"(idesc), "r"(0));
    }
    mma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  for (int c = 0; c < 128; c += 32) {
    uint32_t v[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    for (int j = 0; j < 32; ++j) C[(warp * 32 + lane) * 128 + c + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

int main() {
  std::vector<float> A(128 * 8), B(8 * 128), C(128 * 128), R(128 * 128, 0.f);
  srand(7);
  for (auto& x : A) x = (float)(rand() % 7 - 3);
  for (auto& x : B) x = (float)(rand() % 7 - 3);
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 128; ++j)
      for (int k = 0; k < 8; ++k) R[i * 128 + j] += A[i * 8 + k] * B[k * 128 + j];
  float *dA, *dB, *dC;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dC, C.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  probe<<<1, 128>>>(dA, dB, dC, 0);
  const cudaError_t err = cudaDeviceSynchronize();
  cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 128 * 128; ++i) bad += C[i] != R[i];
  printf("TS tf32 MMA (A in TMEM, lane = row, column = k): %s, %d / %d mismatches\n",
         cudaGetErrorString(err), bad, 128 * 128);
  if (bad)
    for (int i = 0; i < 4; ++i) printf("  C[0][%d] = %g want %g\n", i, C[i], R[i]);
  return bad != 0;
}
