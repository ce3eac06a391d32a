// Micro-benchmark (profiling aid, not product): TMA (cp.async.bulk.tensor) L2/HBM -> SMEM
// throughput on B200 for the box shapes the LMME kernels use. One CTA per SM streams
// 32 KB stages through a ring (no consumer), boxes spread over a complex64 (int64)
// "matrix stack"; reports bytes/clk/SM and TB/s for an L2-resident and an HBM-sized stack.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/ubench_tma tools/ubench_tma.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int kStages = 6;
constexpr int kStage = 32 * 1024;

// shape 0: A-like 3D box (16 k x 128 rows) = 16 KB, x2 per stage
// shape 1: B-like 5D box (8 x 4 x 4 x 16 groups) = 16 KB, x2
// shape 2: row box 3D (128 cols x 16 k) = 16 KB, x2
// shape 3: A-like box with 32 k (32 x 128 rows) = 32 KB
// shape 4: 1-D bulk copy of 32 KB
__global__ void __launch_bounds__(128, 1)
    tma_bench(const __grid_constant__ CUtensorMap m3, const __grid_constant__ CUtensorMap m5,
              const __grid_constant__ CUtensorMap mrow, const __grid_constant__ CUtensorMap m32,
              const char* base, int shape, int iters, int mats, int d, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kStages];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t ring = smem_u32(smem);
  long long t0 = clock64();
  const int kblocks = d / 16;
  for (int g = 0; g < iters; ++g) {
    const int s = g % kStages;
    const uint32_t bar = smem_u32(&full[s]);
    if (g >= kStages)
      asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(bar),
                   "r"((uint32_t)(((g / kStages) - 1) & 1)) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kStage) : "memory");
    const uint32_t dst = ring + s * kStage;
    // walk (matrix, row tile, k block) so different SMs touch different lines
    const int idx = blockIdx.x * 977 + g;
    const int kb = idx % kblocks;
    const int rt = (idx / kblocks) % (d / 128);
    const int mt = (idx / kblocks / (d / 128)) % mats;
    if (shape == 0) {
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(dst), "l"(&m3), "r"(kb * 16), "r"(rt * 128), "r"(mt), "r"(bar) : "memory");
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(dst + 16384), "l"(&m3), "r"(((kb + 1) % kblocks) * 16), "r"(rt * 128), "r"(mt), "r"(bar) : "memory");
    } else if (shape == 1) {
      asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   ::"r"(dst), "l"(&m5), "r"(0), "r"(kb * 4), "r"(0), "r"(rt * 16), "r"(mt), "r"(bar) : "memory");
      asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   ::"r"(dst + 16384), "l"(&m5), "r"(0), "r"(((kb + 1) % kblocks) * 4), "r"(0), "r"(rt * 16), "r"(mt), "r"(bar) : "memory");
    } else if (shape == 2) {
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(dst), "l"(&mrow), "r"(rt * 128), "r"(kb * 16), "r"(mt), "r"(bar) : "memory");
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(dst + 16384), "l"(&mrow), "r"(rt * 128), "r"(((kb + 1) % kblocks) * 16), "r"(mt), "r"(bar) : "memory");
    } else if (shape == 3) {
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(dst), "l"(&m32), "r"((kb / 2) * 32), "r"(rt * 128), "r"(mt), "r"(bar) : "memory");
    } else {
      const char* src = base + ((size_t)mt * d * d + (size_t)(rt * 128 + kb) * d) * 8 % ((size_t)mats * d * d * 8 - kStage);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"((const char*)((uintptr_t)src & ~(uintptr_t)15)), "r"(kStage), "r"(bar) : "memory");
    }
  }
  for (int g = iters; g < iters + kStages; ++g) {
    const int s = g % kStages;
    asm volatile("{\n\t.reg .pred p;\n\tW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2;\n\t}" ::"r"(smem_u32(&full[s])),
                 "r"((uint32_t)(((g / kStages) - 1) & 1)) : "memory");
  }
  cyc[blockIdx.x] = clock64() - t0;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

int main() {
  const int d = 512;
  auto fn = enc();
  for (int mats : {16, 2048}) {  // 16 x 2 MB = 32 MB (L2-resident), 2048 x 2 MB = 4 GB
    void* buf;
    size_t bytes = (size_t)mats * d * d * 8;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    CUtensorMap m3, m5, mrow, m32;
    cuuint32_t e[5] = {1, 1, 1, 1, 1};
    {
      cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)d, (cuuint64_t)mats};
      cuuint64_t str[2] = {(cuuint64_t)d * 8, (cuuint64_t)d * d * 8};
      cuuint32_t box[3] = {16, 128, 1};
      fn(&m3, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, buf, dims, str, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      cuuint32_t box32[3] = {32, 128, 1};
      fn(&m32, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, buf, dims, str, box32, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      cuuint32_t boxr[3] = {128, 16, 1};
      fn(&mrow, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, buf, dims, str, boxr, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    {
      cuuint64_t dims[5] = {8, (cuuint64_t)d / 4, 4, (cuuint64_t)d / 8, (cuuint64_t)mats};
      cuuint64_t str[4] = {(cuuint64_t)d * 8 * 4, (cuuint64_t)d * 8, 64, (cuuint64_t)d * d * 8};
      cuuint32_t box[5] = {8, 4, 4, 16, 1};
      CUresult r = fn(&m5, CU_TENSOR_MAP_DATA_TYPE_INT64, 5, buf, dims, str, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) printf("5d encode failed %d\n", (int)r);
    }
    long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    const int smem = kStages * kStage + 1024;
    cudaFuncSetAttribute(tma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int shape = 0; shape <= 4; ++shape) {
      const int iters = 4000;
      tma_bench<<<148, 128, smem>>>(m3, m5, mrow, m32, (const char*)buf, shape, 200, mats, d, cyc);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      tma_bench<<<148, 128, smem>>>(m3, m5, mrow, m32, (const char*)buf, shape, iters, mats, d, cyc);
      cudaEventRecord(b);
      cudaError_t err = cudaDeviceSynchronize();
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      long long h[148], mx = 0;
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      const double tot = (double)iters * kStage * 148;
      printf("stack %5d MB shape %d: %s %.3f ms  %.2f TB/s  %.1f B/clk/SM\n", (int)(bytes >> 20), shape,
             cudaGetErrorString(err), ms, tot / (ms * 1e-3) / 1e12, (double)iters * kStage / mx);
    }
    cudaFree(buf);
    cudaFree(cyc);
  }
  return 0;
}
