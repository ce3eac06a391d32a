// Micro-benchmark (profiling aid, not product): tcgen05 kind::tf32 MMA issue rate on
// B200 with and without concurrent shared-memory / ALU traffic from other warps,
// cta_group::1 (M=128) and cta_group::2 (M=256 across a CTA pair). Answers: does the
// tensor core's smem operand read share the 128 B/clk LSU crossbar with LDS/STS?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_mma tools/ubench_mma.cu
//   ./ubench_mma
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | (1ull << 16) | ((uint64_t)(sbo >> 4) << 32) |
         (1ull << 46) | (4ull << 61);
}
__host__ __device__ constexpr uint32_t tf32_idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

constexpr int kStage = 48 * 1024;  // A 16 KB + B 32 KB (big/small interleaved like lmme_tc)

template <int CG>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (CG == 1)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// mode: 0 idle, 1 STS.128 loop, 2 LDS.128 loop, 3 MUFU+FFMA loop, 4 LDS+STS
template <int CG, int N>
__global__ void __launch_bounds__(576, 1) bench(int iters, int mode, long long* out, float* sink, unsigned long long* traffic, int no_mma) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t rank = 0;
  if constexpr (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < (kStage + 64 * 1024) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if constexpr (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  const uint32_t base = smem_u32(smem);
  if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = tf32_idesc(128 * CG, N);
      const uint64_t dAb = sw64_desc(base, 1024), dAs = sw64_desc(base + 512, 1024);
      const uint64_t dBb = sw64_desc(base + 16384, 1024), dBs = sw64_desc(base + 16384 + 512, 1024);
      long long t0 = clock64();
      if (no_mma) { while (clock64() - t0 < (long long)iters * 6 * (N / 2)) {} }
      else for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const uint64_t adv = (uint64_t)(kk * 32) >> 4;
          mma<CG>(tmem, dAs + adv, dBb + adv, idesc, (it | kk) != 0);
          mma<CG>(tmem, dAb + adv, dBs + adv, idesc, 1);
          mma<CG>(tmem, dAb + adv, dBb + adv, idesc, 1);
        }
      }
      if constexpr (CG == 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
      else
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
      if (!no_mma) asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
      long long t1 = clock64();
      out[blockIdx.x] = t1 - t0;
      stop = 1;
    } else if (lane == 0 && CG == 2) {
      if (!no_mma) asm volatile("{\n\t.reg .pred p;\n\tW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
      out[blockIdx.x] = 0;
      stop = 1;
    }
    __syncwarp();
  } else if (warp >= 2 && mode != 0) {
    // 16 warps of traffic on a 64 KB region past the stage
    const uint32_t reg = base + kStage + (warp - 2) * 4096 + lane * 16;
    float acc = 0.f, x = lane * 1e-3f;
    int n = 0;
    while (!stop) {
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const uint32_t a = reg + ((j * 512) & 4095);
        if (mode == 1 || mode == 4)
          asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(a), "r"(j) : "memory");
        if (mode == 2 || mode == 4) {
          float4 v;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
          acc += v.x;
        }
        if (mode == 3) {
          float e;
          asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x));
          x = fmaf(e, 0.999f, x * 0.5f);
          acc += x;
        }
      }
      ++n;
    }
    if (acc == 12345.f) sink[0] = acc + n;
    if (lane == 0) atomicAdd(traffic, (unsigned long long)n * 32 * 512);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if constexpr (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

template <int CG, int N>
void run(int mode, int iters, int no_mma = 0) {
  auto k = bench<CG, N>;
  const int smem = kStage + 64 * 1024 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long* out;
  float* sink;
  cudaMalloc(&out, 148 * sizeof(long long));
  cudaMalloc(&sink, 4);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(576);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  unsigned long long* traffic;
  cudaMalloc(&traffic, 8);
  cudaLaunchKernelEx(&cfg, k, iters, mode, out, sink, traffic, no_mma);
  cudaMemset(traffic, 0, 8);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, iters, mode, out, sink, traffic, no_mma);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; i += CG) mx = h[i] > mx ? h[i] : mx;
  const double mmas = 6.0 * iters;
  const double flops = 2.0 * 128 * CG * N * 8 * mmas * (148 / CG);
  unsigned long long tb = 0;
  cudaMemcpy(&tb, traffic, 8, cudaMemcpyDeviceToHost);
  printf("cg=%d N=%d mode=%d nomma=%d: %s  %.1f clk/MMA (leader)  %.1f TF/s (tf32, all SMs)  %.3f ms  LSU %.1f B/clk/SM\n", CG, N,
         mode, no_mma, cudaGetErrorString(err), mx / mmas, no_mma ? 0.0 : flops / (ms * 1e-3) / 1e12, ms, (double)tb / 148 / mx);
  cudaFree(traffic);
  cudaFree(out);
  cudaFree(sink);
}

int main() {
  const int iters = 4096;
  for (int mode = 1; mode <= 4; ++mode) run<1, 256>(mode, iters, 1);
  for (int mode = 0; mode <= 4; ++mode) run<1, 256>(mode, iters);
  for (int mode = 0; mode <= 4; ++mode) run<1, 128>(mode, iters);
  for (int mode = 0; mode <= 4; ++mode) run<2, 256>(mode, iters);
  return 0;
}
