// Micro-benchmark (profiling aid): FP64 FMA throughput per SM on B200 (one CTA, 8 independent
// chains per thread), for 1..32 warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/ubench_dfma_tp tools/ubench_dfma_tp.cu
#include <cstdio>
__global__ void tp(int n, long long* out, double* sink) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7;
  const double y = 1.0000001, z = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    a0 = fma(a0, y, z); a1 = fma(a1, y, z); a2 = fma(a2, y, z); a3 = fma(a3, y, z);
    a4 = fma(a4, y, z); a5 = fma(a5, y, z); a6 = fma(a6, y, z); a7 = fma(a7, y, z);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) *out = t1 - t0;
  sink[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void tpf(int n, long long* out, float* sink) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
        a6 = a0 + 6, a7 = a0 + 7;
  const float y = 1.0000001f, z = 1e-9f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    a0 = fmaf(a0, y, z); a1 = fmaf(a1, y, z); a2 = fmaf(a2, y, z); a3 = fmaf(a3, y, z);
    a4 = fmaf(a4, y, z); a5 = fmaf(a5, y, z); a6 = fmaf(a6, y, z); a7 = fmaf(a7, y, z);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) *out = t1 - t0;
  sink[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
  long long* o;
  double* s;
  float* sf;
  cudaMalloc(&o, 8);
  cudaMalloc(&s, 1024 * 8);
  cudaMalloc(&sf, 1024 * 4);
  const int n = 4096;
  for (int w : {1, 2, 4, 8, 16, 32}) {
    tp<<<1, 32 * w>>>(n, o, s);
    tp<<<1, 32 * w>>>(n, o, s);
    long long c;
    cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);
    tpf<<<1, 32 * w>>>(n, o, sf);
    tpf<<<1, 32 * w>>>(n, o, sf);
    long long cf;
    cudaMemcpy(&cf, o, 8, cudaMemcpyDeviceToHost);
    printf("warps %2d: FP64 %.1f FMA/clk/SM   FP32 %.1f FMA/clk/SM\n", w,
           8.0 * n * 32 * w / c, 8.0 * n * 32 * w / cf);
  }
  return 0;
}
