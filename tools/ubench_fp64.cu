// Micro-benchmark (profiling aid, not product): latencies of the FP64 and sync primitives
// on the selective walk's critical path (B200, one CTA of 256 threads): dependent DFMA,
// IEEE sqrt / division / reciprocal, rsqrt, 4-lane xor shuffles, CTA barrier, and a
// store -> barrier -> load round trip through shared memory.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/ubench_fp64 tools/ubench_fp64.cu
#include <cstdio>

__global__ void lat(double seed, int n, long long* out, double* sink) {
  __shared__ double sh[256];
  double x = seed + threadIdx.x * 1e-3, y = 1.0000001;
  long long t0, t1;
  // 0: dependent DFMA
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
  t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / n;
  // 1: sqrt
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 1.0;
  t1 = clock64();
  if (threadIdx.x == 0) out[1] = (t1 - t0) / n;
  // 2: division
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 3.0 / x + 1.0;
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = (t1 - t0) / n;
  // 3: reciprocal
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __drcp_rn(x) + 1.0;
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = (t1 - t0) / n;
  // 4: rsqrt
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x) + 1.0;
  t1 = clock64();
  if (threadIdx.x == 0) out[4] = (t1 - t0) / n;
  // 5: quad xor shuffle pair
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x *= 0.25;
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[5] = (t1 - t0) / n;
  // 6: __syncthreads alone
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) out[6] = (t1 - t0) / n;
  // 7: store (one thread) -> barrier -> everyone loads, dependent
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (threadIdx.x == (i & 255)) sh[i & 7] = x;
    __syncthreads();
    x = sh[i & 7] * 0.5 + 1.0;
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[7] = (t1 - t0) / n;
  // 8: exp
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = exp(-x) + 1.0;
  t1 = clock64();
  if (threadIdx.x == 0) out[8] = (t1 - t0) / n;
  // 9: log
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = log(x) + 2.0;
  t1 = clock64();
  if (threadIdx.x == 0) out[9] = (t1 - t0) / n;
  sink[threadIdx.x] = x;
}

int main() {
  long long* d_out;
  double* sink;
  cudaMalloc(&d_out, 16 * sizeof(long long));
  cudaMalloc(&sink, 256 * sizeof(double));
  const char* names[10] = {"dfma", "sqrt", "div", "drcp_rn", "rsqrt", "quad shfl+add x2",
                           "syncthreads", "sts-bar-lds", "exp", "log"};
  for (int rep = 0; rep < 2; ++rep) {
    lat<<<1, 256>>>(1.5, 4096, d_out, sink);
    cudaDeviceSynchronize();
  }
  long long h[16];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  for (int i = 0; i < 10; ++i) printf("%-18s %lld cycles\n", names[i], h[i]);
  return 0;
}
