// Micro-benchmark (profiling aid, not product): latency of the selective walk's 64 x 64
// FP64 Householder QR (selective.cu qr_regs) in one CTA, with a per-phase clock64 split
// of an instrumented copy. Built against the library's objects:
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -Ipaper_2510_03426_b200/csrc -o tools/bin/ubench_qr tools/ubench_qr.cu \
//        $(ls paper_2510_03426_b200/csrc/build/*.o | grep -v selective.o)
#include "../paper_2510_03426_b200/csrc/selective.cu"

namespace goom {
namespace {

__device__ long long g_ph[8];

// current qr_regs (tree sums) with a timestamp trace: g_tr[tid][j][pt] for j < 24,
// pt: 0 loop top, 1 after norm, 2 after scalars, 3 after V stores, 4 after barrier, 5 end
__device__ long long g_tr[256][24][6];
template <class Rt>
__device__ void qr_regs_timed(double (&x)[16], int d, const Smem<Rt>& sm, int) {
  const ColLane L = col_lane();
  const int warp = threadIdx.x >> 5, qbase = threadIdx.x & 28;
  double* Vt = sm.W;
  double* tau = sm.vec;
  double* diag = sm.vec + d;
  for (int j = 0; j < d; ++j) {
    if (warp < (j >> 3)) break;
    const bool rec = j < 24;
    if (rec) g_tr[threadIdx.x][j][0] = clock64();
    if (warp == (j >> 3)) {
      double sq[16], alpha = 0.0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int r = L.rc + 4 * i;
        sq[i] = (r > j && r < d) ? x[i] * x[i] : 0.0;
        if (r == j) alpha = x[i];
      }
      const double s = quad_sum(tree_sum16(sq));
      alpha = __shfl_sync(0xffffffffu, alpha, qbase | (j & 3));
      if (rec) g_tr[threadIdx.x][j][1] = clock64();
      if (L.c == j) {
        double t = 0.0, beta = alpha, scale = 0.0;
        if (s != 0.0) {
          const double n2 = fma(alpha, alpha, s);
          const double rn = rsqrt(n2);
          const double nrm = n2 * rn;
          beta = -copysign(nrm, alpha);
          t = fma(fabs(alpha), rn, 1.0);
          scale = copysign(__drcp_rn(fabs(alpha) + nrm), alpha);
        }
        if (rec) g_tr[threadIdx.x][j][2] = clock64();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int r = L.rc + 4 * i;
          if (r < d) Vt[j * d + r] = r > j ? x[i] * scale : (r == j ? 1.0 : 0.0);
        }
        if (L.rc == 0) {
          tau[j] = t;
          diag[j] = beta;
        }
        if (rec) g_tr[threadIdx.x][j][3] = clock64();
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"((kWarps - (j >> 3)) * 32) : "memory");
    if (rec) g_tr[threadIdx.x][j][4] = clock64();
    const double t = tau[j];
    if (t != 0.0) {
      double pr[16], v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int r = L.rc + 4 * i;
        v[i] = (r >= j && r < d) ? Vt[j * d + r] : 0.0;
        pr[i] = v[i] * x[i];
      }
      const double w = t * quad_sum(tree_sum16(pr));
      if (L.c > j && L.c < d) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fma(-w, v[i], x[i]);
      }
    }
    if (rec) g_tr[threadIdx.x][j][5] = clock64();
  }
  __syncthreads();
}


// ablations of the column loop (V = 3: named barrier only; 4: barrier + trailing update;
// 5: owner reflector + barrier, no update)
template <int V>
__device__ void qr_ablate(double (&x)[16], int d, const Smem<double>& sm) {
  const ColLane L = col_lane();
  const int warp = threadIdx.x >> 5, qbase = threadIdx.x & 28;
  double* Vt = sm.W;
  double* tau = sm.vec;
  double* diag = sm.vec + d;
  for (int j = 0; j < d; ++j) {
    if (warp < (j >> 3)) break;
    if (V == 5 && warp == (j >> 3)) {
      double sq[16], alpha = 0.0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int r = L.rc + 4 * i;
        sq[i] = (r > j && r < d) ? x[i] * x[i] : 0.0;
        if (r == j) alpha = x[i];
      }
      const double s = quad_sum(tree_sum16(sq));
      alpha = __shfl_sync(0xffffffffu, alpha, qbase | (j & 3));
      if (L.c == j) {
        double t = 0.0, beta = alpha, scale = 0.0;
        if (s != 0.0) {
          const double n2 = fma(alpha, alpha, s);
          const double rn = rsqrt(n2);
          const double nrm = n2 * rn;
          beta = -copysign(nrm, alpha);
          t = fma(fabs(alpha), rn, 1.0);
          scale = copysign(__drcp_rn(fabs(alpha) + nrm), alpha);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int r = L.rc + 4 * i;
          if (r < d) Vt[j * d + r] = r > j ? x[i] * scale : (r == j ? 1.0 : 0.0);
        }
        if (L.rc == 0) {
          tau[j] = t;
          diag[j] = beta;
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"((kWarps - (j >> 3)) * 32) : "memory");
    if (V == 4) {
      const double t = tau[j];
      if (t != 0.0) {
        double pr[16], v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int r = L.rc + 4 * i;
          v[i] = (r >= j && r < d) ? Vt[j * d + r] : 0.0;
          pr[i] = v[i] * x[i];
        }
        const double w = t * quad_sum(tree_sum16(pr));
        if (L.c > j && L.c < d) {
#pragma unroll
          for (int i = 0; i < 16; ++i) x[i] = fma(-w, v[i], x[i]);
        }
      }
    }
  }
  __syncthreads();
}

template <int V>
__global__ void __launch_bounds__(kThreads, 1) qr_bench(const double* M, int d, int reps, int t_obs,
                                                         long long* cyc, double* diag_out) {
  extern __shared__ __align__(16) char smem_raw[];
  Smem<double> sm = carve<double>(smem_raw, d);
  const ColLane L = col_lane();
  long long total = 0;
  for (int rep = 0; rep < reps; ++rep) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int r = L.rc + 4 * i;
      x[i] = (L.c < d && r < d) ? M[r * d + L.c] : 0.0;
    }
    __syncthreads();
    const long long t0 = clock64();
    if (V == 0) qr_regs(x, d, sm);
    if (V == 1) qr_regs_timed(x, d, sm, t_obs);
    if (V == 2) q_regs(x, d, true, sm);
    if (V >= 3) qr_ablate<V>(x, d, sm);
    __syncthreads();
    total += clock64() - t0;
  }
  if (threadIdx.x == 0) {
    cyc[0] = total / reps;
    for (int i = 0; i < 5; ++i) cyc[1 + i] = g_ph[i] / reps;
  }
  for (int j = threadIdx.x; j < d; j += kThreads) diag_out[j] = sm.vec[d + j];
}

}  // namespace
}  // namespace goom

int main(int argc, char** argv) {
  using namespace goom;
  const int d = argc > 1 ? atoi(argv[1]) : 64, reps = 20;
  static double h[64 * 64];
  unsigned s = 12345;
  for (int i = 0; i < d * d; ++i) {
    s = s * 1664525u + 1013904223u;
    h[i] = (s >> 8) * (1.0 / 16777216.0) - 0.5;
  }
  double *M, *diag;
  long long* cyc;
  cudaMalloc(&M, sizeof(double) * d * d);
  cudaMalloc(&diag, d * sizeof(double));
  cudaMalloc(&cyc, 8 * sizeof(long long));
  cudaMemcpy(M, h, sizeof(double) * d * d, cudaMemcpyHostToDevice);
  const size_t sb = smem_bytes<double>(d);
  cudaFuncSetAttribute(qr_bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
  cudaFuncSetAttribute(qr_bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
  cudaFuncSetAttribute(qr_bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
  long long hc[8];
  qr_bench<0><<<1, kThreads, sb>>>(M, d, reps, 0, cyc, diag);
  qr_bench<0><<<1, kThreads, sb>>>(M, d, reps, 0, cyc, diag);
  cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
  printf("qr_regs d=%d: %lld cycles (%.1f per column) [%s]\n", d, hc[0], hc[0] / (double)d,
         cudaGetErrorString(cudaDeviceSynchronize()));
  if (argc > 2) return 0;
  {
    qr_bench<1><<<1, kThreads, sb>>>(M, d, 1, 0, cyc, diag);
    cudaDeviceSynchronize();
    static long long tr[256][24][6];
    cudaMemcpyFromSymbol(tr, g_tr, sizeof(tr));
    for (int j : {16, 17, 18, 20}) {
      const long long base = tr[0 + 64][j][0];  // warp 2 (owner of 16..23), lane 0
      printf("column %d (owner warp 2):\n", j);
      for (int t : {64 + 4 * (j - 16), 64, 96, 128, 255}) {
        printf("  tid %3d:", t);
        for (int pt = 0; pt < 6; ++pt) printf(" %6lld", tr[t][j][pt] ? tr[t][j][pt] - base : -1);
        printf("\n");
      }
    }
  }
  for (int v = 3; v <= 5; ++v) {
    if (v == 3) { cudaFuncSetAttribute(qr_bench<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb); qr_bench<3><<<1, kThreads, sb>>>(M, d, reps, 0, cyc, diag); }
    if (v == 4) { cudaFuncSetAttribute(qr_bench<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb); qr_bench<4><<<1, kThreads, sb>>>(M, d, reps, 0, cyc, diag); }
    if (v == 5) { cudaFuncSetAttribute(qr_bench<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb); qr_bench<5><<<1, kThreads, sb>>>(M, d, reps, 0, cyc, diag); }
    cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    printf("ablation %d (%s): %lld cycles (%.1f per column)\n", v,
           v == 3 ? "barrier only" : v == 4 ? "barrier + update" : "owner + barrier", hc[0], hc[0] / 64.0);
  }
  qr_bench<2><<<1, kThreads, sb>>>(M, d, reps, 0, cyc, diag);
  cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
  printf("q_regs d=64: %lld cycles\n", hc[0]);
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
