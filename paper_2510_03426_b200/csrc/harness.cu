// Long-chain harness kernels (SPEC.md harness module, run_chain):
//  * a counter-based normal generator writing GOOMs directly, keyed (seed, element
//    index) so a chain leaf t is the same on any GPU / shard / window (Philox4x32-10,
//    the reference's named generator family util.py:8, + Box-Muller);
//  * a per-prefix digest (max log-magnitude, log Frobenius norm, finiteness) so a
//    1M-long 512x512 chain (2 TiB of prefixes) can be checked without storing it.
#include "goom_internal.cuh"

namespace goom {

namespace {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += W0;
    k.y += W1;
  }
  return c;
}

// uniform in (0, 1]
__device__ __forceinline__ float u01(uint32_t x) { return (x + 1.0f) * 2.3283064365386963e-10f; }

__device__ __forceinline__ float2 goom_of(float v) {
  return make_float2(logf(fabsf(v)), v < 0.0f ? kPi : 0.0f);
}

// 4 normals per Philox counter g (Box-Muller on two uniform pairs); MUFU log / sincos:
// the generator is HBM-bound (the accurate libm paths made it 3x slower than its store).
__device__ __forceinline__ float4 normals4(uint64_t g, uint2 key) {
  const uint4 r = philox4x32_10(make_uint4((uint32_t)g, (uint32_t)(g >> 32), 0x474F4F4Du, 0u), key);
  // -2 ln u = lg2(u) * (-2 ln 2) and 2 pi u01(x) = (x + 1) * (2 pi 2^-32): one product each
  // instead of two, bit for bit the same (scaling by a power of two is exact; __logf is
  // lg2 * 0.693147182f)
  constexpr float kNeg2Ln2 = -2.0f * 0.693147182f;
  constexpr float kTwoPiUlp = 6.283185307179586f * 2.3283064365386963e-10f;
  const float a = sqrtf(__log2f(u01(r.x)) * kNeg2Ln2), t0 = (r.y + 1.0f) * kTwoPiUlp;
  const float b = sqrtf(__log2f(u01(r.z)) * kNeg2Ln2), t1 = (r.w + 1.0f) * kTwoPiUlp;
  float s0, c0, s1, c1;
  __sincosf(t0, &s0, &c0);
  __sincosf(t1, &s1, &c1);
  return make_float4(a * c0, a * s0, b * c1, b * s1);
}

__global__ void random_normal_kernel(float2* __restrict__ out, int64_t n, uint64_t seed,
                                     uint64_t offset) {
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q * 4 < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const float4 z = normals4((offset / 4) + (uint64_t)q, key);  // 4 normals per counter
    if (q * 4 + 3 < n) {
      float4* o = reinterpret_cast<float4*>(out + q * 4);
      const float2 g0 = goom_of(z.x), g1 = goom_of(z.y), g2 = goom_of(z.z), g3 = goom_of(z.w);
      o[0] = make_float4(g0.x, g0.y, g1.x, g1.y);
      o[1] = make_float4(g2.x, g2.y, g3.x, g3.y);
    } else {
      const float zz[4] = {z.x, z.y, z.z, z.w};
      for (int j = 0; j < 4 && q * 4 + j < n; ++j) out[q * 4 + j] = goom_of(zz[j]);
    }
  }
}

// the same leaves as tile-scaled fp32 (chain_ts.cu): U = the normals, q = 0, G = bits(0)
template <int kU>
__global__ void random_normal_ts_kernel(float* __restrict__ U, float* __restrict__ qv,
                                        uint32_t* __restrict__ G, int64_t n, int64_t nq,
                                        int64_t ng, uint64_t seed, uint64_t offset) {
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t whole = n / 4;  // whole quads
  int64_t q = tid;
  // kU independent counters per iteration: the Philox rounds of one hide the multiply and
  // MUFU latencies of the others (the generator is ALU-bound). Bitwise the one-counter loop;
  // d = 512 window of 32,768 leaves: kU = 1 / 2 / 3 / 4 10.85 / 9.64 / 9.31 / 9.42 ms
  // (profiles/r2_rng_interleave.txt)
  for (; q + (kU - 1) * stride < whole; q += kU * stride) {
    float4 z[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) z[u] = normals4((offset / 4) + (uint64_t)(q + u * stride), key);
#pragma unroll
    for (int u = 0; u < kU; ++u) reinterpret_cast<float4*>(U)[q + u * stride] = z[u];
  }
  for (; q * 4 < n; q += stride) {
    const float4 z = normals4((offset / 4) + (uint64_t)q, key);
    if (q * 4 + 3 < n) {
      reinterpret_cast<float4*>(U)[q] = z;
    } else {
      const float zz[4] = {z.x, z.y, z.z, z.w};
      for (int j = 0; j < 4 && q * 4 + j < n; ++j) U[q * 4 + j] = zz[j];
    }
  }
  for (int64_t i = tid; i < nq; i += stride) qv[i] = 0.0f;
  for (int64_t i = tid; i < ng; i += stride) G[i] = float_to_ordered(0.0f);
}

// one CTA per matrix: {max log, log Frobenius norm, finite(1/0), 0}
__global__ void digest_kernel(const float2* __restrict__ X, int64_t n, float4* __restrict__ out) {
  const float2* x = X + blockIdx.x * n;
  __shared__ float red[32];
  __shared__ float top_s;
  float m = kNegInf;
  int bad = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const float v = x[i].x;
    m = fmaxf(m, v);
    bad |= (isnan(v) || v == INFINITY);
  }
  m = warp_max(m);
  bad = __syncthreads_or(bad);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = kNegInf;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmaxf(t, red[w]);
    top_s = t;
  }
  __syncthreads();
  const float top = top_s;
  float acc = 0.0f;
  if (top != kNegInf)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += expf(2.0f * (x[i].x - top));
  acc = warp_sum(acc);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.0f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    const float lfro = top == kNegInf ? kNegInf : top + 0.5f * logf(s);
    out[blockIdx.x] = make_float4(top, lfro, bad ? 0.0f : 1.0f, 0.0f);
  }
}

}  // namespace
}  // namespace goom

using namespace goom;

extern "C" {

int goom_random_normal_c64(goom_c64* out, int64_t n, uint64_t seed, uint64_t offset,
                           void* stream) {
  if (n < 0) return fail(GOOM_EINVAL, "n must be >= 0");
  if (n == 0) return GOOM_OK;
  if (!out) return fail(GOOM_EINVAL, "null pointer");
  if (offset % 4) return fail(GOOM_EINVAL, "offset must be a multiple of 4");
  int64_t q = (n + 3) / 4;
  int64_t blocks = (q + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  random_normal_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
      reinterpret_cast<float2*>(out), n, seed, offset);
  GOOM_CHECK_LAUNCH("random_normal_kernel");
  return GOOM_OK;
}

int goom_random_normal_ts(float* U, float* q, uint32_t* G, int64_t T, int d, uint64_t seed,
                          uint64_t t0, void* stream) {
  if (T < 0 || d < 256 || d % 256) return fail(GOOM_EINVAL, "tile-scaled leaves need d % 256 == 0");
  if (T == 0) return GOOM_OK;
  if (!U || !q || !G) return fail(GOOM_EINVAL, "null pointer");
  const int64_t n = T * d * d, offset = (int64_t)t0 * d * d;
  if (offset % 4) return fail(GOOM_EINVAL, "offset must be a multiple of 4");
  int64_t blocks = (n / 4 + 255) / 256;
  // 64 blocks per SM of grid-stride work (16 / 32 / 64 / 128: 9.32 / 9.22 / 9.17 / 9.17 ms per
  // 32,768-leaf window; bitwise the same leaves, profiles/r2_rng_interleave.txt)
  const int64_t cap = (int64_t)num_sms() * 64;
  if (blocks > cap) blocks = cap;
  PhaseTimer timer(as_stream(stream), 0, T);
  random_normal_ts_kernel<3><<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
      U, q, G, n, T * d * (d / 256), T * (d / 256), seed, (uint64_t)offset);
  GOOM_CHECK_LAUNCH("random_normal_ts_kernel");
  timer.stop();
  return GOOM_OK;
}

int goom_digest_c64(const goom_c64* X, int64_t batch, int64_t n, float* out4, void* stream) {
  if (batch < 0 || n < 1) return fail(GOOM_EINVAL, "bad shape");
  if (batch == 0) return GOOM_OK;
  if (!X || !out4) return fail(GOOM_EINVAL, "null pointer");
  digest_kernel<<<(unsigned)batch, 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float2*>(X), n, reinterpret_cast<float4*>(out4));
  GOOM_CHECK_LAUNCH("digest_kernel");
  return GOOM_OK;
}

}  // extern "C"
