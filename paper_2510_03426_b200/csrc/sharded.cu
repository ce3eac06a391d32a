// Time-sharded chain scan over an NCCL communicator: the C-ABI form of sharded.py
// (SURVEY §8b goom_scan_chain_sharded_c64, §8e). Rank g of n holds leaves
// [start_g, start_g + T_local) of the global chain A_{T-1} ... A_0 and gets the global
// prefixes (or their digests) of its leaves. The reference's two-level tree
// (_scan_affine_stack, scan.py:181-214) is split around the one exchange:
//   1. local phases 1-2   L_t = A_t ... A_{block start} (batched over blocks) and the block
//                         carries Cx[k] (sequential fold); Cx[nb] = the chunk total
//   2. all-gather         tot_r = Cx[nb] of every rank    (one ncclAllGather, d x d complex64)
//   3. exclusive carry    C_g = tot_{g-1} (x) ... (x) tot_0 (products accumulate on the left,
//                         so the carry multiplies on the right)
//   4. carried phase 3    Cx'[k] = Cx[k] (x) C_g (one batched LMME of nb products), then
//                         P_t = L_t (x) Cx'[t / block] (one batched LMME; digested per chunk
//                         when only digests are wanted)
// About two LMMEs per leaf — the single-GPU scan's work — plus 2 nb for the carries.
// Results equal the single-GPU chain up to float32 rounding (a different tree),
// deterministic for a fixed (n, T_local, block). NCCL is resolved at run time from the
// libnccl the process already loaded (torch's), so libgoom.so has no link-time NCCL
// dependency.
#include <dlfcn.h>
#include <nccl.h>

#include "goom_internal.cuh"

namespace goom {
namespace {

struct Nccl {
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclCommCount) count = nullptr;
  decltype(&ncclCommUserRank) user_rank = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's, if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) return r;
    r.all_gather = reinterpret_cast<decltype(&ncclAllGather)>(dlsym(h, "ncclAllGather"));
    r.count = reinterpret_cast<decltype(&ncclCommCount)>(dlsym(h, "ncclCommCount"));
    r.user_rank = reinterpret_cast<decltype(&ncclCommUserRank)>(dlsym(h, "ncclCommUserRank"));
    r.error_string = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
    r.ok = r.all_gather && r.count && r.user_rank && r.error_string;
    return r;
  }();
  return n;
}

inline size_t rup(size_t x) { return (x + 255) & ~size_t(255); }

constexpr int64_t kDigestChunk = 512;  // prefixes materialised at a time for digest-only output

struct ShardWs {
  float2* L;         // T_local local products
  float2* Cx;        // nb + 1 block carries (Cx[0] unused: the identity)
  float2* Cy;        // nb carried carries Cx[k] (x) C
  float2* gathered;  // nranks chunk totals
  float2* carry[2];  // fold ping-pong
  float2* P;         // digest-only: a chunk of prefixes
  char* rest;        // LMME workspace
  size_t rest_bytes;
};

// digest-only output: prefixes are materialised a whole number of blocks at a time
int64_t digest_chunk(int64_t T, int64_t s) {
  const int64_t blocks = kDigestChunk / s > 1 ? kDigestChunk / s : 1;
  return T < blocks * s ? T : blocks * s;
}

size_t shard_bytes(int64_t T, int d, int block, int nranks, bool digests_only) {
  const int64_t s = block < T ? block : T;
  const int64_t nb = (T + s - 1) / s;
  const size_t mat = sizeof(float2) * (size_t)d * d;
  const int64_t pchunk = digests_only ? digest_chunk(T, s) : 0;
  return rup(mat * T) + 2 * rup(mat * (nb + 1)) + rup(mat * nranks) + 2 * rup(mat) +
         rup(mat * pchunk) + goom_lmme_workspace_size(T, d, d, d) + 1024;
}

int carve(void* ws, int64_t T, int d, int block, int nranks, bool digests_only, ShardWs& w) {
  const int64_t s = block < T ? block : T;
  const int64_t nb = (T + s - 1) / s;
  const size_t mat = sizeof(float2) * (size_t)d * d;
  const int64_t pchunk = digests_only ? digest_chunk(T, s) : 0;
  char* p = reinterpret_cast<char*>(ws);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += rup(bytes);
    return reinterpret_cast<float2*>(r);
  };
  w.L = take(mat * T);
  w.Cx = take(mat * (nb + 1));
  w.Cy = take(mat * (nb + 1));
  w.gathered = take(mat * nranks);
  w.carry[0] = take(mat);
  w.carry[1] = take(mat);
  w.P = pchunk ? take(mat * pchunk) : nullptr;
  w.rest = p;
  w.rest_bytes = goom_lmme_workspace_size(T, d, d, d);
  return GOOM_OK;
}

int lmme(const float2* a, int64_t sa, int64_t da, const float2* b, int64_t sb, int64_t db,
         float2* c, int64_t sc, int64_t batch, int d, const ShardWs& w, void* stream) {
  goom_operand A{a, sa, da}, B{b, sb, db};
  return goom_lmme_c64(A, B, reinterpret_cast<goom_c64*>(c), sc, batch, d, d, d, w.rest,
                       w.rest_bytes, stream);
}

int sharded_impl(const goom_c64* A_, goom_c64* out_, float* digests4, int64_t T, int d,
                 int block, void* nccl_comm, void* ws, size_t ws_bytes, void* stream) {
  if (T < 1 || d < 1 || block < 1) return fail(GOOM_EINVAL, "T_local, d, block must be >= 1");
  if (!A_ || (!out_ && !digests4) || !nccl_comm || !ws) return fail(GOOM_EINVAL, "null pointer");
  const Nccl& nc = nccl();
  if (!nc.ok) return fail(GOOM_EUNSUPPORTED, "libnccl.so.2 not available in this process");
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(nccl_comm);
  int nranks = 0, rank = 0;
  if (nc.count(comm, &nranks) != ncclSuccess || nc.user_rank(comm, &rank) != ncclSuccess)
    return fail(GOOM_EINVAL, "invalid NCCL communicator");
  const bool digests_only = out_ == nullptr;
  if (ws_bytes < shard_bytes(T, d, block, nranks, digests_only))
    return fail(GOOM_EWORKSPACE, "sharded chain workspace too small");
  cudaStream_t st = as_stream(stream);
  const float2* A = reinterpret_cast<const float2*>(A_);
  float2* out = reinterpret_cast<float2*>(out_);
  const int64_t mat = (int64_t)d * d;
  const int64_t s = block < T ? block : T;
  const int64_t nb = (T + s - 1) / s;
  ShardWs w;
  GOOM_TRY(carve(ws, T, d, block, nranks, digests_only, w));
  // 1. phase 1: L[ks] = A[ks]; L[ks+i] = A[ks+i] (x) L[ks+i-1], batched over blocks
  if (cudaMemcpy2DAsync(w.L, sizeof(float2) * mat * s, A, sizeof(float2) * mat * s,
                        sizeof(float2) * mat, nb, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "sharded phase-1 copy");
  for (int64_t i = 1; i < s; ++i) {
    const int64_t cnt = (T - i + s - 1) / s;
    if (cnt <= 0) break;
    GOOM_TRY(lmme(A + i * mat, s * mat, 1, w.L + (i - 1) * mat, s * mat, 1, w.L + i * mat, s * mat,
                  cnt, d, w, stream));
  }
  //    phase 2: Cx[1] = L[s-1]; Cx[k+1] = L[last of block k] (x) Cx[k] (the reference's fold)
  if (cudaMemcpyAsync(w.Cx + mat, w.L + (s - 1) * mat, sizeof(float2) * mat,
                      cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "sharded carry copy");
  for (int64_t kb = 1; kb < nb; ++kb) {
    const int64_t last = (kb * s + s - 1 < T ? kb * s + s - 1 : T - 1);
    GOOM_TRY(lmme(w.L + last * mat, 0, 1, w.Cx + kb * mat, 0, 1, w.Cx + (kb + 1) * mat, mat, 1,
                  d, w, stream));
  }
  // 2. all-gather the chunk totals Cx[nb] (complex64 as 2 x float32)
  const ncclResult_t r = nc.all_gather(w.Cx + nb * mat, w.gathered, 2 * mat, ncclFloat, comm, st);
  if (r != ncclSuccess) return fail(GOOM_ECUDA, std::string("ncclAllGather: ") + nc.error_string(r));
  // 3. C_rank = tot_{rank-1} (x) ... (x) tot_0
  const float2* C = nullptr;
  if (rank > 0) {
    C = w.gathered;
    for (int q = 1, k = 0; q < rank; ++q, k ^= 1) {
      GOOM_TRY(lmme(w.gathered + q * mat, 0, 1, C, 0, 1, w.carry[k], mat, 1, d, w, stream));
      C = w.carry[k];
    }
  }
  // 4. block carries with the chunk carry on the right: Cy[0] = C, Cy[k] = Cx[k] (x) C;
  //    on rank 0 block 0 has no carry (its prefixes are L) and Cy = Cx
  const float2* carries = w.Cx;
  if (C) {
    if (cudaMemcpyAsync(w.Cy, C, sizeof(float2) * mat, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), "sharded carry copy");
    if (nb > 1)
      GOOM_TRY(lmme(w.Cx + mat, mat, 1, C, 0, 1, w.Cy + mat, mat, nb - 1, d, w, stream));
    carries = w.Cy;
  }
  //    P_t = L_t (x) carries[t / s] (t < s on rank 0: P_t = L_t)
  auto phase3 = [&](int64_t b0, int64_t n, float2* dst) -> int {
    int64_t lo = b0;
    if (!C && lo < s) {  // rank 0, block 0
      const int64_t m = (s < b0 + n ? s : b0 + n) - lo;
      if (cudaMemcpyAsync(dst, w.L + lo * mat, sizeof(float2) * mat * m, cudaMemcpyDeviceToDevice,
                          st) != cudaSuccess)
        return cuda_fail(cudaGetLastError(), "sharded block-0 copy");
      dst += m * mat;
      lo += m;
    }
    const int64_t m = b0 + n - lo;
    if (m <= 0) return GOOM_OK;
    // batch index b' = t - lo; carry index t / s = (b' + lo) / s: offset the carry base so the
    // kernel's b' / s addressing lands right when lo % s == 0 (chunks are block-aligned)
    return lmme(w.L + lo * mat, mat, 1, carries + (lo / s) * mat, mat, s, dst, mat, m, d, w,
                stream);
  };
  if (!digests_only) return phase3(0, T, out);
  const int64_t chunk = digest_chunk(T, s);
  for (int64_t b0 = 0; b0 < T; b0 += chunk) {
    const int64_t n = T - b0 < chunk ? T - b0 : chunk;
    GOOM_TRY(phase3(b0, n, w.P));
    GOOM_TRY(goom_digest_c64(reinterpret_cast<goom_c64*>(w.P), n, mat, digests4 + 4 * b0, stream));
  }
  return GOOM_OK;
}

}  // namespace
}  // namespace goom

using namespace goom;

extern "C" {

size_t goom_scan_chain_sharded_workspace_size(int64_t T_local, int d, int block, int nranks) {
  if (T_local < 1 || d < 1 || block < 1 || nranks < 1) return 0;
  return goom::shard_bytes(T_local, d, block, nranks, false);
}

size_t goom_scan_chain_sharded_digest_workspace_size(int64_t T_local, int d, int block,
                                                     int nranks) {
  if (T_local < 1 || d < 1 || block < 1 || nranks < 1) return 0;
  return goom::shard_bytes(T_local, d, block, nranks, true);
}

int goom_scan_chain_sharded_c64(const goom_c64* A, goom_c64* out, int64_t T_local, int d,
                                int block, void* nccl_comm, void* ws, size_t ws_bytes,
                                void* stream) {
  if (!out) return fail(GOOM_EINVAL, "null pointer");
  return goom::sharded_impl(A, out, nullptr, T_local, d, block, nccl_comm, ws, ws_bytes, stream);
}

int goom_scan_chain_sharded_digest_c64(const goom_c64* A, float* digests4, int64_t T_local, int d,
                                       int block, void* nccl_comm, void* ws, size_t ws_bytes,
                                       void* stream) {
  if (!digests4) return fail(GOOM_EINVAL, "null pointer");
  return goom::sharded_impl(A, nullptr, digests4, T_local, d, block, nccl_comm, ws, ws_bytes,
                            stream);
}

}  // extern "C"
