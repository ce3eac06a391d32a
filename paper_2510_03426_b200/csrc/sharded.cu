// Time-sharded chain scan over an NCCL communicator: the C-ABI form of sharded.py
// (SURVEY §8b goom_scan_chain_sharded_c64, §8e). Rank g of n holds leaves
// [start_g, start_g + T_local) of the global chain A_{T-1} ... A_0 and gets the global
// prefixes of its leaves:
//   1. local scan        L_t = A_t ... A_start            (goom_scan_chain_c64, no carry)
//   2. all-gather        tot_r = L_last of every rank     (one ncclAllGather, d x d complex64)
//   3. exclusive carry   C_g = tot_{g-1} (x) ... (x) tot_0 (products accumulate on the left)
//   4. apply             P_t = L_t (x) C_g                (one batched LMME, C broadcast)
// Two LMMEs per leaf, the single-GPU scan's work; results equal the single-GPU chain up to
// float32 rounding (a different tree), deterministic for a fixed (n, T_local, block).
// NCCL is resolved at run time from the libnccl the process already loaded (torch's), so
// libgoom.so has no link-time NCCL dependency.
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

struct ShardWs {
  float2* L;        // T_local d x d local prefixes (ranks > 0)
  float2* gathered; // nranks d x d totals
  float2* carry[2]; // fold ping-pong
  char* rest;       // scan / LMME workspace
  size_t rest_bytes;
};

size_t inner_bytes(int64_t T, int d, int block) {
  const size_t scan = goom_scan_chain_workspace_size(T, d, block);
  const size_t apply = goom_lmme_workspace_size(T, d, d, d);
  return scan > apply ? scan : apply;
}

}  // namespace
}  // namespace goom

using namespace goom;

extern "C" {

size_t goom_scan_chain_sharded_workspace_size(int64_t T_local, int d, int block, int nranks) {
  if (T_local < 1 || d < 1 || block < 1 || nranks < 1) return 0;
  const size_t mat = sizeof(float2) * (size_t)d * d;
  return rup(mat * T_local) + rup(mat * nranks) + 2 * rup(mat) +
         goom::inner_bytes(T_local, d, block) + 256;
}

int goom_scan_chain_sharded_c64(const goom_c64* A, goom_c64* out, int64_t T_local, int d,
                                int block, void* nccl_comm, void* ws, size_t ws_bytes,
                                void* stream) {
  if (T_local < 1 || d < 1 || block < 1) return fail(GOOM_EINVAL, "T_local, d, block must be >= 1");
  if (!A || !out || !nccl_comm || !ws) return fail(GOOM_EINVAL, "null pointer");
  const Nccl& nc = nccl();
  if (!nc.ok) return fail(GOOM_EUNSUPPORTED, "libnccl.so.2 not available in this process");
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(nccl_comm);
  int nranks = 0, rank = 0;
  if (nc.count(comm, &nranks) != ncclSuccess || nc.user_rank(comm, &rank) != ncclSuccess)
    return fail(GOOM_EINVAL, "invalid NCCL communicator");
  if (ws_bytes < goom_scan_chain_sharded_workspace_size(T_local, d, block, nranks))
    return fail(GOOM_EWORKSPACE, "sharded chain workspace too small");
  cudaStream_t st = as_stream(stream);
  const size_t mat = (size_t)d * d;
  char* p = reinterpret_cast<char*>(ws);
  ShardWs w;
  w.L = reinterpret_cast<float2*>(p);
  p += rup(sizeof(float2) * mat * T_local);
  w.gathered = reinterpret_cast<float2*>(p);
  p += rup(sizeof(float2) * mat * nranks);
  w.carry[0] = reinterpret_cast<float2*>(p);
  p += rup(sizeof(float2) * mat);
  w.carry[1] = reinterpret_cast<float2*>(p);
  p += rup(sizeof(float2) * mat);
  w.rest = p;
  w.rest_bytes = inner_bytes(T_local, d, block);
  // 1. local scan (rank 0's prefixes are already global)
  goom_c64* local = rank == 0 ? out : reinterpret_cast<goom_c64*>(w.L);
  GOOM_TRY(goom_scan_chain_c64(A, local, T_local, d, block, nullptr, w.rest, w.rest_bytes, stream));
  // 2. all-gather the chunk totals (complex64 as 2 x float32)
  const ncclResult_t r = nc.all_gather(local + (T_local - 1) * mat, w.gathered, 2 * mat, ncclFloat,
                                       comm, st);
  if (r != ncclSuccess) return fail(GOOM_ECUDA, std::string("ncclAllGather: ") + nc.error_string(r));
  if (rank == 0) return GOOM_OK;
  // 3. C_rank = tot_{rank-1} (x) ... (x) tot_0
  const float2* C = w.gathered;
  for (int q = 1, k = 0; q < rank; ++q, k ^= 1) {
    goom_operand a{w.gathered + q * mat, 0, 1}, b{C, 0, 1};
    GOOM_TRY(goom_lmme_c64(a, b, reinterpret_cast<goom_c64*>(w.carry[k]), (int64_t)mat, 1, d, d, d,
                           w.rest, w.rest_bytes, stream));
    C = w.carry[k];
  }
  // 4. P_t = L_t (x) C_rank for every local t
  goom_operand a{w.L, (int64_t)mat, 1}, b{C, 0, 1};
  return goom_lmme_c64(a, b, out, (int64_t)mat, T_local, d, d, d, w.rest, w.rest_bytes, stream);
}

}  // extern "C"
