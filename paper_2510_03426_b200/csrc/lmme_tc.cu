// tcgen05 3xTF32 LMME (placeholder until the TMEM kernel lands).
#include "goom_internal.cuh"

namespace goom {

bool lmme_tc_eligible(int n, int k, int m) { (void)n; (void)k; (void)m; return false; }

int lmme_tc(const LmmeProblem& p, cudaStream_t s) {
  (void)p; (void)s;
  return GOOM_EUNSUPPORTED;
}

}  // namespace goom
