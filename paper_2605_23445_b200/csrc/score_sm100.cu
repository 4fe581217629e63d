// score_sm100.cu — K3 tensor-core path (placeholder until the tcgen05 kernel lands).
#include "common.cuh"

namespace dfsgpu {

bool score_sm100_supports(int64_t, int64_t, int64_t) { return false; }
int64_t score_sm100_ws_bytes(int64_t, int64_t, int64_t, int64_t, int64_t) { return 0; }
int score_blocks_sm100(const float*, const float*, int64_t, int64_t, int64_t, int64_t, int64_t, double*, void*,
                       int64_t, cudaStream_t) {
  return fail(DFS_E_UNSUPPORTED, "score_blocks_sm100: not built");
}

}  // namespace dfsgpu
