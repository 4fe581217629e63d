// attn_sm100.cu — K5 tcgen05 path (placeholder until the kernel lands).
#include "common.cuh"

namespace dfsgpu {

bool attn_sm100_supports(const dfs_attn_args&) { return false; }
int sparse_attn_sm100(const dfs_attn_args&, float, cudaStream_t) {
  return fail(DFS_E_UNSUPPORTED, "sparse_attn_sm100: not built");
}

}  // namespace dfsgpu
