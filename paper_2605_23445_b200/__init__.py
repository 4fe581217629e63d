"""DFSAttn sparse self-attention path, B200-native (sm_100a CUDA behind a C ABI).

Importing the package loads libdfs_b200.so (built in-tree by `make lib` /
__graft_entry__.build()); there is no CPU fallback. The host API mirrors the
reference's dfs:: operators — see paper_2605_23445_b200.ops.
"""
from . import _capi  # noqa: F401  (raises ImportError when the CUDA library is missing)
from .ops import (  # noqa: F401
    BlockMask, GridDims, Handle, MaskCache, Permutation, QkPrologue, ScheduleConfig, ScoringParams, SparsitySchedule,
    apply_permutation, block3d_order, block_count_for, block_scores, block_sparse_attention, build_mask,
    default_handle, full_attention_output, hilbert2d_order, hilbert3d_order, invert_permutation, mean_pool,
    order_tokens, raster_order, realized_sparsity, run_step, should_update, sparse_attention_csr, topk_count,
    topk_lut, topk_select, unpermute, validate_permutation, block_recall)

LIBRARY = _capi.LIB_PATH
