"""ctypes binding of the C ABI in include/dfs_gpu.h (libdfs_b200.so, built in-tree).

There is no fallback: if the shared object is missing or was not built for
sm_100a, importing this module raises. Errors from the library become Python
exceptions with the reference's exception semantics:
DFS_E_INVALID -> ValueError (std::invalid_argument), DFS_E_RANGE -> IndexError
(std::out_of_range), everything else -> RuntimeError.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# DFS_B200_LIB points at an alternative build of the same library (A/B kernel measurements)
LIB_PATH = os.environ.get("DFS_B200_LIB") or os.path.join(HERE, "libdfs_b200.so")

DFS_OK, DFS_E_INVALID, DFS_E_RANGE, DFS_E_UNSUPPORTED, DFS_E_CUDA, DFS_E_INTERNAL = 0, -1, -2, -3, -4, -5
DFS_BF16, DFS_F32 = 0, 1
DFS_NHD, DFS_HND = 0, 1
DFS_OPT_GENERIC_SCORE, DFS_OPT_GENERIC_ATTN = 1, 2
ROPE_LAYOUTS = {"none": 0, "interleaved": 1, "half": 2}
ORDERINGS = {"raster": 0, "hilbert2d": 1, "block3d": 2, "hilbert3d": 3}

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make lib` (or __graft_entry__.build()); "
        "there is no CPU fallback for the DFSAttn path")

lib = C.CDLL(LIB_PATH)

_i64, _i32, _dbl, _p, _f = C.c_int64, C.c_int, C.c_double, C.c_void_p, C.c_float


class UnsupportedGeometry(RuntimeError):
    """DFS_E_UNSUPPORTED: outside the compiled kernels' geometry contract."""


class AttnArgs(C.Structure):
    _fields_ = [("q", _p), ("k", _p), ("v", _p), ("o", _p), ("dtype", _i32), ("in_layout", _i32),
                ("out_layout", _i32), ("heads", _i64), ("nq", _i64), ("nk", _i64), ("d", _i64),
                ("block", _i64), ("blk_ptr", _p), ("blk_idx", _p), ("out_rows", _p), ("scale", _f),
                ("force_generic", _i32), ("dv", _i64), ("in_rows", _p), ("out_peers", _p)]


MAX_PEERS = 16


class PeerHandle(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 64), ("offset", _i64)]


class AlltoallStepArgs(C.Structure):
    _fields_ = [("q", _p * MAX_PEERS), ("k", _p * MAX_PEERS), ("v", _p * MAX_PEERS), ("o", _p * MAX_PEERS),
                ("world", _i32), ("rank", _i32), ("n_local", _i64), ("heads", _i64), ("d", _i64),
                ("frames", _i64), ("height", _i64), ("width", _i64), ("block", _i64), ("sub_block", _i64),
                ("layer", _i32), ("step", _i32), ("force_dense", _i32), ("dense_out", C.POINTER(_i32)),
                ("budget_out", C.POINTER(_dbl)), ("updated_out", C.POINTER(_i32)),
                ("sparsity_out", C.POINTER(_dbl))]


class Schedule(C.Structure):
    _fields_ = [("total_steps", _i32), ("warmup_fraction", _dbl), ("phase_budgets", C.POINTER(_dbl)),
                ("n_budgets", _i32), ("phase_fraction", _dbl), ("update_interval", _i32)]


class StepArgs(C.Structure):
    _fields_ = [("q", _p), ("k", _p), ("v", _p), ("o", _p), ("n", _i64), ("heads", _i64), ("d", _i64),
                ("perm", _p), ("frames", _i64), ("height", _i64), ("width", _i64), ("block", _i64),
                ("sub_block", _i64), ("layer", _i32), ("step", _i32), ("force_dense", _i32),
                ("nonfinite", _p), ("dense_out", C.POINTER(_i32)), ("budget_out", C.POINTER(_dbl)),
                ("updated_out", C.POINTER(_i32)), ("sparsity_out", C.POINTER(_dbl)),
                ("recall_out", C.POINTER(_dbl)), ("dtype", _i32), ("dv", _i64), ("prologue", _p)]


class QkPrologueArgs(C.Structure):
    _fields_ = [("q_norm_weight", _p), ("k_norm_weight", _p), ("eps", _f), ("rope_layout", _i32),
                ("rope_cos", _p), ("rope_sin", _p)]


_SIGS = {
    "dfs_last_error": (C.c_char_p, []),
    "dfs_abi_version": (_i32, []),
    "dfs_handle_create": (_i32, [C.POINTER(_p), _i32]),
    "dfs_handle_destroy": (_i32, [_p]),
    "dfs_handle_workspace_bytes": (_i32, [_p, C.POINTER(_i64)]),
    "dfs_handle_set_option": (_i32, [_p, _i32, _i32]),
    "dfs_order_tokens": (_i32, [_i32, _i64, _i64, _i64, _p, _p, _p]),
    "dfs_invert_permutation": (_i32, [_p, _i64, _p, _p]),
    "dfs_validate_permutation": (_i32, [_p, _p, _i64, C.POINTER(_i32), _p]),
    "dfs_permute_rows": (_i32, [_p, _i32, _p, _i32, _i32, _p, _i64, _i64, _i64, _p, _i64, _p, _p]),
    "dfs_unpermute_rows": (_i32, [_p, _i32, _p, _i32, _i32, _p, _i64, _i64, _i64, _p]),
    "dfs_score_blocks": (_i32, [_p, _p, _p, _i64, _i64, _i64, _i64, _i64, _p, _p]),
    "dfs_topk_count": (_i32, [_dbl, _i64, C.POINTER(_i64)]),
    "dfs_topk_select": (_i32, [_p, _i64, _i64, _i64, _p, _p, _p]),
    "dfs_mask_bits_to_csr": (_i32, [_p, _p, _i64, _i64, _p, _p, C.POINTER(_i64), _p]),
    "dfs_lut_row_ptr": (_i32, [_i64, _i64, _i64, _p, _p]),
    "dfs_sparse_attn_fwd": (_i32, [_p, C.POINTER(AttnArgs), _p]),
    "dfs_schedule_budget_at": (_i32, [C.POINTER(Schedule), _i32, C.POINTER(_dbl)]),
    "dfs_schedule_is_update_step": (_i32, [C.POINTER(Schedule), _i32, C.POINTER(_i32)]),
    "dfs_schedule_info": (_i32, [C.POINTER(Schedule), C.POINTER(_i32), C.POINTER(_i32)]),
    "dfs_mask_cache_clear": (_i32, [_p]),
    "dfs_mask_cache_contains": (_i32, [_p, _i32, _i32, C.POINTER(_i32)]),
    "dfs_mask_cache_get": (_i32, [_p, _i32, _i32, _p, C.POINTER(_i32), C.POINTER(_i64), _p]),
    "dfs_mask_cache_store": (_i32, [_p, _i32, _i32, _p, _i64, _i64, _i32, _p]),
    "dfs_mask_cache_size": (_i32, [_p, C.POINTER(_i64)]),
    "dfs_mask_cache_info": (_i32, [_p, _i32, _i32, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i32)]),
    "dfs_cast": (_i32, [_p, _i32, _p, _i32, _i64, _p, _p]),
    "dfs_qk_prologue_apply": (_i32, [_p, _i32, _p, _p, _i32, _p, _i64, _i64, _i64, _p]),
    "dfs_alltoall_export": (_i32, [_p, C.POINTER(PeerHandle)]),
    "dfs_alltoall_import": (_i32, [C.POINTER(PeerHandle), C.POINTER(_p)]),
    "dfs_alltoall_close": (_i32, [_p]),
    "dfs_run_step": (_i32, [_p, C.POINTER(Schedule), C.POINTER(StepArgs), _p]),
    "dfs_alltoall_run_step": (_i32, [_p, C.POINTER(Schedule), C.POINTER(AlltoallStepArgs), _p]),
    "dfs_softmax_scores": (_i32, [_p, _p, _i64, _i64, _i64, _i64, _i64, _i64, _dbl, _p, _p]),
    "dfs_aggregate_scores": (_i32, [_p, _i64, _i64, _i64, _i64, _p, _p]),
    "dfs_top_indices": (_i32, [_p, _i64, _i64, _i64, _p, _p]),
    "dfs_masked_scores": (_i32, [_p, _i64, _i64, _p, _i64, _i64, _p, _p]),
    "dfs_block_recall": (_i32, [_p, _p, _p, _i32, _p, _i64, _i64, _i64, _p, _p, C.POINTER(_dbl), _p]),
    "dfs_check_finite": (_i32, [_p, _i64, _i32, C.POINTER(_i32), _p]),
    "dfs_attention_recall": (_i32, [_p, _i64, _i64, _p, _i64, _i64, C.POINTER(_dbl), _p]),
}

EXPORTS = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)  # AttributeError here = an export declared in dfs_gpu.h is missing
    _fn.restype = _res
    _fn.argtypes = _args


def last_error() -> str:
    msg = lib.dfs_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    if rc == DFS_OK:
        return
    msg = last_error()
    if rc == DFS_E_INVALID:
        raise ValueError(msg)
    if rc == DFS_E_RANGE:
        raise IndexError(msg)
    if rc == DFS_E_UNSUPPORTED:
        raise UnsupportedGeometry(msg)
    raise RuntimeError(f"dfs_gpu error {rc}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib, name)(*args))
