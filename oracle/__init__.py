"""oracle — TEST INFRASTRUCTURE ONLY (the checker, never the product).

numpy/ctypes bindings to
  * ``ora``: the C restatement of the reference hot path (oracle/dfs_oracle.c,
    built to oracle/_build/libdfsoracle.so), and
  * ``ref``: the UNMODIFIED reference library built from /root/reference by
    oracle/Makefile into oracle/_ref/libdfsref.so (None when absent).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
reference arm may import this package. Both backends expose the same Python
functions so a test can run one case through each and compare bytes.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libdfsoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdfsref.so")

ORDERINGS = {"raster": 0, "hilbert2d": 1, "block3d": 2, "hilbert3d": 3}

_i64, _u64, _i32, _dbl = C.c_int64, C.c_uint64, C.c_int, C.c_double
_p = C.c_void_p


class OracleError(ValueError):
    """Raised for reference std::invalid_argument (rc -1)."""


class OracleRange(IndexError):
    """Raised for reference std::out_of_range (rc -2)."""


def build() -> None:
    """Compile the C restatement (and the reference build when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_p)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


class _Backend:
    """Same Python surface over either shared object (prefix 'oracle_' or 'dfsref_')."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        self._err = getattr(self.lib, prefix + "last_error", None)
        if self._err is not None:
            self._err.restype = C.c_char_p

    def _fn(self, name, restype=_i32):
        f = getattr(self.lib, self.prefix + name)
        f.restype = restype
        return f

    def _check(self, rc: int, what: str) -> None:
        if rc == 0:
            return
        msg = self._err().decode() if self._err is not None else what
        if rc == -2:
            raise OracleRange(msg)
        raise OracleError(msg)

    # ---- reorder ----
    def order_tokens(self, ordering: str | int, dims) -> np.ndarray:
        f, h, w = (int(x) for x in dims)
        o = ORDERINGS[ordering] if isinstance(ordering, str) else int(ordering)
        out = np.empty(f * h * w, dtype=np.uint32)
        self._check(self._fn("order_tokens")(_i32(o), _i64(f), _i64(h), _i64(w), _ptr(out)), "order")
        return out

    def hilbert3d_order(self, dims) -> np.ndarray:
        return self.order_tokens("hilbert3d", dims)

    def invert_permutation(self, fwd: np.ndarray) -> np.ndarray:
        fwd = np.ascontiguousarray(fwd, dtype=np.uint32)
        inv = np.empty_like(fwd)
        fn = self._fn("invert_permutation", None if self.prefix == "oracle_" else _i32)
        fn(_ptr(fwd), _i64(fwd.size), _ptr(inv))
        return inv

    def apply_permutation(self, fwd: np.ndarray, x: np.ndarray) -> np.ndarray:
        fwd = np.ascontiguousarray(fwd, dtype=np.uint32)
        x = _f32(x)
        out = np.empty_like(x)
        self._check(self._fn("apply_permutation")(_ptr(fwd), _i64(fwd.size), _ptr(x),
                                                 _i64(x.shape[0]), _i64(x.shape[1]), _ptr(out)),
                    "apply_permutation")
        return out

    # ---- synthetic ----
    def derive_seed(self, seed: int, path) -> int:
        arr = np.asarray(list(path), dtype=np.uint64)
        fn = self._fn("derive_seed", _u64)
        return int(fn(_u64(seed), _ptr(arr), _i32(arr.size)))

    def gen_video_field(self, dims, d: int, smoothness: float, seed: int):
        f, h, w = (int(x) for x in dims)
        n = f * h * w
        q, k, v = (np.empty((n, d), np.float32) for _ in range(3))
        self._check(self._fn("gen_video_field")(_i64(f), _i64(h), _i64(w), _i64(d), _dbl(smoothness),
                                               _u64(seed), _ptr(q), _ptr(k), _ptr(v)), "gen")
        return q, k, v

    def trajectory_at(self, dims, d, smoothness, seed, steps, noise_start, noise_end, step):
        f, h, w = (int(x) for x in dims)
        n = f * h * w
        q, k, v = (np.empty((n, d), np.float32) for _ in range(3))
        self._check(self._fn("trajectory_at")(_i64(f), _i64(h), _i64(w), _i64(d), _dbl(smoothness),
                                             _u64(seed), _i32(steps), _dbl(noise_start),
                                             _dbl(noise_end), _i32(step), _ptr(q), _ptr(k), _ptr(v)),
                    "trajectory")
        return q, k, v

    # ---- score / mask ----
    def mean_pool(self, x: np.ndarray, pool: int) -> np.ndarray:
        x = _f32(x)
        groups = -(-x.shape[0] // pool) if pool >= 1 else 0
        out = np.zeros((max(groups, 1), x.shape[1]), np.float32)
        self._check(self._fn("mean_pool")(_ptr(x), _i64(x.shape[0]), _i64(x.shape[1]), _i64(pool),
                                         _ptr(out)), "mean_pool")
        return out

    def subblock_scores(self, q, k, b: int, bs: int) -> np.ndarray:
        q, k = _f32(q), _f32(k)
        n, d = q.shape
        m = -(-n // b)
        rows = m * (b // bs) if bs >= 1 and b >= bs else 1
        out = np.zeros((rows, rows), np.float32)
        self._check(self._fn("subblock_scores")(_ptr(q), _ptr(k), _i64(n), _i64(d), _i64(b), _i64(bs),
                                               _ptr(out)), "subblock_scores")
        return out

    def block_scores(self, q, k, b: int, bs: int) -> np.ndarray:
        q, k = _f32(q), _f32(k)
        n, d = q.shape
        m = -(-n // b)
        s = np.zeros((m, m), np.float64)
        self._check(self._fn("block_scores")(_ptr(q), _ptr(k), _i64(n), _i64(d), _i64(b), _i64(bs),
                                            _ptr(s)), "block_scores")
        return s

    def topk_count(self, budget: float, m: int) -> int:
        k = C.c_int64(0)
        self._check(self._fn("topk_count")(_dbl(budget), _i64(m), C.byref(k)), "topk_count")
        return k.value

    def topk_select(self, s: np.ndarray, budget: float, b: int = 128) -> np.ndarray:
        """Returns the BlockMask byte payload (MSB-first bits)."""
        s = np.ascontiguousarray(s, dtype=np.float64)
        m = s.shape[0]
        bits = np.zeros((m * m + 7) // 8, np.uint8)
        if self.prefix == "oracle_":
            rc = self._fn("topk_select")(_ptr(s), _i64(m), _dbl(budget), _ptr(bits), None)
        else:
            rc = self._fn("topk_select")(_ptr(s), _i64(m), _dbl(budget), _i64(b), _ptr(bits))
        self._check(rc, "topk_select")
        return bits

    def build_mask(self, q, k, b: int, bs: int, budget: float) -> np.ndarray:
        q, k = _f32(q), _f32(k)
        n, d = q.shape
        m = -(-n // b)
        bits = np.zeros((m * m + 7) // 8, np.uint8)
        self._check(self._fn("build_mask")(_ptr(q), _ptr(k), _i64(n), _i64(d), _i64(b), _i64(bs),
                                          _dbl(budget), _ptr(bits)), "build_mask")
        return bits

    # ---- attention ----
    def block_sparse_attention(self, q, k, v, bits, m: int, b: int, rows=None) -> np.ndarray:
        q, k, v = _f32(q), _f32(k), _f32(v)
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        n, d = q.shape
        out = np.zeros((n, d), np.float32)
        if self.prefix == "oracle_":
            lo, hi = (0, n) if rows is None else rows
            rc = self._fn("block_sparse_attention")(_ptr(q), _ptr(k), _ptr(v), _i64(n), _i64(d),
                                                    _ptr(bits), _i64(m), _i64(b), _i64(lo), _i64(hi),
                                                    _ptr(out))
        else:
            rc = self._fn("block_sparse_attention")(_ptr(q), _ptr(k), _ptr(v), _i64(n), _i64(d),
                                                    _ptr(bits), _i64(m), _i64(b), _ptr(out))
        self._check(rc, "block_sparse_attention")
        return out

    def full_attention_output(self, q, k, v, rows=None) -> np.ndarray:
        q, k, v = _f32(q), _f32(k), _f32(v)
        nq, d = q.shape
        nk = k.shape[0]
        out = np.zeros((nq, v.shape[1]), np.float32)
        if self.prefix == "oracle_":
            lo, hi = (0, nq) if rows is None else rows
            rc = self._fn("full_attention_output")(_ptr(q), _i64(nq), _ptr(k), _ptr(v), _i64(nk), _i64(d),
                                                   _i64(lo), _i64(hi), _ptr(out))
        else:
            rc = self._fn("full_attention_output")(_ptr(q), _i64(nq), _ptr(k), _ptr(v), _i64(nk), _i64(d),
                                                   _ptr(out))
        self._check(rc, "full_attention_output")
        return out

    # ---- schedule ----
    def schedule(self, total=50, warmup=0.25, budgets=(0.3, 0.2, 0.1), phase=0.25, interval=12):
        b = np.asarray(budgets, np.float64)
        bo = np.zeros(total, np.float64)
        uo = np.zeros(total, np.uint8)
        ws, pl = C.c_int(0), C.c_int(0)
        self._check(self._fn("schedule")(_i32(total), _dbl(warmup), _ptr(b), _i32(b.size), _dbl(phase),
                                        _i32(interval), _ptr(bo), _ptr(uo), C.byref(ws), C.byref(pl)),
                    "schedule")
        return bo, uo.astype(bool), ws.value, pl.value


def _load(path, prefix):
    if not os.path.exists(path):
        return None
    return _Backend(path, prefix)


if not os.path.exists(ORACLE_SO):  # build on first import (gcc is on every box in this image)
    try:
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    except Exception:  # pragma: no cover
        pass

ora = _load(ORACLE_SO, "oracle_")
ref = _load(REF_SO, "dfsref_")


def mask_bits_to_lut(bits: np.ndarray, m: int) -> list[list[int]]:
    """BlockMask bytes -> per-row ascending selected key blocks."""
    flat = np.unpackbits(np.asarray(bits, np.uint8))[: m * m].reshape(m, m)
    return [list(np.nonzero(r)[0]) for r in flat]


def mask_bits_to_dense(bits: np.ndarray, m: int) -> np.ndarray:
    return np.unpackbits(np.asarray(bits, np.uint8))[: m * m].reshape(m, m).astype(bool)


def dense_to_mask_bits(dense: np.ndarray) -> np.ndarray:
    m = dense.shape[0]
    flat = np.zeros(((m * m + 7) // 8) * 8, np.uint8)
    flat[: m * m] = dense.reshape(-1).astype(np.uint8)
    return np.packbits(flat)


def fnv1a64(data: bytes) -> str:
    h = 0xCBF29CE484222325
    for byte in data:
        h ^= byte
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def fnv1a64_np(arr: np.ndarray) -> str:
    """FNV-1a-64 over the little-endian bytes of arr."""
    return fnv1a64(np.ascontiguousarray(arr).tobytes())
