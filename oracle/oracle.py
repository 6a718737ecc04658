"""CPU oracle for the zSort stable sort -- TEST INFRASTRUCTURE ONLY.

Python side of ``oracle/zsort_oracle.c`` (a C restatement of the reference
package's algorithm).  Used by ``tests/`` as the parity checker, by
``__graft_entry__.smoke()`` as the checker, and by ``bench.py`` as the timed
CPU baseline ("port").  The product package ``paper_2605_14419_b200`` never
imports this module.

Citations are to /root/reference/pkg/src/zsort/<file>:<line>.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

INT64_MIN = -(2**63)
INT64_MAX = 2**63 - 1
_SIGN = np.uint64(0x8000000000000000)


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        D = ctypes.c_double
        L.zo_zsort.argtypes = [P, P, I, P, P, D, P, P]
        L.zo_zsort.restype = ctypes.c_int
        L.zo_zsort_rec.argtypes = [P, P, I, P, P, I, D, D, I, P, P]
        L.zo_zsort_rec.restype = ctypes.c_int
        L.zo_first_pass.argtypes = [P, I, I, P, P, P, P]
        L.zo_variance_pass.argtypes = [P, I, I, D]
        L.zo_variance_pass.restype = D
        L.zo_bucket_of.argtypes = [I, D, D, D, D, I]
        L.zo_bucket_of.restype = I
        L.zo_estimated_center.argtypes = [I, D, D, D, D]
        L.zo_estimated_center.restype = D
        L.zo_histogram_pass.argtypes = [P, I, I, D, D, D, D, I, P]
        L.zo_exclusive_offsets.argtypes = [P, P, I]
        L.zo_exclusive_offsets.restype = I
        L.zo_scatter_pass.argtypes = [P, P, I, I, D, D, D, D, I, P, P, P, I]
        L.zo_mean_from_limbs.argtypes = [I, I, I]
        L.zo_mean_from_limbs.restype = D
        L.zo_cluster_count.argtypes = [I, D]
        L.zo_cluster_count.restype = I
        L.zo_mapping_params.argtypes = [P, I, I, P]
        L.zo_mapping_params.restype = ctypes.c_int
        L.zo_check_stable_perm.argtypes = [P, P, P, I, P]
        L.zo_check_stable_perm.restype = ctypes.c_uint64
        L.zo_mt19937_64.argtypes = [ctypes.c_uint64, P, I]
        L.zo_apply_index_swaps.argtypes = [P, P, I]
        L.zo_merge_sort_range.argtypes = [P, P, I, I, P, P]
        L.zo_insertion_sort_range.argtypes = [P, P, I, I]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ------------------------------------------------------------------ config

@dataclass(frozen=True)
class OracleConfig:
    """Mirror of SortConfig (core.py:63-89)."""

    alpha: float = 0.6
    insertion_threshold: int = 96
    counting_range_threshold: int = 65000
    depth_guard: int = 32


@dataclass
class OracleStats:
    """Mirror of SortStats (core.py:135-143)."""

    max_depth_reached: int = 0
    fallback_invocations: int = 0
    counting_sort_invocations: int = 0
    insertion_sort_invocations: int = 0
    total_scatter_passes: int = 0


def _stats(c: np.ndarray) -> OracleStats:
    return OracleStats(*[int(x) for x in c[:5]])


def _icfg(cfg: OracleConfig) -> np.ndarray:
    return np.array([cfg.insertion_threshold, cfg.counting_range_threshold, cfg.depth_guard], np.int64)


# ------------------------------------------------------------ key images

def ordered_u64(keys: np.ndarray) -> np.ndarray:
    """Order-preserving uint64 image of int64 or float64 keys.

    int64: flip the sign bit.  float64: -0.0 is canonicalised to +0.0 (IEEE
    equality, as np.argsort(kind="stable") treats them), then the standard
    sign-magnitude flip.  NaN is rejected by the product wrapper and must not
    reach here.
    """
    keys = np.ascontiguousarray(keys)
    if keys.dtype == np.int64:
        return keys.view(np.uint64) ^ _SIGN
    if keys.dtype == np.float64:
        b = keys.view(np.uint64).copy()
        b[b == _SIGN] = np.uint64(0)  # -0.0 -> +0.0
        neg = (b & _SIGN) != 0
        out = np.where(neg, ~b, b | _SIGN)
        return out.astype(np.uint64)
    raise TypeError(f"unsupported key dtype {keys.dtype}")


def f2i(keys: np.ndarray) -> np.ndarray:
    """int64 image with the same order as ordered_u64 (SURVEY §0.3 f2i with -0.0
    canonicalised), so float keys can go through the int64-only reference."""
    return (ordered_u64(keys) ^ _SIGN).view(np.int64)


# ------------------------------------------------------------------ sorts

def zsort_ref(keys, payload=None, config: OracleConfig | None = None):
    """Restatement of core.zsort (core.py:348-400) for int64 keys.

    Returns ``(sorted_keys, sorted_payload_or_None, OracleStats)`` with the
    reference's payload carry rules (core.py:168-181).
    """
    cfg = config or OracleConfig()
    keys = np.ascontiguousarray(np.asarray(keys))
    if keys.ndim != 1:
        raise ValueError("keys must be one-dimensional")
    if keys.dtype != np.int64:
        if keys.dtype.kind == "i" or (keys.dtype.kind == "u" and keys.dtype.itemsize < 8):
            keys = keys.astype(np.int64)
        elif keys.size == 0:
            keys = np.empty(0, np.int64)
        else:
            raise TypeError(f"keys must be signed 64-bit integers, got dtype {keys.dtype}")
    n = keys.size
    if payload is None:
        carry, restore = np.arange(n, dtype=np.int64), (lambda c: None)
    else:
        arr = np.asanyarray(payload)
        if arr.shape != (n,):
            raise ValueError(f"payload must have shape ({n},), got {arr.shape}")
        if arr.dtype.hasobject or arr.dtype.itemsize != 8 or arr.dtype.names:
            src = arr
            carry, restore = np.arange(n, dtype=np.int64), (lambda c: src[c])
        else:
            flat = np.ascontiguousarray(arr)
            carry, restore = flat.view(np.int64), (lambda c: c.view(flat.dtype))
    out_k = np.empty(n, np.int64)
    out_c = np.empty(n, np.int64)
    counters = np.zeros(8, np.int64)
    rc = lib().zo_zsort(_p(keys), _p(carry), n, _p(out_k), _p(out_c), float(cfg.alpha), _p(_icfg(cfg)),
                        _p(counters))
    if rc == 1:
        raise ValueError("segment too large for exact two-limb summation")
    if rc != 0:
        raise MemoryError(f"oracle zsort failed rc={rc}")
    return out_k, restore(out_c), _stats(counters)


def zsort_rec_ref(keys, k, scale, mean_est, depth=1, payload=None, config: OracleConfig | None = None):
    """Restatement of core.zsort_rec (core.py:403-437)."""
    cfg = config or OracleConfig()
    if depth < 1 or k < 2 or not (scale > 0):
        raise ValueError("invalid zsort_rec arguments")
    keys = np.ascontiguousarray(np.asarray(keys, dtype=np.int64))
    n = keys.size
    if n <= cfg.insertion_threshold:
        raise ValueError("zsort_rec requires a segment larger than the insertion threshold")
    if payload is None:
        carry, restore = np.arange(n, dtype=np.int64), (lambda c: None)
    else:
        arr = np.asanyarray(payload)
        if arr.dtype.itemsize != 8 or arr.dtype.hasobject:
            src = arr
            carry, restore = np.arange(n, dtype=np.int64), (lambda c: src[c])
        else:
            flat = np.ascontiguousarray(arr)
            carry, restore = flat.view(np.int64), (lambda c: c.view(flat.dtype))
    out_k = np.empty(n, np.int64)
    out_c = np.empty(n, np.int64)
    counters = np.zeros(8, np.int64)
    rc = lib().zo_zsort_rec(_p(keys), _p(carry), n, _p(out_k), _p(out_c), int(k), float(scale), float(mean_est),
                            int(depth), _p(_icfg(cfg)), _p(counters))
    if rc != 0:
        raise MemoryError(f"oracle zsort_rec failed rc={rc}")
    return out_k, restore(out_c), _stats(counters)


def stable_sort(keys: np.ndarray, payload: np.ndarray | None = None, config: OracleConfig | None = None):
    """Oracle stable sort for int64 or float64 keys (any payload).

    int64 keys go straight through the restated zsort; float64 keys go
    through their order-preserving int64 image (f2i) with the index as carry,
    and the original float bits are gathered back.  Returns
    ``(sorted_keys, sorted_payload_or_None, perm)``.
    """
    keys = np.ascontiguousarray(keys)
    if keys.dtype == np.float64:
        if np.isnan(keys).any():
            raise ValueError("NaN keys have no order")
        img = f2i(keys)
    elif keys.dtype == np.int64:
        img = keys
    else:
        img = keys.astype(np.int64)
    idx = np.arange(keys.size, dtype=np.int64)
    _, perm, _ = zsort_ref(img, idx, config)
    out_k = keys[perm]
    out_p = None if payload is None else np.asarray(payload)[perm]
    return out_k, out_p, perm


def check_stable_permutation(in_keys: np.ndarray, out_keys: np.ndarray, out_index: np.ndarray) -> int:
    """Structural check (verify.py:55-108): out is sorted, out_index is a
    permutation of [0, n) with out_keys == in_keys[out_index], and equal keys
    keep increasing index.  Returns 0 if stable, else (kind << 56 | position)."""
    n = in_keys.size
    a = np.ascontiguousarray(ordered_u64(in_keys))
    b = np.ascontiguousarray(ordered_u64(out_keys))
    p = np.ascontiguousarray(out_index.astype(np.int64, copy=False))
    bitmap = np.empty((n + 7) // 8 + 1, np.uint8)
    return int(lib().zo_check_stable_perm(_p(a), _p(b), _p(p), n, _p(bitmap)))


# ------------------------------------------------------- building blocks

def first_pass(keys: np.ndarray):
    """core.py:184-197 -> (exact sum, min, max)."""
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    out = np.zeros(4, np.int64)
    lib().zo_first_pass(_p(keys), 0, keys.size, _p(out[0:]), _p(out[1:]), _p(out[2:]), _p(out[3:]))
    return (int(out[0]) << 32) + int(out[1]), int(out[2]), int(out[3])


def mapping_params(keys: np.ndarray, k: int):
    """core.py:212-234 -> (mean, std, zmin, scale) or None when degenerate."""
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    out = np.zeros(4, np.float64)
    rc = lib().zo_mapping_params(_p(keys), keys.size, int(k), _p(out))
    return None if rc else tuple(float(x) for x in out)


def histogram(keys: np.ndarray, mean, std, zmin, scale, k):
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    counts = np.zeros(k, np.int64)
    lib().zo_histogram_pass(_p(keys), 0, keys.size, mean, std, zmin, scale, k, _p(counts))
    return counts


def bucket_of(key: int, mean, std, zmin, scale, k) -> int:
    return int(lib().zo_bucket_of(int(key), mean, std, zmin, scale, int(k)))


def stable_scatter(keys, carry, mean, std, zmin, scale, k):
    """core.py:259-276 over an int64 carry; returns (keys, carry, counts)."""
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    carry = np.ascontiguousarray(carry, dtype=np.int64)
    counts = histogram(keys, mean, std, zmin, scale, k)
    offs = np.zeros(k, np.int64)
    lib().zo_exclusive_offsets(_p(counts), _p(offs), k)
    dk = np.empty_like(keys)
    dc = np.empty_like(carry)
    lib().zo_scatter_pass(_p(keys), _p(carry), 0, keys.size, mean, std, zmin, scale, k, _p(offs), _p(dk), _p(dc), 0)
    return dk, dc, counts


def cluster_count(n: int, alpha: float) -> int:
    return int(lib().zo_cluster_count(int(n), float(alpha)))


# ---------------------------------------------------------------- datagen

def mt19937_64(seed: int, count: int) -> np.ndarray:
    """_mt19937.py:24-48 raw words."""
    out = np.empty(count, np.uint64)
    if count:
        lib().zo_mt19937_64(np.uint64(seed), _p(out), count)
    return out


_TWO_POW_MINUS_53 = 1.0 / 9007199254740992.0
_INT64_MAX_F = 9223372036854774784.0
_INT64_MIN_F = -9223372036854775808.0


def _to_int64(x):
    return np.clip(x, _INT64_MIN_F, _INT64_MAX_F).astype(np.int64)


def generate_family(kind: str, size: int, seed: int = 1, normal_mu=0.0, normal_sigma=1e9, pareto_alpha=1.5,
                    pareto_xm=1.0, swap_fraction=0.01, dup_range=1000) -> np.ndarray:
    """Restatement of datagen.generate key families (datagen.py:92-162)."""
    if kind == "uniform":  # datagen.py:106-107
        return mt19937_64(seed, size).view(np.int64).copy()
    if kind == "normal":  # datagen.py:110-122
        pairs = (size + 1) // 2
        raw = mt19937_64(seed, 2 * pairs)
        u1 = ((raw[:pairs] >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * _TWO_POW_MINUS_53
        u2 = (raw[pairs:] >> np.uint64(11)).astype(np.float64) * _TWO_POW_MINUS_53
        radius = np.sqrt(-2.0 * np.log(u1))
        angle = (2.0 * np.pi) * u2
        z = np.empty(2 * pairs, np.float64)
        z[0::2] = radius * np.cos(angle)
        z[1::2] = radius * np.sin(angle)
        return _to_int64(np.rint(normal_mu + normal_sigma * z[:size]))
    if kind == "skewed":  # datagen.py:125-128
        u = ((mt19937_64(seed, size) >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * _TWO_POW_MINUS_53
        return _to_int64(np.floor(pareto_xm * u ** (-1.0 / pareto_alpha)))
    if kind == "nearly_sorted":  # datagen.py:131-138
        swaps = int(swap_fraction * size)
        raw = mt19937_64(seed, size + 2 * swaps)
        keys = np.sort(raw[:size].view(np.int64))
        if swaps:
            idx = np.ascontiguousarray((raw[size:] % np.uint64(size)).astype(np.int64))
            lib().zo_apply_index_swaps(_p(keys), _p(idx), swaps)
        return keys
    if kind == "high_duplicate":  # datagen.py:141-143
        return (mt19937_64(seed, size) % np.uint64(dup_range)).astype(np.int64)
    raise ValueError(f"unknown distribution {kind!r}")


FAMILIES = ("uniform", "normal", "skewed", "nearly_sorted", "high_duplicate")


# ------------------------------------------------------ BASELINE configs

def make_config(index: int, n: int | None = None):
    """Seeded synthetic inputs for BASELINE.json configs (SURVEY §8(d) recipes).

    index 1..4 -> (keys, payload) numpy arrays.  ``n`` overrides the size for
    the scaled-down parity variants (same recipe, smaller n).  Config 5 is
    generated on the device by a counter-based generator (see
    paper_2605_14419_b200.datagen) and is not produced here.
    """
    if index == 1:  # 10^6 int64 uniform over the full range, seed 0
        n = n or 10**6
        keys = np.random.default_rng(0).integers(INT64_MIN, INT64_MAX, size=n, endpoint=True, dtype=np.int64)
    elif index == 2:  # 10^7 float64 N(0,1), seed 1
        n = n or 10**7
        keys = np.random.default_rng(1).standard_normal(n)
    elif index == 3:  # 10^7 int64 from 1000 distinct values in [0, 2^40), seed 2
        n = n or 10**7
        r = np.random.default_rng(2)
        while True:
            vals = r.integers(0, 2**40, 1000, dtype=np.int64)
            if np.unique(vals).size == 1000:
                break
        keys = vals[r.integers(0, 1000, n)]
    elif index == 4:  # 10^8 float64 lognormal skew + partially sorted half, seed 3
        n = n or 10**8
        r = np.random.default_rng(3)
        h = n // 2
        first = r.lognormal(0.0, 2.0, h)
        second = np.sort(r.lognormal(0.0, 2.0, n - h))
        swaps = int(0.01 * (n - h))  # 1% swap pairs, datagen.py:131-138 convention
        pairs = r.integers(0, n - h, size=(swaps, 2))
        second = _apply_swaps_f64(second, pairs)
        keys = np.concatenate([first, second])
    else:
        raise ValueError("configs 1..4 are host-generated; config 5 is device-generated")
    payload = np.arange(keys.size, dtype=np.int32)
    return np.ascontiguousarray(keys), payload


def _apply_swaps_f64(arr: np.ndarray, pairs: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(arr).view(np.int64).copy()
    p = np.ascontiguousarray(pairs.astype(np.int64))
    lib().zo_apply_index_swaps(_p(a), _p(p), p.shape[0])
    return a.view(np.float64)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Counter-based generator used for config 5 (device and host agree)."""
    with np.errstate(over="ignore"):
        z = (x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))
