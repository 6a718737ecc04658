"""Host-side mirror of the reference's sort API, running on the B200.

Same names, signatures, argument meaning and error behaviour as
/root/reference/pkg/src/zsort/core.py, so the parity tests read like the
reference's own tests.  Every numeric pass runs in the CUDA kernels of
libzsort_b200.so through its C ABI (include/zsort_b200.h); Python only
validates arguments, moves host arrays to and from the device, and maps error
codes to exceptions.  There is no CPU fallback.

Deliberate deviations:
  * float64 keys are accepted (NaN rejected with ValueError); the reference
    raises TypeError for floats (core.py:151-165, test_zsort.py:80-82).
    -0.0 and +0.0 compare equal (IEEE), as in numpy's stable argsort.
  * 4-byte payloads move natively (the reference gathers them by index after
    the sort, core.py:168-181); the result is identical.
  * SortStats counts GPU work units (partition levels, segment scatters,
    shared-memory finish runs, exact-split fallbacks); sorted output and the
    payload permutation are bit-identical to the reference whatever the
    counters say, because a stable sort's output is unique.
"""

from __future__ import annotations

import ctypes as _ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

__all__ = [
    "DegenerateSpreadError", "FirstPassStats", "MappingParams", "PartitionPlan", "SortConfig", "SortStats",
    "all_equal", "build_mapping_params", "build_partition_plan", "cluster_count", "estimated_mean",
    "first_pass", "map_to_cluster", "stable_scatter", "zsort", "zsort_rec", "insertion_sort_stable",
    "counting_sort_stable", "fallback_sort_stable", "check_stable_permutation_device",
]

INT64_MIN = -(2**63)
INT64_MAX = 2**63 - 1
_MAX_SEGMENT = 2**32 - 1  # per-device limit of the 32-bit position arithmetic


class DegenerateSpreadError(ValueError):
    """Standard deviation underflowed to zero on a segment with unequal keys
    (core.py:55-60)."""


@dataclass(frozen=True)
class SortConfig:
    """Tuning knobs (core.py:63-89) plus the GPU bucket mapping.

    ``mapping="fitted"`` (default) fits the z-score scale to the segment's
    z-range; ``mapping="paper"`` uses Eq. 1 exactly at level 1
    (k = round(alpha*sqrt(n)), scale = k/4).  Output is identical.
    """

    alpha: float = 0.6
    insertion_threshold: int = 96
    counting_range_threshold: int = 65000
    depth_guard: int = 32
    collect_stats: bool = False
    mapping: str = "fitted"

    def __post_init__(self):
        if not (0 < self.alpha <= 2):
            raise ValueError(f"alpha must be in (0, 2], got {self.alpha}")
        if self.insertion_threshold < 1:
            raise ValueError("insertion_threshold must be >= 1")
        if self.counting_range_threshold < 1:
            raise ValueError("counting_range_threshold must be >= 1")
        if self.depth_guard < 3:
            raise ValueError("depth_guard must be >= 3")
        if self.mapping not in ("fitted", "paper"):
            raise ValueError("mapping must be 'fitted' or 'paper'")

    def to_c(self) -> _lib.ZsbConfig:
        return _lib.ZsbConfig(float(self.alpha), int(self.insertion_threshold), int(self.counting_range_threshold),
                              int(self.depth_guard), int(bool(self.collect_stats)),
                              0 if self.mapping == "fitted" else 1)


@dataclass(frozen=True)
class FirstPassStats:
    sum: int
    min_key: int
    max_key: int


@dataclass(frozen=True)
class MappingParams:
    """core.py:101-123."""

    mean: float
    std: float
    zmin: float
    scale: float
    k: int

    def __post_init__(self):
        if not (self.std > 0):
            raise ValueError("std must be positive")
        if self.zmin < 0:
            raise ValueError("zmin must be nonnegative")
        if not (self.scale > 0):
            raise ValueError("scale must be positive")
        if self.k < 2:
            raise ValueError("k must be >= 2")


@dataclass(frozen=True)
class PartitionPlan:
    k: int
    counts: np.ndarray
    offsets: np.ndarray


@dataclass
class SortStats:
    """core.py:135-143 (GPU work-unit semantics, see module docstring)."""

    max_depth_reached: int = 0
    fallback_invocations: int = 0
    counting_sort_invocations: int = 0
    insertion_sort_invocations: int = 0
    total_scatter_passes: int = 0


def cluster_count(n: int, alpha: float) -> int:
    """core.py:146-148."""
    return max(2, int(round(alpha * math.sqrt(n))))


# ------------------------------------------------------------ coercion

def _is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("zsort_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


_KEY_CODES = {torch.int64: 0, torch.float64: 1}


def _coerce_keys(keys):
    """Key dtype gate (core.py:151-165) widened to float64.

    Returns (tensor, kind) where kind is 'numpy' or 'torch'.  Integer keys
    narrower than 8 bytes are widened to int64 like the reference.
    """
    if _is_torch(keys):
        t = keys
        if t.dim() != 1:
            raise ValueError("keys must be one-dimensional")
        if t.dtype in (torch.int64, torch.float64):
            pass
        elif t.dtype in (torch.int8, torch.int16, torch.int32, torch.uint8, torch.uint16, torch.uint32):
            t = t.to(torch.int64)
        elif t.numel() == 0:
            t = t.to(torch.int64)
        else:
            raise TypeError(f"keys must be 64-bit integers or float64, got dtype {t.dtype}")
        return t.contiguous(), "torch"
    arr = np.asarray(keys)
    if arr.ndim != 1:
        raise ValueError("keys must be one-dimensional")
    if arr.size == 0 and arr.dtype not in (np.float64,):
        arr = np.empty(0, np.int64)
    if arr.dtype == np.int64 or arr.dtype == np.float64:
        arr = np.ascontiguousarray(arr)
    elif arr.dtype.kind == "i" or (arr.dtype.kind == "u" and arr.dtype.itemsize < 8):
        arr = arr.astype(np.int64)
    else:
        raise TypeError(f"keys must be signed 64-bit integers or float64, got dtype {arr.dtype}")
    return torch.from_numpy(arr), "numpy"


def _stream_ptr(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _to_dev(t: torch.Tensor, dev: torch.device) -> torch.Tensor:
    if t.device == dev:
        return t
    return t.to(dev, non_blocking=t.is_pinned())


def _np_payload_kind(arr: np.ndarray) -> int:
    if arr.dtype.hasobject or arr.dtype.names:
        return 0
    return arr.dtype.itemsize if arr.dtype.itemsize in (4, 8) else 0


# ----------------------------------------------------------------- zsort

def zsort(keys, payload=None, config: SortConfig | None = None, *, out=None):
    """Stably sort records by key on the GPU; returns ``(keys, payload, stats)``.

    Drop-in for core.zsort (core.py:348-400): inputs are never modified and
    new arrays are returned.  numpy inputs give numpy outputs (host round
    trip included); torch tensors give torch tensors on the input's device.
    ``out=(keys_out, payload_out)`` (torch tensors, e.g. pinned host buffers)
    receives the result instead of fresh allocations (extension).
    """
    return _sort(keys, payload, config, out=out)


def zsort_rec(keys, k: int, scale: float, mean_est: float, depth: int = 1, payload=None,
              config: SortConfig | None = None):
    """Recursive-phase sort of one segment given an estimated mean
    (core.py:403-437 -> _kernels.zsort_rec_driver, _kernels.py:453-473).

    Same validation as the reference (depth >= 1, k >= 2, scale > 0, more
    records than the insertion threshold).  On the device the segment starts
    at level depth + 1: one fused pass gathers min, max and the squared
    deviation around ``mean_est`` and Eq. 1 buckets it with the caller's k
    (clamped to one pass's fan-out, 2048) and scale; deeper levels size k to
    their segments.  Returns ``(keys, payload, stats)``; the sorted output is
    the unique stable order, identical to the reference's.
    """
    cfg = config if config is not None else SortConfig()
    if depth < 1:
        raise ValueError("depth must be >= 1")
    if k < 2:
        raise ValueError("k must be >= 2")
    if not (scale > 0):
        raise ValueError("scale must be positive")
    kt, _ = _coerce_keys(keys)
    if kt.numel() <= cfg.insertion_threshold:
        raise ValueError("zsort_rec requires a segment larger than the insertion threshold")
    if not math.isfinite(float(mean_est)):
        raise ValueError("mean_est must be finite")
    return _sort(keys, payload, cfg, rec=(int(k), float(scale), float(mean_est), int(depth)))


def _sort(keys, payload=None, config: SortConfig | None = None, *, out=None, rec=None):
    cfg = config if config is not None else SortConfig()
    kt, kind = _coerce_keys(keys)
    n = kt.numel()
    # payload carry rules (core.py:168-181)
    pay_t = None
    gather_src = None
    pb = 0
    if payload is not None:
        if _is_torch(payload):
            if tuple(payload.shape) != (n,):
                raise ValueError(f"payload must have shape ({n},), got {tuple(payload.shape)}")
            if payload.element_size() in (4, 8):
                pay_t, pb = payload.contiguous(), payload.element_size()
            else:
                gather_src, pb = payload, 4 if n < 2**31 else 8
        else:
            parr = np.asanyarray(payload)
            if parr.shape != (n,):
                raise ValueError(f"payload must have shape ({n},), got {parr.shape}")
            pk = _np_payload_kind(parr)
            if pk:
                pay_t, pb = torch.from_numpy(np.ascontiguousarray(parr).view(np.int32 if pk == 4 else np.int64)), pk
            else:
                gather_src, pb = parr, 4 if n < 2**31 else 8
    if n == 0:
        out_k = kt.clone() if kind == "torch" else kt.numpy().copy()
        if payload is None:
            return out_k, None, SortStats()
        return out_k, (payload.clone() if _is_torch(payload) else np.asanyarray(payload).copy()), SortStats()
    if n > _MAX_SEGMENT:
        raise ValueError("segment too large for one device; shard it with paper_2605_14419_b200.dist")
    dev = kt.device if kt.is_cuda else _device()
    L = _lib.load()
    kd = _KEY_CODES[kt.dtype]
    with torch.cuda.device(dev):
        d_keys = _to_dev(kt, dev)
        if gather_src is not None:
            d_pay = torch.arange(n, dtype=torch.int32 if pb == 4 else torch.int64, device=dev)
        elif pay_t is not None:
            d_pay = _to_dev(pay_t, dev)
        else:
            d_pay = None
        out_k = torch.empty_like(d_keys)
        out_p = torch.empty_like(d_pay) if d_pay is not None else None
        c = cfg.to_c()
        stats = (_ctypes.c_int64 * 5)()
        dp_ptr = d_pay.data_ptr() if d_pay is not None else None
        op_ptr = out_p.data_ptr() if out_p is not None else None
        if rec is None:
            ws_bytes = L.zsb_workspace_bytes(n, kd, pb, c)
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
            rc = L.zsb_sort(d_keys.data_ptr(), kd, dp_ptr, pb, out_k.data_ptr(), op_ptr, n, c,
                            ws.data_ptr(), ws_bytes, stats, _stream_ptr(dev))
        else:
            rk, rscale, rmean, rdepth = rec
            ws_bytes = L.zsb_rec_workspace_bytes(n, kd, pb, rk)
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
            rc = L.zsb_sort_rec(d_keys.data_ptr(), kd, dp_ptr, pb, out_k.data_ptr(), op_ptr, n, rk, rscale, rmean,
                                rdepth, c, ws.data_ptr(), ws_bytes, stats, _stream_ptr(dev))
        _lib.check(rc)
        st = SortStats(*[int(x) for x in stats])
        if out is not None and kind == "torch" and gather_src is None:
            ok_t, op_t = out
            ok_t.copy_(out_k, non_blocking=ok_t.is_pinned())
            if op_t is not None and out_p is not None:
                op_t.copy_(out_p, non_blocking=op_t.is_pinned())
            torch.cuda.current_stream(dev).synchronize()
            return ok_t, op_t, st
        res_p = None
        if payload is not None:
            if gather_src is not None:
                if _is_torch(gather_src):
                    res_p = gather_src[out_p.to(gather_src.device).long()]
                else:
                    res_p = gather_src[out_p.cpu().numpy()]
            elif _is_torch(payload):
                res_p = out_p if payload.is_cuda else out_p.to("cpu")
            else:
                res_p = out_p.cpu().numpy().view(np.asanyarray(payload).dtype)
        if kind == "numpy":
            return out_k.cpu().numpy(), res_p, st
        if not kt.is_cuda:
            out_k = out_k.to("cpu")
        return out_k, res_p, st


# ------------------------------------------------------- building blocks

def insertion_sort_stable(keys, payload=None):
    """core.py:288-296.  On the GPU every segment of at most the finish
    capacity is one shared-memory finish run (rank by (key, index)); longer
    inputs take the full partition pipeline.  Returns ``(keys, payload)``."""
    k, p, _ = _sort(keys, payload)
    return k, p


def counting_sort_stable(keys, min_key: int, max_key: int, payload=None,
                         range_threshold: int = SortConfig.counting_range_threshold):
    """core.py:299-323: the exact range [min_key, max_key] is validated with
    Python integers (span < 0, span >= range_threshold, keys outside the
    range: ValueError); the keys' min/max come from the K1 moments kernel.
    The finish's direct-digit mode is the GPU counting sort (one digit per
    key value when the range fits its sub-buckets).  Returns ``(keys, payload)``."""
    kt, _ = _coerce_keys(keys)
    if kt.dtype != torch.int64:
        raise TypeError("counting_sort_stable is defined for integer keys")
    span = int(max_key) - int(min_key)
    if span < 0:
        raise ValueError("max_key must be >= min_key")
    if span >= range_threshold:
        raise ValueError(f"key range {span} is not below the counting threshold {range_threshold}")
    if kt.numel():
        st = first_pass(kt)
        if st.min_key < int(min_key) or st.max_key > int(max_key):
            raise ValueError("keys fall outside [min_key, max_key]")
    k, p, _ = _sort(keys, payload)
    return k, p


def fallback_sort_stable(keys, payload=None):
    """core.py:326-335 (the reference's merge-sort termination path).  On the
    GPU termination is the exact MSD digit split inside the same pipeline
    (K7), so this is the full stable sort.  Returns ``(keys, payload)``."""
    k, p, _ = _sort(keys, payload)
    return k, p


def _moments(keys):
    kt, _ = _coerce_keys(keys)
    n = kt.numel()
    if n == 0:
        raise ValueError("first_pass requires a nonempty segment")
    if n > 2**31 - 1:
        raise ValueError("segment too large for exact two-limb summation")
    dev = kt.device if kt.is_cuda else _device()
    L = _lib.load()
    with torch.cuda.device(dev):
        d = _to_dev(kt, dev)
        ws_bytes = L.zsb_workspace_bytes(n, _KEY_CODES[kt.dtype], 0, None)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        out = (_ctypes.c_double * 8)()
        limbs = (_ctypes.c_int64 * 2)()
        mm = (_ctypes.c_uint64 * 2)()
        _lib.check(L.zsb_moments(d.data_ptr(), _KEY_CODES[kt.dtype], n, ws.data_ptr(), ws_bytes, out, limbs, mm,
                                 _stream_ptr(dev)))
    return kt, list(out), (int(limbs[0]), int(limbs[1]) & 0xFFFFFFFFFFFFFFFF), (int(mm[0]), int(mm[1]))


def _signed(u: int) -> int:
    return u - (1 << 64) if u >= 1 << 63 else u


def first_pass(keys) -> FirstPassStats:
    """Exact sum, min and max (core.py:184-197) from the K1 moments kernel."""
    kt, out, (hi, lo), (mn, mx) = _moments(keys)
    if kt.dtype != torch.int64:
        raise TypeError("first_pass is defined for integer keys")
    return FirstPassStats(sum=(hi << 32) + lo, min_key=_signed(mn), max_key=_signed(mx))


def all_equal(stats: FirstPassStats, size: int) -> bool:
    """core.py:200-209."""
    if size < 1:
        raise ValueError("size must be >= 1")
    return stats.sum == stats.min_key * size


def build_mapping_params(keys, stats: FirstPassStats, k: int) -> MappingParams:
    """core.py:212-234: mean is the correctly rounded exact quotient; the
    variance comes from the one-pass fp64 reduction of K1 (agrees with the
    reference's sequential pass to rounding noise)."""
    if k < 2:
        raise ValueError("k must be >= 2")
    kt, out, _, _ = _moments(keys)
    size = kt.numel()
    mean = stats.sum / size
    var = out[2] / size
    std = math.sqrt(var)
    if not (std > 0.0) or not math.isfinite(std):
        raise DegenerateSpreadError("standard deviation underflowed to zero; segment cannot be bucketed")
    zmin = abs((stats.min_key - mean) / std)
    return MappingParams(mean=mean, std=std, zmin=zmin, scale=k / 4, k=k)


def _params_array(params: MappingParams):
    return (_ctypes.c_double * 4)(params.mean, params.std, params.zmin, params.scale)


def build_partition_plan(keys, params: MappingParams) -> PartitionPlan:
    """core.py:248-256 on the K2 histogram kernel (parameter injection)."""
    kt, _ = _coerce_keys(keys)
    n = kt.numel()
    counts = np.zeros(params.k, np.int64)
    if n:
        dev = kt.device if kt.is_cuda else _device()
        L = _lib.load()
        with torch.cuda.device(dev):
            d = _to_dev(kt, dev)
            dc = torch.zeros(params.k, dtype=torch.int64, device=dev)
            ws_bytes = L.zsb_workspace_bytes(n, _KEY_CODES[kt.dtype], 0, None) + params.k * 4096 * 4
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
            _lib.check(L.zsb_histogram(d.data_ptr(), _KEY_CODES[kt.dtype], n, _params_array(params), params.k,
                                       dc.data_ptr(), ws.data_ptr(), ws_bytes, _stream_ptr(dev)))
            counts = dc.cpu().numpy()
    offsets = np.concatenate(([0], np.cumsum(counts)[:-1])).astype(np.int64)
    return PartitionPlan(k=params.k, counts=counts, offsets=offsets)


def map_to_cluster(key: int, params: MappingParams) -> int:
    """core.py:237-245 (one key through the device bucket function)."""
    plan = build_partition_plan(np.array([key], np.int64), params)
    return int(np.flatnonzero(plan.counts)[0])


def stable_scatter(keys, plan: PartitionPlan, params: MappingParams, payload=None):
    """core.py:259-276 on K2+K3+K4 (parameter injection)."""
    kt, kind = _coerce_keys(keys)
    n = kt.numel()
    if int(np.asarray(plan.counts).sum()) != n:
        raise ValueError("partition plan does not match segment size")
    if payload is None:
        pay = np.arange(n, dtype=np.int64)
        restore = lambda c: None  # noqa: E731
    else:
        parr = np.asanyarray(payload)
        if parr.dtype.itemsize == 8 and not parr.dtype.hasobject:
            pay = np.ascontiguousarray(parr).view(np.int64)
            restore = lambda c: c.view(parr.dtype)  # noqa: E731
        else:
            pay = np.arange(n, dtype=np.int64)
            restore = lambda c: parr[c]  # noqa: E731
    dev = kt.device if kt.is_cuda else _device()
    L = _lib.load()
    with torch.cuda.device(dev):
        d = _to_dev(kt, dev)
        dp = torch.from_numpy(pay).to(dev)
        ok = torch.empty_like(d)
        op = torch.empty_like(dp)
        ws_bytes = L.zsb_workspace_bytes(n, _KEY_CODES[kt.dtype], 8, None) + params.k * 4096 * 4
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        _lib.check(L.zsb_scatter(d.data_ptr(), _KEY_CODES[kt.dtype], dp.data_ptr(), 8, n, _params_array(params),
                                 params.k, ok.data_ptr(), op.data_ptr(), ws.data_ptr(), ws_bytes, _stream_ptr(dev)))
        return ok.cpu().numpy(), restore(op.cpu().numpy())


def estimated_mean(bucket: int, params: MappingParams) -> float:
    """core.py:279-285 / _kernels.py:103-106 (scalar arithmetic)."""
    if not (0 <= bucket < params.k):
        raise ValueError(f"bucket must be in [0, {params.k}), got {bucket}")
    return ((float(bucket) + 0.5) / params.scale - params.zmin) * params.std + params.mean


def check_stable_permutation_device(in_keys: torch.Tensor, out_keys: torch.Tensor, out_index: torch.Tensor,
                                    index_base: int = 0) -> int:
    """K8: structural stable-permutation check on the device (verify.py:55-108
    for payload = original index).  Returns the number of violations."""
    L = _lib.load()
    n = in_keys.numel()
    dev = in_keys.device
    with torch.cuda.device(dev):
        ws_bytes = L.zsb_check_workspace_bytes(n)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        res = _ctypes.c_int64(0)
        _lib.check(L.zsb_check_sorted(in_keys.data_ptr(), out_keys.data_ptr(), out_index.data_ptr(),
                                      out_index.element_size(), _KEY_CODES[in_keys.dtype], n, int(index_base),
                                      ws.data_ptr(), _ctypes.byref(res), _stream_ptr(dev)))
    return int(res.value)
