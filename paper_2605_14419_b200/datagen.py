"""Synthetic inputs: BASELINE configs 1-4 (numpy recipes) and config 5
(counter-based, on the device) -- SURVEY.md §8(d).

Config 5 is n = 2^31 int64 keys uniform over the full int64 range with 10%
of positions overwritten by one repeated value, sharded evenly over the
GPUs.  A counter-based generator (splitmix64 of the global index) lets every
rank build its own shard on its device and lets any checker regenerate any
key.  Choices the BASELINE text leaves open, recorded here and in DESIGN.md:
  * key_i = splitmix64(SEED_MIX + i), SEED_MIX = 4 << 56 (seed 4);
  * position i is overwritten iff the 53-bit uniform from
    splitmix64(SALT + i) is < 0.1 (Bernoulli(0.1), not exactly floor(0.1 n));
  * the repeated value is splitmix64(4).
Float-free integer arithmetic, identical on host (oracle.splitmix64) and
device.
"""

from __future__ import annotations

import torch

SEED_MIX = 4 << 56
SALT = 0x5A5A5A5A << 32
_TENTH_53 = int(0.1 * (1 << 53))


def _i64(x: int) -> int:
    x &= (1 << 64) - 1
    return x - (1 << 64) if x >= 1 << 63 else x


def _lsr(z: torch.Tensor, s: int) -> torch.Tensor:
    return (z >> s) & ((1 << (64 - s)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (wrapping arithmetic)."""
    z = x + _i64(0x9E3779B97F4A7C15)
    z = (z ^ _lsr(z, 30)) * _i64(0xBF58476D1CE4E5B9)
    z = (z ^ _lsr(z, 27)) * _i64(0x94D049BB133111EB)
    return z ^ _lsr(z, 31)


def repeated_value() -> int:
    return int(splitmix64(torch.tensor([4], dtype=torch.int64))[0])


def config5_keys(offset: int, count: int, n_total: int, device="cuda", chunk: int = 1 << 27) -> torch.Tensor:
    """Keys for global positions [offset, offset + count) of config 5."""
    assert 0 <= offset and offset + count <= n_total
    out = torch.empty(count, dtype=torch.int64, device=device)
    rep = repeated_value()
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        i = torch.arange(offset + s, offset + e, dtype=torch.int64, device=device)
        k = splitmix64(i + SEED_MIX)
        u = _lsr(splitmix64(i + SALT), 11)
        k = torch.where(u < _TENTH_53, torch.full_like(k, rep), k)
        out[s:e] = k
        del i, k, u
    return out


# ---------------------------------------------------------------- configs 1-4
# Host recipes of BASELINE configs 1-4: numpy default_rng,
# identical arrays to the committed input digests (tests/golden/golden.json,
# checked in tests/test_datagen.py against the oracle's copy of the recipes).

def baseline_config(index: int, n: int | None = None):
    """(keys, payload) numpy arrays of BASELINE config ``index`` in 1..4; ``n``
    overrides the size (same recipe) for scaled-down variants."""
    import numpy as np

    i64min, i64max = -(2**63), 2**63 - 1
    if index == 1:  # 10^6 int64 uniform over the full range, seed 0
        n = n or 10**6
        keys = np.random.default_rng(0).integers(i64min, i64max, size=n, endpoint=True, dtype=np.int64)
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
    elif index == 4:  # 10^8 float64 lognormal(0, 2) half + sorted half with 1% index-pair swaps, seed 3
        n = n or 10**8
        r = np.random.default_rng(3)
        h = n // 2
        first = r.lognormal(0.0, 2.0, h)
        second = np.sort(r.lognormal(0.0, 2.0, n - h))
        pairs = r.integers(0, n - h, size=(int(0.01 * (n - h)), 2))
        second = _swap_pairs(second, pairs)
        keys = np.concatenate([first, second])
    else:
        raise ValueError("configs 1..4 are host recipes; config 5 is config5_keys")
    return np.ascontiguousarray(keys), np.arange(keys.size, dtype=np.int32)


def _swap_pairs(arr, pairs):
    """Apply the index swaps in order (later pairs see earlier swaps), on the
    device: pairs are processed in rounds of mutually disjoint positions, each
    round a vectorised exchange."""
    import numpy as np

    a = torch.from_numpy(np.ascontiguousarray(arr).copy())
    p = torch.from_numpy(np.ascontiguousarray(pairs.astype(np.int64)))
    dev = torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")
    a, p = a.to(dev), p.to(dev)
    start, m = 0, p.shape[0]
    while start < m:
        # longest prefix of the remaining pairs whose positions are all distinct
        chunk = p[start:start + 8192]
        flat = chunk.reshape(-1)
        order = torch.argsort(flat, stable=True)
        sf = flat[order]
        dup = torch.zeros_like(flat, dtype=torch.bool)
        dup[order[1:]] = sf[1:] == sf[:-1]
        first_conflict = torch.nonzero(dup.reshape(-1, 2).any(dim=1))
        take = int(first_conflict[0]) if first_conflict.numel() else chunk.shape[0]
        take = max(take, 1)
        sel = chunk[:take]
        i, j = sel[:, 0], sel[:, 1]
        ai, aj = a[i].clone(), a[j].clone()
        a[i], a[j] = aj, ai
        start += take
    return a.cpu().numpy()


# ------------------------------------------------- device family generator
# The reference's key families (datagen.py:92-162: uniform, normal, skewed,
# nearly_sorted, high_duplicate) drawn on the device by the library's
# counter-based generator (zsb_generate, csrc/gen_kernels.cuh): key i is a
# pure function of (family, seed, i, params), so 10^8-10^9-key workloads are
# built in HBM in milliseconds and any shard can be regenerated.

FAMILIES = ("uniform", "normal", "skewed", "nearly_sorted", "high_duplicate")
FAMILY_DEFAULTS = {"normal_mu": 0.0, "normal_sigma": 1e9, "pareto_alpha": 1.5, "pareto_xm": 1.0,
                   "swap_fraction": 0.01, "dup_range": 1000}  # the reference's DistributionSpec defaults


def device_family(kind: str, n: int, seed: int = 1, offset: int = 0, n_total: int | None = None,
                  device="cuda", **params) -> torch.Tensor:
    """int64 keys of positions [offset, offset + n) of an n_total-key workload
    of family ``kind`` (defaults of the reference's DistributionSpec unless
    overridden), generated on ``device`` by the CUDA kernel."""
    import ctypes

    from . import _lib

    if kind not in FAMILIES:
        raise ValueError(f"unknown family {kind!r}; one of {FAMILIES}")
    unknown = set(params) - set(FAMILY_DEFAULTS)
    if unknown:
        raise TypeError(f"unknown family parameters {sorted(unknown)}")
    p = dict(FAMILY_DEFAULTS, **params)
    n_total = n if n_total is None else n_total
    out = torch.empty(n, dtype=torch.int64, device=device)
    arr = (ctypes.c_double * 6)(p["normal_mu"], p["normal_sigma"], p["pareto_alpha"], p["pareto_xm"],
                                p["swap_fraction"], float(p["dup_range"]))
    L = _lib.load()
    stream = torch.cuda.current_stream(out.device).cuda_stream
    _lib.check(L.zsb_generate(FAMILIES.index(kind), int(offset), int(n), int(n_total),
                              ctypes.c_uint64(seed & ((1 << 64) - 1)), arr, out.data_ptr(), stream))
    return out
