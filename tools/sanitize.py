"""Small sorts that exercise every kernel path under compute-sanitizer:
level-1 sampled map + scatter + finish (C1-sized), paper mapping, recursion,
refine runs, the small single-finish path, float64 with -0.0, NaN error path,
int64 payload, and the device checker.  Exits 0 when every result matches the
CPU oracle."""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_2605_14419_b200 as Z  # noqa: E402
from oracle import oracle as O  # noqa: E402


def check(keys, pay, cfg=None):
    ok, op, _ = Z.zsort(keys, pay, cfg)
    ek, ep, _ = O.stable_sort(keys, pay)
    assert np.array_equal(ok.view(np.uint64), ek.view(np.uint64)) and np.array_equal(op, ep)


rng = np.random.default_rng(0)
n = 10**6
keys = rng.integers(-(2**63), 2**63 - 1, size=n, endpoint=True, dtype=np.int64)
check(keys, np.arange(n, dtype=np.int32))                                   # C1 shape
check(keys, np.arange(n, dtype=np.int32), Z.SortConfig(mapping="paper"))    # paper mapping
f = rng.standard_normal(300_000)
f[::1000] = -0.0
check(f, np.arange(f.size, dtype=np.int64))                                  # float64, int64 payload
check(rng.integers(0, 1000, size=400_000).astype(np.int64) << 20, np.arange(400_000, dtype=np.int32))  # ties
check(np.repeat(rng.integers(0, 2**40, 300), 100).astype(np.int64), np.arange(30_000, dtype=np.int32))
small = rng.standard_normal(5000)
check(small, np.arange(small.size, dtype=np.int32))                         # single finish
outl = rng.integers(0, 1000, size=12000, dtype=np.int64)
outl[rng.permutation(12000)[:36]] = rng.integers(10**6, 10**15, size=36)     # refine runs
check(outl, np.arange(outl.size, dtype=np.int32))
bad = small.copy()
bad[3] = np.nan
try:
    Z.zsort(bad)
    raise SystemExit("NaN not rejected")
except ValueError:
    pass
kr = rng.integers(0, 10**9, size=200_000).astype(np.int64)
ok, op, _ = Z.zsort_rec(kr, k=60, scale=15.0, mean_est=float(kr.mean()), depth=1, payload=np.arange(kr.size))
ek, ep, _ = O.stable_sort(kr, np.arange(kr.size))
assert np.array_equal(ok, ek) and np.array_equal(op, ep)
d = torch.from_numpy(keys).cuda()
ix = torch.arange(n, dtype=torch.int64, device="cuda")
k, p, _ = Z.zsort(d, ix)
assert Z.check_stable_permutation_device(d, k, p) == 0
print("sanitize workload ok", flush=True)
