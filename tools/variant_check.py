"""Correctness of an experiment build (ZSB_LIB_VARIANT) on float64 keys with an
int32 index payload: bench configs 2/4 through the device structural check, and
skewed / clustered / heavy-tie inputs sized to produce team runs against the CPU
oracle.  Exit 0 when everything matches."""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_2605_14419_b200 as Z  # noqa: E402
from paper_2605_14419_b200 import datagen  # noqa: E402
from oracle import oracle as O  # noqa: E402

rng = np.random.default_rng(7)
cases = {
    "lognormal3e6": rng.lognormal(0, 2, 3_000_000),
    "normal2e6": rng.standard_normal(2_000_000),
    "clusters": np.repeat(rng.standard_normal(40), 50_000) + rng.standard_normal(2_000_000) * 1e-9,
    "ties": rng.integers(0, 300, 2_500_000).astype(np.float64),
    "fewvalues_big": np.repeat(rng.standard_normal(3), 400_000)[rng.permutation(1_200_000)],
    "negzero": np.where(rng.random(1_500_000) < 0.3, -0.0, rng.standard_normal(1_500_000)),
    "tiny_spread": 1.0 + rng.integers(0, 1 << 20, 2_000_000) * 2.0 ** -52,
}
bad = 0
for name, keys in cases.items():
    pay = np.arange(keys.size, dtype=np.int32)
    k, p, st = Z.zsort(keys, pay)
    ek, ep, _ = O.stable_sort(keys, pay)
    ok = np.array_equal(k.view(np.uint64), ek.view(np.uint64)) and np.array_equal(p, ep)
    bad += not ok
    print(f"{name:14s} n={keys.size:9d} {'ok' if ok else 'MISMATCH'} {st}", flush=True)
for c in (2, 4):
    kh, ph = datagen.baseline_config(c, None)
    keys, pay = torch.from_numpy(kh).cuda(), torch.from_numpy(ph).cuda()
    k, p, st = Z.zsort(keys, pay)
    v = Z.check_stable_permutation_device(keys, k, p)
    bad += v != 0
    print(f"config {c}: violations {v} {st}", flush=True)
sys.exit(1 if bad else 0)
