"""One profiled sort of a bench workload (for ncu launch lists / captures and
compute-sanitizer): a warm-up sort, then cudaProfilerStart, one sort,
cudaProfilerStop.  Run ncu with --profile-from-start off.

    python tools/prof_sort.py --config 4 [--mapping fitted] [--n N]
"""
import argparse
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_2605_14419_b200 as Z  # noqa: E402
from paper_2605_14419_b200 import datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--mapping", default="fitted")
ap.add_argument("--check", action="store_true")
a = ap.parse_args()
if a.config == 5:
    n = a.n or (1 << 28)
    keys = datagen.config5_keys(0, n, 1 << 31, device="cuda")
    pay = torch.arange(n, dtype=torch.int64, device="cuda")
else:
    kh, ph = datagen.baseline_config(a.config, a.n)
    keys, pay = torch.from_numpy(kh).cuda(), torch.from_numpy(ph).cuda()
cfg = Z.SortConfig(mapping=a.mapping)
k, p, st = Z.zsort(keys, pay, cfg)
torch.cuda.synchronize()
torch.cuda.profiler.start()
k, p, st = Z.zsort(keys, pay, cfg)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
if a.check:
    v = Z.check_stable_permutation_device(keys, k, p)
    assert v == 0, v
print(f"config {a.config} n {keys.numel()} stats {st}", flush=True)
