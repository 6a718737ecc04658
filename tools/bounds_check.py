"""Bounds-check run (the compute-sanitizer stand-in: that tool is closed on
this GPU pool).  Loads the -DZSB_CHECKS build (ZSB_LIB_VARIANT=checks, built
by `bash tools/build_variant.sh checks -DZSB_CHECKS`), runs every sort path
-- tools/sanitize.py's small cases, BASELINE configs 1-4 at full size, the
config-5 recipe at 2^26 with an int64 payload, the five device families at
10^7, team runs, zsort_rec, the multi-GPU kernels on simulated ranks -- and
checks each result (CPU oracle or the device structural checker), then
asserts that no kernel saw an out-of-range shared or global index."""
import os
import subprocess
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
assert os.environ.get("ZSB_LIB_VARIANT") == "checks", "run with ZSB_LIB_VARIANT=checks"

import paper_2605_14419_b200 as Z  # noqa: E402
from paper_2605_14419_b200 import _lib, datagen  # noqa: E402

L = _lib.load()
assert L.zsb_check_violations(1) == 0, "not a fresh bounds-check build"
# 1. the sanitizer workload (small cases of every path, oracle-checked)
subprocess.run([sys.executable, os.path.join(REPO, "tools", "sanitize.py")], check=True)
dev = torch.device("cuda", 0)
# 2. BASELINE configs 1-4 at full size, device-checked
for c in (1, 2, 3, 4):
    kh, ph = datagen.baseline_config(c)
    keys = torch.from_numpy(kh).to(dev)
    for mapping in ("fitted", "paper"):
        k, p, st = Z.zsort(keys, torch.from_numpy(ph).to(dev), Z.SortConfig(mapping=mapping))
        v = Z.check_stable_permutation_device(keys, k, p)
        print(f"config {c} {mapping}: violations {v} {st}", flush=True)
        assert v == 0
# 3. config-5 recipe at 2^26, int64 payload
n = 1 << 26
keys = datagen.config5_keys(0, n, 1 << 31, device="cuda")
k, p, st = Z.zsort(keys, torch.arange(n, dtype=torch.int64, device=dev))
assert Z.check_stable_permutation_device(keys, k, p) == 0
print("config 5 (2^26)", st, flush=True)
# 4. device families
for kind in datagen.FAMILIES:
    keys = datagen.device_family(kind, 10**7, seed=2)
    k, p, st = Z.zsort(keys, torch.arange(keys.numel(), dtype=torch.int32, device=dev))
    assert Z.check_stable_permutation_device(keys, k, p) == 0
    print(kind, st, flush=True)
# 5. multi-GPU kernels on simulated ranks (real DeviceOps)
sys.path.insert(0, os.path.join(REPO, "tests"))
from tests.dist_testlib import config5_small, run_threads  # noqa: E402
from paper_2605_14419_b200.dist import DeviceOps  # noqa: E402

ks = config5_small(1 << 20)
shards = [(torch.from_numpy(np.ascontiguousarray(ks[r * ks.size // 4:(r + 1) * ks.size // 4])).to(dev),
           torch.arange(r * ks.size // 4, (r + 1) * ks.size // 4, dtype=torch.int64, device=dev)) for r in range(4)]
outs = run_threads(shards, lambda: DeviceOps(dev), k=4096)
ok = torch.cat([o[0] for o in outs]).cpu().numpy()
assert np.array_equal(np.sort(ks, kind="stable"), ok)
viol = L.zsb_check_violations(0)
print(f"bounds-check violations: {viol}", flush=True)
sys.exit(1 if viol else 0)
