"""Large-n robustness: sort 2^28 and 2^30 keys on one B200 and verify with the
device structural checker (K8).  Prints time per sort."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2605_14419_b200 as Z
from paper_2605_14419_b200 import datagen

for logn, kind in [(28, "c5"), (28, "f64normal"), (30, "c5")]:
    n = 1 << logn
    if kind == "c5":
        keys = datagen.config5_keys(0, n, n, device="cuda")
    else:
        g = torch.Generator(device="cuda").manual_seed(5)
        keys = torch.randn(n, generator=g, device="cuda", dtype=torch.float64)
    idx = torch.arange(n, dtype=torch.int64, device="cuda")
    ok, op = torch.empty_like(keys), torch.empty_like(idx)
    Z.zsort(keys, idx, out=(ok, op))
    torch.cuda.synchronize()
    t = time.perf_counter()
    _, _, st = Z.zsort(keys, idx, out=(ok, op))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    viol = Z.check_stable_permutation_device(keys, ok, op)
    print(f"n=2^{logn} {kind}: {dt*1e3:.1f} ms ({n/dt/1e9:.2f} G keys/s), violations={viol}, stats={st}", flush=True)
    del keys, idx, ok, op
    torch.cuda.empty_cache()
