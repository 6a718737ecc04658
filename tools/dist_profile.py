"""Per-rank local traffic of the multi-GPU path, for an ncu launch list: G
simulated ranks (threads) on one B200 run dist_zsort on the config-5 recipe
(int64 keys, int64 index payload), DeviceOps = the product kernels.  The
collectives are ThreadComm device copies (on real GPUs: NCCL over NVLink).

    ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        --csv --log-file gpurun_out/dist_launches.csv python tools/dist_profile.py --world 4 --log2n 26
"""
import argparse
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2605_14419_b200 import datagen  # noqa: E402
from paper_2605_14419_b200.dist import DeviceOps  # noqa: E402
from tests.dist_testlib import run_threads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=4)
ap.add_argument("--log2n", type=int, default=26, help="records per rank = 2^log2n")
ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"])
a = ap.parse_args()
dev = torch.device("cuda", 0)
per = 1 << a.log2n
n = per * a.world
keys = datagen.config5_keys(0, n, 1 << 31, device="cuda")
shards = [(keys[r * per:(r + 1) * per], torch.arange(r * per, (r + 1) * per, dtype=torch.int64, device=dev))
          for r in range(a.world)]
run_threads(shards, lambda: DeviceOps(dev), k=4096, exchange=a.exchange)  # warm-up
torch.cuda.synchronize()
torch.cuda.profiler.start()
outs = run_threads(shards, lambda: DeviceOps(dev), k=4096, exchange=a.exchange)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
ok = torch.cat([o[0] for o in outs])
assert bool((ok[1:] >= ok[:-1]).all()), "not sorted"
print(f"world {a.world} x {per} records: sizes {[o[0].numel() for o in outs]}", flush=True)
