"""Benchmark: stable-sorted 64-bit keys/s on B200 vs the HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4]

One step = one full stable sort (keys + payload) of the configured workload.
N=1 default workload: BASELINE config 4 (10^8 float64 keys, lognormal half +
nearly sorted half, seed 3, int32 original-index payload): the largest
BASELINE config that fits one GPU and that the reference can run, inside the
north star's 10^8-10^9 range.  N>1: config 5 (2^31 int64 keys with an int64
index payload, sharded 2^31/N per GPU: strong scaling over NCCL).
Inputs are resident in HBM for `value`; `e2e` times the public API on
pinned host buffers (H2D + sort + D2H inside the timed region).  L2 is
flushed (512 MiB write) between timed steps, outside the timed region.

`--impl reference` times the reference algorithm's CPU implementation (the
C restatement in oracle/, single-threaded like the reference) on the host,
same workload and metric, each step a bounded sample of the workload (every
4th key of C4: same shape, ~2 s of CPU).  Under torchrun only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "stable-sorted 64-bit keys/sec at 1/2/4/8 B200; achieved HBM GB/s vs roofline"
CONFIG_DESC = {
    1: "C1: 1e6 int64 uniform full range (seed 0), int32 index payload",
    2: "C2: 1e7 float64 N(0,1) (seed 1), int32 index payload",
    3: "C3: 1e7 int64 from 1000 distinct values in [0,2^40) (seed 2), int32 index payload",
    4: "C4: 1e8 float64 lognormal(0,2) half + sorted half with 1% swaps (seed 3), int32 index payload",
    5: "C5: 2^31/N int64 per GPU (uniform, 10% one repeated value, seed 4), int64 index payload",
    9: "X9: 1e9 int64 uniform full range (seed 9), int32 index payload",
}


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# CPU sample of each workload for the reference arm and cpu_baseline (bounded
# CPU time): a stride keeps the workload's shape (C4: lognormal half + nearly
# sorted half)
CPU_SAMPLE_STRIDE = {1: 1, 2: 1, 3: 1, 4: 4, 9: 40}


def cpu_sample(cfg: int, keys, payload):
    st = CPU_SAMPLE_STRIDE.get(cfg, 1)
    if st == 1:
        return keys, payload, f"full workload ({keys.size} keys)"
    ks = np.ascontiguousarray(keys[::st])
    return ks, np.arange(ks.size, dtype=payload.dtype), (f"every {st}th key of the workload ({ks.size} keys, same "
                                                         f"shape), index payload")


def bench_config(args, n, pb):
    """The config dict both arms print (identical keys and values)."""
    return {"workload": CONFIG_DESC[args.config], "n_per_gpu": int(n), "payload_bytes": int(pb),
            "mapping": args.mapping, "l2": "flushed (512 MiB write) between timed steps",
            "parallelism": "single" if args.gpus == 1 else f"dp{args.gpus}"}


def make_workload(cfg: int, rank: int = 0, world: int = 1):
    """Host arrays (keys, payload) for one rank."""
    from paper_2605_14419_b200 import datagen

    if cfg in (1, 2, 3, 4):
        return datagen.baseline_config(cfg)
    if cfg == 9:
        keys = np.random.default_rng(9).integers(-(2**63), 2**63 - 1, size=10**9, endpoint=True, dtype=np.int64)
        return keys, np.arange(keys.size, dtype=np.int32)
    raise ValueError(cfg)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def run_reference(args, rank: int):
    """CPU arm: the reference algorithm's C restatement on the host (1 core)."""
    from oracle import oracle as O

    if args.config == 5:  # the reference cannot run config 5 (n > 2^31 - 1, core.py:51-52): one 2^24 shard
        from paper_2605_14419_b200 import datagen
        import torch
        n_full = 1 << 31
        keys = datagen.config5_keys(0, 1 << 24, n_full, device="cpu").numpy()
        payload = np.arange(keys.size, dtype=np.int64)
        sample = f"first 2^24 keys of config 5 (the reference cannot sort n > 2^31 - 1)"
        n_full_local = n_full // args.gpus
        pb = 8
    else:
        keys_w, pay_w = make_workload(args.config)
        keys, payload, sample = cpu_sample(args.config, keys_w, pay_w)
        n_full_local, pb = keys_w.size, pay_w.dtype.itemsize
        del keys_w, pay_w
    n = keys.size
    for _ in range(args.warmup if args.warmup < 2 else 1):
        O.stable_sort(keys[: min(n, 10**6)], payload[: min(n, 10**6)])
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.stable_sort(keys, payload)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = n * len(times) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
        "scaling": "weak" if args.config != 5 else "strong", "vs_baseline": None,
        "dtype": "int64" if keys.dtype == np.int64 else "f64",
        "data": "synthetic", "config": bench_config(args, n_full_local, pb),
        "cpu_baseline": {"value": value, "unit": "keys/s", "cores": 1, "kind": "port",
                         "sample": f"{sample} x {len(times)} steps (oracle/zsort_oracle.c, the reference algorithm's "
                                   f"C restatement); the reference is single-threaded by design (SPEC.md:222-223); "
                                   f"host cpu_count={os.cpu_count()}"},
        "e2e": {"value": value, "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(keys, payload, sample, budget_s=12.0, max_reps=5):
    from oracle import oracle as O

    times = []
    t_start = time.perf_counter()
    while len(times) < max_reps and (time.perf_counter() - t_start) < budget_s:
        t0 = time.perf_counter()
        O.stable_sort(keys, payload)
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    return {"value": keys.size / med, "unit": "keys/s", "cores": 1, "kind": "port",
            "sample": f"{sample}, median of {len(times)} runs of the oracle restatement "
                      f"(oracle/zsort_oracle.c) on this host; cpu_count={os.cpu_count()}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=None, help="default: 4 at N=1, 5 at N>1")
    ap.add_argument("--mapping", default="fitted", choices=["fitted", "paper"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-comparators", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the paper-mapping and config-5 single-GPU legs")
    ap.add_argument("--exchange", default="auto", choices=["auto", "p2p", "nccl"],
                    help="N>1: fused peer-store exchange or NCCL all_to_all (auto: p2p when peers are accessible)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config is None:
        args.config = 4 if max(world, args.gpus) == 1 else 5
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, rank)
        return

    import torch

    import paper_2605_14419_b200 as Z
    from paper_2605_14419_b200 import _lib

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        return run_dist(args, rank, world, dev)
    if args.config == 5:
        raise SystemExit("config 5 at N=1 is reported inside the default line (c5_single_gpu); use --gpus N>1")
    L = _lib.load()
    keys_h, pay_h = make_workload(args.config, rank, world)
    n = keys_h.size
    pb = pay_h.dtype.itemsize
    kd = 1 if keys_h.dtype == np.float64 else 0
    cfg = Z.SortConfig(mapping=args.mapping)
    d_keys = torch.from_numpy(keys_h).to(dev)
    d_pay = torch.from_numpy(pay_h).to(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    S = Sorter(L, d_keys, d_pay, cfg, stream)
    for _ in range(max(3, args.warmup)):
        S.sort()
    torch.cuda.synchronize()
    # correctness gate on the benchmarked output (device structural check)
    viol = Z.check_stable_permutation_device(d_keys, S.out_k, S.out_p)
    if viol and os.environ.get("ZSB_LIB_VARIANT", "").startswith("whatif"):
        print(f"what-if build ({viol} violations): timing only", file=sys.stderr)  # tools/gpu_ab.sh experiments
    elif viol:
        raise SystemExit(f"benchmarked output failed the structural check: {viol} violations")

    import ctypes
    ms_phase = (ctypes.c_double * 8)()
    launches = (ctypes.c_int64 * 8)()
    with ClockSampler(local) as clk:
        # keep the GPU busy with the same workload while nvidia-smi starts
        # sampling (the timed region itself is only milliseconds long)
        t_end = time.perf_counter() + 1.5
        while time.perf_counter() < t_end:
            S.sort()
        torch.cuda.synchronize()
        step_ms = timed_steps(lambda: S.sort(with_stats=False), args.steps, flush, stream)
    # per-phase breakdown (CUDA events around each launch group) in a separate
    # pass of the same steps, so the events do not perturb the timed steps
    L.zsb_timing_read(ms_phase, launches, 8, 1)
    L.zsb_timing_enable(1)
    for _ in range(args.steps):
        flush.zero_()
        S.sort()
    torch.cuda.synchronize()
    L.zsb_timing_enable(0)
    records = (ctypes.c_int64 * 8)()
    L.zsb_timing_records(records, 8)
    L.zsb_timing_read(ms_phase, launches, 8, 1)
    ms_per_step = sum(step_ms) / args.steps
    value = n / (ms_per_step / 1e3)

    hbm_peak, peak_kind = peaks()
    rec = 8 + pb
    roof, phase_ms = roofline_from_phases(n, rec, ms_phase, launches, args.steps, args.config, records)
    sort_alg_bytes = (16 + 4 * rec) * n
    gpu_launches = int(sum(launches[i] for i in range(8)) / args.steps)
    st = S.stats
    line = {
        "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": 1, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if kd == 1 else "int64", "data": "synthetic",
        "config": bench_config(args, n, pb),
        "roofline": roof,
        "sort_roofline": {"alg_bytes_per_key": 16 + 4 * rec, "achieved_gbs": sort_alg_bytes / (ms_per_step / 1e3) / 1e9,
                          "frac": sort_alg_bytes / (ms_per_step / 1e3) / 1e9 / hbm_peak},
        "phases_ms_per_step": {k: round(v, 4) for k, v in phase_ms.items()},
        "gpu_launches": gpu_launches,
        "stats": {"max_depth": st[0], "fallbacks": st[1], "finish_runs": st[3], "scatters": st[4]},
    }
    line["clocks"] = clk.summary()
    line["clocks"]["window"] = "nvidia-smi sampled every 100 ms over a 1.5 s warm loop of the same sort plus the timed steps"

    if not args.no_e2e:
        line["e2e"] = e2e_leg(Z, keys_h, pay_h, cfg, S, flush, stream, args.steps)
    if args.mapping == "fitted" and not args.no_extras:
        # the paper's exact Eq. 1 level 1 (k = round(0.6 sqrt n), scale = k/4), same input
        Sp = Sorter(L, d_keys, d_pay, Z.SortConfig(mapping="paper"), stream)
        for _ in range(2):
            Sp.sort()
        pms = sum(timed_steps(lambda: Sp.sort(with_stats=False), max(3, args.steps // 2), flush, stream))
        pms /= max(3, args.steps // 2)
        line["paper_mapping"] = {"ms_per_step": pms, "keys_per_s": n / (pms / 1e3),
                                 "sort_roofline_frac": sort_alg_bytes / (pms / 1e3) / 1e9 / hbm_peak,
                                 "stats": {"max_depth": Sp.stats[0], "scatters": Sp.stats[4]},
                                 "same_output": bool(torch.equal(Sp.out_k, S.out_k) and torch.equal(Sp.out_p, S.out_p)),
                                 "note": "mapping='paper': exact Eq. 1 at level 1, k = round(0.6 sqrt(n)), scale = k/4"}
        del Sp
    if not args.no_comparators:
        line["comparators"] = comparators(d_keys, d_pay, S.out_k, S.out_p, flush, stream, args.steps, ms_per_step)
    if not args.no_cpu_baseline:
        ks, ps, sample = cpu_sample(args.config, keys_h, pay_h)
        line["cpu_baseline"] = cpu_baseline(ks, ps, sample)
    del S, d_keys, d_pay
    torch.cuda.empty_cache()
    if not args.no_extras:
        line["c5_single_gpu"] = c5_single_gpu(Z, L, dev, flush, stream, max(3, args.steps // 2), hbm_peak)
    print(json.dumps(line), flush=True)


class Sorter:
    """Preallocated zsb_sort call on device-resident inputs (the timed unit)."""

    def __init__(self, L, d_keys, d_pay, cfg, stream):
        import ctypes
        import torch

        self.L, self.d_keys, self.d_pay, self.stream = L, d_keys, d_pay, stream
        self.n = d_keys.numel()
        self.kd = 1 if d_keys.dtype == torch.float64 else 0
        self.pb = d_pay.element_size()
        self.c = cfg.to_c()
        self.out_k = torch.empty_like(d_keys)
        self.out_p = torch.empty_like(d_pay)
        self.ws_bytes = L.zsb_workspace_bytes(self.n, self.kd, self.pb, self.c)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=d_keys.device)
        self.stats = (ctypes.c_int64 * 5)()

    def sort(self, with_stats=True):
        # timed steps pass no stats buffer: the call is then stream-ordered and
        # returns once the sort is enqueued (the CUDA events bracket its GPU
        # work); with stats it adds one host round trip for the counters
        from paper_2605_14419_b200 import _lib

        rc = self.L.zsb_sort(self.d_keys.data_ptr(), self.kd, self.d_pay.data_ptr(), self.pb, self.out_k.data_ptr(),
                             self.out_p.data_ptr(), self.n, self.c, self.ws.data_ptr(), self.ws_bytes,
                             self.stats if with_stats else None, self.stream.cuda_stream)
        _lib.check(rc)


def timed_steps(fn, steps, flush, stream):
    """CUDA-event time of `fn` per step, L2 flushed before each step (outside
    the events), synchronised on both sides."""
    import torch

    out = []
    torch.cuda.synchronize()
    for _ in range(steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    return out


def e2e_leg(Z, keys_h, pay_h, cfg, S, flush, stream, steps):
    """The public API on pinned host tensors: H2D + sort + D2H per step."""
    import torch

    n, rec = keys_h.size, 8 + pay_h.dtype.itemsize
    hk = torch.from_numpy(keys_h).pin_memory()
    hp = torch.from_numpy(pay_h).pin_memory()
    hok = torch.empty_like(hk).pin_memory()
    hop = torch.empty_like(hp).pin_memory()
    for _ in range(2):
        Z.zsort(hk, hp, cfg, out=(hok, hop))
    e2e_ms = timed_steps(lambda: Z.zsort(hk, hp, cfg, out=(hok, hop)), max(3, min(steps, 10)), flush, stream)
    e2e_step = sum(e2e_ms) / len(e2e_ms)
    if not (np.array_equal(hok.numpy(), S.out_k.cpu().numpy()) and np.array_equal(hop.numpy(), S.out_p.cpu().numpy())):
        raise SystemExit("e2e output differs from the device-resident run")
    # the copies alone (same pinned buffers, same sizes): every output key
    # depends on every input key, so no output can leave before the last input
    # has arrived -- H2D + D2H is the floor of ONE end-to-end sort over PCIe
    dk, dp = torch.empty(hk.shape, dtype=hk.dtype, device="cuda"), torch.empty(hp.shape, dtype=hp.dtype, device="cuda")
    h2d = timed_steps(lambda: (dk.copy_(hk, non_blocking=True), dp.copy_(hp, non_blocking=True)), 3, flush, stream)
    d2h = timed_steps(lambda: (hok.copy_(dk, non_blocking=True), hop.copy_(dp, non_blocking=True)), 3, flush, stream)
    copy_floor = min(h2d) + min(d2h)
    del dk, dp
    # The headline: the same steps as a stream through the public
    # SortPipeline (every step uploads its inputs from pinned host memory and
    # downloads its result, inside the timed region), two device buffer sets and
    # three streams: step i+1's upload and step i-1's download overlap step i's
    # sort, so both PCIe directions are busy.  Inputs (1.2 GB per step at C4)
    # exceed the L2, no flush between steps.  Timed by CUDA events from before
    # the first upload to after the last download, and by the host clock.
    hk2, hp2 = hk.clone().pin_memory(), hp.clone().pin_memory()  # alternate input and output buffers
    hok2, hop2 = torch.empty_like(hk).pin_memory(), torch.empty_like(hp).pin_memory()
    hok3, hop3 = torch.empty_like(hk).pin_memory(), torch.empty_like(hp).pin_memory()
    pipe = Z.SortPipeline(n, hk.dtype, hp.dtype, cfg)
    # three host output sets: a step waits for the step that last used its set,
    # whose download ended a whole step earlier (no bubble on the upload engine)
    ins, outs = [(hk, hp), (hk2, hp2)], [(hok, hop), (hok2, hop2), (hok3, hop3)]
    NW = 6
    for i in range(NW):
        pipe.submit(*ins[i % 2], *outs[i % 3])
    pipe.drain()
    ksteps = max(6, min(2 * steps, 18))
    for ok_h, op_h in outs:
        ok_h.zero_(), op_h.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(pipe.s_in)
    for i in range(ksteps):
        if i >= 3:
            pipe.wait(NW + i - 3)  # the step that used these host output buffers
        pipe.submit(*ins[i % 2], *outs[i % 3])
    pipe.drain()
    e1.record(pipe.s_out)
    e1.synchronize()
    wall_ms = (time.perf_counter() - t0) * 1e3
    pipe_ms = max(e0.elapsed_time(e1), 0.0) / ksteps
    torch.cuda.synchronize()
    for ok_h, op_h in outs:
        if not (np.array_equal(ok_h.numpy(), S.out_k.cpu().numpy()) and np.array_equal(op_h.numpy(), S.out_p.cpu().numpy())):
            raise SystemExit("pipelined e2e output differs from the device-resident run")
    del pipe
    torch.cuda.empty_cache()
    duplex_floor = max(min(h2d), min(d2h))
    return {"value": n / (pipe_ms / 1e3), "unit": "keys/s", "h2d_bytes_per_step": int(n * rec),
            "d2h_bytes_per_step": int(n * rec), "ms_per_step": pipe_ms, "steps": ksteps,
            "wall_ms_per_step": wall_ms / ksteps,
            "pipeline_floor_ms": duplex_floor, "vs_pipeline_floor": pipe_ms / duplex_floor,
            "api": "paper_2605_14419_b200.SortPipeline(n, f64, i32).submit(pinned host keys, payload, pinned host "
                   "outputs) per step; wait()/drain(): uploads, sorts and downloads of consecutive steps overlap",
            "single_sort": {"ms_per_step": e2e_step, "keys_per_s": n / (e2e_step / 1e3),
                            "copy_floor_ms": copy_floor, "vs_copy_floor": e2e_step / copy_floor,
                            "api": "paper_2605_14419_b200.zsort(pinned host tensors, out=pinned host tensors): "
                                   "one sort, H2D + sort + D2H in series (latency)"},
            "h2d_gbs": n * rec / min(h2d) / 1e6, "d2h_gbs": n * rec / min(d2h) / 1e6}


def c5_single_gpu(Z, L, dev, flush, stream, steps, hbm_peak):
    """BASELINE config 5 at its full size on this one GPU: 2^31 int64 keys
    (counter-based, generated on the device) + int64 index payload, ~101 GB of
    HBM; 80 B/key roofline; device structural check of the output."""
    import torch

    from paper_2605_14419_b200 import datagen

    n = 1 << 31
    free, _ = torch.cuda.mem_get_info(dev)
    if free < 125 * (1 << 30):
        return {"skipped": f"needs ~125 GB free HBM, {free / 2**30:.0f} GB free"}
    try:
        keys = datagen.config5_keys(0, n, n, device=dev)
        idx = torch.arange(n, dtype=torch.int64, device=dev)
        S5 = Sorter(L, keys, idx, Z.SortConfig(), stream)
        S5.sort()
        torch.cuda.synchronize()
        viol = Z.check_stable_permutation_device(keys, S5.out_k, S5.out_p)
        ms = timed_steps(lambda: S5.sort(with_stats=False), steps, flush, stream)
        t = sum(ms) / len(ms)
        out = {"n": n, "payload_bytes": 8, "ms_per_step": t, "keys_per_s": n / (t / 1e3),
               "sort_roofline": {"alg_bytes_per_key": 80, "frac": 80 * n / (t / 1e3) / 1e9 / hbm_peak},
               "structural_check_violations": int(viol),
               "stats": {"max_depth": S5.stats[0], "finish_runs": S5.stats[3], "scatters": S5.stats[4]}}
        del S5, keys, idx
        torch.cuda.empty_cache()
        return out
    except torch.cuda.OutOfMemoryError as e:  # noqa: F841
        torch.cuda.empty_cache()
        return {"skipped": "out of memory"}


def roofline_from_phases(n, rec, ms_phase, launches, steps, cfg, records=None):
    """Roofline of the dominant kernel from the library's per-phase CUDA-event
    times (a separate pass of the same steps).  Per launch: algorithmic bytes =
    the per-record figure of the kernel (2 x (8 + payload) for the
    scatter and the finish, 8 for the histogram and the moments) x the records
    its launches passed over (zsb_timing_records: every partition level's
    records for the histogram and the scatter, n for the finish), over the
    kernel's CUDA-event time.  `one_pass_frac` is the stricter figure that
    credits a single pass over the n records whatever the number of levels
    (the whole-sort `sort_roofline` uses the same convention).  `traffic`
    comes from the committed ncu capture of the same config
    (profiles/*_traffic_c<cfg>.json), else null."""
    from paper_2605_14419_b200 import _lib

    hbm_peak, peak_kind = peaks()
    per_rec = {"moments": 8, "histogram": 8, "scatter": 2 * rec, "finish": 2 * rec}
    phase_ms = {name: ms_phase[i] / steps for i, name in enumerate(_lib.PHASES)}
    phase_launch = {name: launches[i] / steps for i, name in enumerate(_lib.PHASES)}
    phase_rec = {name: (records[i] / steps if records is not None and records[i] > 0 else n)
                 for i, name in enumerate(_lib.PHASES)}
    dominant = max(("moments", "histogram", "scatter", "finish"), key=lambda k: phase_ms[k])
    ms = max(phase_ms[dominant], 1e-9)
    nl = max(phase_launch[dominant], 1.0)
    alg_step = per_rec[dominant] * phase_rec[dominant]  # all launches of the kernel in one sort
    achieved = alg_step / (ms / 1e3) / 1e9
    one_pass = per_rec[dominant] * n / (ms / 1e3) / 1e9
    traffic, traffic_src = None, None
    try:
        import glob
        tf = sorted(glob.glob(os.path.join(REPO, "profiles", f"*_traffic_c{cfg}.json")))
        if tf:
            rec_t = json.load(open(tf[-1]))
            if int(rec_t.get("n", n)) == n:
                per = rec_t["bytes_per_step"].get(f"k_{dominant}")
                if per:
                    traffic, traffic_src = float(per) / nl, os.path.relpath(tf[-1], REPO)
    except Exception:
        traffic = None
    roof = {"bound": "hbm", "kernel": f"k_{dominant}", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved / hbm_peak, "traffic": traffic, "traffic_source": traffic_src, "peak_kind": peak_kind,
            "alg_bytes_per_launch": alg_step / nl, "launch_ms": ms / nl, "launches_per_step": nl,
            "records_per_step": phase_rec[dominant], "one_pass_frac": one_pass / hbm_peak,
            "note": f"per launch of k_{dominant}: alg bytes = {per_rec[dominant]} B x the records the launch passes "
                    "over (each partition level's launch passes over that level's records), time = the kernel's "
                    "CUDA-event time / its launches, measured live; one_pass_frac credits one pass over n only; "
                    "traffic = ncu DRAM bytes per launch of the same config"}
    return roof, phase_ms


def comparators(d_keys, d_pay, out_k, out_p, flush, stream, steps, ms_ours):
    """SURVEY §8(f)3, the paper's bit-width-wall contrast on the GPU: the same
    stable sort (keys + payload permuted alongside) with torch.sort(stable=True)
    -- CUB's LSD radix sort, one pass per 8-bit digit of the 64-bit key -- plus
    the payload gather, same inputs, same L2 flush and CUDA-event timing.  The
    outputs are checked equal to ours."""
    import torch

    def run():
        k, perm = torch.sort(d_keys, stable=True)
        return k, d_pay[perm]

    k, p = run()
    same = bool(torch.equal(k.view(torch.int64), out_k.view(torch.int64)) and torch.equal(p, out_p))
    ms = []
    for _ in range(max(3, steps)):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = sum(ms) / len(ms)
    return {"torch.sort(stable=True)+gather": {"ms_per_step": t, "keys_per_s": d_keys.numel() / (t / 1e3),
                                               "ours_speedup": t / ms_ours, "same_output": same}}


def run_dist(args, rank, world, dev):
    """N > 1: config 5, strong scaling of the globally stable sort over NCCL
    (dist.py): n = 2^31 int64 keys (uniform, 10% one repeated value,
    counter-based, each rank generates its shard on its device) with the int64
    global-index payload, 2^31/N records per GPU.  One step = D1 allreduce, D2
    allgather, stable partition, NCCL all-to-all, local stable sort; the
    concatenation of the rank outputs is the global stable sort (checked on
    the device per rank plus the boundary records across ranks)."""
    import torch
    import torch.distributed as dist

    from paper_2605_14419_b200 import datagen
    from paper_2605_14419_b200.dist import dist_zsort
    import paper_2605_14419_b200 as Z

    if args.config != 5:
        raise SystemExit("N>1 runs config 5 (strong scaling of 2^31 keys)")
    n_total = 1 << 31
    n = n_total // world
    base = rank * n
    dk = datagen.config5_keys(base, n, n_total, device=dev)
    dp = torch.arange(base, base + n, dtype=torch.int64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    # the exchange: fused into the partition kernel (stores into the peers'
    # receive buffers over NVLink) when every pair of the ranks' GPUs has peer
    # access, else NCCL all_to_all; a failure of the fused path falls back
    exchange = args.exchange
    if exchange == "auto":
        peer = torch.tensor([1 if all(torch.cuda.can_device_access_peer(dev.index, d)
                                      for d in range(torch.cuda.device_count()) if d != dev.index) else 0],
                            device=dev)
        dist.all_reduce(peer, op=dist.ReduceOp.MIN)
        exchange = "p2p" if int(peer.item()) else "nccl"
    try:
        for _ in range(max(3, args.warmup)):
            ok, op, info = dist_zsort(dk, dp, base, exchange=exchange)
        torch.cuda.synchronize()
    except Exception as exc:  # keep the scaling run alive on the proven path
        if exchange != "p2p":
            raise
        print(f"[bench] fused p2p exchange failed ({exc}); using nccl", file=sys.stderr, flush=True)
        exchange = "nccl"
        dist.barrier()
        for _ in range(max(3, args.warmup)):
            ok, op, info = dist_zsort(dk, dp, base, exchange=exchange)
        torch.cuda.synchronize()
    # global correctness: per-rank structural check (keys regenerated from the
    # global index) and ordered boundaries between consecutive ranks
    viol = check_dist_output(Z, datagen, ok, op, n_total, dev)
    bnd = torch.tensor([ok[0].item() if ok.numel() else 0, ok[-1].item() if ok.numel() else 0,
                        op[0].item() if op.numel() else -1, op[-1].item() if op.numel() else -1], device=dev)
    allb = [torch.empty_like(bnd) for _ in range(world)]
    dist.all_gather(allb, bnd)
    for r in range(world - 1):
        a, b = allb[r].tolist(), allb[r + 1].tolist()
        if a[1] > b[0] or (a[1] == b[0] and a[3] >= b[2]):
            viol += 1
    vt = torch.tensor([viol], device=dev)
    dist.all_reduce(vt)
    if int(vt.item()):
        raise SystemExit(f"distributed output failed the structural check: {int(vt.item())} violations")
    del ok, op
    step_ms = []
    with ClockSampler(dev.index) as clk:
        t_end = time.perf_counter() + 1.5
        while time.perf_counter() < t_end:
            dist_zsort(dk, dp, base, exchange=exchange)
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.zero_()
            dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ok, op, info = dist_zsort(dk, dp, base, exchange=exchange)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            del ok, op
        dist.barrier()
    t = torch.tensor([sum(step_ms)], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    # our kernel launches per timed step and the per-phase breakdown of the
    # local work, from a separate pass of the same steps
    import ctypes
    from paper_2605_14419_b200 import _lib
    L = _lib.load()
    ms_phase = (ctypes.c_double * 8)()
    launches = (ctypes.c_int64 * 8)()
    L.zsb_timing_read(ms_phase, launches, 8, 1)
    L.zsb_timing_enable(1)
    for _ in range(args.steps):
        flush.zero_()
        dist.barrier()
        dist_zsort(dk, dp, base, exchange=exchange)
    torch.cuda.synchronize()
    L.zsb_timing_enable(0)
    records = (ctypes.c_int64 * 8)()
    L.zsb_timing_records(records, 8)
    L.zsb_timing_read(ms_phase, launches, 8, 1)
    roof, phase_ms = roofline_from_phases(n, 16, ms_phase, launches, args.steps, args.config, records)
    gpu_launches = int(sum(launches[i] for i in range(8)) / args.steps)
    # e2e: pinned host shard -> device -> distributed sort -> pinned host result
    e2e = None
    try:
        import psutil
        need = 4 * n * 16 * world
        room = psutil.virtual_memory().available
    except Exception:
        need, room = 1, 0
    if need < 0.6 * room and not args.no_e2e:
        hk = dk.cpu().pin_memory()
        hp = dp.cpu().pin_memory()
        times = []
        for _ in range(3):
            dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            k_, p_, _ = dist_zsort(hk.to(dev, non_blocking=True), hp.to(dev, non_blocking=True), base,
                                   exchange=exchange)
            rk = torch.empty(k_.shape, dtype=k_.dtype, pin_memory=True)
            rp = torch.empty(p_.shape, dtype=p_.dtype, pin_memory=True)
            rk.copy_(k_, non_blocking=True)
            rp.copy_(p_, non_blocking=True)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        te = torch.tensor([sum(times) / len(times)], device=dev, dtype=torch.float64)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": n_total / (float(te.item()) / 1e3), "unit": "keys/s",
               "h2d_bytes_per_step": int(n_total * 16), "d2h_bytes_per_step": int(n_total * 16),
               "ms_per_step": float(te.item()),
               "api": "paper_2605_14419_b200.dist.dist_zsort(pinned host shard copied in; result copied to pinned host)"}
    else:
        dist.barrier()
    if rank == 0:
        hbm_peak, peak_kind = peaks()
        t_roof_hbm = n * 80 / (hbm_peak * 1e9)
        t_roof_nvl = n * 16 * (world - 1) / world / 900e9
        line = {
            "metric": METRIC, "value": n_total / (ms_per_step / 1e3), "unit": "keys/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": bench_config(args, n, 8),
            "sort_roofline": {"alg_bytes_per_key": 80, "model_ms": 1e3 * max(t_roof_hbm, t_roof_nvl),
                              "frac_of_model": 1e3 * max(t_roof_hbm, t_roof_nvl) / ms_per_step,
                              "note": "T_roof(G) = max(n/G * 80 B / HBM peak, n/G * 16 (G-1)/G B / 900 GB/s)"},
            "exchange": {"mode": exchange, "sent_per_rank": info.get("sent"), "received_rank0": info.get("received"),
                         "note": "p2p: the partition kernel stores into the peers' receive buffers (CUDA IPC, NVLink); "
                                 "nccl: partition to a send buffer + all_to_all_single"},
            "gpu_launches": gpu_launches, "roofline": roof,
            "phases_ms_per_step": {k: round(v, 4) for k, v in phase_ms.items()}, "clocks": clk.summary(),
        }
        if e2e:
            line["e2e"] = e2e
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def check_dist_output(Z, datagen, ok, op, n_total, dev):
    """Per-rank structural check of a distributed sort's local output: the
    received keys are sorted and stable by global index, and each key equals
    the config-5 key regenerated from its global index."""
    import torch

    if ok.numel() == 0:
        return 0
    viol = int(((ok[1:] < ok[:-1]) | ((ok[1:] == ok[:-1]) & (op[1:] <= op[:-1]))).sum().item())
    for s in range(0, ok.numel(), 1 << 26):
        e = min(ok.numel(), s + (1 << 26))
        gi = op[s:e]
        i = gi.to(torch.int64)
        k = datagen.splitmix64(i + datagen.SEED_MIX)
        u = datagen._lsr(datagen.splitmix64(i + datagen.SALT), 11)
        k = torch.where(u < datagen._TENTH_53, torch.full_like(k, datagen.repeated_value()), k)
        viol += int((k != ok[s:e]).sum().item())
    return viol


if __name__ == "__main__":
    main()
