"""B200 bench seam.

Two ways to time the GPU sort the way the reference harness times its
algorithms (``zsort.bench``: ``register_algorithm`` at bench.py:163-170,
``run_trial`` at bench.py:196-232):

* ``register()`` plugs ``adapter`` into the reference registry, so the
  reference's own ``run_trial`` / ``build_matrix`` time and verify the GPU
  sort on host arrays (wall clock, host copies included -- the reference's
  contract).
* ``run_trial_gpu()`` is the B200 version of ``run_trial``: inputs resident in
  HBM, the L2 flushed between repetitions (a 512 MiB device write instead of
  ``flush_cache``), CUDA events on the sort's stream instead of
  ``perf_counter_ns``, and every repetition verified on the device by the
  structural checker (K8, ``zsb_check_sorted``) -- the equivalent of
  ``check_stable_permutation`` (verify.py:55-108).  It returns the reference's
  ``TrialResult`` fields.
"""

from __future__ import annotations

import statistics
from dataclasses import dataclass

import numpy as np

from . import core as _core

__all__ = ["adapter", "register", "TrialResultGPU", "run_trial_gpu"]


def _config_from(sort_config) -> _core.SortConfig:
    if sort_config is None:
        return _core.SortConfig()
    if isinstance(sort_config, _core.SortConfig):
        return sort_config
    # the reference's SortConfig (core.py:63-89): same field names
    return _core.SortConfig(alpha=sort_config.alpha, insertion_threshold=sort_config.insertion_threshold,
                            counting_range_threshold=sort_config.counting_range_threshold,
                            depth_guard=sort_config.depth_guard,
                            collect_stats=getattr(sort_config, "collect_stats", False))


def adapter(keys, payload, sort_config):
    """Registry adapter: ``(keys, payload, sort_config) -> (keys, payload)``
    (the contract of ``register_algorithm``, bench.py:163-170)."""
    out_k, out_p, _ = _core.zsort(keys, payload, _config_from(sort_config))
    return out_k, out_p


def register(register_algorithm=None, name: str = "zsort_b200") -> str:
    """Register ``adapter`` under ``name`` in the reference harness (or in the
    given ``register_algorithm`` callable).  Returns the name."""
    if register_algorithm is None:
        from zsort.bench import register_algorithm  # the reference package, when installed
    register_algorithm(name, adapter)
    return name


@dataclass(frozen=True)
class TrialResultGPU:
    algorithm: str
    size: int
    repetitions: int
    mean_ms: float
    median_ms: float
    min_ms: float
    stddev_ms: float
    verified: bool
    keys_per_s: float


def run_trial_gpu(keys, payload=None, repetitions: int = 10, config=None, flush_bytes: int = 512 << 20,
                  algorithm: str = "zsort_b200") -> TrialResultGPU:
    """Cold-L2, verified-only GPU timing of the sort on device-resident inputs."""
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    tk = keys if isinstance(keys, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(keys))
    tk = tk.to(dev)
    if payload is None:
        tp = torch.arange(tk.numel(), dtype=torch.int64, device=dev)
    else:
        tp = (payload if isinstance(payload, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(payload))).to(dev)
    cfg = _config_from(config)
    out_k, out_p = torch.empty_like(tk), torch.empty_like(tp)
    flush = torch.empty(max(1, flush_bytes), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    _core.zsort(tk, tp, cfg, out=(out_k, out_p))  # warm-up (library load, workspace)
    idx = torch.arange(tk.numel(), dtype=torch.int64, device=dev)
    perm = torch.empty_like(idx)
    times = []
    for _ in range(repetitions):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _core.zsort(tk, tp, cfg, out=(out_k, out_p))
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        # verification (untimed): the index permutation of the same sort must be
        # the stable one, and the timed payload must be the input payload under it
        _core.zsort(tk, idx, cfg, out=(torch.empty_like(tk), perm))
        if _core.check_stable_permutation_device(tk, out_k, perm) != 0 or not torch.equal(out_p, tp[perm]):
            raise RuntimeError(f"{algorithm} failed verification on n={tk.numel()}")
    med = statistics.median(times)
    return TrialResultGPU(algorithm=algorithm, size=int(tk.numel()), repetitions=repetitions,
                          mean_ms=statistics.fmean(times), median_ms=med, min_ms=min(times),
                          stddev_ms=statistics.stdev(times) if len(times) > 1 else 0.0, verified=True,
                          keys_per_s=tk.numel() / (med / 1e3))
