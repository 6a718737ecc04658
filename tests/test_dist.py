"""Multi-GPU path (paper_2605_14419_b200/dist.py): range assignment, exchange
and cross-rank stability.

CPU: world_size-2 gloo processes and 2..8 simulated ranks (threads) with the
numpy stand-ins for the local CUDA operations.  GPU (-m gpu): simulated ranks
on one B200 running the real partition / histogram / sort kernels (the
driver gives this run one GPU; the NCCL path is the same code with
TorchComm).  Every result is compared with the CPU oracle's stable sort of
the global input.
"""

import socket
import tempfile

import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.dist_testlib import NumpyOps, config5_small, gloo_device_worker, gloo_worker, run_threads

INT64_MIN, INT64_MAX = -(2**63), 2**63 - 1


def datasets():
    rng = np.random.default_rng(7)
    yield "uniform_i64", rng.integers(INT64_MIN, INT64_MAX, size=20_000, endpoint=True, dtype=np.int64)
    yield "config5_recipe", config5_small(30_000)
    yield "normal_f64", rng.standard_normal(20_000)
    d = rng.integers(0, 5, size=15_000, dtype=np.int64)
    yield "few_values", d
    yield "all_equal", np.full(9_000, 42, np.int64)
    z = rng.choice(np.array([0.0, -0.0, 1.5, -2.0]), 12_000)
    yield "signed_zeros", z
    h = rng.integers(-1000, 1000, size=20_000, dtype=np.int64)
    h[rng.random(20_000) < 0.6] = 7  # a 60% run: several cuts land inside one bucket
    yield "heavy_run", h


def check(keys_all, outs):
    ok = np.concatenate([o[0].cpu().numpy() for o in outs])
    op = np.concatenate([o[1].cpu().numpy() for o in outs])
    ek, _, perm = O.stable_sort(keys_all, None)
    assert np.array_equal(ok.view(np.uint64), ek.view(np.uint64))
    assert np.array_equal(op, perm)


def shards_of(keys_all, world, device="cpu"):
    n = keys_all.size
    out = []
    for r in range(world):
        lo, hi = r * n // world, (r + 1) * n // world
        out.append((torch.from_numpy(np.ascontiguousarray(keys_all[lo:hi])).to(device),
                    torch.arange(lo, hi, dtype=torch.int64, device=device)))
    return out


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_simulated_ranks_cpu(world):
    for name, keys in datasets():
        outs = run_threads(shards_of(keys, world), NumpyOps, k=512)
        check(keys, outs)


def test_balance_with_heavy_run_cpu():
    keys = config5_small(80_000)
    outs = run_threads(shards_of(keys, 4), NumpyOps, k=1024)
    sizes = [o[0].numel() for o in outs]
    assert max(sizes) - min(sizes) <= 1, sizes  # cuts are exact: the 10% run is split by position
    check(keys, outs)


def test_empty_and_tiny_shards_cpu():
    keys = np.array([5, 3, 5, 1], np.int64)
    outs = run_threads(shards_of(keys, 4), NumpyOps, k=64)
    check(keys, outs)
    keys = np.arange(7, dtype=np.int64)[::-1].copy()
    outs = run_threads(shards_of(keys, 8), NumpyOps, k=64)  # one empty shard
    check(keys, outs)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name", ["config5_recipe", "normal_f64", "heavy_run"])
def test_gloo_world2(name):
    import torch.multiprocessing as mp

    keys = dict(datasets())[name]
    pay = np.arange(keys.size, dtype=np.int64)
    with tempfile.TemporaryDirectory() as td:
        mp.start_processes(gloo_worker, args=(2, _free_port(), keys, pay, td, 512), nprocs=2, join=True,
                           start_method="spawn")
        outs = [(torch.from_numpy(np.load(f"{td}/k{r}.npy")), torch.from_numpy(np.load(f"{td}/p{r}.npy")))
                for r in range(2)]
    check(keys, outs)


# ------------------------------------------------------------------ GPU

@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
def test_simulated_ranks_gpu(world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_14419_b200.dist import DeviceOps

    dev = torch.device("cuda", 0)
    for name, keys in datasets():
        outs = run_threads(shards_of(keys, world, dev), lambda: DeviceOps(dev), k=1024)
        check(keys, outs)
    keys = config5_small(1 << 21)
    outs = run_threads(shards_of(keys, world, dev), lambda: DeviceOps(dev), k=4096)
    sizes = [o[0].numel() for o in outs]
    assert max(sizes) - min(sizes) <= 1, sizes  # exact cuts
    check(keys, outs)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 8])
def test_simulated_ranks_gpu_fused_exchange(world):
    """exchange="p2p": the partition kernel stores every record into its
    destination rank's buffer (here the ranks are threads of one process, so
    the peer pointers are plain device pointers)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_14419_b200.dist import DeviceOps

    dev = torch.device("cuda", 0)
    for name, keys in datasets():
        outs = run_threads(shards_of(keys, world, dev), lambda: DeviceOps(dev), k=1024, exchange="p2p")
        check(keys, outs)
    keys = config5_small(1 << 21)
    outs = run_threads(shards_of(keys, world, dev), lambda: DeviceOps(dev), k=4096, exchange="p2p")
    sizes = [o[0].numel() for o in outs]
    assert max(sizes) - min(sizes) <= 1, sizes
    check(keys, outs)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["config5_recipe", "heavy_run", "signed_zeros"])
def test_two_processes_fused_exchange_ipc(name):
    """The fused exchange across real processes: each rank's receive
    buffers are opened by the other through CUDA IPC and the partition kernel
    stores straight into them (on one GPU here; across GPUs the same stores
    travel over NVLink)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    keys = dict(datasets())[name]
    if name == "config5_recipe":
        keys = config5_small(1 << 20)
    pay = np.arange(keys.size, dtype=np.int64)
    with tempfile.TemporaryDirectory() as td:
        mp.start_processes(gloo_device_worker, args=(2, _free_port(), keys, pay, td, 4096, "p2p"), nprocs=2,
                           join=True, start_method="spawn")
        outs = [(torch.from_numpy(np.load(f"{td}/k{r}.npy")), torch.from_numpy(np.load(f"{td}/p{r}.npy")))
                for r in range(2)]
    check(keys, outs)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["config5_recipe", "normal_f64", "heavy_run", "signed_zeros"])
def test_two_processes_device_ops_gloo(name):
    """The product distributed path in real processes: two ranks on cuda:0,
    DeviceOps (CUDA kernels through the C ABI: D1 moments, D2 histograms and
    cut refinement, the device occurrence search, the MODE_DEST partition,
    the local sort) with TorchComm over gloo, collectives staged through host
    memory.  No kernel of one process waits on the other."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    keys = dict(datasets())[name]
    if name == "config5_recipe":
        keys = config5_small(1 << 20)
    pay = np.arange(keys.size, dtype=np.int64)
    with tempfile.TemporaryDirectory() as td:
        mp.start_processes(gloo_device_worker, args=(2, _free_port(), keys, pay, td, 4096), nprocs=2, join=True,
                           start_method="spawn")
        outs = [(torch.from_numpy(np.load(f"{td}/k{r}.npy")), torch.from_numpy(np.load(f"{td}/p{r}.npy")))
                for r in range(2)]
    sizes = [o[0].numel() for o in outs]
    if name in ("config5_recipe", "heavy_run"):
        assert max(sizes) - min(sizes) <= 1, sizes  # exact cuts, the long run split by position
    check(keys, outs)
