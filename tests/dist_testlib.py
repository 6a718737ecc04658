"""Test helpers for the multi-GPU path (test infrastructure only).

ThreadComm simulates G ranks inside one process (one thread per rank) with
the collective semantics dist.py needs; NumpyOps are CPU stand-ins for the
CUDA local operations so the distributed planning and exchange logic can be
exercised without a GPU (gloo multi-process tests and thread tests).
"""

from __future__ import annotations

import os
import threading

import numpy as np
import torch

from oracle import oracle as O


class ThreadGroup:
    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world


class ThreadComm:
    def __init__(self, group: ThreadGroup, rank: int):
        self.g, self.rank, self.world = group, rank, group.world

    def _exchange(self, obj):
        self.g.slots[self.rank] = obj
        self.g.barrier.wait()
        vals = list(self.g.slots)
        self.g.barrier.wait()
        return vals

    def all_reduce(self, t, op):
        vals = self._exchange(t.clone())
        acc = vals[0].clone()
        for v in vals[1:]:
            v = v.to(acc.device)
            acc = acc + v if op == "sum" else (torch.minimum(acc, v) if op == "min" else torch.maximum(acc, v))
        t.copy_(acc)
        return t

    def all_gather(self, t):
        return [v.to(t.device) for v in self._exchange(t.clone())]

    def barrier(self):
        self.g.barrier.wait()

    def share_cuda(self, tensors):
        return self._exchange(list(tensors))  # one process: every rank's buffers are plain device memory

    def all_to_all_single(self, out, inp, out_splits=None, in_splits=None):
        if in_splits is None:
            in_splits = [inp.numel() // self.world] * self.world
        chunks = list(torch.split(inp, list(in_splits)))
        allc = self._exchange([c.clone() for c in chunks])
        mine = [allc[r][self.rank].to(out.device) for r in range(self.world)]
        out.copy_(torch.cat(mine) if mine else out)


class NumpyOps:
    """CPU stand-ins of dist.DeviceOps (same semantics, numpy/oracle based)."""

    device = torch.device("cpu")

    @staticmethod
    def kind(keys):
        return "int64" if keys.dtype == torch.int64 else "float64"

    @staticmethod
    def _vals(k: np.ndarray):
        return k if k.dtype == np.float64 else k.astype(np.float64)

    def local_moments(self, keys):
        k = keys.numpy()
        if k.size == 0:
            return torch.zeros(4, dtype=torch.float64), torch.tensor([-1, 0], dtype=torch.int64)
        c = float(self._vals(k[:1])[0])
        d = self._vals(k) - c
        o = O.ordered_u64(k)
        return (torch.tensor([float(k.size), float(d.sum()), float((d * d).sum()), c], dtype=torch.float64),
                torch.tensor(np.array([o.min(), o.max()], np.uint64).view(np.int64)))

    @staticmethod
    def bucket_ids(keys, p):
        x = NumpyOps._vals(keys.numpy())
        with np.errstate(invalid="ignore", over="ignore"):
            h = ((x - p.center) / p.std + p.zmin) * p.scale
            f = np.floor(h)
        b = np.where(f > 0.0, np.where(f >= p.k, p.k - 1, f), 0.0)
        return b.astype(np.int64)

    def bucket_histogram(self, keys, params):
        return torch.from_numpy(np.bincount(self.bucket_ids(keys, params), minlength=params.k).astype(np.int64))

    def bucket_minmax(self, keys, params, buckets):
        ids = self.bucket_ids(keys, params)
        o = O.ordered_u64(keys.numpy())
        mn, mx = [], []
        for b in buckets:
            sel = o[ids == b]
            mn.append(int(sel.min()) if sel.size else (1 << 64) - 1)
            mx.append(int(sel.max()) if sel.size else 0)
        return (torch.tensor(np.array(mn, np.uint64).view(np.int64)),
                torch.tensor(np.array(mx, np.uint64).view(np.int64)))

    def range_histogram(self, keys, params, buckets, lo, hi, shifts, nbins):
        ids = self.bucket_ids(keys, params)
        o = O.ordered_u64(keys.numpy())
        out = np.zeros((len(buckets), nbins), np.int64)
        for q, (b, a, z, sh) in enumerate(zip(buckets, lo, hi, shifts)):
            sel = o[(ids == b) & (o >= np.uint64(a)) & (o <= np.uint64(z))]
            d = ((sel - np.uint64(a)) >> np.uint64(sh)).astype(np.int64)
            out[q] = np.bincount(d, minlength=nbins)[:nbins]
        return torch.from_numpy(out.reshape(-1))

    def occurrence_index(self, keys, key_bits, occurrence, kind):
        o = O.ordered_u64(keys.numpy())
        target = O.ordered_u64(np.array([key_bits], np.uint64).view(np.int64 if kind == "int64" else np.float64))[0]
        return int(np.flatnonzero(o == target)[occurrence])

    def partition(self, keys, payload, params, gidx_base, cuts):
        ids = self.bucket_ids(keys, params)
        o = O.ordered_u64(keys.numpy())
        g = gidx_base + np.arange(keys.numel())
        dest = np.zeros(keys.numel(), np.int64)
        for c in cuts:
            ge = (ids > c.bucket) | ((ids == c.bucket) & ((o > np.uint64(c.ord)) | ((o == np.uint64(c.ord)) & (g >= c.gidx))))
            dest += ge
        order = np.argsort(dest, kind="stable")
        counts = np.bincount(dest, minlength=len(cuts) + 1)
        pk = keys[torch.from_numpy(order)]
        pp = payload[torch.from_numpy(order)] if payload is not None else None
        return pk, pp, [int(x) for x in counts]

    def local_sort(self, keys, payload):
        k, p, _ = O.stable_sort(keys.numpy(), payload.numpy() if payload is not None else None)
        return torch.from_numpy(np.ascontiguousarray(k)), (torch.from_numpy(np.ascontiguousarray(p)) if p is not None else None)


def run_threads(shards, ops_factory, k=1024, exchange="nccl"):
    """Run dist_zsort on len(shards) simulated ranks; returns per-rank outputs."""
    from paper_2605_14419_b200.dist import dist_zsort

    world = len(shards)
    grp = ThreadGroup(world)
    results = [None] * world
    errors = []
    bases = np.concatenate(([0], np.cumsum([s[0].numel() for s in shards])))

    def work(r):
        try:
            keys, pay = shards[r]
            ops = ops_factory()
            if hasattr(ops.device, "type") and ops.device.type == "cuda":
                torch.cuda.set_device(ops.device)
            results[r] = dist_zsort(keys, pay, int(bases[r]), ops=ops, comm=ThreadComm(grp, r), k=k,
                                    exchange=exchange)
        except BaseException as exc:  # surface in the main thread
            errors.append(exc)
            grp.barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errors:
        raise errors[0]
    return results


def gloo_worker(rank, world, port, keys_all, pay_all, out_dir, k):
    """torch.multiprocessing target: one gloo rank running dist_zsort with NumpyOps."""
    import torch.distributed as dist

    from paper_2605_14419_b200.dist import dist_zsort

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = keys_all.size
        lo, hi = rank * n // world, (rank + 1) * n // world
        keys = torch.from_numpy(np.ascontiguousarray(keys_all[lo:hi]))
        pay = torch.from_numpy(np.ascontiguousarray(pay_all[lo:hi]))
        ok, op, info = dist_zsort(keys, pay, lo, ops=NumpyOps(), k=k)
        np.save(os.path.join(out_dir, f"k{rank}.npy"), ok.numpy())
        np.save(os.path.join(out_dir, f"p{rank}.npy"), op.numpy())
    finally:
        dist.destroy_process_group()


class StagedComm:
    """dist.TorchComm over gloo for CUDA tensors: every collective copies its
    operands to host memory, runs the gloo collective there and copies the
    result back (gloo has no CUDA all_to_all).  Lets real processes run the
    product DeviceOps path on one GPU without kernels that wait on another
    process."""

    def __init__(self):
        from paper_2605_14419_b200.dist import TorchComm

        self.inner = TorchComm()
        self.world, self.rank = self.inner.world, self.inner.rank

    def all_reduce(self, t, op):
        h = t.cpu()
        self.inner.all_reduce(h, op)
        t.copy_(h)
        return t

    def all_gather(self, t):
        return [x.to(t.device) for x in self.inner.all_gather(t.cpu())]

    def all_to_all_single(self, out, inp, out_splits=None, in_splits=None):
        h = torch.empty(out.shape, dtype=out.dtype)
        self.inner.all_to_all_single(h, inp.cpu(), out_splits, in_splits)
        out.copy_(h)

    def barrier(self):
        self.inner.barrier()

    def share_cuda(self, tensors):
        return self.inner.share_cuda(tensors)


def gloo_device_worker(rank, world, port, keys_all, pay_all, out_dir, k, exchange="nccl"):
    """torch.multiprocessing target: one process per rank on cuda:0 running
    dist_zsort with the product DeviceOps (CUDA kernels through the C ABI)
    and TorchComm over gloo (staged through host memory)."""
    import torch.distributed as dist

    from paper_2605_14419_b200.dist import DeviceOps, dist_zsort

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        n = keys_all.size
        lo, hi = rank * n // world, (rank + 1) * n // world
        keys = torch.from_numpy(np.ascontiguousarray(keys_all[lo:hi])).to(dev)
        pay = torch.from_numpy(np.ascontiguousarray(pay_all[lo:hi])).to(dev)
        ok, op, info = dist_zsort(keys, pay, lo, ops=DeviceOps(dev), comm=StagedComm(), k=k, exchange=exchange)
        np.save(os.path.join(out_dir, f"k{rank}.npy"), ok.cpu().numpy())
        np.save(os.path.join(out_dir, f"p{rank}.npy"), op.cpu().numpy())
    finally:
        dist.destroy_process_group()


def config5_small(n: int, seed_frac=0.1):
    """Config 5 recipe at small n (splitmix64 keys, 10% one repeated value)."""
    from paper_2605_14419_b200 import datagen

    return datagen.config5_keys(0, n, n, device="cpu").numpy()
