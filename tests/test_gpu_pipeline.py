"""SortPipeline (paper_2605_14419_b200/pipeline.py): a stream of host-to-host
sorts with uploads, sorts and downloads of consecutive tickets overlapped.
Same contract as zsort (reference core.py:348-400): every ticket's output is
the stable sort of its own input, checked against the CPU oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def Z():
    import paper_2605_14419_b200 as Z

    return Z


def test_pipeline_needs_cuda_and_validates(Z):
    # no CPU fallback: without a device the constructor raises
    if not torch.cuda.is_available():
        with pytest.raises(RuntimeError):
            Z.SortPipeline(16, torch.float64, torch.int32)
        return
    with pytest.raises(TypeError):
        Z.SortPipeline(16, torch.float32, torch.int32)
    with pytest.raises(TypeError):
        Z.SortPipeline(16, torch.float64, torch.int16)
    with pytest.raises(ValueError):
        Z.SortPipeline(0, torch.float64, torch.int32)


def _mk(rng, n, kdt, i):
    if kdt == torch.float64:
        k = rng.standard_normal(n) * (10.0 ** (i % 4))
        if i % 3 == 1:
            k = np.round(k)  # heavy ties
    else:
        k = rng.integers(-10**9, 10**9, size=n, dtype=np.int64) * (1 if i % 2 else 1 << 20)
    return k


@pytest.mark.gpu
@pytest.mark.parametrize("depth", [1, 2, 3])
@pytest.mark.parametrize("kdt,pdt", [(torch.float64, torch.int32), (torch.int64, torch.int64), (torch.float64, None)])
def test_pipeline_tickets_match_oracle(Z, depth, kdt, pdt):
    rng = np.random.default_rng(depth * 17 + (0 if pdt is None else 3))
    n, tickets = 200_003, 6
    pipe = Z.SortPipeline(n, kdt, pdt, depth=depth)
    ins, outs, ids = [], [], []
    for i in range(tickets):
        k = torch.from_numpy(_mk(rng, n, kdt, i)).pin_memory()
        p = None if pdt is None else torch.arange(n, dtype=pdt).pin_memory()
        ok = torch.empty_like(k).pin_memory()
        op = None if pdt is None else torch.empty_like(p).pin_memory()
        ins.append((k, p))
        outs.append((ok, op))
        ids.append(pipe.submit(k, p, ok, op))
        if i == 2:
            pipe.wait(ids[0])  # out of order with the submissions still in flight
    pipe.drain()
    pipe.wait(ids[3])  # waiting twice is a no-op
    for (k, p), (ok, op) in zip(ins, outs):
        ek, ep, _ = O.stable_sort(k.numpy(), None if p is None else p.numpy())
        assert np.array_equal(ok.numpy().view(np.uint64), ek.view(np.uint64))
        if p is not None:
            assert np.array_equal(op.numpy(), ep)


@pytest.mark.gpu
def test_pipeline_two_levels_and_pageable_buffers(Z):
    # 3e6 lognormal keys: two partition levels; pageable host tensors (the copies
    # are then synchronous, the result is the same)
    rng = np.random.default_rng(5)
    n = 3_000_000
    pipe = Z.SortPipeline(n, torch.float64, torch.int32)
    datas = [rng.lognormal(0, 2, n), np.sort(rng.standard_normal(n))[::-1].copy()]
    outs = []
    for d in datas:
        ok, op = torch.empty(n, dtype=torch.float64), torch.empty(n, dtype=torch.int32)
        outs.append((ok, op))
        pipe.submit(torch.from_numpy(d), torch.arange(n, dtype=torch.int32), ok, op)
    pipe.drain()
    for d, (ok, op) in zip(datas, outs):
        ek, ep, _ = O.stable_sort(d, np.arange(n, dtype=np.int32))
        assert np.array_equal(ok.numpy().view(np.uint64), ek.view(np.uint64)) and np.array_equal(op.numpy(), ep)


@pytest.mark.gpu
def test_pipeline_rejects_nan_and_bad_arguments(Z):
    n = 50_000
    pipe = Z.SortPipeline(n, torch.float64, torch.int32)
    k = torch.randn(n, dtype=torch.float64)
    p = torch.arange(n, dtype=torch.int32)
    ok, op = torch.empty_like(k), torch.empty_like(p)
    with pytest.raises(ValueError):
        pipe.submit(k[:-1], p, ok, op)
    with pytest.raises(ValueError):
        pipe.submit(k, p.to(torch.int64), ok, op)
    with pytest.raises(ValueError):
        pipe.wait(7)
    k[n // 2] = float("nan")
    with pytest.raises(ValueError):
        pipe.submit(k, p, ok, op)
        pipe.drain()
