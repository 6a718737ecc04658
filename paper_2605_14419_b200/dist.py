"""Multi-GPU stable z-score partitioning sort (one process per GPU, NCCL).

The reference is single-threaded and has no distributed
path; this is the B200 extension of its algorithm described in SURVEY.md
§8(e).  Each rank holds a contiguous shard of the global input (global
positions [gidx_base, gidx_base + n_local)); the global stable order is
(key, global position).

  D1  one pass over each shard (count, sum and sum of squares around the
      shard's first key, ordered extremes) and one all_gather of those six
      numbers; every rank merges them in rank order (Chan's parallel
      variance) and derives bit-identical fitted z-score parameters
      (core.py:212-234 with the fitted scale of the single-GPU path);
  D2  all_gather of the k-bucket z-score histograms -> G-1 cuts at the
      target positions j*N/G.  A cut falls on a bucket boundary, except
      inside an all-equal bucket (checked with an all_reduce of per-bucket
      min/max), where it splits the run by global position -- config 5's
      10% repeated value is spread over ranks this way;
  D3  stable partition of every shard by destination rank (the scatter
      kernel in MODE_DEST, records keep input order) and an NCCL
      all_to_all_single of keys and payload; chunks arrive in source-rank
      order, so each rank's received sequence is in global input order;
  local stable zsort of the received records (the single-GPU path).

The concatenation of the ranks' outputs in rank order is the stable sort of
the global input.  Local operations are pluggable (`ops`): DeviceOps runs the
CUDA kernels through the C ABI (the product path); the gloo CPU tests plug in
numpy stand-ins to exercise the planning and exchange logic without a GPU.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as tdist

from . import _lib

SIGN = 1 << 63
INT64_MIN = -(1 << 63)
DEFAULT_K = 4096


# ------------------------------------------------------------ key images

def ord_to_value(o: int, kind: str) -> float:
    """Value of the key whose order-preserving image is `o` (as double)."""
    if kind == "int64":
        v = (o ^ SIGN)
        return float(v - (1 << 64) if v >= SIGN else v)
    b = (o ^ SIGN) if o & SIGN else (~o & ((1 << 64) - 1))
    return float(np.array([b], np.uint64).view(np.float64)[0])


@dataclass(frozen=True)
class GlobalParams:
    """Fitted z-score mapping shared by all ranks (same arithmetic everywhere)."""

    center: float
    std: float
    zmin: float
    scale: float
    k: int

    def as_array(self):
        return (ctypes.c_double * 4)(self.center, self.std, self.zmin, self.scale)


def plan_params(count: float, s1: float, s2: float, shift: float, vmin: float, vmax: float, k: int) -> GlobalParams:
    """Fitted Eq. 1 parameters from allreduced moments (finalize_params in
    sort_kernels.cuh, fitted branch).  Degenerate inputs map every key to bucket
    0, which is still correct (no cut can then fall inside a non-constant
    bucket), only unbalanced."""
    mean = shift + s1 / count
    var = max(0.0, s2 / count - (s1 / count) ** 2)
    sd = math.sqrt(var)
    if sd > 0.0 and math.isfinite(sd) and vmax > vmin:
        span = (vmax - vmin) / sd
        if span > 0.0 and math.isfinite(span):
            zmin = (mean - vmin) / sd
            scale = (k * (1.0 - 2.0 ** -20)) / span
            if scale > 0.0 and math.isfinite(scale) and math.isfinite(zmin):
                return GlobalParams(mean, sd, zmin, scale, k)
    return GlobalParams(0.0, 1.0, 0.0, 1e-300, k)


def merge_moments(rows: np.ndarray):
    """Global (count, mean, M2, ordered min, ordered max) from the per-rank D1
    rows {count, sum(x - c), sum((x - c)^2), c, min bits, max bits}: Chan's
    pairwise merge in rank order, so every rank computes the same doubles."""
    n = mean = m2 = 0.0
    omin, omax = MASK64, 0
    bits = np.ascontiguousarray(rows[:, 4:6]).view(np.uint64)
    for r in range(rows.shape[0]):
        nr = float(rows[r, 0])
        if nr <= 0.0:
            continue
        s1, s2, c = float(rows[r, 1]), float(rows[r, 2]), float(rows[r, 3])
        mr = c + s1 / nr
        m2r = max(0.0, s2 - s1 * s1 / nr)
        tot = n + nr
        d = mr - mean
        mean = mean + d * (nr / tot)
        m2 = m2 + m2r + d * d * (n * nr / tot)
        n = tot
        omin = min(omin, int(bits[r, 0]))
        omax = max(omax, int(bits[r, 1]))
    return n, mean, m2, omin, omax


@dataclass(frozen=True)
class Cut:
    bucket: int
    ord: int
    gidx: int


def plan_cuts(counts: np.ndarray, nparts: int, all_equal, occurrence_gidx):
    """G-1 cuts over the global bucket sequence (SURVEY §8(e) range assignment).

    counts: (G, k) per-rank bucket counts.  all_equal(b) -> (bool, ord) says
    whether bucket b holds a single key value.  occurrence_gidx(b, t) returns
    the global index of the t-th record of bucket b in (rank, local) order.
    """
    glob = counts.sum(axis=0)
    total = int(glob.sum())
    excl = np.concatenate(([0], np.cumsum(glob)))
    cuts = []
    for j in range(1, nparts):
        target = (j * total) // nparts
        b = int(np.searchsorted(excl, target, side="right") - 1)  # excl[b] <= target < excl[b+1]
        b = min(max(b, 0), len(glob) - 1) if total else 0
        if target <= excl[b]:
            cuts.append(Cut(b, 0, INT64_MIN))
            continue
        eq, o = all_equal(b)
        if eq:
            t = target - int(excl[b])
            cuts.append(Cut(b, o, occurrence_gidx(b, t)))
        else:
            nxt = b + 1 if (excl[b + 1] - target) < (target - excl[b]) else b
            cuts.append(Cut(nxt, 0, INT64_MIN))
    return cuts


REFINE_BITS = 12


def plan_cuts_exact(counts, world, rank, keys, params, gidx_base, ops, comm, kind):
    """Exact G-1 cuts at the target positions j*N/G of the global stable order.

    A target on a bucket boundary cuts there.  A target inside bucket B is
    refined with exact integer-digit histograms of B's ordered key range
    (REFINE_BITS per round, batched over targets, one all_gather each) until
    it lands on a key boundary -- a key-level cut -- or on a single key value,
    whose run is then cut by global position (the record at that position is
    found by the rank that owns it).  Every rank computes identical cuts.
    """
    dev = ops.device
    glob = counts.sum(axis=0)
    total = int(glob.sum())
    excl = np.concatenate(([0], np.cumsum(glob)))
    cuts = [None] * (world - 1)
    pending = []  # [j, bucket, t (offset inside the current range), lo, hi, per-rank counts]
    for j in range(1, world):
        target = (j * total) // world
        b = int(np.searchsorted(excl, target, side="right") - 1)
        b = min(max(b, 0), len(glob) - 1)
        if target <= excl[b]:
            cuts[j - 1] = Cut(b, 0, INT64_MIN)
        else:
            pending.append([j, b, int(target - excl[b]), None, None, counts[:, b].astype(np.int64)])
    if pending:
        bs = sorted({q[1] for q in pending})
        bmn, bmx = ops.bucket_minmax(keys, params, bs)
        bmn = (bmn ^ INT64_MIN).clone()
        bmx = (bmx ^ INT64_MIN).clone()
        comm.all_reduce(bmn, "min")
        comm.all_reduce(bmx, "max")
        ext = {b: ((a ^ INT64_MIN) & MASK64, (z ^ INT64_MIN) & MASK64) for b, a, z in zip(bs, bmn.tolist(), bmx.tolist())}
        for q in pending:
            q[3], q[4] = ext[q[1]]
    requests = []
    for _round in range(64 // REFINE_BITS + 3):
        active = []
        for q in pending:
            if cuts[q[0] - 1] is not None:
                continue
            if q[3] == q[4]:  # one key value: cut its run by global position
                requests.append(q)
                cuts[q[0] - 1] = "pos"
            else:
                active.append(q)
        if not active:
            break
        shifts = [max(0, (q[4] - q[3]).bit_length() - REFINE_BITS) for q in active]
        nbins = 1 << REFINE_BITS
        h = ops.range_histogram(keys, params, [q[1] for q in active], [q[3] for q in active],
                                [q[4] for q in active], shifts, nbins)
        allh = torch.stack(comm.all_gather(h)).cpu().numpy().reshape(world, len(active), nbins)
        for qi, (q, sh) in enumerate(zip(active, shifts)):
            g = allh[:, qi, :].sum(axis=0)
            ex = np.concatenate(([0], np.cumsum(g)))
            d = int(np.searchsorted(ex, q[2], side="right") - 1)
            if q[2] == ex[d]:  # on a key boundary: records with ord >= that key go right
                cuts[q[0] - 1] = Cut(q[1], q[3] + (d << sh), INT64_MIN)
            else:
                q[2] -= int(ex[d])
                lo = q[3] + (d << sh)
                q[3], q[4] = lo, min(q[4], lo + (1 << sh) - 1)
                q[5] = allh[:, qi, d].astype(np.int64)
    if requests:
        answers = torch.full((len(requests),), INT64_MIN, dtype=torch.int64, device=dev)
        for qi, q in enumerate(requests):
            before = 0
            for r in range(world):
                c = int(q[5][r])
                if before <= q[2] < before + c:
                    if r == rank:
                        answers[qi] = gidx_base + ops.occurrence_index(keys, _ord_to_bits(q[3], kind), q[2] - before,
                                                                      kind)
                    break
                before += c
        comm.all_reduce(answers, "max")
        for q, g in zip(requests, answers.tolist()):
            cuts[q[0] - 1] = Cut(q[1], q[3], int(g))
    assert all(isinstance(c, Cut) for c in cuts), cuts
    return cuts


MASK64 = (1 << 64) - 1


# ------------------------------------------------------------ local ops

class DeviceOps:
    """Local work on the rank's GPU through the C ABI (the product path)."""

    def __init__(self, device: torch.device):
        self.device = device
        self.L = _lib.load()

    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    @staticmethod
    def kind(keys: torch.Tensor) -> str:
        return "int64" if keys.dtype == torch.int64 else "float64"

    @staticmethod
    def _kd(keys):
        return 0 if keys.dtype == torch.int64 else 1

    def local_moments(self, keys: torch.Tensor):
        """One pass: ({count, sum(x - c), sum((x - c)^2), c}, {ordered min, max}),
        c = the shard's first key."""
        out = torch.empty(4, dtype=torch.float64, device=self.device)
        bits = torch.empty(2, dtype=torch.int64, device=self.device)
        _lib.check(self.L.zsb_local_moments(keys.data_ptr(), self._kd(keys), keys.numel(), float("nan"),
                                            out.data_ptr(), bits.data_ptr(), self._stream()))
        return out, bits

    def bucket_histogram(self, keys, params: GlobalParams) -> torch.Tensor:
        c = torch.empty(params.k, dtype=torch.int64, device=self.device)
        _lib.check(self.L.zsb_bucket_histogram(keys.data_ptr(), self._kd(keys), keys.numel(), params.as_array(),
                                               params.k, c.data_ptr(), self._stream()))
        return c

    def bucket_minmax(self, keys, params: GlobalParams, buckets):
        nb = len(buckets)
        db = torch.tensor(list(buckets) or [0], dtype=torch.int32, device=self.device)
        mn = torch.empty(max(nb, 1), dtype=torch.int64, device=self.device)
        mx = torch.empty(max(nb, 1), dtype=torch.int64, device=self.device)
        _lib.check(self.L.zsb_bucket_minmax(keys.data_ptr(), self._kd(keys), keys.numel(), params.as_array(), params.k,
                                            nb, db.data_ptr(), mn.data_ptr(), mx.data_ptr(), self._stream()))
        return mn[:nb], mx[:nb]

    def range_histogram(self, keys, params: GlobalParams, buckets, lo, hi, shifts, nbins):
        nq = len(buckets)
        qb = torch.tensor(buckets, dtype=torch.int32, device=self.device)
        qlo = torch.tensor([x - (1 << 64) if x >= SIGN else x for x in lo], dtype=torch.int64, device=self.device)
        qhi = torch.tensor([x - (1 << 64) if x >= SIGN else x for x in hi], dtype=torch.int64, device=self.device)
        qs = torch.tensor(shifts, dtype=torch.int32, device=self.device)
        c = torch.empty(nq * nbins, dtype=torch.int64, device=self.device)
        _lib.check(self.L.zsb_range_histogram(keys.data_ptr(), self._kd(keys), keys.numel(), params.as_array(),
                                              params.k, nq, qb.data_ptr(), qlo.data_ptr(), qhi.data_ptr(),
                                              qs.data_ptr(), nbins, c.data_ptr(), self._stream()))
        return c

    def occurrence_index(self, keys, key_bits: int, occurrence: int, kind: str) -> int:
        """Local index of the `occurrence`-th record equal to the key with bits
        key_bits (for float64, -0.0 and +0.0 are the same key): the device
        search k_occ_count / k_occ_find."""
        ws = torch.empty(int(self.L.zsb_occurrence_workspace_bytes()), dtype=torch.uint8, device=self.device)
        out = ctypes.c_int64(-1)
        _lib.check(self.L.zsb_occurrence_index(keys.data_ptr(), self._kd(keys), keys.numel(),
                                               ctypes.c_uint64(key_bits & MASK64), int(occurrence), ws.data_ptr(),
                                               ctypes.byref(out), self._stream()))
        if out.value < 0:
            raise RuntimeError("occurrence not found: the cut plan and the shard disagree")
        return int(out.value)

    def partition(self, keys, payload, params: GlobalParams, gidx_base: int, cuts):
        n = keys.numel()
        nparts = len(cuts) + 1
        pb = payload.element_size() if payload is not None else 0
        ok = torch.empty_like(keys)
        op = torch.empty_like(payload) if payload is not None else None
        wsb = self.L.zsb_partition_workspace_bytes(n, pb, nparts)
        ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
        cb = (ctypes.c_int32 * max(1, len(cuts)))(*[c.bucket for c in cuts])
        co = (ctypes.c_uint64 * max(1, len(cuts)))(*[c.ord for c in cuts])
        cg = (ctypes.c_int64 * max(1, len(cuts)))(*[c.gidx for c in cuts])
        counts = (ctypes.c_int64 * nparts)()
        _lib.check(self.L.zsb_partition_to_ranks(keys.data_ptr(), self._kd(keys),
                                                 payload.data_ptr() if payload is not None else None, pb, n,
                                                 params.as_array(), params.k, int(gidx_base), len(cuts), cb, co, cg,
                                                 ok.data_ptr(), op.data_ptr() if op is not None else None, counts,
                                                 ws.data_ptr(), wsb, self._stream()))
        return ok, op, [int(x) for x in counts]

    def partition_plan(self, keys, payload, params: GlobalParams, gidx_base: int, cuts):
        """Fused exchange, step 1: the destination counts of the stable
        partition (histogram + scan, kept in the returned workspace)."""
        n = keys.numel()
        nparts = len(cuts) + 1
        pb = payload.element_size() if payload is not None else 0
        wsb = self.L.zsb_partition_workspace_bytes(n, pb, nparts)
        ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
        cb = (ctypes.c_int32 * max(1, len(cuts)))(*[c.bucket for c in cuts])
        co = (ctypes.c_uint64 * max(1, len(cuts)))(*[c.ord for c in cuts])
        cg = (ctypes.c_int64 * max(1, len(cuts)))(*[c.gidx for c in cuts])
        counts = (ctypes.c_int64 * nparts)()
        _lib.check(self.L.zsb_partition_to_ranks(keys.data_ptr(), self._kd(keys),
                                                 payload.data_ptr() if payload is not None else None, pb, n,
                                                 params.as_array(), params.k, int(gidx_base), len(cuts), cb, co, cg,
                                                 None, None, counts, ws.data_ptr(), wsb, self._stream()))
        return ws, [int(x) for x in counts]

    def partition_send(self, keys, payload, ws, dest_keys, dest_payload, dest_offsets):
        """Fused exchange, step 2: the partition's scatter stores every record
        straight into its destination's receive buffers (peer pointers)."""
        nparts = len(dest_keys)
        pb = payload.element_size() if payload is not None else 0
        dk = (ctypes.c_uint64 * nparts)(*[t.data_ptr() for t in dest_keys])
        dp = (ctypes.c_uint64 * nparts)(*[t.data_ptr() for t in dest_payload]) if payload is not None else None
        off = (ctypes.c_int64 * nparts)(*dest_offsets)
        _lib.check(self.L.zsb_partition_send(keys.data_ptr(), self._kd(keys),
                                             payload.data_ptr() if payload is not None else None, pb, keys.numel(),
                                             nparts, dk, dp, off, ws.data_ptr(), ws.numel(), self._stream()))

    def local_sort(self, keys, payload):
        from .core import zsort
        k, p, _ = zsort(keys, payload)
        return k, p


# ------------------------------------------------------------- comms

class TorchComm:
    """Collectives over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    _OPS = {"sum": tdist.ReduceOp.SUM, "min": tdist.ReduceOp.MIN, "max": tdist.ReduceOp.MAX}

    def __init__(self, group=None):
        self.group = group
        self.world = tdist.get_world_size(group) if tdist.is_initialized() else 1
        self.rank = tdist.get_rank(group) if tdist.is_initialized() else 0

    def all_reduce(self, t: torch.Tensor, op: str) -> torch.Tensor:
        if self.world > 1:
            tdist.all_reduce(t, op=self._OPS[op], group=self.group)
        return t

    def all_gather(self, t: torch.Tensor):
        out = [torch.empty_like(t) for _ in range(self.world)]
        tdist.all_gather(out, t, group=self.group)
        return out

    def all_to_all_single(self, out, inp, out_splits=None, in_splits=None):
        tdist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits,
                                group=self.group)

    def barrier(self):
        if self.world > 1:
            tdist.barrier(group=self.group)

    def share_cuda(self, tensors):
        """Every rank's `tensors` as device tensors usable here: this rank's own,
        the others' opened through CUDA IPC (torch's tensor reductions: the
        allocation's IPC handle plus offset; peer access over NVLink between
        GPUs of a node, plain device memory between processes of one GPU)."""
        from torch.multiprocessing.reductions import reduce_tensor

        mine = [reduce_tensor(t) for t in tensors]
        objs = [None] * self.world
        tdist.all_gather_object(objs, mine, group=self.group)
        out = []
        for r, o in enumerate(objs):
            out.append(list(tensors) if r == self.rank else [fn(*args) for fn, args in o])
        return out


# ------------------------------------------------------------- the sort

def dist_zsort(keys: torch.Tensor, payload: torch.Tensor | None, gidx_base: int, group=None, ops=None,
               k: int = DEFAULT_K, comm=None, exchange: str = "nccl"):
    """Globally stable sort of sharded records; returns this rank's slice.

    exchange: "nccl" -- stable partition into a send buffer, then
    all_to_all_single of keys and payload; "p2p" -- the fused exchange: the
    partition's scatter stores every record straight into its destination
    rank's receive buffer through CUDA IPC peer pointers (one kernel, no send
    buffer, no all_to_all; needs peer access between the ranks' GPUs).

    keys/payload: this rank's shard (contiguous global positions starting at
    gidx_base).  Returns (keys, payload, info) where concatenating every
    rank's result in rank order gives the stable sort of the global input.
    """
    ops = ops or DeviceOps(keys.device)
    comm = comm or TorchComm(group)
    world, rank = comm.world, comm.rank
    dev = ops.device
    kind = ops.kind(keys)
    n = keys.numel()
    info = {"world": world}

    # ---- D1: one pass per shard, one all_gather of six numbers per rank
    if n:
        mom, bits = ops.local_moments(keys)
        row = torch.cat([mom.to(torch.float64), bits.view(torch.float64)])
    else:
        row = torch.zeros(6, dtype=torch.float64, device=dev)
    rows = torch.stack(comm.all_gather(row)).cpu().numpy()  # (G, 6): count, s1, s2, c, min bits, max bits
    count, mean, m2, omin, omax = merge_moments(rows)
    info.update(total=int(count), omin=omin, omax=omax)
    if count == 0:
        return keys.clone(), (payload.clone() if payload is not None else None), info
    if omin == omax or world == 1:  # globally constant (already stable) or nothing to exchange
        k_, p_ = ops.local_sort(keys, payload) if n else (keys.clone(), payload)
        return k_, p_, info
    vmin, vmax = ord_to_value(omin, kind), ord_to_value(omax, kind)
    params = plan_params(count, 0.0, m2, mean, vmin, vmax, k)

    # ---- D2: per-rank histograms (all_gather) -> cuts
    hist = ops.bucket_histogram(keys, params)
    counts = torch.stack(comm.all_gather(hist)).cpu().numpy()  # (G, k)
    cuts = plan_cuts_exact(counts, world, rank, keys, params, gidx_base, ops, comm, kind)
    info["cuts"] = cuts

    # ---- D3: stable partition by destination and the exchange
    if exchange == "p2p":
        rk, rp, send, recv = _exchange_p2p(keys, payload, params, gidx_base, cuts, ops, comm, world, rank, dev)
    else:
        pk, pp, send = ops.partition(keys, payload, params, gidx_base, cuts)
        send_t = torch.tensor(send, dtype=torch.int64, device=dev)
        recv_t = torch.empty_like(send_t)
        comm.all_to_all_single(recv_t, send_t)
        recv = [int(x) for x in recv_t.tolist()]
        rk = torch.empty(sum(recv), dtype=keys.dtype, device=dev)
        comm.all_to_all_single(rk, pk, recv, send)
        rp = None
        if payload is not None:
            rp = torch.empty(sum(recv), dtype=payload.dtype, device=dev)
            comm.all_to_all_single(rp, pp, recv, send)
    info.update(sent=send, received=recv, exchange=exchange)
    # ---- local stable sort of the received records (global input order)
    if rk.numel() == 0:
        return rk, rp, info
    ok, op = ops.local_sort(rk, rp)
    return ok, op, info


def _exchange_p2p(keys, payload, params, gidx_base, cuts, ops, comm, world, rank, dev):
    """Fused partition + exchange: counts (all_gather), receive buffers shared
    by IPC, then one scatter kernel writes every record into its destination
    rank's buffer at (records of that destination from lower-ranked sources)
    + its stable position.  Chunks land in source-rank order, as all_to_all
    delivers them."""
    ws, send = ops.partition_plan(keys, payload, params, gidx_base, cuts)
    allc = torch.stack(comm.all_gather(torch.tensor(send, dtype=torch.int64, device=dev))).cpu().numpy()  # (src, dst)
    recv = [int(x) for x in allc[:, rank]]
    rk = torch.empty(sum(recv), dtype=keys.dtype, device=dev)
    rp = torch.empty(sum(recv), dtype=payload.dtype, device=dev) if payload is not None else None
    shared = comm.share_cuda([rk] + ([rp] if rp is not None else []))  # per rank: [keys buf, payload buf]
    offsets = [int(allc[:rank, d].sum()) for d in range(world)]
    ops.partition_send(keys, payload, ws, [shared[d][0] for d in range(world)],
                       [shared[d][1] for d in range(world)] if payload is not None else None, offsets)
    comm.barrier()  # every rank's stores into this rank's buffers are done
    del shared
    comm.barrier()  # the peers' mappings are released before the buffers can be freed
    return rk, rp, send, recv


def _ord_to_bits(o: int, kind: str) -> int:
    if kind == "int64":
        return o ^ SIGN
    return (o ^ SIGN) if o & SIGN else (~o & ((1 << 64) - 1))
