"""Host-to-host sorts as a stream: both PCIe directions busy at once.

One ``zsort`` of host data is three serial steps -- host-to-device copy of
the keys and payload, the sort, device-to-host copy of the result -- and
every output key depends on every input key, so inside one sort nothing
overlaps: at 10^8 keys the copies are 43 ms and the sort 3.4 ms.  A caller
with a *sequence* of arrays to sort (the reference's benchmark harness and
file workflows, bench.py:e2e) does not have to pay the two directions one
after the other: ``SortPipeline`` keeps ``depth`` sets of device buffers and
three CUDA streams, so the upload of sort i+1, sort i and the download of
sort i-1 run concurrently.  Steady state is one sort per max(H2D, D2H, sort)
instead of their sum.

Same contract as ``core.zsort`` (reference core.py:348-400): stable, inputs
untouched, NaN raises ValueError, the CUDA library is the only path.

    pipe = SortPipeline(n, torch.float64, torch.int32)
    t0 = pipe.submit(keys0, pay0, out_k0, out_p0)   # pinned host tensors
    t1 = pipe.submit(keys1, pay1, out_k1, out_p1)
    pipe.wait(t0); pipe.wait(t1)                    # or pipe.drain()
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .core import SortConfig, _KEY_CODES


class _Slot:
    def __init__(self, n, kdt, pdt, ws_bytes, dev):
        self.d_keys = torch.empty(n, dtype=kdt, device=dev)
        self.d_pay = torch.empty(n, dtype=pdt, device=dev) if pdt is not None else None
        self.d_ok = torch.empty_like(self.d_keys)
        self.d_op = torch.empty_like(self.d_pay) if pdt is not None else None
        self.ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        self.ev_in = torch.cuda.Event()      # inputs of the slot's current sort are on the device
        self.ev_sorted = torch.cuda.Event()  # its sort is done: inputs consumed, outputs ready
        self.ev_out = torch.cuda.Event()     # its outputs are on the host (the event of its latest ticket)
        self.busy = False
        self.dst = None


class SortPipeline:
    """``depth`` device buffer sets and three streams (upload, sort,
    download).  ``submit`` enqueues the upload at once and launches the sort
    of the *previous* ticket behind it: the library's sort call holds the
    host until the last partition level is enqueued (one wait per level), so
    the next upload has to be in flight before that call starts.  A ticket's
    host tensors belong to the pipeline until ``wait(ticket)`` returns.  One
    pipeline per host thread (the object itself is not thread-safe; separate
    pipelines on separate threads are independent, like separate ``zsort``
    calls)."""

    def __init__(self, n, key_dtype, payload_dtype=None, config: SortConfig | None = None, depth: int = 2,
                 device=None):
        if key_dtype not in _KEY_CODES:
            raise TypeError("keys must be int64 or float64")
        if payload_dtype is not None and torch.empty(0, dtype=payload_dtype).element_size() not in (4, 8):
            raise TypeError("pipeline payloads are 4 or 8 bytes wide")
        if n < 1 or depth < 1:
            raise ValueError("n and depth must be positive")
        if not torch.cuda.is_available():
            raise RuntimeError("SortPipeline needs a CUDA device (there is no CPU fallback)")
        self.n, self.kdt, self.pdt = int(n), key_dtype, payload_dtype
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.cfg = (config if config is not None else SortConfig()).to_c()
        self.L = _lib.load()
        self.kd = _KEY_CODES[key_dtype]
        self.pb = 0 if payload_dtype is None else torch.empty(0, dtype=payload_dtype).element_size()
        with torch.cuda.device(self.dev):
            self.ws_bytes = self.L.zsb_workspace_bytes(self.n, self.kd, self.pb, self.cfg)
            self.slots = [_Slot(self.n, key_dtype, payload_dtype, self.ws_bytes, self.dev) for _ in range(depth)]
            self.s_in, self.s_sort, self.s_out = (torch.cuda.Stream(self.dev) for _ in range(3))
        self.tickets = 0
        self.pending = None  # ticket whose upload is enqueued and whose sort is not launched yet
        self.done = {}       # ticket -> event recorded behind its download, until waited for

    def _check(self, t, name, dt):
        if not isinstance(t, torch.Tensor) or t.dtype != dt or tuple(t.shape) != (self.n,) or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous {dt} tensor of shape ({self.n},)")

    def submit(self, keys, payload=None, out_keys=None, out_payload=None) -> int:
        """Enqueue one sort: ``keys``/``payload`` are read (pinned host tensors
        make the copies asynchronous), the result lands in ``out_keys`` /
        ``out_payload`` once ``wait(ticket)`` returns."""
        self._check(keys, "keys", self.kdt)
        self._check(out_keys, "out_keys", self.kdt)
        if self.pdt is not None:
            self._check(payload, "payload", self.pdt)
            self._check(out_payload, "out_payload", self.pdt)
        t = self.tickets
        slot = self.slots[t % len(self.slots)]
        if slot.busy:  # the slot's previous sort: launched (inputs consumed on ev_sorted), outputs downloaded
            self._launch_pending_upto(t - len(self.slots))
        with torch.cuda.device(self.dev):
            if slot.busy:
                self.s_in.wait_event(slot.ev_sorted)
            with torch.cuda.stream(self.s_in):
                slot.d_keys.copy_(keys, non_blocking=True)
                if self.pdt is not None:
                    slot.d_pay.copy_(payload, non_blocking=True)
                slot.ev_in.record(self.s_in)
        # the previous ticket's sort goes in behind this upload
        prev = self.pending
        slot.dst = (out_keys, out_payload)
        slot.busy = True
        self.tickets += 1
        self.pending = t
        if prev is not None:
            self._launch(prev)
        return t

    def _launch_pending_upto(self, t):
        if self.pending is not None and self.pending <= t:
            p, self.pending = self.pending, None
            self._launch(p)

    def _launch(self, t):
        slot = self.slots[t % len(self.slots)]
        with torch.cuda.device(self.dev):
            self.s_sort.wait_event(slot.ev_in)
            self.s_sort.wait_event(slot.ev_out)  # the slot's previous download has left the output buffers
            rc = self.L.zsb_sort(slot.d_keys.data_ptr(), self.kd,
                                 slot.d_pay.data_ptr() if slot.d_pay is not None else None, self.pb,
                                 slot.d_ok.data_ptr(), slot.d_op.data_ptr() if slot.d_op is not None else None,
                                 self.n, self.cfg, slot.ws.data_ptr(), self.ws_bytes, None,
                                 ctypes.c_void_p(self.s_sort.cuda_stream))
            _lib.check(rc)  # ZSB_ERR_NAN -> ValueError, like core.zsort
            slot.ev_sorted.record(self.s_sort)
            self.s_out.wait_event(slot.ev_sorted)
            ok, op = slot.dst
            with torch.cuda.stream(self.s_out):
                ok.copy_(slot.d_ok, non_blocking=True)
                if self.pdt is not None:
                    op.copy_(slot.d_op, non_blocking=True)
                slot.ev_out = torch.cuda.Event()
                slot.ev_out.record(self.s_out)
                self.done[t] = slot.ev_out
        if self.pending == t:
            self.pending = None

    def wait(self, ticket: int) -> None:
        """Block until the outputs of ``ticket`` are in its host tensors."""
        if ticket < 0 or ticket >= self.tickets:
            raise ValueError("unknown ticket")
        self._launch_pending_upto(ticket)
        ev = self.done.pop(ticket, None)
        if ev is not None:  # None: already waited for
            ev.synchronize()

    def drain(self) -> None:
        """Launch what is pending and wait for every outstanding sort."""
        self._launch_pending_upto(self.tickets - 1)
        for t in sorted(self.done):
            self.done.pop(t).synchronize()
