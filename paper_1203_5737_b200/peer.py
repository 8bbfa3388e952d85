"""Fused SpMV + all-gather over peer memory (the B200-native multi-GPU step).

The NCCL step (multigpu.py) is "SpMV into my chunk of x', then an
all-gather of the chunks".  Here the all-gather disappears into the SpMV:
every rank's kernel epilogue stores each y row into its own next-x buffer AND
into every peer's next-x buffer through the NVLink peer mapping
(argcsr_dev_spmv_peer), so the slices travel tile by tile while the SpMV
streams the matrix.  Completion is announced with one flag per (receiver,
sender) -- a monotone step counter stored with system-scope release after the
SpMV (argcsr_peer_signal) and awaited with acquire loads by the receiver
(argcsr_peer_wait) -- which also carries each rank's partial ||y||^2 for the
power iteration.

Buffers, per rank, in ONE device allocation shared through CUDA IPC
(argcsr_peer_alloc / argcsr_peer_open):

    x[2][num_cols]  (dtype)   double-buffered x of the power iteration
    flags[world]    (u64)     flags[p] = last step rank p has completed here
    partial[2][world] (f64)   partial[b][p] = rank p's ||y_p||^2 for buffer b

Step k (reads buffer k % 2, writes (k + 1) % 2 on every GPU):
    wait until flags[p] >= k for all peers p       (x_k complete here, and every
                                                    peer is done reading (k+1)%2)
    scale = 1 / sqrt(sum_p partial[k % 2][p])      (k > 0; same order on all ranks)
    y = A (scale * x_k), stored locally and into each peer's x[(k+1)%2][r0:r1]
    partial[(k+1)%2][rank] = ||y||^2, copied to every peer, then flags = k + 1

Double buffering is enough: a rank writes a peer's buffer (k+1)%2 only after
it has seen that peer's flag k, i.e. after the peer's SpMV k-1 (the last
reader of that buffer) completed.

Only one GPU is available to this repo's tests, so the protocol is checked
(tests/test_peer.py) with P virtual ranks on one device (peer "mappings" are
plain device pointers) and with two processes sharing one GPU through real
CUDA IPC handles.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch

from . import _ext

_TYPESTR = {torch.float64: "<f8", torch.float32: "<f4", torch.int64: "<i8"}


class _DevArray:
    """A raw device range as a __cuda_array_interface__ object (zero-copy torch view)."""

    def __init__(self, ptr: int, n: int, dtype: torch.dtype):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": _TYPESTR[dtype], "data": (ptr, False),
                                         "version": 3, "strides": None}


def _view(ptr: int, n: int, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    return torch.as_tensor(_DevArray(ptr, n, dtype), device=device)


def needed_ranges(columns, bounds) -> np.ndarray:
    """[world, 2]: for each owner p, the global rows [lo, hi) of p's slice that
    `columns` (this rank's slice) reference; (0, 0) when none.  A rank sends
    peer q only rows in q's range for it (a halo for banded matrices)."""
    c = torch.as_tensor(np.asarray(columns) if isinstance(columns, np.ndarray) else columns).to(torch.int64)
    b = np.asarray(bounds, dtype=np.int64)
    out = np.zeros((b.size - 1, 2), dtype=np.int64)
    for p in range(b.size - 1):
        sel = c[(c >= int(b[p])) & (c < int(b[p + 1]))]
        if sel.numel():
            out[p] = (int(sel.min()), int(sel.max()) + 1)
    return out


class PeerBuffers:
    """One rank's shared buffers (layout in the module docstring) and the
    device addresses of every peer's copy of them."""

    def __init__(self, rank: int, world: int, num_cols: int, dtype: torch.dtype, device: torch.device):
        if world > 8:
            raise ValueError("the peer step supports up to 8 GPUs (7 peers)")
        self.rank, self.world, self.num_cols, self.dtype, self.device = rank, world, num_cols, dtype, device
        es = torch.empty(0, dtype=dtype).element_size()
        self.es = es
        self.off_x = [0, ((num_cols * es + 255) // 256) * 256]
        self.off_flags = 2 * self.off_x[1]
        self.off_partial = self.off_flags + ((world * 8 + 255) // 256) * 256
        self.bytes = self.off_partial + 2 * world * 8
        self.base, self.handle = _ext.peer_alloc(self.bytes, device.index if device.index is not None else 0)
        self.x = [_view(self.base + o, num_cols, dtype, device) for o in self.off_x]
        self.flags = _view(self.base + self.off_flags, world, torch.int64, device)
        self.partial = [_view(self.base + self.off_partial + b * world * 8, world, torch.float64, device)
                        for b in range(2)]
        self.peer_base: dict[int, int] = {}
        self._opened: list[int] = []

    # ----------------------------------------------------------- connection
    def connect_local(self, others: Sequence["PeerBuffers"]) -> None:
        """Single-process ranks on one device: peers' buffers are plain pointers."""
        for o in others:
            if o.rank != self.rank:
                self.peer_base[o.rank] = o.base

    def connect_ipc(self, handles: Sequence[bytes]) -> None:
        """Multi-process: open every other rank's IPC handle on this device."""
        dev = self.device.index if self.device.index is not None else 0
        for p, h in enumerate(handles):
            if p != self.rank:
                b = _ext.peer_open(h, dev)
                self._opened.append(b)
                self.peer_base[p] = b

    @property
    def peers(self) -> list[int]:
        return sorted(self.peer_base)

    def peer_x(self, b: int, row0: int) -> list[int]:
        return [self.peer_base[q] + self.off_x[b] + row0 * self.es for q in self.peers]

    def peer_flag_slots(self) -> list[int]:
        return [self.peer_base[q] + self.off_flags + self.rank * 8 for q in self.peers]

    def peer_partial_slots(self, b: int) -> list[int]:
        return [self.peer_base[q] + self.off_partial + (b * self.world + self.rank) * 8 for q in self.peers]

    def close(self) -> None:
        for b in self._opened:
            _ext.peer_close(b)
        self._opened = []
        self.peer_base = {}
        if self.base:
            torch.cuda.synchronize(self.device)
            self.x = self.flags = self.partial = None
            _ext.peer_free(self.base)
            self.base = 0


class PeerPowerIteration:
    """One rank's power iteration with the fused SpMV + peer-store exchange
    (normalize=False: the plain iterated SpMV x_{k+1} = A x_k, no norms).

    `engine` is the rank's DeviceEngine (its converted row slice [r0, r1))."""

    def __init__(self, engine, r0: int, r1: int, bufs: PeerBuffers, normalize: bool = True,
                 send_ranges: Optional[dict] = None):
        self.engine, self.r0, self.r1, self.bufs = engine, r0, r1, bufs
        self.normalize = normalize
        self.device = bufs.device
        # rows (local to the slice) each peer reads from this rank: q -> (lo, hi)
        self.peer_rows = []
        if send_ranges is not None:
            for q in bufs.peers:
                lo, hi = send_ranges[q]
                lo, hi = (lo - r0, hi - r0) if hi > lo else (0, 0)
                self.peer_rows += [max(lo, 0), max(hi, 0)]
        self.scale = torch.ones(1, dtype=torch.float64, device=bufs.device)
        # Step numbers are absolute and never reset: the flags compare against
        # them, so a second run on the same buffers cannot pass a wait on a
        # stale flag of the first run.
        self.k = 0
        self.k0 = 0  # first step of the current run

    def _cur(self) -> int:
        """The caller's current stream: the peer kernels, the SpMV and the
        torch ops on the norms are all ordered on it."""
        return torch.cuda.current_stream(self.device).cuda_stream

    def begin(self, x0: torch.Tensor) -> None:
        """Start a run from x0 (collective: every rank calls it).  Only this
        rank's own buffer is written; peers store into it only after seeing
        this rank's flag for the step before theirs."""
        self.bufs.x[self.k % 2].copy_(x0)
        self.scale.fill_(1.0)
        self.k0 = self.k

    def wait(self, k: int) -> None:
        if self.bufs.peers and k > 0:
            _ext.peer_wait(self.bufs.flags.data_ptr(), self.bufs.world, k, self._cur())

    def step(self, full: bool = False) -> None:
        """One step; `full` stores every row into every peer (the last step of
        a run, so that all GPUs end with the whole x), else only the rows each
        peer reads."""
        k, b = self.k, self.k % 2
        nb = (k + 1) % 2
        bufs = self.bufs
        self.wait(k)
        if k > self.k0 and self.normalize:
            torch.reciprocal(torch.sqrt(bufs.partial[b].sum().reshape(1)), out=self.scale)
        y = bufs.x[nb][self.r0:self.r1]
        self.engine.m.spmv_peer_device(bufs.x[b].data_ptr(), self.scale.data_ptr() if self.normalize else 0, 0,
                                       self.engine.num_groups, y.data_ptr(), bufs.peer_x(nb, self.r0),
                                       [] if full else self.peer_rows, 0, self._cur())
        own = bufs.partial[nb][bufs.rank:bufs.rank + 1]
        if self.normalize:
            y64 = y.to(torch.float64)
            own.copy_(torch.dot(y64, y64).reshape(1))
        if bufs.peers:
            _ext.peer_signal(bufs.peer_flag_slots(), k + 1, own.data_ptr() if self.normalize else 0,
                             bufs.peer_partial_slots(nb) if self.normalize else [], self._cur())
        bufs.flags[bufs.rank:bufs.rank + 1].fill_(k + 1)  # own slot: the wait covers all `world` slots
        self.k = k + 1

    def current(self) -> torch.Tensor:
        """x_k (after the wait for the peers' slices), this rank's buffer view."""
        self.wait(self.k)
        return self.bufs.x[self.k % 2]

    def finish(self):
        """(lambda, x): lambda = ||A x_{k-1}|| and the normalised last x."""
        b = self.k % 2
        self.wait(self.k)
        s2 = self.bufs.partial[b].sum()
        lam = float(torch.sqrt(s2).item())
        x = self.bufs.x[b] * torch.reciprocal(torch.sqrt(s2))
        return lam, x


def power_iteration_local(engines: Sequence, bounds: Sequence[int], num_cols: int, x0: torch.Tensor, iters: int,
                          dtype: torch.dtype = torch.float64, normalize: bool = True,
                          slice_columns: Optional[Sequence] = None):
    """P virtual ranks on ONE device (tests): each rank's engine, the peer
    protocol with plain device pointers, steps interleaved rank by rank
    (halo-only stores when the ranks' slice columns are given, the last step
    full).  Returns per rank (lambda, x) -- or x_iters (a copy) when not
    normalize."""
    P = len(engines)
    dev = x0.device
    bufs = [PeerBuffers(p, P, num_cols, dtype, dev) for p in range(P)]
    for b in bufs:
        b.connect_local(bufs)
    need = [needed_ranges(slice_columns[p], bounds) for p in range(P)] if slice_columns is not None else None
    runs = [PeerPowerIteration(engines[p], int(bounds[p]), int(bounds[p + 1]), bufs[p], normalize,
                               {q: tuple(need[q][p]) for q in range(P) if q != p} if need is not None else None)
            for p in range(P)]
    try:
        for r in runs:
            r.begin(x0)
        for i in range(iters):
            for r in runs:
                r.step(full=i == iters - 1)
        return [r.finish() if normalize else r.current().clone() for r in runs]
    finally:
        torch.cuda.synchronize(dev)
        for b in bufs:
            b.close()
