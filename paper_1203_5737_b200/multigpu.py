"""Single-box multi-GPU layer: row-partitioned ARG-CSR.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch):

* rows are split into contiguous, nnz-balanced ranges (argcsr_partition_rows:
  r_p = lower_bound(row_pointers, p * nnz / P));
* every rank converts ITS OWN slice on its own GPU (row pointers rebased to 0,
  all columns kept), so slice p equals the reference argcsr_from_csr(slice_p)
  bit-for-bit (group boundaries restart at each slice start);
* x is replicated; a step is the local SpMV followed by the all-gather of the
  y slices into every rank's next x.  With equal slices that is one
  ncclAllGather straight into x; otherwise one broadcast per owner into its
  row range of x (no padding, no compaction copy).

The power iteration (config C5) is x_{k+1} = fl(y_k * fl(1 / ||y_k||_2)),
y_k = A x_k.  The scaling of step k is fused into the gathers of SpMV k+1
(argcsr_dev_spmv_scaled, bit-identical to scaling x first), and
||y_k||^2 is one 8-byte all-reduce of the per-rank partial sums.

Overlap.  Each rank finds the longest run of its groups whose
rows reference only columns it owns (interior groups; on a stencil slice all
but the first and last ~n^2 rows).  A step computes the interior groups first
(their x entries are the rank's own y from the previous step), then waits for
the previous step's all-gather -- which ran on NCCL's stream meanwhile -- and
computes the boundary groups; y is written straight into the rank's chunk of
the next x buffer and the in-place all-gather of step k overlaps the interior
SpMV of step k+1.

The collectives and the per-rank engine are separable so the host logic runs
on CPU with the gloo backend in tests (tests/test_multigpu_gloo.py), where a
test-only engine (the oracle) stands in for the device.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist


def partition_bounds(row_pointers: np.ndarray, parts: int) -> np.ndarray:
    """nnz-balanced contiguous row ranges (same rule as argcsr_partition_rows).

    bounds[p] = lower_bound(rp, rp[0] + floor(nnz * p / parts)), clamped so
    every part keeps at least one row when num_rows >= parts."""
    rp = np.asarray(row_pointers, dtype=np.uint64)
    n = rp.size - 1
    nnz = int(rp[-1] - rp[0])
    b = np.zeros(parts + 1, dtype=np.uint64)
    for p in range(1, parts):
        target = int(rp[0]) + (nnz * p) // parts
        r = int(np.searchsorted(rp, np.uint64(target), side="left"))
        lo = int(b[p - 1]) + (1 if n >= parts else 0)
        hi = n - (parts - p) if n >= parts else n
        b[p] = min(max(r, lo), hi)
    b[parts] = n
    return b


@dataclass
class CsrSlice:
    """Rows [row_begin, row_end) of a CSR matrix, row pointers rebased to 0."""

    row_begin: int
    row_end: int
    num_cols: int
    row_pointers: np.ndarray | torch.Tensor
    columns: np.ndarray | torch.Tensor
    values: np.ndarray | torch.Tensor

    @property
    def num_rows(self) -> int:
        return self.row_end - self.row_begin


def interior_group_range(row_pointers, columns, first_rows, r0: int, r1: int) -> tuple[int, int]:
    """Longest run [ga, gb) of groups whose rows reference only columns in
    [r0, r1).  `first_rows` has G + 1 entries (the last one is num_rows);
    row_pointers / columns are the slice's (rebased) arrays; works on numpy
    arrays or torch tensors (device-side for the big ones)."""
    t = torch.as_tensor(np.asarray(columns) if isinstance(columns, np.ndarray) else columns)
    rp = torch.as_tensor(np.asarray(row_pointers, dtype=np.int64) if isinstance(row_pointers, np.ndarray)
                         else row_pointers.to(torch.int64)).to(t.device)
    bad = ((t < r0) | (t >= r1)).to(torch.int64)
    cbad = torch.cat([torch.zeros(1, dtype=torch.int64, device=t.device), torch.cumsum(bad, 0)])
    row_bad = (cbad[rp[1:]] - cbad[rp[:-1]] > 0).to(torch.int64)
    rbad = torch.cat([torch.zeros(1, dtype=torch.int64, device=t.device), torch.cumsum(row_bad, 0)])
    fr = torch.as_tensor(np.asarray(first_rows, dtype=np.int64)).to(t.device)
    good = ~(rbad[fr[1:]] - rbad[fr[:-1]] > 0)
    g = np.concatenate([[False], good.cpu().numpy(), [False]]).astype(np.int8)
    edges = np.flatnonzero(np.diff(g))  # run starts and ends alternate
    if edges.size == 0:
        return 0, 0
    starts, ends = edges[0::2], edges[1::2]
    k = int(np.argmax(ends - starts))
    return int(starts[k]), int(ends[k])


def slice_rows(row_pointers, columns, values, num_cols: int, r0: int, r1: int) -> CsrSlice:
    a, b = int(row_pointers[r0]), int(row_pointers[r1])
    return CsrSlice(r0, r1, num_cols, row_pointers[r0:r1 + 1] - row_pointers[r0], columns[a:b], values[a:b])


class DeviceEngine:
    """The product engine: this rank's slice converted and multiplied on its GPU."""

    def __init__(self, sl: CsrSlice, tpg: int, dcs: int, device: torch.device, dtype=torch.float64,
                 layout: str = "compact"):
        import paper_1203_5737_b200 as argcsr

        self.device = device
        self.dtype = dtype
        rp = torch.as_tensor(np.asarray(sl.row_pointers).astype(np.int64)) if isinstance(sl.row_pointers, np.ndarray) \
            else sl.row_pointers.to(torch.int64)
        cols = torch.as_tensor(sl.columns) if isinstance(sl.columns, np.ndarray) else sl.columns
        vals = torch.as_tensor(sl.values) if isinstance(sl.values, np.ndarray) else sl.values
        self.stream = torch.cuda.current_stream(device)
        self.m = argcsr.argcsr_from_torch(sl.num_rows, sl.num_cols, rp.to(device).contiguous(),
                                          cols.to(device, torch.int32).contiguous(),
                                          vals.to(device, dtype).contiguous(), tpg, dcs, stream=self.stream,
                                          layout=layout)
        self.stream.synchronize()  # the handle is used from other streams afterwards

    def cur(self) -> int:
        """The caller's current stream: products are ordered with the torch
        ops around them (norms, copies), whatever stream the conversion used."""
        return torch.cuda.current_stream(self.device).cuda_stream

    def spmv(self, x: torch.Tensor, y: torch.Tensor, x_scale: Optional[torch.Tensor] = None) -> None:
        """y = A (s * x), s = x_scale[0] read on the device (None: 1)."""
        self.m.spmv_scaled_device(x.data_ptr(), 0 if x_scale is None else x_scale.data_ptr(), y.data_ptr(),
                                  self.cur())

    def spmv_range(self, x: torch.Tensor, y: torch.Tensor, g0: int, g1: int, x_scale: Optional[torch.Tensor] = None,
                   reuse_x: bool = False) -> None:
        """Rows of groups [g0, g1) of y = A (s * x) (argcsr_dev_spmv_ex)."""
        if g1 <= g0:
            return
        self.m.spmv_ex_device(x.data_ptr(), 0 if x_scale is None else x_scale.data_ptr(), g0, g1, y.data_ptr(),
                              1 if reuse_x else 0, self.cur())

    @property
    def num_groups(self) -> int:
        return self.m.num_groups

    def group_first_rows(self) -> np.ndarray:
        g = self.m.groups_array
        return np.concatenate([g[:, 0], [self.m.num_rows]]).astype(np.int64)


class DistributedArgCsr:
    """A row-partitioned ARG-CSR matrix across the ranks of `group`
    (world size 1 without torch.distributed)."""

    def __init__(self, num_rows: int, num_cols: int, row_pointers, columns, values, tpg: int = 128, dcs: int = 1,
                 group=None, device: Optional[torch.device] = None,
                 engine_factory: Optional[Callable[[CsrSlice], object]] = None, dtype=torch.float64,
                 layout: str = "compact", overlap: bool = True, exchange: str = "auto"):
        self.group = group
        self.distributed = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.distributed else 1
        self.rank = dist.get_rank(group) if self.distributed else 0
        rp_host = row_pointers.cpu().numpy() if isinstance(row_pointers, torch.Tensor) else np.asarray(row_pointers)
        self.bounds = partition_bounds(rp_host.astype(np.uint64), self.world)
        self.counts = [int(self.bounds[p + 1] - self.bounds[p]) for p in range(self.world)]
        self.num_rows, self.num_cols = num_rows, num_cols
        r0, r1 = int(self.bounds[self.rank]), int(self.bounds[self.rank + 1])
        self.slice = slice_rows(row_pointers, columns, values, num_cols, r0, r1)
        self.nnz_local = int(self.slice.row_pointers[-1])
        self.nnz_total = int(rp_host[-1] - rp_host[0])
        if engine_factory is None:
            dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
            self.engine = DeviceEngine(self.slice, tpg, dcs, dev, dtype, layout)
        else:
            self.engine = engine_factory(self.slice)
        self.device = self.engine.device
        self.dtype = dtype
        self.y = torch.empty(self.slice.num_rows, dtype=dtype, device=self.device)
        self.r0, self.r1 = r0, r1
        self.overlap = overlap and self.world > 1
        self.interior = (0, 0)
        self._pending = []  # outstanding async gather works (overlap mode)
        if self.overlap:
            self.interior = interior_group_range(self.slice.row_pointers, self.slice.columns,
                                                 self.engine.group_first_rows(), r0, r1)
        # x exchange between steps: the all-gather of every y slice, or only
        # the halo -- the x entries of other ranks this rank's columns use
        # (auto: halo when it moves < 1/4 of the all-gather's volume)
        if exchange not in ("auto", "allgather", "halo", "p2p"):
            raise ValueError("exchange must be 'auto', 'allgather', 'halo' or 'p2p'")
        self.halo = None
        self.peer = self.pstep = None
        if exchange == "p2p":
            # fused SpMV + peer stores over NVLink (peer.py): no collective in the step
            from .peer import PeerBuffers, PeerPowerIteration

            self.overlap = False
            from .peer import needed_ranges

            self.peer = PeerBuffers(self.rank, self.world, num_cols, dtype, self.device)
            send = None
            if self.world > 1:
                handles = [None] * self.world
                dist.all_gather_object(handles, self.peer.handle, group=self.group)
                self.peer.connect_ipc(handles)
                # rows each peer reads from this rank (its columns in our row range)
                need = [None] * self.world
                dist.all_gather_object(need, needed_ranges(self.slice.columns, self.bounds), group=self.group)
                send = {q: tuple(need[q][self.rank]) for q in range(self.world) if q != self.rank}
            self.pstep = PeerPowerIteration(self.engine, r0, r1, self.peer, send_ranges=send)
            self.exchange = "p2p"
            return
        if self.overlap and exchange != "allgather":
            self.halo = self._build_halo()
            total = int(self.halo["recv_total"].item())
            if exchange == "auto" and total * 4 >= self.num_rows:
                self.halo = None
        self.exchange = "halo" if self.halo is not None else ("allgather" if self.world > 1 else "none")

    def _build_halo(self) -> dict:
        """Halo plan: per peer, the global rows this rank needs (recv) and the
        global rows it must send (learned with two all-to-alls)."""
        cols = self.slice.columns
        c = torch.as_tensor(np.asarray(cols) if isinstance(cols, np.ndarray) else cols).to(self.device, torch.int64)
        need = torch.unique(c[(c < self.r0) | (c >= self.r1)])  # sorted
        b = torch.as_tensor(self.bounds.astype(np.int64), device=self.device)
        cuts = torch.searchsorted(need, b)
        recv_counts = (cuts[1:] - cuts[:-1]).to(torch.int64)
        dev_cc = self.device if self.device.type == "cuda" else torch.device("cpu")
        sc = torch.empty(self.world, dtype=torch.int64, device=dev_cc)
        dist.all_to_all_single(sc, recv_counts.to(dev_cc), group=self.group)
        rc_l, sc_l = recv_counts.cpu().tolist(), sc.cpu().tolist()
        send_rows = torch.empty(sum(sc_l), dtype=torch.int64, device=dev_cc)
        dist.all_to_all_single(send_rows, need.to(dev_cc), output_split_sizes=sc_l, input_split_sizes=rc_l,
                               group=self.group)
        return {"recv_rows": need, "recv_counts": rc_l, "send_local": (send_rows.to(self.device) - self.r0),
                "send_counts": sc_l, "recv_total": torch.tensor(sum(rc_l)),
                "recv_buf": torch.empty(sum(rc_l), dtype=self.dtype, device=self.device),
                "send_buf": torch.empty(sum(sc_l), dtype=self.dtype, device=self.device)}

    # ------------------------------------------------------------ collectives
    def gather(self, y_local: torch.Tensor, x_full: torch.Tensor) -> None:
        """All-gather the y slices into x_full (every rank)."""
        if self.world == 1:
            x_full.copy_(y_local)
            return
        if len(set(self.counts)) == 1:
            dist.all_gather_into_tensor(x_full, y_local, group=self.group)
            return
        off = 0
        for p, n in enumerate(self.counts):
            seg = x_full[off:off + n]
            if p == self.rank:
                seg.copy_(y_local)
            dist.broadcast(seg, src=dist.get_global_rank(self.group, p) if self.group is not None else p,
                           group=self.group)
            off += n

    def gather_async(self, x_full: torch.Tensor) -> None:
        """In-place all-gather: this rank's chunk x_full[r0:r1] already holds
        its y slice; the works complete on the collective stream."""
        if len(set(self.counts)) == 1:
            self._pending.append(dist.all_gather_into_tensor(x_full, x_full[self.r0:self.r1], group=self.group,
                                                             async_op=True))
            return
        off = 0
        for p, n in enumerate(self.counts):
            src = dist.get_global_rank(self.group, p) if self.group is not None else p
            self._pending.append(dist.broadcast(x_full[off:off + n], src=src, group=self.group, async_op=True))
            off += n

    def halo_async(self, x_full: torch.Tensor) -> None:
        """Send the rows peers need from this rank's chunk x_full[r0:r1] and
        receive this rank's halo; the scatter into x_full follows the wait."""
        h = self.halo
        torch.index_select(x_full[self.r0:self.r1], 0, h["send_local"], out=h["send_buf"])
        self._pending.append(dist.all_to_all_single(h["recv_buf"], h["send_buf"],
                                                    output_split_sizes=h["recv_counts"],
                                                    input_split_sizes=h["send_counts"], group=self.group,
                                                    async_op=True))
        self._halo_target = x_full

    def exchange_async(self, x_full: torch.Tensor) -> None:
        if self.halo is not None:
            self.halo_async(x_full)
        else:
            self.gather_async(x_full)

    def close(self) -> None:
        """Release the peer buffers (exchange='p2p'); call on every rank."""
        if self.peer is not None:
            torch.cuda.synchronize(self.device)
            if self.world > 1:
                dist.barrier(group=self.group)  # no peer still stores into our buffers
            self.peer.close()
            self.peer = self.pstep = None

    def wait_gather(self) -> None:
        """Stream-order (NCCL) or complete (gloo) the outstanding exchange."""
        for w in self._pending:
            w.wait()
        if self._pending and self.halo is not None:
            self._halo_target.index_copy_(0, self.halo["recv_rows"], self.halo["recv_buf"])
        self._pending = []

    def assemble(self, x_full: torch.Tensor) -> None:
        """All-gather every rank's chunk of x_full (after a halo-only step,
        the other ranks' rows of x_full are stale)."""
        self.wait_gather()
        if self.world > 1:
            y = x_full[self.r0:self.r1].clone()
            self.gather(y, x_full)

    def _spmv_overlapped(self, xin: torch.Tensor, xout: torch.Tensor, x_scale: Optional[torch.Tensor]) -> torch.Tensor:
        """Interior groups, wait for xin's gather, boundary groups; y into
        xout's own chunk (returned as a view)."""
        y = xout[self.r0:self.r1]
        ga, gb = self.interior
        G = self.engine.num_groups
        self.engine.spmv_range(xin, y, ga, gb, x_scale)
        self.wait_gather()
        self.engine.spmv_range(xin, y, 0, ga, x_scale)
        self.engine.spmv_range(xin, y, gb, G, x_scale, reuse_x=ga > 0)
        return y

    def allreduce_sum(self, v: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            dist.all_reduce(v, op=dist.ReduceOp.SUM, group=self.group)
        return v

    # ------------------------------------------------------------------ steps
    def spmv_gather(self, x_full: torch.Tensor, out_full: torch.Tensor, x_scale: Optional[torch.Tensor] = None,
                    wait: bool = True) -> None:
        """out = A (x_scale * x) assembled on every rank (iterated-SpMV step).
        In overlap mode the gather is left in flight unless `wait`; the next
        spmv_gather on `out_full` (or wait_gather) orders it."""
        if not self.overlap:
            self.engine.spmv(x_full, self.y, x_scale)
            self.gather(self.y, out_full)
            return
        self._spmv_overlapped(x_full, out_full, x_scale)
        self.exchange_async(out_full)
        if wait:
            self.wait_gather()
            if self.halo is not None:
                self.assemble(out_full)

    def power_iteration(self, x0: torch.Tensor, iters: int):
        """`iters` steps of x <- A x / ||A x||; returns (lambda, x) with
        lambda = ||A x_{iters-1}|| (x normalised), on every rank."""
        if self.pstep is not None:
            self.pstep.normalize = True
            self.pstep.begin(x0)
            for i in range(iters):
                self.pstep.step(full=i == iters - 1)  # halo stores, the last step assembles all of x
            return self.pstep.finish()
        buf = [x0.clone(), torch.empty_like(x0)]
        scale = torch.ones(1, dtype=torch.float64, device=self.device)
        s2 = torch.zeros(1, dtype=torch.float64, device=self.device)
        for k in range(iters):
            self.step(buf[k % 2], buf[(k + 1) % 2], scale, s2)
        self.wait_gather()
        if self.halo is not None:
            self.assemble(buf[iters % 2])
        lam = float(torch.sqrt(s2).item())  # the only host synchronisation
        x = buf[iters % 2] * scale  # materialise the last normalisation
        return lam, x

    def step(self, xin: torch.Tensor, xout: torch.Tensor, scale: torch.Tensor, s2: torch.Tensor) -> None:
        """One power-iteration step, device-side only: y = A (scale * xin);
        s2 = ||y||^2 (all-reduced); xout = all-gather(y); scale = 1/sqrt(s2)."""
        if self.overlap:
            y = self._spmv_overlapped(xin, xout, scale)
        else:
            y = xout if self.world == 1 else self.y  # one GPU: y is the next x, no copy
            self.engine.spmv(xin, y, scale)
        y64 = y.to(torch.float64)
        s2.copy_(torch.dot(y64, y64).reshape(1))
        self.allreduce_sum(s2)
        if self.overlap:
            self.exchange_async(xout)  # in flight under the next step's interior groups
        elif self.world > 1:
            self.gather(y, xout)
        torch.reciprocal(torch.sqrt(s2), out=scale)
