"""Single-box multi-GPU layer: a thin Python wrapper over
the C-ABI argcsr_mgpu_* (csrc/mgpu.cu, include/argcsr_gpu.h).

One process per GPU (torch.distributed is only the launcher's plumbing: it
carries the 128-byte ncclUniqueId from rank 0 to the others, and -- for the
NCCL-free p2p form -- the 64-byte CUDA IPC handles).  Everything else runs in
C++/CUDA behind the ABI:

* rows split into contiguous nnz-balanced slices (argcsr_partition_rows'
  rule), each rank converting ITS slice (bit-exact with the reference
  argcsr_from_csr(slice_p));
* x replicated; a step is the slice SpMV plus the exchange of y into every
  rank's next x: NCCL all-gather (in place) or grouped broadcasts, the halo
  (grouped send/recv of the rows other slices read), or p2p (the SpMV epilogue
  stores y into the peers' x over NVLink, flags + partial norms in peer
  memory);
* the power iteration with ||y||^2 fused into the SpMV epilogue, an 8-byte
  all-reduce, and the scaling fused into the next SpMV; the NCCL exchange of
  step k overlaps the interior groups of step k+1.

Replaces the reference's parallel_over / spmv_argcsr_parallel
(proj/src/bench.cpp:48-71, 109-116).
"""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _ext
from . import _layout_flags

EXCHANGES = {"auto": 0, "allgather": 1, "halo": 2, "p2p": 3}
EXCHANGE_NAMES = {0: "auto", 1: "allgather", 2: "halo", 3: "p2p", 4: "none"}


def partition_bounds(row_pointers, parts: int) -> np.ndarray:
    """nnz-balanced contiguous row ranges (argcsr_partition_rows)."""
    return np.asarray(_ext.partition_rows(np.asarray(row_pointers, dtype=np.uint64), parts), dtype=np.uint64)


def interior_group_range(row_pointers, columns, group_first, r0: int, r1: int) -> tuple[int, int]:
    """Longest run of groups whose rows read only columns in [r0, r1)
    (argcsr_plan_interior); group_first has G + 1 entries."""
    return tuple(_ext.plan_interior(np.asarray(row_pointers, np.uint64), np.asarray(columns, np.int32),
                                    np.asarray(group_first, np.uint64), r0, r1))


def needed_rows(columns, num_cols: int, bounds, self_rank: int) -> list:
    """Per owner p, the distinct rows of p's slice the columns read (argcsr_plan_needed)."""
    return _ext.plan_needed(np.asarray(columns, np.int32), num_cols, np.asarray(bounds, np.uint64), self_rank)


def _as_tensor(a, dtype=None) -> torch.Tensor:
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


class DistributedArgCsr:
    """A row-partitioned ARG-CSR matrix over the ranks of `group` (world size 1
    without torch.distributed).  Every rank passes the FULL matrix (host or
    device tensors / numpy arrays)."""

    def __init__(self, num_rows: int, num_cols: int, row_pointers, columns, values, tpg: int = 128, dcs: int = 1,
                 group=None, device: Optional[torch.device] = None, dtype=torch.float64, layout: str = "compact",
                 exchange: str = "auto", nccl: bool = True):
        if exchange not in EXCHANGES:
            raise ValueError("exchange must be 'auto', 'allgather', 'halo' or 'p2p'")
        self.group = group
        self.distributed = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.distributed else 1
        self.rank = dist.get_rank(group) if self.distributed else 0
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dtype = dtype
        self.num_rows, self.num_cols = num_rows, num_cols
        rp = _as_tensor(row_pointers, torch.int64)
        cols = _as_tensor(columns, torch.int32)
        vals = _as_tensor(values, dtype)
        on_dev = rp.is_cuda
        if on_dev and not (cols.is_cuda and vals.is_cuda):
            raise ValueError("row_pointers, columns and values must all be host or all be device tensors")
        if on_dev:
            torch.cuda.current_stream(self.device).synchronize()  # the CSR is read on other streams
        nccl_id = None
        if self.world > 1 and (nccl or exchange != "p2p"):
            box = [_ext.mgpu_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(box, src=self._global(0), group=group)
            nccl_id = box[0]
        self.h = _ext.MultiGpu.create_rank(
            num_rows, num_cols, int(cols.numel()), rp.data_ptr(), cols.data_ptr(), vals.data_ptr(),
            "float64" if dtype == torch.float64 else "float32", on_dev, self.rank, self.world, nccl_id, tpg, dcs,
            self.device.index if self.device.index is not None else 0, _layout_flags(layout), EXCHANGES[exchange])
        if exchange == "p2p" and self.world > 1 and nccl_id is None:
            # the NCCL-free form: IPC handles and need tables over the caller's channel
            mine = self.h.p2p_export()
            allx = [None] * self.world
            dist.all_gather_object(allx, mine, group=group)
            self.h.p2p_connect([a[0] for a in allx], [a[1] for a in allx])
        info = self.h.info()
        self.r0, self.r1 = int(info["row_begin"]), int(info["row_end"])
        self.interior = (int(info["interior_begin"]), int(info["interior_end"]))
        self.exchange = EXCHANGE_NAMES[int(info["exchange"])]
        self.halo_recv_rows = int(info["halo_recv_rows"])
        self.nnz_total = int(info["nnz"])
        self.local_matrix = self.h.local(0)
        self.bounds = partition_bounds(rp.cpu().numpy().view(np.uint64) if not on_dev else rp.cpu().numpy(),
                                       self.world)
        self.counts = [int(self.bounds[p + 1] - self.bounds[p]) for p in range(self.world)]

    def _global(self, r: int) -> int:
        return dist.get_global_rank(self.group, r) if self.group is not None else r

    def _stream(self) -> list:
        return [torch.cuda.current_stream(self.device).cuda_stream]

    # ------------------------------------------------------------------ steps
    def spmv_gather(self, x_full: torch.Tensor, out_full: torch.Tensor) -> None:
        """out = A x assembled on every rank (stream-ordered on the current stream)."""
        self.h.spmv_gather([x_full.data_ptr()], [out_full.data_ptr()], self._stream())

    def begin(self, x0: torch.Tensor, normalize: bool = True) -> None:
        """Start a run of iterated SpMVs (normalize: the power iteration) from x0."""
        self.h.begin([x0.contiguous().data_ptr()], normalize, self._stream())

    def step(self, last: bool = False) -> None:
        """One step; `last` exchanges every row (halo / p2p modes otherwise move
        only the rows other slices read)."""
        self.h.step(last, self._stream())

    def drain(self) -> None:
        """The current stream waits for the last exchange (end of a timed region)."""
        self.h.wait(self._stream())

    def finish(self):
        """(lambda, x): lambda = ||A x_{k-1}|| for the power iteration, and the
        current (normalised) x on this rank; synchronises."""
        x = torch.empty(self.num_cols, dtype=self.dtype, device=self.device)
        lam = self.h.finish([x.data_ptr()], self._stream())
        return lam, x

    def power_iteration(self, x0: torch.Tensor, iters: int):
        """`iters` steps of x <- A x / ||A x||; returns (lambda, x) on every rank."""
        self.begin(x0, normalize=True)
        for i in range(iters):
            self.step(last=i == iters - 1)
        return self.finish()

    # ----------------------------------------------------------- reporting
    def launches_per_step(self) -> int:
        m = self.local_matrix
        per = (1 if m.heavy_ctas else 0) + (1 if m.light_tiles else 0)
        if self.exchange == "p2p":
            return per + (1 if m.x_remap else 0) + (2 if self.world > 1 else 0) + 2  # + norm reduce(s), own flag
        if self.world > 1 and self.interior[1] > self.interior[0]:
            return 3 * per + (2 if m.x_remap else 0) + 2  # interior + two boundary ranges + 2-level norm reduce
        return per + (1 if m.x_remap else 0) + 2

    def step_description(self) -> str:
        if self.exchange == "p2p":
            return ("SpMV with y stored into every GPU's next x by its epilogue + fused ||y||^2 partials, "
                    "step flags and partial norms over peer memory, scaling fused into the next SpMV")
        return ("SpMV (interior groups, then boundary groups once the exchange landed) with fused ||y||^2, "
                f"8-byte NCCL all-reduce, {self.exchange} exchange of y on a collective stream, scaling fused "
                "into the next SpMV")

    def close(self) -> None:
        """Free the handle; collective (no peer still stores into our buffers)."""
        if self.h is None:
            return
        torch.cuda.synchronize(self.device)
        if self.world > 1 and self.distributed:
            dist.barrier(group=self.group)
        self.local_matrix = None
        self.h.free()
        self.h = None

    def __del__(self):
        try:
            if self.h is not None and self.world == 1:
                self.h.free()
        except Exception:
            pass
