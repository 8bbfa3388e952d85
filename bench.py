#!/usr/bin/env python
"""ARG-CSR SpMV benchmark (BASELINE.json metric: SpMV GFLOP/s and effective HBM
GB/s (% of 8 TB/s) at 1/2/4/8 B200 vs the CPU reference).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--tpg 128] [--dcs 1]
  python bench.py --impl reference ...      # the reference CPU path (oracle/_ref)

A "step" is one ARG-CSR SpMV y = A x over the whole synthetic matrix of the
config with x, y and the matrix resident in HBM (N = 1).  At N > 1 the rows
are nnz-balanced across ranks, each rank converts its own slice, and a step
is the local SpMV plus the all-gather of y into every rank's next x (the
iterated-SpMV / power-iteration step of config C5); value = 2 * nnz(total) /
max-over-ranks step time (strong scaling).

Rank 0 prints ONE JSON line.  Algorithmic bytes per SpMV:
alg_bytes = nnz*(S_v + 4) + (rows + cols)*S_v, S_v = 8 (fp64) / 4 (fp32);
flops = 2*nnz.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

NOMINAL_HBM_GBS = 8000.0
FALLBACK_HBM_GBS = 6650.0


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C4f32", "C5"])
    p.add_argument("--tpg", type=int, default=128)
    p.add_argument("--dcs", type=int, default=1)
    p.add_argument("--layout", default="compact", choices=["compact", "reference"],
                   help="device storage of the value/column blocks (include/argcsr_gpu.h ARGCSR_LAYOUT_REFERENCE)")
    p.add_argument("--x-remap", default="auto", choices=["auto", "on", "off"],
                   help="device column order (single-GPU path): library decision, or forced")
    p.add_argument("--no-variants", action="store_true", help="skip the tuned-dcs and cuSPARSE side runs")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-steps", type=int, default=20)
    p.add_argument("--exchange", default="auto", choices=["auto", "allgather", "halo", "p2p"],
                   help="multi-GPU x exchange: NCCL all-gather / halo all-to-all (auto picks), or p2p: "
                        "the SpMV epilogue stores y straight into the peers' x over NVLink (peer.py)")
    p.add_argument("--power-iteration", action="store_true",
                   help="a step is one power-iteration step (SpMV, ||y|| all-reduce, all-gather, fused scaling)")
    return p.parse_args()


# ------------------------------------------------------------------ helpers
def measured_peak():
    f = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def alg_bytes(nnz: int, rows: int, cols: int, sv: int) -> int:
    return nnz * (sv + 4) + (rows + cols) * sv


def traffic_from_profiles(key: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the
    committed ncu --set full summary (profiles/ncu_traffic.json), or None."""
    f = ROOT / "profiles" / "ncu_traffic.json"
    try:
        return json.loads(f.read_text()).get(key)
    except Exception:
        return None


class ClockSampler:
    """Polls NVML (SM clock, throttle reasons) from a thread; the samples taken
    between mark_start() and mark_end() are the timed-region record."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples = []
        self.period = period_s
        self.t0 = self.t1 = None
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()
        self._th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((time.perf_counter(), sm, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self._th.start()

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_end(self):
        self.t1 = time.perf_counter()

    def stop(self):
        self._stop.set()
        if self.ok:
            self._th.join(timeout=1)

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "note": "NVML unavailable"}
        inside = [s for s in self.samples if self.t0 <= s[0] <= self.t1]
        note = "sampled during the timed region"
        if not inside:  # region shorter than the polling period: nearest samples under load
            inside = sorted(self.samples, key=lambda s: abs(s[0] - self.t1))[:3]
            note = "timed region shorter than the 5 ms NVML poll; nearest samples"
        reasons = set()
        for _, _, rs in inside:
            for bit, name in self.REASONS.items():
                if rs & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[1] for s in inside) if inside else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(inside), "note": note}


def cpu_info():
    cores = os.cpu_count()
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return cores, model


# ----------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's own CPU path: argcsr_from_csr + spmv_argcsr_parallel
    (proj/src/argcsr.cpp:123-155, bench.cpp:109-116) from oracle/_ref, with
    all host threads, timed like run_benchmark (bench.cpp:128-141)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import torch

    import oracle
    from paper_1203_5737_b200 import synthetic

    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libargcsr_ref.so not built"}))
        return
    cfg = synthetic.CONFIGS[args.config]
    if cfg["dtype"] != "float64":
        print(json.dumps({"impl": "reference", "unavailable": "the reference library is fp64-only (SPEC.md:82)"}))
        return
    ref = oracle.ref()
    t = time.perf_counter()
    A = cfg["gen"]("cpu")
    csr = oracle.Csr(A.num_rows, A.num_cols, A.row_pointers.numpy().view(np.uint64), A.columns.numpy(),
                     A.values.numpy())
    gen_s = time.perf_counter() - t
    t = time.perf_counter()
    h = ref.argcsr_handle(csr, args.tpg, args.dcs)
    conv_s = time.perf_counter() - t
    workers = os.cpu_count()
    x = oracle.bench_input(A.num_cols)
    times, _ = ref.time_spmv_argcsr_parallel(h, x, workers, args.warmup, args.steps, A.num_rows)
    ref.free_argcsr(h)
    med = float(np.median(times))
    gflops = 2.0 * A.nnz / med / 1e9
    cores, model = cpu_info()
    sample = (f"{args.steps} x spmv_argcsr_parallel over the full {args.config} matrix "
              f"(tpg={args.tpg}, dcs={args.dcs}) after {args.warmup} warm-up, median; workers={workers}")
    out = {
        "impl": "reference", "metric": "SpMV GFLOP/s", "value": round(gflops, 4), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": med * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": args.config, "matrix": A.name, "rows": A.num_rows,
                                        "nnz": A.nnz, "threads_per_group": args.tpg,
                                        "desired_chunk_size": args.dcs},
        "cpu_baseline": {"value": round(gflops, 4), "unit": "GFLOP/s", "cores": workers, "kind": "reference",
                         "sample": sample, "cpu_model": model},
        "e2e": {"value": round(gflops, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "conversion_s": conv_s, "generation_s": gen_s,
        "eff_GBps": alg_bytes(A.nnz, A.num_rows, A.num_cols, 8) / med / 1e9,
    }
    print(json.dumps(out))


# ----------------------------------------------------------------- B200 arm
def time_spmv(m, x, y, steps, warmup, stream, spmv_fn, flush=None):
    """Per-step CUDA-event times (ms) of `steps` SpMVs on `stream`."""
    import torch

    for _ in range(warmup):
        spmv_fn(m, x, y, stream)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    with torch.cuda.stream(stream):
        for a, b in ev:
            if flush is not None:
                flush()
            a.record(stream)
            spmv_fn(m, x, y, stream)
            b.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1203_5737_b200 as argcsr
    from paper_1203_5737_b200 import synthetic

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = synthetic.CONFIGS[args.config]
    tdtype = torch.float64 if cfg["dtype"] == "float64" else torch.float32
    sv = 8 if tdtype == torch.float64 else 4

    # ---------------------------------------------------------- setup
    t = time.perf_counter()
    A = cfg["gen"](dev)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t
    nnz_total, rows_total, cols_total = A.nnz, A.num_rows, A.num_cols
    stream = torch.cuda.Stream(dev)
    ce0, ce1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    D = None
    with torch.cuda.stream(stream):
        ce0.record(stream)
        if world > 1 or args.power_iteration or os.environ.get("ARGCSR_BENCH_DIST") == "1":
            # nnz-balanced row slices, each rank converts its own (multigpu.py)
            from paper_1203_5737_b200.multigpu import DistributedArgCsr

            D = DistributedArgCsr(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values.to(tdtype),
                                  args.tpg, args.dcs, device=dev, dtype=tdtype, layout=args.layout,
                                  exchange=args.exchange)
            m = D.engine.m
            S = D.slice
        else:
            S = A
            m = argcsr.argcsr_from_torch(A.num_rows, A.num_cols, A.row_pointers.contiguous(), A.columns.contiguous(),
                                         A.values.to(tdtype).contiguous(), args.tpg, args.dcs, stream=stream,
                                         layout=args.layout, x_remap=args.x_remap)
        ce1.record(stream)
    torch.cuda.synchronize()
    conv_ms = ce0.elapsed_time(ce1)

    x = synthetic.bench_input(A.num_cols, dev, tdtype)
    xg = torch.empty_like(x) if D is not None else None
    y = torch.empty(m.num_rows, dtype=tdtype, device=dev)

    def spmv_fn(mm, xx, yy, s):
        mm.spmv_device(xx.data_ptr(), yy.data_ptr(), s.cuda_stream)

    ab = alg_bytes(nnz_total, rows_total, cols_total, sv)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_buf = None
    working_set = m.stored_slots * (sv + 4) + (m.num_rows + m.num_cols) * sv
    if working_set < 4 * l2:
        flush_buf = torch.empty(2 * l2 // 4 + 1024, dtype=torch.int32, device=dev)

    def flush():
        flush_buf.zero_()

    # --------------------------------------------------- timed region
    sampler = ClockSampler(local)
    sampler.start()
    pi_lambda = None
    if D is None:
        spmv_times = time_spmv(m, x, y, args.warmup, 0, stream, spmv_fn)  # warm-up pass
        sampler.mark_start()
        if flush_buf is None:
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                for _ in range(args.steps):
                    spmv_fn(m, x, y, stream)
                e1.record(stream)
            torch.cuda.synchronize()
            total_ms = e0.elapsed_time(e1)
            step_ms = total_ms / args.steps
        else:
            spmv_times = time_spmv(m, x, y, args.steps, 0, stream, spmv_fn, flush)
            total_ms = sum(spmv_times)
            step_ms = total_ms / args.steps
        sampler.mark_end()
        launches = args.steps * ((1 if m.heavy_ctas else 0) + (1 if m.light_tiles else 0) + (1 if m.x_remap else 0))
    else:
        bufs = [x, xg]
        it = [0]
        pscale = torch.ones(1, dtype=torch.float64, device=dev)
        ps2 = torch.zeros(1, dtype=torch.float64, device=dev)

        if D.pstep is not None:
            D.pstep.normalize = args.power_iteration  # else the iterated SpMV x <- A x
            D.pstep.begin(x)

        def step():
            # y = A_p x_i on this rank's rows, then the all-gather of y into
            # every rank's x_{i+1} (NCCL over NVLink), double-buffered x;
            # power iteration adds the 8-byte ||y||^2 all-reduce and the
            # scaling fused into the next SpMV's gathers.  p2p: the SpMV
            # stores y into every GPU's next x itself; flags + partial norms.
            if D.pstep is not None:
                D.pstep.step()
            elif args.power_iteration:
                D.step(bufs[it[0] % 2], bufs[(it[0] + 1) % 2], pscale, ps2)
            else:
                D.spmv_gather(bufs[it[0] % 2], bufs[(it[0] + 1) % 2], wait=False)
            it[0] += 1

        def drain():
            if D.pstep is not None:
                D.pstep.wait(D.pstep.k)
            else:
                D.wait_gather()

        for _ in range(args.warmup):
            step()
        drain()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        sampler.mark_start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        drain()  # the last all-gather (p2p: the last peers' flags) is part of the timed region
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        sampler.mark_end()
        total_ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total_ms = float(t.item())
        if D.pstep is not None:
            pi_lambda = D.pstep.finish()[0]
        elif args.power_iteration:
            pi_lambda = float(torch.sqrt(ps2).item())
        step_ms = total_ms / args.steps
        per_call = (1 if m.heavy_ctas else 0) + (1 if m.light_tiles else 0)
        if D.pstep is not None:  # one SpMV (+ x' gather), signal and wait kernels
            launches = args.steps * (per_call + (1 if m.x_remap else 0) + (2 if world > 1 else 0))
        elif D.overlap:  # interior + two boundary ranges; the last reuses the x' gather
            launches = args.steps * (3 * per_call + (2 if m.x_remap else 0))
        else:
            launches = args.steps * (per_call + (1 if m.x_remap else 0))
    sampler.stop()
    clocks = sampler.summary()

    gflops = 2.0 * nnz_total / (step_ms * 1e-3) / 1e9
    eff_gbs = ab / (step_ms * 1e-3) / 1e9
    e2e_dist = None
    if D is not None and not args.power_iteration and D.pstep is None:
        # e2e at N GPUs through the multi-GPU API: every step each rank uploads
        # its input x from pinned host memory, runs the SpMV + exchange
        # (spmv_gather) and downloads its y slice; max over ranks of the time.
        try:
            xh = torch.empty(A.num_cols, dtype=tdtype, pin_memory=True)
            xh.copy_(x.cpu())
            yh = torch.empty(D.r1 - D.r0, dtype=tdtype, pin_memory=True)
            xd, od = torch.empty_like(x), torch.empty_like(x)

            def e2e_step():
                xd.copy_(xh, non_blocking=True)
                D.spmv_gather(xd, od, wait=True)
                yh.copy_(od[D.r0:D.r1], non_blocking=True)

            for _ in range(3):
                e2e_step()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            k2 = max(10, min(args.steps, 50))
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record()
            for _ in range(k2):
                e2e_step()
            f1.record()
            torch.cuda.synchronize()
            t2 = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(t2, op=dist.ReduceOp.MAX)
            e2e_ms = float(t2.item()) / k2
            e2e_dist = {"value": round(2.0 * nnz_total / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                        "h2d_bytes_per_step": world * A.num_cols * sv, "d2h_bytes_per_step": A.num_rows * sv,
                        "ms_per_step": e2e_ms, "steps": k2,
                        "path": "per rank: pinned host x -> H2D, DistributedArgCsr.spmv_gather (SpMV + "
                                f"{D.exchange} exchange), D2H of the rank's y slice; max over ranks"}
        except Exception as exc:  # report, do not lose the bench line
            e2e_dist = {"value": None, "error": f"{type(exc).__name__}: {exc}"[:200]}
    if D is not None and D.peer is not None:
        D.close()  # collective over the ranks: nobody stores into freed peer buffers
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak, peak_src = measured_peak()
    info = {"layout": m.layout, "groups": m.num_groups, "total_slots": m.total_slots,
            "stored_slots": m.stored_slots, "x_remap": m.x_remap, "x_used_columns": m.x_used_columns, "unit_len_bytes": m.unit_len_bytes,
            "heavy_groups": m.heavy_groups,
            "light_tiles": m.light_tiles, "max_chunk": m.max_chunk_size, "device_bytes": m.device_bytes,
            "heavy_ctas": m.heavy_ctas, "l2_persist_bytes": m.l2_persist_bytes}
    key = f"{args.config}_tpg{args.tpg}_dcs{args.dcs}_{args.layout}"
    traffic = traffic_from_profiles(key)
    out = {
        "metric": "SpMV GFLOP/s", "value": round(gflops, 3), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if sv == 8 else "f32", "data": "synthetic",
        "config": {"workload": args.config, "matrix": A.name, "desc": cfg["desc"], "rows": rows_total,
                   "nnz": nnz_total, "threads_per_group": args.tpg, "desired_chunk_size": args.dcs,
                   "layout": args.layout,
                   "l2": ("flushed between steps (working set < 4x L2)" if flush_buf is not None else
                          f"inputs larger than L2 (ARG-CSR arrays {m.stored_slots * (sv + 4) / 1e9:.2f} GB); "
                          "x kept L2-resident by design (access-policy window)"),
                   "parallelism": ("single GPU" if world == 1 else
                                   f"rows nnz-balanced over {world} GPU(s), SpMV epilogue stores y into every "
                                   f"GPU's next x over NVLink (p2p), flag + partial-norm signals" if D.exchange == "p2p"
                                   else f"rows nnz-balanced over {world} GPU(s), {D.exchange} x exchange overlapped "
                                   f"with the interior groups")},
        "eff_GBps": round(eff_gbs, 1), "pct_of_8TBps": round(100 * eff_gbs / NOMINAL_HBM_GBS, 2),
        "pct_of_measured": round(100 * eff_gbs / peak, 2),
        "roofline": {"bound": "hbm", "achieved": round(eff_gbs, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(eff_gbs / peak, 4), "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes_per_launch": ab, "kernel": "spmv_kernel"},
        "conversion_ms": round(conv_ms, 3), "generation_s": round(gen_s, 3), "format": info,
        "clocks": clocks, "gpu_launches": launches,
    }
    if args.power_iteration:
        out["power_iteration"] = {"steps_total": args.warmup + args.steps, "lambda": pi_lambda,
                                  "step": ("SpMV with y stored into every GPU's next x by its epilogue + ||y||^2 "
                                           "partials and step flags over peer memory + scaling fused into the next SpMV"
                                           if D.exchange == "p2p" else
                                           "SpMV + ||y||^2 all-reduce + all-gather of y + scaling fused into the next SpMV")}

    if e2e_dist is not None:
        out["e2e"] = e2e_dist
        out["gpu_launches"] = launches
    elif world == 1 and not args.power_iteration:
        # ------------------------------------------------ e2e through the C-ABI with host buffers
        xh = torch.empty(A.num_cols, dtype=tdtype, pin_memory=True)
        xh.copy_(x.cpu())
        yh = torch.empty(A.num_rows, dtype=tdtype, pin_memory=True)
        xd = torch.empty_like(x)
        yd = torch.empty_like(y)
        for _ in range(3):
            m.spmv_host_staged(xh.data_ptr(), xd.data_ptr(), yd.data_ptr(), yh.data_ptr(), stream.cuda_stream)
        e2e_steps = max(10, min(args.steps, 100))
        t = time.perf_counter()
        for _ in range(e2e_steps):
            m.spmv_host_staged(xh.data_ptr(), xd.data_ptr(), yd.data_ptr(), yh.data_ptr(), stream.cuda_stream)
        sync_s = (time.perf_counter() - t) / e2e_steps
        # A stream of SpMVs from host memory through the non-blocking C-ABI call:
        # every step uploads its x and downloads its y (two alternating pinned
        # y buffers); step i+1's upload overlaps step i's SpMV and step i-1's
        # download (the handle double-buffers its device staging).
        yh2 = [yh, torch.empty_like(yh, pin_memory=True)]
        for i in range(3):
            m.spmv_host_async(xh.data_ptr(), yh2[i % 2].data_ptr(), stream.cuda_stream)
        m.host_wait()
        t = time.perf_counter()
        for i in range(e2e_steps):
            m.spmv_host_async(xh.data_ptr(), yh2[i % 2].data_ptr(), stream.cuda_stream)
        m.host_wait()
        e2e_s = (time.perf_counter() - t) / e2e_steps
        out["e2e"] = {"value": round(2.0 * nnz_total / e2e_s / 1e9, 3), "unit": "GFLOP/s",
                      "h2d_bytes_per_step": A.num_cols * sv, "d2h_bytes_per_step": A.num_rows * sv,
                      "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
                      "path": "argcsr_dev_spmv_host_async per step (pinned host x -> H2D on copy engine 1 -> SpMV "
                              "-> D2H into alternating pinned y buffers on copy engine 2), argcsr_dev_host_wait "
                              "after the last step; consecutive steps overlap",
                      "single_call": {"value": round(2.0 * nnz_total / sync_s / 1e9, 3), "ms_per_step": sync_s * 1e3,
                                      "path": "argcsr_dev_spmv_host_staged, synchronous per call: x up in 8 "
                                              "pieces, light-tile chunks launched as their x window lands, y "
                                              "chunks down meanwhile; one-shot with heavy groups or the x remap"}}
        out["gpu_launches"] = launches

        if not args.no_variants:
            out["variants"] = variants(args, A, x, tdtype, sv, stream, spmv_fn, m.x_remap)

        if not args.no_cpu_baseline and cfg["dtype"] == "float64":
            out["cpu_baseline"] = cpu_baseline(args, m, A, x, y, stream)
    print(json.dumps(out))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def variants(args, A, x, tdtype, sv, stream, spmv_fn, x_remap=False):
    """Side runs on the same matrix: the tuned chunk budget and the cuSPARSE
    CSR yardstick (torch.sparse CSR matvec -> cusparseSpMV)."""
    import torch

    import paper_1203_5737_b200 as argcsr

    res = []
    ab = alg_bytes(A.nnz, A.num_rows, A.num_cols, sv)
    y = torch.empty(A.num_rows, dtype=tdtype, device=x.device)
    other = "reference" if args.layout == "compact" else "compact"
    runs = [(args.dcs, other, "auto")] + [(d, args.layout, "auto") for d in sorted({32, 4} - {args.dcs})]
    if x_remap:
        runs.append((args.dcs, args.layout, "off"))
    for dcs, layout, xr in runs:
        m2 = argcsr.argcsr_from_torch(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values.to(tdtype),
                                      args.tpg, dcs, stream=stream, layout=layout, x_remap=xr)
        ts = time_spmv(m2, x, y, min(args.steps, 100), args.warmup, stream, spmv_fn)
        ms = statistics.median(ts)
        res.append({"impl": "argcsr_b200", "threads_per_group": args.tpg, "desired_chunk_size": dcs,
                    "layout": layout, "x_remap": m2.x_remap, "ms": ms, "gflops": 2 * A.nnz / ms / 1e6, "eff_GBps": ab / ms / 1e6,
                    "total_slots": m2.total_slots, "stored_slots": m2.stored_slots, "groups": m2.num_groups})
        m2.free()
        del m2
    # the paper's comparison formats on the device (csrc/ellpack.cu)
    for name, slice_size in (("sliced_ellpack_32", 32), ("ellpack", 0)):
        try:
            E = argcsr._ext.sell_from_device_csr(
                A.num_rows, A.num_cols, A.nnz, A.row_pointers.data_ptr(), A.columns.data_ptr(),
                A.values.to(tdtype).contiguous().data_ptr(), "float64" if sv == 8 else "float32", slice_size,
                x.device.index, stream.cuda_stream)

            def ell(_m, xx, yy, st, E=E):
                E.spmv_device(xx.data_ptr(), yy.data_ptr(), st.cuda_stream)

            ts = time_spmv(None, x, y, min(args.steps, 50), args.warmup, stream, ell)
            ms = statistics.median(ts)
            res.append({"impl": name, "ms": ms, "gflops": 2 * A.nnz / ms / 1e6, "eff_GBps": ab / ms / 1e6,
                        "total_slots": E.total_slots})
            del E
        except Exception as e:  # ELLPACK pads every row to the widest: power-law rows do not fit
            res.append({"impl": name, "error": str(e)[:160]})
        torch.cuda.empty_cache()
    try:
        csr = torch.sparse_csr_tensor(A.row_pointers, A.columns.to(torch.int64), A.values.to(tdtype),
                                      size=(A.num_rows, A.num_cols))

        def cus(_m, xx, yy, s):
            torch.mv(csr, xx)

        with torch.cuda.stream(stream):
            ts = time_spmv(None, x, y, min(args.steps, 50), args.warmup, stream, cus)
        ms = statistics.median(ts)
        res.append({"impl": "cusparse_csr (torch.mv on a sparse CSR tensor -> cusparseSpMV)", "ms": ms,
                    "gflops": 2 * A.nnz / ms / 1e6, "eff_GBps": ab / ms / 1e6})
        del csr
    except Exception as e:  # the yardstick is informational
        res.append({"impl": "cusparse_csr", "error": str(e)[:200]})
    torch.cuda.empty_cache()
    return res


def cpu_baseline(args, m, A, x, y, stream):
    """The reference CPU path (oracle/_ref spmv_argcsr_parallel, all host
    threads) on the bit-identical ARG-CSR arrays exported from the device,
    bounded sample; also the parity check of the timed GPU result."""
    import numpy as np
    import torch

    try:
        import oracle
    except Exception as e:
        return {"value": None, "error": f"oracle unavailable: {e}"}
    if not oracle.ref_available():
        return {"value": None, "error": "oracle/_ref not built"}
    ref = oracle.ref()
    g4 = m.groups_array.copy()
    M = oracle.ArgCsr(m.num_rows, m.num_cols, m.threads_per_group, g4, np.asarray(m.threads_mapping),
                      np.asarray(m.values), np.asarray(m.columns))
    h = ref.import_argcsr(M)
    del M
    workers = os.cpu_count()
    xh = x.double().cpu().numpy()
    times, y_ref = ref.time_spmv_argcsr_parallel(h, xh, workers, 2, args.cpu_sample_steps, A.num_rows)
    ref.free_argcsr(h)
    with torch.cuda.stream(stream):
        m.spmv_device(x.data_ptr(), y.data_ptr(), stream.cuda_stream)
    torch.cuda.synchronize()
    y_gpu = y.double().cpu().numpy()
    med = float(np.median(times))
    cores, model = cpu_info()
    return {"value": round(2.0 * A.nnz / med / 1e9, 4), "unit": "GFLOP/s", "cores": workers, "kind": "reference",
            "sample": f"{args.cpu_sample_steps} x spmv_argcsr_parallel (oracle/_ref, {workers} threads) over the "
                      f"full matrix, median; matrix = the device export (bit-identical to argcsr_from_csr)",
            "ms_per_step": med * 1e3, "cpu_model": model,
            "parity": "bit-exact" if y_gpu.tobytes() == y_ref.tobytes() else
            f"max|dy|={float(np.max(np.abs(y_gpu - y_ref))):.3e}"}


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
