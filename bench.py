#!/usr/bin/env python
"""ARG-CSR SpMV benchmark (BASELINE.json metric: SpMV GFLOP/s and effective HBM
GB/s (% of 8 TB/s) at 1/2/4/8 B200 vs the CPU reference).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--tpg 128] [--dcs 1]
  python bench.py --impl reference ...      # the reference CPU path (oracle/_ref)

A "step" is one ARG-CSR SpMV y = A x over the whole synthetic matrix of the
config with x, y and the matrix resident in HBM (N = 1).  At N > 1 the rows
are nnz-balanced across ranks, each rank converts its own slice, and a step
is the local SpMV plus the exchange of y into every rank's next x (the
iterated-SpMV step of config C5); value = 2 * nnz(total) / max-over-ranks
step time (strong scaling).  `--power-iteration` times the C5 step
(SpMV + fused ||y||^2 + all-reduce + exchange + fused scaling).

Rank 0 prints ONE JSON line.  Algorithmic bytes per SpMV:
alg_bytes = nnz*(S_v + 4) + (rows + cols)*S_v, S_v = 8 (fp64) / 4 (fp32);
flops = 2*nnz.

Parity gate (like run_benchmark's CorrectnessError, proj/src/bench.cpp:
220-226): at N = 1 the default run converts the SAME CSR with the compiled
reference (oracle/_ref argcsr_from_csr), compares groups / threads_mapping /
values / columns byte for byte with the device export, and compares the timed
SpMV's y with the reference spmv_argcsr_parallel bit for bit; any mismatch
prints the line and exits with status 3.

Both arms build their matrix with workloads.py (device-independent hash RNG),
so they time the same input; config.input_sha256 proves it.  The reference
arm never imports the product package (no native library of the B200 path is
mapped in that process).
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
PARITY_FAIL_RC = 3


def parse_args(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=None, help="timed steps (default 200; 100 with --power-iteration)")
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--config", default=None, choices=["C1", "C2", "C3", "C4", "C4f32", "C5"],
                   help="workload (default C2; C5 with --power-iteration)")
    p.add_argument("--tpg", type=int, default=128)
    p.add_argument("--dcs", type=int, default=1)
    p.add_argument("--layout", default="compact", choices=["compact", "reference"],
                   help="device storage of the value/column blocks (include/argcsr_gpu.h ARGCSR_LAYOUT_REFERENCE)")
    p.add_argument("--x-remap", default="auto", choices=["auto", "on", "off"],
                   help="device column order (single-GPU path): library decision, or forced")
    p.add_argument("--no-variants", action="store_true", help="skip the tuned-dcs / ELL / cuSPARSE side runs")
    p.add_argument("--no-configs", action="store_true", help="skip the C1/C3/C4/C4f32 block of the default run")
    p.add_argument("--no-cpu-baseline", action="store_true", help="skip the reference CPU leg (and the parity gate)")
    p.add_argument("--cpu-sample-steps", type=int, default=20)
    p.add_argument("--exchange", default="auto", choices=["auto", "allgather", "halo", "p2p"],
                   help="multi-GPU x exchange: NCCL all-gather / halo send-recv (auto picks), or p2p: "
                        "the SpMV epilogue stores y straight into the peers' x over NVLink")
    p.add_argument("--power-iteration", action="store_true",
                   help="a step is one power-iteration step (SpMV + fused ||y||^2, all-reduce, exchange, "
                        "scaling fused into the next SpMV)")
    a = p.parse_args(argv)
    if a.config is None:
        a.config = "C5" if a.power_iteration else "C2"
    if a.steps is None:
        a.steps = 100 if a.power_iteration else 200
    return a


# ------------------------------------------------------------------ helpers
def measured_peak():
    f = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


READ_CEILING_GBS = 7320.0  # contiguous-read stream probe on this B200 pool (profiles/r01_stream_probe.txt)


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


def make_config(args, A, world: int, cfg: dict) -> dict:
    """The `config` object -- identical in both arms for the same command."""
    sv = 8 if cfg["dtype"] == "float64" else 4
    ws = A.nnz * (sv + 4) + (A.num_rows + A.num_cols) * sv
    return {
        "workload": args.config, "matrix": A.name, "desc": cfg["desc"], "rows": A.num_rows, "cols": A.num_cols,
        "nnz": A.nnz, "threads_per_group": args.tpg, "desired_chunk_size": args.dcs,
        "input_sha256": A.digest(),
        "l2": ("inputs larger than L2 (CSR arrays %.2f GB > 126 MB); x kept L2-resident by design" % (ws / 1e9)
               if ws > 4 * 126e6 else "L2 flushed between timed steps (working set < 4x L2)"),
        "parallelism": ("single GPU" if world == 1 else f"rows nnz-balanced over {world} GPUs"),
        "step": "power-iteration step" if args.power_iteration else "one SpMV y = A x",
    }


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


def ref_csr(A):
    """The workload's CSR as the oracle's numpy view (host)."""
    import numpy as np

    import oracle

    return oracle.Csr(A.num_rows, A.num_cols, A.row_pointers.cpu().numpy().view(np.uint64), A.columns.cpu().numpy(),
                      A.values.cpu().numpy().astype(np.float64))


# ----------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's own CPU path: argcsr_from_csr + spmv_argcsr_parallel
    (proj/src/argcsr.cpp:123-155, bench.cpp:109-116) from oracle/_ref, with
    all host threads, timed like run_benchmark's timed_median
    (bench.cpp:128-141: warm-up, then the median of individually timed
    runs), and checked like it (relative error vs spmv_csr <= 1e-10,
    bench.cpp:151, 220-226)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    import workloads

    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libargcsr_ref.so not built"}))
        return 0
    cfg = workloads.CONFIGS[args.config]
    if cfg["dtype"] != "float64":
        print(json.dumps({"impl": "reference", "unavailable": "the reference library is fp64-only (SPEC.md:82)"}))
        return 0
    ref = oracle.ref()
    t = time.perf_counter()
    A = cfg["gen"]("cpu")
    config = make_config(args, A, args.gpus, cfg)
    slice_note = ""
    if args.config == "C5":
        # bounded sample: the reference would need ~50 GB of host memory for all
        # 879 M nnz at (128, 1); time one GPU's share at 8 GPUs (rows [0, N/8))
        A = A.slice_rows(0, A.num_rows // 8)
        slice_note = f"; rows [0, {A.num_rows}) = one GPU's share of C5 at 8 GPUs (bounded host memory)"
    csr = oracle.Csr(A.num_rows, A.num_cols, A.row_pointers.numpy().view(np.uint64), A.columns.numpy(),
                     A.values.numpy())
    gen_s = time.perf_counter() - t
    t = time.perf_counter()
    h = ref.argcsr_handle(csr, args.tpg, args.dcs)
    conv_s = time.perf_counter() - t
    workers = os.cpu_count()
    x = oracle.bench_input(A.num_cols)
    steps = args.steps
    if args.power_iteration:
        steps = max(args.steps, 1)
    times, y = ref.time_spmv_argcsr_parallel(h, x, workers, args.warmup, steps, A.num_rows)
    ref.free_argcsr(h)
    y_csr = ref.spmv_csr(csr, x)
    rel = float(np.max(np.abs(y - y_csr)) / max(float(np.max(np.abs(y_csr))), 1.0)) if y.size else 0.0
    med = float(np.median(times))
    gflops = 2.0 * A.nnz / med / 1e9
    cores, model = cpu_info()
    sample = (f"{steps} x spmv_argcsr_parallel over the full {args.config} matrix "
              f"(tpg={args.tpg}, dcs={args.dcs}) after {args.warmup} warm-up, median of individually timed runs; "
              f"workers={workers}{slice_note}")
    out = {
        "impl": "reference", "metric": "SpMV GFLOP/s", "value": round(gflops, 4), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup, "ms_per_step": med * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (workloads.py, hash RNG: the same matrix as the B200 arm)", "config": config,
        "cpu_baseline": {"value": round(gflops, 4), "unit": "GFLOP/s", "cores": workers, "kind": "reference",
                         "sample": sample, "cpu_model": model},
        "e2e": {"value": round(gflops, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "conversion_s": conv_s, "generation_s": gen_s,
        "eff_GBps": alg_bytes(A.nnz, A.num_rows, A.num_cols, 8) / med / 1e9,
        "check": {"relative_error_vs_spmv_csr": rel, "tolerance": 1e-10, "ok": rel <= 1e-10},
    }
    print(json.dumps(out))
    return 0 if rel <= 1e-10 else PARITY_FAIL_RC


# ----------------------------------------------------------------- B200 arm
def time_steps(fn, steps: int, stream, flush=None):
    """Per-step CUDA-event times (ms) of `steps` calls of fn() on `stream`
    (events recorded on that stream), plus the time of the whole bracket."""
    import torch

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    fl = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)] \
        if flush is not None else None
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for i in range(steps):
            if flush is not None:
                flush()
                fl[i][0].record(stream)
            else:
                ev[i].record(stream)
            fn()
            if flush is not None:
                fl[i][1].record(stream)
        ev[steps].record(stream)
    torch.cuda.synchronize()
    if flush is not None:
        per = [a.elapsed_time(b) for a, b in fl]
        return per, sum(per)
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    return per, ev[0].elapsed_time(ev[steps])


def l2_flusher(dev):
    import torch

    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    buf = torch.empty(2 * l2 // 4 + 1024, dtype=torch.int32, device=dev)
    return lambda: buf.zero_()


def launches_per_spmv(m) -> int:
    return (1 if m.heavy_ctas else 0) + (1 if m.light_tiles else 0) + (1 if m.x_remap else 0)


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1203_5737_b200 as argcsr
    import workloads

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = workloads.CONFIGS[args.config]
    tdtype = torch.float64 if cfg["dtype"] == "float64" else torch.float32
    sv = 8 if tdtype == torch.float64 else 4

    # ---------------------------------------------------------- setup
    t = time.perf_counter()
    A = cfg["gen"](dev)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t
    config = make_config(args, A, world, cfg)
    nnz_total, rows_total, cols_total = A.nnz, A.num_rows, A.num_cols
    stream = torch.cuda.Stream(dev)
    D = None
    distributed_path = world > 1 or args.power_iteration or os.environ.get("ARGCSR_BENCH_DIST") == "1"
    # one small conversion + SpMV first, so that lazy kernel-module loading and
    # first-call setup are not charged to the conversion time below
    _w = workloads.stencil3d27(12, dev)
    _wm = argcsr.argcsr_from_torch(_w.num_rows, _w.num_cols, _w.row_pointers, _w.columns, _w.values.to(tdtype),
                                   args.tpg, args.dcs, stream=stream, layout=args.layout, x_remap=args.x_remap)
    _wy = torch.empty(_w.num_rows, dtype=tdtype, device=dev)
    _wm.spmv_device(workloads.bench_input(_w.num_cols, dev, tdtype).data_ptr(), _wy.data_ptr(), stream.cuda_stream)
    torch.cuda.synchronize()
    _wm.free()
    del _w, _wm, _wy
    t_conv = time.perf_counter()
    with torch.cuda.stream(stream):
        if distributed_path:
            # nnz-balanced row slices, each rank converts its own (multigpu.py over the C-ABI)
            from paper_1203_5737_b200.multigpu import DistributedArgCsr

            D = DistributedArgCsr(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values.to(tdtype),
                                  args.tpg, args.dcs, device=dev, dtype=tdtype, layout=args.layout,
                                  exchange=args.exchange)
            m = D.local_matrix
        else:
            m = argcsr.argcsr_from_torch(A.num_rows, A.num_cols, A.row_pointers.contiguous(), A.columns.contiguous(),
                                         A.values.to(tdtype).contiguous(), args.tpg, args.dcs, stream=stream,
                                         layout=args.layout, x_remap=args.x_remap)
    torch.cuda.synchronize()
    conv_ms = 1e3 * (time.perf_counter() - t_conv)  # host wall clock: conversion synchronises
    conv_repeat_ms = None
    if not distributed_path:
        # the same conversion again: the first one also pays the driver's first
        # mapping of ~1.4 GB of fresh device memory
        t_conv = time.perf_counter()
        with torch.cuda.stream(stream):
            argcsr.argcsr_from_torch(A.num_rows, A.num_cols, A.row_pointers.contiguous(), A.columns.contiguous(),
                                     A.values.to(tdtype).contiguous(), args.tpg, args.dcs, stream=stream,
                                     layout=args.layout, x_remap=args.x_remap).free()
        torch.cuda.synchronize()
        conv_repeat_ms = round(1e3 * (time.perf_counter() - t_conv), 3)

    x = workloads.bench_input(A.num_cols, dev, tdtype)
    y = torch.empty(m.num_rows, dtype=tdtype, device=dev)
    ab = alg_bytes(nnz_total, rows_total, cols_total, sv)
    working_set = A.nnz * (sv + 4) + (A.num_rows + A.num_cols) * sv
    flush = l2_flusher(dev) if working_set < 4 * 126e6 else None

    # --------------------------------------------------- timed region
    sampler = ClockSampler(local)
    sampler.start()
    pi_lambda = None
    timing = {}
    if D is None:
        def one():
            m.spmv_device(x.data_ptr(), y.data_ptr(), stream.cuda_stream)

        time_steps(one, args.warmup, stream)  # warm-up
        sampler.mark_start()
        per, total_ms = time_steps(one, args.steps, stream, flush)
        sampler.mark_end()
        step_ms = total_ms / args.steps
        timing = {"mean_ms": step_ms, "median_ms": statistics.median(per), "min_ms": min(per),
                  "per_step_events": "CUDA events on the launching stream around every step",
                  "l2_flushed": flush is not None}
        launches = args.steps * launches_per_spmv(m)
    else:
        D.begin(x, normalize=args.power_iteration)
        for _ in range(args.warmup):
            D.step()
        D.drain()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        sampler.mark_start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            D.step()
        D.drain()  # the last exchange is part of the timed region
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        sampler.mark_end()
        total_ms = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            total_ms = float(tt.item())
        lam, _ = D.finish()
        pi_lambda = lam if args.power_iteration else None
        step_ms = total_ms / args.steps
        timing = {"mean_ms": step_ms, "max_over_ranks": True}
        launches = args.steps * D.launches_per_step()
    sampler.stop()
    clocks = sampler.summary()

    gflops = 2.0 * nnz_total / (step_ms * 1e-3) / 1e9
    eff_gbs = ab / (step_ms * 1e-3) / 1e9
    e2e_dist = None
    if D is not None and not args.power_iteration:
        e2e_dist = e2e_distributed(D, A, x, tdtype, sv, world, dev, args)
    if D is not None:
        D.close()  # collective over the ranks
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    peak, peak_src = measured_peak()
    info = {"layout": m.layout, "groups": m.num_groups, "total_slots": m.total_slots,
            "stored_slots": m.stored_slots, "x_remap": m.x_remap, "x_used_columns": m.x_used_columns,
            "unit_len_bytes": m.unit_len_bytes, "heavy_groups": m.heavy_groups, "light_tiles": m.light_tiles,
            "max_chunk": m.max_chunk_size, "device_bytes": m.device_bytes, "heavy_ctas": m.heavy_ctas,
            "l2_persist_bytes": m.l2_persist_bytes}
    key = f"{args.config}_tpg{args.tpg}_dcs{args.dcs}_{args.layout}"
    out = {
        "metric": "SpMV GFLOP/s", "value": round(gflops, 3), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if sv == 8 else "f32",
        "data": "synthetic (workloads.py, hash RNG: the same matrix as the reference arm)", "config": config,
        "timing": timing,
        "eff_GBps": round(eff_gbs, 1), "pct_of_8TBps": round(100 * eff_gbs / NOMINAL_HBM_GBS, 2),
        "pct_of_measured": round(100 * eff_gbs / peak, 2),
        "frac_of_read_ceiling": round(eff_gbs / READ_CEILING_GBS, 4),
        "roofline": {"bound": "hbm", "achieved": round(eff_gbs, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(eff_gbs / peak, 4), "traffic": traffic_from_profiles(key),
                     "peak_source": peak_src, "alg_bytes_per_launch": ab,
                     "kernel": "spmv_light_kernel (+ spmv_heavy_kernel when heavy groups exist), one SpMV",
                     "read_ceiling_GBps": READ_CEILING_GBS},
        "conversion_ms": round(conv_ms, 3), "conversion_repeat_ms": conv_repeat_ms,
        "conversion_note": ("per-GPU slice conversions plus the multi-GPU handle setup (NCCL communicator, halo plan)"
                            if distributed_path else "host wall clock around argcsr_from_torch after a warm-up "
                            "conversion; conversion_repeat_ms = the same conversion again"),
        "generation_s": round(gen_s, 3), "format": info,
        "clocks": clocks, "gpu_launches": launches,
        "layout": args.layout,
    }
    if args.power_iteration:
        out["power_iteration"] = {"steps_total": args.warmup + args.steps, "lambda": pi_lambda,
                                  "exchange": D.exchange, "step": D.step_description()}
    rc = 0
    if args.power_iteration and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_c5_share(args, A)
    if e2e_dist is not None:
        out["e2e"] = e2e_dist
    elif world == 1 and D is None:
        out["e2e"] = e2e_single(m, A, x, y, tdtype, sv, stream, args)
        if not args.no_variants:
            out["variants"] = variants(args, A, x, tdtype, sv, stream, m.x_remap)
        if not args.no_cpu_baseline and cfg["dtype"] == "float64":
            out["cpu_baseline"], ok = cpu_baseline_and_parity(args, m, A, x, y, stream)
            out["parity"] = out["cpu_baseline"].pop("parity")
            if not ok:
                rc = PARITY_FAIL_RC
        if not args.no_configs and args.config == "C2":
            del m
            torch.cuda.empty_cache()
            out["configs"] = other_configs(args, dev, stream, peak)
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return rc


def e2e_single(m, A, x, y, tdtype, sv, stream, args):
    """The same metric end to end through the C-ABI with host buffers."""
    import torch

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
    # every step uploads its x and downloads its y (two alternating pinned y
    # buffers); step i+1's upload overlaps step i's SpMV and step i-1's
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
    return {"value": round(2.0 * A.nnz / e2e_s / 1e9, 3), "unit": "GFLOP/s",
            "h2d_bytes_per_step": A.num_cols * sv, "d2h_bytes_per_step": A.num_rows * sv,
            "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
            "path": "argcsr_dev_spmv_host_async per step (pinned host x -> H2D on copy engine 1 -> SpMV "
                    "-> D2H into alternating pinned y buffers on copy engine 2), argcsr_dev_host_wait "
                    "after the last step; consecutive steps overlap",
            "single_call": {"value": round(2.0 * A.nnz / sync_s / 1e9, 3), "ms_per_step": sync_s * 1e3,
                            "path": "argcsr_dev_spmv_host_staged, synchronous per call: x up in 8 "
                                    "pieces, light-tile chunks launched as their x window lands, y "
                                    "chunks down meanwhile; one-shot with heavy groups or the x remap"}}


def e2e_distributed(D, A, x, tdtype, sv, world, dev, args):
    """e2e at N GPUs through the multi-GPU API: every step each rank uploads
    its input x from pinned host memory, runs the SpMV + exchange and
    downloads its y slice; max over ranks of the time."""
    import torch
    import torch.distributed as dist

    try:
        xh = torch.empty(A.num_cols, dtype=tdtype, pin_memory=True)
        xh.copy_(x.cpu())
        yh = torch.empty(D.r1 - D.r0, dtype=tdtype, pin_memory=True)
        xd, od = torch.empty_like(x), torch.empty_like(x)

        def e2e_step():
            xd.copy_(xh, non_blocking=True)
            D.spmv_gather(xd, od)
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
        return {"value": round(2.0 * A.nnz / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                "h2d_bytes_per_step": world * A.num_cols * sv, "d2h_bytes_per_step": A.num_rows * sv,
                "ms_per_step": e2e_ms, "steps": k2,
                "path": "per rank: pinned host x -> H2D, argcsr_mgpu_spmv_gather (SpMV + "
                        f"{D.exchange} exchange), D2H of the rank's y slice; max over ranks"}
    except Exception as exc:  # report, do not lose the bench line
        return {"value": None, "error": f"{type(exc).__name__}: {exc}"[:200]}


def cusparse_yardstick(A, x, tdtype, stream, steps: int, warmup: int):
    """cusparseSpMV (CSR, ALG1 and ALG2) called directly on the same CSR and x
    (yardstick/libcusparse_yardstick.so, a bench-only helper); median of
    CUDA-event-timed runs."""
    import ctypes as C

    import torch

    lib_path = ROOT / "yardstick" / "libcusparse_yardstick.so"
    if not lib_path.exists():
        return [{"impl": "cusparse", "error": "yardstick/libcusparse_yardstick.so not built"}]
    lib = C.CDLL(str(lib_path))
    lib.ys_spmv_csr_median_ms.restype = C.c_int
    lib.ys_spmv_csr_median_ms.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                          C.POINTER(C.c_double), C.c_char_p, C.c_int]
    if A.nnz >= 2 ** 31:
        return [{"impl": "cusparse", "error": "nnz >= 2^31: no 32-bit CSR for cuSPARSE"}]
    y = torch.empty(A.num_rows, dtype=tdtype, device=x.device)
    vals = A.values.to(tdtype).contiguous()
    rp32 = A.row_pointers.to(torch.int32)
    out = []
    for alg in (1, 2):
        ms = C.c_double(0)
        err = C.create_string_buffer(256)
        rc = lib.ys_spmv_csr_median_ms(A.num_rows, A.num_cols, A.nnz, rp32.data_ptr(),
                                       A.columns.data_ptr(), vals.data_ptr(), 1 if tdtype == torch.float64 else 0,
                                       x.data_ptr(), y.data_ptr(), alg, warmup, steps, C.c_void_p(stream.cuda_stream),
                                       C.byref(ms), err, 256)
        if rc != 0:
            out.append({"impl": f"cusparse_csr_alg{alg}", "error": err.value.decode()[:200]})
        else:
            out.append({"impl": f"cusparse_csr_alg{alg}", "ms": ms.value})
    del vals, rp32
    return out


def variants(args, A, x, tdtype, sv, stream, x_remap=False):
    """Side runs on the same matrix: the other layout, the tuned chunk
    budget, ELLPACK / SELL, and the cuSPARSE CSR yardstick (ALG1, ALG2)."""
    import torch

    import paper_1203_5737_b200 as argcsr

    res = []
    ab = alg_bytes(A.nnz, A.num_rows, A.num_cols, sv)
    y = torch.empty(A.num_rows, dtype=tdtype, device=x.device)
    other = "reference" if args.layout == "compact" else "compact"
    runs = [(args.dcs, other, "auto")] + [(d, args.layout, "auto") for d in sorted({32, 4} - {args.dcs})]
    if x_remap:
        runs.append((args.dcs, args.layout, "off"))
    nsteps = min(args.steps, 50)
    for dcs, layout, xr in runs:
        m2 = argcsr.argcsr_from_torch(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values.to(tdtype),
                                      args.tpg, dcs, stream=stream, layout=layout, x_remap=xr)
        fn = lambda: m2.spmv_device(x.data_ptr(), y.data_ptr(), stream.cuda_stream)  # noqa: E731
        time_steps(fn, args.warmup, stream)
        per, _ = time_steps(fn, nsteps, stream)
        ms = statistics.median(per)
        res.append({"impl": "argcsr_b200", "threads_per_group": args.tpg, "desired_chunk_size": dcs,
                    "layout": layout, "x_remap": m2.x_remap, "ms": ms, "gflops": 2 * A.nnz / ms / 1e6,
                    "eff_GBps": ab / ms / 1e6, "total_slots": m2.total_slots, "stored_slots": m2.stored_slots,
                    "groups": m2.num_groups})
        m2.free()
        del m2
    # the paper's comparison formats on the device (csrc/ellpack.cu)
    for name, slice_size in (("sliced_ellpack_32", 32), ("ellpack", 0)):
        try:
            E = argcsr._ext.sell_from_device_csr(
                A.num_rows, A.num_cols, A.nnz, A.row_pointers.data_ptr(), A.columns.data_ptr(),
                A.values.to(tdtype).contiguous().data_ptr(), "float64" if sv == 8 else "float32", slice_size,
                x.device.index, stream.cuda_stream)
            fn = lambda E=E: E.spmv_device(x.data_ptr(), y.data_ptr(), stream.cuda_stream)  # noqa: E731
            time_steps(fn, args.warmup, stream)
            per, _ = time_steps(fn, min(nsteps, 20), stream)
            ms = statistics.median(per)
            res.append({"impl": name, "ms": ms, "gflops": 2 * A.nnz / ms / 1e6, "eff_GBps": ab / ms / 1e6,
                        "total_slots": E.total_slots})
            del E
        except Exception as e:  # ELLPACK pads every row to the widest: power-law rows do not fit
            res.append({"impl": name, "error": str(e)[:160]})
        torch.cuda.empty_cache()
    for r in cusparse_yardstick(A, x, tdtype, stream, nsteps, args.warmup):
        if "ms" in r:
            r.update(gflops=2 * A.nnz / r["ms"] / 1e6, eff_GBps=ab / r["ms"] / 1e6)
        res.append(r)
    torch.cuda.empty_cache()
    return res


def cpu_baseline_c5_share(args, A):
    """CPU baseline of the power-iteration config, bounded: the reference's
    spmv_argcsr_parallel (oracle/_ref, all host threads) on one GPU's share of
    the rows at 8 GPUs (rows [0, N/8)), the unit each GPU converts and
    multiplies in the row-partitioned step; same metric (GFLOP/s)."""
    import numpy as np

    try:
        import oracle
    except Exception as e:
        return {"value": None, "error": f"oracle unavailable: {e}"}
    if not oracle.ref_available():
        return {"value": None, "error": "oracle/_ref not built"}
    ref = oracle.ref()
    S = A.slice_rows(0, A.num_rows // 8)
    csr = ref_csr(S)
    h = ref.argcsr_handle(csr, args.tpg, args.dcs)
    workers = os.cpu_count()
    xh = oracle.bench_input(S.num_cols)
    times, _ = ref.time_spmv_argcsr_parallel(h, xh, workers, 2, args.cpu_sample_steps, S.num_rows)
    ref.free_argcsr(h)
    med = float(np.median(times))
    _, model = cpu_info()
    return {"value": round(2.0 * S.nnz / med / 1e9, 4), "unit": "GFLOP/s", "cores": workers, "kind": "reference",
            "sample": f"{args.cpu_sample_steps} x spmv_argcsr_parallel (oracle/_ref, {workers} threads) on rows "
                      f"[0, {S.num_rows}) of {args.config} ({S.nnz} nnz: one GPU's share at 8 GPUs; the full matrix "
                      f"would need ~50 GB of host memory in the reference layout), after 2 warm-up, median",
            "ms_per_step": med * 1e3, "cpu_model": model}


def cpu_baseline_and_parity(args, m, A, x, y, stream):
    """The reference CPU path on the box's host cores: oracle/_ref
    argcsr_from_csr of the SAME CSR (timed as the reference conversion), then
    spmv_argcsr_parallel on all host threads (bounded sample, median).  Also
    the parity gate: the device export must equal the reference conversion
    byte for byte, and the timed y the reference product bit for bit."""
    import numpy as np
    import torch

    try:
        import oracle
    except Exception as e:
        return {"value": None, "error": f"oracle unavailable: {e}", "parity": {"checked": False}}, True
    if not oracle.ref_available():
        return {"value": None, "error": "oracle/_ref not built", "parity": {"checked": False}}, True
    ref = oracle.ref()
    csr = ref_csr(A)
    t = time.perf_counter()
    h = ref.argcsr_handle(csr, args.tpg, args.dcs)
    ref_conv_s = time.perf_counter() - t
    R = ref.export(h)
    conv = {"groups": np.array_equal(m.groups_array, R.groups),
            "threads_mapping": np.array_equal(np.asarray(m.threads_mapping), R.threads_mapping)}
    dv = np.asarray(m.values)
    conv["values"] = dv.tobytes() == R.values.tobytes()
    del dv
    dc = np.asarray(m.columns)
    conv["columns"] = np.array_equal(dc, R.columns)
    del dc, R
    workers = os.cpu_count()
    xh = x.double().cpu().numpy()
    times, y_ref = ref.time_spmv_argcsr_parallel(h, xh, workers, 2, args.cpu_sample_steps, A.num_rows)
    ref.free_argcsr(h)
    with torch.cuda.stream(stream):
        m.spmv_device(x.data_ptr(), y.data_ptr(), stream.cuda_stream)
    torch.cuda.synchronize()
    y_gpu = y.double().cpu().numpy()
    spmv_ok = y_gpu.tobytes() == y_ref.tobytes()
    conv_ok = all(conv.values())
    med = float(np.median(times))
    cores, model = cpu_info()
    parity = {
        "conversion": "bit-exact" if conv_ok else "MISMATCH: " + ",".join(k for k, v in conv.items() if not v),
        "conversion_checked": "groups, threads_mapping, values, columns of the device export vs oracle/_ref "
                              "argcsr_from_csr of the same CSR (memcmp)",
        "spmv": "bit-exact" if spmv_ok else f"MISMATCH max|dy|={float(np.max(np.abs(y_gpu - y_ref))):.3e}",
        "spmv_checked": "y of the timed kernel vs oracle/_ref spmv_argcsr_parallel on the reference's own conversion",
    }
    return {"value": round(2.0 * A.nnz / med / 1e9, 4), "unit": "GFLOP/s", "cores": workers, "kind": "reference",
            "sample": f"{args.cpu_sample_steps} x spmv_argcsr_parallel (oracle/_ref, {workers} threads) over the "
                      f"full matrix after 2 warm-up, median; matrix = the reference's own argcsr_from_csr",
            "ms_per_step": med * 1e3, "cpu_model": model, "reference_conversion_s": round(ref_conv_s, 3),
            "parity": parity}, conv_ok and spmv_ok


def other_configs(args, dev, stream, peak):
    """The other single-GPU configs of BASELINE.json measured in the same run
    (fp64 C1 with L2 flushed per step -- it is L2-resident otherwise --, C3,
    C4, and C4 in fp32): GFLOP/s, roofline fraction, the L2-flushed median,
    and cuSPARSE ALG1/ALG2 on the same CSR."""
    import torch

    import paper_1203_5737_b200 as argcsr
    import workloads

    res = []
    for name in ("C3", "C4", "C4f32", "C1"):
        try:
            cfg = workloads.CONFIGS[name]
            tdtype = torch.float64 if cfg["dtype"] == "float64" else torch.float32
            sv = 8 if tdtype == torch.float64 else 4
            # warm-up conversion of this dtype first: the first use of a dtype's
            # kernels (lazy module loading) is not part of the conversion time
            _w = workloads.stencil3d27(12, dev)
            argcsr.argcsr_from_torch(_w.num_rows, _w.num_cols, _w.row_pointers, _w.columns, _w.values.to(tdtype),
                                     args.tpg, args.dcs, stream=stream).free()
            del _w
            A = cfg["gen"](dev)
            vals = A.values.to(tdtype).contiguous()
            torch.cuda.synchronize()  # the CSR is produced on the default stream
            t_conv = time.perf_counter()
            with torch.cuda.stream(stream):
                m = argcsr.argcsr_from_torch(A.num_rows, A.num_cols, A.row_pointers, A.columns, vals, args.tpg,
                                             args.dcs, stream=stream)
            torch.cuda.synchronize()
            conv_ms = 1e3 * (time.perf_counter() - t_conv)
            x = workloads.bench_input(A.num_cols, dev, tdtype)
            y = torch.empty(A.num_rows, dtype=tdtype, device=dev)
            fn = lambda: m.spmv_device(x.data_ptr(), y.data_ptr(), stream.cuda_stream)  # noqa: E731
            ab = alg_bytes(A.nnz, A.num_rows, A.num_cols, sv)
            flush = l2_flusher(dev)
            time_steps(fn, args.warmup, stream)
            steps = min(args.steps, 50)
            entry = {"workload": name, "matrix": A.name, "dtype": "f64" if sv == 8 else "f32", "nnz": A.nnz,
                     "rows": A.num_rows, "groups": m.num_groups, "heavy_groups": m.heavy_groups,
                     "stored_slots": m.stored_slots, "total_slots": m.total_slots, "x_remap": m.x_remap,
                     "conversion_ms": round(conv_ms, 3), "alg_bytes": ab}
            if name != "C1":
                per, total = time_steps(fn, steps, stream)
                ms = total / steps
                entry.update(ms_per_step=ms, median_ms=statistics.median(per), gflops=2 * A.nnz / ms / 1e6,
                             frac=round(ab / ms / 1e6 / peak, 4))
            per_f, _ = time_steps(fn, steps, stream, flush)
            mf = statistics.median(per_f)
            entry.update(l2_flushed_median_ms=mf, l2_flushed_gflops=2 * A.nnz / mf / 1e6,
                         l2_flushed_frac=round(ab / mf / 1e6 / peak, 4))
            if name == "C1":
                per_b, total_b = time_steps(fn, steps, stream)
                entry.update(gflops=entry["l2_flushed_gflops"], frac=entry["l2_flushed_frac"],
                             back_to_back_ms=total_b / steps,
                             note="L2-resident working set: the headline numbers are L2-flushed per step; "
                                  "back_to_back_ms is the same product unflushed, the condition cuSPARSE is "
                                  "timed in")
            m.free()
            del m
            entry["cusparse"] = [dict(r, gflops=2 * A.nnz / r["ms"] / 1e6) if "ms" in r else r
                                 for r in cusparse_yardstick(A, x, tdtype, stream, steps, args.warmup)]
            res.append(entry)
            del A, vals, x, y
        except Exception as e:
            res.append({"workload": name, "error": f"{type(e).__name__}: {e}"[:200]})
        torch.cuda.empty_cache()
    return res


def main(argv=None):
    args = parse_args(argv)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
