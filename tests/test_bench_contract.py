"""The bench's reference arm (`bench.py --impl reference`) keeps the driver
contract on the CPU: one JSON line with the B200 arm's metric, unit and
config keys, `impl: reference`, a `cpu_baseline` describing the run, a
zero-byte `e2e`, and the reference's own correctness check
(bench.cpp:220-226) -- and it maps none of this package's native libraries.
Runs C1 (5 M nnz) so it finishes in seconds."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

pytestmark = pytest.mark.skipif(not (ROOT / "oracle" / "_ref" / "libargcsr_ref.so").exists(),
                                reason="oracle/_ref not built")

PROBE = r"""
import atexit, json, runpy, sys
def maps():
    libs = sorted({l.split()[-1] for l in open('/proc/self/maps') if '.so' in l})
    print('MAPPED ' + json.dumps(libs), file=sys.stderr)
atexit.register(maps)
sys.argv = ['bench.py', '--impl', 'reference', '--config', 'C1', '--steps', '2', '--warmup', '1']
runpy.run_path('bench.py', run_name='__main__')
"""


def test_reference_arm_contract():
    env = dict(os.environ, PYTHONWARNINGS="ignore")
    r = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == "SpMV GFLOP/s" and line["unit"] == "GFLOP/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["steps"] == 2 and line["warmup"] == 1
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["value"] == line["value"] and cb["cores"] >= 1 and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    cfg = line["config"]
    for k in ("workload", "matrix", "rows", "cols", "nnz", "threads_per_group", "desired_chunk_size",
              "input_sha256"):
        assert k in cfg, k
    assert cfg["workload"] == "C1" and cfg["nnz"] == 5238784
    assert line["check"]["ok"] and line["check"]["relative_error_vs_spmv_csr"] <= 1e-10
    mapped = json.loads(r.stderr.split("MAPPED ", 1)[1].splitlines()[0])
    ours = [p for p in mapped if "paper_1203_5737_b200" in p]
    assert not ours, f"the reference arm mapped this package's libraries: {ours}"
    assert any(p.endswith("oracle/_ref/libargcsr_ref.so") for p in mapped)
