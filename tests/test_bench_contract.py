"""bench.py's JSON-line contract, on the CPU (no GPU needed).

The reference arm (`--impl reference`) times the oracle itself, so it runs
here on C1 and its line is checked key by key against the contract (metric
and unit of BASELINE.json, one measured full census equal to the oracle-only
golden file, `e2e` with zero copy bytes, `cpu_baseline` describing the run).
The GPU arm must fail loudly on a host without a GPU: no CPU fallback ever
prints a bench line.
"""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout)


def test_reference_arm_line_c1():
    r = _run(["--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["impl"] == "reference"
    assert d["metric"] == base["metric"]
    assert d["unit"] == "arcs/s" and d["higher_is_better"] is True
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["config"]["workload"].startswith("C1")
    assert d["census_matches_golden"] is True
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "census_C1.json")))
    want = golden["census"] if isinstance(golden, dict) else golden
    assert [int(x) for x in d["census"]] == [int(x) for x in want]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == d["value"] and cb["cores"] >= 1
    assert cb["sample"]


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure")
def test_gpu_arm_fails_loudly_without_gpu():
    r = _run(["--config", "C1", "--steps", "1", "--warmup", "3"])
    assert r.returncode != 0
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
