"""bench.py output contract (the JSON line the driver parses).

CPU: the reference arm (`--impl reference`, the oracle timed on the host cores on a bounded
sample) prints one line with the required keys, and non-zero ranks of a torchrun launch exit 0
without output.  GPU: the default arm (C3b, one GPU) prints one line with the required keys,
a roofline of the dominant kernel, e2e through host buffers, clocks and the launch count."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def _run(args, env_extra=None, timeout=900):
    env = dict(os.environ)
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    return lines


def test_reference_arm_line():
    lines = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "evals/s" and d["higher_is_better"] is True
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]


def test_reference_arm_other_ranks_silent():
    lines = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"],
                 env_extra={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, timeout=300)
    assert lines == []


@pytest.mark.gpu
def test_gpu_arm_line():
    lines = _run(["--steps", "1", "--warmup", "3", "--no-alt"], timeout=1200)
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d) and {"roofline", "clocks", "gpu_launches"} <= set(d)
    assert d["n_gpus"] == 1 and d["warmup"] >= 3 and d["dtype"] == "f64"
    assert d["config"]["workload"].startswith("C3b") and d["config"]["ndof_per_rank"] == 1003686
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1.2
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["e2e"]["h2d_bytes_per_step"] == 8 * 1003686 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 1000  # the CG loop's kernels, counted by the library
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["clocks"]["samples"] >= 1
    cert = d["extra"]["certification"]
    assert cert["true_rel_res"] < 1e-9 and cert["lanczos_lmin"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["C1", "C2"])
def test_gpu_latency_lines(workload):
    lines = _run(["--workload", workload, "--steps", "20", "--warmup", "3"], timeout=600)
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d) and d["metric"].startswith(workload) and d["value"] > 0
    assert d["roofline"]["bound"] == "latency" and d["roofline"]["achieved"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["extrapolated"] is False
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0


@pytest.mark.gpu
def test_gpu_c5_line():
    lines = _run(["--workload", "C5", "--steps", "1", "--warmup", "3"], timeout=900)
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d) and d["unit"] == "designs/s" and d["scaling"] == "weak" and d["value"] > 0
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.2
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["gpu_launches"] > 0
    assert d["config"]["cg_iters_max"] >= d["config"]["cg_iters_min"] > 0
