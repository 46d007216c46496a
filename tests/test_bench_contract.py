"""The driver's bench.py contract on CPU: the reference arm (`--impl reference`,
the CPU port of the reference kernels) prints exactly one JSON line with the
keys the driver reads, at N = 1 and under torchrun at N = 2 (rank 0 alone
prints). The GPU arm is exercised by `tests/test_scale_gpu.py` and the round-end
bench run."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.strip().startswith("{")]


def _check_reference_line(d, n):
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["impl"] == "reference" and d["n_gpus"] == n and d["steps"] == 1 and d["warmup"] == 1
    assert d["value"] > 0 and d["unit"] == "TFLOP/s" and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb)
    assert cb["kind"] in ("port", "reference") and cb["value"] == d["value"] and cb["cores"] >= 1
    e2e = d["e2e"]
    assert e2e["value"] == d["value"] and e2e["unit"] == d["unit"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def test_reference_arm_single_process():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--exp-max", "10"], capture_output=True, text=True, cwd=str(ROOT),
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = _json_lines(out.stdout)
    assert len(lines) == 1
    _check_reference_line(lines[0], 1)


def test_reference_arm_single_workload():
    """configs[0]: the full 1024^3 op through both CPU reference paths."""
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--workload", "single", "--single", "256"],
                         capture_output=True, text=True, cwd=str(ROOT), timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = _json_lines(out.stdout)
    assert len(lines) == 1
    _check_reference_line(lines[0], 1)
    assert "configs[0]" in lines[0]["config"]["workload"]


def test_reference_arm_under_torchrun():
    env = dict(os.environ, OMP_NUM_THREADS="1")
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl",
         "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--exp-max", "10"],
        capture_output=True, text=True, cwd=str(ROOT), timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = _json_lines(out.stdout)
    assert len(lines) == 1  # rank 0 alone prints
    _check_reference_line(lines[0], 2)


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["sweep", "fcn", "single"])
def test_gpu_arm_line(workload):
    """The GPU arm's JSON line on a reduced sweep (m,n,k <= 512) and the FCN
    step: roofline, cpu_baseline (sweep), e2e with host copies, launches and
    sampled clocks are all present and consistent."""
    args = [sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--workload", workload]
    if workload == "sweep":
        args += ["--exp-max", "9"]
    out = subprocess.run(args, capture_output=True, text=True, cwd=str(ROOT), timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = _json_lines(out.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert r["bound"] == "tensor" and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["verify"]["failed"] == 0 and d["verify"]["worst_rel_frobenius"] < 1e-5
    if workload in ("sweep", "single"):
        cb = d["cpu_baseline"]
        assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["value"] > 0
        # the reference arm reports the same config (same workload, same cases)
        ref = subprocess.run(args + ["--impl", "reference", "--steps", "1", "--warmup", "1"],
                             capture_output=True, text=True, cwd=str(ROOT), timeout=900)
        assert ref.returncode == 0, ref.stderr[-2000:]
        assert _json_lines(ref.stdout)[0]["config"] == d["config"]
    if workload == "sweep":
        mb = d["mtnn_vs_best_of_both"]
        assert 0 < mb["mean_per_case_ratio"] <= 1.05 and mb["aggregate_ratio"] <= 1.02
