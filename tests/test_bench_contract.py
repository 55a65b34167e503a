"""bench.py's output contract: one JSON line per run with the keys the driver reads, the same
`config` dict on the GPU arm and the reference arm (the fp64 oracle on host cores), and the
reference arm under torchrun printing from rank 0 only.  Small config (C1) so the CPU tests stay
fast; the GPU arm's line is checked on the box."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=600, env=None):
    r = subprocess.run([sys.executable] + args, cwd=ROOT, capture_output=True, text=True, timeout=timeout,
                       env=dict(os.environ, **(env or {})))
    assert r.returncode == 0, r.stderr[-2000:]
    return [json.loads(x) for x in r.stdout.strip().splitlines() if x.startswith("{")]


def _expected_config(name, lam=1e-2):
    import bench
    from paper_2202_08627_b200 import synth
    return bench.bench_config(synth.CONFIGS[name], lam)


def test_reference_arm_line():
    lines = _run(["bench.py", "--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "3"])
    assert len(lines) == 1
    d = lines[0]
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["dtype"] == "f64" and d["higher_is_better"] is True
    import bench
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 3
    assert d["config"] == _expected_config("C1")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_torchrun_rank0_only():
    """Under torchrun (N > 1) rank 0 alone runs the oracle and prints; the other ranks exit 0."""
    lines = _run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
                  "127.0.0.1", "--master-port", "29531", "bench.py", "--impl", "reference", "--config", "C1",
                  "--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2


@pytest.mark.gpu
def test_gpu_arm_line():
    lines = _run(["bench.py", "--config", "C1", "--steps", "5", "--warmup", "3", "--no-cpu-baseline"])
    assert len(lines) == 1
    d = lines[0]
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["config"] == _expected_config("C1")          # same dict as the reference arm
    assert d["dtype"] == "f32" and d["scaling"] == "weak" and d["n_gpus"] == 1 and d["steps"] == 5
    assert d["value"] > 0 and abs(d["value"] - 1000.0 / d["ms_per_step"]) < 1e-3 * d["value"] + 1e-3
    rf = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(rf)
    assert rf["peak"] > 0 and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] < d["value"]                         # host copies inside the timed region
    assert d["gpu_launches"] >= 4 * d["steps"]             # K0..K3 per evaluation, all libei kernels
    assert d["clocks"]["sm_mhz"] and d["clocks"]["sm_max_mhz"]
    assert set(d["kernels"]) >= {"K0_pack", "K1_project", "K2_curve", "K3_backproject"}
    pct = d["ms_per_step_pct"]                           # per-step spread of the device times
    assert 0 < pct["p10"] <= pct["p50"] <= pct["p90"]
