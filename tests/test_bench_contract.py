"""bench.py's driver contract on CPU: the reference arm (the oracle C port of the reference's CPU path) prints
one JSON line with the contract's keys; under torchrun only rank 0 works and prints; and the GPU arm's
options exist.  (The GPU arm itself runs in the gpu tier and at round end.)"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT, env=env)
    return r


def test_reference_arm_prints_one_contract_line():
    r = _bench(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "frames/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1 and d["n_gpus"] == 1
    assert d["config"]["workload"].startswith("c1")
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["vs_baseline"] is None


def test_reference_arm_only_rank0_prints_under_torchrun():
    r = _bench(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0"],
               {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]


def test_gpu_arm_refuses_a_world_size_mismatch():
    """Under torchrun, --gpus must equal WORLD_SIZE (a plain `bench.py --gpus 8` re-launches itself instead)."""
    r = _bench(["--gpus", "3", "--config", "c1", "--steps", "1"], {"RANK": "0", "WORLD_SIZE": "2", "LOCAL_RANK": "0"},
               timeout=120)
    assert r.returncode == 2
    assert "WORLD_SIZE" in r.stdout


def test_reference_arm_reports_the_requested_gpu_count():
    r = _bench(["--impl", "reference", "--gpus", "4", "--config", "c1", "--steps", "1", "--warmup", "0"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["n_gpus"] == 4


def test_gpu_arm_options():
    r = _bench(["--help"], timeout=120)
    assert r.returncode == 0
    for opt in ("--gpus", "--steps", "--warmup", "--impl", "--config", "--streams", "--view-group", "--coverage",
                "--band-output"):
        assert opt in r.stdout, opt


@pytest.mark.gpu
def test_gpu_arm_line_has_the_contract_keys():
    """bench.py's own arm on the GPU (small config): value, e2e with byte counts, roofline, clocks, launches."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = _bench(["--config", "c1", "--steps", "4", "--warmup", "3", "--no-cpu-baseline"], timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 4 and d["warmup"] == 3 and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    rf = d["roofline"]
    assert rf["bound"] in ("hbm", "tensor", "issue") and rf["peak"] > 0 and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["clocks"]["sm_mhz"] > 0
