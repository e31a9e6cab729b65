"""CPU: bench.py's reference arm runs here (the reference's CPU lane through
oracle/_ref) and prints the driver's JSON contract: one line, the shared
keys, the reference-arm extras (impl, cpu_baseline, zero-copy e2e)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libocm_ref.so")),
                    reason="oracle/_ref not built")
def test_reference_arm_json_contract():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--config", "1"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert "workload" in d["config"] and "model" not in d["config"]


@pytest.mark.gpu
def test_device_arm_json_contract():
    """B200: the device arm's line carries every key the driver reads."""
    out = subprocess.run([sys.executable, "bench.py", "--steps", "1", "--warmup", "3", "--config", "1",
                          "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches",
              "clocks", "certified"):
        assert k in d, k
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] == r["achieved"] / r["peak"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 2 and d["certified"] == {"min": True, "max": True}
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libocm_ref.so")),
                    reason="oracle/_ref not built")
def test_reference_arm_never_loads_the_product():
    """The reference arm builds its graph with the checkers' generators and
    solves it with oracle/_ref: the product library is never mapped."""
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', "
            "'--warmup', '0', '--config', '1']; runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "assert 'libocm_b200' not in maps, 'product library loaded'; "
            "assert 'libocm_ref' in maps; "
            "assert 'paper_1111_0627_b200' not in sys.modules")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][0])
    # the same graph as the device arm: config 1 at full size, not a sample
    assert d["config"]["n"] == 10_000 and "SAMPLE" not in d["config"]["workload"]
    assert d["mu"] == {"min": "419/40", "max": "632/7"}  # tests/golden/config_golden.json


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libocm_ref.so")),
                    reason="oracle/_ref not built")
def test_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` without a torchrun environment starts two ranks
    itself (torch.distributed.run on 127.0.0.1); rank 0 alone prints."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "0", "--config", "1"], cwd=ROOT,
                         capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"


def test_gpus_flag_refuses_missing_devices():
    """More ranks than visible GPUs fails loudly instead of measuring fewer."""
    import torch
    n = max(2, torch.cuda.device_count() + 1)
    out = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--steps", "1"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300,
                         env={k: v for k, v in os.environ.items() if k != "WORLD_SIZE"})
    assert out.returncode != 0 and "visible" in out.stderr


@pytest.mark.gpu
def test_gpus_2_self_launch_on_one_gpu():
    """`bench.py --gpus 2` starts two ranks itself; with both on this box's
    one GPU (OCM_BENCH_SHARE_GPU=1: gloo plumbing, half the SMs each) the
    fused strong-scaling lane solves config 2 across them and rank 0 prints
    one line with n_gpus 2 and the reference's mu (config_golden.json)."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["OCM_BENCH_SHARE_GPU"] = "1"
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "2", "--steps", "1",
                          "--warmup", "1", "--no-cpu-baseline", "--no-e2e"], cwd=ROOT,
                         capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and "fused" in d["config"]["parallelism"]
    assert d["mu"] == {"min": "229/45", "max": "193/2"}
    assert d["policy_iterations"] == {"min": 44, "max": 26}
    assert all(d["time_to_ocm_s"][o] > 0 for o in ("min", "max"))
    assert abs(sum(d["time_to_ocm_s"].values()) * 1e3 - d["ms_per_step"]) < 1e-6 * d["ms_per_step"]
    # the strong-scaling reference point: the same graph on one GPU alone
    single = d["single_gpu_same_config"]
    assert single["value"] > 0 and single["unit"] == d["unit"] and single["steps"] == 2
    assert d["e2e"] is None
