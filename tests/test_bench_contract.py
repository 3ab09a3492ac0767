"""bench.py's output contract: one JSON line with the keys the driver reads.

CPU: the reference arm (`--impl reference`, the oracle) on the small c1 config, and the
roofline helpers.  GPU: our arm on c1 with the roofline / cpu_baseline / e2e / clocks /
gpu_launches objects.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

COMMON = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
          "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1")
    assert COMMON <= set(d), COMMON - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "nnz·R/s"
    assert d["higher_is_better"] is True and d["vs_baseline"] is None and d["dtype"] == "f64"
    assert d["config"]["workload"] == "c1"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_self_launch_two_ranks():
    """`bench.py --gpus 2` outside torchrun re-executes itself under torch.distributed.run with
    two ranks on 127.0.0.1 (what a driver's `bench.py --gpus 8` relies on); rank 0 alone prints
    the line.  The reference arm runs without a GPU, so the launcher is checked on CPU."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--config", "c1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["world_size"] == 2 and d["n_gpus"] == 2 and d["impl"] == "reference"
    assert "torch.distributed.run" in out.stderr


def test_gather_view_helper():
    sys.path.insert(0, ROOT)
    import bench
    st = [{"iters": 2, "csf_nodes": [[10, 40, 100], [5, 60, 100], [20, 50, 100]]}]
    g = bench.gather_view(st, 3, 35, 1e-3, "all")
    rows = 2 * ((40 + 100) + (60 + 100) + (50 + 100))
    assert g["rows_per_s"] == pytest.approx(rows / 1e-3)
    assert g["row_bytes"] == 288 and g["peak_rows_per_s"] > 0
    assert g["frac"] == pytest.approx(g["rows_per_s"] / g["peak_rows_per_s"])
    assert bench.gather_view(st, 3, 35, 1e-3, "one") is None
    assert bench.gather_view(st, 3, 12, 1e-3, "all")["frac"] is None  # no measured peak (96 B)


@pytest.mark.gpu
def test_our_arm_line(cuda_ok):
    d = run_bench("--config", "c1", "--steps", "3", "--warmup", "3")
    assert COMMON <= set(d), COMMON - set(d)
    assert "impl" not in d and d["value"] > 0 and d["n_gpus"] == 1
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert r["alg_bytes_per_launch"] > r["min_bytes_per_launch"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert d["comm"]["nranks"] == 1
    assert {"alg_frac_of_hbm", "dram_frac_of_hbm", "l1tex_wavefront_pct"} <= set(r["views"])
    assert "one_thread" in cb and cb["one_thread"]["value"] > 0 and cb["host"]["logical_cpus"]
    clk = d["clocks"]
    assert clk is None or {"sm_mhz", "sm_max_mhz", "reasons"} <= set(clk)
