"""bench.py's JSON line carries every key the driver's contract names: the
reference arm runs here on the CPU (it never touches a GPU); our arm on a B200."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(*args, timeout=600):
    res = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1")
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "Gpixel/s"
    assert d["higher_is_better"] is True and d["config"]["workload"]
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == d["value"] and d["dtype"] == "u32"
    assert cb["host"]["cpu_count"] >= cb["cores"]
    assert d["e2e"] == {"value": d["value"], "unit": "Gpixel/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_line(cuda_dev):
    d = _run("--config", "c1", "--steps", "2000", "--warmup", "3")
    assert BASE_KEYS | {"roofline", "cpu_baseline", "gpu_launches", "clocks"} <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 2000 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    cb = d["cpu_baseline"]
    assert cb["cores"] == 1 and cb["kind"] in ("reference", "port") and cb["value"] > 0
    assert cb["sample"] and d["dtype"] == "u32"
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 256 * 256 and e["d2h_bytes_per_step"] == 256 * 8 * 4
    assert d["gpu_launches"] >= 2000
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["parity"]["ok"] and d["parity"]["checked_px"] == 256 * 256
    assert d["e2e"]["dropin"]["per_call_us"] > 0


def test_both_arms_share_config():
    """The driver compares the two arms' `config` dicts: one function makes both."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    assert b.DEFAULT_CONFIG == "c4"
    for cfg in b.CONFIGS:
        for world in (1, 2, 8):
            c = b.workload_config(cfg, world, False)
            assert c == b.workload_config(cfg, world, False) and c["config_id"] == cfg
    ref = _run("--impl", "reference", "--config", "c2", "--steps", "2", "--warmup", "1")
    assert ref["config"] == b.workload_config("c2", 1, False)
    assert ref["cpu_baseline"]["sample"].startswith("the whole config every step (16777216 px")
