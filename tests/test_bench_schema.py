"""The committed bench lines (profiles/r01/) carry every key the driver contract asks for."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def line(name, rnd="r02"):
    return json.loads(open(os.path.join(ROOT, "profiles", rnd, name)).read().strip().splitlines()[-1])


@pytest.mark.parametrize("name", ["bench_final.json", "bench_final_c3.json", "bench_final_c7se.json"])
def test_bench_line_schema(name):
    d = line(name)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["warmup"] >= 3 and d["value"] > 0 and d["gpu_launches"] > 0
    assert "workload" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] in ("hbm", "tensor", "alu") and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["clocks"]
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in c, k
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert not bad & set(c["reasons"])


def test_default_bench_line_has_cpu_baseline():
    d = line("bench_final.json")
    cb = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "sweeps"):
        assert k in cb, k
    assert cb["kind"] == "oracle" and cb["cores"] >= 1
    # whole oracle sweeps (c2, c3), not a scaled sample, carry the value
    assert set(cb["sweeps"]) == {"c2", "c3"} and cb["value"] == cb["sweeps"]["c3"]["value"]


def test_default_roofline_is_the_whole_sweep():
    """north_star's quantity: the sweep's algorithmic bytes (40 B/dof for c5) over the
    measured HBM peak; per-kernel lines under `kernels`."""
    d = line("bench_final.json")
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["scope"].startswith("whole sweep") and r["bytes_per_dof"] == 40
    assert abs(r["achieved"] - r["algorithmic_bytes_per_step"] / (d["ms_per_step"] * 1e-3) / 1e9) < 1e-6 * r["achieved"]
    assert "k1" in d["kernels"] and "dominant" in d["kernels"]


def test_gmres_step_line():
    d = line("bench_final_c4_gmres.json")
    r = d["roofline"]
    assert r["bound"] == "hbm" and len(r["step_ms"]) == d["steps"] == 3
    assert 0 < r["frac"] <= 1


def test_reference_line():
    d = line("bench_reference_final.json")
    assert d["config"]["workload"] == line("bench_final.json")["config"]["workload"]
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def _run_bench(*argv, env=None):
    import subprocess
    import sys

    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], capture_output=True, text=True,
                       timeout=300, env=e, cwd=ROOT)
    return p


def test_bench_self_launches_n_ranks():
    """bench.py --gpus 2 without a torchrun environment starts 2 ranks itself (gloo here, NCCL
    on a GPU box): every rank joins one process group and rank 0 reports n_gpus = 2."""
    p = _run_bench("--gpus", "2", "--launch-check")
    assert p.returncode == 0, p.stderr
    d = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    assert d["n_gpus"] == 2 and d["world_size_ok"] and d["allreduce_sum"] == 2.0


def test_bench_rejects_world_size_mismatch():
    p = _run_bench("--gpus", "1", "--launch-check", env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert p.returncode != 0 and "WORLD_SIZE" in p.stderr
