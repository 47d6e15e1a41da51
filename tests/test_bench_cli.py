"""bench.py's contract on CPU: the reference arm (the oracle, per the task's
tier rules) prints one JSON line with the required keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                        "--steps", "1", "--warmup", "0", "--cpu-sample-n", "64"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ["impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"]:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert "workload" in d["config"]


import pytest  # noqa: E402


@pytest.mark.gpu
def test_mine_arm_json_line_is_consistent():
    """bench.py's own arm on the GPU (config 1, short): one JSON line with the
    contract's keys, and the numbers agree with one another -- value =
    pairs x steps / time, the e2e value is the same pair count over the
    (longer) end-to-end time, the roofline fraction is achieved / peak."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "1", "--steps", "3",
                        "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"]:
        assert k in d, k
    pairs = sum(d["pairs_per_step"].values())
    assert abs(d["value"] - pairs / (d["ms_per_step"] / 1e3)) <= 1e-6 * d["value"]
    e = d["e2e"]
    assert abs(e["value"] - pairs / (e["ms_per_step"] / 1e3)) <= 1e-6 * e["value"]
    assert e["ms_per_step"] >= d["ms_per_step"] * 0.5 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    ro = d["roofline"]
    assert abs(ro["frac"] - ro["achieved"] / ro["peak"]) <= 1e-9 and 0 < ro["frac"] < 1
    assert d["gpu_launches"] > 0
    # per-step device times (sum = the timed total within event skew), partition GEMM
    # rooflines, per-collective bytes (nothing leaves the GPU at N = 1)
    assert len(d["step_ms_rank0"]) == 3 and len(d["host_segments_ms_rank0"]) == 3
    assert sum(d["step_ms_rank0"]) <= 3 * d["ms_per_step"] * 1.01
    pr = d["partition_roofline"]
    for g in ("S2a_gemm", "S2d_gemm"):
        assert pr[g]["pairs"] > 0 and abs(pr[g]["frac"] - pr[g]["achieved"] / pr["peak"]) <= 1e-9
    assert all(v == 0 for v in d["collectives"]["bytes_sent_per_rank_per_step"].values())
