"""bench.py's reference arm runs on the CPU and prints one JSON line with the driver's
contract keys (metric/value/unit/..., impl, cpu_baseline, e2e with zero copies)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
         "--warmup", "1", "--matrix-order", "600"],
        capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference"
    assert d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["n"] == 600 and "non-default" in d["metric"]


def test_guarded_leg_reports_errors_and_abandons_a_stuck_leg():
    """bench.guarded_leg: an exception becomes the leg's error entry; a leg still running
    at the limit makes rank 0 print the headline line (with the error) and exit 0, so a
    rank stuck in a collective never costs the headline."""
    sys.path.insert(0, ROOT)
    import bench

    def boom():
        raise RuntimeError("collective failed")

    out = bench.guarded_leg({"value": 1.0}, 0, boom, limit_s=30.0)
    assert out == {"error": "RuntimeError: collective failed"}
    assert bench.guarded_leg(None, 1, lambda: {"s_per_solve": 1.0}, limit_s=30.0) == \
        {"s_per_solve": 1.0}
    code = ("import sys, time; sys.path.insert(0, %r); import bench; "
            "bench.guarded_leg({'metric': 'm', 'value': 2.0}, 0, lambda: time.sleep(60), "
            "limit_s=1.0); print('not reached')" % ROOT)
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=120, cwd=ROOT)
    assert res.returncode == 0
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and "not reached" not in res.stdout
    d = json.loads(lines[0])
    assert d["value"] == 2.0 and "abandoned" in d["solve_c4"]["error"]


def test_time_budget_skips_a_leg_that_would_overrun():
    """bench.in_budget: an optional leg starts only when its usual duration still fits in
    --time-budget-s of process time, so the JSON line is printed before an outer limit."""
    import argparse
    sys.path.insert(0, ROOT)
    import bench

    elapsed = bench.time.monotonic() - bench.T_PROCESS_START
    roomy = argparse.Namespace(time_budget_s=elapsed + 10_000.0)
    tight = argparse.Namespace(time_budget_s=elapsed + 60.0)
    assert bench.in_budget(roomy, "sequence_c4")
    assert not bench.in_budget(tight, "sequence_c4")      # ~190 s does not fit in 60 s
    assert bench.in_budget(tight, "tail")                  # ~10 s does
    assert bench.in_budget(tight, "e2e") and bench.in_budget(tight, "cpu_baseline")
