"""The bench contract on CPU: `bench.py --impl reference` (the reference arm:
the reference's own hvbem from baseline/_ref timed on the host cores, the
oracle port when baseline/_ref is absent) prints one JSON line with the
metric, unit, cpu_baseline and e2e keys the driver reads."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    env = dict(os.environ, RANK="0")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--scale", "0.1",
                          "--steps", "1", "--warmup", "0", "--cpu-rows", "4"], capture_output=True, text=True,
                         timeout=600, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["impl"] == "reference" and d["metric"] == base["metric"]
    assert d["unit"] == "entries/s" and d["higher_is_better"] is True and d["value"] > 0
    cb = d["cpu_baseline"]
    want = "reference" if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "hvbem")) else "port"
    assert cb["kind"] == want and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_silently():
    env = dict(os.environ, RANK="1")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--scale", "0.1"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert res.returncode == 0 and res.stdout.strip() == ""
