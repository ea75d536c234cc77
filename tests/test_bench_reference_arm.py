"""bench.py --impl reference (the driver's reference arm) runs on CPU and
prints one JSON line with the contract's keys -- through the stock
reference package when baseline/_ref is staged, else the restated driver."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                        "--steps", "1", "--warmup", "0", "--cpu-seconds", "1", "--no-restated"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "signals/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
    if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "sfft_dt")):
        assert "unmodified reference package" in d["cpu_baseline"]["sample"]
