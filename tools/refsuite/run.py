"""Run the reference's own test suite (staged in baseline/_ref/tests) in one
or more modes of sfdt_refsuite_plugin and print one JSON line per mode:

    python tools/refsuite/run.py [stock] [seam] [dropin]

Needs a GPU for seam / dropin.  Exit 0 iff every requested mode passed.
"""

import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
STAGE = os.path.join(ROOT, "baseline", "_ref")


def run(mode: str) -> dict:
    env = dict(os.environ, SFDT_REFSUITE_MODE=mode,
               PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "tools", "refsuite"), ROOT]))
    cmd = [sys.executable, "-m", "pytest", "tests", "-q", "-p", "sfdt_refsuite_plugin", "-p", "no:cacheprovider",
           "-c", os.devnull, "--rootdir", STAGE]
    r = subprocess.run(cmd, cwd=STAGE, env=env, capture_output=True, text=True)
    tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
    counts = {k: int(v) for v, k in re.findall(r"(\d+) (passed|failed|error|errors|skipped)", tail)}
    return {"mode": mode, "returncode": r.returncode, "summary": tail, **counts,
            "failures": [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")][:20]}


def main(argv):
    if not os.path.isdir(os.path.join(STAGE, "tests")):
        print(json.dumps({"unavailable": "baseline/_ref/tests not staged (tools/stage_reference.sh)"}))
        return 0
    ok = True
    for mode in argv or ["stock", "seam", "dropin"]:
        res = run(mode)
        ok &= res["returncode"] == 0
        print(json.dumps(res), flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
