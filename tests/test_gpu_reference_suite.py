"""The reference's own test suite (/root/reference/pkg/tests: 49 tests of
spectral.py and syndrome.py, staged into baseline/_ref/tests by
tools/stage_reference.sh) run against the B200 implementation
(tools/refsuite/): with the reference's kernel seam bound to
paper_1407_8315_b200.kernels, and with `sfft_dt` resolved to
paper_1407_8315_b200 itself.  Skipped where the staging is absent (it is
git-ignored; it travels to the GPU box with the gpurun snapshot)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("mode", ["seam", "dropin"])
def test_reference_suite(mode):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "tests")):
        pytest.skip("reference suite not staged (tools/stage_reference.sh)")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "refsuite", "run.py"), mode],
                       capture_output=True, text=True, timeout=900)
    res = json.loads(r.stdout.strip().splitlines()[-1])
    print(res["summary"])
    assert res["returncode"] == 0, res
    assert res.get("passed", 0) >= 49 and not res.get("failed")
