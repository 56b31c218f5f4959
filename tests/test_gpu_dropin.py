"""The drop-in, proven with the reference's own acceptance suite
(/root/reference/proj/tests/acceptance.cpp, unchanged): integration/Makefile
links it against the unmodified reference objects with forward / inverse /
denoise taken from integration/transform_b200.cpp over libshearlet_b200.so
(the B200 path). Criteria that exercise the transform (1 exact
reconstruction, 5 oracle equivalence, 7 denoising, 8 inpainting, 9
separation, 10 invariants) must PASS exactly as with the CPU reference."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "accept", "acceptance_b200")


def test_reference_acceptance_suite_on_b200(cuda):
    if not os.path.exists(BIN):
        pytest.fail("oracle/_ref/accept/acceptance_b200 not built (make -C integration, in the build container)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=1200)
    print(r.stdout)
    res = dict(re.findall(r"criterion (\w+) \([^)]*\): (PASS|FAIL)", r.stdout))
    # 3 (frame-bound ratio pin) fails for the CPU reference build too; 11 times
    # forward() against an R N log N model, which host-copy-bound GPU calls do not follow
    for c in ("1", "2", "4", "5", "6", "7", "8", "9", "10"):
        assert res.get(c) == "PASS", (c, r.stdout)
