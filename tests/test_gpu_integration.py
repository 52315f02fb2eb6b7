"""The drop-in itself: the reference driver's own load_run_config +
materialize + execute_mode("oracle") against the added execute_mode("b200")
(integration/ixsum_b200_mode.cpp), on the reference corpus specs. The check
binary links the reference library compiled in place and libixb.so."""
import glob
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "b200_mode_check")
SPECS = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "specs", "*.json")))


def test_reference_driver_b200_mode_on_corpus():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/b200_mode_check not built (needs the reference sources)")
    r = subprocess.run([BIN] + SPECS, capture_output=True, text=True, timeout=600)
    lines = [json.loads(x) for x in r.stdout.strip().splitlines()]
    assert r.returncode == 0, r.stdout + r.stderr
    assert len(lines) == len(SPECS) >= 6
    assert all(x["ok"] for x in lines), lines
