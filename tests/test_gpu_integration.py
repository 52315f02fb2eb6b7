"""The drop-in itself: the reference driver's own load_run_config +
materialize + execute_mode("oracle") against the drop-in's device-built
materialize (integration/ixsum_b200_formats.cpp) + execute_mode("b200")
(integration/ixsum_b200_mode.cpp), on the reference corpus specs; and the
drop-in builders against the reference builders at BASELINE scale. The
check binary links the reference library compiled in place and libixb.so."""
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
    assert all(x["ok"] and x["formats_identical"] for x in lines), lines


def test_reference_builders_drop_in_at_baseline_scale():
    """ixsum::b200::{dense_to_coo, canonicalize, coo_to_groupcoo,
    dense_to_blockgroupcoo, group_coo_tensor, tune} (integration/
    ixsum_b200_formats.cpp, the reference's signatures over the device
    builders) equal the reference builders bit for bit on cfg1's and cfg2's
    full matrices and on rank-3/4 COO tensors, real and int64; errors have the
    reference's types and messages."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/b200_mode_check not built (needs the reference sources)")
    r = subprocess.run([BIN, "--builders"], capture_output=True, text=True, timeout=900)
    lines = [json.loads(x) for x in r.stdout.strip().splitlines()]
    assert r.returncode == 0, r.stdout + r.stderr
    assert len(lines) >= 20 and all(x["ok"] for x in lines), lines
