"""Every selectable kernel variant (env knobs) stays bit-exact: the
north_star's per-warp match_any bins (K2a), one key per byte at B = 16, the previous
adjacent-pixel pairing, the pre-PRMT table layout, the bytewise SWAR downsample, the LDG downsample kernel, the downsample output
staged in the ring slot and written by the producer's TMA bulk stores, the fused
kernel's previous 96 KB table layout (SCN_FUSED_SPLIT=0; the split layout is the
default), and non-default warp counts / tile sizes."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

VARIANTS = [
    {"SCN_HIST_IMPL": "match"},
    {"SCN_HIST_SINGLE": "1"},
    {"SCN_HIST_VAR": "8"},
    {"SCN_HIST_VAR": "64"},
    {"SCN_DS_VAR": "0"},
    {"SCN_DS_VAR": "1"},
    {"SCN_DS_VAR": "2"},
    {"SCN_DS_IMPL": "1"},
    {"SCN_DS_STORE": "1"},
    {"SCN_FUSED_SPLIT": "0"},
    {"SCN_FLUSH_ZERO": "1"},
    {"SCN_MAX_STAGES": "2"},
    {"SCN_L2_PREFETCH": "0"},
    {"SCN_L2_PREFETCH": "3"},
    {"SCN_FUSED_TILE": "23040"},
    {"SCN_HIST_WARPS": "8", "SCN_FUSED_WARPS": "16"},
    {"SCN_HIST_TILE": "15360", "SCN_FUSED_TILE": "23040", "SCN_DS_TILE": "64512"},
]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_variant_parity(env):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "helpers", "variant_parity.py")],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "variant_parity ok" in r.stdout
