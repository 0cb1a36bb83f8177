"""Every selectable kernel variant stays bit-exact against the oracle: the north_star's
per-warp __match_any_sync bins (K2a) and its packed-key amortisation (K2a'), chosen
through the ABI (scn_set_hist_impl), and the measurement build libscn_tuning.so
(`make tuning`, SCN_LIB=tuning) under non-default grid / tile / ring-depth / L2-prefetch
knobs. The product library reads no environment variables."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

T = {"SCN_LIB": "tuning"}
VARIANTS = [
    {"SCN_TEST_HIST_IMPL": "1"},
    {"SCN_TEST_HIST_IMPL": "2"},
    {**T},
    {**T, "SCN_MAX_STAGES": "2"},
    {**T, "SCN_L2_PREFETCH": "0"},
    {**T, "SCN_L2_PREFETCH": "3"},
    {**T, "SCN_FUSED_TILE": "23040"},
    {**T, "SCN_GRID": "7"},
    {**T, "SCN_HIST_TILE": "15360", "SCN_FUSED_TILE": "23040", "SCN_DS_TILE": "64512"},
]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_variant_parity(env):
    if env.get("SCN_LIB") == "tuning" and not os.path.exists(os.path.join(ROOT, "paper_1805_07339_b200",
                                                                          "libscn_tuning.so")):
        subprocess.run(["make", "-C", ROOT, "tuning"], check=True, capture_output=True)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "helpers", "variant_parity.py")],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "variant_parity ok" in r.stdout
