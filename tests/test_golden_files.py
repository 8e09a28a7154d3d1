"""Provenance of the config-size golden histories (tests/golden/hist_cfg*.json): every file was
written by tests/scripts/golden_histories.py from the oracle only.  Config 1 is recomputed here and
must match the stored file exactly; every file pair (own / reversed summation order) describes the
same run, and the reversed-order spread is at rounding level while the iteration is not blown up."""
import glob
import json
import os
import subprocess
import sys

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _pairs():
    return sorted(f[:-5] for f in glob.glob(os.path.join(GOLD, "hist_cfg*_*.json")) if not f.endswith("_alt.json"))


def test_config1_recomputes_exactly(tmp_path):
    env = dict(os.environ, GOLDEN_OUT=str(tmp_path))
    subprocess.check_call([sys.executable, os.path.join(ROOT, "tests", "scripts", "golden_histories.py"), "1", "vanka"],
                          env=env, stdout=subprocess.DEVNULL)
    new = json.load(open(tmp_path / "hist_cfg1_vanka.json"))
    old = json.load(open(os.path.join(GOLD, "hist_cfg1_vanka.json")))
    for key in ("hist", "floor8", "opts", "material", "cycles", "n", "levels"):
        assert new[key] == old[key], key
    assert new["final"] == old["final"]


@pytest.mark.parametrize("base", _pairs())
def test_pair_consistency(base):
    g = json.load(open(base + ".json"))
    a = json.load(open(base + "_alt.json"))
    assert not g["alt_order"] and a["alt_order"]
    for key in ("config", "n", "levels", "relax", "opts", "cycles", "b_seed", "K_seed", "material"):
        assert g[key] == a[key], key
    hO, hA = np.array(g["hist"]), np.array(a["hist"])
    assert len(hO) == g["cycles"] + 1 and np.all(np.isfinite(hO))
    assert g["final"]["slots"] == a["final"]["slots"]
    # two legal summation orders agree to a small multiple of the a-priori rounding scale
    assert np.all(np.abs(hO - hA) <= 1e3 * np.array(g["floor8"]) + 1e-12 * hO)
