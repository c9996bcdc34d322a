"""The stored full-size oracle results (tests/golden/oracle_<cfg>.npz, written by scripts/make_oracle_golden.py,
which calls only oracle/) belong to the current inputs and the current oracle source, and a fresh oracle run on
windows of each configuration reproduces them (root intervals and group starts bit for bit, W exactly)."""
import hashlib
import json
import os

import numpy as np
import pytest

import mrrr_inputs as mi
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load(name):
    z = np.load(os.path.join(ROOT, "tests", "golden", f"oracle_{name}.npz"))
    out = {k: z[k] for k in z.files if k != "meta"}
    out["meta"] = json.loads(str(z["meta"]))
    return out


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5b", "C5a"])
def test_golden_matches_inputs_oracle_and_a_fresh_window(cfg):
    c = mi.CONFIGS[cfg]
    d, e = c.matrix()
    G = _load(cfg)
    h = hashlib.sha256()
    h.update(d.tobytes())
    h.update(e.tobytes())
    assert G["meta"]["input_sha256"] == h.hexdigest()
    with open(os.path.join(ROOT, "oracle", "mrrr_oracle.c"), "rb") as f:
        assert G["meta"]["oracle_sha256"] == hashlib.sha256(f.read()).hexdigest()
    assert G["W"].size == c.k and G["root_lo"].size == c.n
    assert np.all(np.diff(G["W"]) >= 0)
    # a window in the middle of the index range, same root side as the stored all-range solve
    width = 6
    a = c.il + (c.k // 2) - 3
    r = oracle.mrrr(d, e, a, a + width - 1, root_side=int(G["side"][0]))
    assert r.info == 0
    pos = np.nonzero(~np.isnan(r.root_lo))[0]
    assert np.array_equal(r.root_lo[pos], G["root_lo"][pos]) and np.array_equal(r.root_hi[pos], G["root_hi"][pos])
    assert np.array_equal(r.root_gstart[pos[1:]], G["root_gstart"][pos[1:]])
    assert np.array_equal(r.W, G["W"][a - c.il:a - c.il + width])
