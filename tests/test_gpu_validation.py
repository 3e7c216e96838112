"""GPU exhaustive validator against the reference validator's own reports
(tests/golden/validation.*, made by tools/make_golden_validation.py from
/root/reference/pkg/src/palettecolor/validation.py:41-131), and beyond its 20k cap."""

import json
import os

import numpy as np
import pytest

import paper_2401_06713_b200 as b200
from paper_2401_06713_b200 import validation
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

with open(os.path.join(GOLDEN, "validation.json")) as _f:
    CASES = json.load(_f)


@pytest.fixture(scope="module")
def arrays():
    return dict(np.load(os.path.join(GOLDEN, "validation.npz")))


@pytest.fixture(scope="module")
def runs():
    out = {}
    for c in CASES:
        key = (c["n"], c["q"], c["gen_seed"])
        if key not in out:
            ps = b200.PauliSet.from_strings(b200.random_pauli_strings(c["n"], c["q"], seed=c["gen_seed"]))
            out[key] = (ps, b200.run(b200.pauli_view(ps), b200.PaletteParams(12.5, 2.0, seed=0)))
    return out


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_report_matches_reference(case, arrays, runs):
    ps, res = runs[(case["n"], case["q"], case["gen_seed"])]
    view = b200.pauli_view(ps)
    if case["subset"]:
        view = view.induce(arrays[case["name"] + "/active"])
    res.color = arrays[case["name"] + "/color"].copy()
    rep = validation.validate(view, res, "exhaustive")
    assert rep.proper == case["proper"]
    assert rep.violation_count == case["violation_count"]
    assert [list(p) for p in rep.violations] == case["violations"]
    assert rep.oracle_edges == case["oracle_edges"]
    assert rep.pairs_checked == case["pairs_checked"]
    assert rep.colors_used == case["colors_used"]
    assert rep.ec_max_pct == pytest.approx(case["ec_max_pct"])


def test_beyond_reference_cap():
    """A 30k-vertex run (above the reference's 20k exhaustive cap) validates as proper, with
    |E| equal to the run's own oracle_edges; breaking one color is caught exactly."""
    ps = b200.PauliSet.from_strings(b200.random_pauli_strings(30000, 32, seed=5))
    view = b200.pauli_view(ps)
    res = b200.run(view, b200.PaletteParams(12.5, 2.0, seed=0))
    with pytest.raises(b200.errors.TooLargeForExactError):
        validation.validate(view, res)  # the reference's cap is the default
    rep = validation.validate(view, res, uncapped=True)
    assert rep.proper and rep.violation_count == 0
    assert rep.oracle_edges == res.oracle_edges
    # give vertex v the color of a commuting partner u < v: exactly the violations of v
    v = 29999
    u = int(np.flatnonzero(view.pair_mask(np.arange(v), np.full(v, v)))[0])
    bad = res.color.copy()
    bad[v] = bad[u]
    same = np.flatnonzero((bad == bad[v]) & (np.arange(bad.size) != v))
    commuting = same[view.pair_mask(same, np.full(same.size, v))]
    res.color = bad
    rep = validation.validate(view, res, uncapped=True)
    assert rep.violation_count == commuting.size >= 1
    assert rep.violations[: len(commuting)] == sorted((int(a), v) for a in commuting)
