"""Host helpers of the validation module against the reference's own (CPU, this container).

verify_palette_discipline / partition_groups / partition_export (validation.py:134-201) run on
a reference whole run (the reference's own builder, small view); the outputs and the first
failure messages must be the reference's.  The exhaustive cap is the reference's by default.
"""

import copy
import os
import sys

import numpy as np
import pytest

REF_SRC = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present")


@pytest.fixture(scope="module")
def ref_run():
    sys.path.insert(0, REF_SRC)
    try:
        import palettecolor as pc
        from palettecolor import validation as rv
    finally:
        sys.path.remove(REF_SRC)
    ps = pc.PauliSet.from_strings(pc.random_pauli_strings(400, 10, seed=3))
    view = pc.pauli_view(ps)
    res = pc.run(view, pc.PaletteParams(12.5, 2.0, seed=0))
    return pc, rv, ps, res


def _raises(fn, res):
    try:
        fn(res)
    except AssertionError as e:
        return str(e)
    return None


def test_partitions_match_reference(ref_run):
    from paper_2401_06713_b200 import validation as mv

    pc, rv, ps, res = ref_run
    assert mv.partition_groups(res) == rv.partition_groups(res)
    assert mv.partition_export(res, ps) == rv.partition_export(res, ps)


def test_palette_discipline_matches_reference(ref_run):
    from paper_2401_06713_b200 import validation as mv

    pc, rv, ps, res = ref_run
    assert _raises(mv.verify_palette_discipline, res) is None
    assert _raises(rv.verify_palette_discipline, res) is None
    colored = np.flatnonzero(res.color >= 0)
    # a color outside its iteration's palette; a color in the palette but not in the list
    for how in ("range", "list", "iteration"):
        bad = copy.deepcopy(res)
        v = int(colored[len(colored) // 3])
        it = int(bad.colored_at[v])
        plan = [r for r in bad.iterations if r.iteration == it][0]
        if how == "range":
            bad.color[v] = plan.palette_base + plan.palette_size + 5
        elif how == "list":
            lists = pc.driver.assign_random_lists(
                pc.driver.IterationPlan(iteration=it, palette_size=plan.palette_size,
                                        palette_base=plan.palette_base, list_size=plan.list_size),
                np.array([v], dtype=np.int64), res.params.seed)
            row = set(int(c) for c in lists.colors_for(v))
            bad.color[v] = next(c for c in range(plan.palette_base, plan.palette_base + plan.palette_size)
                                if c not in row)
        else:
            bad.colored_at[v] = 999
        want = _raises(rv.verify_palette_discipline, bad)
        assert want is not None
        assert _raises(mv.verify_palette_discipline, bad) == want


def test_exhaustive_cap_is_the_reference_default():
    import paper_2401_06713_b200 as b200
    from paper_2401_06713_b200 import validation as mv
    from paper_2401_06713_b200.graph import EXACT_ENUMERATION_CAP

    n = EXACT_ENUMERATION_CAP + 1
    ps = b200.PauliSet.from_strings(b200.random_pauli_strings(n, 8, seed=1))
    view = b200.pauli_view(ps)

    class R:
        color = np.zeros(n, dtype=np.int64)
        iterations = []
        peak_conflict_edges = 0

    with pytest.raises(b200.errors.TooLargeForExactError):
        mv.validate(view, R(), "exhaustive")
