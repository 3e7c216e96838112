"""Shared fixtures.  GPU tests are marked ``gpu``; everything else runs on CPU."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running (minutes)")


@pytest.fixture(scope="session")
def golden_ref():
    with open(os.path.join(GOLDEN, "reference.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_builds():
    return dict(np.load(os.path.join(GOLDEN, "builds_small.npz")))


def sha(a) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()[:16]


class GoldenCase:
    """One stored reference build: inputs + expected CSR."""

    def __init__(self, meta: dict, arrays: dict):
        import paper_2401_06713_b200 as b200
        from paper_2401_06713_b200.driver import ColorLists
        from paper_2401_06713_b200.graph import EdgeOracleView

        name = meta["name"]
        self.meta = meta
        words = arrays[f"{name}/words"]
        q = meta["num_qubits"]
        strings = ["I" * q] * words.shape[0]  # strings are not used by the build
        ps = b200.PauliSet(strings, np.array(words, dtype=np.uint64))
        self.view = EdgeOracleView(ps, "implicit-complement", active=arrays[f"{name}/active"])
        if f"{name}/lists" in arrays:
            self.lists = ColorLists.from_array(self.view.active, arrays[f"{name}/lists"],
                                               meta["palette_base"], meta["palette_size"])
        else:
            data, off = arrays[f"{name}/list_data"], arrays[f"{name}/list_off"]
            rows = [data[off[k]:off[k + 1]] for k in range(off.size - 1)]
            self.lists = ColorLists(self.view.active, rows, meta["palette_base"], meta["palette_size"])
        self.members = arrays[f"{name}/members"]
        self.offsets = arrays[f"{name}/offsets"]
        self.neighbors = arrays[f"{name}/neighbors"].astype(np.int64)

    def check(self, got) -> None:
        assert np.array_equal(got.members, self.members)
        assert got.edge_count == self.meta["edge_count"]
        assert np.array_equal(got.graph.offsets if hasattr(got, "graph") else got.offsets, self.offsets)
        nb = got.graph.neighbors if hasattr(got, "graph") else got.neighbors
        assert np.array_equal(nb, self.neighbors)
        assert got.view_edges_scanned == self.meta["view_edges_scanned"]


@pytest.fixture(scope="session")
def golden_cases(golden_ref, golden_builds):
    return [GoldenCase(m, golden_builds) for m in golden_ref["cases"]]


def pauli_view(n, q, seed):
    import paper_2401_06713_b200 as b200

    return b200.pauli_view(b200.PauliSet.from_strings(b200.random_pauli_strings(n, q, seed=seed)))


def random_lists(view, pct=12.5, alpha=2.0, seed=0, iteration=1, base=0):
    import paper_2401_06713_b200 as b200

    plan = b200.plan_iteration(iteration, view.n_active, b200.PaletteParams(pct, alpha, seed),
                               palette_base=base)
    return b200.assign_random_lists(plan, view.active, seed)


def oracle_builder(view, lists, **kw):
    """The C oracle wrapped as a ``build``-compatible function (tests only)."""
    from oracle.oracle import oracle_build
    from paper_2401_06713_b200.conflict import ConflictGraph
    from paper_2401_06713_b200.graph import ExplicitGraph

    o = oracle_build(view, lists)
    return ConflictGraph(o.members, ExplicitGraph(int(o.members.size), o.offsets, o.neighbors),
                         o.edge_count, o.view_edges_scanned)
