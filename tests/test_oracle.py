"""The oracle (oracle/conflict_oracle.c) pinned against the reference's own outputs."""

import numpy as np
import pytest

from conftest import pauli_view, random_lists, sha
from oracle.oracle import OracleInstance, oracle_build


def test_oracle_matches_every_golden_build(golden_cases):
    for case in golden_cases:
        case.check(oracle_build(case.view, case.lists, threads=4))


@pytest.mark.parametrize("n", [5000, 10000])
def test_oracle_matches_hashed_q32_builds(golden_ref, n):
    g = golden_ref["builds_hashed"][f"q32_n{n}"]
    v = pauli_view(n, 32, 0)
    lists = random_lists(v, seed=0)
    assert sha(lists.array) == g["lists_sha"]
    o = oracle_build(v, lists)
    assert (sha(o.members), sha(o.offsets), sha(o.neighbors)) == (
        g["members_sha"], g["offsets_sha"], g["neighbors_sha"])
    assert o.edge_count == g["edge_count"]
    assert o.view_edges_scanned == g["view_edges_scanned"]


def test_oracle_thread_count_independent(golden_cases):
    case = next(c for c in golden_cases if c.meta["name"] == "c1_iter1")
    a = oracle_build(case.view, case.lists, threads=1)
    b = oracle_build(case.view, case.lists, threads=7)
    assert np.array_equal(a.neighbors, b.neighbors) and np.array_equal(a.offsets, b.offsets)


def test_oracle_rows_and_commute_count(golden_cases):
    case = next(c for c in golden_cases if c.meta["name"] == "c1_iter1")
    inst = OracleInstance(case.view.backing.words, case.view.active, case.lists)
    assert inst.commute_count() == case.meta["view_edges_scanned"]
    for i in (0, 1, 777, 1999):
        row, _ = inst.row(i)
        # row i of the golden CSR (all members here: compact id == local id)
        assert np.array_equal(row, case.neighbors[case.offsets[i]:case.offsets[i + 1]])


def test_oracle_scan_rows_counts(golden_cases):
    case = next(c for c in golden_cases if c.meta["name"] == "c1_iter1")
    inst = OracleInstance(case.view.backing.words, case.view.active, case.lists)
    pairs, seen, adm = inst.scan_rows(0, inst.n)
    assert pairs == inst.n * (inst.n - 1) // 2
    assert seen == case.meta["view_edges_scanned"]
    assert adm == case.meta["edge_count"]
