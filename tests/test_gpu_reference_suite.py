"""The reference's own hot-path tests, unchanged, against the installed B200 builder (GPU).

SURVEY §4: the parity suite the new build must pass unchanged is the reference's
``tests/test_conflict.py`` (every Pauli build vs its naive ``build_reference``, all oracle
modes, subset views, determinism across threads/blocks/one-phase, the edge budget with the
reference's own exception class, CSR invariants), ``test_acceptance.py`` (acceptance
criteria incl. whole runs) and ``test_driver.py`` (Algorithm 1).  They run from an untracked
copy of the reference package under ``baseline/_ref/pkg`` (git-ignored; it travels to the GPU
box with the snapshot) with ``install_into(palettecolor)`` applied by
``tests/ref_dropin_plugin.py``; the plugin counts the builds the CUDA path served.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref", "pkg")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")),
                                 reason="no reference copy under baseline/_ref/pkg "
                                        "(cp -r /root/reference/pkg baseline/_ref/)")]


def _recorded_outcome(suite):
    """The reference's own recorded run of its suite (pkg/test_output.txt): the tests that
    failed there, and the ACCEPTANCE report lines (the acceptance criteria print measured
    values; test_criterion_05 and _10 are expected to fail at these sizes, see
    test_acceptance.py:203-210)."""
    failed, report = set(), {}
    with open(os.path.join(REF, "test_output.txt")) as f:
        for line in f:
            if line.startswith("FAILED tests/" + suite):
                failed.add(line.split()[1].split("::")[1])
            if line.startswith("tests/" + suite) and "ACCEPTANCE" in line:
                tail = line.split("ACCEPTANCE", 1)[1]
                report[int(tail.split()[0])] = tail.rsplit("; runtime", 1)[0].strip()
    return failed, report


@pytest.mark.parametrize("suite", ["test_conflict.py", "test_acceptance.py", "test_driver.py"])
def test_reference_suite_passes_unchanged(suite, tmp_path):
    """Same outcome as the reference's own run: every test it passed passes, and the two
    acceptance criteria it fails (by design, at these sizes) fail with identical measured
    values."""
    count = tmp_path / "count"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REF, "src"), os.path.join(ROOT, "tests"), ROOT,
                                         env.get("PYTHONPATH", "")])
    env["PICASSO_DROPIN_COUNT"] = str(count)
    r = subprocess.run([sys.executable, "-m", "pytest", "-v", "-s", "-p", "ref_dropin_plugin",
                        "-p", "no:cacheprovider", "--rootdir", REF, os.path.join(REF, "tests", suite)],
                       cwd=REF, env=env, capture_output=True, text=True, timeout=1800)
    out = r.stdout
    print(out[-3000:])
    failed = {ln.split()[1].split("::")[1] for ln in out.splitlines()
              if ln.startswith("FAILED tests/" + suite)}
    report = {}
    for ln in out.splitlines():
        if "ACCEPTANCE" in ln:
            tail = ln.split("ACCEPTANCE", 1)[1]
            report[int(tail.split()[0])] = tail.rsplit("; runtime", 1)[0].strip()
    want_failed, want_report = _recorded_outcome(suite)
    assert " error" not in out.splitlines()[-1], out[-5000:] + r.stderr[-3000:]
    assert failed == want_failed, (failed, want_failed, out[-5000:])
    # criteria 1 and 11 report wall times, 4 the host's thread counts (1, 2, nproc):
    # compare their verdicts only
    timed = (1, 4, 11)
    for k, v in want_report.items():
        got = report.get(k) or ""
        if k in timed:
            assert got.split(" - ")[0] == v.split(" - ")[0], (k, got, v)
        else:
            assert got == v, (k, got, v)
    served = int(count.read_text())
    print(f"{suite}: {served} conflict builds served by the CUDA builder; "
          f"failed as in the reference's own run: {sorted(failed)}")
    assert served > 0
