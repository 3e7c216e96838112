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


@pytest.mark.parametrize("suite", ["test_conflict.py", "test_acceptance.py", "test_driver.py"])
def test_reference_suite_passes_unchanged(suite, tmp_path):
    count = tmp_path / "count"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REF, "src"), os.path.join(ROOT, "tests"), ROOT,
                                         env.get("PYTHONPATH", "")])
    env["PICASSO_DROPIN_COUNT"] = str(count)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "ref_dropin_plugin",
                        "-p", "no:cacheprovider", "--rootdir", REF, os.path.join(REF, "tests", suite)],
                       cwd=REF, env=env, capture_output=True, text=True, timeout=1800)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-5000:] + r.stderr[-3000:]
    served = int(count.read_text())
    print(f"{suite}: {served} conflict builds served by the CUDA builder")
    assert served > 0
