"""pytest plugin: run the reference's own test suite with the B200 builder installed.

``python -m pytest -p ref_dropin_plugin <reference tests>`` (tests/ on PYTHONPATH, the
reference's ``src`` first on it) swaps ``palettecolor.conflict.build`` for this package's
CUDA builder before any test runs (``install_into``, the integration a maintainer adds), and
counts how many builds the CUDA path served (written to $PICASSO_DROPIN_COUNT at exit), so the
caller can check the suite really went through the GPU.  Test infrastructure only.
"""
import os

_calls = {"gpu": 0}


def pytest_configure(config):
    import palettecolor

    import paper_2401_06713_b200 as b200
    from paper_2401_06713_b200 import conflict as b200_conflict

    real = b200_conflict.build

    def counted(view, lists, **kw):
        _calls["gpu"] += 1
        return real(view, lists, **kw)

    b200_conflict.build = counted
    b200.build = counted
    # install_into binds the package-level build at call time
    b200.install_into(palettecolor)
    routed = palettecolor.conflict.build
    assert routed is not palettecolor.conflict._reference_build


def pytest_unconfigure(config):
    path = os.environ.get("PICASSO_DROPIN_COUNT")
    if path:
        with open(path, "w") as f:
            f.write(str(_calls["gpu"]))
