"""pytest plugin: run the reference's own test files with `ringmix` routed through
libringmix_b200 (integration/ringmix_b200.py).

  PYTHONPATH=baseline/_ref:integration python -m pytest -p pytest_ringmix_b200 \
      baseline/_ref/ringmix_ref_tests/test_mixing.py ...

XFAIL may list tests that compare `apply_mixing(W, T)` bit for bit with numpy's `W @ T`
where our FMA chain and OpenBLAS's kernel for that matrix shape could round differently
(OpenBLAS's small-matrix and remainder kernels are an implementation-defined choice of the
BLAS).  It is empty: with numpy 2.3.5 / OpenBLAS 0.3.30 every one of the
reference's tests passes through the binding (test_mixing.py's bitwise W @ T check
included).  The terminal summary prints how many calls went through the GPU."""

from __future__ import annotations

import os

import pytest

XFAIL: dict[str, str] = {}


def pytest_configure(config):
    import ringmix
    import ringmix_b200

    ringmix_b200.install(ringmix)
    config._ringmix_b200 = ringmix_b200


def pytest_collection_modifyitems(config, items):
    for item in items:
        key = f"{os.path.basename(str(item.fspath))}::{item.name}"
        if key in XFAIL:
            item.add_marker(pytest.mark.xfail(reason=XFAIL[key], strict=False))


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    calls = config._ringmix_b200.CALLS
    terminalreporter.write_sep("-", "libringmix_b200 binding")
    terminalreporter.write_line("RINGMIX_B200_CALLS " + " ".join(f"{k}={v}" for k, v in
                                                                 calls.items()))
