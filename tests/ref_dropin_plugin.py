"""pytest plugin: the reference's own test suite with the B200 drop-in
installed (paper_1303_1651_b200.install). Test infrastructure, loaded by
tests/test_gpu_reference_suite.py as `-p ref_dropin_plugin`.

At configure time — before the reference's test modules are imported, so
their `from sparsemm.kernels import multiply_rowmajor` binds the GPU
version — the drop-in replaces the reference's entry points, each wrapped
with a call counter; the counts go to $SPMMM_DROPIN_REPORT at the end, so the
outer test can prove the GPU path served the suite.

Deselected (they test the reference's CPU internals, not the entry point):
TestRowMajor::test_result_never_exceeds_reservation swaps the reference's
CsrBuilder class and expects multiply_rowmajor to instantiate it
(test_kernels.py:92-108); the drop-in sizes C on the device and never calls
that class.
"""

from __future__ import annotations

import functools
import json
import os

DESELECT = ("test_kernels.py::TestRowMajor::test_result_never_exceeds_reservation",)
_counts: dict = {}
_handle = None


def _counting(name, fn):
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        _counts[name] = _counts.get(name, 0) + 1
        return fn(*args, **kwargs)
    return wrapper


def pytest_configure(config):
    global _handle
    import sparsemm

    import importlib

    import paper_1303_1651_b200 as drop_in

    inst = importlib.import_module("paper_1303_1651_b200.install")

    for name in list(inst._NAMES):
        inst._NAMES[name] = _counting(name, inst._NAMES[name])
    _handle = drop_in.install(sparsemm)
    import sparsemm.kernels as k

    assert k.multiply_rowmajor.__wrapped__.__module__ == "paper_1303_1651_b200.kernels"


def pytest_collection_modifyitems(config, items):
    keep, drop = [], []
    for it in items:
        (drop if any(it.nodeid.endswith(d) for d in DESELECT) else keep).append(it)
    if drop:
        config.hook.pytest_deselected(items=drop)
        items[:] = keep


def pytest_unconfigure(config):
    path = os.environ.get("SPMMM_DROPIN_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump({"calls": _counts}, f)
    if _handle is not None:
        _handle.uninstall()
