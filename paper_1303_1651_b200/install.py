"""Drop-in installation into the reference package.

The reference's plug points are its module globals (test_kernels.py:98-107
swaps `sparsemm.kernels.CsrBuilder` the same way). `multiply_mixed` looks
`multiply_rowmajor` up in `sparsemm.kernels` (kernels.py:428-429, 436-437)
and the harness binds its own copy at import (bench.py:27-34), so both
names are replaced, plus the package re-export (__init__.py:304-315):

    import sparsemm, paper_1303_1651_b200
    handle = paper_1303_1651_b200.install(sparsemm)
    ...                      # every reference caller now runs on the B200
    handle.uninstall()
"""

from __future__ import annotations

import importlib
import sys

from .kernels import multiply_rowmajor

_TARGETS = ("kernels", "bench", "")


class Installation:
    def __init__(self, saved):
        self._saved = saved

    def uninstall(self):
        for mod, old in self._saved:
            mod.multiply_rowmajor = old
        self._saved = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.uninstall()


def install(package=None) -> Installation:
    """Point the reference's `multiply_rowmajor` names at the GPU version."""
    if package is None:
        package = importlib.import_module("sparsemm")
    name = package.__name__
    saved = []
    for sub in _TARGETS:
        modname = f"{name}.{sub}" if sub else name
        mod = sys.modules.get(modname)
        if mod is None and sub:
            try:
                mod = importlib.import_module(modname)
            except ImportError:
                continue
        if mod is not None and hasattr(mod, "multiply_rowmajor"):
            saved.append((mod, mod.multiply_rowmajor))
            mod.multiply_rowmajor = multiply_rowmajor
    return Installation(saved)
