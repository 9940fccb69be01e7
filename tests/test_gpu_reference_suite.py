"""The reference's own tests, run through the drop-in on the B200.

`baseline/_ref/` holds the unmodified reference package (pip-installed from
/root/reference/pkg with the contract's offline command) and a copy of its
tests (pkg/tests); it is git-ignored and travels to the GPU box with the
repo. tests/ref_dropin_plugin.py installs paper_1303_1651_b200 into the
reference's `sparsemm` before the test modules load, so every
multiply_rowmajor / multiply_colmajor / multiply_mixed the suite calls runs
the CUDA path; the plugin's call counts prove it. Anchors:
pkg/tests/test_kernels.py:41-351, pkg/tests/test_acceptance.py:72-105."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, have_gpu

REF = os.path.join(ROOT, "baseline", "_ref")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device"),
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")),
                                 reason="baseline/_ref (the installed reference + its tests) absent")]


@pytest.mark.parametrize("files", [("test_kernels.py",), ("test_acceptance.py",),
                                   ("test_bench.py", "test_formats.py", "test_perfmodel.py")])
def test_reference_suite_through_drop_in(files, tmp_path):
    report = str(tmp_path / "calls.json")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests")]),
               SPMMM_DROPIN_REPORT=report)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        "-p", "ref_dropin_plugin", "--rootdir", os.path.join(REF, "tests"),
                        *[os.path.join(REF, "tests", f) for f in files]],
                       env=env, capture_output=True, text=True, timeout=1500, cwd=tmp_path)
    tail = r.stdout[-4000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    calls = json.load(open(report))["calls"]
    assert calls.get("multiply_rowmajor", 0) > 0, calls
    if files[0] in ("test_kernels.py", "test_acceptance.py"):
        assert calls.get("multiply_colmajor", 0) > 0 and calls.get("multiply_mixed", 0) > 0, calls
    print(files, calls, tail.strip().splitlines()[-1])
