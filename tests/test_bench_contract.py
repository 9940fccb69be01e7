"""The bench.py JSON line the driver parses: the reference arm runs on the CPU
here; our arm needs the GPU (marked)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import have_gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "3"])
    assert BASE_KEYS <= set(d), set(d) ^ BASE_KEYS
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["config"]["workload"].startswith("C1")
    # the reference arm never maps the product library (its operands come
    # from oracle/gen_oracle.c)
    assert not any("libspmmm" in p for p in d["native_libs_mapped"]), d["native_libs_mapped"]
    assert "oracle/liboracle.so" in d["native_libs_mapped"]


@pytest.mark.gpu
@pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")
def test_our_arm_line():
    d = _run(["--config", "C1", "--steps", "3", "--warmup", "3", "--cpu-budget", "0.5"])
    assert BASE_KEYS <= set(d), set(d) ^ BASE_KEYS
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= d["steps"]  # (C1: one count-free k_fused per product)
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    cb = d["cpu_baseline"]
    assert cb["cores"] == 1 and cb["value"] > 0 and cb["kind"] == "port"
    assert d["e2e_pageable"]["value"] > 0
    assert "paper_1303_1651_b200/libspmmm.so" in d["native_libs_mapped"]
    # both arms print the same config for the same workload
    ref = _run(["--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "3"])
    assert ref["config"] == d["config"]


@pytest.mark.gpu
@pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")
def test_multi_rank_line_functional():
    """`--gpus 2` launches two ranks itself (torch.distributed.run). With one
    GPU the ranks share it over gloo: a functional run of the N>1 path."""
    d = _run(["--gpus", "2", "--backend", "gloo", "--config", "C3", "--steps", "3",
              "--warmup", "3", "--e2e-steps", "2"], timeout=900)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "strong"
    assert len(d["rank_products"]) == 2 and sum(d["rank_products"]) == d["config"]["products"]
    assert d["balance"] < 1.01
    assert d["e2e"]["value"] > 0 and d["gather_ms"] > 0 and d["b_allgather_ms"] > 0
    assert d["gpu_launches"] >= 2 * 2 * d["steps"]
