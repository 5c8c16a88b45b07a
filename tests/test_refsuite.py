"""The reference's OWN unit tests, compiled unmodified from
/root/reference/proj/tests against our drop-in headers (include/odcsim) and
libodc.so by tests/refsuite/Makefile (doctest replaced by a small shim).

The binaries are built here (build() / this test) and travel to the GPU box;
nothing reads /root/reference at run time there."""
import os
import subprocess

import pytest

from conftest import ROOT

SUITE = os.path.join(ROOT, "tests", "refsuite")
BUILD = os.path.join(SUITE, "_build")


def _binary(name):
    path = os.path.join(BUILD, name)
    if not os.path.exists(path) and os.path.isdir("/root/reference/proj/tests"):
        subprocess.run(["make", "-C", SUITE, f"_build/{name}"], check=True, capture_output=True)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (no /root/reference here and no prebuilt copy)")
    return path


def _run(path):
    p = subprocess.run([path], capture_output=True, text=True, timeout=600,
                       env={**os.environ, "ODC_SIM_LOG": "quiet"})
    tail = (p.stdout + p.stderr)[-3000:]
    assert p.returncode == 0, tail
    assert "failed: 0 |" in p.stdout, tail
    return p.stdout


def test_reference_partition_tests_pass_on_b200_lb():
    out = _run(_binary("ref_partition_tests"))
    assert "test cases: 23" in out


@pytest.mark.gpu
def test_reference_primitives_tests_pass_on_gpu_fabric():
    out = _run(_binary("ref_primitives_tests"))
    assert "test cases: 13" in out or "test cases: 14" in out


def test_reference_workload_tests_pass_on_facade():
    """tests/test_workload.cpp (generators, length files, scaling, summarize,
    dist-spec strings) against include/odcsim/workload.hpp + libodc.so."""
    out = _run(_binary("ref_workload_tests"))
    assert "test cases: 16" in out


def test_reference_cost_model_tests_pass_on_facade():
    out = _run(_binary("ref_cost_model_tests"))
    assert "test cases: 9" in out
