"""C-ABI boundary checks (CPU): libodc.so loads without a GPU, exports every
function include/odc/odc.h declares, the Python binding covers exactly that
set, and the layout entry point matches the reference's shard map."""
import os
import re
import subprocess

import pytest

from conftest import ROOT
from oracle import odc_oracle as O
from paper_2601_19362_b200 import _lib
from paper_2601_19362_b200 import errors as E
from paper_2601_19362_b200.primitives import shard_range

HEADER = os.path.join(ROOT, "include", "odc", "odc.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^\s*[A-Za-z_][\w\s\*]*?\b(odc_\w+)\s*\(", src, flags=re.M))


def test_header_declares_the_api():
    d = declared()
    for must in ("odc_fetch", "odc_push", "odc_push_slice", "odc_minibatch_end", "odc_adam_step", "odc_shard_range",
                 "odc_fabric_gather", "odc_fabric_scatter_accumulate", "odc_fabric_finalize", "odc_plan_json"):
        assert must in d


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(odc_\w+)$", out, flags=re.M))
    missing = declared() - exported
    assert not missing, missing


def test_binding_covers_header():
    assert set(_lib.SIGNATURES) == declared()
    L = _lib.lib()  # loads on a GPU-less host
    for name in _lib.SIGNATURES:
        assert getattr(L, name)


def test_shard_range_matches_reference_layout():
    for M in list(range(1, 40)) + [46797824, 218112000, 275268608]:
        for N in (1, 2, 3, 4, 5, 7, 8, 16):
            for r in range(N):
                assert shard_range(M, N, r) == O.shard_range(M, N, r)
    assert [shard_range(5, 4, r) for r in range(4)] == [(0, 2), (2, 2), (4, 1), (5, 0)]
    with pytest.raises(E.ParamError):
        shard_range(0, 2, 0)
    with pytest.raises(E.ParamError):
        shard_range(10, 2, 2)


def test_no_oracle_in_product():
    pkg = os.path.join(ROOT, "paper_2601_19362_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".hpp", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "from oracle" not in txt and "import oracle" not in txt and "odcref" not in txt, f
