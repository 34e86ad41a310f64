"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
every symbol include/tsnet.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tsnet.h")


def declared_symbols():
    src = open(HEADER).read()
    return re.findall(r"TSNET_API\s+[\w\s\*]+?\b(tsnet_\w+)\s*\(", src)


@pytest.fixture(scope="module")
def libpath():
    from paper_2509_19785_b200 import build
    return build.build()


def test_header_declares_the_survey_entry_points():
    syms = set(declared_symbols())
    for s in ("tsnet_build_P", "tsnet_grad", "tsnet_step", "tsnet_cost", "tsnet_workspace_bytes",
              "tsnet_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(libpath):
    L = ctypes.CDLL(libpath)
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    # and the binding's signature table covers exactly the header
    from paper_2509_19785_b200.tsnet import SIGNATURES
    assert sorted(n for n, _, _ in SIGNATURES) == sorted(set(declared_symbols()))


def test_library_is_sm100a(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_host_only_entry_points(libpath):
    from paper_2509_19785_b200 import tsnet as T
    assert T.tsnet_resolve_k(10 ** 6, 40.0) == 120
    assert T.tsnet_resolve_k(50, 40.0) == 49
    assert T.tsnet_resolve_k(1000, 2.5) == 8
    gp = T.GradParams()
    b1 = T.tsnet_workspace_bytes(1000, 100000, gp)
    b2 = T.tsnet_workspace_bytes(2000, 100000, gp)
    assert 0 < b1 < b2


def test_binding_refuses_cpu_tensors():
    import torch
    from paper_2509_19785_b200 import tsnet as T
    with pytest.raises(ValueError):
        T.CSR(torch.zeros(2, dtype=torch.int64), torch.zeros(0, dtype=torch.int32), torch.zeros(0))


def test_product_does_not_import_oracle():
    """The product path shares no code with oracle/ and never imports it."""
    pkg = os.path.join(ROOT, "paper_2509_19785_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
                assert "liboracle" not in txt and "oracle/" not in txt, f
