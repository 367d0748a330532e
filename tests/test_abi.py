"""CPU checks of the C-ABI boundary: libevospec.so builds for sm_100a, loads,
and exports every entry point include/evospec.h declares (no compute calls)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2605_27390_b200 import _build
    return _build.build()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "evospec.h")).read()
    return sorted(set(re.findall(r"\b(evospec_[a-z_]+)\s*\(", hdr)))


def test_header_declares_the_three_calls():
    syms = declared_symbols()
    for s in ["evospec_build_subset", "evospec_subset_logits_topk", "evospec_merge_shards"]:
        assert s in syms


def test_exports_every_declared_symbol(libpath):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath]).decode()
    exported = set(re.findall(r" T (evospec_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    # nothing but the C ABI leaks out (hidden visibility for everything else)
    assert all(s.startswith("evospec_") for s in re.findall(r" T (\w+)", out) if not s.startswith("_"))


def test_binding_loads_and_matches_header(libpath):
    import paper_2605_27390_b200 as es
    L = es.lib()
    assert set(es.EXPORTED) == set(declared_symbols())
    for s in es.EXPORTED:
        assert hasattr(L, s)
    assert "sm_100a" in es.version()
    assert es.lib().evospec_status_string(2).decode() == "input error"


def test_sass_is_sm100a(libpath):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath]).decode()
    assert "sm_100a" in out


def test_no_gpu_context_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2605_27390_b200 as es
    with pytest.raises(RuntimeError):
        es.Context(V=16, d=8, w_dtype=torch.float32, h_dtype=torch.float32, max_subset=16, max_rows=1)


def test_struct_layouts_match_header():
    import ctypes as C
    import paper_2605_27390_b200 as es
    assert C.sizeof(es.Config) == 13 * 4
    assert C.sizeof(es.BuildParams) == 6 * 4
