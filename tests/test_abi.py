"""The C-ABI library loads on CPU and exports every entry point include/samu.h declares
(no compute calls without a GPU); the binding fails loudly without a device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "samu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(samu_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libsamu():
    import __graft_entry__  # noqa: F401
    from paper_2503_16893_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_boundary():
    fns = declared_functions()
    for need in ("samu_ecdf_load", "samu_sample_lengths", "samu_simulate_batch", "samu_plan_greedy"):
        assert need in fns


def test_library_exports_every_declared_symbol(libsamu):
    for fn in declared_functions():
        assert hasattr(libsamu, fn), f"libsamu.so does not export {fn}"


def test_binding_names_match_abi():
    from paper_2503_16893_b200 import binding
    assert set(binding.EXPORTED) == set(declared_functions())


def test_struct_layouts():
    from paper_2503_16893_b200 import binding as B
    assert ctypes.sizeof(B.samu_trial_rec) == 40
    assert ctypes.sizeof(B.samu_request) == 20
    assert ctypes.sizeof(B.samu_candidate) == 24


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2503_16893_b200 import Samu
    with pytest.raises(RuntimeError):
        Samu(0)
