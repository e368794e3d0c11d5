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


def test_struct_layouts(tmp_path):
    # every struct the binding marshals has the C compiler's size (and a few pinned ones)
    import subprocess
    from paper_2503_16893_b200 import binding as B
    assert ctypes.sizeof(B.samu_trial_rec) == 40
    assert ctypes.sizeof(B.samu_request) == 20
    assert ctypes.sizeof(B.samu_candidate) == 24
    names = ["samu_model_spec", "samu_engine_cfg", "samu_request", "samu_trial_rec", "samu_candidate",
             "samu_cand_summary", "samu_plan_stage", "samu_plan", "samu_plan_opts", "samu_replay_stage",
             "samu_replay"]
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "samu.h"\nint main(void){\n' +
                   "".join(f'printf("%zu\\n", sizeof({n}));\n' for n in names) + "return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    sizes = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    for n, sz in zip(names, sizes):
        assert ctypes.sizeof(getattr(B, n)) == sz, n


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2503_16893_b200 import Samu
    with pytest.raises(RuntimeError):
        Samu(0)


def test_product_and_oracle_share_nothing():
    # the CUDA path and the oracle are independent: no imports, includes or links either way
    import re
    pkg = os.path.join(ROOT, "paper_2503_16893_b200")
    for d, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(d, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
                assert not re.search(r'#include\s*[<"][^>"]*oracle', src), f
                assert "liboracle" not in src, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".cpp", ".h")):
            src = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(import|from)\s+paper_2503_16893_b200\b", src, re.M), f
            assert "libsamu" not in src, f
            assert not re.search(r'#include\s*[<"][^>"]*samu', src), f
