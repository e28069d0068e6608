"""CPU-side checks of the boundary: libriki.so builds, loads and exports every symbol that
include/riki.h declares; without a usable device the calls fail loudly (no fallback)."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import paper_2001_06770_b200 as P
from paper_2001_06770_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_builds_and_exports_all_declared_symbols():
    B.build()
    lib = P.load()
    declared = P.declared_symbols()
    assert len(declared) >= 20
    out = subprocess.check_output(["nm", "-D", "--defined-only", P.riki.LIB_PATH], text=True)
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(declared) <= exported, set(declared) - exported
    for s in declared:
        assert hasattr(lib, s)
    assert lib.riki_version().startswith(b"riki-b200")


def test_library_is_sm100a_only():
    out = subprocess.check_output(["cuobjdump", "--list-elf", P.riki.LIB_PATH], text=True)
    assert "sm_100a" in out


def test_no_oracle_in_product_path():
    # the product package must not import, link or execute oracle/
    pkg = os.path.join(ROOT, "paper_2001_06770_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "riki_oracle" not in txt, f
    out = subprocess.check_output(["nm", "-D", P.riki.LIB_PATH], text=True)
    assert "orc_" not in out


def test_params_default():
    lib = P.load()
    p = P.riki.Params()
    lib.riki_params_default(C.byref(p))
    assert p.gamma == 0.5 and p.beam_w == 0 and p.beam_mode == 0 and p.ptc_mode == 0 and p.early_term == 0


def test_fails_loudly_without_device():
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises(P.RikiError) as e:
        P.Graph(3, np.array([0, 1], np.uint32), np.array([1, 0], np.uint32), None,
                np.array([0, 1], np.uint64), np.array([0], np.uint32))
    assert e.value.name == "RIKI_ECUDA"


def _build_c_client(tmp_path):
    """tests/c/abi_smoke.c compiled and linked against libriki.so with the plain C compiler and
    include/riki.h only (no C++ or CUDA headers): the boundary is a C ABI."""
    B.build()
    exe = str(tmp_path / "abi_smoke")
    libdir = os.path.dirname(P.riki.LIB_PATH)
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-o", exe, "-L", libdir, "-lriki",
                           "-Wl,-rpath," + libdir])
    return exe


def test_plain_c_client_compiles_and_links(tmp_path):
    exe = _build_c_client(tmp_path)
    assert os.path.exists(exe)
    out = subprocess.check_output(["nm", "-u", exe], text=True)
    assert "riki_rpq_search" in out and "riki_load_graph" in out


@pytest.mark.gpu
def test_plain_c_client_runs(tmp_path):
    exe = _build_c_client(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ABI_SMOKE_OK" in r.stdout
