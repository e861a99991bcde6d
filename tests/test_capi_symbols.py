"""The C-ABI library builds, loads without a GPU and exports every symbol include/*.h declares."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sinkhorn_nfft.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_ ]*\**\s+\**([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2201_07524_b200 import build
    path = build.build()
    return ctypes.CDLL(path), path


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ["sinkhorn_init", "fastsum_plan", "fastsum_apply", "sinkhorn_run", "sinkhorn_divergence",
                     "sinkhorn_finalize", "fastsum_plan_destroy", "sk_last_error"]:
        assert required in names, names


def test_library_exports_every_declared_symbol(lib):
    L, path = lib
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    for n in declared_functions():
        assert re.search(rf"\bT {n}$", out, flags=re.M), n


def test_library_is_sm100a_only(lib):
    _, path = lib
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_binding_loads_and_matches_header():
    from paper_2201_07524_b200 import capi
    assert set(capi.EXPORTED) >= set(declared_functions()) - {"sk_last_error"}
    # no compute without a GPU: only error paths that do not touch the device
    assert capi._lib.sinkhorn_run(None, None, None, 1, 0.0, 0, None, None, None) == capi.SK_EINVAL
    assert b"NULL plan" in capi._lib.sk_last_error()


def test_missing_library_fails_loudly():
    """The product path has no CPU fallback: without the CUDA library the binding refuses to import."""
    import sys
    env = dict(os.environ, SK_LIB_PATH="/nonexistent/libsk_nfft.so")
    r = subprocess.run([sys.executable, "-c", "import paper_2201_07524_b200.capi"], cwd=ROOT, env=env,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "ImportError" in r.stderr
