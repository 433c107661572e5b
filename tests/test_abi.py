"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports
every symbol declared in include/vecattn.h, and rejects bad arguments
synchronously (no launch happens on an invalid call, so these run without a GPU).
"""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "vecattn.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2603_29494_b200 import _build
    _build.build()
    import paper_2603_29494_b200.vecattn as va
    return va.load()


def declared_functions():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"\b(vecattn_[a-z_]+)\s*\(", txt)))


def test_header_declares_expected_entry_points():
    names = declared_functions()
    for n in ["vecattn_select", "vecattn_sparse_fwd", "vecattn_dense_fwd", "vecattn_pool",
              "vecattn_select_workspace_bytes", "vecattn_sparse_workspace_bytes", "vecattn_status_string"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2603_29494_b200 import _build
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (vecattn_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    for n in declared_functions():
        getattr(lib, n)


def test_library_is_sm100a_code():
    from paper_2603_29494_b200 import _build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_tcgen05_and_tma_in_sass():
    # B200_PROFILING.md: tcgen05.mma -> UTC*MMA, tcgen05.ld/st -> LDTM/STTM, TMA -> UTMALDG
    from paper_2603_29494_b200 import _build
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _build.LIB], capture_output=True,
                          text=True).stdout
    assert re.search(r"UTC\w*MMA", sass)
    assert "LDTM" in sass and "STTM" in sass
    assert "UTMALDG" in sass
    assert not re.search(r"\bHMMA\b", sass)  # no legacy mma.sync path


def test_status_strings_and_version(lib):
    assert lib.vecattn_abi_version() == 1
    assert lib.vecattn_status_string(0) == b"ok"
    assert lib.vecattn_status_string(4) == b"workspace too small"


def _prob(va, **kw):
    d = dict(B=1, Hq=2, Hkv=1, N=1024, D=128, causal=0, scale=0.0)
    d.update(kw)
    return va.Problem(d["B"], d["Hq"], d["Hkv"], d["N"], d["D"], d["causal"], d["scale"])


def test_argument_errors_are_synchronous(lib):
    import paper_2603_29494_b200.vecattn as va
    fake = ctypes.c_void_p(0x10000)  # never dereferenced: validation fails first
    st = ctypes.c_void_p(0)
    pr = _prob(va)
    sp = va.SelectConfig(mode="alg1", pq=64, bk=16, gk=16, alpha=0.5).params()
    ws_bytes = lib.vecattn_select_workspace_bytes(ctypes.byref(pr), ctypes.byref(sp))
    assert ws_bytes > 0
    # workspace too small
    rc = lib.vecattn_select(ctypes.byref(pr), ctypes.byref(sp), fake, fake, fake, None, 0, fake, fake, 16, st)
    assert rc == 4
    # bad shapes / params
    for kw, code in [(dict(D=96), 2), (dict(N=0), 2), (dict(Hq=3, Hkv=2), 1), (dict(scale=-1.0), 1)]:
        p2 = _prob(va, **kw)
        assert lib.vecattn_select(ctypes.byref(p2), ctypes.byref(sp), fake, fake, fake, None, 0, fake, fake,
                                  ws_bytes, st) == code
    for cfg, code in [(va.SelectConfig(pq=32), 1), (va.SelectConfig(alpha=-1.0), 1),
                      (va.SelectConfig(bk=4), 1), (va.SelectConfig(bk=48), 1), (va.SelectConfig(bk=512), 1),
                      (va.SelectConfig(gk=0), 1),
                      (va.SelectConfig(mode="topk", topk=0, keep_frac=0.0), 1),
                      (va.SelectConfig(alpha=float("nan")), 1)]:
        s2 = cfg.params()
        assert lib.vecattn_select(ctypes.byref(pr), ctypes.byref(s2), fake, fake, fake, None, 0, fake, fake,
                                  ws_bytes, st) == code
    # NULL tensor pointers
    assert lib.vecattn_select(ctypes.byref(pr), ctypes.byref(sp), None, fake, fake, None, 0, fake, fake,
                              ws_bytes, st) == 1
    # unaligned pointer
    odd = ctypes.c_void_p(0x10008)
    assert lib.vecattn_dense_fwd(ctypes.byref(pr), odd, fake, fake, fake, None, fake, 256, st) == 2
    # sparse workspace sizing and error
    need = lib.vecattn_sparse_workspace_bytes(ctypes.byref(pr), 64, 1000)
    assert need >= 4000
    assert lib.vecattn_sparse_fwd(ctypes.byref(pr), 64, fake, fake, fake, fake, fake, 1000, fake, None, fake,
                                  need - 1, st) == 4
    assert lib.vecattn_sparse_fwd(ctypes.byref(pr), 48, fake, fake, fake, fake, fake, 1000, fake, None, fake,
                                  need, st) == 1


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2603_29494_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(//|#).*", "", txt).lower() or f == "synth.py", f
