"""C-ABI library checks that need no GPU: it loads, exports every symbol include/pi.h declares,
and validates configurations on the host (-m "not gpu")."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2406_16091_b200 import build
    build.build()
    from paper_2406_16091_b200 import _lib
    return _lib.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "pi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pi_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert "pi_create" in syms and "pi_interact" in syms and "pi_step" in syms
    for s in syms:
        assert hasattr(lib, s), f"libpi.so does not export {s}"


def test_only_c_abi_exported():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2406_16091_b200", "libpi.so")],
                         capture_output=True, text=True).stdout
    names = [l.split()[-1] for l in out.splitlines() if l.strip()]
    ours = [n for n in names if n.startswith("pi_")]
    assert set(ours) == set(declared_symbols())


def test_binding_matches_header(lib):
    from paper_2406_16091_b200 import _lib
    assert set(_lib.SIGNATURES) == set(declared_symbols())
    assert lib.pi_abi_version() == 1


def _cfg(**kw):
    from paper_2406_16091_b200 import _lib
    c = _lib.pi_config()
    d = dict(dims=(16, 16, 16), w=1 / 16, rc=1 / 16, cap=4096, nranks=1, rank=0)
    d.update(kw)
    for a in range(3):
        c.dims[a] = d["dims"][a]
    c.cell_width = d["w"]
    c.r_c = d["rc"]
    c.capacity = d["cap"]
    c.nranks = d["nranks"]
    c.rank = d["rank"]
    return c


def test_workspace_bytes_validation(lib):
    ok = lib.pi_workspace_bytes(ctypes.byref(_cfg()))
    assert ok > 4096 * 16
    # grows with capacity and with the grid
    assert lib.pi_workspace_bytes(ctypes.byref(_cfg(cap=8192))) > ok
    assert lib.pi_workspace_bytes(ctypes.byref(_cfg(dims=(32, 16, 16)))) > ok
    # invalid: r_c > cell width, dims <= 0, nranks not dividing dims[0]
    assert lib.pi_workspace_bytes(ctypes.byref(_cfg(rc=0.1))) == 0
    assert lib.pi_workspace_bytes(ctypes.byref(_cfg(dims=(0, 16, 16)))) == 0
    assert lib.pi_workspace_bytes(ctypes.byref(_cfg(nranks=3, dims=(16, 16, 16)))) == 0
    assert lib.pi_workspace_bytes(None) == 0
    # x_subcells: 0 (default) or a power of two <= 16; finer X order needs more fine offsets
    c1, c8 = _cfg(), _cfg()
    c1.x_subcells, c8.x_subcells = 1, 8
    assert 0 < lib.pi_workspace_bytes(ctypes.byref(c1)) < lib.pi_workspace_bytes(ctypes.byref(c8))
    for bad in (3, 32, -1):
        c = _cfg()
        c.x_subcells = bad
        assert lib.pi_workspace_bytes(ctypes.byref(c)) == 0
    # the fine (X sub-cell) index is 32-bit in the kernels: cells x x_subcells must stay < 2^31
    # (ADVICE r01); 1024^3 cells with 4 sub-cells is refused, 512^3 with 8 accepted
    big = _cfg(dims=(1024, 1024, 1024))
    assert lib.pi_workspace_bytes(ctypes.byref(big)) == 0
    ok8 = _cfg(dims=(512, 512, 512))
    ok8.x_subcells = 8
    assert lib.pi_workspace_bytes(ctypes.byref(ok8)) > 0
    ok8.x_subcells = 16
    assert lib.pi_workspace_bytes(ctypes.byref(ok8)) == 0
    # every kernel id 0..5 (the cost sweep's LOWFLOP / HIGHFLOP included), nothing above
    for k in range(6):
        c = _cfg()
        c.kernel = k
        assert lib.pi_workspace_bytes(ctypes.byref(c)) > 0
    c = _cfg()
    c.kernel = 6
    assert lib.pi_workspace_bytes(ctypes.byref(c)) == 0


def test_create_rejects_bad_arguments_without_gpu(lib):
    from paper_2406_16091_b200 import _lib
    h = ctypes.c_void_p()
    c = _cfg(rc=0.5)
    assert lib.pi_create(ctypes.byref(c), None, 0, ctypes.byref(h)) == _lib.PI_EINVAL
    c = _cfg()
    # workspace too small / NULL
    assert lib.pi_create(ctypes.byref(c), None, 10, ctypes.byref(h)) == _lib.PI_EINVAL
    assert lib.pi_create(ctypes.byref(c), ctypes.c_void_p(256), 10, None) == _lib.PI_EINVAL
    # calls on a NULL context
    assert lib.pi_bin(None, 0, None, None, None, None, None) == _lib.PI_EINVAL
    assert lib.pi_interact(None, 0, None, None, None, None) == _lib.PI_EINVAL
    assert lib.pi_step(None, 0, ctypes.c_float(0.0)) == _lib.PI_EINVAL
    assert lib.pi_last_error(None) == b"NULL context"


def test_product_does_not_import_oracle():
    """The product path never touches oracle/ (it is test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2406_16091_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("oracle/", ""), f
