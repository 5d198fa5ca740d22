"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, and exports
every symbol include/cutfem.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "cutfem.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cutfem_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("cutfem_setup", "cutfem_apply", "cutfem_csr_apply", "cutfem_destroy", "cutfem_last_error"):
        assert s in syms


def test_library_builds_loads_and_exports_all_symbols():
    import paper_2404_07911_b200 as m
    path = m.build()
    lib = ctypes.CDLL(path)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) <= set(m._lib.EXPORTS) | {"cutfem_csr_nnz"}


def test_missing_library_fails_loudly(tmp_path):
    import paper_2404_07911_b200._lib as L
    with pytest.raises(RuntimeError, match="not built"):
        L.load(str(tmp_path / "nope.so"))


def test_sass_is_sm100a_and_atomic_free():
    """The hot-path kernels are compiled for sm_100a and contain no atomics (north_star)."""
    import shutil
    import subprocess
    import paper_2404_07911_b200 as m
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    out = subprocess.run(["cuobjdump", "-sass", m.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    funcs = re.split(r"\n\s*Function : ", out)
    hot = [f for f in funcs if re.match(r"_Z\d+k_(uncw|cut|tile|cell)", f)]
    # k_cut1<2,3>, k_cell<2,3>, k_cutp<4>, k_tile2<4>, k_uncw<4..9>, k_cut<5..9>
    assert len(hot) >= 17
    for f in hot:
        assert not re.search(r"\b(ATOM|ATOMS|ATOMG|RED)\b", f), f.split("\n")[0]
