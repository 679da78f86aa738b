"""The C-ABI library loads and exports every entry point include/find_b200.h declares (CPU only)."""

import ctypes as C
import re

from conftest import ROOT


def declared_symbols():
    text = (ROOT / "include" / "find_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(find_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_header_symbols():
    from paper_1104_0623_b200 import _native

    lib = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 14
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) <= set(_native.EXPORTED)


def test_status_struct_layout():
    from paper_1104_0623_b200 import _native

    assert C.sizeof(_native.FindStatus) == 4 + 4 + 8 + 8 + 8 + 160


def test_ledger_key_names():
    from paper_1104_0623_b200 import _native

    lib = _native.lib()
    assert lib.find_ledger_key_name(0) == b"naive_dense"
    assert lib.find_ledger_key_name(1) == b"sigma_naive"


def test_solve_rejects_bad_arguments_without_gpu():
    import ctypes as C

    from paper_1104_0623_b200 import _native

    lib = _native.lib()
    st = _native.FindStatus()
    rc = lib.find_solve(None, None, None, 1, 1, 1, 1e-12, None, None, None, 0, None, C.byref(st))
    assert rc == _native.FIND_EINVAL


def test_dense_primitives_reject_bad_arguments_without_gpu():
    from paper_1104_0623_b200 import _native

    lib = _native.lib()
    st = _native.FindStatus()
    h = C.c_void_p()
    assert lib.find_dense_create(0, 1, C.byref(h), C.byref(st)) == _native.FIND_EINVAL
    assert lib.find_dense_create(8, 0, C.byref(h), C.byref(st)) == _native.FIND_EINVAL
    assert lib.find_dense_inverse(None, None, None, None, None, C.byref(st)) == _native.FIND_EINVAL
    rc = lib.find_zgemm_batched(1, 4, 4, 4, None, 4, 16, None, 4, 16, 0, None, 4, 16, 0, None, C.byref(st))
    assert rc == _native.FIND_EINVAL
    lib.find_dense_destroy(None)  # no-op
