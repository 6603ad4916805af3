"""The C-ABI library loads and exports every entry point include/bal.h declares (CPU only)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "bal.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:bal_status|int64_t|const char\*|void)\s+(bal_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = header_functions()
    for required in ("bal_init", "bal_step", "bal_assemble", "bal_spmv", "bal_pcg", "bal_destroy", "bal_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    import paper_2407_00046_b200 as pkg
    lib = ctypes.CDLL(pkg.lib_path)
    for name in header_functions():
        assert hasattr(lib, name), name
    assert set(header_functions()) <= set(pkg._lib.EXPORTS)


def test_init_error_paths_without_gpu():
    """bal_init validates its arguments before touching the device."""
    import paper_2407_00046_b200 as pkg
    h = ctypes.c_void_p()
    assert pkg._lib.lib.bal_init(None, None, 0, None, 0, ctypes.byref(h)) == -1
    assert not h.value
