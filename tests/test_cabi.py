"""The C-ABI library loads and exports every entry point include/bal.h declares (CPU only)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "bal.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:bal_status|int64_t|int32_t|const char\*|void)\s+(bal_\w+)\s*\(", src, flags=re.M)
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
    assert pkg._lib.lib.bal_init(None, None, 0, None, None, ctypes.byref(h)) == -1
    assert not h.value


def test_init_rejects_bad_dist_without_gpu():
    """A bal_dist with rank outside [0, world) or half a host transport is rejected up front."""
    import numpy as np

    import paper_2407_00046_b200 as pkg
    import scenes
    sc = scenes.make_single_tet(0)
    for rank, world in ((2, 2), (-1, 2), (0, 0)):
        try:
            pkg.bal_init(sc, rank=rank, world=world)
            raise AssertionError("expected BalError")
        except pkg.BalError as e:
            assert e.status == -1
    assert np.all(pkg.bal_halo_pack(np.zeros(0, np.int32), np.zeros(3)) == np.zeros(0))
