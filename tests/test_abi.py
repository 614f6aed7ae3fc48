"""CPU-side checks of the C ABI: the library builds/loads and exports every
symbol include/pot3d.h declares; host-side logic of the binding."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    src = (ROOT / "include" / "pot3d.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pot3d_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_boundary():
    syms = declared_symbols()
    for s in ["pot3d_setup", "pot3d_solve", "pot3d_field", "pot3d_destroy", "pot3d_last_error"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1709_01126_b200 import build

    lib = build.build()
    L = ctypes.CDLL(str(lib))
    for s in declared_symbols():
        assert hasattr(L, s), s


def test_binding_export_list_matches_header():
    from paper_1709_01126_b200 import pot3d

    assert sorted(pot3d.EXPORTS) == declared_symbols()


def test_no_cuda_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import synth
    from paper_1709_01126_b200 import Pot3d

    rf, tf, pf = synth.grid(4, 6, 8)
    with pytest.raises(RuntimeError):
        Pot3d(rf, tf, pf, synth.br0_map(tf, pf, 0))


def test_setup_error_without_device_is_reported():
    """Invalid arguments are rejected before any device work."""
    from paper_1709_01126_b200 import pot3d

    L = pot3d.library()
    import numpy as np

    rf = np.linspace(1, 2.5, 2)  # nr = 1 < 2
    tf = np.linspace(0, np.pi, 5)
    pf = np.linspace(0, 2 * np.pi, 9)
    g = pot3d._Grid(1, 4, 8, rf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                    tf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                    pf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    br = np.zeros((8, 4))
    ctx = ctypes.c_void_p()
    rc = L.pot3d_setup(ctypes.byref(g), ctypes.c_void_p(br.ctypes.data), 0, 1, None,
                       ctypes.byref(ctx))
    assert rc == -1
    assert b">= 2" in L.pot3d_last_error(None)
