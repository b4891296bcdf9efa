"""CPU-side checks of the C-ABI boundary: the in-tree library builds/loads, exports every
function include/dgvv.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes as C
import os

import pytest

from paper_2506_14424_b200 import _abi as A


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(A.LIB_PATH):
        from paper_2506_14424_b200 import build
        build.build()
    return A.lib()


def test_exports_every_header_symbol(lib):
    names = A.header_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n


def test_header_has_no_torch_types():
    txt = open(A.HEADER).read()
    assert "torch" not in txt.lower().replace("pytorch", "")
    assert 'extern "C"' in txt


def test_fails_loudly_without_device(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = C.c_void_p()
    st = lib.dgvv_setup(None, 3, None, None, None, None, C.byref(h))
    assert st == A.ECUDA
    assert b"CUDA" in lib.dgvv_last_error()
    assert not h.value


def test_binding_is_marshalling_only():
    """The binding modules contain no numerical kernels of the method (no basis, metric,
    flux or law arithmetic): they never import the oracle and only pack arguments."""
    here = os.path.dirname(A.__file__)
    for f in ("_abi.py", "dgvv.py", "__init__.py"):
        src = open(os.path.join(here, f)).read()
        assert "oracle" not in src.replace("no arithmetic", "")
        for bad in ("einsum", "leggauss", "np.sin", "np.exp", "sqrt("):
            assert bad not in src, (f, bad)
