"""B200-native matrix-free SIPG viscous-operator hot path of arXiv 2506.14424.

The product is the C-ABI library libdgvv.so (include/dgvv.h; CUDA kernels for sm_100a in
csrc/).  This package holds its build script and a thin ctypes binding (argument
marshalling only).  There is no CPU fallback: without the built library or a CUDA device
the calls raise.
"""
from . import _abi  # noqa: F401
from ._abi import (BC_DIRICHLET, BC_NEUMANN, FORM_DIVERGENCE, FORM_LAPLACE, OP_POISSON,  # noqa: F401
                   OP_VISCOUS, DgvvError)


def Context(*args, **kwargs):
    from .dgvv import Context as _C
    return _C(*args, **kwargs)
