"""ctypes mirror of include/dgvv.h (argument marshalling only; no arithmetic of the method).

Loads the in-tree paper_2506_14424_b200/lib/libdgvv.so and fails loudly when it is missing:
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DGVV_LIB_PATH") or os.path.join(HERE, "lib", "libdgvv.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "dgvv.h")

STATUS = {0: "DGVV_OK", 1: "DGVV_EINVAL", 2: "DGVV_EDOMAIN", 3: "DGVV_ENOMEM", 4: "DGVV_ECUDA",
          5: "DGVV_ENCCL", 6: "DGVV_ESTATE", 7: "DGVV_EUNSUPPORTED"}
OK, EINVAL, EDOMAIN, ENOMEM, ECUDA, ENCCL, ESTATE, EUNSUPPORTED = range(8)
BC_DIRICHLET, BC_NEUMANN = 1, 2
LAW_CONST, LAW_SIN3, LAW_EXP, LAW_CARREAU = 0, 1, 2, 3
OP_VISCOUS, OP_POISSON, OP_PENALTY = 0, 1, 2
PRECOND_NONE, PRECOND_JACOBI, PRECOND_VCYCLE, PRECOND_VCYCLE_FP32 = 0, 1, 2, 3
FORM_DIVERGENCE, FORM_LAPLACE = 0, 1
GHOST_VISCOUS, GHOST_POISSON, GHOST_ULIN, GHOST_TRANSPORT = 0, 1, 2, 3


class DgvvLaw(C.Structure):
    _fields_ = [("kind", C.c_int32), ("p", C.c_double * 8)]


class DgvvMesh(C.Structure):
    _fields_ = [("n_cells", C.c_int32), ("n_ghost", C.c_int32), ("first_global_cell", C.c_int64),
                ("neighbor", C.POINTER(C.c_int64)), ("ghost_global_id", C.POINTER(C.c_int64)),
                ("ghost_owner", C.POINTER(C.c_int32)), ("map_degree", C.c_int32),
                ("nodes", C.POINTER(C.c_double))]


class DgvvOptions(C.Structure):
    _fields_ = [("n_levels", C.c_int32), ("degrees", C.POINTER(C.c_int32)), ("ip_factor", C.c_double),
                ("formulation", C.c_int32), ("nccl_comm", C.c_void_p)]


class DgvvError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None

VP, D, I32, I64 = C.c_void_p, C.c_double, C.c_int32, C.c_int64
PD = C.POINTER(C.c_double)
_SIGS = {
    "dgvv_setup": [C.POINTER(DgvvMesh), I32, C.POINTER(DgvvLaw), C.POINTER(DgvvLaw), C.POINTER(DgvvOptions), VP, C.POINTER(VP)],
    "dgvv_update_viscosity": [VP, VP, VP],
    "dgvv_apply_viscous": [VP, I32, VP, VP, VP],
    "dgvv_apply_viscous_host": [VP, I32, VP, VP, VP],
    "dgvv_set_mass": [VP, I32, D],
    "dgvv_vcycle_fp32": [VP, I32, VP, VP, PD, VP],
    "dgvv_set_penalty_parameters": [VP, PD, PD],
    "dgvv_apply_penalty": [VP, VP, VP, VP],
    "dgvv_apply_penalty_level": [VP, I32, VP, VP, VP],
    "dgvv_cg_solve": [VP, I32, VP, VP, D, I32, I32, PD, C.POINTER(I32), PD, VP],
    "dgvv_set_transport": [VP, VP, VP],
    "dgvv_set_coarse_context": [VP, VP, C.POINTER(I32), C.POINTER(C.c_int8)],
    "dgvv_prolongate_h": [VP, I32, VP, VP, D, VP],
    "dgvv_restrict_h": [VP, I32, VP, VP, D, VP],
    "dgvv_setup_coarse_solver": [VP, I32, C.POINTER(I32)],
    "dgvv_set_continuous_level": [VP, I32],
    "dgvv_continuous_level_info": [VP, C.POINTER(I32), C.POINTER(I32)],
    "dgvv_apply_continuous": [VP, I32, VP, VP, VP],
    "dgvv_embed_continuous": [VP, I32, I32, VP, VP, D, VP],
    "dgvv_apply_convective": [VP, VP, VP, VP],
    "dgvv_apply_oseen": [VP, D, VP, VP, VP],
    "dgvv_gmres_solve": [VP, D, VP, VP, D, I32, I32, I32, PD, C.POINTER(I32), PD, VP],
    "dgvv_apply_linearized_viscous": [VP, VP, VP, VP],
    "dgvv_apply_poisson": [VP, I32, VP, VP, VP],
    "dgvv_inverse_diagonal": [VP, I32, I32, VP, VP],
    "dgvv_estimate_lambda_max": [VP, I32, I32, I32, VP, PD, VP],
    "dgvv_chebyshev_smooth": [VP, I32, I32, VP, VP, I32, D, D, I32, VP, VP],
    "dgvv_prolongate": [VP, I32, I32, VP, VP, D, VP],
    "dgvv_restrict": [VP, I32, I32, VP, VP, D, VP],
    "dgvv_vcycle": [VP, I32, VP, VP, PD, VP],
    "dgvv_dot": [VP, I32, I32, VP, VP, PD, VP],
    "dgvv_sizes": [VP, I32, C.POINTER(I64), C.POINTER(I64)],
    "dgvv_coefficient_range": [VP, I32, I32, PD, PD],
    "dgvv_ghost_layout": [VP, C.POINTER(I32), C.POINTER(I32), C.POINTER(I32), C.POINTER(I32)],
    "dgvv_pack_ghosts": [VP, I32, I32, VP, VP, VP],
    "dgvv_ghost_buffer": [VP, I32, I32, C.POINTER(VP)],
    "dgvv_nccl_get_unique_id": [C.c_char_p],
    "dgvv_nccl_comm_init": [C.c_char_p, I32, I32, C.POINTER(VP)],
    "dgvv_nccl_comm_destroy": [VP],
    "dgvv_thread_group_create": [I32, C.POINTER(VP)],
    "dgvv_thread_group_comm": [VP, I32, C.POINTER(VP)],
    "dgvv_thread_group_destroy": [VP],
    "dgvv_exchange_bytes": [VP, I32, I32, C.POINTER(I64), C.POINTER(I64)],
}


def lib():
    """The loaded libdgvv.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libdgvv.so not built ({LIB_PATH}); run python -m paper_2506_14424_b200.build")
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    for name, args in _SIGS.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    L.dgvv_last_error.restype = C.c_char_p
    L.dgvv_last_error.argtypes = []
    L.dgvv_version.restype = C.c_char_p
    L.dgvv_destroy.restype = None
    L.dgvv_destroy.argtypes = [VP]
    _lib = L
    return L


def check(status):
    if status != OK:
        raise DgvvError(status, lib().dgvv_last_error().decode())
    return status


def header_functions():
    """Names of all functions declared in include/dgvv.h."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(dgvv_[a-z_]+)\s*\(", txt)))
