"""ctypes binding of libvoxb200.so (the C ABI in include/voxb200.h).

There is no CPU fallback: importing the package on a machine without the
built library raises, and every compute entry point raises when no CUDA
device is present.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import NumericalError, SetupError, SolverBreakdown, VolumeInfeasible

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VT_LIB_PATH") or os.path.join(_HERE, "libvoxb200.so")

VT_OK, VT_EINVAL, VT_ECUDA, VT_ESETUP, VT_EBREAKDOWN, VT_EVOLUME, VT_ENUMERICAL, VT_ENOMEM, VT_EDENSITY = range(9)

P = C.c_void_p
D = C.c_double
I = C.c_int
I64 = C.c_int64


class SolveReportC(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("final_rel_residual", C.c_double),
        ("precond_applications", C.c_int),
        ("converged", C.c_int),
        ("residual_drift", C.c_double),
        ("breakdown", C.c_int),
        ("breakdown_iter", C.c_int),
        ("breakdown_value", C.c_double),
    ]


_SIGS = {
    "vt_last_error": (C.c_char_p, []),
    "vt_version": (I, []),
    "vt_launch_count": (C.c_uint64, []),
    "vt_copy": (I, [P, P, I64, P]),
    "vt_debug_trace": (I, [P, I, P, I]),
    "vt_grid_create": (I, [C.POINTER(P), I, I, I, D, D, P, I, I, I]),
    "vt_grid_destroy": (I, [P]),
    "vt_vec_len": (I64, [P]),
    "vt_elem_len": (I64, [P]),
    "vt_n_fixed": (I64, [P]),
    "vt_vec_upload": (I, [P, P, P, P]),
    "vt_vec_download": (I, [P, P, P, P]),
    "vt_scale_from_density": (I, [P, P, D, D, D, P, P]),
    "vt_apply": (I, [P, P, P, P, P]),
    "vt_apply_projected": (I, [P, P, P, P, P]),
    "vt_apply_host": (I, [P, P, P, P, I, P]),
    "vt_diagonal": (I, [P, P, P, P]),
    "vt_residual": (I, [P, P, P, P, P, P]),
    "vt_dot": (I, [P, P, P, C.POINTER(D), P]),
    "vt_axpy": (I, [P, I, D, P, P, P]),
    "vt_project": (I, [P, P, P, P]),
    "vt_assemble_dense": (I, [P, P, P, P, P]),
    "vt_hier_create": (I, [C.POINTER(P), P, I, D, I]),
    "vt_hier_destroy": (I, [P]),
    "vt_hier_create_ex": (I, [C.POINTER(P), P, I, D, I, I]),
    "vt_hier_scheme": (I, [P]),
    "vt_tail_config": (C.c_longlong, [C.c_longlong]),
    "vt_hier_tail_level": (I, [P]),
    "vt_tail_trace": (I, [I, P, I]),
    "vt_hier_level_mats": (P, [P, I]),
    "vt_hier_levels": (I, [P]),
    "vt_hier_grid": (P, [P, I]),
    "vt_hier_refresh": (I, [P, P, P, D, D, D, P]),
    "vt_hier_vcycle": (I, [P, P, P, P]),
    "vt_hier_restrict": (I, [P, I, P, P, P]),
    "vt_hier_prolong": (I, [P, I, P, P, P]),
    "vt_hier_jacobi": (I, [P, I, P, P, I, P, P]),
    "vt_hier_level_apply": (I, [P, I, P, P, P]),
    "vt_hier_level_diag": (I, [P, I, P, P]),
    "vt_hier_coarse_solve": (I, [P, P, P, P]),
    "vt_hier_level_scale": (P, [P, I]),
    "vt_hier_level_rho": (P, [P, I]),
    "vt_pcg": (I, [P, P, I, P, P, P, I, D, I, C.POINTER(SolveReportC), P]),
    "vt_compliance": (I, [P, P, P, C.POINTER(D), P]),
    "vt_sensitivities": (I, [P, P, P, D, D, D, I, D, P, P]),
    "vt_gravity_load": (I, [P, P, I, D, P, I, P, P]),
    "vt_scale_two_material": (I, [P, P, P, D, D, D, D, P, P, P]),
    "vt_sensitivities_two_material": (I, [P, P, P, P, D, D, D, D, I, D, P, P, P]),
    "vt_filter_create": (I, [C.POINTER(P), P, I, P]),
    "vt_filter_destroy": (I, [P]),
    "vt_filter_wsum": (P, [P]),
    "vt_filter_apply": (I, [P, P, P, D, P, P]),
    "vt_filter_correlate": (I, [P, P, P, P]),
    "vt_oc_update": (I, [P, P, P, P, P, D, D, D, D, P, C.POINTER(D), C.POINTER(I), P]),
    "vt_oc_update_flat": (I, [I64, P, P, P, P, D, D, D, D, P, C.POINTER(D), C.POINTER(I), P]),
    "vt_change_volume": (I, [P, P, P, P, C.POINTER(D), C.POINTER(D), P]),
    "vt_nccl_id_bytes": (I, []),
    "vt_nccl_unique_id": (I, [P, I]),
    "vt_dist_create": (I, [C.POINTER(P), I, I, I, D, D, P, I, D, I, I, I, P, I, P, I]),
    "vt_dist_set_scheme": (I, [P, I]),
    "vt_dist_scheme": (I, [P]),
    "vt_dist_create_peer": (I, [C.POINTER(P), I, I, I, D, D, P, I, D, I, I, P, I, I]),
    "vt_peer_handle_bytes": (I, []),
    "vt_dist_peer_handle": (I, [P, P, I]),
    "vt_dist_peer_open": (I, [P, P, I]),
    "vt_dist_destroy": (I, [P]),
    "vt_dist_levels": (I, [P]),
    "vt_dist_dist_level": (I, [P]),
    "vt_dist_nlocal": (I, [P]),
    "vt_dist_grid": (P, [P, I, I]),
    "vt_dist_tail": (P, [P]),
    "vt_dist_graph_nodes": (C.c_uint64, [P]),
    "vt_dist_set_scale": (I, [P, P, P]),
    "vt_dist_refresh": (I, [P, P, P, D, D, D, P]),
    "vt_dist_apply": (I, [P, P, P, P]),
    "vt_dist_dot": (I, [P, P, P, C.POINTER(D), P]),
    "vt_dist_vcycle": (I, [P, P, P, P]),
    "vt_dist_pcg": (I, [P, P, P, I, D, I, C.POINTER(SolveReportC), P]),
    "vt_dist_sensitivities": (I, [P, P, P, D, D, D, I, D, P, P]),
    "vt_dist_sensitivities_two_material": (I, [P, P, P, P, D, D, D, D, I, D, P, P, P]),
    "vt_dist_gravity_load": (I, [P, P, I, D, P, I, P, P]),
    "vt_dist_filter_create": (I, [P, I, P]),
    "vt_dist_filter_apply": (I, [P, P, P, D, P, P]),
    "vt_dist_oc_update": (I, [P, P, P, P, P, D, D, D, D, P, C.POINTER(D), C.POINTER(I), P]),
    "vt_dist_change_volume": (I, [P, P, P, P, C.POINTER(D), C.POINTER(D), P]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c \"import __graft_entry__ as g; g.build()\"` "
            "(nvcc, sm_100a). There is no CPU fallback."
        )
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    msg = lib.vt_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    """Map a vt_status to the reference's exception classes (errors.py:7-24)."""
    if status == VT_OK:
        return
    msg = last_error() or what
    if status in (VT_EINVAL, VT_EDENSITY):
        raise ValueError(msg)
    if status == VT_ESETUP:
        raise SetupError(msg)
    if status == VT_EBREAKDOWN:
        raise SolverBreakdown(msg)
    if status == VT_EVOLUME:
        raise VolumeInfeasible(msg)
    if status == VT_ENUMERICAL:
        raise NumericalError(msg)
    if status == VT_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libvoxb200: {msg}")
