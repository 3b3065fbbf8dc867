"""ctypes binding of libb200hydro.so (include/b200hydro.h).

The shared library is built in-tree by `paper_2112_07075_b200.build` (nvcc,
sm_100a).  There is no fallback: if the library or a CUDA device is missing,
every entry point raises `BackendUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# HX_LIB: alternative in-tree build of the same library (A/B measurements of compile-time variants)
LIB_PATH = os.environ.get("HX_LIB") or os.path.join(HERE, "libb200hydro.so")

HX_OK, HX_EINVAL, HX_EINVERTED, HX_ECG_BREAKDOWN, HX_ECG_MAXITER, HX_ECUDA, HX_ENCCL, HX_EUNDERFLOW = range(8)
HX_SPACE_H1, HX_SPACE_L2 = 0, 1


class BackendUnavailable(RuntimeError):
    """The sm_100a library or a CUDA device is missing (no CPU fallback exists)."""


class MeshDesc(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("order", C.c_int32), ("q1d", C.c_int32), ("thermo_order", C.c_int32),
        ("num_elements", C.c_int64), ("num_nodes", C.c_int64),
        ("dofmap_host", C.POINTER(C.c_int64)),
        ("B_host", C.POINTER(C.c_double)), ("G_host", C.POINTER(C.c_double)),
        ("Bt_host", C.POINTER(C.c_double)), ("qweights_host", C.POINTER(C.c_double)),
        ("device", C.c_int32),
    ]


class Params(C.Structure):
    _fields_ = [
        ("gamma", C.c_double), ("q1", C.c_double), ("q2", C.c_double),
        ("rel_tol", C.c_double), ("max_iter", C.c_int32), ("max_retries", C.c_int32),
        ("cfl", C.c_double), ("dt_min", C.c_double), ("dt_max", C.c_double), ("t_final", C.c_double),
    ]


class Inverted(C.Structure):
    _fields_ = [("inverted", C.c_int32), ("element", C.c_int64), ("point", C.c_int64), ("detj", C.c_double)]


class CGInfo(C.Structure):
    _fields_ = [("code", C.c_int32), ("iterations", C.c_int32), ("n_residuals", C.c_int32)]


class StepInfo(C.Structure):
    _fields_ = [
        ("code", C.c_int32), ("cg_iterations", C.c_int32 * 2), ("retries", C.c_int32),
        ("clamped", C.c_int64), ("dt", C.c_double), ("min_h_over_speed", C.c_double),
        ("t_new", C.c_double), ("inv", Inverted), ("failed_stage", C.c_int32),
    ]


P = C.c_void_p
_SIGS = {
    "hx_create": (C.c_int, [C.POINTER(MeshDesc), C.POINTER(C.c_void_p)]),
    "hx_destroy": (C.c_int, [P]),
    "hx_set_stream": (C.c_int, [P, P]),
    "hx_last_error": (C.c_char_p, [P]),
    "hx_kernel_launches": (C.c_int64, [P]),
    "hx_layout": (C.c_int, [P]),
    "hx_set_material": (C.c_int, [P, P]),
    "hx_diffusion_create": (C.c_int, [P, P, P, P, P, C.POINTER(C.c_void_p)]),
    "hx_convection_create": (C.c_int, [P, P, P, P, P, C.POINTER(C.c_void_p)]),
    "hx_op_apply": (C.c_int, [P, P, P]),
    "hx_op_destroy": (C.c_int, [P]),
    "hx_gather": (C.c_int, [P, C.c_int, P, C.c_int, P]),
    "hx_scatter_add": (C.c_int, [P, C.c_int, P, C.c_int, P]),
    "hx_geometry": (C.c_int, [P, P, P, P, P, P, C.POINTER(Inverted)]),
    "hx_mass_create": (C.c_int, [P, P, C.POINTER(C.c_void_p)]),
    "hx_mass_destroy": (C.c_int, [P]),
    "hx_mass_apply": (C.c_int, [P, P, C.c_int, P]),
    "hx_mass_diagonal": (C.c_int, [P, P]),
    "hx_mass_cg": (C.c_int, [P, P, C.c_int, P, P, C.c_double, C.c_int, P, P, C.POINTER(CGInfo)]),
    "hx_force_create": (C.c_int, [P, P, P, P, P, C.POINTER(C.c_void_p)]),
    "hx_force_destroy": (C.c_int, [P]),
    "hx_force_apply": (C.c_int, [P, P, P]),
    "hx_force_apply_t": (C.c_int, [P, P, P]),
    "hx_phase_begin": (C.c_int, [P, P, P, P, P, P, P]),
    "hx_stress": (C.c_int, [P, C.POINTER(Params), P, P, P, P, P, C.POINTER(C.c_double),
                            C.POINTER(C.c_int64), C.POINTER(Inverted)]),
    "hx_tmop_create": (C.c_int, [P, P, P, P, P, C.c_int, C.c_double, C.c_double, C.c_double, C.POINTER(P)]),
    "hx_tmop_set_gamma": (C.c_int, [P, C.c_double]),
    "hx_tmop_terms": (C.c_int, [P, P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    "hx_tmop_gradient": (C.c_int, [P, P, P]),
    "hx_tmop_hessian_action": (C.c_int, [P, P, P, P]),
    "hx_tmop_hessian_diagonal": (C.c_int, [P, P, P]),
    "hx_tmop_destroy": (C.c_int, [P]),
    "hx_timestep_ratio": (C.c_int, [P, C.POINTER(Params), P, P, P, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                    C.POINTER(Inverted)]),
    "hx_energy_solve": (C.c_int, [P, P, P]),
    "hx_rates": (C.c_int, [P, C.POINTER(Params), P, P, P, P, P, C.POINTER(StepInfo)]),
    "hx_step": (C.c_int, [P, C.POINTER(Params), C.c_double, P, P, P, P, P, P, C.POINTER(StepInfo)]),
    "hx_rk2_step": (C.c_int, [P, C.POINTER(Params), C.c_double, C.c_double, P, P, P, P, P, P,
                              C.POINTER(StepInfo)]),
    "hx_step_host": (C.c_int, [P, C.POINTER(Params), C.c_double, P, P, P, C.POINTER(StepInfo)]),
    "hx_energies": (C.c_int, [P, P, P, P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "hx_prof_enable": (C.c_int, [P, C.c_int]),
    "hx_prof_read": (C.c_int, [P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "hx_prof_reset": (C.c_int, [P]),
    "hx_prof_dup": (C.c_int, [P, C.c_int]),
    "hx_fp64_peak": (C.c_int, [C.POINTER(C.c_double)]),
    "hx_peer_setup": (C.c_int, [P, C.c_int, C.c_int, C.c_int, C.c_int, P, P, P, C.c_int, P, P, P, C.c_int, P, P,
                                C.POINTER(C.c_void_p)]),
    "hx_peer_connect": (C.c_int, [P, P]),
    "hx_peer_disconnect": (C.c_int, [P]),
    "hx_peer_ipc_handle": (C.c_int, [P, P]),
    "hx_peer_ipc_open": (C.c_int, [P, C.POINTER(C.c_void_p)]),
    "hx_peer_ipc_close": (C.c_int, [P]),
    "hx_peer_state": (C.c_int, [P, P]),
    "hx_comm_active": (C.c_int, [P]),
}

_lib = None


def exported_symbols():
    """Names declared in include/b200hydro.h that the library must export."""
    return sorted(_SIGS)


def load(require_cuda: bool = True):
    """Load the library (once).  Raises BackendUnavailable when it cannot run."""
    global _lib
    if _lib is not None:
        if require_cuda:
            _require_cuda()
        return _lib
    if not os.path.exists(LIB_PATH):
        raise BackendUnavailable(
            f"{LIB_PATH} is missing: build it with `python -m paper_2112_07075_b200.build` "
            "(nvcc, sm_100a).  There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    if require_cuda:
        _require_cuda()
    return lib


def _require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device visible: the B200 path has no CPU fallback")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def current_stream_ptr() -> int:
    import torch

    return torch.cuda.current_stream().cuda_stream


def as_f64_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def as_i64_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))
