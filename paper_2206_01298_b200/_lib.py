"""ctypes binding of the C ABI in include/odeblock.h (``libodeblock.so``).

The library is loaded from the package directory only; there is no fallback:
if it is missing or fails to load, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libodeblock.so")
# experiments only: load another in-tree build of the same ABI (e.g. a variant under tools/)
if os.environ.get("OB_LIB_VARIANT"):
    LIB_PATH = os.path.join(os.path.dirname(PKG), os.environ["OB_LIB_VARIANT"])

OB_OK = 0
OB_ERR_VALUE = 1
OB_ERR_INTEGRATION = 2
OB_ERR_STIFFNESS = 3
OB_ERR_CONVERGENCE = 4
OB_ERR_GRADIENT_EXPLOSION = 5
OB_ERR_CUDA = 6
OB_ERR_UNSUPPORTED = 7

OB_F32, OB_F64 = 0, 1
OB_FIELD_MLP, OB_FIELD_STIFF, OB_FIELD_CNF, OB_FIELD_CONV = 0, 1, 2, 3
OB_SCHEME_RK, OB_SCHEME_THETA = 0, 1
OB_POLICY = {"store_all": 0, "store_solutions": 1, "revolve": 2}
OB_LOSS = {"half_sqnorm": 0, "mse": 4, "mae": 5, "ce_head": 2, "cnf_nll": 3, "seed": 6}
# (code 1 = the ABI's K=1 terminal MSE; the host routes mse through the general
#  observation path, code 4)
OB_MAX_LAYERS = 8
OB_MAX_STAGES = 8
OB_NSTATS = 8   # nfe_f, nfe_b, newton, gmres_f, gmres_b, accepted, rejected, recomputed

EXPORTS = (
    "ob_version", "ob_last_error", "ob_device_count", "ob_revolve_count", "ob_revolve_schedule",
    "ob_grad_workspace_size", "ob_grad", "ob_debug_phase_cycles", "ob_field_eval", "ob_field_jvp", "ob_field_vjp",
    "ob_field_vjp_u", "ob_adamw_step", "ob_grad_norm", "ob_optim_last_error", "ob_continuous_adjoint",
    "ob_forward_pass", "ob_backward_sweep", "ob_adamw_step_gated",
)


class FieldDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dtype", C.c_int32), ("n_layers", C.c_int32),
                ("widths", C.c_int32 * (OB_MAX_LAYERS + 1)), ("activation", C.c_int32),
                ("time_input", C.c_int32), ("out_scale", C.c_double), ("n_params", C.c_int64)]


class SchemeDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("stages", C.c_int32), ("fsal", C.c_int32), ("_pad", C.c_int32),
                ("theta", C.c_double), ("a", C.c_double * (OB_MAX_STAGES * OB_MAX_STAGES)),
                ("b", C.c_double * OB_MAX_STAGES), ("c", C.c_double * OB_MAX_STAGES),
                ("b_emb", C.c_double * OB_MAX_STAGES), ("order", C.c_int32), ("has_emb", C.c_int32)]


class SolverDesc(C.Structure):
    _fields_ = [("newton_tol", C.c_double), ("gmres_tol", C.c_double), ("newton_maxit", C.c_int32),
                ("gmres_maxit", C.c_int32), ("gmres_restart", C.c_int32), ("_pad", C.c_int32)]


class Problem(C.Structure):
    _fields_ = [("field", FieldDesc), ("scheme", SchemeDesc), ("solver", SolverDesc),
                ("batch", C.c_int64), ("batch_global", C.c_int64), ("n_steps", C.c_int32),
                ("policy", C.c_int32), ("nc", C.c_int32), ("loss", C.c_int32),
                ("times", C.POINTER(C.c_double)), ("flags", C.c_int32), ("n_obs", C.c_int32),
                ("obs_steps", C.POINTER(C.c_int32)),
                ("adaptive", C.c_int32), ("max_accepted", C.c_int32),
                ("abstol", C.c_double), ("reltol", C.c_double), ("h_init", C.c_double),
                ("h_min", C.c_double), ("h_max", C.c_double), ("safety", C.c_double),
                ("max_steps", C.c_int64), ("t0", C.c_double), ("tF", C.c_double),
                ("obs_times", C.POINTER(C.c_double)), ("tile_rows", C.c_int32), ("_pad2", C.c_int32)]


class Buffers(C.Structure):
    _fields_ = [("theta", C.c_void_p), ("aux", C.c_void_p), ("u0", C.c_void_p),
                ("targets", C.c_void_p), ("u_final", C.c_void_p), ("du0", C.c_void_p),
                ("dtheta", C.c_void_p), ("loss", C.c_void_p), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("sample_stats", C.c_void_p),
                ("head", C.c_void_p), ("labels", C.c_void_p), ("dhead", C.c_void_p),
                ("n_classes", C.c_int32), ("_pad", C.c_int32),
                ("obs_values", C.c_void_p), ("scale_lo", C.c_void_p), ("scale_hi", C.c_void_p),
                ("predictions", C.c_void_p), ("grid", C.c_void_p), ("n_accepted", C.c_void_p),
                ("seed", C.c_void_p), ("dtheta_seed", C.c_void_p)]


class Counters(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "nfe_forward", "nfe_backward", "steps_accepted", "steps_rejected", "steps_recomputed",
        "stored_states", "stored_stage_vectors", "max_live_slots", "recomputed_steps",
        "kernel_launches", "device_rhs_evals", "device_vjp_evals", "tile_rows", "tiles",
        "tensor_cores")] + [
        (n, C.c_double) for n in ("ms_pack", "ms_forward", "ms_reverse", "ms_reduce")]

    def as_dict(self):
        return {n: (float(getattr(self, n)) if n.startswith("ms_") else int(getattr(self, n)))
                for n, _ in self._fields_}


_lib = None
_lock = threading.Lock()


class LibraryMissing(RuntimeError):
    pass


def load():
    """Load the in-tree libodeblock.so; raise if it is absent (no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} is missing: build it with `python -m paper_2206_01298_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        lib.ob_version.restype = C.c_char_p
        lib.ob_last_error.restype = C.c_char_p
        lib.ob_device_count.argtypes = [C.POINTER(i32)]
        lib.ob_revolve_count.argtypes = [i32, i32, C.POINTER(i64)]
        lib.ob_revolve_schedule.argtypes = [i32, i32, C.POINTER(i32), i64, C.POINTER(i64)]
        lib.ob_grad_workspace_size.argtypes = [C.POINTER(Problem), C.POINTER(C.c_size_t)]
        lib.ob_grad.argtypes = [C.POINTER(Problem), C.POINTER(Buffers), C.POINTER(Counters), vp]
        lib.ob_forward_pass.argtypes = lib.ob_grad.argtypes
        lib.ob_backward_sweep.argtypes = lib.ob_grad.argtypes
        lib.ob_debug_phase_cycles.argtypes = [C.POINTER(C.c_uint64), C.c_int32, C.c_int32]
        dbl = C.c_double
        lib.ob_adamw_step.argtypes = [i32, vp, vp, vp, vp, i64, i64, dbl, dbl, dbl, dbl, dbl, vp]
        lib.ob_grad_norm.argtypes = [i32, vp, i64, C.POINTER(dbl), vp]
        lib.ob_adamw_step_gated.argtypes = [i32, vp, vp, vp, vp, i64, i64, dbl, dbl, dbl, dbl, dbl, dbl,
                                            vp, vp, vp]
        lib.ob_continuous_adjoint.argtypes = [C.POINTER(Problem), vp, vp, vp, vp, vp, vp, vp,
                                              C.c_size_t, C.POINTER(Counters), vp]
        fd = C.POINTER(FieldDesc)
        lib.ob_field_eval.argtypes = [fd, i64, vp, vp, vp, C.c_double, vp, vp]
        lib.ob_field_jvp.argtypes = [fd, i64, vp, vp, vp, C.c_double, vp, vp, vp]
        lib.ob_field_vjp.argtypes = [fd, i64, vp, vp, vp, C.c_double, vp, vp, vp, vp]
        lib.ob_field_vjp_u.argtypes = [fd, i64, vp, vp, vp, C.c_double, vp, vp, vp]
        for name in EXPORTS:
            getattr(lib, name).restype = C.c_int if name not in (
                "ob_version", "ob_last_error", "ob_optim_last_error") else C.c_char_p
        _lib = lib
        return lib


def last_error() -> str:
    return load().ob_last_error().decode()


def optim_last_error() -> str:
    return load().ob_optim_last_error().decode()


def version() -> str:
    return load().ob_version().decode()
