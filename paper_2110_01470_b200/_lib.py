"""ctypes binding of libpsso.so (the C ABI declared in include/psso.h).

The library is loaded with ``ctypes.CDLL`` so the GIL is released for the
duration of every foreign call.  There is no CPU fallback: if the shared
library is missing or no CUDA device is present, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("PSSO_LIB") or Path(__file__).resolve().parent / "libpsso.so")

PSSO_OK = 0
PSSO_E_INVALID = 1
PSSO_E_CUDA = 2
PSSO_E_NONFINITE = 3
PSSO_E_UNSUPPORTED = 4
PSSO_E_NCCL = 5

PSSO_F64 = 0
PSSO_F32 = 1
PSSO_RNG_REFERENCE = 0
PSSO_RNG_PHILOX = 1
PSSO_FN_PROBE = 0

#: every symbol include/psso.h declares (checked by tests/test_lib_exports.py)
EXPORTS = (
    "psso_version", "psso_last_error", "psso_create", "psso_destroy", "psso_bind",
    "psso_init", "psso_step", "psso_run", "psso_search", "psso_evaluate",
    "psso_update_pbests", "psso_update_gbest", "psso_candidate_bytes", "psso_init_local",
    "psso_step_local", "psso_apply_candidates", "psso_check", "psso_result", "psso_set_gbest_index", "psso_nonfinite",
    "psso_iteration_stats", "psso_batch_failure", "psso_run_p2p",
    "psso_launch_count",
    "psso_rng_uniform", "psso_eval_rows", "psso_solve", "psso_profile", "psso_profile_read",
    "psso_kernel_name", "psso_solve_batch", "psso_p2p_buffer_bytes", "psso_p2p_alloc",
    "psso_p2p_free", "psso_p2p_handle", "psso_p2p_open", "psso_p2p_close", "psso_publish_p2p",
    "psso_apply_p2p", "psso_run_sequential", "psso_sequential_passes",
    "psso_solve_sequential_batch", "psso_nccl_unique_id", "psso_comm_create", "psso_comm_destroy",
    "psso_attach_comm", "psso_init_sharded",
    "psso_run_sharded",
)


class PssoConfig(ctypes.Structure):
    _fields_ = [
        ("fn_id", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("rng_mode", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("nsol", ctypes.c_int64),
        ("nvar", ctypes.c_int64),
        ("row_lo", ctypes.c_int64),
        ("row_hi", ctypes.c_int64),
        ("cw", ctypes.c_double),
        ("cp", ctypes.c_double),
        ("cg", ctypes.c_double),
        ("var_min", ctypes.c_double),
        ("var_max", ctypes.c_double),
        ("seed", ctypes.c_uint64),
        ("probe_level", ctypes.c_double),
    ]


class PssoBuffers(ctypes.Structure):
    _fields_ = [
        ("sol", ctypes.c_void_p),
        ("pbests", ctypes.c_void_p),
        ("sol_f", ctypes.c_void_p),
        ("p_f", ctypes.c_void_p),
        ("gbest", ctypes.c_void_p),
        ("g_f", ctypes.c_void_p),
        ("traj", ctypes.c_void_p),
    ]


class PssoError(RuntimeError):
    def __init__(self, code: int, message: str):
        self.code = code
        super().__init__(message)


_lib = None


def load():
    """Load libpsso.so once; raises loudly when the CUDA extension is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"CUDA extension {LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)"
        )
    L = ctypes.CDLL(str(LIB_PATH))
    vp, i64, i32, u64, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double
    cfgp = ctypes.POINTER(PssoConfig)
    L.psso_version.restype = ctypes.c_char_p
    L.psso_last_error.restype = ctypes.c_char_p
    L.psso_last_error.argtypes = [vp]
    L.psso_create.argtypes = [cfgp, ctypes.POINTER(vp)]
    L.psso_destroy.argtypes = [vp]
    L.psso_destroy.restype = None
    L.psso_bind.argtypes = [vp, ctypes.POINTER(PssoBuffers), vp]
    L.psso_init.argtypes = [vp]
    L.psso_step.argtypes = [vp, i64]
    L.psso_run.argtypes = [vp, i64, i64]
    L.psso_search.argtypes = [vp, i64]
    L.psso_evaluate.argtypes = [vp, i64]
    L.psso_update_pbests.argtypes = [vp]
    L.psso_update_gbest.argtypes = [vp]
    L.psso_candidate_bytes.argtypes = [cfgp]
    L.psso_candidate_bytes.restype = i64
    L.psso_init_local.argtypes = [vp, vp]
    L.psso_step_local.argtypes = [vp, i64, vp]
    L.psso_apply_candidates.argtypes = [vp, i64, vp, i32, i32]
    L.psso_check.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.psso_set_gbest_index.argtypes = [vp, i64]
    L.psso_run_p2p.argtypes = [vp, i64, i64, vp, vp, i32, i32]
    L.psso_batch_failure.argtypes = [ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64),
                                     ctypes.POINTER(dbl)]
    L.psso_iteration_stats.argtypes = [vp, i64, i64, ctypes.POINTER(dbl), ctypes.POINTER(i64),
                                       ctypes.POINTER(i64)]
    L.psso_nccl_unique_id.argtypes = [vp]
    L.psso_comm_create.argtypes = [vp, i32, i32, ctypes.POINTER(vp)]
    L.psso_comm_destroy.argtypes = [vp]
    L.psso_comm_destroy.restype = None
    L.psso_attach_comm.argtypes = [vp, vp]
    L.psso_init_sharded.argtypes = [vp]
    L.psso_run_sharded.argtypes = [vp, i64, i64]
    L.psso_nonfinite.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(dbl)]
    L.psso_result.argtypes = [vp, ctypes.POINTER(dbl), ctypes.POINTER(i64), ctypes.POINTER(i64),
                              ctypes.POINTER(i64)]
    L.psso_launch_count.argtypes = [vp]
    L.psso_launch_count.restype = i64
    L.psso_profile.argtypes = [vp, i32]
    L.psso_profile_read.argtypes = [vp, ctypes.POINTER(dbl), ctypes.POINTER(i64)]
    L.psso_rng_uniform.argtypes = [u64, u64, u64, vp, vp, i64, vp, vp]
    L.psso_eval_rows.argtypes = [i32, i32, i64, vp, i64, vp, dbl, vp]
    L.psso_solve.argtypes = [cfgp, i64, vp, vp, ctypes.POINTER(dbl), ctypes.POINTER(dbl)]
    L.psso_solve_batch.argtypes = [cfgp, vp, i32, i64, vp, vp, vp, ctypes.POINTER(dbl)]
    L.psso_solve_sequential_batch.argtypes = L.psso_solve_batch.argtypes
    L.psso_kernel_name.argtypes = [vp]
    L.psso_kernel_name.restype = ctypes.c_char_p
    L.psso_p2p_buffer_bytes.argtypes = [cfgp, i32]
    L.psso_p2p_buffer_bytes.restype = i64
    L.psso_p2p_alloc.argtypes = [i64, ctypes.POINTER(vp)]
    L.psso_p2p_free.argtypes = [vp]
    L.psso_p2p_handle.argtypes = [vp, vp]
    L.psso_p2p_open.argtypes = [vp, ctypes.POINTER(vp)]
    L.psso_p2p_close.argtypes = [vp]
    L.psso_publish_p2p.argtypes = [vp, vp, vp, i32, i32, u64]
    L.psso_apply_p2p.argtypes = [vp, i64, vp, i32, u64, i32]
    L.psso_run_sequential.argtypes = [vp, i64, i64]
    L.psso_sequential_passes.argtypes = [vp, ctypes.POINTER(i64)]
    for name in EXPORTS:
        if not hasattr(L, name):
            raise RuntimeError(f"{LIB_PATH} does not export {name}")
    _lib = L
    return L


def last_error(ctx=None) -> str:
    msg = load().psso_last_error(ctx)
    return msg.decode() if msg else ""


def check(rc: int, ctx=None) -> None:
    if rc == PSSO_OK:
        return
    msg = last_error(ctx)
    if rc in (PSSO_E_INVALID,):
        raise ValueError(msg)
    raise PssoError(rc, msg)


def require_device() -> None:
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the PSSO engine runs on CUDA (sm_100a) only; no GPU is visible")
    load()


def env_flag(name: str) -> bool:
    return os.environ.get(name, "") not in ("", "0", "false")
