"""ctypes binding of libpevd.so (the C ABI declared in include/pevd.h).

The product path has no CPU fallback: if the shared library or a CUDA device is missing, every
compute entry point raises.  Device memory and streams come from PyTorch (plumbing only).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpevd.so")

PEVD_OK, PEVD_ERR_CUDA, PEVD_ERR_VALUE, PEVD_ERR_CONVERGE, PEVD_ERR_NOMEM = 0, 1, 2, 3, 4
ORDER_CODES = {"pipelined": 0, "sequential": 1, "conventional": 2}

_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double
_vp = ctypes.c_void_p


class PevdStats(ctypes.Structure):
    _fields_ = [("sbr_ms", _dbl * 2), ("bc_ms", _dbl * 2), ("solver_ms", _dbl * 2),
                ("sbr_back_ms", _dbl * 2), ("bc_back_ms", _dbl * 2), ("final_ms", _dbl * 2),
                ("total_ms", _dbl), ("n_reflectors", _i64), ("n_rounds", _i64),
                ("flops", _dbl * 6)]

# order of PevdStats.flops (pevd.h): the FlopCounter stage names
FLOP_STAGES = ("SBR", "BC", "SBR-Back", "BC-Back", "Solver", "FinalMultiply")


# name -> (restype, argtypes); must cover every function declared in include/pevd.h
SIGNATURES = {
    "pevd_last_error": (ctypes.c_char_p, []),
    "pevd_version": (ctypes.c_char_p, []),
    "pevd_kernel_launches": (_i64, []),
    "pevd_syevd_workspace_bytes": (_i64, [_i64, _int, _int, _int]),
    "pevd_syevd_device": (_int, [_i64, _int, _vp, _i64, _vp, _vp, _i64, _int, _int, _vp, _i64,
                                 _vp, ctypes.POINTER(PevdStats)]),
    "pevd_syevd": (_int, [_i64, _int, _vp, _i64, _vp, _vp, _i64, _int, _int,
                          ctypes.POINTER(PevdStats)]),
    "pevd_dgemm": (_int, [_int, _int, _i64, _i64, _i64, _dbl, _vp, _i64, _vp, _i64, _dbl, _vp,
                          _i64, _vp, _i64, _vp]),
    "pevd_dsymm_lower": (_int, [_i64, _i64, _dbl, _vp, _i64, _vp, _i64, _dbl, _vp, _i64, _vp, _i64,
                                _vp]),
    "pevd_panel_qr_workspace_bytes": (_i64, []),
    "pevd_panel_qr": (_int, [_i64, _int, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp]),
    "pevd_sbr_workspace_bytes": (_i64, [_i64, _int]),
    "pevd_sbr": (_int, [_i64, _int, _vp, _i64, _vp, _vp, _vp, _vp]),
    "pevd_bc_num_reflectors": (_i64, [_i64, _int]),
    "pevd_bc_workspace_bytes": (_i64, [_i64, _int]),
    "pevd_bc": (_int, [_i64, _int, _vp, _vp, _vp, _vp, _vp, _int, _vp, _vp]),
    "pevd_bc_partition": (_int, [_i64, _int, _int, _vp, _i64, _vp, _vp, _vp, _int, _vp, _vp]),
    "pevd_stedc_workspace_bytes": (_i64, [_i64]),
    "pevd_stedc": (_int, [_i64, _vp, _vp, _vp, _i64, _vp, _vp]),
    "pevd_stedc_cols": (_int, [_i64, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp]),
    "pevd_sbr_back_workspace_bytes": (_i64, [_i64, _int]),
    "pevd_sbr_back_form": (_int, [_i64, _int, _vp, _i64, _vp, _vp, _i64, _vp, _vp]),
    "pevd_sbr_back_left": (_int, [_i64, _int, _vp, _i64, _vp, _vp, _i64, _i64, _vp, _vp]),
    "pevd_bc_back_workspace_bytes": (_i64, [_i64, _i64]),
    "pevd_bc_back_right": (_int, [_i64, _int, _vp, _vp, _int, _vp, _i64, _i64, _vp, _vp]),
    "pevd_bc_back_left": (_int, [_i64, _int, _vp, _vp, _int, _vp, _i64, _i64, _vp, _vp]),
}

_lib = None


class PevdError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def load():
    """Load libpevd.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc != PEVD_OK:
        msg = load().pevd_last_error().decode(errors="replace")
        err = PevdError(rc, f"{what}: {msg}")
        if rc == PEVD_ERR_VALUE:
            raise ValueError(str(err))
        raise err


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2511_16174_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    load()
    return torch
