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


# stage codes of pevd_trace_event / pevd_message (pevd.h PEVD_TRACE_* / PEVD_LEDGER_*)
TRACE_STAGES = ("SBR", "BC", "SBR-Back", "BC-Back", "Solver", "FinalMultiply", "Comm")
LEDGER_STAGES = ("SBR", "SBR-panel", "BandStage", "BC", "U-gather", "Qd", "Result", "Gather")


class PevdTraceEvent(ctypes.Structure):
    _fields_ = [("worker", ctypes.c_int32), ("stage", ctypes.c_int32), ("block", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("t_start_ms", _dbl), ("t_end_ms", _dbl),
                ("words", _i64)]


class PevdMessage(ctypes.Structure):
    _fields_ = [("src", ctypes.c_int32), ("dst", ctypes.c_int32), ("stage", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("words", _i64)]


class PevdDistStats(ctypes.Structure):
    _fields_ = [("stages", PevdStats), ("t0_mono_ns", _dbl),
                ("events", ctypes.POINTER(PevdTraceEvent)), ("events_cap", _i64),
                ("n_events", _i64), ("msgs", ctypes.POINTER(PevdMessage)), ("msgs_cap", _i64),
                ("n_msgs", _i64)]


def new_dist_stats(events_cap: int = 1 << 15, msgs_cap: int = 1 << 15):
    """A PevdDistStats with caller-owned event / message arrays (kept alive on the object)."""
    st = PevdDistStats()
    st._ev = (PevdTraceEvent * events_cap)()
    st._ms = (PevdMessage * msgs_cap)()
    st.events = ctypes.cast(st._ev, ctypes.POINTER(PevdTraceEvent))
    st.events_cap = events_cap
    st.msgs = ctypes.cast(st._ms, ctypes.POINTER(PevdMessage))
    st.msgs_cap = msgs_cap
    return st


# name -> (restype, argtypes); must cover every function declared in include/pevd.h
SIGNATURES = {
    "pevd_last_error": (ctypes.c_char_p, []),
    "pevd_version": (ctypes.c_char_p, []),
    "pevd_kernel_launches": (_i64, []),
    "pevd_syevd_workspace_bytes": (_i64, [_i64, _int, _int, _int]),
    "pevd_syevd_device": (_int, [_i64, _int, _vp, _i64, _vp, _vp, _i64, _int, _int, _vp, _i64,
                                 _vp, ctypes.POINTER(PevdStats)]),
    "pevd_syevd_device_host_q": (_int, [_i64, _int, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _int,
                                        _int, _int, _vp, _i64, _vp, ctypes.POINTER(PevdStats)]),
    "pevd_syevd": (_int, [_i64, _int, _vp, _i64, _vp, _vp, _i64, _int, _int,
                          ctypes.POINTER(PevdStats)]),
    "pevd_syevd_checked": (_int, [_i64, _int, _vp, _i64, _vp, _vp, _i64, _int, _int, _dbl,
                                  _int, ctypes.POINTER(PevdStats)]),
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
    "pevd_bc_back_workspace_bytes": (_i64, [_i64, _i64, _int]),
    "pevd_bc_back_right": (_int, [_i64, _int, _vp, _vp, _int, _vp, _i64, _i64, _vp, _vp]),
    "pevd_bc_back_left": (_int, [_i64, _int, _vp, _vp, _int, _vp, _i64, _i64, _vp, _vp]),
    "pevd_asymmetry": (_int, [_i64, _vp, _i64, ctypes.POINTER(_dbl), _vp]),
    "pevd_transpose": (_int, [_i64, _i64, _vp, _i64, _vp, _i64, _vp]),
    "pevd_nccl_unique_id": (_int, [ctypes.c_char_p]),
    "pevd_comm_nccl_create": (_int, [_int, _int, ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "pevd_comm_destroy": (None, [_vp]),
    "pevd_dist_syevd": (_int, [_vp, _i64, _int, _vp, _i64, ctypes.POINTER(_i64),
                               ctypes.POINTER(_i64), _vp, _vp, _i64, _int, _int, _vp,
                               ctypes.POINTER(PevdDistStats)]),
    "pevd_syevd_multi": (_int, [_int, ctypes.POINTER(_int), _i64, _int, _vp, _i64,
                                ctypes.POINTER(_i64), ctypes.POINTER(_i64), _vp, _vp, _int, _int,
                                ctypes.POINTER(PevdDistStats)]),
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
