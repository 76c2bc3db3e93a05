"""B200-native pipelined two-stage FP64 symmetric EVD (arXiv 2511.16174), a drop-in for the
hot path of the reference package `pipeevd` (pkg/src/pipeevd/__init__.py:10-47).

All arithmetic runs in libpevd.so (hand-written sm_100a CUDA: FP64 DMMA GEMMs, cooperative
panel QR, wavefront bulge chase, device divide and conquer, BLAS2 register-window BC-Back)
behind the C ABI in include/pevd.h.  There is no CPU fallback: importing works anywhere, but
every compute call raises without a CUDA device and the built library.
"""
from .core import (EPS, BandMatrix, EigenResult, FlopCounter, ProtocolError, ReflectorPanel,
                   SymmetricMatrix, TridiagonalMatrix)
from .messaging import BROADCAST, HOST, CommLedger, TraceEvent, TraceLog
from .pipeline import ORDERS, PipelineConfig, PipelineError, run, run_auto_skew
from .schedule import (BackPlan, back_plan_sizes, comm_broadcast_words, comm_triangular_words,
                       crossover_bandwidth, make_back_plan, mean_idle_fraction, partition,
                       round_schedule, validate_trace)
from .stages import (BcPartitionResult, BulgeReflectorSet, OverlapBlock, RowAccumulator, SbrConfig, SbrFactors,
                     application_order, apply_block_reflector, bc_back_apply, bc_reduce,
                     bc_reduce_partition,
                     final_gemm, form_z, house_vector, panel_qr, sbr_back_accumulate,
                     sbr_back_rows, sbr_reduce, sym_rank2k_update, trailing_update, tridiag_eig)

__version__ = "0.1.0"

__all__ = [
    "BackPlan", "BandMatrix", "BcPartitionResult", "bc_reduce_partition", "BulgeReflectorSet", "OverlapBlock", "RowAccumulator",
    "application_order", "apply_block_reflector", "form_z", "sym_rank2k_update", "trailing_update", "CommLedger", "EigenResult", "FlopCounter",
    "HOST", "BROADCAST", "ORDERS", "PipelineConfig", "PipelineError", "ProtocolError",
    "ReflectorPanel", "SbrConfig", "SbrFactors", "SymmetricMatrix", "TraceEvent", "TraceLog",
    "TridiagonalMatrix", "back_plan_sizes", "bc_back_apply", "bc_reduce", "comm_broadcast_words",
    "comm_triangular_words", "crossover_bandwidth", "final_gemm", "house_vector",
    "make_back_plan", "panel_qr", "partition", "round_schedule", "run", "run_auto_skew",
    "sbr_back_accumulate", "sbr_back_rows", "sbr_reduce", "tridiag_eig", "validate_trace",
    "mean_idle_fraction",
]
