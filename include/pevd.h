/*
 * pevd.h -- C ABI of libpevd.so, the B200 (sm_100a) pipelined two-stage FP64 symmetric EVD.
 *
 * Drop-in boundary for the reference package `pipeevd` (a pure-Python package; its "FFI" is the
 * Python call `pipeevd.run(a, PipelineConfig(...))`, pkg/src/pipeevd/pipeline.py:511-548).  The
 * Python package `paper_2511_16174_b200` binds these symbols with ctypes and re-exposes the
 * reference's API names on top (see INTEGRATION.md for the binding).  Every entry point takes
 * plain pointers and sizes; matrices are column-major (Fortran order, as SymmetricMatrix stores
 * them, core.py:65-93).
 *
 * Return codes map to the reference's exception taxonomy:
 *   PEVD_ERR_VALUE    -> ValueError     (bad shape / bandwidth / config, pipeline.py:74-82)
 *   PEVD_ERR_CUDA     -> PipelineError  (device failure, pipeline.py:540-544)
 *   PEVD_ERR_CONVERGE -> RuntimeError   (solver did not converge, tridiag.py:314-320)
 * pevd_last_error() returns the message of the calling thread's last failure.
 */
#ifndef PEVD_H
#define PEVD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PEVD_OK 0
#define PEVD_ERR_CUDA 1
#define PEVD_ERR_VALUE 2
#define PEVD_ERR_CONVERGE 3
#define PEVD_ERR_NOMEM 4

/* back-transformation orders, PipelineConfig.order (pipeline.py:45, 57-82) */
#define PEVD_ORDER_PIPELINED 0
#define PEVD_ORDER_SEQUENTIAL 1
#define PEVD_ORDER_CONVENTIONAL 2

/* Per-stage device times (CUDA events on the launching streams), for TraceEvent /
 * FlopCounter population (messaging.py:51-108).  Offsets are relative to the first event. */
typedef struct pevd_stats {
  double sbr_ms[2];        /* [start, end] */
  double bc_ms[2];
  double solver_ms[2];
  double sbr_back_ms[2];
  double bc_back_ms[2];
  double final_ms[2];
  double total_ms;         /* first start .. last end */
  int64_t n_reflectors;    /* bulge reflector slots (sum_j (n-2-jb), b the chase bandwidth: roundup8(b) <= 64) */
  int64_t n_rounds;        /* SBR panels */
  /* EXECUTED flops per stage, in the order SBR, BC, SBR-Back, BC-Back, Solver, FinalMultiply
   * (FlopCounter stages, core.py:26-62): GEMM launches as issued (2 m n k; the lower-tile
   * rank-2k update counts its tiles), the divide and conquer's deflated merge GEMMs summed on the
   * device from their descriptors, the BC-Back DMMA kernel as the DMMAs it issues (1.25x the
   * BLAS2 count), panel QR and the chase analytically (2 m k^2 + 2 m k^2; 14 b^2 per reflector). */
  double flops[6];
} pevd_stats;

/* ---------------------------------------------------------------- multi-GPU (blockwise)
 * Trace events and ledger messages of one rank of a distributed EVD (TraceEvent / CommLedger,
 * messaging.py:51-167).  Stages of events: PEVD_TRACE_*; stages of messages: PEVD_LEDGER_*.
 * dst of a message: >= 0 a rank, -1 the host, -2 a broadcast (messaging.py HOST / BROADCAST). */
#define PEVD_TRACE_SBR 0
#define PEVD_TRACE_BC 1
#define PEVD_TRACE_SBR_BACK 2
#define PEVD_TRACE_BC_BACK 3
#define PEVD_TRACE_SOLVER 4
#define PEVD_TRACE_FINAL 5
#define PEVD_TRACE_COMM 6
#define PEVD_LEDGER_SBR 0
#define PEVD_LEDGER_SBR_PANEL 1
#define PEVD_LEDGER_BANDSTAGE 2
#define PEVD_LEDGER_BC 3
#define PEVD_LEDGER_UGATHER 4
#define PEVD_LEDGER_QD 5
#define PEVD_LEDGER_RESULT 6
#define PEVD_LEDGER_GATHER 7

typedef struct pevd_trace_event {
  int32_t worker, stage, block, pad;
  double t_start_ms, t_end_ms;  /* device time from the rank's t0 (CUDA events) */
  int64_t words;                /* FP64 words moved (Comm spans) */
} pevd_trace_event;

typedef struct pevd_message {
  int32_t src, dst, stage, pad;
  int64_t words;
} pevd_message;

/* Caller-owned arrays; the library fills min(count, cap) entries and reports the full count. */
typedef struct pevd_dist_stats {
  pevd_stats stages;        /* this rank's stage spans (ms from t0) and executed flops */
  double t0_mono_ns;        /* CLOCK_MONOTONIC at t0 (after a barrier of all ranks) */
  pevd_trace_event* events;
  int64_t events_cap, n_events;
  pevd_message* msgs;       /* this rank's SENDS, as words actually handed to the transport */
  int64_t msgs_cap, n_msgs;
} pevd_dist_stats;

const char* pevd_last_error(void);
const char* pevd_version(void);
/* Number of CUDA kernels this library has launched since it was loaded. */
int64_t pevd_kernel_launches(void);

/* ---------------------------------------------------------------- whole EVD
 * Replaces pipeevd.run (pipeline.py:511) for one GPU: A = Q diag(lam) Q^T.
 * lam ascending (tridiag.py:321); Q with columns the eigenvectors. */

/* Device workspace needed by pevd_syevd_device (bytes). */
int64_t pevd_syevd_workspace_bytes(int64_t n, int b, int want_vectors, int order);

/* All pointers are DEVICE pointers.  A (n x n, lda; only the lower triangle is read) is
 * destroyed.  Q (n x n, ldq) may be NULL when want_vectors == 0.  `stream` is a cudaStream_t
 * (NULL = legacy default stream).  Synchronous: returns after the result is complete. */
int pevd_syevd_device(int64_t n, int b, double* A, int64_t lda, double* lam, double* Q,
                      int64_t ldq, int want_vectors, int order, void* workspace,
                      int64_t workspace_bytes, void* stream, pevd_stats* stats);

/* As pevd_syevd_device, but Q (a DEVICE buffer it computes in) is also delivered to the HOST
 * buffer Qh (ldqh >= n): in conventional order the last back-transformation runs in column
 * slabs and each slab's copy overlaps the next slab's compute, so only the last slab's copy is
 * exposed.  q_row_major = 0: Qh column-major.  q_row_major = 1 (pipelined / sequential orders
 * only, PEVD_ERR_VALUE otherwise): Qh receives Q row-major -- the C-ordered Q of pipeline.py:503
 * -- from a final GEMM that forms Q^T in slabs, streamed the same way (the device buffer Q then
 * holds Q^T).  Pinned Qh is copied by the copy engines; pageable Qh through pinned
 * staging chunks worked by several host threads (PEVD_STAGE_THREADS, default 8). */
int pevd_syevd_device_host_q(int64_t n, int b, double* A, int64_t lda, double* lam, double* Q,
                             int64_t ldq, double* Qh, int64_t ldqh, int q_row_major,
                             int want_vectors, int order, void* workspace,
                             int64_t workspace_bytes, void* stream, pevd_stats* stats);

/* HOST pointers (A column-major, lda; only its lower triangle is read and copied to the
 * device); allocates device memory itself.  Q comes back as pevd_syevd_device_host_q delivers
 * it.  Q may be NULL when want_vectors == 0.  A is not modified. */
int pevd_syevd(int64_t n, int b, const double* A, int64_t lda, double* lam, double* Q,
               int64_t ldq, int want_vectors, int order, pevd_stats* stats);

/* pevd_syevd with the input check of SymmetricMatrix (core.py:75-84, pipeline.py:517-518)
 * folded in: all of A goes up and max |A_ij - A_ji| > sym_tol * max(1, ||A||_F) returns
 * PEVD_ERR_VALUE ("asymmetry ... exceeds tolerance") before any reduction runs; sym_tol < 0
 * skips the check (and uploads only the lower triangle).  q_row_major as in
 * pevd_syevd_device_host_q. */
int pevd_syevd_checked(int64_t n, int b, const double* A, int64_t lda, double* lam, double* Q,
                       int64_t ldq, int want_vectors, int order, double sym_tol, int q_row_major,
                       pevd_stats* stats);

/* The input check of SymmetricMatrix (core.py:75-84) on the device: out2[0] = max |A_ij - A_ji|,
 * out2[1] = ||A||_F (HOST array of 2).  A device pointer (column-major, lda).  Synchronous. */
int pevd_asymmetry(int64_t n, const double* A, int64_t lda, double* out2, void* stream);
/* out (cols x rows, ldo) = in^T (in: rows x cols, ldi), device pointers: the C-order Q of
 * pipeline.py:503 without a host transpose. */
int pevd_transpose(int64_t rows, int64_t cols, const double* in, int64_t ldi, double* out,
                   int64_t ldo, void* stream);

/* ---------------------------------------------------------------- per-stage (device pointers)
 * Each replaces one reference function; `stream` is a cudaStream_t; all are asynchronous except
 * where noted. */

/* C = alpha op(A) op(B) + beta C (FP64 DMMA GEMM); core.py:309-319 matmul_counted. */
int pevd_dgemm(int transA, int transB, int64_t m, int64_t n, int64_t k, double alpha,
               const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
               int64_t ldc, void* workspace, int64_t workspace_bytes, void* stream);

/* C = alpha A B + beta C with A symmetric (m x m) read from its lower triangle only
 * (the A W product of form_z, sbr.py:119-130). */
int pevd_dsymm_lower(int64_t m, int64_t n, double alpha, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                     void* workspace, int64_t workspace_bytes, void* stream);

/* Householder panel QR, sbr.py:69-116.  P (m x k, ldp) read; R (k x k), Y (m x k, ldy),
 * W (m x k, ldw), T (k x k) written (any output may be NULL except Y).  k <= 32. */
int64_t pevd_panel_qr_workspace_bytes(void);
int pevd_panel_qr(int64_t m, int k, const double* P, int64_t ldp, double* R, double* Y,
                  int64_t ldy, double* W, int64_t ldw, double* T, void* workspace, void* stream);

/* Band reduction sbr.py:155-188: A (n x n, lda, lower triangle) -> bands ((b+1) x n, C order,
 * bands[d*n + j] = A[j+d, j], core.py:118-135).  A becomes the explicit-Y staircase, Tall
 * (rounds x b x b) receives the panels' T factors (may be NULL). */
int64_t pevd_sbr_workspace_bytes(int64_t n, int b);
int pevd_sbr(int64_t n, int b, double* A, int64_t lda, double* bands, double* Tall,
             void* workspace, void* stream);

/* Bulge chasing bulge.py:299-309: bands -> d (n), e (n-1); reflectors (tau, V with stride vld)
 * in fixed slots, canonical chase-step-major order (bulge.py:51-60): slot(i, j) =
 * j (n-2) - b j (j-1)/2 + i; tau = 0 marks a step the reference skips.  tau/V may be NULL. */
int64_t pevd_bc_num_reflectors(int64_t n, int b);
int64_t pevd_bc_workspace_bytes(int64_t n, int b);
int pevd_bc(int64_t n, int b, const double* bands, double* d, double* e, double* tau, double* V,
            int vld, void* workspace, void* stream);

/* Tridiagonal divide and conquer (replaces tridiag_eig, tridiag.py:298-334): d in/out (lam
 * ascending), e (n-1) preserved, Q (n x n, ldq) eigenvectors with the reference sign convention.
 * Synchronous (returns PEVD_ERR_CONVERGE on non-convergence). */
/* bc_reduce_partition (bulge.py:348-385): chase the sweeps [0, sweep_end) down a band of
 * semi-bandwidth bw <= 2b (the tail relayed by the predecessor, columns renumbered from the
 * partition start); band_out ((2b+1) x n, bands[d, j] layout) receives the band afterwards
 * (finished rows + residual fill of the tail); reflectors in the pevd_bc slot layout of size n. */
int pevd_bc_partition(int64_t n, int b, int bw, const double* bands, int64_t sweep_end,
                      double* band_out, double* tau, double* V, int vld, void* workspace,
                      void* stream);
int64_t pevd_stedc_workspace_bytes(int64_t n);
int pevd_stedc(int64_t n, double* d, const double* e, double* Q, int64_t ldq, void* workspace,
               void* stream);

/* SBR-Back: Qs (n x n, ldq) = prod_x (I - Y_x T_x Y_x^T) (backtrans.py:128-192). */
/* pevd_stedc restricted to the eigenvector columns [col_lo, col_hi) (all eigenvalues; the other
 * columns of Q are left zero): the top-level merge GEMM only forms the wanted columns, as the
 * distributed conventional order needs for a rank's column block. */
int pevd_stedc_cols(int64_t n, double* d, const double* e, double* Q, int64_t ldq, int64_t col_lo,
                    int64_t col_hi, void* workspace, void* stream);
int64_t pevd_sbr_back_workspace_bytes(int64_t n, int b);
/* Ystair: the Y staircase pevd_sbr / pevd_syevd_device leave in A (leading dimension ldy = lda). */
int pevd_sbr_back_form(int64_t n, int b, const double* Ystair, int64_t ldy, const double* Tall,
                       double* Qs, int64_t ldq, void* workspace, void* stream);
/* X (n x ncols, ldx) <- Q_s X (conventional order, pipeline.py:380-384). */
int pevd_sbr_back_left(int64_t n, int b, const double* Ystair, int64_t ldy, const double* Tall,
                       double* X, int64_t ldx, int64_t ncols, void* workspace, void* stream);

/* BC-Back backtrans.py:277-310.  right: X (nrows x n, ldx) <- X Q_b ("reordered", i.e. the
 * transpose of Q_b^T X^T).  left: X (n x ncols, ldx) <- Q_b X ("conventional"; for the DMMA
 * bandwidths b in {8, 16, ..., 64} it runs on X^T in the workspace, the kernel's coalesced
 * layout; other b apply the reflectors one by one).  The workspace
 * (pevd_bc_back_workspace_bytes(n, rows or cols, b)) holds scheduler counters, the (V, Z)
 * records of the reflector blocks and that transpose. */
int64_t pevd_bc_back_workspace_bytes(int64_t n, int64_t nrows, int b);
int pevd_bc_back_right(int64_t n, int b, const double* tau, const double* V, int vld, double* X,
                       int64_t ldx, int64_t nrows, void* workspace, void* stream);
int pevd_bc_back_left(int64_t n, int b, const double* tau, const double* V, int vld, double* X,
                      int64_t ldx, int64_t ncols, void* workspace, void* stream);

/* ---------------------------------------------------------------- multi-GPU entry points
 * The reference's `run(a, PipelineConfig(workers=G))` (pipeline.py:511-548) with G cooperating
 * devices and the paper's blockwise column distribution (schedule.py:21-33).  col_lo (G+1) is
 * the SBR column partition (`partition(n, G)`), back_lo (G+1) the back-transform partition
 * (`back_plan_sizes`, backtrans.py:108-121): columns of Q in conventional order, rows otherwise.
 * b <= 32. */

/* 128-byte NCCL unique id (rank 0 creates it; the caller shares it, e.g. over torch.distributed). */
int pevd_nccl_unique_id(char* out128);
/* One process per GPU: an NCCL communicator for this rank (the current CUDA device). */
int pevd_comm_nccl_create(int rank, int size, const char* id128, void** comm);
void pevd_comm_destroy(void* comm);

/* One rank of the distributed EVD (every rank calls it; device pointers).  blk: this rank's
 * column block [col_lo[r], col_lo[r+1]) with all n rows (n x w, ldb; destroyed).  lam: n (every
 * rank).  Q: conventional -> the rank's back columns (n x nb, ldq, Fortran order); pipelined /
 * sequential -> the rank's back rows stored as an n x nb column-major block (the rows of Q in C
 * order).  Synchronous. */
int pevd_dist_syevd(void* comm, int64_t n, int b, double* blk, int64_t ldb, const int64_t* col_lo,
                    const int64_t* back_lo, double* lam, double* Q, int64_t ldq, int want_vectors,
                    int order, void* stream, pevd_dist_stats* stats);

/* One process, G workers (one host thread each) on devices devs[0..G) (entries may repeat: workers
 * then share a GPU), peer-to-peer transfers over NVLink.  HOST buffers: A column-major (lda),
 * lam (n), Q n x n: Fortran order in conventional order, C order otherwise (pipeline.py:495,503).
 * stats: G entries (may be NULL). */
int pevd_syevd_multi(int G, const int* devs, int64_t n, int b, const double* A, int64_t lda,
                     const int64_t* col_lo, const int64_t* back_lo, double* lam, double* Q,
                     int want_vectors, int order, pevd_dist_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* PEVD_H */
