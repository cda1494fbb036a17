/*
 * egsolve.h — C ABI of the B200-native mixed-precision BiCGStab Helmholtz solver.
 *
 * Implements the hot path of Maynard & Walters, "Precision of the ENDGame: Mixed-precision
 * arithmetic in the iterative solver of the Unified Model" (arXiv 1811.03852).  Citations "P:L"
 * are lines of the paper's text; "A-n" are the readings listed in DESIGN.md §Readings.
 *
 *   A x = b                                (Eq. 1)  pressure-correction / Helmholtz system
 *   D_g^-1 A C C^-1 x = D_g^-1 b           (Eq. 5) diagonal scaling outside the solver,
 *                                           right ("post-") preconditioned BiCGStab
 *   C^-1 = T^-1, T the vertical tridiagonal of Ahat (Eq. 6; reading A-3)
 *   halt when R = ||r|| / ||b|| < R_c      (Eq. 8-9)
 *   MIXED: x 64-bit, matrix / vectors / arithmetic / halos 32-bit, global sums 64-bit
 *          (P:151-154); mandatory restart every 150 iterations.
 *
 * Every step runs in this library's sm_100a kernels; there is no CPU fallback.  No torch or CUDA
 * types cross this boundary: device buffers are plain pointers, streams are `void*`
 * (a cudaStream_t), sizes are int64_t / size_t.
 *
 * GRID AND LAYOUT.  nx longitudes (periodic, nx >= 3), ny latitudes (zero-flux at j = 0 and
 * j = ny-1), nz levels (zero-flux at k = 0 and k = nz-1).  Every field — bands, b, x, vectors —
 * is stored longitude-fastest ("IKJ"):  q = i + nx*(k + nz*j_local),  j_local = j - j_begin.
 * A latitude row is one contiguous block of nx*nz values, so a latitude band is one contiguous
 * chunk.  (The paper fixes no layout; DESIGN.md §Layout explains the choice.)
 *
 * BANDS.  Seven unscaled fp64 coefficient arrays in the order C (diagonal), E (i+1), W (i-1),
 * N (j+1), S (j-1), U (k+1), D (k-1); band d at point q multiplies x at neighbour d of q.
 * A band at an absent neighbour (N at j = ny-1, S at j = 0, U at k = nz-1, D at k = 0) must be 0.
 *
 * THREADING.  One handle is not thread-safe; separate handles are independent.  All device work
 * is ordered on the stream given to eg_solver_create.  The fused phase kernels keep
 * one CTA per SM and synchronise CTAs through ready flags, which needs every CTA of a launch
 * resident: they are launched COOPERATIVELY, so the runtime either makes the whole grid resident or
 * fails the launch (EG_ERR_CUDA), never a partly resident grid that waits forever — also with MPS
 * or other work on the GPU.  Concurrent eg_solve / eg_solve_batch calls of handles that use them
 * are additionally serialised per device inside this process (they block until done anyway).
 */
#ifndef EGSOLVE_H
#define EGSOLVE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (returned by every int function; 0 = success) ---- */
#define EG_OK 0
#define EG_ERR_ARG 1             /* invalid argument / grid / decomposition / layout            */
#define EG_ERR_SINGULAR_DIAG 2   /* some a_C is 0 or non-finite                         */
#define EG_ERR_DEGENERATE_RHS 3  /* ||D_g^-1 b|| = 0                                    */
#define EG_ERR_BREAKDOWN 4       /* two consecutive BiCGStab breakdowns without progress (A-12) */
#define EG_ERR_NONFINITE 5       /* non-finite value in the iteration               */
#define EG_ERR_CUDA 6            /* CUDA runtime error (see eg_last_error)                      */
#define EG_ERR_NCCL 7            /* NCCL error (see eg_last_error)                              */
#define EG_ERR_WORKSPACE 8       /* workspace too small or misaligned                           */

typedef struct eg_solver eg_solver;

typedef struct {
    int64_t nx, ny, nz; /* GLOBAL grid */
} eg_grid;

/* Precision policy (Table 1 "Mixed-precision" vs "Double precision").
 *   EG_FP64  : everything binary64 ("DP").
 *   EG_MIXED : x binary64; scaled bands, Krylov vectors, their arithmetic and the halo exchange
 *              binary32; global sums binary64 ("MP" after the 64-bit-sum fix).
 *   EG_FP32  : everything binary32 including the global sums (the original MP sums / toy SP). */
typedef enum { EG_FP64 = 0, EG_MIXED = 1, EG_FP32 = 2 } eg_precision;

/* Latitude-band decomposition over nranks GPUs (one process per GPU).  Rows [j_begin, j_end) are
 * local.  NULL = one GPU owning all rows.  With nranks > 1 the bands must be contiguous in rank
 * order and aligned to the 8 fixed reduction row-groups (group g = rows [g*ny/G, (g+1)*ny/G),
 * G = min(8, ny)), i.e. nranks must divide G; that fixed grouping makes every global sum — and
 * so x and the history — bitwise identical for any nranks.  nccl_unique_id points to the 128-byte
 * ncclUniqueId from eg_nccl_unique_id() on rank 0, broadcast by the caller (NULL if nranks == 1),
 * or to an id from eg_loopback_id() (the in-process test transport, below). */
typedef struct {
    int64_t j_begin, j_end;
    int32_t rank, nranks;
    const void* nccl_unique_id;
} eg_dist;

/* flags for eg_solve_params.flags */
#define EG_SOLVE_NO_GRAPH 1u  /* launch each kernel directly instead of replaying a CUDA graph  */
#define EG_SOLVE_PROFILE 2u   /* record CUDA events around every kernel (implies NO_GRAPH);     */
                              /* read with eg_profile_get                                       */

typedef struct {
    double tol;             /* R_c; 0 = no halting criterion, run maxit   */
    int32_t maxit;          /* >= 0                                                          */
    int32_t restart_every;  /* mandatory restart period (P:553-557, 150 in the UM); <= 0 off */
    uint32_t flags;         /* EG_SOLVE_*                                                    */
    int32_t check_every;    /* iterations between host polls of the device flags; 0 = auto   */
    const double* rhat0;    /* NULL (default): the shadow residual of BiCGStab is rhat0 = r0    */
                            /* (reading A-1).  Else a DEVICE fp64 array of the local rows, used */
                            /* (rounded to the working precision) as rhat0 at the FIRST start   */
                            /* only; restarts set rhat0 = r (A-11).  If rho = rhat0 . r0 fails  */
                            /* the breakdown test (A-12: 0, non-finite, or |rho| < eps_V        */
                            /* ||rhat0|| ||r0||) the solve restarts at once with rhat0 = r0.    */
                            /* (BiCGStab leaves rhat0 free; used to inject breakdowns in tests.) */
} eg_solve_params;

typedef struct {
    int32_t iters;       /* completed BiCGStab iterations (an s-step exit counts, A-7/A-8)   */
    int32_t converged;   /* 1 iff the verified true residual R_true < tol (A-6)             */
    int32_t restarts;    /* mandatory + breakdown + failed-verification restarts             */
    int32_t breakdowns;  /* scalar-weight breakdowns (A-12)                                  */
    int32_t status;      /* same code eg_solve returns                                       */
    double final_R;      /* last recorded R (history[iters])                                 */
    double true_R;       /* ||bhat - Ahat x|| / ||bhat|| recomputed with fp64 accumulation   */
} eg_solve_info;

/* Bytes of device workspace the caller must provide to eg_solver_create for this grid, local
 * band and precision (PyTorch owns all device memory).  Returns EG_OK or EG_ERR_ARG. */
int eg_workspace_bytes(const eg_grid* grid, const eg_dist* dist, eg_precision prec, size_t* bytes);

/* Same, for a solver that will also use optional features.  features: bit mask of
 *   EG_FEATURE_TRISOR: room for colour-split copies of the scaled bands, of the preconditioner's
 *     right-hand side and of the sweeps' iterate (8 working-precision values per point plus two
 *     ghost rows), which the red-black tri-SOR sweeps
 *     (EG_PRECOND_TRISOR) read instead of every other value of the natural-order arrays.  A solver
 *     created with this feature (eg_solver_create_ex) uses them; without it tri-SOR still runs, on
 *     the natural-order arrays (same results, bitwise).
 * features = 0 gives eg_workspace_bytes.  Returns EG_OK or EG_ERR_ARG. */
#define EG_FEATURE_TRISOR 1u
/*   EG_FEATURE_BATCH: room for two device staging buffers each of b and x (4 fp64 values per point)
 *     used by eg_solve_batch. */
#define EG_FEATURE_BATCH 2u
int eg_workspace_bytes_ex(const eg_grid* grid, const eg_dist* dist, eg_precision prec, uint32_t features,
                          size_t* bytes);

/* a1 — create a solver: scales the operator "outside the solver" (Eq. 5):
 * Ahat_d = a_d / a_C (binary64 IEEE division, then rounded to the working precision), the fp64
 * diagonal kept for scaling b.  bands[7]: DEVICE fp64 arrays of the local rows (layout above);
 * read during this call only — the caller may free them after return.  workspace: DEVICE buffer
 * of >= eg_workspace_bytes, 256-byte aligned, owned by the caller, must outlive the solver.
 * stream: the cudaStream_t all work is ordered on.  With dist->nranks > 1 this call is collective
 * (creates the NCCL communicator).  Blocks until the validation flags are read.
 * Errors: EG_ERR_ARG (dims, nx < 3, decomposition, nonzero band at an absent neighbour or
 * non-finite band), EG_ERR_SINGULAR_DIAG, EG_ERR_WORKSPACE, EG_ERR_CUDA, EG_ERR_NCCL.
 * On error *out is NULL. */
int eg_solver_create(const eg_grid* grid, const eg_dist* dist, const double* const bands[7],
                     eg_precision prec, void* workspace, size_t workspace_bytes, void* stream,
                     eg_solver** out);

/* The same with optional features (EG_FEATURE_* bit mask, as passed to eg_workspace_bytes_ex): the
 * workspace must be at least eg_workspace_bytes_ex(grid, dist, prec, features) bytes (else
 * EG_ERR_WORKSPACE), and exactly the requested optional regions are carved from it — a larger
 * workspace never turns a feature on.  eg_solver_create(...) == eg_solver_create_ex(..., 0, ...).
 * Errors: those of eg_solver_create; EG_ERR_ARG for an unknown feature bit. */
int eg_solver_create_ex(const eg_grid* grid, const eg_dist* dist, const double* const bands[7],
                        eg_precision prec, uint32_t features, void* workspace, size_t workspace_bytes,
                        void* stream, eg_solver** out);

/* a1 again on an existing solver: re-scale a NEW operator of the same grid / band / precision into
 * the workspace ("the matrix is time varying and so needs to be recomputed at every time step",
 * P:217-220).  Same inputs, errors and blocking behaviour as eg_solver_create, without allocation
 * or communicator setup.  On error the previous operator is no longer valid. */
int eg_solver_set_operator(eg_solver* s, const double* const bands[7]);

/* NEXT-1 — choose the preconditioner C^-1.
 *   EG_PRECOND_TRIDIAG (default): C^-1 = T^-1, one Jacobi-ordered Eq. 7 sweep from 0 (reading A-3).
 *   EG_PRECOND_TRISOR: `sweeps` sweeps (the UM uses "typically three") of the tri-SOR
 *     fixed point (Eq. 7, over-relaxation `omega`, 1.5 in the UM) from x = 0, columns in
 *     red-black order ((i + j) % 2; L = couplings to already-updated columns, U = to the others).
 *     Requires nx even (periodic 2-colouring), sweeps >= 1, 0 < omega < 2.
 * Applies to eg_solve and eg_precondition.  Errors: EG_ERR_ARG. */
#define EG_PRECOND_TRIDIAG 0
#define EG_PRECOND_TRISOR 1
int eg_solver_set_preconditioner(eg_solver* s, int kind, int sweeps, double omega);

/* y = Ahat x, the scaled operator the solver iterates with (unit diagonal + 6 bands; periodic in i,
 * absent neighbours contribute 0).  x, y: DEVICE arrays of the local rows in the working precision
 * (float for EG_MIXED / EG_FP32, double for EG_FP64).  Exchanges halo rows when distributed
 * (collective).  Stream-ordered; returns without synchronising.  x and y must not overlap (EG_ERR_ARG). */
int eg_apply_operator(eg_solver* s, const void* x, void* y);

/* z = C^-1 r, the applied preconditioner, in the working precision.  EG_PRECOND_TRIDIAG (default):
 * z = T^-1 r per column (reading A-3), T = tridiag(D_k, 1, U_k) of the scaled vertical bands,
 * Thomas recurrence without pivoting (A-14), no communication (no vertical decomposition,
 * P:263-264).  EG_PRECOND_TRISOR: the red-black tri-SOR sweeps from z = 0, which exchange halo rows
 * after every half-sweep when distributed (collective).  Stream-ordered.  r and z must not overlap
 * (EG_ERR_ARG). */
int eg_precondition(eg_solver* s, const void* r, void* z);

/* Solve Ahat x = D_g^-1 b by right-preconditioned BiCGStab (algorithm in DESIGN.md).
 * b: fp64 local rows.  x0: fp64 local rows or NULL (= 0).  x: fp64 output, local rows.
 * b, x0 and x may each be DEVICE or HOST memory (host buffers are copied in / out inside the call).
 * history: HOST array of >= params->maxit + 1 doubles: history[0] = true R of x0,
 * history[i] = R after iteration i (may be NULL).  info: HOST, may be NULL.
 * Blocks until done.  Not converging within maxit is NOT an error (info->converged = 0).
 * Errors: EG_ERR_ARG, EG_ERR_DEGENERATE_RHS, EG_ERR_NONFINITE, EG_ERR_BREAKDOWN, EG_ERR_CUDA,
 * EG_ERR_NCCL; info / history / x stay valid up to the failure point. */
int eg_solve(eg_solver* s, const double* b, const double* x0, const eg_solve_params* params,
             double* x, double* history, eg_solve_info* info);

/* A sequence of `count` solves, e.g. one per time step ("the solver is called ... every time step",
 * P:191-192), with the host <-> device transfers of neighbouring solves overlapped with the solves:
 *   for k = 0 .. count-1:  [eg_solver_set_operator(s, bands) if bands != NULL];
 *                          eg_solve(s, b[k], NULL, params, x[k], history + k*(maxit+1), info + k)
 * b[k], x[k]: fp64 local rows, HOST (pinned memory overlaps; pageable works but is serialised by the
 * driver) or DEVICE.  bands: DEVICE, as for eg_solver_set_operator, or NULL.  history (HOST,
 * count*(maxit+1) doubles) and info (HOST, count entries) may be NULL.  While solve k runs, the
 * upload of b[k+1] and the download of x[k-1] run on the library's own copy streams, staged
 * through two device buffers for b and two for x in the workspace: requires a solver created with
 * EG_FEATURE_BATCH (eg_solver_create_ex; else EG_ERR_WORKSPACE).  Each solve's
 * x / history / info are bitwise those of the individual eg_solve call.  Blocks until every x[k] is
 * written.  Stops at the first failing solve; *done (may be NULL) = the number of solves completed.
 * Errors: those of eg_solve, EG_ERR_ARG, EG_ERR_WORKSPACE. */
int eg_solve_batch(eg_solver* s, int count, const double* const* b, double* const* x,
                   const double* const bands[7], const eg_solve_params* params, double* history,
                   eg_solve_info* info, int* done);

/* Release the NCCL communicator (or the loopback-group membership), the peer mappings of the P2P
 * transport, streams, events and graphs (not the caller's workspace).  With latitude bands the
 * other ranks write into this rank's workspace during solves: destroy a handle (and free its
 * workspace) only once every rank's last collective call on it has returned.  NULL is a no-op. */
void eg_solver_destroy(eg_solver* s);

/* Human-readable detail of the last error on this handle ("" if none).  Valid until the next call. */
const char* eg_last_error(const eg_solver* s);
const char* eg_status_str(int status);

/* Fill out[128] with a fresh ncclUniqueId (call on rank 0, broadcast to the others). */
int eg_nccl_unique_id(char out[128]);

/* In-process loopback transport, for testing the latitude-band decomposition (DESIGN.md
 * §Multi-GPU) on ONE GPU.  Fills out[128] with an id naming a new group of nranks ranks; pass it
 * as eg_dist.nccl_unique_id to exactly nranks eg_solver_create calls in this process (one per
 * rank), all on the same device and the SAME stream (EG_ERR_ARG otherwise).  Every call that
 * exchanges data (eg_apply_operator, tri-SOR eg_precondition, eg_solve, eg_solve_batch) must then
 * be made on all ranks concurrently, one host thread per rank: each halo exchange and group-sum
 * all-gather is a host barrier plus device-to-device copies on the shared stream, so the ranks'
 * kernels run one after another in enqueue order and never wait on each other.  Solves are
 * launched kernel by kernel (no CUDA graph).  A rank that fails or stops calling makes the others'
 * exchange fail with EG_ERR_NCCL after 120 s.  The group is freed with its last member; an id must
 * not be reused after that.  Errors: EG_ERR_ARG (out NULL, nranks < 1). */
int eg_loopback_id(int nranks, char out[128]);

/* ---- the transport of a latitude-band decomposition ----
 * EG_TRANSPORT_P2P (the default for nranks > 1): the kernels that produce the band-edge rows of
 * z / z_s and the reduction groups' sums store them straight into the neighbours' ghost rows and
 * every rank's gather buffer through peer memory (CUDA IPC handles of the workspaces, exchanged at
 * create over NCCL; NVLink / NVSwitch peer access), then stamp flags the consuming kernels wait
 * on: no NCCL call and no copy inside an iteration, which is then one CUDA graph of kernels only.
 * It needs every rank's workspace to be IPC-exportable (cudaMalloc memory, as PyTorch's default
 * allocator gives) and peer access between all ranks; otherwise — or with the environment variable
 * EG_P2P=0 — the handle keeps EG_TRANSPORT_NCCL (send / recv of ghost rows on a side stream,
 * ncclAllGather of the group sums).  All ranks agree on the choice (collective at create).  A wait
 * that a peer never satisfies ends the solve with EG_ERR_NCCL after EG_P2P_TIMEOUT_MS (default
 * 60000) instead of hanging.  The loopback test transport uses the same P2P kernels on one GPU
 * (EG_TRANSPORT_LOOPBACK_P2P, built at the first solve) or host-barrier copies (EG_P2P=0,
 * EG_TRANSPORT_LOOPBACK).  Results are bitwise identical under every transport.  The tri-SOR
 * preconditioner's halo after each red-black half-sweep (it needs every rank created with the
 * same features) and the ghost rows of x before a restart / the verification go the same way, as
 * a push kernel and a wait kernel.  eg_apply_operator keeps the NCCL / copy exchange, which the
 * receiver writes itself: consecutive applies have no global sum between them that would keep a
 * pushing neighbour from overwriting a ghost row not yet read. */
#define EG_TRANSPORT_NONE 0          /* one GPU, no exchange                               */
#define EG_TRANSPORT_NCCL 1
#define EG_TRANSPORT_P2P 2
#define EG_TRANSPORT_LOOPBACK 3
#define EG_TRANSPORT_LOOPBACK_P2P 4
int eg_solver_transport(const eg_solver* s);

/* Test hooks for the P2P transport's CUDA IPC step (the one part of it a single-GPU box can check
 * across processes).  eg_debug_ipc_export: the 80-byte record (IPC handle of the allocation that
 * contains ptr, ptr's offset in it) that the NCCL ranks all-gather at create; EG_ERR_CUDA if the
 * memory cannot be exported (e.g. cuMemCreate-backed).  eg_debug_ipc_open, in another process:
 * *ptr = the same bytes as mapped here (peer access enabled lazily), *opened = the mapping to pass
 * to eg_debug_ipc_close.  Errors: EG_ERR_ARG, EG_ERR_CUDA. */
int eg_debug_ipc_export(const void* ptr, unsigned char out[80]);
int eg_debug_ipc_open(const unsigned char in[80], void** ptr, void** opened);
int eg_debug_ipc_close(void* opened);

/* ---- kernel-level profiling (EG_SOLVE_PROFILE): CUDA events on the solver's stream ---- */
int eg_num_kernels(void);
const char* eg_kernel_name(int kernel_id);
/* Accumulated device time (ms) and launch count of one kernel since the last reset, and its
 * ALGORITHMIC HBM bytes per launch for this solver's grid / precision. */
int eg_profile_get(const eg_solver* s, int kernel_id, double* total_ms, int64_t* launches,
                   double* alg_bytes_per_launch);
int eg_profile_reset(eg_solver* s);

#ifdef __cplusplus
}
#endif
#endif
