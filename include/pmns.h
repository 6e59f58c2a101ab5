/*
 * pmns.h — C ABI of the B200 gPLMM-preconditioned Newton-FGMRES library
 * (arXiv 2510.22077, Li & Mehmani, "Preconditioning and Reduced-Order
 * Modeling of Navier-Stokes Equations in Complex Porous Microstructures").
 *
 * Citations: "P:n" = line n of the paper's PAPER.md (LaTeX source) with the
 * section / equation label; readings A*, D* refer to DESIGN.md §3 (they
 * follow SURVEY.md §8(c)).
 *
 * Conventions
 *  - Every entry point returns pmns_status; no C++ exception crosses the ABI.
 *    On a non-OK status, pmns_last_error() returns a thread-local message.
 *  - Device vectors are fp64 arrays of length N = n_f + n_c in DEVICE ORDER
 *    (the permutation W of Eq. permute: unknowns grouped by primary
 *    grid, then interface cells, then interface faces).  pmns_export_layout
 *    gives the map device slot -> canonical index; pmns_permute converts.
 *  - Canonical order (for host-side users): x-face DOFs by i+(nx+1)(j+ny k),
 *    then y-face DOFs by i+nx(j+ny k) (face j = low-y face of cell j), then
 *    z-faces likewise, then cells by i+nx(j+ny k).
 *  - The caller owns every pointer it passes; device pointers must stay
 *    valid until the given stream has passed the call.  The library owns all
 *    internal allocations (made in create/build, freed in destroy).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - CUDA failures are sticky: after PMNS_ECUDA the context must be destroyed.
 */
#ifndef PMNS_H
#define PMNS_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PMNS_OK = 0,
  PMNS_EINVAL = 1,     /* bad argument */
  PMNS_ENONPERC = 2,   /* no void connected to the inlet/outlet planes (reading D1) */
  PMNS_ESINGULAR = 3,  /* a local or coarse block is singular (reading A20) */
  PMNS_ENOCONV = 4,    /* Krylov or Newton iteration limit; best iterate written */
  PMNS_EDIVERGED = 5,  /* Newton residual grew > 10x its minimum */
  PMNS_ENOMEM = 6,
  PMNS_ECUDA = 7,
  PMNS_ENCCL = 8,      /* a collective or halo exchange failed (NCCL); sticky, destroy the context */
  PMNS_ESTATE = 9      /* call out of order (e.g. solve before build) */
} pmns_status;

/* Problem statement: binary image, rho, mu, body force,
 * inlet/outlet pressure, optional backward-Euler dt.  SI units. */
typedef struct {
  int32_t dim;              /* 2 or 3; flow axis is x */
  int64_t n[3];             /* nx, ny, nz (nz = 1 in 2D) */
  const uint8_t *solid;     /* HOST, nx*ny*nz, x fastest, 1 = grain, 0 = void; read during create */
  double h, rho, mu;        /* voxel edge [m], density [kg/m^3], viscosity [Pa s] */
  double body_force[3];     /* b [m/s^2] */
  double p_in, p_out;       /* [Pa] at ghost cell centres h/2 outside x-min / x-max (reading A3) */
  uint32_t periodic;        /* bit 0 => y periodic, bit 1 => z periodic (x is never periodic) */
  double dt;                /* 0 => steady; > 0 => backward Euler (reading A7) */
  double ws_merge_h;        /* watershed merge threshold h_m [voxels] (reading D5) */
  int32_t ws_min_cells;     /* small-basin threshold n_min (reading D5) */
  int32_t dual_layers;      /* dual-grid dilation steps k_d (reading D8; configs use 1) */
  int32_t mask_band;        /* inertia-mask band width (reading D9) */
} pmns_problem;

typedef struct pmns_ctx pmns_ctx;

typedef struct {
  int64_t n_c, n_f, N;      /* pressure cells, face velocities, total unknowns */
  int64_t n_p, n_iface;     /* primary grids N^p, contact interfaces N^c (= N^d) */
  int64_t n_coarse;         /* N^c + N^p_B (coarse unknowns, reading A15); 0 before build */
  int64_t nx, ny, nz;
  int64_t dual_unknowns;    /* sum of dual-block sizes */
  int64_t mp_bytes, md_bytes, coarse_bytes, prolong_bytes;  /* stored local operators (after build) */
  int64_t raw_basins;       /* watershed basins before merging (D3) */
  int64_t h2d_bytes;        /* bytes uploaded host->device by pmns_create */
  int64_t rank, world;      /* pmns_set_comm (1 rank by default) */
  int64_t own_lo, own_hi;   /* owned primaries [own_lo, own_hi) of this rank */
} pmns_sizes;

typedef struct {
  double newton_tol;        /* ||r(x)|| / ||b0|| (reading A23), default 1e-8 */
  double krylov_tol;        /* ||r + J d|| / ||b0||, default 1e-9 */
  int32_t restart;          /* FGMRES restart m (reading A21), default 50 */
  int32_t max_krylov;       /* per Newton step, default 2000 */
  int32_t max_newton;       /* default 30 */
  int32_t variant;          /* 0 = gPLMM (default), 1 = aPLMM_S, 2 = aPLMM_NS (see solve_steady) */
} pmns_solve_opts;

typedef struct {
  int32_t newton_iters;     /* Newton steps taken (linear solves) */
  int32_t converged;
  int32_t krylov_iters[64]; /* FGMRES iterations per Newton step */
  double res_hist[65];      /* ||r(x^k)|| / ||b0|| for k = 0..newton_iters */
  double b0_norm;
  double t_mg_ms, t_ml_ms, t_sol_ms;   /* build M_G, build M_L (factorisations), Krylov */
  int32_t builds;           /* preconditioner builds performed */
  int32_t total_krylov;
  int64_t kernel_launches;  /* library kernels launched during the call */
  int32_t n_steps;          /* transient: time steps completed */
  int32_t step_newton[64];  /* transient: Newton steps per time step */
  double t_setup_ms;        /* pmns_create host set-up (S1/S2) of this context */
  int64_t bytes_per_iter;   /* the library's stored bytes streamed per FGMRES iteration (M_p + M_d + coarse +
                               shape vectors + 3 J applies + CGS2 at the mean basis size); SURVEY 8(d)'s
                               algorithmic bytes are computed by bench.py from the oracle's factor nnz */
  int32_t failed_subdomain; /* ESINGULAR: the block / front id named by the failure, else -1 */
} pmns_report;

/* Setup (S1/S2): clean-up, decomposition D1-D10, numbering, device layout.
 * Host work + upload.  *out owns the device data.  device < 0 creates a
 * host-only context (setup + pmns_query/pmns_export_layout/pmns_halo_plan
 * only; every device call then returns PMNS_ESTATE).  SURVEY 8(b) passes the
 * distribution (pmns_dist) here; this library takes the device id here and
 * the rank/world/transport in pmns_set_comm / pmns_set_comm_loopback, one
 * call for both transports. */
pmns_status pmns_create(const pmns_problem *prob, int32_t device, pmns_ctx **out);
void pmns_destroy(pmns_ctx *ctx);
const char *pmns_last_error(void);

pmns_status pmns_query(const pmns_ctx *ctx, pmns_sizes *out);

/* Memory plan (SURVEY 8(d) sizing; DESIGN.md section 8 memory budget): what
 * the local operators of Eq. Mp_Md will occupy once built and
 * what one factorisation costs, from the structural nested-dissection plans
 * alone (no numeric build; joins the layout thread pmns_create started).
 * HOST struct written.  PMNS_ESTATE on a host-only context. */
typedef struct {
  int64_t mp_bytes, md_bytes;       /* stored M_p / M_d operators [bytes] */
  double mp_flops, md_flops;        /* flops of one factorisation of each */
  int64_t mp_fronts, md_fronts;     /* nested-dissection fronts */
  int64_t mp_max_pivots, mp_max_boundary, mp_levels;
  int64_t krylov_bytes;             /* FGMRES(50) bases V and Z */
  int64_t index_bytes;              /* per-row stencil table + row position/mask */
  int64_t max_primary_unknowns;     /* largest primary block */
  int64_t stencil_runs;             /* maximal runs of consecutive rows whose stencil codes advance together
                                       (N / stencil_runs = mean run length of a run-length coded table) */
} pmns_memplan;
pmns_status pmns_memory_plan(pmns_ctx *ctx, pmns_memplan *out);

/* Host exports (bit-exact integer parity, reading D1-D10):
 * perm[N]: canonical index of each device slot; labels[nvox]: primary id or
 * -1; iface[nvox]: interface id or -1; dual_ptr[n_iface+1] / dual_cells[...]:
 * flat voxel indices of each dual grid (pass NULL to skip any). */
pmns_status pmns_export_layout(const pmns_ctx *ctx, int64_t *perm, int32_t *labels, int32_t *iface,
                               int64_t *dual_ptr, int64_t *dual_cells, uint8_t *mask_faces_canonical);

/* dst = src permuted: dir = 0 canonical -> device order, 1 device -> canonical. Device pointers. */
pmns_status pmns_permute(pmns_ctx *ctx, const double *src, double *dst, int32_t dir, void *stream);

/* a1: r(x) (Eq. Ax=b with Eq. mod_res w = u; readings A3-A8).  u_prev may be NULL (steady). */
pmns_status pmns_residual(pmns_ctx *ctx, const double *x, const double *u_prev, double *r, void *stream);

/* a2: y = J(x^k) v (reading A9: exact Jacobian, upwind selector frozen). */
pmns_status pmns_apply_jacobian(pmns_ctx *ctx, const double *xk, const double *v, double *y, void *stream);

/* y = b - J(x_k) v: the fused form of the same apply used inside the
 * preconditioner (Eq. mono_struct steps s = v - J z_G and t = s - J z_d,
 * the residual update costs one more 8N read instead of a
 * separate pass).  Same layout, ownership and errors as pmns_apply_jacobian;
 * b must not alias y. */
pmns_status pmns_apply_jacobian_fused(pmns_ctx *ctx, const double *xk, const double *v, const double *b, double *y,
                                      void *stream);

/* y = J~_w v (Eq. mod_res; reading A10): Oseen with wind w = u(w_state),
 * inertia removed on the mask band.  Used to build M_G; exported for tests. */
pmns_status pmns_apply_jacobian_modified(pmns_ctx *ctx, const double *w_state, const double *v, double *y,
                                         void *stream);

/* B1 + B2: build gPLMM.  M_G from J~_w with w = u(x_b); M_L local
 * blocks from J(x_b) (reading A17).  x_b == NULL => x_b = 0 (Stokes, = aPLMM_S,
 * P:763).  Replaces any previous build. */
pmns_status pmns_build_preconditioner(pmns_ctx *ctx, const double *x_b, void *stream);

/* z = M^{-1} v (Eq. mono_struct, n_st = 1, M_l = M_dp) with J(xk) as the
 * matrix of the composition steps s = v - J z_G, t = s - J z_d.  The Newton
 * solvers pass xk = x_b, the build state (reading A18 as revised in DESIGN.md
 * R9: Eq. mono_struct / Mdp use the same A^ as the local blocks of Eq. Mp_Md,
 * and the preconditioner is built once before the Newton loop); any
 * other state gives the round-1 composition with the current Jacobian. */
pmns_status pmns_apply_preconditioner(pmns_ctx *ctx, const double *xk, const double *v, double *z, void *stream);
/* z = M_G^{-1} v (Eq. iMG with Remark 1). */
pmns_status pmns_apply_mg(pmns_ctx *ctx, const double *v, double *z, void *stream);

/* Newton with the current preconditioner (Eq. Ax=b; readings A21-A23).  x is
 * the initial guess on entry, the iterate on exit.  u_prev: previous time
 * level (required iff dt > 0). */
pmns_status pmns_newton_solve(pmns_ctx *ctx, double *x, const double *u_prev, const pmns_solve_opts *opts,
                              pmns_report *rep, void *stream);

/* The steady pipeline (reading A19): build with x_b = 0, one Newton step
 * (the Stokes solve), rebuild with x_b = x^1 (wind = Stokes velocity),
 * Newton to convergence.  x: device, output (input ignored; starts at 0).
 * opts->variant selects the preconditioner family: gPLMM (M_G from
 * J~_w, rebuilt after step 0); aPLMM_S (the step-0 Stokes build reused for
 * every Newton step); aPLMM_NS (rebuilt after step 0 with M_G from the plain
 * Jacobian J(x^1): no wind linearisation, no inertia mask). */
pmns_status pmns_solve_steady(pmns_ctx *ctx, double *x, const pmns_solve_opts *opts, pmns_report *rep,
                              void *stream);

/* The transient pipeline (reading A7/A19, SURVEY config 4; "rebuilt ...
 * not in between dt steps or Newton iterations"): Newton step 0 of the steady
 * problem gives the Stokes state x_S; ONE build from x_S (wind u(x_S), M_L
 * from J(x_S), rho/dt included); then n_steps backward-Euler steps, each a
 * Newton solve from x^n with u^n = x^n.  Requires dt > 0.  x: device, in =
 * u^0 state (e.g. zeros = from rest), out = state after n_steps. */
pmns_status pmns_solve_transient(pmns_ctx *ctx, double *x, int32_t n_steps, const pmns_solve_opts *opts,
                                 pmns_report *rep, void *stream);

/* Re continuation (homotopy): drive increments k = 1..n_incr
 * (p_in, p_out, b scaled by k/n_incr).  Increment 1 = pmns_solve_steady;
 * increment k >= 2 rebuilds gPLMM once at its start with the previous
 * solution as wind and M_L state, then Newton from that solution.
 * report: step_newton[k] = Newton steps of increment k, krylov_iters in
 * order; res_hist[k] = final ||r||/||b0|| of increment k. */
pmns_status pmns_solve_continuation(pmns_ctx *ctx, double *x, int32_t n_incr, const pmns_solve_opts *opts,
                                    pmns_report *rep, void *stream);

/* Coarse-scale steady Navier-Stokes solver, Algorithm 1: drive
 * increments k = 1..n_ramp (p_in, p_out, b scaled by k/n_ramp); per
 * increment an M_G-only build from J~_w with the previous increment's
 * velocity (w = 0 first: Stokes fallback), then Newton on the coarse
 * unknowns only: r_c = R^ r~(x^), J_c = R^ J~^k P^, x^ += P^ delta_c, until
 * ||r_c|| / ||r_c^0|| < opts->newton_tol (default 1e-6), at most max_newton
 * (default 50).  x (device, out) = the approximate fine-scale solution x^.
 * report: step_newton[k] = Newton iterations of increment k. */
pmns_status pmns_coarse_solve(pmns_ctx *ctx, double *x, int32_t n_ramp, const pmns_solve_opts *opts,
                              pmns_report *rep, void *stream);

/* Same with HOST buffers (canonical order), copies inside (the e2e path). */
pmns_status pmns_solve_steady_host(pmns_ctx *ctx, double *x_host_canonical, const pmns_solve_opts *opts,
                                   pmns_report *rep);
/* pmns_solve_continuation with HOST buffers (canonical order, copies inside;
 * n_incr == 1 is pmns_solve_steady_host): the e2e path of the continuation
 * pipeline (config 3). */
pmns_status pmns_solve_continuation_host(pmns_ctx *ctx, double *x_host_canonical, int32_t n_incr,
                                         const pmns_solve_opts *opts, pmns_report *rep);
/* pmns_solve_transient from rest (x^0 = 0) with a HOST output buffer
 * (canonical order, the D2H copy inside): the e2e path of the transient
 * pipeline (config 4). */
pmns_status pmns_solve_transient_host(pmns_ctx *ctx, double *x_host_canonical, int32_t n_steps,
                                      const pmns_solve_opts *opts, pmns_report *rep);

/* Live kernel timing with CUDA events on the launching stream.  kind:
 * 0 = M_p local-solve GEMV launches (a9, the dominant kernel: every level
 * sweep of the nested-dissection fronts), 1 = M_d GEMV (a7), 2 = Jacobian
 * apply (a2/a6/a8/a10), 3 = one whole M_p apply, 4 = one whole M_d apply,
 * 5 = one whole preconditioner apply M^{-1} (a3-a9 inside FGMRES; bytes 0:
 * the caller supplies SURVEY §8(d)'s B_M).  Kinds 3-5 time the production
 * path (the captured level-sweep graphs); kinds 0/1 record per launch only
 * with PMNS_PROF_LAUNCHES=1.  pmns_profile(ctx, 1) clears and enables
 * the record; pmns_profile_query sums the recorded launches of one kind
 * (count, device milliseconds, algorithmic bytes per SURVEY §8(d)). */
pmns_status pmns_profile(pmns_ctx *ctx, int32_t enable);

/* Multi-GPU (one process per GPU).  pmns_comm_unique_id fills a
 * 128-byte NCCL unique id (call on rank 0, broadcast the bytes to every rank,
 * e.g. with torch.distributed).  pmns_set_comm(ctx, rank, world, id) must be
 * called on every rank before the first build: the primaries are split into
 * `world` contiguous ranges (primary ids follow the z-major first voxel, so
 * ranges are slabs) balanced by sum n_i^2; rank r factorises and applies only
 * the M_p / folded-Abar local solves of its range (Eq. Mp_Md, Eq. prolong_2/3)
 * and the M_d solves of a contiguous, n^2-balanced range of dual grids;
 * everything else (J, M_G, FGMRES) is replicated.  The owned M_p output and
 * shape vectors are combined with ncclAllReduce over disjoint supports
 * (exact); the M_d output (overlapping duals) with ncclAllReduce(sum), which
 * returns the same bits to every rank, so every rank holds identical iterates.
 * id == NULL with world > 1 gives a partition-only context (no communicator,
 * no coarse solver: for testing the partition with pmns_apply_mp).  Errors:
 * EINVAL (bad rank/world), ECUDA (NCCL). */
pmns_status pmns_comm_unique_id(uint8_t *out128);
pmns_status pmns_set_comm(pmns_ctx *ctx, int32_t rank, int32_t world, const uint8_t *id128);

/* In-process loopback transport for the multi-rank path on ONE device: create
 * a group of `world` virtual ranks, then call pmns_set_comm_loopback on one
 * context per rank, each driven by its own host thread (all collectives of a
 * solve are entered by every rank in the same order).  Exchanges are
 * host-synchronised device copies: no kernel ever waits on another.  The group
 * must outlive its contexts.  Used by the tests; a real run uses NCCL
 * (pmns_set_comm).  Errors: EINVAL (bad rank/world or a world mismatch). */
/* Host-side multi-GPU plan of rank `rank` of `world` (no device needed; the
 * same computation pmns_set_comm performs): counts[4 p + q] = number of slots
 * (device order) in list q with peer p -- q = 0 forward halo received from p,
 * 1 forward halo sent to p, 2 dual partial sums sent to p, 3 received from p --
 * then counts[4 world .. 4 world + 5] = this rank's owned ranges [lo, hi) of
 * primary rows, interface cells and interface f-faces.  slots (nullable; size
 * = sum of the 4 world counts) receives the lists in (p, q) order.  Errors:
 * EINVAL. */
pmns_status pmns_halo_plan(pmns_ctx *ctx, int32_t rank, int32_t world, int64_t *counts, int64_t *slots);

void *pmns_loopback_create(int32_t world);
void pmns_loopback_destroy(void *group);
pmns_status pmns_set_comm_loopback(pmns_ctx *ctx, int32_t rank, int32_t world, void *group);

/* z = M_p^{-1} t restricted to this rank's owned primaries (zeros elsewhere;
 * Eq. Mp_Md), device vectors of N doubles in W order, after a build.  No
 * collective: the sum over ranks of pmns_apply_mp equals the one-GPU M_p. */
pmns_status pmns_apply_mp(pmns_ctx *ctx, const double *t, double *z, void *stream);

/* z = M_d^{-1} v over this rank's owned dual grids (Eq. Mp_Md: the additive
 * dual-grid solves, overlapping contributions summed in dual order), device
 * vectors of N doubles in W order, after a build; no collective (with a
 * communicator the preconditioner all-reduces this sum over ranks). */
pmns_status pmns_apply_md(pmns_ctx *ctx, const double *v, double *z, void *stream);

/* Device memory and execution resources are cached process-wide (a caching
 * allocator keyed by device and a pool of build streams), so a context
 * created after another one was destroyed reuses them.  pmns_release_cache
 * returns every cached block and pooled stream that no live context uses to
 * the driver.  Never fails; safe to call at any time from the host. */
void pmns_release_cache(void);
pmns_status pmns_profile_query(pmns_ctx *ctx, int32_t kind, int64_t *count, double *total_ms,
                               int64_t *total_bytes);

/* The library's fp64 GEMM (DMMA tensor path, csrc/dgemm.inc), exposed for
 * tests and rate measurements: C = alpha op(A) B + beta C on `batch`
 * column-major matrices with strides sA, sB, sC (elements); op(A) = A^T if
 * transA != 0.  Device pointers; no context needed.  This is the contraction
 * of the build-time dense front updates and Schur inversions (the "LU of
 * local systems" cost T_ML).  EINVAL on negative sizes or
 * k = 0 with beta != 1. */
pmns_status pmns_dgemm(int32_t transA, int32_t m, int32_t n, int32_t k, double alpha, const double *A, int32_t lda,
                       int64_t sA, const double *B, int32_t ldb, int64_t sB, double beta, double *C, int32_t ldc,
                       int64_t sC, int32_t batch, void *stream);

/* In-place inverse of one n x n column-major device matrix (ld) by the
 * library's blocked Gauss-Jordan with partial pivoting (the local-solve
 * fallback and the coarse matrix A°, Eq. coarse_prob).  Synchronous
 * on `stream`; ESINGULAR if a pivot column is zero.  Exposed for tests. */
pmns_status pmns_dense_inverse(double *A, int32_t n, int32_t ld, void *stream);

#ifdef __cplusplus
}
#endif
#endif
