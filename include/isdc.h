/*
 * isdc.h -- C ABI of the B200 (sm_100a) ISDC hot-path library  libisdc.so
 *
 * Inexact spectral deferred corrections (Speck, Ruprecht, Minion, Emmett, Krause,
 * arXiv:1401.7824; /root/reference/PAPER.md, cited as P:<line>).  Each semi-implicit SDC sweep
 * (Eq. 4) is written in the weighted Mehrstellen form (Eq. 5)
 *
 *     (B_h - dt_m nu L_h) u_{m+1}^{k+1} = B_h v_m + L_h w_m
 *
 * and solved only approximately with L V(nu1,nu2) multigrid cycles (ISDC) or to a tolerance
 * (classical SDC).  Convergence is monitored with the max norm of the (B_h-weighted)
 * SDC residual (reading R15).
 *
 * Conventions shared by every call
 *  - Grid: d in {2,3}; n interior points per direction with n + 1 = 2^p (p >= 2); h = 1/(n+1);
 *    homogeneous Dirichlet data on the unit square/cube.  Periodic grids (grid.bc =
 *    ISDC_BC_PERIODIC, NEXT f3, Burgers P:106-112): n = 2^p points (p >= 2) x_i = -1 + i h of
 *    [-1,1)^d, h = 2/n, wrap-around neighbours (readings R30, R31).
 *  - Field layout at the boundary: dense fp64, n^d values, C-contiguous with x fastest
 *    (index i + n*(j + n*k)) -- a torch tensor of shape (n,n) or (n,n,n).  Internally the library
 *    keeps pitched copies (row pitch n+1 doubles; periodic: n) inside the caller's workspace.
 *  - Ownership: the caller owns every buffer passed in (device fields, host arrays, the
 *    workspace).  The library never calls cudaMalloc; it owns only the handle, host-side tables
 *    and CUDA graphs.  Pointers named *_dev are device pointers, *_host are host pointers.
 *  - Streams: all device work is ordered on the stream given to isdc_create (NULL = legacy
 *    default stream).  Calls that return host scalars synchronise that stream.
 *  - Threads: a handle is not thread-safe; distinct handles are independent.
 *  - Errors: every call returns an isdc_status and never aborts or throws across the ABI.
 *    ISDC_ERR_CUDA carries the CUDA error text in isdc_last_error(h).  Non-convergence (sweep
 *    cap, SDC inner cap) is NOT an error: it is reported through *converged and counters.
 *  - Arithmetic: fp64, no FMA contraction, canonical expression trees of DESIGN.md §4 -- the
 *    results are bit-identical to the CPU oracle (oracle/), which shares no code with this library.
 */
#ifndef ISDC_H
#define ISDC_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct isdc_ctx *isdc_handle;

typedef enum {
    ISDC_OK = 0,
    ISDC_ERR_INVALID_ARG = 1,  /* n != 2^p - 1, d not in {2,3}, dt <= 0, nu <= 0, L < 1, NULL ptr */
    ISDC_ERR_UNSUPPORTED = 2,  /* node type other than Gauss-Lobatto, M outside [2, 8]           */
    ISDC_ERR_CUDA = 3,         /* a CUDA runtime error; text in isdc_last_error                   */
    ISDC_ERR_NONFINITE = 4,    /* a norm came out NaN/Inf; state kept for inspection              */
    ISDC_ERR_WORKSPACE = 5     /* workspace NULL, too small or not 256-byte aligned               */
} isdc_status;

/* Collocation node family.  Only Gauss-Lobatto is built. */
typedef enum {
    ISDC_NODES_GAUSS_LOBATTO = 0,
    ISDC_NODES_GAUSS_RADAU_RIGHT = 1,
    ISDC_NODES_GAUSS_LEGENDRE = 2
} isdc_nodes;

/* Explicit part f^E of the IMEX split.  Kinds of B:configs (R20-R22). */
typedef enum {
    ISDC_FE_NONE = 0,          /* f^E == 0: implicit SDC, Eq. (3)                                 */
    ISDC_FE_CUBIC = 1,         /* f^E(u) = u - u^3 (Allen-Cahn type, config 2)                    */
    ISDC_FE_FORCING = 2,       /* f^E(x,t) = G(x) cos(t), G given as a field (config 3)           */
    ISDC_FE_ADVECTION_CD4 = 3, /* f^E(u) = -a . grad u, 4th-order central differences (config 5) */
    ISDC_FE_BURGERS_WENO5 = 4  /* f^E(u) = -(u u_x + u u_y [+ u u_z]) = -sum_a d_a(u^2/2): WENO5-JS on
                                  Lax-Friedrichs split fluxes, alpha = max|u| of the evaluated field
                                  (R31).  Periodic grids only.          */
} isdc_fe_kind;

typedef enum {
    ISDC_BC_DIRICHLET = 0,     /* homogeneous Dirichlet on [0,1]^d, n = 2^p - 1 interior points  */
    ISDC_BC_PERIODIC = 1       /* periodic on [-1,1)^d, n = 2^p points (NEXT f3)                  */
} isdc_bc;

typedef enum {
    ISDC_MODE_ISDC_FIXED = 0,  /* exactly L V-cycles per node solve                        */
    ISDC_MODE_SDC_TOL = 1,     /* V-cycles until ||b - S u|| <= inner_tol*max(1,||b||)  */
    ISDC_MODE_ISDC_CAPPED = 2  /* the SDC_TOL test before every cycle, at most L cycles: the
                                  reading of Table 1's ISDC counts below K~(M-1)L (P:82 vs
                                  P:126-136, R10)                     */
} isdc_mode;

typedef struct {
    int dim;          /* 2 or 3                                                                  */
    int n;            /* points per direction: Dirichlet n = 2^p - 1 (interior), periodic n = 2^p, p >= 2 */
    int coarsest_n;   /* 0 or the coarsest level: 3 (Dirichlet, exact 3^d solve), 4 (periodic, 4^d) */
    int bc;           /* isdc_bc                                                                 */
} isdc_grid;

typedef struct {
    int nu1, nu2;     /* pre/post weighted-Jacobi sweeps per level (2, 2)                        */
    double omega;     /* Jacobi damping (0.8)                                                    */
} isdc_mg_opts;

typedef struct {
    isdc_mode mode;
    int L;            /* ISDC: V-cycles per node solve (2)                                */
    double inner_tol; /* SDC: relative defect tolerance (1e-12, R18)                   */
    int inner_cap;    /* SDC: max V-cycles per node solve (50)                                   */
    double sweep_tol; /* sweep until ||r~||_inf < sweep_tol (strict)                      */
    int max_sweeps;   /* sweep cap per step (200)                                                */
    int fixed_sweeps; /* > 0: exactly this many sweeps per step, no tolerance test (config 1)     */
    int guess;        /* node-solve initial guess: 0 = u_{m+1}^k, 1 = zero, 2 = u_m^{k+1} */
} isdc_solve_opts;

typedef struct {
    isdc_grid grid;
    int M;                       /* collocation nodes, 2 <= M <= 8                               */
    isdc_nodes nodes;
    double dt, nu;               /* step size and diffusion coefficient                          */
    isdc_fe_kind fe;
    double fe_params[3];         /* ADVECTION_CD4: velocity a = (a_x, a_y, a_z)                  */
    const double *fe_field_dev;  /* FORCING: G, dense n^d device field (copied at create), else NULL */
    isdc_mg_opts mg;
    isdc_solve_opts solve;
    /* Residual in the sweep test (NEXT f2): 0 = weighted ||r~|| = ||B_h r|| (R15);
     * 1 = the paper's unweighted ||r|| = ||W^{-1} r~||, 2D only, W^{-1} applied by
     * V-cycles on B_h from zero until ||r~ - B_h x|| <= w_tol*||r~|| (at most w_cap; R15b).
     * The W-cycles are counted apart from the V-cycles. */
    int residual_kind;
    double w_tol;                /* 1e-6 */
    int w_cap;                   /* 50   */
    /* Two-level MLSDC with ISDC sweeps (NEXT f4; "SDC sweeps in a multigrid-like way on
     * multiple levels ... connected through an FAS correction term"; reading R32).
     * mlsdc_levels 0 or 1: single-level ISDC; 2: every iteration is a fine ISDC sweep (stop test on
     * the fine residual), then -- unless the step stops -- injection of the iterate to the next
     * coarser grid n_c = (n-1)/2, the FAS correction fas_m = r~_H(R u)_m - R_fw r~_h,m, coarse_sweeps
     * ISDC sweeps of the FAS-corrected coarse collocation problem, and the 4th-order interpolation of
     * the coarse correction back onto every fine node.  Dirichlet grids with n >= 7, mode
     * ISDC_MODE_ISDC_FIXED, residual_kind 0 (else ISDC_ERR_UNSUPPORTED). */
    int mlsdc_levels;
    int coarse_sweeps;           /* coarse ISDC sweeps per MLSDC iteration (1) */
} isdc_problem;

/* Per-step statistics (Table 1 accounting; SPEC RunStats S:249-252). */
typedef struct {
    int sweeps;          /* K (SDC) or K~ (ISDC) sweeps performed in the step                   */
    long vcycles;        /* V-cycles over all node solves of the step (K~(M-1)L in ISDC)        */
    int cap_hits;        /* SDC node solves that stopped at inner_cap                           */
    int converged;       /* residual < sweep_tol reached (always 1 with fixed_sweeps)           */
    double final_residual;
    long wcycles;        /* W-cycles of the unweighted residual (residual_kind 1)         */
    long coarse_vcycles; /* MLSDC: V-cycles of the coarse-level sweeps (counted apart)          */
} isdc_step_stats;

/* Bytes of device workspace a problem needs (fields, MG hierarchy, reductions, tables). */
isdc_status isdc_workspace_bytes(const isdc_problem *prob, size_t *bytes);

/* Validate prob, lay out the workspace (device, >= isdc_workspace_bytes, 256-B aligned), build the
 * quadrature tables (binary128 -> binary64), level coefficients and coarse inverses, and bind
 * cuda_stream (a cudaStream_t or NULL).  On success *out is a new handle. */
isdc_status isdc_create(const isdc_problem *prob, void *workspace_dev, size_t bytes,
                        void *cuda_stream, isdc_handle *out);

/* Set u_0 (dense device field, copied) and the step counter (t_n = (double)step_index*dt,
 * DESIGN.md R28); spreads u_j = u_0 for all nodes. */
isdc_status isdc_set_initial(isdc_handle h, const double *u0_dev, int step_index);
/* Same with a host buffer (pinned or pageable); the H2D copy is stream-ordered. */
isdc_status isdc_set_initial_host(isdc_handle h, const double *u0_host, int step_index);

/* One sweep k -> k+1 over nodes m = 1..M-1: RHS assembly, node solves, then the residual
 * of the new iterate.  res_per_node[M-1], res_max and cycles[M-1] are host outputs (nullable). */
isdc_status isdc_sweep(isdc_handle h, double *res_per_node, double *res_max, int *cycles);

/* One time step: spread (already done by set_initial or the previous step), sweep until the
 * residual is below sweep_tol (or fixed_sweeps / max_sweeps), then u_0 <- u_M, step_index++.
 * res_hist (host, capacity max(max_sweeps, fixed_sweeps)) receives the residual after each sweep;
 * node_cycles (host, capacity cap*(M-1)) the V-cycles of every node solve.  Both nullable. */
isdc_status isdc_step(isdc_handle h, isdc_step_stats *stats, double *res_hist, int *node_cycles);

/* Run nsteps time steps (equivalent to nsteps isdc_step calls); stats[nsteps] nullable. */
isdc_status isdc_run(isdc_handle h, int nsteps, isdc_step_stats *stats);

/* One V(nu1,nu2)-cycle on the node system S u = b, S = B_h - gamma_m L_h, of substep node_m
 * (0-based, 0..M-2; gamma_m = nu*(dt*dtau_m)), applied in place to the dense device field u_dev
 * with right-hand side b_dev.  defect_before/after: ||b - S u||_inf before/after the cycle
 * (host, nullable). */
isdc_status mg_vcycle(isdc_handle h, int node_m, const double *b_dev, double *u_dev,
                      double *defect_before, double *defect_after);

/* Weighted SDC residual max_m ||r~_m||_inf of the current node state (R15). */
isdc_status residual_norm(isdc_handle h, double *per_node, double *max_norm);

/* Copy node `node` (0..M-1; M-1 = end of step) of the current iterate into a dense field. */
isdc_status isdc_get_solution(isdc_handle h, int node, double *out_dev);
isdc_status isdc_get_solution_host(isdc_handle h, int node, double *out_host);

/* ---- PFASST slice operations (NEXT f4b; "SDC sweeps on multiple levels combined with
 * a forward transfer of updated initial values in a manner similar to Parareal ... only a single
 * SDC sweep is performed" per level and iteration; reading R33) ------------------------
 * A PFASST time slice is a handle with mlsdc_levels = 2 (ISDC_ERR_INVALID_ARG otherwise).  A block
 * starts with isdc_set_initial (the block's u0 spread, the slice's step index); then, per R33:
 *   isdc_pfasst_restrict     phase B: fine residual fields of the current iterate (predictor: the
 *                            spread state), injection Ubar_j = U_j = R_i u_j, FAS correction
 *   isdc_pfasst_coarse       phase C: coarse node 0 <- U0 (dense n_c^d device field; NULL keeps it),
 *                            coarse_sweeps coarse ISDC sweeps, the coarse end value U_M -> Uend
 *                            (dense device, nullable), the coarse V-cycles -> *coarse_vcycles
 *   isdc_pfasst_interpolate  phase D: u_j += P4(U_j - Ubar_j), j = 1..M-1; the fine end value
 *                            u_M -> uend (dense n^d device, nullable)
 *   isdc_pfasst_set_u0       step 1: node 0 of the fine iterate <- u0 (dense device), in both iterate
 *                            sets (the forward transfer)
 *   isdc_sweep               phase A: one fine ISDC sweep + the fine weighted residual
 * Calls with device outputs synchronise the handle's stream before returning.  The caller moves the
 * dense end values between slices (on one GPU, or between ranks: paper_1401_7824_b200/pfasst.py). */
isdc_status isdc_pfasst_set_u0(isdc_handle h, const double *u0_dev);
isdc_status isdc_pfasst_restrict(isdc_handle h);
isdc_status isdc_pfasst_coarse(isdc_handle h, const double *U0_dev, double *Uend_dev, long *coarse_vcycles);
isdc_status isdc_pfasst_interpolate(isdc_handle h, double *uend_dev);

/* Load a full node state u[0..M-1] (dense device fields; used by parity tests). */
isdc_status isdc_set_state(isdc_handle h, const double *const *u_dev, int step_index);

/* Host copies of the tables: tau[M], Q[M*M], S[(M-1)*M], dtau[M-1] (nullable each). */
isdc_status isdc_get_tables(isdc_handle h, double *tau, double *Q, double *S, double *dtau);

/* RHS b of Eq. (5) for substep node_m (0..M-2) at time t_n = (double)step_index*dt, from the
 * previous iterate uold_dev[0..M-1] and the new value unew_m_dev = u_m^{k+1}; all dense device
 * fields (parity tests). */
isdc_status isdc_rhs(isdc_handle h, int node_m, const double *const *uold_dev,
                     const double *unew_m_dev, double *b_dev);

/* Number of kernels executed by this handle since creation, counting every kernel node of each
 * CUDA-graph launch (launch accounting). */
long isdc_kernel_launches(isdc_handle h);

/* Live kernel timing (bench.py's roofline): on = 1 brackets every fine-level launch (classes 0-2)
 * with CUDA events on the handle's stream, on = 2 every launch of every class, on = 16 + c only
 * class c, on = 0 none (events inside CUDA graphs are captured as external event-record nodes).
 * Classes: 0 fine-level smoother pass, 1 fine (pre-smoother +) defect + restriction, 2 fine
 * prolongation + correction (+ post-smoother), 3 RHS assembly, 4 residual, 5 coarse levels.
 * isdc_profile_get synchronises, returns the summed event time (ms), the launch count and the
 * ALGORITHMIC bytes those launches must move, and keeps accumulating. */
isdc_status isdc_profile_enable(isdc_handle h, int on);   /* 0 off, 1 fine-level classes 0-2, 2 all, 16+c class c only */
isdc_status isdc_profile_reset(isdc_handle h);
isdc_status isdc_profile_get(isdc_handle h, int cls, double *total_ms, long *launches, double *alg_bytes);

isdc_status isdc_destroy(isdc_handle h);
const char *isdc_last_error(isdc_handle h);
const char *isdc_status_string(isdc_status s);

#ifdef __cplusplus
}
#endif
#endif /* ISDC_H */
