/*
 * include/stokes.h -- C ABI of the B200-native matrix-free multigrid Stokes solver
 * (paper_2603_14040_b200, library libstokes_b200.so).
 *
 * Problem (PAPER.md:262-291 Eqs. xmom/ymom/mass, PAPER.md:716-741 Eq. stokes_saddle):
 * given a box [0,Lx]x[0,Ly] (y pointing DOWN), per-side boundary conditions, viscosity
 * on basic nodes (eta_b) and on pressure nodes (eta_p), density on basic nodes (rho_b)
 * and gravity (gx, gy), find the velocity v = (vx, vy) and the zero-mean pressure p with
 *      [ L  G ] [v]   [f]        L v = div_h(eta (grad_h v + grad_h v^T))
 *      [ D  0 ] [p] = [0],       G p = -grad_h p,  D v = div_h v
 * on the fully staggered grid of PAPER.md:611-624 with the stress-conservative finite
 * differences of PAPER.md:626-661 (x row = Listing vx_op_point).
 * Body force f = -g * rho averaged to the velocity node (reading R4/R23).
 * Method: inexact Uzawa (sign reading R3) with geometric-multigrid
 * V-cycle velocity solves, optionally accelerated by flexible
 * GCR(m); stopping test = relative energy residual E
 * (PAPER.md:1696-1701).  All arithmetic is IEEE FP64 on the GPU.
 *
 * ---------------------------------------------------------------- conventions
 * Sizes: nx x ny CELLS (reading R1: the paper's n_x, n_y count basic nodes = cells + 1).
 * Arrays: FP64, C-contiguous row-major, DEVICE pointers on the handle's GPU unless a
 * function says HOST.  "User layout" (physical nodes only, no ghosts), cell spacing
 * dx = Lx/nx, dy = Ly/ny:
 *     vx    : ny x (nx+1)   vx[i][j] at (j dx, (i+1/2) dy); columns 0 and nx are walls
 *     vy    : (ny+1) x nx   vy[i][j] at ((j+1/2) dx, i dy); rows 0 and ny are walls
 *     p     : ny x nx       P node [i][j] at ((j+1/2) dx, (i+1/2) dy)
 *     eta_p : ny x nx       (P nodes)
 *     eta_b : (ny+1) x (nx+1)   basic node [i][j] at (j dx, i dy)
 *     rho_b : (ny+1) x (nx+1)
 * Wall entries of vx/vy inputs are IGNORED (the normal velocity on a wall is zero) and
 * are written 0 on output.
 * Boundary conditions bc[4] = {West, East, North(top, y=0), South(bottom, y=Ly)}, each
 * STOKES_FREE_SLIP or STOKES_NO_SLIP; tangential mirrors of
 * PAPER.md:613 (free slip: +mirror, no slip: -mirror).
 * Ownership: the caller owns every array; inputs are borrowed for the duration of the
 * call; set_* functions COPY.  The handle owns its workspace (or borrows the caller's
 * workspace passed to stokes_create, which must outlive the handle).
 * Streams: all device work is enqueued on the handle's stream (cudaStream_t passed as
 * void*; NULL = legacy default stream).  Functions returning HOST scalars synchronise
 * that stream.  A handle is not thread safe.
 * Errors: every function returns an int status: 0 OK, >0 warning with valid outputs,
 * <0 error (outputs undefined).  stokes_strerror() gives a message; the last CUDA/NCCL
 * error text is available from stokes_last_error().
 */
#ifndef PAPER_2603_14040_B200_STOKES_H
#define PAPER_2603_14040_B200_STOKES_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the library is built with -fvisibility=hidden */
#endif

typedef struct stokes_s *stokes_t;

enum { STOKES_FREE_SLIP = 0, STOKES_NO_SLIP = 1 };

enum {
    STOKES_OK = 0,
    STOKES_NOT_CONVERGED = 1, /* max_iter reached; outputs are the last iterate          */
    STOKES_EINVAL = -1,       /* bad size / pointer / option / non-positive viscosity    */
    STOKES_ENOMEM = -2,       /* device allocation failed or workspace too small         */
    STOKES_ECUDA = -3,        /* CUDA runtime error (see stokes_last_error)               */
    STOKES_ENCCL = -4,        /* NCCL error (distributed handles)                         */
    STOKES_EDIVERGED = -5,    /* E non-finite or > 1e6 E0; last iterate kept */
    STOKES_ESTATE = -6        /* call order: set_viscosity / set_density missing          */
};

enum { STOKES_SMOOTH_JACOBI = 0, STOKES_SMOOTH_RBGS = 1, STOKES_SMOOTH_RAS = 2, STOKES_SMOOTH_MIXED = 3 };
enum { STOKES_ACCEL_NONE = 0, STOKES_ACCEL_GCR = 1, STOKES_ACCEL_ANDERSON = 2 };

/* Solver options.  stokes_opts_default() fills the paper's setting (PAPER.md:1765-1788:
 * omega_v 0.3, omega_p 0.6, 5+5 sweeps) with the readings of DESIGN.md §3 (growth g = 1,
 * direct coarsest).  The field order is part of the ABI. */
typedef struct {
    int smoother;         /* STOKES_SMOOTH_JACOBI, _RBGS, _RAS
                             (Alg. 3) or _MIXED (Jacobi finest, RAS below)  */
    double omega_v;       /* velocity relaxation omega_v                                        */
    double alpha_p;       /* pressure relaxation alpha (= omega_p)                              */
    int nu1;              /* pre- and post-smoothing sweeps on the finest level                 */
    double nu_growth;     /* nu_l = floor(nu1 * g^(l-1) + 1/2)  (reading R9)      */
    int coarse_min;       /* coarsen by 2 while both sizes even and min(nx,ny)/2 >= coarse_min  */
    int coarse_direct;    /* 1: exact coarsest solve (reading R10); 0: 2*nu_L smoothing sweeps  */
    int vcycles_per_iter; /* V-cycles per Uzawa step                            */
    int accel;            /* STOKES_ACCEL_NONE (plain Uzawa), _GCR or _ANDERSON (single domain)  */
    int gcr_restart;      /* m of GCR(m)                                                        */
    int max_iter;         /* cap on iterations (V-cycle applications)                           */
    int pressure_sign;    /* +1 physical reading R3 (default); -1 literal PAPER.md:824 (diverges) */
    double theta_step;    /* viscosity rescaling: stages theta = 0, step, ..
                             < 1 with eta_comp = (1-theta) eta_min + theta eta, then theta = 1;
                             0 = off (default).  Single-domain handles only                      */
    int theta_every;      /* Uzawa / GCR iterations per stage before theta = 1 (25) */
    int aa_depth;         /* STOKES_ACCEL_ANDERSON (Alg. 5): depth m, 0..15   */
    double aa_beta;       /* Anderson mixing beta in (0, 1] (0.5-0.8)              */
    int ras_tile;         /* RAS tile edge T in cells, 2..32 (32)                  */
    int ras_inner;        /* RAS inner sweeps T_inner (4)                          */
    uint64_t ras_seed;    /* seed of the counter-based tile-shift generator (reading R27)         */
    int gcr_true_restart; /* GCR restart (reading R13): 1 (default) restarts
                             from the true residual b - A x; 0 keeps the recursive r (Alg. 4)   */
} stokes_opts;

/* Fill *o with the defaults.  Returns STOKES_EINVAL if o is NULL. */
int stokes_opts_default(stokes_opts *o);

/* Device workspace (bytes) stokes_create needs for an nx x ny problem with these
 * options; *bytes written on success. */
int stokes_workspace_bytes(int nx, int ny, const stokes_opts *opts, size_t *bytes);

/* Create a single-GPU handle on the current CUDA device.
 *   nx, ny >= 2 cells; Lx, Ly > 0; bc[4] in {0,1}; opts may be NULL (defaults);
 *   cuda_stream: cudaStream_t as void* (NULL = default stream);
 *   workspace: device memory of >= stokes_workspace_bytes() bytes, 256-B aligned,
 *   owned by the caller (e.g. a torch tensor), or NULL to let the library cudaMalloc.
 * Builds the level hierarchy (reading R8).  Errors: EINVAL, ENOMEM, ECUDA. */
int stokes_create(int nx, int ny, double Lx, double Ly, const int bc[4], const stokes_opts *opts,
                  void *cuda_stream, void *workspace, size_t workspace_bytes, stokes_t *out);

/* 2D domain decomposition.  The global nx x ny grid is
 * split into px x py tiles of (nx/px) x (ny/py) cells (nx % px == ny % py == 0); tile
 * (tx, ty) = (rank % px, rank / px).  Exact: iterates equal the single-domain solve's up to
 * the order of global sums.  Levels whose tiles are >= dmin cells wide (NCCL 512, in-process
 * 64; STOKES_DIST_DMIN) are distributed (width-2 halo exchange after every pass that writes a
 * velocity / correction / right-hand side / pressure); the coarser levels are agglomerated:
 * every process holds the global grid of the first coarse level and runs the coarse tail
 * redundantly.  Options: accel STOKES_ACCEL_NONE (Uzawa-MG), STOKES_ACCEL_GCR (GCR(m) with
 * the distributed V-cycle as preconditioner and global inner products) or
 * STOKES_ACCEL_ANDERSON (AA(m, beta) over the decomposed Uzawa iteration, global Gram row);
 * viscosity-rescaling stages (theta_step > 0; eta_min reduced over all tiles) with any of
 * them; the RAS / Mixed smoothers: STOKES_EINVAL.
 *   rank = -1 VIRTUAL: all tiles in this process on the current GPU; every array of the
 *             calls below is the GLOBAL user-layout array (tests of the decomposition).
 *   rank = -2 LOOPBACK: as VIRTUAL, but halos and the agglomeration go through the NCCL
 *             path's packing / unpacking with device copies standing in for the NCCL calls.
 *   rank = -3 NCCL_SELF: as LOOPBACK, but every transfer is a real ncclSend / ncclRecv /
 *             ncclAllReduce on a one-rank communicator (the NCCL code path on one GPU).
 *   rank >= 0 NCCL: this process owns tile `rank` (one GPU per process), nccl_unique_id =
 *             128 bytes from stokes_nccl_unique_id() on rank 0, shared by the caller; every
 *             array is the tile's WINDOW of the global user layout, i.e. the user layout of
 *             an (nx/px) x (ny/py) problem (shared edge nodes appear in both windows).
 *             nccl_unique_id = NULL: the same handle as a schedule-recording DRY RUN -- no
 *             communicator; every NCCL call the transport would issue is recorded instead
 *             (stokes_dist_schedule) and the collectives keep the local part, so the ranks'
 *             schedules can be built one after another in one process on one GPU and checked
 *             against NCCL's matching rules.  Its numerical results are meaningless.
 * Supported calls on a decomposed handle: set_viscosity, set_density, set_gravity,
 * residual (energy only: rx = ry = rp = NULL), solve, num_levels, launch_count, destroy;
 * the per-step entry points return STOKES_EINVAL.  The library allocates its own memory. */
int stokes_create_dist(int nx, int ny, double Lx, double Ly, const int bc[4], int px, int py, int rank,
                       const void *nccl_unique_id, const stokes_opts *opts, void *cuda_stream, stokes_t *out);
/* The NCCL calls recorded by a dry-run decomposed handle (rank >= 0, nccl_unique_id NULL),
 * in issue order, 5 values per call: op (1 group start, 2 group end, 3 ncclSend, 4 ncclRecv,
 * 5 ncclAllGather, 6 ncclAllReduce; markers 7 / 8 = begin / end of the capture of one plain
 * Uzawa iteration's graph, peer = its pressure parity), peer rank (-1 for collectives and groups), element
 * count (per rank for all-gathers), ncclDataType_t, ncclRedOp_t (-1 if none).  Calls made
 * during a CUDA-graph capture are recorded once, when captured.  rec: host buffer of cap
 * records (may be NULL if cap = 0); *n = the number recorded (may exceed cap: call again
 * with a larger buffer).  STOKES_EINVAL for any other handle.  Verification of the multi-
 * process schedule (tests/test_gpu_nccl_schedule.py). */
int stokes_dist_schedule(stokes_t h, long long *rec, int cap, int *n);
/* 128-byte NCCL unique id for stokes_create_dist (call on rank 0, broadcast it). */
int stokes_nccl_unique_id(void *id128);

/* Release the handle (and its own allocations). */
int stokes_destroy(stokes_t h);

/* Number of multigrid levels and the cell counts / sweeps of level l (0 = finest). */
int stokes_num_levels(stokes_t h, int *nlev);
int stokes_level_shape(stokes_t h, int level, int *nx, int *ny, int *nu);

/* Copy viscosities (device, user layout eta_b (ny+1)x(nx+1), eta_p ny x nx), check
 * eta > 0 (EINVAL otherwise, by a device min-reduction), build the coarse-level
 * viscosities by normalised bilinear restriction (a7, reading R7)
 * and the coarsest-level inverse (a8).  Synchronises the stream. */
int stokes_set_viscosity(stokes_t h, const double *eta_b, const double *eta_p);

/* Copy the basic-node density (device, (ny+1)x(nx+1)). */
int stokes_set_density(stokes_t h, const double *rho_b);

/* Gravity vector; f = -(gx, gy) * rho averaged to velocity nodes (y down). */
int stokes_set_gravity(stokes_t h, double gx, double gy);

/* ax, ay = L v + G p (vx / vy layouts, walls 0); ap = D v (P layout).  (a2) */
int stokes_apply_operator(stokes_t h, const double *vx, const double *vy, const double *p, double *ax,
                          double *ay, double *ap);

/* rx, ry = f - L v - G p; rp = -D v (rx, ry, rp may be NULL); *rel_energy (HOST, may be
 * NULL) = E = sqrt((sum r_v^2/d_v + sum r_p^2 eta_p/(2/dx^2+2/dy^2)) / sum f^2/d_v) with
 * d_v = -a_ii (reading R5/R12); E = 0 if f == 0.  (a3) */
int stokes_residual(stokes_t h, const double *vx, const double *vy, const double *p, double *rx, double *ry,
                    double *rp, double *rel_energy);

/* One V-cycle (a9) on L v = b, warm-started from (vx, vy) (in/out);
 * bx, by in vx / vy layouts (walls ignored). */
int stokes_vcycle(stokes_t h, const double *bx, const double *by, double *vx, double *vy);

/* Solve to E <= rtol (a12).  vx, vy, p: in = initial guess, out = solution (p zero-mean).
 * *iters (HOST) = number of V-cycle applications; *rel_energy (HOST) = final E.  With GCR the
 * stopping test runs on the recursive residual and, once that passes, on the true residual
 * (restarting from it if it does not pass); the E returned is the true one.
 * Returns OK, NOT_CONVERGED, EDIVERGED (last iterate kept) or an error. */
int stokes_solve(stokes_t h, double rtol, double *vx, double *vy, double *p, int *iters, double *rel_energy);
/* stokes_solve that also writes E after every iteration: hist[k] (HOST, hist_len doubles,
 * caller-owned; entries past *iters are untouched) = E after iteration k + 1 -- the energy
 * residual of the new (v, p) (Uzawa, Anderson: of G(x^k)) or of the recursive residual (GCR),
 * counted across viscosity-rescaling stages.  Single-domain handles (EINVAL otherwise). */
int stokes_solve_hist(stokes_t h, double rtol, double *vx, double *vy, double *p, int *iters, double *rel_energy,
                      double *hist, int hist_len);

/* ---- per-step entry points (parity tests of each hot-path step; same layouts at the
 * given level's size; all device pointers) ------------------------------------------- */
/* nsweeps smoother sweeps (a4) on level `level` for L v = b, in place on (vx, vy). */
int stokes_smooth(stokes_t h, int level, const double *bx, const double *by, double *vx, double *vy,
                  int nsweeps);
/* r = b - L v on level `level`. */
int stokes_level_residual(stokes_t h, int level, const double *bx, const double *by, const double *vx,
                          const double *vy, double *rx, double *ry);
/* Restriction (a5 / a7) level -> level+1 of a field of kind 0 vx, 1 vy, 2 P, 3 basic. */
int stokes_restrict(stokes_t h, int level, int kind, const double *fine, double *coarse);
/* (vx, vy) at `level` += P (ex, ey) from level+1, then mirror refresh (a6). */
int stokes_prolong(stokes_t h, int level, const double *ex, const double *ey, double *vx, double *vy);
/* Viscosities of a level as built by set_viscosity (a7). */
int stokes_get_viscosity(stokes_t h, int level, double *eta_b, double *eta_p);
/* Exact coarsest-level solve L_c v = b (a8); EINVAL if coarse_direct == 0. */
int stokes_coarse_solve(stokes_t h, const double *bx, const double *by, double *vx, double *vy);

/* ---- instrumentation ---------------------------------------------------------- */
/* Lithostatic pressure, the initial guess the paper uses with gravity:
 * p(x, y) = int_0^y rho g_y dy' from the top wall, discretely the hydrostatic balance of the
 * y-momentum row with v = 0 (reading R4, density at vy nodes R23):
 *   p(1,j) = g_y (dy/2) rho_vy(0,j),  p(i+1,j) = p(i,j) + g_y dy rho_vy(i,j).
 * p: DEVICE, P layout ny x nx, written (not de-meaned).  Needs stokes_set_density
 * (STOKES_ESTATE otherwise); single-domain handles only (STOKES_EINVAL otherwise). */
int stokes_lithostatic(stokes_t h, double *p);

/* Number of kernels this library launched on the handle since creation / last reset. */
int stokes_launch_count(stokes_t h, long long *count, int reset);
/* Time `reps` back-to-back launches of a hot-path kernel on the handle's stream with CUDA
 * events (after 2 warm-ups); *avg_ms (HOST) = mean duration of one launch, *bytes (HOST)
 * = algorithmic bytes one launch moves.  kernel: 0 fine Jacobi sweep
 * (Uzawa RHS), 1 fine residual+energy, 2 fine residual+restriction, 3 prolongation,
 * 4 pressure update (fused with the energy residual), 5 RBGS sweep (4 phases), 6 pressure
 * update + energy residual + first Jacobi sweep of the next V-cycle, 7 two Jacobi sweeps in
 * one pass (6 and 7: fine grid >= 128 x 8 only, else STOKES_EINVAL), 8 one RAS outer
 * iteration (ras_inner sweeps on shared-memory tiles), 9 the last post-smoothing sweep of a
 * V-cycle fused with kernel 6 (k_jju; single-domain fine grid >= 128 x 8, else EINVAL).
 * Uses the handle's current fields. */
int stokes_time_kernel(stokes_t h, int kernel, int reps, double *avg_ms, double *bytes);

/* ---- marker-in-cell ------------------------
 * Markers: n FP64 positions (xm, ym) in the box frame of the handle (y down), DEVICE arrays
 * of length n (n < 2^31 - 1).  Positions outside the closed box are clamped into it (R28/
 * R30); they must be finite.  Single-domain handles only (STOKES_EINVAL otherwise).  The
 * first call allocates marker scratch (~64 B per marker + 12 B per cell, freed by
 * stokes_destroy; STOKES_ENOMEM if that fails).  Results are bit-identical to the serial
 * CPU loops of the paper (the node sums are taken in ascending marker index). */
enum { STOKES_ADVECT_EULER = 0, STOKES_ADVECT_HEUN = 1, STOKES_ADVECT_RK4 = 2, STOKES_ADVECT_LPI2 = 3,
       STOKES_ADVECT_LPI3 = 4 };

/* Marker -> grid (§4.2 steps 1-5; reading R28): every node value is
 *   phi(node) = sum_m w_m phi_m / sum_m w_m
 * over the markers whose surrounding cell of that grid has the node as a corner, with the
 * bilinear weights of PAPER.md:480-484 (w = (1 - r_x/dx or r_x/dx)(1 - r_y/dy or r_y/dy),
 * r measured from the cell's top-left reference node).  eta_m -> eta_b (basic nodes) and
 * eta_p (pressure nodes), rho_m -> rho_b (basic nodes): the inputs of stokes_set_viscosity /
 * stokes_set_density, user layouts.  Nodes with zero accumulated weight are written 0 and
 * counted in *n_empty (HOST, nullable; non-NULL synchronises).  Any of eta_b, eta_p, rho_b
 * may be NULL (not written); rho_m may be NULL when rho_b is. */
int stokes_markers_to_grid(stokes_t h, long long n, const double *xm, const double *ym, const double *eta_m,
                           const double *rho_m, double *eta_b, double *eta_p, double *rho_b, long long *n_empty);
/* Grid -> marker (R29): (vxm, vym)[m] = the four-node bilinear sum of the
 * caller's velocity (user layout; wall entries taken as 0, mirror rows/columns from the
 * boundary conditions of the handle) at marker m. */
int stokes_grid_to_markers(stokes_t h, long long n, const double *xm, const double *ym, const double *vx,
                           const double *vy, double *vxm, double *vym);
/* One advection step of every marker IN PLACE (R30) with the velocity
 * frozen: scheme STOKES_ADVECT_EULER (Eq. euler_advection), _HEUN
 * (Eq. heun_method), _RK4 (Eq. rk4_method, Listing rk4_agnostic order) or the locally
 * polynomial integrator _LPI2 / _LPI3 (Eq. lpi_update truncated after the J or the H term;
 * J and H are the derivatives of the bilinear velocity interpolant, reading R32).  Stage and final
 * positions are clamped into the closed box; *n_clamped (HOST, nullable; synchronises) =
 * markers whose final position was clamped. */
int stokes_advect_markers(stokes_t h, long long n, double *xm, double *ym, const double *vx, const double *vy,
                          double dt, int scheme, long long *n_clamped);
/* CFL-like time step (R31): *dt (HOST) = min(max_dt, cfl min(dx/max|vx|,
 * dy/max|vy|)) over the velocity unknowns (a zero component drops its term).  cfl > 0,
 * max_dt > 0.  Synchronises. */
int stokes_marker_timestep(stokes_t h, const double *vx, const double *vy, double cfl, double max_dt, double *dt);

const char *stokes_strerror(int status);
const char *stokes_last_error(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif
