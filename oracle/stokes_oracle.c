/*
 * oracle/stokes_oracle.c -- CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_2603_14040_b200/) never links,
 * imports or executes anything under oracle/, and this file includes no header from
 * the product tree: it shares no code with the CUDA path.
 *
 * A plain, slow, single-threaded FP64 implementation of the matrix-free geometric
 * multigrid Stokes solve of arXiv 2603.14040 (Pyroclast), written from PAPER.md:
 *   - staggered grid, "lower-right" indexing, ghost/boundary nodes  (§4.4.1)
 *   - stress-conservative FD; the x-momentum row is Listing vx_op_point;
 *     the y-momentum row follows "the same procedure" -> DESIGN.md reading R2
 *   - saddle system [L G; D 0][v;p] = [f;0]       (Eq. stokes_saddle)
 *   - inexact Uzawa + diagonal Schur surrogate    (Eq. uzawa_iteration;
 *     sign reading R3), zero-mean pressure        (Eq. pressure_normalization)
 *   - V-cycle (Eq. multigrid_levels), bilinear prolongation
 *     (PAPER.md:970-982), normalised bilinear restriction (Alg. 2),
 *     damped Jacobi (Eq. damped_jacobi), damped RBGS
 *     (Eq. sor_update; 4-phase reading R11)
 *   - flexible GCR(m) with MGS (Alg. 4), preconditioner M^-1 of the
 *     Uzawa splitting
 *   - relative energy residual
 * Readings where the paper is silent/garbled are the R-numbers of DESIGN.md §3 (they
 * follow SURVEY.md §8(c) Q1..Q23).
 *
 * Arithmetic: IEEE FP64, round to nearest, compiled with -O2 -ffp-contract=off;
 * reductions are pairwise sums in row-major order (vx, then vy, then p).
 *
 * Pins: every function below is pinned by a -m "not gpu" test in tests/test_oracle_*.py
 * (dense assembly from the stress formulas, MMS second order, hydrostatics, transfer
 * identities, spectral radius of the Uzawa map, GCR on dense systems).  The iteration
 * COUNT of a solve is "parity unpinned" by the paper (it prints none): pinned only
 * oracle <-> GPU, see DESIGN.md §4.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXLEV 24

typedef struct {
    int smoother;        /* 0 damped Jacobi, 1 RBGS 4-phase, 2 RAS-type temporal blocking (Alg. 3),
                            3 mixed: Jacobi on the finest level, RAS on the coarser ones */
    double omega_v;      /* velocity relaxation */
    double alpha_p;      /* pressure relaxation (omega_p) */
    int nu1;             /* sweeps on the finest level (pre and post) */
    double nu_growth;    /* per-level growth g of the sweep count */
    int coarse_min;      /* coarsen while min(ncx,ncy)/2 >= coarse_min */
    int coarse_direct;   /* 1 exact coarsest solve, 0 2*nu_L smoothing sweeps */
    int vcycles_per_iter;
    int accel;           /* 0 plain Uzawa, 1 flexible GCR(m) */
    int gcr_restart;     /* m */
    int max_iter;
    int pressure_sign;   /* +1 physical reading R3 (default); -1 literal PAPER.md:824 */
    double theta_step;   /* viscosity rescaling: theta += step per stage, 0 = off */
    int theta_every;     /* Uzawa iterations per stage before theta = 1 (25) */
    int aa_depth;        /* Anderson acceleration (accel = 2, Alg. 5): depth m */
    double aa_beta;      /* Anderson mixing beta in (0, 1] */
    int ras_tile;        /* RAS tile edge T_I = T_J in cells (32) */
    int ras_inner;       /* RAS inner iterations T_inner (4) */
    uint64_t ras_seed;   /* seed of the counter-based tile-shift generator (reading R27) */
    int gcr_true_restart; /* 1: true residual at every GCR restart (R13), 0: recursive r (Alg. 4) */
    int gcr_inner;        /* GCR inner product: 0 Euclidean over unknowns (default),
                             1 energy-weighted (the weights of E; reading R33) */
} oracle_opts;

typedef struct {
    int ncx, ncy;          /* cells */
    double dx, dy;
    int W;                 /* padded row length = ncx + 2 */
    double *etab, *etap;   /* padded (ncy+2) x (ncx+2) */
    /* scratch (padded) */
    double *rx, *ry, *bx, *by, *ex, *ey, *tx, *ty;
    int nu;                /* sweeps per pre/post smoothing on this level */
} olevel;

typedef struct {
    int nx, ny;
    double Lx, Ly;
    int bc[4];             /* W, E, N(top), S(bottom): 0 free slip, 1 no slip */
    double gx, gy;
    oracle_opts o;
    int nlev;
    olevel lev[MAXLEV];
    double *rhob;          /* padded, fine */
    double *fx, *fy;       /* padded body force at vx / vy nodes (fine) */
    int have_eta, have_rho, force_override;
    /* coarsest direct solve: Cholesky factor of -L_c (dense, lower, row-major) */
    int nc;                /* coarsest unknowns */
    double *chol;
    /* fine-level work fields */
    double *vx, *vy, *p;
    /* the caller's viscosities (padded, fine) -- viscosity rescaling blends from them */
    double *etab_user, *etap_user;
    /* RAS shift counter: draw index q = ras_k * 65536 + ras_c (reading R27) */
    int ras_k, ras_c;
} oracle_t;

/* ------------------------------------------------------------------ helpers */
static inline int IX(const olevel *L, int i, int j) { return i * L->W + j; }
static double sgn_of(int bc) { return bc == 0 ? 1.0 : -1.0; } /* free slip +1, no slip -1 */

static double *zalloc(size_t n) { return (double *)calloc(n ? n : 1, sizeof(double)); }
static size_t padn(const olevel *L) { return (size_t)(L->ncy + 2) * (size_t)(L->ncx + 2); }

/* Pairwise summation of a[0..n-1] (fixed order). */
static double pairwise(const double *a, size_t n) {
    if (n == 0) return 0.0;
    if (n <= 8) {
        double s = 0.0;
        for (size_t k = 0; k < n; ++k) s += a[k];
        return s;
    }
    size_t h = n / 2;
    return pairwise(a, h) + pairwise(a + h, n - h);
}

/* ----------------------------------------------- boundary conditions (R1, R5)
 * Mirror ("boundary") nodes: vx rows 0 and ncy+1 mirror rows 1 and ncy with sign s_N/s_S;
 * vy columns 0 and ncx+1 mirror columns 1 and ncx with sign s_W/s_E; the wall-normal
 * nodes (vx columns 0, ncx; vy rows 0, ncy) are zero. */
static void refresh_mirrors(const oracle_t *S, const olevel *L, double *vx, double *vy) {
    int ncx = L->ncx, ncy = L->ncy;
    double sW = sgn_of(S->bc[0]), sE = sgn_of(S->bc[1]), sN = sgn_of(S->bc[2]), sS = sgn_of(S->bc[3]);
    for (int i = 0; i <= ncy + 1; ++i) { vx[IX(L, i, 0)] = 0.0; vx[IX(L, i, ncx)] = 0.0; }
    for (int j = 1; j <= ncx - 1; ++j) {
        vx[IX(L, 0, j)] = sN * vx[IX(L, 1, j)];
        vx[IX(L, ncy + 1, j)] = sS * vx[IX(L, ncy, j)];
    }
    for (int j = 0; j <= ncx + 1; ++j) { vy[IX(L, 0, j)] = 0.0; vy[IX(L, ncy, j)] = 0.0; }
    for (int i = 1; i <= ncy - 1; ++i) {
        vy[IX(L, i, 0)] = sW * vy[IX(L, i, 1)];
        vy[IX(L, i, ncx + 1)] = sE * vy[IX(L, i, ncx)];
    }
}

/* ------------------------------------------------ the operator (a2)
 * x-momentum row at vx(i,j): Listing vx_op_point, verbatim
 * (velocity part; the pressure part is grad_x below). */
static double Lx_point(const olevel *L, const double *vx, const double *vy, int i, int j) {
    double dx = L->dx, dy = L->dy;
    double etaA = L->etap[IX(L, i, j)];
    double etaB = L->etap[IX(L, i, j + 1)];
    double eta1 = L->etab[IX(L, i - 1, j)];
    double eta2 = L->etab[IX(L, i, j)];
    double vx1 = 2.0 * etaA / (dx * dx);
    double vx2 = eta1 / (dy * dy);
    double vx3 = -(eta1 + eta2) / (dy * dy) - 2.0 * (etaA + etaB) / (dx * dx);
    double vx4 = eta2 / (dy * dy);
    double vx5 = 2.0 * etaB / (dx * dx);
    double vy1 = eta1 / (dx * dy);
    double vy2 = -eta2 / (dx * dy);
    double vy3 = -eta1 / (dx * dy);
    double vy4 = eta2 / (dx * dy);
    return vx1 * vx[IX(L, i, j - 1)] + vx2 * vx[IX(L, i - 1, j)] + vx3 * vx[IX(L, i, j)] +
           vx4 * vx[IX(L, i + 1, j)] + vx5 * vx[IX(L, i, j + 1)] + vy1 * vy[IX(L, i - 1, j)] +
           vy2 * vy[IX(L, i, j)] + vy3 * vy[IX(L, i - 1, j + 1)] + vy4 * vy[IX(L, i, j + 1)];
}
static double Lx_center(const olevel *L, int i, int j) {
    double dx = L->dx, dy = L->dy;
    double etaA = L->etap[IX(L, i, j)], etaB = L->etap[IX(L, i, j + 1)];
    double eta1 = L->etab[IX(L, i - 1, j)], eta2 = L->etab[IX(L, i, j)];
    return -(eta1 + eta2) / (dy * dy) - 2.0 * (etaA + etaB) / (dx * dx);
}

/* y-momentum row at vy(i,j) (reading R2): "the same procedure is applied":
 *   (sxx -> syy) d(syy)/dy with syy(P(i,j)) = 2 etaP(i,j) (vy(i,j)-vy(i-1,j))/dy,
 *   d(sxy)/dx with sxy(B(i,j)) = etaB(i,j) ((vx(i+1,j)-vx(i,j))/dy + (vy(i,j+1)-vy(i,j))/dx)
 *   (PAPER.md:643-661).  Written as the stress differences, not as coefficients, so the
 *   dense pin P1 (coefficients assembled in numpy) is an independent check. */
static double Ly_point(const olevel *L, const double *vx, const double *vy, int i, int j) {
    double dx = L->dx, dy = L->dy;
    double syy_S = 2.0 * L->etap[IX(L, i + 1, j)] * (vy[IX(L, i + 1, j)] - vy[IX(L, i, j)]) / dy;
    double syy_N = 2.0 * L->etap[IX(L, i, j)] * (vy[IX(L, i, j)] - vy[IX(L, i - 1, j)]) / dy;
    double sxy_E = L->etab[IX(L, i, j)] *
                   ((vx[IX(L, i + 1, j)] - vx[IX(L, i, j)]) / dy + (vy[IX(L, i, j + 1)] - vy[IX(L, i, j)]) / dx);
    double sxy_W = L->etab[IX(L, i, j - 1)] *
                   ((vx[IX(L, i + 1, j - 1)] - vx[IX(L, i, j - 1)]) / dy +
                    (vy[IX(L, i, j)] - vy[IX(L, i, j - 1)]) / dx);
    return (syy_S - syy_N) / dy + (sxy_E - sxy_W) / dx;
}
static double Ly_center(const olevel *L, int i, int j) {
    double dx = L->dx, dy = L->dy;
    double etaN = L->etap[IX(L, i, j)], etaS = L->etap[IX(L, i + 1, j)];
    double etaW = L->etab[IX(L, i, j - 1)], etaE = L->etab[IX(L, i, j)];
    return -2.0 * (etaN + etaS) / (dy * dy) - (etaW + etaE) / (dx * dx);
}
/* Diagonal a_ii of the velocity block L of the linear system (reading R5): the centre
 * coefficient plus, for a row adjacent to a mirror node, the mirror's coefficient times
 * the mirror sign s (the mirror is s times this very unknown).  This is the
 * a_ii of Eq. jacobi_update and the diag(-L) of PAPER.md:1615. */
static double Lx_diag(const oracle_t *S, const olevel *L, int i, int j) {
    double a = Lx_center(L, i, j);
    if (i == 1) a += sgn_of(S->bc[2]) * L->etab[IX(L, i - 1, j)] / (L->dy * L->dy);
    if (i == L->ncy) a += sgn_of(S->bc[3]) * L->etab[IX(L, i, j)] / (L->dy * L->dy);
    return a;
}
static double Ly_diag(const oracle_t *S, const olevel *L, int i, int j) {
    double a = Ly_center(L, i, j);
    if (j == 1) a += sgn_of(S->bc[0]) * L->etab[IX(L, i, j - 1)] / (L->dx * L->dx);
    if (j == L->ncx) a += sgn_of(S->bc[1]) * L->etab[IX(L, i, j)] / (L->dx * L->dx);
    return a;
}
/* G p = -grad_h p (Eq. gradient_discrete); pressure terms of the Listing. */
static double Gx_point(const olevel *L, const double *p, int i, int j) {
    return -p[IX(L, i, j + 1)] / L->dx + p[IX(L, i, j)] / L->dx;
}
static double Gy_point(const olevel *L, const double *p, int i, int j) {
    return -p[IX(L, i + 1, j)] / L->dy + p[IX(L, i, j)] / L->dy;
}
/* D v = div_h v (Eq. divergence_discrete; SPEC continuity_apply). */
static double D_point(const olevel *L, const double *vx, const double *vy, int i, int j) {
    return (vx[IX(L, i, j)] - vx[IX(L, i, j - 1)]) / L->dx + (vy[IX(L, i, j)] - vy[IX(L, i - 1, j)]) / L->dy;
}

/* index ranges of unknowns (Listing loop bounds PAPER.md:2352-2353, reading R1) */
#define FOR_VX(L) for (int i = 1; i <= (L)->ncy; ++i) for (int j = 1; j <= (L)->ncx - 1; ++j)
#define FOR_VY(L) for (int i = 1; i <= (L)->ncy - 1; ++i) for (int j = 1; j <= (L)->ncx; ++j)
#define FOR_P(L) for (int i = 1; i <= (L)->ncy; ++i) for (int j = 1; j <= (L)->ncx; ++j)

/* r = b - L v on unknowns (mirrors of v must be current); Eq. mg_residual */
static void residual_v(const olevel *L, const double *vx, const double *vy, const double *bx, const double *by,
                       double *rx, double *ry) {
    memset(rx, 0, padn(L) * sizeof(double));
    memset(ry, 0, padn(L) * sizeof(double));
    FOR_VX(L) rx[IX(L, i, j)] = bx[IX(L, i, j)] - Lx_point(L, vx, vy, i, j);
    FOR_VY(L) ry[IX(L, i, j)] = by[IX(L, i, j)] - Ly_point(L, vx, vy, i, j);
}

/* ------------------------------------------------ smoothers (a4)
 * Damped Jacobi, Eq. damped_jacobi: x_i <- x_i + w (b - A x)_i / a_ii,
 * all reads from the old iterate; a_ii = diagonal of L (reading R5). */
static void smooth_jacobi(const oracle_t *S, olevel *L, double *vx, double *vy, const double *bx,
                          const double *by, int nu) {
    double w = S->o.omega_v;
    for (int s = 0; s < nu; ++s) {
        residual_v(L, vx, vy, bx, by, L->tx, L->ty);
        FOR_VX(L) vx[IX(L, i, j)] += w * L->tx[IX(L, i, j)] / Lx_diag(S, L, i, j);
        FOR_VY(L) vy[IX(L, i, j)] += w * L->ty[IX(L, i, j)] / Ly_diag(S, L, i, j);
        refresh_mirrors(S, L, vx, vy);
    }
}
/* Damped red-black Gauss-Seidel, Eq. sor_update, reading R11: four phases
 * (vx,red)(vx,black)(vy,red)(vy,black), red = (i+j) even on global indices; within a
 * phase each unknown is updated serially in row-major order with current values. */
static void smooth_rbgs(const oracle_t *S, olevel *L, double *vx, double *vy, const double *bx,
                        const double *by, int nu) {
    double w = S->o.omega_v;
    for (int s = 0; s < nu; ++s) {
        for (int colour = 0; colour < 2; ++colour) {
            FOR_VX(L) if (((i + j) & 1) == colour) {
                double r = bx[IX(L, i, j)] - Lx_point(L, vx, vy, i, j);
                vx[IX(L, i, j)] += w * r / Lx_diag(S, L, i, j);
            }
            refresh_mirrors(S, L, vx, vy);
        }
        for (int colour = 0; colour < 2; ++colour) {
            FOR_VY(L) if (((i + j) & 1) == colour) {
                double r = by[IX(L, i, j)] - Ly_point(L, vx, vy, i, j);
                vy[IX(L, i, j)] += w * r / Ly_diag(S, L, i, j);
            }
            refresh_mirrors(S, L, vx, vy);
        }
    }
}
/* RAS-type temporal blocking, Alg. 3, reading R27.  N_outer =
 * ceil(nu / T_inner), made even; per outer iteration a shift (s_i, s_j) in [0, T)^2 from
 * the counter-based generator below partitions the cells into tiles ((i-1+s_i) div T,
 * (j-1+s_j) div T), clipped at the walls; a vx / vy node belongs to the tile of its cell
 * (i, j).  Each tile runs T_inner damped-Jacobi sweeps on its own unknowns with every
 * value outside the tile frozen at the start of the outer iteration (its mirrors follow
 * the tile's own values), then writes its unknowns back (single writer). */
static uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static void ras_shift(oracle_t *S, int *si, int *sj) {
    const uint64_t q = (uint64_t)S->ras_k * 65536u + (uint64_t)(S->ras_c++);
    const uint64_t u = splitmix64(S->o.ras_seed ^ (q * 0x9E3779B97F4A7C15ull));
    *si = (int)((u & 0xffffffffull) % (uint64_t)S->o.ras_tile);
    *sj = (int)((u >> 32) % (uint64_t)S->o.ras_tile);
}
static void smooth_ras(oracle_t *S, olevel *L, double *vx, double *vy, const double *bx, const double *by, int nu) {
    const int T = S->o.ras_tile, Tin = S->o.ras_inner;
    int nout = (nu + Tin - 1) / Tin;
    nout += nout % 2;
    const double w = S->o.omega_v;
    const double sW = sgn_of(S->bc[0]), sE = sgn_of(S->bc[1]), sN = sgn_of(S->bc[2]), sS = sgn_of(S->bc[3]);
    size_t n = padn(L);
    double *x0 = zalloc(n), *y0 = zalloc(n), *nx_ = zalloc(n), *ny_ = zalloc(n);
    for (int t = 0; t < nout; ++t) {
        int si, sj;
        ras_shift(S, &si, &sj);
        memcpy(x0, vx, n * sizeof(double)); /* frozen state of this outer iteration */
        memcpy(y0, vy, n * sizeof(double));
        /* view arrays = frozen state; a tile overlays its own current values while it works */
        memcpy(L->tx, vx, n * sizeof(double));
        memcpy(L->ty, vy, n * sizeof(double));
        const int nti = (L->ncy + si + T - 1) / T, ntj = (L->ncx + sj + T - 1) / T;
        for (int ti = 0; ti < nti; ++ti)
            for (int tj = 0; tj < ntj; ++tj) {
                const int i0 = ti * T - si + 1 > 1 ? ti * T - si + 1 : 1;
                const int i1 = (ti + 1) * T - si < L->ncy ? (ti + 1) * T - si : L->ncy;
                const int j0 = tj * T - sj + 1 > 1 ? tj * T - sj + 1 : 1;
                const int j1 = (tj + 1) * T - sj < L->ncx ? (tj + 1) * T - sj : L->ncx;
                if (i0 > i1 || j0 > j1) continue;
                const int xj1 = j1 < L->ncx - 1 ? j1 : L->ncx - 1, yi1 = i1 < L->ncy - 1 ? i1 : L->ncy - 1;
                for (int tau = 0; tau < Tin; ++tau) {
                    for (int i = i0; i <= i1; ++i)
                        for (int j = j0; j <= xj1; ++j)
                            nx_[IX(L, i, j)] = L->tx[IX(L, i, j)] + w * (bx[IX(L, i, j)] - Lx_point(L, L->tx, L->ty, i, j)) /
                                                                      Lx_diag(S, L, i, j);
                    for (int i = i0; i <= yi1; ++i)
                        for (int j = j0; j <= j1; ++j)
                            ny_[IX(L, i, j)] = L->ty[IX(L, i, j)] + w * (by[IX(L, i, j)] - Ly_point(L, L->tx, L->ty, i, j)) /
                                                                      Ly_diag(S, L, i, j);
                    for (int i = i0; i <= i1; ++i)
                        for (int j = j0; j <= xj1; ++j) {
                            L->tx[IX(L, i, j)] = nx_[IX(L, i, j)];
                            if (i == 1) L->tx[IX(L, 0, j)] = sN * nx_[IX(L, i, j)];
                            if (i == L->ncy) L->tx[IX(L, L->ncy + 1, j)] = sS * nx_[IX(L, i, j)];
                        }
                    for (int i = i0; i <= yi1; ++i)
                        for (int j = j0; j <= j1; ++j) {
                            L->ty[IX(L, i, j)] = ny_[IX(L, i, j)];
                            if (j == 1) L->ty[IX(L, i, 0)] = sW * ny_[IX(L, i, j)];
                            if (j == L->ncx) L->ty[IX(L, i, L->ncx + 1)] = sE * ny_[IX(L, i, j)];
                        }
                }
                /* single writer: the tile's unknowns go to the result; the view gets the frozen
                 * values back for the next tile */
                for (int i = i0; i <= i1; ++i)
                    for (int j = j0; j <= xj1; ++j) {
                        vx[IX(L, i, j)] = L->tx[IX(L, i, j)];
                        L->tx[IX(L, i, j)] = x0[IX(L, i, j)];
                        if (i == 1) L->tx[IX(L, 0, j)] = x0[IX(L, 0, j)];
                        if (i == L->ncy) L->tx[IX(L, L->ncy + 1, j)] = x0[IX(L, L->ncy + 1, j)];
                    }
                for (int i = i0; i <= yi1; ++i)
                    for (int j = j0; j <= j1; ++j) {
                        vy[IX(L, i, j)] = L->ty[IX(L, i, j)];
                        L->ty[IX(L, i, j)] = y0[IX(L, i, j)];
                        if (j == 1) L->ty[IX(L, i, 0)] = y0[IX(L, i, 0)];
                        if (j == L->ncx) L->ty[IX(L, i, L->ncx + 1)] = y0[IX(L, i, L->ncx + 1)];
                    }
            }
        refresh_mirrors(S, L, vx, vy);
    }
    free(x0); free(y0); free(nx_); free(ny_);
}
static void smooth(oracle_t *S, olevel *L, double *vx, double *vy, const double *bx, const double *by, int nu) {
    const int ras = S->o.smoother == 2 || (S->o.smoother == 3 && L != &S->lev[0]);
    if (ras) smooth_ras(S, L, vx, vy, bx, by, nu);
    else if (S->o.smoother == 1) smooth_rbgs(S, L, vx, vy, bx, by, nu);
    else smooth_jacobi(S, L, vx, vy, bx, by, nu);
}

/* ------------------------------------------------ transfers (a5, a6, a7)
 * Node types: position of index (i,j) in units of the spacing is (j + ox, i + oy):
 *   basic (0,0), vx (0,-1/2), vy (-1/2,0), P (-1/2,-1/2)  (PAPER.md:615 lower-right rule). */
enum { T_VX = 0, T_VY = 1, T_P = 2, T_B = 3 };
static void type_offsets(int t, double *ox, double *oy) {
    *ox = (t == T_VY || t == T_P) ? -0.5 : 0.0;
    *oy = (t == T_VX || t == T_P) ? -0.5 : 0.0;
}
/* index ranges of the nodes of type t "inside the closed domain" (reading R6):
 * unknowns and wall nodes; mirror/ghost nodes excluded. */
static void type_range(int t, int ncx, int ncy, int *i0, int *i1, int *j0, int *j1) {
    switch (t) {
    case T_VX: *i0 = 1; *i1 = ncy; *j0 = 0; *j1 = ncx; break;
    case T_VY: *i0 = 0; *i1 = ncy; *j0 = 1; *j1 = ncx; break;
    case T_P: *i0 = 1; *i1 = ncy; *j0 = 1; *j1 = ncx; break;
    default: *i0 = 0; *i1 = ncy; *j0 = 0; *j1 = ncx; break;
    }
}
static double hat(double d, double H) { /* bilinear weight, Alg. 2: w = (1-|r_x|)(1-|r_y|) */
    double r = fabs(d) / H;
    return r < 1.0 ? 1.0 - r : 0.0;
}
/* Normalised bilinear restriction (Alg. 2 weights, reading R6):
 *   u^H(I,J) = sum_p w_Ip u^h(p) / sum_p w_Ip,  w = hat_H(dx) hat_H(dy),
 * over fine nodes p of the same type inside the closed domain; each fine node counted once.
 * Writes coarse nodes in [ci0,ci1]x[cj0,cj1]. */
static void restrict_generic(const olevel *F, const olevel *C, int t, const double *uf, double *uc, int ci0,
                             int ci1, int cj0, int cj1) {
    double ox, oy;
    type_offsets(t, &ox, &oy);
    int i0, i1, j0, j1;
    type_range(t, F->ncx, F->ncy, &i0, &i1, &j0, &j1);
    double Hx = C->dx, Hy = C->dy;
    for (int I = ci0; I <= ci1; ++I)
        for (int J = cj0; J <= cj1; ++J) {
            double X = (J + ox) * Hx, Y = (I + oy) * Hy;
            double num = 0.0, den = 0.0;
            /* candidate fine nodes: |x - X| < Hx  <=>  j within a window around 2J */
            for (int i = 2 * I - 3; i <= 2 * I + 3; ++i) {
                if (i < i0 || i > i1) continue;
                double wy = hat((i + oy) * F->dy - Y, Hy);
                if (wy == 0.0) continue;
                for (int j = 2 * J - 3; j <= 2 * J + 3; ++j) {
                    if (j < j0 || j > j1) continue;
                    double wx = hat((j + ox) * F->dx - X, Hx);
                    if (wx == 0.0) continue;
                    double w = wx * wy;
                    num += w * uf[IX(F, i, j)];
                    den += w;
                }
            }
            uc[IX(C, I, J)] = num / den;
        }
}
/* Bilinear prolongation: each fine node receives the hat-weighted sum of
 * the surrounding coarse nodes of the same type, coarse mirror nodes holding the
 * homogeneous-BC image and wall nodes zero (reading R6/Appendix B).  u_f += P u_c. */
static void prolong_add(const olevel *F, const olevel *C, int t, const double *uc, double *uf) {
    double ox, oy;
    type_offsets(t, &ox, &oy);
    int fi0, fi1, fj0, fj1;
    if (t == T_VX) { fi0 = 1; fi1 = F->ncy; fj0 = 1; fj1 = F->ncx - 1; }
    else { fi0 = 1; fi1 = F->ncy - 1; fj0 = 1; fj1 = F->ncx; }
    for (int i = fi0; i <= fi1; ++i)
        for (int j = fj0; j <= fj1; ++j) {
            double x = (j + ox) * F->dx, y = (i + oy) * F->dy;
            double s = 0.0;
            for (int I = i / 2 - 2; I <= i / 2 + 2; ++I) {
                if (I < 0 || I > C->ncy + 1) continue;
                double wy = hat((I + oy) * C->dy - y, C->dy);
                if (wy == 0.0) continue;
                for (int J = j / 2 - 2; J <= j / 2 + 2; ++J) {
                    if (J < 0 || J > C->ncx + 1) continue;
                    double wx = hat((J + ox) * C->dx - x, C->dx);
                    if (wx == 0.0) continue;
                    s += wx * wy * uc[IX(C, I, J)];
                }
            }
            uf[IX(F, i, j)] += s;
        }
}

/* ------------------------------------------------ coarsest solve (a8, reading R10)
 * Dense -L_c with the mirror relations folded in (the true operator), Cholesky. */
static int nunk(const olevel *L) { return L->ncy * (L->ncx - 1) + (L->ncy - 1) * L->ncx; }
static void pack_unknowns(const olevel *L, const double *vx, const double *vy, double *u) {
    int k = 0;
    FOR_VX(L) u[k++] = vx[IX(L, i, j)];
    FOR_VY(L) u[k++] = vy[IX(L, i, j)];
}
static void unpack_unknowns(const olevel *L, const double *u, double *vx, double *vy) {
    int k = 0;
    FOR_VX(L) vx[IX(L, i, j)] = u[k++];
    FOR_VY(L) vy[IX(L, i, j)] = u[k++];
}
static int build_coarse_direct(oracle_t *S) {
    olevel *L = &S->lev[S->nlev - 1];
    int n = nunk(L);
    S->nc = n;
    free(S->chol);
    S->chol = zalloc((size_t)n * n);
    double *e = zalloc(n), *vx = zalloc(padn(L)), *vy = zalloc(padn(L)), *col = zalloc(n);
    double *ax = zalloc(padn(L)), *ay = zalloc(padn(L)), *zero = zalloc(padn(L));
    for (int c = 0; c < n; ++c) {
        memset(e, 0, n * sizeof(double));
        e[c] = 1.0;
        memset(vx, 0, padn(L) * sizeof(double));
        memset(vy, 0, padn(L) * sizeof(double));
        unpack_unknowns(L, e, vx, vy);
        refresh_mirrors(S, L, vx, vy);
        residual_v(L, vx, vy, zero, zero, ax, ay); /* = -L e */
        pack_unknowns(L, ax, ay, col);
        for (int r = 0; r < n; ++r) S->chol[(size_t)r * n + c] = col[r];
    }
    /* symmetrise against rounding of the two equal off-diagonal formulas */
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < r; ++c) {
            double a = 0.5 * (S->chol[(size_t)r * n + c] + S->chol[(size_t)c * n + r]);
            S->chol[(size_t)r * n + c] = a;
            S->chol[(size_t)c * n + r] = a;
        }
    /* in-place Cholesky, lower triangle */
    int ok = 1;
    for (int j = 0; j < n && ok; ++j) {
        double d = S->chol[(size_t)j * n + j];
        for (int k = 0; k < j; ++k) d -= S->chol[(size_t)j * n + k] * S->chol[(size_t)j * n + k];
        if (!(d > 0.0)) { ok = 0; break; }
        d = sqrt(d);
        S->chol[(size_t)j * n + j] = d;
        for (int i = j + 1; i < n; ++i) {
            double s = S->chol[(size_t)i * n + j];
            for (int k = 0; k < j; ++k) s -= S->chol[(size_t)i * n + k] * S->chol[(size_t)j * n + k];
            S->chol[(size_t)i * n + j] = s / d;
        }
    }
    free(e); free(vx); free(vy); free(col); free(ax); free(ay); free(zero);
    return ok ? 0 : -1;
}
/* solve L_c v = b, i.e. (-L_c) v = -b */
static void coarse_direct_solve(const oracle_t *S, olevel *L, double *vx, double *vy, const double *bx,
                                const double *by) {
    int n = S->nc;
    double *u = zalloc(n);
    pack_unknowns(L, bx, by, u);
    for (int k = 0; k < n; ++k) u[k] = -u[k];
    for (int i = 0; i < n; ++i) { /* forward */
        double s = u[i];
        for (int k = 0; k < i; ++k) s -= S->chol[(size_t)i * n + k] * u[k];
        u[i] = s / S->chol[(size_t)i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) { /* backward */
        double s = u[i];
        for (int k = i + 1; k < n; ++k) s -= S->chol[(size_t)k * n + i] * u[k];
        u[i] = s / S->chol[(size_t)i * n + i];
    }
    unpack_unknowns(L, u, vx, vy);
    refresh_mirrors(S, L, vx, vy);
    free(u);
}

/* ------------------------------------------------ V-cycle (a9), Eq. multigrid_levels */
static void vcycle_level(oracle_t *S, int l, double *vx, double *vy, const double *bx, const double *by) {
    olevel *L = &S->lev[l];
    if (l == S->nlev - 1) {
        if (S->o.coarse_direct) coarse_direct_solve(S, L, vx, vy, bx, by);
        else smooth(S, L, vx, vy, bx, by, 2 * L->nu);
        return;
    }
    olevel *C = &S->lev[l + 1];
    smooth(S, L, vx, vy, bx, by, L->nu);                               /* (1) pre-smoothing */
    residual_v(L, vx, vy, bx, by, L->rx, L->ry);                       /* (2) residual */
    memset(C->bx, 0, padn(C) * sizeof(double));
    memset(C->by, 0, padn(C) * sizeof(double));
    restrict_generic(L, C, T_VX, L->rx, C->bx, 1, C->ncy, 1, C->ncx - 1); /* (3) restrict */
    restrict_generic(L, C, T_VY, L->ry, C->by, 1, C->ncy - 1, 1, C->ncx);
    memset(C->ex, 0, padn(C) * sizeof(double));                         /* coarse guess 0 */
    memset(C->ey, 0, padn(C) * sizeof(double));
    vcycle_level(S, l + 1, C->ex, C->ey, C->bx, C->by);                 /* (4) recurse */
    refresh_mirrors(S, C, C->ex, C->ey);
    prolong_add(L, C, T_VX, C->ex, vx);                                 /* (5) correct */
    prolong_add(L, C, T_VY, C->ey, vy);
    refresh_mirrors(S, L, vx, vy);
    smooth(S, L, vx, vy, bx, by, L->nu);                               /* (6) post-smoothing */
}

/* ------------------------------------------------ energy norm (a3) */
static void body_force(const oracle_t *S, double *fx, double *fy) {
    const olevel *L = &S->lev[0];
    memset(fx, 0, padn(L) * sizeof(double));
    memset(fy, 0, padn(L) * sizeof(double));
    /* reading R4/R23: f = -g * rho averaged to the velocity node (y down, g_y > 0 downward) */
    FOR_VX(L) fx[IX(L, i, j)] = -S->gx * (S->rhob[IX(L, i - 1, j)] + S->rhob[IX(L, i, j)]) / 2.0;
    FOR_VY(L) fy[IX(L, i, j)] = -S->gy * (S->rhob[IX(L, i, j - 1)] + S->rhob[IX(L, i, j)]) / 2.0;
}
/* weighted sums: Sv = sum r^2/d over vx then vy, d = -a_ii (diag(-L), reading R5); Sp = sum rp^2 eta/(2/dx^2+2/dy^2) */
static double sum_vel_energy(const oracle_t *S, const olevel *L, const double *rx, const double *ry) {
    size_t n = (size_t)nunk(L), k = 0;
    double *t = zalloc(n);
    FOR_VX(L) t[k++] = rx[IX(L, i, j)] * rx[IX(L, i, j)] / (-Lx_diag(S, L, i, j));
    FOR_VY(L) t[k++] = ry[IX(L, i, j)] * ry[IX(L, i, j)] / (-Ly_diag(S, L, i, j));
    double s = pairwise(t, n);
    free(t);
    return s;
}
static double sum_p_energy(const olevel *L, const double *rp) {
    size_t n = (size_t)L->ncx * L->ncy, k = 0;
    double *t = zalloc(n);
    double c = 2.0 / (L->dx * L->dx) + 2.0 / (L->dy * L->dy);
    FOR_P(L) t[k++] = rp[IX(L, i, j)] * rp[IX(L, i, j)] * (L->etap[IX(L, i, j)] / c);
    double s = pairwise(t, n);
    free(t);
    return s;
}
static double p_mean(const olevel *L, const double *p) {
    size_t n = (size_t)L->ncx * L->ncy, k = 0;
    double *t = zalloc(n);
    FOR_P(L) t[k++] = p[IX(L, i, j)];
    double s = pairwise(t, n) / (double)n;
    free(t);
    return s;
}
/* full residual of the saddle system: rv = f - L v - G p, rp = 0 - D v */
static void full_residual(const oracle_t *S, const double *vx, const double *vy, const double *p, double *rx,
                          double *ry, double *rp) {
    const olevel *L = &S->lev[0];
    memset(rx, 0, padn(L) * sizeof(double));
    memset(ry, 0, padn(L) * sizeof(double));
    memset(rp, 0, padn(L) * sizeof(double));
    FOR_VX(L) rx[IX(L, i, j)] = S->fx[IX(L, i, j)] - (Lx_point(L, vx, vy, i, j) + Gx_point(L, p, i, j));
    FOR_VY(L) ry[IX(L, i, j)] = S->fy[IX(L, i, j)] - (Ly_point(L, vx, vy, i, j) + Gy_point(L, p, i, j));
    FOR_P(L) rp[IX(L, i, j)] = -D_point(L, vx, vy, i, j);
}
static double energy_of(const oracle_t *S, const double *rx, const double *ry, const double *rp, double Sf) {
    const olevel *L = &S->lev[0];
    return sqrt((sum_vel_energy(S, L, rx, ry) + sum_p_energy(L, rp)) / Sf);
}

/* ------------------------------------------------ layout conversion (user <-> padded)
 * user layout (no ghosts): vx ny x (nx+1), vy (ny+1) x nx, p/eta_p ny x nx, eta_b/rho_b (ny+1) x (nx+1) */
static void in_vx(const olevel *L, const double *u, double *a) {
    for (int i = 0; i < L->ncy; ++i)
        for (int j = 0; j <= L->ncx; ++j) a[IX(L, i + 1, j)] = u[(size_t)i * (L->ncx + 1) + j];
}
static void in_vy(const olevel *L, const double *u, double *a) {
    for (int i = 0; i <= L->ncy; ++i)
        for (int j = 0; j < L->ncx; ++j) a[IX(L, i, j + 1)] = u[(size_t)i * L->ncx + j];
}
static void in_p(const olevel *L, const double *u, double *a) {
    for (int i = 0; i < L->ncy; ++i)
        for (int j = 0; j < L->ncx; ++j) a[IX(L, i + 1, j + 1)] = u[(size_t)i * L->ncx + j];
}
static void in_b(const olevel *L, const double *u, double *a) {
    for (int i = 0; i <= L->ncy; ++i)
        for (int j = 0; j <= L->ncx; ++j) a[IX(L, i, j)] = u[(size_t)i * (L->ncx + 1) + j];
}
static void out_vx(const olevel *L, const double *a, double *u) {
    for (int i = 0; i < L->ncy; ++i)
        for (int j = 0; j <= L->ncx; ++j)
            u[(size_t)i * (L->ncx + 1) + j] = (j == 0 || j == L->ncx) ? 0.0 : a[IX(L, i + 1, j)];
}
static void out_vy(const olevel *L, const double *a, double *u) {
    for (int i = 0; i <= L->ncy; ++i)
        for (int j = 0; j < L->ncx; ++j)
            u[(size_t)i * L->ncx + j] = (i == 0 || i == L->ncy) ? 0.0 : a[IX(L, i, j + 1)];
}
static void out_p(const olevel *L, const double *a, double *u) {
    for (int i = 0; i < L->ncy; ++i)
        for (int j = 0; j < L->ncx; ++j) u[(size_t)i * L->ncx + j] = a[IX(L, i + 1, j + 1)];
}
static void out_b(const olevel *L, const double *a, double *u) {
    for (int i = 0; i <= L->ncy; ++i)
        for (int j = 0; j <= L->ncx; ++j) u[(size_t)i * (L->ncx + 1) + j] = a[IX(L, i, j)];
}
/* velocity input: unknowns from the user array, walls zero, mirrors from their partners */
static void in_velocity(const oracle_t *S, const olevel *L, const double *ux, const double *uy, double *vx,
                        double *vy) {
    memset(vx, 0, padn(L) * sizeof(double));
    memset(vy, 0, padn(L) * sizeof(double));
    FOR_VX(L) vx[IX(L, i, j)] = ux[(size_t)(i - 1) * (L->ncx + 1) + j];
    FOR_VY(L) vy[IX(L, i, j)] = uy[(size_t)i * L->ncx + (j - 1)];
    refresh_mirrors(S, L, vx, vy);
}

/* ================================================================== public API */
#define O_OK 0
#define O_NOT_CONVERGED 1
#define O_EINVAL (-1)
#define O_ENOMEM (-2)
#define O_EDIVERGED (-5)
#define O_ESTATE (-6)

int oracle_opts_default(oracle_opts *o) {
    if (!o) return O_EINVAL;
    o->smoother = 0;
    o->omega_v = 0.3;
    o->alpha_p = 0.6;
    o->nu1 = 5;
    o->nu_growth = 1.0;
    o->coarse_min = 8;
    o->coarse_direct = 1;
    o->vcycles_per_iter = 1;
    o->accel = 0;
    o->gcr_restart = 10;
    o->gcr_true_restart = 1;
    o->gcr_inner = 0;
    o->max_iter = 10000;
    o->pressure_sign = 1;
    o->theta_step = 0.0;
    o->theta_every = 25;
    o->aa_depth = 5;
    o->aa_beta = 0.7;
    o->ras_tile = 32;
    o->ras_inner = 4;
    o->ras_seed = 2603;
    return O_OK;
}

static void alloc_level(olevel *L, int ncx, int ncy, double Lx, double Ly) {
    L->ncx = ncx; L->ncy = ncy; L->W = ncx + 2;
    L->dx = Lx / ncx; L->dy = Ly / ncy;
    size_t n = padn(L);
    L->etab = zalloc(n); L->etap = zalloc(n);
    L->rx = zalloc(n); L->ry = zalloc(n); L->bx = zalloc(n); L->by = zalloc(n);
    L->ex = zalloc(n); L->ey = zalloc(n); L->tx = zalloc(n); L->ty = zalloc(n);
}

int oracle_create(int nx, int ny, double Lx, double Ly, const int *bc, const oracle_opts *opts, oracle_t **out) {
    if (!out || nx < 2 || ny < 2 || !(Lx > 0) || !(Ly > 0) || !bc) return O_EINVAL;
    for (int k = 0; k < 4; ++k) if (bc[k] != 0 && bc[k] != 1) return O_EINVAL;
    oracle_t *S = (oracle_t *)calloc(1, sizeof(oracle_t));
    S->nx = nx; S->ny = ny; S->Lx = Lx; S->Ly = Ly;
    memcpy(S->bc, bc, sizeof(S->bc));
    if (opts) S->o = *opts; else oracle_opts_default(&S->o);
    if (S->o.nu1 < 0 || S->o.coarse_min < 2 || S->o.vcycles_per_iter < 1 || S->o.gcr_restart < 1 ||
        !(S->o.theta_step >= 0.0 && S->o.theta_step <= 1.0) || S->o.theta_every < 1 || S->o.accel < 0 ||
        S->o.accel > 2 || S->o.aa_depth < 0 || S->o.aa_depth > 15 || !(S->o.aa_beta > 0.0 && S->o.aa_beta <= 1.0) ||
        S->o.smoother < 0 || S->o.smoother > 3 || S->o.ras_tile < 2 || S->o.ras_inner < 1) {
        free(S);
        return O_EINVAL;
    }
    S->gx = 0.0; S->gy = 0.0;
    /* hierarchy (reading R8): factor 2 while both even and min/2 >= coarse_min */
    int cx = nx, cy = ny, l = 0;
    for (;;) {
        alloc_level(&S->lev[l], cx, cy, Lx, Ly);
        double nu = floor(S->o.nu1 * pow(S->o.nu_growth, (double)l) + 0.5);
        S->lev[l].nu = (int)nu;
        ++l;
        if (l >= MAXLEV) break;
        if ((cx % 2) || (cy % 2)) break;
        int m = cx < cy ? cx : cy;
        if (m / 2 < S->o.coarse_min) break;
        cx /= 2; cy /= 2;
    }
    S->nlev = l;
    size_t n = padn(&S->lev[0]);
    S->rhob = zalloc(n); S->fx = zalloc(n); S->fy = zalloc(n);
    S->vx = zalloc(n); S->vy = zalloc(n); S->p = zalloc(n);
    S->etab_user = zalloc(n); S->etap_user = zalloc(n);
    *out = S;
    return O_OK;
}

int oracle_destroy(oracle_t *S) {
    if (!S) return O_EINVAL;
    for (int l = 0; l < S->nlev; ++l) {
        olevel *L = &S->lev[l];
        free(L->etab); free(L->etap); free(L->rx); free(L->ry); free(L->bx); free(L->by);
        free(L->ex); free(L->ey); free(L->tx); free(L->ty);
    }
    free(S->rhob); free(S->fx); free(S->fy); free(S->vx); free(S->vy); free(S->p); free(S->chol);
    free(S->etab_user); free(S->etap_user);
    free(S);
    return O_OK;
}

int oracle_num_levels(const oracle_t *S) { return S ? S->nlev : O_EINVAL; }
int oracle_level_shape(const oracle_t *S, int l, int *ncx, int *ncy, int *nu) {
    if (!S || l < 0 || l >= S->nlev) return O_EINVAL;
    *ncx = S->lev[l].ncx; *ncy = S->lev[l].ncy; *nu = S->lev[l].nu;
    return O_OK;
}

static void update_force(oracle_t *S) {
    if (!S->force_override) body_force(S, S->fx, S->fy);
}

/* coarse viscosities (a7, reading R7: the same normalised bilinear restriction,
 * arithmetic) and the coarsest factorisation (a8) from the fine-level viscosities */
static int build_hierarchy(oracle_t *S) {
    for (int l = 0; l + 1 < S->nlev; ++l) {
        olevel *A = &S->lev[l], *C = &S->lev[l + 1];
        restrict_generic(A, C, T_B, A->etab, C->etab, 0, C->ncy, 0, C->ncx);
        restrict_generic(A, C, T_P, A->etap, C->etap, 1, C->ncy, 1, C->ncx);
    }
    S->have_eta = 1;
    if (S->o.coarse_direct) {
        if (nunk(&S->lev[S->nlev - 1]) > 1024) return O_EINVAL; /* same cap as the library */
        if (build_coarse_direct(S) != 0) return O_EINVAL;
    }
    return O_OK;
}

/* set_viscosity: copies eta (kept as the caller's field for viscosity rescaling) and
 * builds the hierarchy. */
int oracle_set_viscosity(oracle_t *S, const double *eta_b, const double *eta_p) {
    if (!S || !eta_b || !eta_p) return O_EINVAL;
    olevel *F = &S->lev[0];
    for (size_t k = 0; k < (size_t)(S->ny + 1) * (S->nx + 1); ++k) if (!(eta_b[k] > 0)) return O_EINVAL;
    for (size_t k = 0; k < (size_t)S->ny * S->nx; ++k) if (!(eta_p[k] > 0)) return O_EINVAL;
    in_b(F, eta_b, F->etab);
    in_p(F, eta_p, F->etap);
    memcpy(S->etab_user, F->etab, padn(F) * sizeof(double));
    memcpy(S->etap_user, F->etap, padn(F) * sizeof(double));
    return build_hierarchy(S);
}

/* Viscosity rescaling: eta_comp = (1 - theta) eta_min + theta eta on
 * both fine viscosity fields, eta_min = the minimum over both caller fields (basic nodes
 * [0,ncy]x[0,ncx], P nodes [1,ncy]x[1,ncx]); then the hierarchy is rebuilt from eta_comp.
 * theta = 1 restores the caller's field exactly. */
int oracle_blend_viscosity(oracle_t *S, double theta) {
    if (!S || !S->have_eta || !(theta >= 0.0 && theta <= 1.0)) return O_EINVAL;
    olevel *F = &S->lev[0];
    double emin = INFINITY;
    for (int i = 0; i <= F->ncy; ++i)
        for (int j = 0; j <= F->ncx; ++j) emin = fmin(emin, S->etab_user[IX(F, i, j)]);
    FOR_P(F) emin = fmin(emin, S->etap_user[IX(F, i, j)]);
    for (int i = 0; i <= F->ncy; ++i)
        for (int j = 0; j <= F->ncx; ++j)
            F->etab[IX(F, i, j)] = (1.0 - theta) * emin + theta * S->etab_user[IX(F, i, j)];
    FOR_P(F) F->etap[IX(F, i, j)] = (1.0 - theta) * emin + theta * S->etap_user[IX(F, i, j)];
    return build_hierarchy(S);
}
int oracle_set_density(oracle_t *S, const double *rho_b) {
    if (!S || !rho_b) return O_EINVAL;
    in_b(&S->lev[0], rho_b, S->rhob);
    S->have_rho = 1;
    update_force(S);
    return O_OK;
}
int oracle_set_gravity(oracle_t *S, double gx, double gy) {
    if (!S) return O_EINVAL;
    S->gx = gx; S->gy = gy;
    update_force(S);
    return O_OK;
}
/* test hook: arbitrary body force (vx / vy user layouts) -- used by the no-slip MMS pin P3 */
int oracle_set_force(oracle_t *S, const double *fx, const double *fy) {
    if (!S || !fx || !fy) return O_EINVAL;
    olevel *L = &S->lev[0];
    double *tx = zalloc(padn(L)), *ty = zalloc(padn(L));
    in_vx(L, fx, tx); in_vy(L, fy, ty);
    memset(S->fx, 0, padn(L) * sizeof(double));
    memset(S->fy, 0, padn(L) * sizeof(double));
    FOR_VX(L) S->fx[IX(L, i, j)] = tx[IX(L, i, j)];
    FOR_VY(L) S->fy[IX(L, i, j)] = ty[IX(L, i, j)];
    free(tx); free(ty);
    S->force_override = 1; S->have_rho = 1;
    return O_OK;
}
int oracle_get_viscosity(const oracle_t *S, int l, double *eta_b, double *eta_p) {
    if (!S || l < 0 || l >= S->nlev || !S->have_eta) return O_EINVAL;
    out_b(&S->lev[l], S->lev[l].etab, eta_b);
    out_p(&S->lev[l], S->lev[l].etap, eta_p);
    return O_OK;
}

/* Lithostatic pressure: p(x, y) = int_0^y rho(x, y') g_y dy', the
 * column integral from the top wall to each P node with the density at the vy nodes
 * (reading R23) -- the discrete hydrostatic balance of the y-momentum row with v = 0
 * (f_y = -g_y rho, G_y p = -(p(i+1,j) - p(i,j))/dy; reading R4):
 *   p(1, j) = g_y (dy/2) rho_vy(0, j),   p(i+1, j) = p(i, j) + g_y dy rho_vy(i, j).
 * Output in the P layout (ny x nx), not de-meaned. */
int oracle_lithostatic(const oracle_t *S, double *p) {
    if (!S || !p) return O_EINVAL;
    if (!S->have_rho) return O_ESTATE;
    const olevel *L = &S->lev[0];
    const double *rb = S->rhob;
    for (int j = 1; j <= L->ncx; ++j) {
        double acc = S->gy * (0.5 * L->dy) * (0.5 * (rb[IX(L, 0, j - 1)] + rb[IX(L, 0, j)]));
        p[(size_t)0 * L->ncx + (j - 1)] = acc;
        for (int i = 1; i < L->ncy; ++i) {
            acc = acc + S->gy * L->dy * (0.5 * (rb[IX(L, i, j - 1)] + rb[IX(L, i, j)]));
            p[(size_t)i * L->ncx + (j - 1)] = acc;
        }
    }
    return O_OK;
}

/* apply_operator: ax, ay = L v + G p (vx/vy layouts, walls 0), ap = D v (P layout) */
int oracle_apply_operator(oracle_t *S, const double *vx, const double *vy, const double *p, double *ax,
                          double *ay, double *ap) {
    if (!S || !S->have_eta) return O_ESTATE;
    olevel *L = &S->lev[0];
    in_velocity(S, L, vx, vy, S->vx, S->vy);
    memset(S->p, 0, padn(L) * sizeof(double));
    in_p(L, p, S->p);
    double *tx = zalloc(padn(L)), *ty = zalloc(padn(L)), *tp = zalloc(padn(L));
    FOR_VX(L) tx[IX(L, i, j)] = Lx_point(L, S->vx, S->vy, i, j) + Gx_point(L, S->p, i, j);
    FOR_VY(L) ty[IX(L, i, j)] = Ly_point(L, S->vx, S->vy, i, j) + Gy_point(L, S->p, i, j);
    FOR_P(L) tp[IX(L, i, j)] = D_point(L, S->vx, S->vy, i, j);
    out_vx(L, tx, ax); out_vy(L, ty, ay); out_p(L, tp, ap);
    free(tx); free(ty); free(tp);
    return O_OK;
}

static double force_energy(const oracle_t *S) { return sum_vel_energy(S, &S->lev[0], S->fx, S->fy); }

/* residual: rx, ry = f - L v - G p; rp = -D v; rel_energy = E */
int oracle_residual(oracle_t *S, const double *vx, const double *vy, const double *p, double *rx, double *ry,
                    double *rp, double *rel_energy) {
    if (!S || !S->have_eta || !S->have_rho) return O_ESTATE;
    olevel *L = &S->lev[0];
    in_velocity(S, L, vx, vy, S->vx, S->vy);
    memset(S->p, 0, padn(L) * sizeof(double));
    in_p(L, p, S->p);
    double *tx = zalloc(padn(L)), *ty = zalloc(padn(L)), *tp = zalloc(padn(L));
    full_residual(S, S->vx, S->vy, S->p, tx, ty, tp);
    if (rx) out_vx(L, tx, rx);
    if (ry) out_vy(L, ty, ry);
    if (rp) out_p(L, tp, rp);
    if (rel_energy) {
        double Sf = force_energy(S);
        *rel_energy = Sf > 0 ? energy_of(S, tx, ty, tp, Sf) : 0.0;
    }
    free(tx); free(ty); free(tp);
    return O_OK;
}

/* ------------------------------------------------ extended-precision residual (verification)
 * The residual and energy norm of oracle_residual -- the same formulas (Listing x row, stress
 * y row, G, D, the weights of E) -- evaluated in long
 * double (x87 80-bit: 64-bit significand, unit roundoff 5.4e-20 against 1.1e-16).  Verification
 * only (reading R34): near convergence the Listing's coefficient form cancels terms
 * ~h^-2 larger than the residual, so the FP64 evaluation of E carries rounding noise growing
 * like h^-2 (a few % of E = 1e-8 at 16384^2); this evaluation does not. */
typedef long double ldbl;
static ldbl Lx_point_ld(const olevel *L, const double *vx, const double *vy, int i, int j) {
    ldbl dx = L->dx, dy = L->dy;
    ldbl etaA = L->etap[IX(L, i, j)], etaB = L->etap[IX(L, i, j + 1)];
    ldbl eta1 = L->etab[IX(L, i - 1, j)], eta2 = L->etab[IX(L, i, j)];
    ldbl vx1 = 2.0L * etaA / (dx * dx), vx2 = eta1 / (dy * dy);
    ldbl vx3 = -(eta1 + eta2) / (dy * dy) - 2.0L * (etaA + etaB) / (dx * dx);
    ldbl vx4 = eta2 / (dy * dy), vx5 = 2.0L * etaB / (dx * dx);
    ldbl vy1 = eta1 / (dx * dy), vy2 = -eta2 / (dx * dy), vy3 = -eta1 / (dx * dy), vy4 = eta2 / (dx * dy);
    return vx1 * vx[IX(L, i, j - 1)] + vx2 * vx[IX(L, i - 1, j)] + vx3 * vx[IX(L, i, j)] +
           vx4 * vx[IX(L, i + 1, j)] + vx5 * vx[IX(L, i, j + 1)] + vy1 * vy[IX(L, i - 1, j)] +
           vy2 * vy[IX(L, i, j)] + vy3 * vy[IX(L, i - 1, j + 1)] + vy4 * vy[IX(L, i, j + 1)];
}
static ldbl Ly_point_ld(const olevel *L, const double *vx, const double *vy, int i, int j) {
    ldbl dx = L->dx, dy = L->dy;
    ldbl syy_S = 2.0L * L->etap[IX(L, i + 1, j)] * ((ldbl)vy[IX(L, i + 1, j)] - vy[IX(L, i, j)]) / dy;
    ldbl syy_N = 2.0L * L->etap[IX(L, i, j)] * ((ldbl)vy[IX(L, i, j)] - vy[IX(L, i - 1, j)]) / dy;
    ldbl sxy_E = L->etab[IX(L, i, j)] *
                 (((ldbl)vx[IX(L, i + 1, j)] - vx[IX(L, i, j)]) / dy + ((ldbl)vy[IX(L, i, j + 1)] - vy[IX(L, i, j)]) / dx);
    ldbl sxy_W = L->etab[IX(L, i, j - 1)] *
                 (((ldbl)vx[IX(L, i + 1, j - 1)] - vx[IX(L, i, j - 1)]) / dy +
                  ((ldbl)vy[IX(L, i, j)] - vy[IX(L, i, j - 1)]) / dx);
    return (syy_S - syy_N) / dy + (sxy_E - sxy_W) / dx;
}
int oracle_residual_ld(oracle_t *S, const double *vx, const double *vy, const double *p, double *rx, double *ry,
                       double *rp, double *rel_energy) {
    if (!S || !S->have_eta || !S->have_rho) return O_ESTATE;
    olevel *L = &S->lev[0];
    in_velocity(S, L, vx, vy, S->vx, S->vy);
    memset(S->p, 0, padn(L) * sizeof(double));
    in_p(L, p, S->p);
    const double *V = S->vx, *U = S->vy, *P = S->p;
    double *tx = zalloc(padn(L)), *ty = zalloc(padn(L)), *tp = zalloc(padn(L));
    ldbl dx = L->dx, dy = L->dy, c = 2.0L / (dx * dx) + 2.0L / (dy * dy), sv = 0.0L, sp = 0.0L, sf = 0.0L;
    FOR_VX(L) {
        ldbl g = -(ldbl)P[IX(L, i, j + 1)] / dx + (ldbl)P[IX(L, i, j)] / dx;
        ldbl r = (ldbl)S->fx[IX(L, i, j)] - (Lx_point_ld(L, V, U, i, j) + g), d = -(ldbl)Lx_diag(S, L, i, j);
        tx[IX(L, i, j)] = (double)r;
        sv += r * r / d;
        sf += (ldbl)S->fx[IX(L, i, j)] * S->fx[IX(L, i, j)] / d;
    }
    FOR_VY(L) {
        ldbl g = -(ldbl)P[IX(L, i + 1, j)] / dy + (ldbl)P[IX(L, i, j)] / dy;
        ldbl r = (ldbl)S->fy[IX(L, i, j)] - (Ly_point_ld(L, V, U, i, j) + g), d = -(ldbl)Ly_diag(S, L, i, j);
        ty[IX(L, i, j)] = (double)r;
        sv += r * r / d;
        sf += (ldbl)S->fy[IX(L, i, j)] * S->fy[IX(L, i, j)] / d;
    }
    FOR_P(L) {
        ldbl r = -(((ldbl)V[IX(L, i, j)] - V[IX(L, i, j - 1)]) / dx + ((ldbl)U[IX(L, i, j)] - U[IX(L, i - 1, j)]) / dy);
        tp[IX(L, i, j)] = (double)r;
        sp += r * r * ((ldbl)L->etap[IX(L, i, j)] / c);
    }
    if (rx) out_vx(L, tx, rx);
    if (ry) out_vy(L, ty, ry);
    if (rp) out_p(L, tp, rp);
    if (rel_energy) *rel_energy = sf > 0 ? (double)sqrtl((sv + sp) / sf) : 0.0;
    free(tx); free(ty); free(tp);
    return O_OK;
}

/* energy partial sums (Sv, Sp, Sf) of a residual -- exposes the reduction itself */
int oracle_energy_sums(oracle_t *S, const double *vx, const double *vy, const double *p, double *sums3) {
    if (!S || !S->have_eta || !S->have_rho) return O_ESTATE;
    olevel *L = &S->lev[0];
    in_velocity(S, L, vx, vy, S->vx, S->vy);
    memset(S->p, 0, padn(L) * sizeof(double));
    in_p(L, p, S->p);
    double *tx = zalloc(padn(L)), *ty = zalloc(padn(L)), *tp = zalloc(padn(L));
    full_residual(S, S->vx, S->vy, S->p, tx, ty, tp);
    sums3[0] = sum_vel_energy(S, L, tx, ty);
    sums3[1] = sum_p_energy(L, tp);
    sums3[2] = force_energy(S);
    free(tx); free(ty); free(tp);
    return O_OK;
}

/* one V-cycle on L v = b (level 0); bx/by in vx/vy user layouts (walls ignored) */
int oracle_vcycle(oracle_t *S, const double *bx, const double *by, double *vx, double *vy) {
    if (!S || !S->have_eta) return O_ESTATE;
    olevel *L = &S->lev[0];
    double *pbx = zalloc(padn(L)), *pby = zalloc(padn(L));
    in_vx(L, bx, pbx); in_vy(L, by, pby);
    in_velocity(S, L, vx, vy, S->vx, S->vy);
    S->ras_k = 0; S->ras_c = 0;
    vcycle_level(S, 0, S->vx, S->vy, pbx, pby);
    out_vx(L, S->vx, vx); out_vy(L, S->vy, vy);
    free(pbx); free(pby);
    return O_OK;
}

/* test hooks on an arbitrary level l (arrays in that level's user layout) */
int oracle_smooth(oracle_t *S, int l, const double *bx, const double *by, double *vx, double *vy, int nsweeps) {
    if (!S || !S->have_eta || l < 0 || l >= S->nlev) return O_ESTATE;
    olevel *L = &S->lev[l];
    double *pbx = zalloc(padn(L)), *pby = zalloc(padn(L)), *wx = zalloc(padn(L)), *wy = zalloc(padn(L));
    in_vx(L, bx, pbx); in_vy(L, by, pby);
    in_velocity(S, L, vx, vy, wx, wy);
    S->ras_k = 0; S->ras_c = 0;
    smooth(S, L, wx, wy, pbx, pby, nsweeps);
    out_vx(L, wx, vx); out_vy(L, wy, vy);
    free(pbx); free(pby); free(wx); free(wy);
    return O_OK;
}
/* residual b - L v at level l (vx/vy layouts) */
int oracle_level_residual(oracle_t *S, int l, const double *bx, const double *by, const double *vx,
                          const double *vy, double *rx, double *ry) {
    if (!S || !S->have_eta || l < 0 || l >= S->nlev) return O_ESTATE;
    olevel *L = &S->lev[l];
    double *pbx = zalloc(padn(L)), *pby = zalloc(padn(L)), *wx = zalloc(padn(L)), *wy = zalloc(padn(L));
    double *tx = zalloc(padn(L)), *ty = zalloc(padn(L));
    in_vx(L, bx, pbx); in_vy(L, by, pby);
    in_velocity(S, L, vx, vy, wx, wy);
    residual_v(L, wx, wy, pbx, pby, tx, ty);
    out_vx(L, tx, rx); out_vy(L, ty, ry);
    free(pbx); free(pby); free(wx); free(wy); free(tx); free(ty);
    return O_OK;
}
/* restriction level l -> l+1 of a field of type t (0 vx, 1 vy, 2 P, 3 basic) */
int oracle_restrict(oracle_t *S, int l, int t, const double *fine, double *coarse) {
    if (!S || l < 0 || l + 1 >= S->nlev || t < 0 || t > 3) return O_EINVAL;
    olevel *F = &S->lev[l], *C = &S->lev[l + 1];
    double *a = zalloc(padn(F)), *b = zalloc(padn(C));
    switch (t) {
    case T_VX: in_vx(F, fine, a); restrict_generic(F, C, t, a, b, 1, C->ncy, 1, C->ncx - 1); out_vx(C, b, coarse); break;
    case T_VY: in_vy(F, fine, a); restrict_generic(F, C, t, a, b, 1, C->ncy - 1, 1, C->ncx); out_vy(C, b, coarse); break;
    case T_P: in_p(F, fine, a); restrict_generic(F, C, t, a, b, 1, C->ncy, 1, C->ncx); out_p(C, b, coarse); break;
    default: in_b(F, fine, a); restrict_generic(F, C, t, a, b, 0, C->ncy, 0, C->ncx); out_b(C, b, coarse); break;
    }
    free(a); free(b);
    return O_OK;
}
/* prolongation + correction: (vx,vy) at level l += P (ex,ey) from level l+1; mirrors refreshed */
int oracle_prolong(oracle_t *S, int l, const double *ex, const double *ey, double *vx, double *vy) {
    if (!S || l < 0 || l + 1 >= S->nlev) return O_EINVAL;
    olevel *F = &S->lev[l], *C = &S->lev[l + 1];
    double *cx = zalloc(padn(C)), *cy = zalloc(padn(C)), *wx = zalloc(padn(F)), *wy = zalloc(padn(F));
    in_velocity(S, C, ex, ey, cx, cy);
    in_velocity(S, F, vx, vy, wx, wy);
    prolong_add(F, C, T_VX, cx, wx);
    prolong_add(F, C, T_VY, cy, wy);
    refresh_mirrors(S, F, wx, wy);
    out_vx(F, wx, vx); out_vy(F, wy, vy);
    free(cx); free(cy); free(wx); free(wy);
    return O_OK;
}
/* exact coarsest-level solve L_c v = b */
int oracle_coarse_solve(oracle_t *S, const double *bx, const double *by, double *vx, double *vy) {
    if (!S || !S->have_eta || !S->o.coarse_direct) return O_ESTATE;
    olevel *L = &S->lev[S->nlev - 1];
    double *pbx = zalloc(padn(L)), *pby = zalloc(padn(L)), *wx = zalloc(padn(L)), *wy = zalloc(padn(L));
    in_vx(L, bx, pbx); in_vy(L, by, pby);
    coarse_direct_solve(S, L, wx, wy, pbx, pby);
    out_vx(L, wx, vx); out_vy(L, wy, vy);
    free(pbx); free(pby); free(wx); free(wy);
    return O_OK;
}

/* ------------------------------------------------ solve (a10-a12) */
static int solve_uzawa(oracle_t *S, double rtol, double Sf, double E0, int *iters, double *E_out,
                       double *hist, int hist_len) {
    olevel *L = &S->lev[0];
    size_t n = padn(L);
    double *bx = zalloc(n), *by = zalloc(n), *rx = zalloc(n), *ry = zalloc(n), *rp = zalloc(n);
    int status = O_NOT_CONVERGED, k;
    double E = E0;
    for (k = 1; k <= S->o.max_iter; ++k) {
        /* velocity subproblem L v = f - G p^k, 1 V-cycle warm-started (R15) */
        FOR_VX(L) bx[IX(L, i, j)] = S->fx[IX(L, i, j)] - Gx_point(L, S->p, i, j);
        FOR_VY(L) by[IX(L, i, j)] = S->fy[IX(L, i, j)] - Gy_point(L, S->p, i, j);
        S->ras_k = k - 1; S->ras_c = 0;  /* RAS shift counter: iteration index (R27) */
        for (int c = 0; c < S->o.vcycles_per_iter; ++c) vcycle_level(S, 0, S->vx, S->vy, bx, by);
        /* pressure update, reading R3: p += alpha eta_P r_p, r_p = -D v^{k+1} */
        FOR_P(L) {
            double r = -D_point(L, S->vx, S->vy, i, j);
            S->p[IX(L, i, j)] += S->o.pressure_sign * S->o.alpha_p * L->etap[IX(L, i, j)] * r;
        }
        /* nullspace: subtract the arithmetic mean */
        double m = p_mean(L, S->p);
        FOR_P(L) S->p[IX(L, i, j)] -= m;
        /* energy residual of the new (v, p) (reading R17) */
        full_residual(S, S->vx, S->vy, S->p, rx, ry, rp);
        E = energy_of(S, rx, ry, rp, Sf);
        if (hist && k - 1 < hist_len) hist[k - 1] = E;
        if (!(E == E) || isinf(E) || E > 1e6 * E0) { status = O_EDIVERGED; break; }
        if (E <= rtol) { status = O_OK; break; }
    }
    if (k > S->o.max_iter) k = S->o.max_iter;
    *iters = k;
    *E_out = E;
    free(bx); free(by); free(rx); free(ry); free(rp);
    return status;
}

/* Flexible GCR(m) with MGS, Alg. 4, readings R13/R14.
 * The iteration is written once (gcr_core) over an abstract vector space: the Stokes solve
 * plugs in x = (vx, vy, p) on the unknowns with <.,.> Euclidean over unknowns (vx, vy, p)
 * and M^-1 = the Uzawa-splitting preconditioner; oracle_gcr_dense plugs in a dense n x n
 * system so that the same code is pinned against a numpy Alg. 4 on small dense systems.
 * Restart (option gcr_true_restart): 1 (default, reading R13) replaces the recursive residual
 * by the true b - A x at every restart (over ~100 steps the recursive r drifts ~1e-9 from
 * the true one); 0 keeps the recursive r, literally Alg. 4.  Exit (reading R13):
 * when E(recursive r) <= rtol the TRUE residual is evaluated; the solve stops only if its E
 * is <= rtol too, otherwise it restarts from that true residual.  The E returned is always
 * the true one. */
typedef struct { double *x, *y, *p; } ovec;
typedef struct {
    void *ctx;
    void (*precond)(void *ctx, ovec r, ovec z);   /* z = M^-1 r */
    void (*apply)(void *ctx, ovec z, ovec w);     /* w = A z */
    double (*dot)(void *ctx, ovec a, ovec b);
    void (*axpy)(void *ctx, double a, ovec x, ovec y);  /* y += a x */
    void (*scale)(void *ctx, double a, ovec x);
    void (*residual)(void *ctx, ovec x, ovec r);  /* r = b - A x */
    double (*energy)(void *ctx, ovec r);          /* stopping-test measure of a residual */
    void (*step)(void *ctx, int k);               /* before preconditioner application k */
} gcr_ops;

static int gcr_core(const gcr_ops *op, ovec x, ovec r, ovec *z, ovec *w, int m, int max_iter, int true_restart,
                    double rtol, double E0, int *iters, double *E_out, double *hist, int hist_len) {
    void *c = op->ctx;
    op->residual(c, x, r);  /* r0 = b - A x0 */
    int k = 0, status = O_NOT_CONVERGED, fresh = 1;
    double E = E0;
    while (k < max_iter && status == O_NOT_CONVERGED) {
        if (!fresh && true_restart) op->residual(c, x, r);  /* restart from the true residual (R13) */
        fresh = 0;
        for (int i = 0; i < m && k < max_iter; ++i) {
            op->step(c, k);
            op->precond(c, r, z[i]);          /* z_i = M^-1 r      (Alg. 4 line 5) */
            op->apply(c, z[i], w[i]);         /* w_i = A z_i       (line 6) */
            for (int j = 0; j < i; ++j) {     /* modified Gram-Schmidt (lines 7-10) */
                double g = op->dot(c, w[i], w[j]);
                op->axpy(c, -g, w[j], w[i]);
                op->axpy(c, -g, z[j], z[i]);
            }
            double nu = sqrt(op->dot(c, w[i], w[i]));
            double rn = sqrt(op->dot(c, r, r));
            ++k;
            if (!(nu > 1e-14 * rn)) { status = O_EDIVERGED; break; } /* breakdown (R13) */
            op->scale(c, 1.0 / nu, w[i]);     /* lines 11-12 */
            op->scale(c, 1.0 / nu, z[i]);
            double beta = op->dot(c, r, w[i]);  /* line 13 */
            op->axpy(c, beta, z[i], x);       /* line 14 */
            op->axpy(c, -beta, w[i], r);      /* line 15 */
            E = op->energy(c, r);
            if (hist && k - 1 < hist_len) hist[k - 1] = E;
            if (!(E == E) || isinf(E) || E > 1e6 * E0) { status = O_EDIVERGED; break; }
            if (E <= rtol) {                  /* exit test on the true residual (R13) */
                op->residual(c, x, r);
                fresh = 1;
                if (op->energy(c, r) <= rtol) status = O_OK;
                break;                        /* else: restart from that true residual */
            }
        }
    }
    op->residual(c, x, r);  /* the E reported is the true one */
    *E_out = op->energy(c, r);
    *iters = k;
    return status;
}

static ovec ovec_new(size_t n) { ovec v = {zalloc(n), zalloc(n), zalloc(n)}; return v; }
static void ovec_free(ovec v) { free(v.x); free(v.y); free(v.p); }
static double ovec_dot(const olevel *L, ovec a, ovec b) {
    size_t n = (size_t)nunk(L) + (size_t)L->ncx * L->ncy, k = 0;
    double *t = zalloc(n);
    FOR_VX(L) t[k++] = a.x[IX(L, i, j)] * b.x[IX(L, i, j)];
    FOR_VY(L) t[k++] = a.y[IX(L, i, j)] * b.y[IX(L, i, j)];
    FOR_P(L) t[k++] = a.p[IX(L, i, j)] * b.p[IX(L, i, j)];
    double s = pairwise(t, n);
    free(t);
    return s;
}
static void ovec_axpy(const olevel *L, double a, ovec x, ovec y) { /* y += a x */
    FOR_VX(L) y.x[IX(L, i, j)] += a * x.x[IX(L, i, j)];
    FOR_VY(L) y.y[IX(L, i, j)] += a * x.y[IX(L, i, j)];
    FOR_P(L) y.p[IX(L, i, j)] += a * x.p[IX(L, i, j)];
}
static void ovec_scale(const olevel *L, double a, ovec x) {
    FOR_VX(L) x.x[IX(L, i, j)] *= a;
    FOR_VY(L) x.y[IX(L, i, j)] *= a;
    FOR_P(L) x.p[IX(L, i, j)] *= a;
}
/* z = M^-1 r: dv = Vcycle(0; r_v), dp = alpha eta_P (r_p - D dv), de-mean dp (R3, R14) */
static void apply_precond(oracle_t *S, ovec r, ovec z) {
    olevel *L = &S->lev[0];
    size_t n = padn(L);
    memset(z.x, 0, n * sizeof(double)); memset(z.y, 0, n * sizeof(double)); memset(z.p, 0, n * sizeof(double));
    for (int c = 0; c < S->o.vcycles_per_iter; ++c) vcycle_level(S, 0, z.x, z.y, r.x, r.y);
    FOR_P(L) z.p[IX(L, i, j)] = S->o.alpha_p * L->etap[IX(L, i, j)] * (r.p[IX(L, i, j)] - D_point(L, z.x, z.y, i, j));
    double m = p_mean(L, z.p);
    FOR_P(L) z.p[IX(L, i, j)] -= m;
}
/* w = A z = [L z_v + G z_p; D z_v] */
static void apply_A(oracle_t *S, ovec z, ovec w) {
    olevel *L = &S->lev[0];
    size_t n = padn(L);
    refresh_mirrors(S, L, z.x, z.y);
    memset(w.x, 0, n * sizeof(double)); memset(w.y, 0, n * sizeof(double)); memset(w.p, 0, n * sizeof(double));
    FOR_VX(L) w.x[IX(L, i, j)] = Lx_point(L, z.x, z.y, i, j) + Gx_point(L, z.p, i, j);
    FOR_VY(L) w.y[IX(L, i, j)] = Ly_point(L, z.x, z.y, i, j) + Gy_point(L, z.p, i, j);
    FOR_P(L) w.p[IX(L, i, j)] = D_point(L, z.x, z.y, i, j);
}
/* the Stokes instance of gcr_ops */
typedef struct { oracle_t *S; double Sf; } stokes_gcr;
static void sg_precond(void *c, ovec r, ovec z) { apply_precond(((stokes_gcr *)c)->S, r, z); }
static void sg_apply(void *c, ovec z, ovec w) { apply_A(((stokes_gcr *)c)->S, z, w); }
/* energy-weighted inner product (option gcr_inner = 1, reading R33): the weights of the
 * stopping test E (sum_vel_energy / sum_p_energy), so GCR minimises E itself */
static double ovec_dot_energy(const oracle_t *S, ovec a, ovec b) {
    const olevel *L = &S->lev[0];
    size_t n = (size_t)nunk(L) + (size_t)L->ncx * L->ncy, k = 0;
    double *t = zalloc(n);
    const double c = 2.0 / (L->dx * L->dx) + 2.0 / (L->dy * L->dy);
    FOR_VX(L) t[k++] = a.x[IX(L, i, j)] * b.x[IX(L, i, j)] / (-Lx_diag(S, L, i, j));
    FOR_VY(L) t[k++] = a.y[IX(L, i, j)] * b.y[IX(L, i, j)] / (-Ly_diag(S, L, i, j));
    FOR_P(L) t[k++] = a.p[IX(L, i, j)] * b.p[IX(L, i, j)] * (L->etap[IX(L, i, j)] / c);
    double s = pairwise(t, n);
    free(t);
    return s;
}
static double sg_dot(void *c, ovec a, ovec b) {
    oracle_t *S = ((stokes_gcr *)c)->S;
    return S->o.gcr_inner ? ovec_dot_energy(S, a, b) : ovec_dot(&S->lev[0], a, b);
}
static void sg_axpy(void *c, double a, ovec x, ovec y) { ovec_axpy(&((stokes_gcr *)c)->S->lev[0], a, x, y); }
static void sg_scale(void *c, double a, ovec x) { ovec_scale(&((stokes_gcr *)c)->S->lev[0], a, x); }
static void sg_residual(void *c, ovec x, ovec r) {
    oracle_t *S = ((stokes_gcr *)c)->S;
    refresh_mirrors(S, &S->lev[0], x.x, x.y);
    full_residual(S, x.x, x.y, x.p, r.x, r.y, r.p);
}
static double sg_energy(void *c, ovec r) { return energy_of(((stokes_gcr *)c)->S, r.x, r.y, r.p, ((stokes_gcr *)c)->Sf); }
static void sg_step(void *c, int k) { ((stokes_gcr *)c)->S->ras_k = k; ((stokes_gcr *)c)->S->ras_c = 0; } /* R27 */

static int solve_gcr(oracle_t *S, double rtol, double Sf, double E0, int *iters, double *E_out, double *hist,
                     int hist_len) {
    olevel *L = &S->lev[0];
    size_t n = padn(L);
    int m = S->o.gcr_restart;
    ovec r = ovec_new(n), xv = {S->vx, S->vy, S->p};
    ovec *z = (ovec *)calloc(m, sizeof(ovec)), *w = (ovec *)calloc(m, sizeof(ovec));
    for (int k = 0; k < m; ++k) { z[k] = ovec_new(n); w[k] = ovec_new(n); }
    stokes_gcr ctx = {S, Sf};
    gcr_ops op = {&ctx, sg_precond, sg_apply, sg_dot, sg_axpy, sg_scale, sg_residual, sg_energy, sg_step};
    int status = gcr_core(&op, xv, r, z, w, m, S->o.max_iter, S->o.gcr_true_restart, rtol, E0, iters, E_out, hist,
                          hist_len);
    refresh_mirrors(S, L, S->vx, S->vy);
    for (int q = 0; q < m; ++q) { ovec_free(z[q]); ovec_free(w[q]); }
    free(z); free(w); ovec_free(r);
    return status;
}

/* the dense instance (pins only): A x = b with an explicit n x n preconditioner Minv,
 * <.,.> Euclidean (pairwise sums), E = ||r|| / ||b|| */
typedef struct { int n; const double *A, *Minv, *b; double nb; } dense_gcr;
static void dmatvec(int n, const double *M, const double *u, double *v) {
    double *t = zalloc(n);
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) t[j] = M[(size_t)i * n + j] * u[j];
        v[i] = pairwise(t, n);
    }
    free(t);
}
static void dg_precond(void *c, ovec r, ovec z) { dense_gcr *d = c; dmatvec(d->n, d->Minv, r.x, z.x); }
static void dg_apply(void *c, ovec z, ovec w) { dense_gcr *d = c; dmatvec(d->n, d->A, z.x, w.x); }
static double dg_dot(void *c, ovec a, ovec b) {
    dense_gcr *d = c;
    double *t = zalloc(d->n);
    for (int i = 0; i < d->n; ++i) t[i] = a.x[i] * b.x[i];
    double s = pairwise(t, d->n);
    free(t);
    return s;
}
static void dg_axpy(void *c, double a, ovec x, ovec y) { dense_gcr *d = c; for (int i = 0; i < d->n; ++i) y.x[i] += a * x.x[i]; }
static void dg_scale(void *c, double a, ovec x) { dense_gcr *d = c; for (int i = 0; i < d->n; ++i) x.x[i] *= a; }
static void dg_residual(void *c, ovec x, ovec r) {
    dense_gcr *d = c;
    dmatvec(d->n, d->A, x.x, r.x);
    for (int i = 0; i < d->n; ++i) r.x[i] = d->b[i] - r.x[i];
}
static double dg_energy(void *c, ovec r) { return sqrt(dg_dot(c, r, r)) / ((dense_gcr *)c)->nb; }
static void dg_step(void *c, int k) { (void)c; (void)k; }

/* GCR(m) of gcr_core on a dense system (test entry point: pins the Krylov code on small
 * dense systems).  x: in initial guess, out iterate.  W (nullable, n x m row-
 * major by vector): the normalised w_i of the last cycle, for the orthogonality pin. */
int oracle_gcr_dense(int n, const double *A, const double *Minv, const double *b, double *x, int m, int max_iter,
                     int true_restart, double rtol, int *iters, double *E, double *hist, int hist_len, double *W) {
    if (n < 1 || m < 1 || max_iter < 0 || !A || !Minv || !b || !x || !iters || !E) return O_EINVAL;
    dense_gcr ctx = {n, A, Minv, b, 0.0};
    ovec bb = {(double *)b, NULL, NULL};
    ctx.nb = sqrt(dg_dot(&ctx, bb, bb));
    if (!(ctx.nb > 0)) return O_EINVAL;
    gcr_ops op = {&ctx, dg_precond, dg_apply, dg_dot, dg_axpy, dg_scale, dg_residual, dg_energy, dg_step};
    ovec r = {zalloc(n), NULL, NULL}, xv = {x, NULL, NULL};
    ovec *z = (ovec *)calloc(m, sizeof(ovec)), *w = (ovec *)calloc(m, sizeof(ovec));
    for (int k = 0; k < m; ++k) { z[k].x = zalloc(n); w[k].x = zalloc(n); }
    op.residual(&ctx, xv, r);
    double E0 = dg_energy(&ctx, r);
    int st = gcr_core(&op, xv, r, z, w, m, max_iter, true_restart, rtol, E0, iters, E, hist, hist_len);
    if (W) for (int k = 0; k < m; ++k) memcpy(W + (size_t)k * n, w[k].x, (size_t)n * sizeof(double));
    for (int k = 0; k < m; ++k) { free(z[k].x); free(w[k].x); }
    free(z); free(w); free(r.x);
    return st;
}

/* solve(rtol): in = initial guess (v, p), out = solution; zero-mean p on exit.
 * iters = number of V-cycle applications ("preconditioner applications" in GCR mode).
 * hist (optional): E after every iteration. */
/* Anderson acceleration AA(m) with mixing beta, Alg. 5, reading R26.
 * G(x) = one Uzawa iteration (V-cycle on L v = f - G p, p += alpha eta_P r_p, de-mean),
 * x = (vx, vy, p).  x^1 = G(x^0); for k >= 1: m_k = min(m, k), R = [r^{k-m_k} .. r^k] with
 * r^i = G(x^i) - x^i, alpha = argmin ||R alpha||_2 subject to 1^T alpha = 1, solved as
 * (R^T R + lambda I) z = 1, alpha = z / 1^T z (lambda = 1e-10 max diag: rank-deficient
 * histories), x^{k+1} = (1 - beta) sum alpha_i x^i + beta sum alpha_i G(x^i), de-meaned.
 * <.,.> Euclidean over the unknowns (R13).  Stopping test on the energy residual of the
 * newest G(x^k) (computed by the Uzawa step), which is returned; iterations = G calls. */
static void aa_copy(const olevel *L, ovec d, const double *vx, const double *vy, const double *p) {
    size_t n = padn(L);
    memcpy(d.x, vx, n * sizeof(double));
    memcpy(d.y, vy, n * sizeof(double));
    memcpy(d.p, p, n * sizeof(double));
}
/* solve (H + lambda I) z = 1 by Gaussian elimination with partial pivoting; alpha = z / sum z */
static int aa_alpha(int n, const double *H, double *alpha) {
    double A[16][17];
    double dmax = 0.0;
    for (int i = 0; i < n; ++i) dmax = fmax(dmax, H[i * n + i]);
    double lam = 1e-10 * dmax;
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) A[i][j] = H[i * n + j] + (i == j ? lam : 0.0);
        A[i][n] = 1.0;
    }
    for (int c = 0; c < n; ++c) {
        int piv = c;
        for (int r = c + 1; r < n; ++r) if (fabs(A[r][c]) > fabs(A[piv][c])) piv = r;
        if (!(fabs(A[piv][c]) > 0.0)) return -1;
        if (piv != c) for (int j = 0; j <= n; ++j) { double t = A[c][j]; A[c][j] = A[piv][j]; A[piv][j] = t; }
        for (int r = c + 1; r < n; ++r) {
            double f = A[r][c] / A[c][c];
            for (int j = c; j <= n; ++j) A[r][j] -= f * A[c][j];
        }
    }
    double z[16], sz = 0.0;
    for (int i = n - 1; i >= 0; --i) {
        double t = A[i][n];
        for (int j = i + 1; j < n; ++j) t -= A[i][j] * z[j];
        z[i] = t / A[i][i];
    }
    for (int i = 0; i < n; ++i) sz += z[i];
    if (!(fabs(sz) > 0.0)) return -1;
    for (int i = 0; i < n; ++i) alpha[i] = z[i] / sz;
    return 0;
}
/* test entry point: the Alg. 5 argmin of solve_anderson on a given Gram matrix H = R^T R */
int oracle_aa_alpha(int n, const double *H, double *alpha) {
    if (n < 1 || n > 16 || !H || !alpha) return O_EINVAL;
    return aa_alpha(n, H, alpha) == 0 ? O_OK : O_EINVAL;
}
static int solve_anderson(oracle_t *S, double rtol, double Sf, double E0, int *iters, double *E_out, double *hist,
                          int hist_len) {
    olevel *L = &S->lev[0];
    size_t n = padn(L);
    const int m = S->o.aa_depth, ns = m + 1;
    const double beta = S->o.aa_beta;
    ovec *X = (ovec *)calloc(ns, sizeof(ovec)), *GX = (ovec *)calloc(ns, sizeof(ovec));
    ovec *R = (ovec *)calloc(ns, sizeof(ovec));
    for (int i = 0; i < ns; ++i) { X[i] = ovec_new(n); GX[i] = ovec_new(n); R[i] = ovec_new(n); }
    double *bx = zalloc(n), *by = zalloc(n), *rx = zalloc(n), *ry = zalloc(n), *rp = zalloc(n);
    double H[16 * 16], alpha[16];
    int status = O_NOT_CONVERGED, k;
    double E = E0;
    for (k = 0; k < S->o.max_iter; ++k) {
        const int slot = k % ns;
        aa_copy(L, X[slot], S->vx, S->vy, S->p);  /* x^k */
        /* G(x^k): one Uzawa iteration (as solve_uzawa) */
        FOR_VX(L) bx[IX(L, i, j)] = S->fx[IX(L, i, j)] - Gx_point(L, S->p, i, j);
        FOR_VY(L) by[IX(L, i, j)] = S->fy[IX(L, i, j)] - Gy_point(L, S->p, i, j);
        S->ras_k = k; S->ras_c = 0;  /* RAS shift counter: iteration index (R27) */
        for (int c = 0; c < S->o.vcycles_per_iter; ++c) vcycle_level(S, 0, S->vx, S->vy, bx, by);
        FOR_P(L) {
            double r = -D_point(L, S->vx, S->vy, i, j);
            S->p[IX(L, i, j)] += S->o.pressure_sign * S->o.alpha_p * L->etap[IX(L, i, j)] * r;
        }
        double pm = p_mean(L, S->p);
        FOR_P(L) S->p[IX(L, i, j)] -= pm;
        full_residual(S, S->vx, S->vy, S->p, rx, ry, rp);
        E = energy_of(S, rx, ry, rp, Sf);
        if (hist && k < hist_len) hist[k] = E;
        if (!(E == E) || isinf(E) || E > 1e6 * E0) { status = O_EDIVERGED; break; }
        if (E <= rtol) { status = O_OK; break; }
        aa_copy(L, GX[slot], S->vx, S->vy, S->p);  /* G(x^k) */
        FOR_VX(L) R[slot].x[IX(L, i, j)] = GX[slot].x[IX(L, i, j)] - X[slot].x[IX(L, i, j)];
        FOR_VY(L) R[slot].y[IX(L, i, j)] = GX[slot].y[IX(L, i, j)] - X[slot].y[IX(L, i, j)];
        FOR_P(L) R[slot].p[IX(L, i, j)] = GX[slot].p[IX(L, i, j)] - X[slot].p[IX(L, i, j)];
        if (k == 0) continue;  /* x^1 = G(x^0): the working fields already hold it */
        const int mk = k < m ? k : m, nn = mk + 1;
        for (int a = 0; a < nn; ++a)
            for (int b = 0; b < nn; ++b) {
                const int sa = (k - mk + a) % ns, sb = (k - mk + b) % ns;
                H[a * nn + b] = ovec_dot(L, R[sa], R[sb]);
            }
        if (aa_alpha(nn, H, alpha) != 0) continue;  /* degenerate history: plain step */
        /* x^{k+1} = (1 - beta) sum alpha_i x^i + beta sum alpha_i G(x^i) (unknowns; mirrors refreshed) */
        FOR_VX(L) {
            double sx = 0.0, sg = 0.0;
            for (int a = 0; a < nn; ++a) {
                const int sa = (k - mk + a) % ns;
                sx += alpha[a] * X[sa].x[IX(L, i, j)];
                sg += alpha[a] * GX[sa].x[IX(L, i, j)];
            }
            S->vx[IX(L, i, j)] = (1.0 - beta) * sx + beta * sg;
        }
        FOR_VY(L) {
            double sx = 0.0, sg = 0.0;
            for (int a = 0; a < nn; ++a) {
                const int sa = (k - mk + a) % ns;
                sx += alpha[a] * X[sa].y[IX(L, i, j)];
                sg += alpha[a] * GX[sa].y[IX(L, i, j)];
            }
            S->vy[IX(L, i, j)] = (1.0 - beta) * sx + beta * sg;
        }
        FOR_P(L) {
            double sx = 0.0, sg = 0.0;
            for (int a = 0; a < nn; ++a) {
                const int sa = (k - mk + a) % ns;
                sx += alpha[a] * X[sa].p[IX(L, i, j)];
                sg += alpha[a] * GX[sa].p[IX(L, i, j)];
            }
            S->p[IX(L, i, j)] = (1.0 - beta) * sx + beta * sg;
        }
        refresh_mirrors(S, L, S->vx, S->vy);
        pm = p_mean(L, S->p);
        FOR_P(L) S->p[IX(L, i, j)] -= pm;
    }
    if (k >= S->o.max_iter) k = S->o.max_iter - 1;
    *iters = k + 1;
    *E_out = E;
    for (int i = 0; i < ns; ++i) { ovec_free(X[i]); ovec_free(GX[i]); ovec_free(R[i]); }
    free(X); free(GX); free(R); free(bx); free(by); free(rx); free(ry); free(rp);
    return status;
}

int oracle_solve_hist(oracle_t *S, double rtol, double *vx, double *vy, double *p, int *iters, double *rel_energy,
                      double *hist, int hist_len) {
    if (!S || !iters || !rel_energy) return O_EINVAL;
    if (!S->have_eta || !S->have_rho) return O_ESTATE;
    olevel *L = &S->lev[0];
    size_t n = padn(L);
    in_velocity(S, L, vx, vy, S->vx, S->vy);
    memset(S->p, 0, n * sizeof(double));
    in_p(L, p, S->p);
    double Sf = force_energy(S);
    if (!(Sf > 0)) { /* f == 0: zero solution, 0 iterations */
        for (size_t k = 0; k < (size_t)S->ny * (S->nx + 1); ++k) vx[k] = 0.0;
        for (size_t k = 0; k < (size_t)(S->ny + 1) * S->nx; ++k) vy[k] = 0.0;
        for (size_t k = 0; k < (size_t)S->ny * S->nx; ++k) p[k] = 0.0;
        *iters = 0; *rel_energy = 0.0;
        return O_OK;
    }
    double *rx = zalloc(n), *ry = zalloc(n), *rp = zalloc(n);
    full_residual(S, S->vx, S->vy, S->p, rx, ry, rp);
    double E0 = energy_of(S, rx, ry, rp, Sf);
    free(rx); free(ry); free(rp);
    int status;
    if (E0 <= rtol) { *iters = 0; *rel_energy = E0; status = O_OK; }
    else if (S->o.theta_step > 0.0) {
        /* viscosity rescaling: stages theta = 0, step, 2 step, .. < 1 of
         * theta_every iterations each (no stopping test: the staged systems are not the
         * problem), warm-started from the previous stage; then theta = 1 (the caller's
         * viscosity) to E <= rtol with the remaining iteration budget. */
        const int budget = S->o.max_iter;
        int used = 0, it = 0;
        double E = E0;
        status = O_OK;
        for (int k = 0;; ++k) {
            double theta = k * S->o.theta_step;
            if (theta >= 1.0 || used >= budget) break;
            oracle_blend_viscosity(S, theta);
            double Sfk = force_energy(S);
            rx = zalloc(n); ry = zalloc(n); rp = zalloc(n);
            full_residual(S, S->vx, S->vy, S->p, rx, ry, rp);
            double E0k = energy_of(S, rx, ry, rp, Sfk);
            free(rx); free(ry); free(rp);
            S->o.max_iter = budget - used < S->o.theta_every ? budget - used : S->o.theta_every;
            int hoff = used < hist_len ? used : hist_len;
            status = S->o.accel == 1   ? solve_gcr(S, -1.0, Sfk, E0k, &it, &E, hist ? hist + hoff : NULL, hist_len - hoff)
                     : S->o.accel == 2 ? solve_anderson(S, -1.0, Sfk, E0k, &it, &E, hist ? hist + hoff : NULL,
                                                        hist_len - hoff)
                                       : solve_uzawa(S, -1.0, Sfk, E0k, &it, &E, hist ? hist + hoff : NULL, hist_len - hoff);
            S->o.max_iter = budget;
            used += it;
            if (status == O_EDIVERGED) break;
        }
        oracle_blend_viscosity(S, 1.0);
        Sf = force_energy(S);
        if (status != O_EDIVERGED && used < budget) {
            rx = zalloc(n); ry = zalloc(n); rp = zalloc(n);
            full_residual(S, S->vx, S->vy, S->p, rx, ry, rp);
            double E1 = energy_of(S, rx, ry, rp, Sf);
            free(rx); free(ry); free(rp);
            if (E1 <= rtol) { it = 0; E = E1; status = O_OK; }
            else {
                S->o.max_iter = budget - used;
                int hoff = used < hist_len ? used : hist_len;
                status = S->o.accel == 1   ? solve_gcr(S, rtol, Sf, E1, &it, &E, hist ? hist + hoff : NULL, hist_len - hoff)
                         : S->o.accel == 2 ? solve_anderson(S, rtol, Sf, E1, &it, &E, hist ? hist + hoff : NULL,
                                                            hist_len - hoff)
                                           : solve_uzawa(S, rtol, Sf, E1, &it, &E, hist ? hist + hoff : NULL, hist_len - hoff);
                S->o.max_iter = budget;
            }
            used += it;
        } else if (status != O_EDIVERGED) {
            status = O_NOT_CONVERGED;
        }
        *iters = used;
        *rel_energy = E;
    }
    else if (S->o.accel == 1) status = solve_gcr(S, rtol, Sf, E0, iters, rel_energy, hist, hist_len);
    else if (S->o.accel == 2) status = solve_anderson(S, rtol, Sf, E0, iters, rel_energy, hist, hist_len);
    else status = solve_uzawa(S, rtol, Sf, E0, iters, rel_energy, hist, hist_len);
    double m = p_mean(L, S->p);
    FOR_P(L) S->p[IX(L, i, j)] -= m;
    out_vx(L, S->vx, vx); out_vy(L, S->vy, vy); out_p(L, S->p, p);
    return status;
}
int oracle_solve(oracle_t *S, double rtol, double *vx, double *vy, double *p, int *iters, double *rel_energy) {
    return oracle_solve_hist(S, rtol, vx, vy, p, iters, rel_energy, NULL, 0);
}

const char *oracle_strerror(int e) {
    switch (e) {
    case O_OK: return "ok";
    case O_NOT_CONVERGED: return "max_iter reached";
    case O_EINVAL: return "invalid argument";
    case O_ENOMEM: return "out of memory";
    case O_EDIVERGED: return "diverged";
    case O_ESTATE: return "call order (set_viscosity/set_density first)";
    default: return "unknown";
    }
}
