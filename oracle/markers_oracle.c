/*
 * oracle/markers_oracle.c -- CPU ORACLE of the marker-in-cell transfers and marker
 * advection.  TEST INFRASTRUCTURE ONLY: loaded by tests/ and
 * bench tooling through oracle/oracle.py; the product path never links it, and this file
 * includes no header from the product tree.
 *
 * Plain single-threaded FP64 loops in the paper's order (gcc -O2 -ffp-contract=off):
 *   - marker -> grid (§4.2 "Marker-to-grid interpolation", steps 1-5):
 *     for every marker IN INDEX ORDER find the reference node at the top-left corner of the
 *     surrounding cell of the target grid, compute r_x, r_y, the four bilinear weights of
 *     PAPER.md:480-484 and accumulate w*phi and w into temporaries; then divide
 *     (PAPER.md:488-491).  Targets: basic nodes (eta_b, rho_b) and pressure nodes (eta_p).
 *   - grid -> marker: phi_m = sum of the four weighted node values.
 *   - advection: forward Euler (Eq. euler_advection), Heun
 *     (Eq. heun_method), classical RK4 (Eq. rk4_method, combination in the order of
 *     Listing rk4_agnostic) and the locally polynomial integrator of
 *     order 2 / 3 (Eq. lpi_update, J and H of the bilinear interpolant: reading R32),
 *     velocity frozen during the step.
 *   - time step: CFL-like limit (formula of SPEC.md:151-154).
 * Readings: R28 stagger offsets, reference-node clamping and empty nodes;
 * R29 velocity mirrors in grid->marker; R30 closed-box clamping of stage and final
 * positions (the paper's listing wraps periodically, our box has walls); R31 time step.
 *
 * Layouts are the C-ABI user layouts (include/stokes.h): eta_b, rho_b (ny+1)x(nx+1) at
 * (j dx, i dy); eta_p ny x nx at ((j+1/2)dx, (i+1/2)dy); vx ny x (nx+1) at
 * (j dx, (i+1/2)dy) with wall columns 0, nx; vy (ny+1) x nx at ((j+1/2)dx, i dy) with
 * wall rows 0, ny.  y points down.  Marker arrays are length-n FP64 vectors.
 *
 * Pins: tests/test_oracle_markers.py (brute force with the hat-function definition of the
 * weights over every node, single marker on a node, constants, exact reproduction of
 * linear fields, the closed-form stability polynomials of Euler/Heun/RK4 on a linear
 * field, mirror images at the walls, the time-step formula).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define M_EINVAL (-1)
#define M_ENOMEM (-2)

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }
static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* Reference node of a grid whose node k sits at k*h + o (R28): k = floor((x - o)/h),
 * clamped to [kmin, kmax]; returns k and the normalised offset t = (x - (k h + o))/h. */
static int ref_node(double x, double h, double o, int kmin, int kmax, double *t) {
    int k = clampi((int)floor((x - o) / h), kmin, kmax);
    double xn = (double)k * h + o;
    *t = (x - xn) / h;
    return k;
}

/* ---------------------------------------------------------- marker -> grid (R28) */
int oracle_markers_to_grid(int nx, int ny, double Lx, double Ly, long long n, const double *xm,
                           const double *ym, const double *eta_m, const double *rho_m, double *eta_b,
                           double *eta_p, double *rho_b, long long *n_empty) {
    if (nx < 2 || ny < 2 || !(Lx > 0) || !(Ly > 0) || n < 0) return M_EINVAL;
    if (n > 0 && (!xm || !ym || !eta_m || !rho_m)) return M_EINVAL;
    double dx = Lx / nx, dy = Ly / ny;
    size_t nb = (size_t)(ny + 1) * (nx + 1), np = (size_t)ny * nx;
    double *swb = calloc(nb, sizeof(double)), *seb = calloc(nb, sizeof(double)),
           *srb = calloc(nb, sizeof(double)), *swp = calloc(np, sizeof(double)),
           *sep = calloc(np, sizeof(double));
    if (!swb || !seb || !srb || !swp || !sep) {
        free(swb); free(seb); free(srb); free(swp); free(sep);
        return M_ENOMEM;
    }
    for (long long m = 0; m < n; m++) {
        double x = clampd(xm[m], 0.0, Lx), y = clampd(ym[m], 0.0, Ly); /* R28/R30 */
        double tx, ty;
        /* basic nodes at (j dx, i dy): reference cell j in [0, nx-1], i in [0, ny-1] */
        int jr = ref_node(x, dx, 0.0, 0, nx - 1, &tx);
        int ir = ref_node(y, dy, 0.0, 0, ny - 1, &ty);
        double w[4] = {(1.0 - tx) * (1.0 - ty), tx * (1.0 - ty), (1.0 - tx) * ty, tx * ty};
        int ii[4] = {ir, ir, ir + 1, ir + 1}, jj[4] = {jr, jr + 1, jr, jr + 1};
        for (int k = 0; k < 4; k++) {
            size_t q = (size_t)ii[k] * (nx + 1) + jj[k];
            swb[q] += w[k];
            seb[q] += w[k] * eta_m[m];
            srb[q] += w[k] * rho_m[m];
        }
        /* pressure nodes at ((j+1/2) dx, (i+1/2) dy); reference node j in [-1, nx-1]
         * (j = -1 and j = nx are ghost nodes outside the domain: their sums are dropped) */
        jr = ref_node(x, dx, 0.5 * dx, -1, nx - 1, &tx);
        ir = ref_node(y, dy, 0.5 * dy, -1, ny - 1, &ty);
        double wp[4] = {(1.0 - tx) * (1.0 - ty), tx * (1.0 - ty), (1.0 - tx) * ty, tx * ty};
        int pi[4] = {ir, ir, ir + 1, ir + 1}, pj[4] = {jr, jr + 1, jr, jr + 1};
        for (int k = 0; k < 4; k++) {
            if (pi[k] < 0 || pi[k] >= ny || pj[k] < 0 || pj[k] >= nx) continue;
            size_t q = (size_t)pi[k] * nx + pj[k];
            swp[q] += wp[k];
            sep[q] += wp[k] * eta_m[m];
        }
    }
    long long empty = 0;
    for (size_t q = 0; q < nb; q++) { /* weighted average */
        if (swb[q] == 0.0) {
            empty++;
            if (eta_b) eta_b[q] = 0.0;
            if (rho_b) rho_b[q] = 0.0;
        } else {
            if (eta_b) eta_b[q] = seb[q] / swb[q];
            if (rho_b) rho_b[q] = srb[q] / swb[q];
        }
    }
    for (size_t q = 0; q < np; q++) {
        if (swp[q] == 0.0) {
            empty++;
            if (eta_p) eta_p[q] = 0.0;
        } else if (eta_p) {
            eta_p[q] = sep[q] / swp[q];
        }
    }
    if (n_empty) *n_empty = empty;
    free(swb); free(seb); free(srb); free(swp); free(sep);
    return 0;
}

/* ---------------------------------------------------------- grid -> marker (R29) */
typedef struct {
    int nx, ny;
    double dx, dy;
    double sW, sE, sN, sS; /* mirror signs: free slip +1, no slip -1 */
    const double *vx, *vy;
} vgrid;

static double vx_node(const vgrid *G, int i, int j) { /* i in [-1, ny], j in [0, nx] */
    if (j <= 0 || j >= G->nx) return 0.0;                      /* walls */
    if (i < 0) return G->sN * G->vx[(size_t)0 * (G->nx + 1) + j]; /* top mirror */
    if (i >= G->ny) return G->sS * G->vx[(size_t)(G->ny - 1) * (G->nx + 1) + j];
    return G->vx[(size_t)i * (G->nx + 1) + j];
}
static double vy_node(const vgrid *G, int i, int j) { /* i in [0, ny], j in [-1, nx] */
    if (i <= 0 || i >= G->ny) return 0.0;
    if (j < 0) return G->sW * G->vy[(size_t)i * G->nx + 0];
    if (j >= G->nx) return G->sE * G->vy[(size_t)i * G->nx + (G->nx - 1)];
    return G->vy[(size_t)i * G->nx + j];
}

/* phi_m = sum_(4 nodes) w phi, the sum taken in the weight order of
 * PAPER.md:480-484 (w00, w01, w10, w11). */
static double interp4(double tx, double ty, double v00, double v01, double v10, double v11) {
    double w00 = (1.0 - tx) * (1.0 - ty), w01 = tx * (1.0 - ty), w10 = (1.0 - tx) * ty, w11 = tx * ty;
    return w00 * v00 + w01 * v01 + w10 * v10 + w11 * v11;
}

static void velocity_at(const vgrid *G, double Lx, double Ly, double x, double y, double *u, double *v) {
    x = clampd(x, 0.0, Lx);
    y = clampd(y, 0.0, Ly);
    double tx, ty;
    int jr = ref_node(x, G->dx, 0.0, 0, G->nx - 1, &tx);
    int ir = ref_node(y, G->dy, 0.5 * G->dy, -1, G->ny - 1, &ty);
    *u = interp4(tx, ty, vx_node(G, ir, jr), vx_node(G, ir, jr + 1), vx_node(G, ir + 1, jr),
                 vx_node(G, ir + 1, jr + 1));
    jr = ref_node(x, G->dx, 0.5 * G->dx, -1, G->nx - 1, &tx);
    ir = ref_node(y, G->dy, 0.0, 0, G->ny - 1, &ty);
    *v = interp4(tx, ty, vy_node(G, ir, jr), vy_node(G, ir, jr + 1), vy_node(G, ir + 1, jr),
                 vy_node(G, ir + 1, jr + 1));
}

/* LPI (reading R32): value, gradient and mixed second derivative of the
 * same bilinear interpolant at (tx, ty) of a cell with spacings (h1, h2):
 *   d/dx = ((1-ty)(v01-v00) + ty(v11-v10))/dx,  d/dy = ((1-tx)(v10-v00) + tx(v11-v01))/dy,
 *   d2/dxdy = (v11 - v10 - v01 + v00)/(dx dy)   (the pure second derivatives of a bilinear
 *   function vanish). */
static void jet4(double tx, double ty, double dx, double dy, double v00, double v01, double v10, double v11,
                 double *val, double *gx, double *gy, double *gxy) {
    *val = interp4(tx, ty, v00, v01, v10, v11);
    *gx = ((1.0 - ty) * (v01 - v00) + ty * (v11 - v10)) / dx;
    *gy = ((1.0 - tx) * (v10 - v00) + tx * (v11 - v01)) / dy;
    *gxy = (v11 - v10 - v01 + v00) / (dx * dy);
}

/* u, v and J = [[du/dx, du/dy], [dv/dx, dv/dy]], Hu = d2u/dxdy, Hv = d2v/dxdy at (x, y) */
static void velocity_jet(const vgrid *G, double Lx, double Ly, double x, double y, double *u, double *v, double *J,
                         double *Hu, double *Hv) {
    x = clampd(x, 0.0, Lx);
    y = clampd(y, 0.0, Ly);
    double tx, ty;
    int jr = ref_node(x, G->dx, 0.0, 0, G->nx - 1, &tx);
    int ir = ref_node(y, G->dy, 0.5 * G->dy, -1, G->ny - 1, &ty);
    jet4(tx, ty, G->dx, G->dy, vx_node(G, ir, jr), vx_node(G, ir, jr + 1), vx_node(G, ir + 1, jr),
         vx_node(G, ir + 1, jr + 1), u, &J[0], &J[1], Hu);
    jr = ref_node(x, G->dx, 0.5 * G->dx, -1, G->nx - 1, &tx);
    ir = ref_node(y, G->dy, 0.0, 0, G->ny - 1, &ty);
    jet4(tx, ty, G->dx, G->dy, vy_node(G, ir, jr), vy_node(G, ir, jr + 1), vy_node(G, ir + 1, jr),
         vy_node(G, ir + 1, jr + 1), v, &J[2], &J[3], Hv);
}

static int make_vgrid(vgrid *G, int nx, int ny, double Lx, double Ly, const int *bc, const double *vx,
                      const double *vy) {
    if (nx < 2 || ny < 2 || !(Lx > 0) || !(Ly > 0) || !bc || !vx || !vy) return M_EINVAL;
    for (int s = 0; s < 4; s++)
        if (bc[s] != 0 && bc[s] != 1) return M_EINVAL;
    G->nx = nx; G->ny = ny; G->dx = Lx / nx; G->dy = Ly / ny;
    G->sW = bc[0] ? -1.0 : 1.0; G->sE = bc[1] ? -1.0 : 1.0;
    G->sN = bc[2] ? -1.0 : 1.0; G->sS = bc[3] ? -1.0 : 1.0;
    G->vx = vx; G->vy = vy;
    return 0;
}

int oracle_grid_to_markers(int nx, int ny, double Lx, double Ly, const int *bc, long long n,
                           const double *xm, const double *ym, const double *vx, const double *vy,
                           double *vxm, double *vym) {
    vgrid G;
    int st = make_vgrid(&G, nx, ny, Lx, Ly, bc, vx, vy);
    if (st) return st;
    for (long long m = 0; m < n; m++) velocity_at(&G, Lx, Ly, xm[m], ym[m], &vxm[m], &vym[m]);
    return 0;
}

/* ---------------------------------------------------------- advection (R30) */
int oracle_advect_markers(int nx, int ny, double Lx, double Ly, const int *bc, long long n, double *xm,
                          double *ym, const double *vx, const double *vy, double dt, int scheme,
                          long long *n_clamped) {
    vgrid G;
    int st = make_vgrid(&G, nx, ny, Lx, Ly, bc, vx, vy);
    if (st) return st;
    if (scheme < 0 || scheme > 4 || !isfinite(dt)) return M_EINVAL;
    long long clamped = 0;
    for (long long m = 0; m < n; m++) {
        double xA = xm[m], yA = ym[m], xn, yn;
        double u1, v1, u2, v2, u3, v3, u4, v4;
        if (scheme >= 3) { /* Eq. lpi_update: order 2 (scheme 3) or 3 (scheme 4), reading R32 */
            double J[4], Hu, Hv;
            velocity_jet(&G, Lx, Ly, xA, yA, &u1, &v1, J, &Hu, &Hv);
            double c2 = 0.5 * dt * dt, c3 = (1.0 / 6.0) * dt * dt * dt;
            double jx = J[0] * u1 + J[1] * v1, jy = J[2] * u1 + J[3] * v1; /* J v0 */
            xn = xA + dt * u1;
            yn = yA + dt * v1;
            xn = xn + c2 * jx;
            yn = yn + c2 * jy;
            if (scheme == 4) { /* (H : v0 v0)_i = 2 d2v_i/dxdy v0x v0y */
                xn = xn + c3 * (2.0 * Hu * u1 * v1);
                yn = yn + c3 * (2.0 * Hv * u1 * v1);
            }
            if (xn < 0.0 || xn > Lx || yn < 0.0 || yn > Ly) clamped++;
            xm[m] = clampd(xn, 0.0, Lx);
            ym[m] = clampd(yn, 0.0, Ly);
            continue;
        }
        velocity_at(&G, Lx, Ly, xA, yA, &u1, &v1);
        if (scheme == 0) { /* Eq. euler_advection */
            xn = xA + dt * u1;
            yn = yA + dt * v1;
        } else if (scheme == 1) { /* Eq. heun_method */
            double xs = clampd(xA + dt * u1, 0.0, Lx), ys = clampd(yA + dt * v1, 0.0, Ly);
            velocity_at(&G, Lx, Ly, xs, ys, &u2, &v2);
            xn = xA + 0.5 * dt * (u1 + u2);
            yn = yA + 0.5 * dt * (v1 + v2);
        } else { /* Eq. rk4_method, Listing rk4_agnostic */
            double xB = clampd(xA + 0.5 * dt * u1, 0.0, Lx), yB = clampd(yA + 0.5 * dt * v1, 0.0, Ly);
            velocity_at(&G, Lx, Ly, xB, yB, &u2, &v2);
            double xC = clampd(xA + 0.5 * dt * u2, 0.0, Lx), yC = clampd(yA + 0.5 * dt * v2, 0.0, Ly);
            velocity_at(&G, Lx, Ly, xC, yC, &u3, &v3);
            double xD = clampd(xA + dt * u3, 0.0, Lx), yD = clampd(yA + dt * v3, 0.0, Ly);
            velocity_at(&G, Lx, Ly, xD, yD, &u4, &v4);
            double ue = (1.0 / 6.0) * (u1 + 2.0 * u2 + 2.0 * u3 + u4);
            double ve = (1.0 / 6.0) * (v1 + 2.0 * v2 + 2.0 * v3 + v4);
            xn = xA + dt * ue;
            yn = yA + dt * ve;
        }
        if (xn < 0.0 || xn > Lx || yn < 0.0 || yn > Ly) clamped++;
        xm[m] = clampd(xn, 0.0, Lx);
        ym[m] = clampd(yn, 0.0, Ly);
    }
    if (n_clamped) *n_clamped = clamped;
    return 0;
}

/* ---------------------------------------------------------- time step (R31) */
int oracle_marker_timestep(int nx, int ny, double Lx, double Ly, const double *vx, const double *vy,
                           double cfl, double max_dt, double *dt) {
    if (nx < 2 || ny < 2 || !(Lx > 0) || !(Ly > 0) || !vx || !vy || !dt) return M_EINVAL;
    if (!(cfl > 0) || !(max_dt > 0)) return M_EINVAL;
    double dx = Lx / nx, dy = Ly / ny, mx = 0.0, my = 0.0;
    for (int i = 0; i < ny; i++) /* unknowns only: wall columns 0, nx are ignored */
        for (int j = 1; j < nx; j++) mx = fmax(mx, fabs(vx[(size_t)i * (nx + 1) + j]));
    for (int i = 1; i < ny; i++)
        for (int j = 0; j < nx; j++) my = fmax(my, fabs(vy[(size_t)i * nx + j]));
    double d = max_dt;
    if (mx > 0.0) d = fmin(d, cfl * (dx / mx));
    if (my > 0.0) d = fmin(d, cfl * (dy / my));
    *dt = d;
    return 0;
}
