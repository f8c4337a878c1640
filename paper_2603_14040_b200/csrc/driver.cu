// Host runtime of libstokes_b200: handle, level hierarchy, workspace carving, V-cycle
// driver (a9), Uzawa loop (a10, a12), flexible GCR (a11), CUDA-graph capture, and the
// C ABI of include/stokes.h.  Every step of the numerical path runs in kernels.cu; this
// file only sequences launches on the handle's stream.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>

#include <nccl.h>

#include "handle.h"

bool first_on_device(unsigned long long *mask) {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long bit = 1ull << (d & 63);
    if (__atomic_load_n(mask, __ATOMIC_ACQUIRE) & bit) return false;
    return !(__atomic_fetch_or(mask, bit, __ATOMIC_ACQ_REL) & bit);
}

namespace sk {

thread_local std::string g_last_error;

int fail_cuda(cudaError_t e, const char *what) {
    char buf[256];
    snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
    g_last_error = buf;
    return STOKES_ECUDA;
}

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

GridL make_grid(int ncx, int ncy, double Lx, double Ly, const int bc[4]) {
    GridL g;
    g.ncx = ncx;
    g.ncy = ncy;
    // columns -1 .. ncx+2 inside the row (width-2 halos of decomposed tiles)
    g.P = (int)round_up((size_t)ncx + 3 + COL_OFF, 32);
    g.dx = Lx / ncx;
    g.dy = Ly / ncy;
    g.idx = 1.0 / g.dx;
    g.idy = 1.0 / g.dy;
    g.idx2 = 1.0 / (g.dx * g.dx);
    g.idy2 = 1.0 / (g.dy * g.dy);
    g.idxdy = 1.0 / (g.dx * g.dy);
    g.idx2x2 = 2.0 * g.idx2;
    g.idy2x2 = 2.0 * g.idy2;
    g.sW = bc[0] == STOKES_FREE_SLIP ? 1.0 : -1.0;
    g.sE = bc[1] == STOKES_FREE_SLIP ? 1.0 : -1.0;
    g.sN = bc[2] == STOKES_FREE_SLIP ? 1.0 : -1.0;
    g.sS = bc[3] == STOKES_FREE_SLIP ? 1.0 : -1.0;
    g.bN = g.bS = g.bW = g.bE = 1;  // single domain: every side is a global boundary
    g.nvxj = ncx - 1;
    g.nvyi = ncy - 1;
    g.par = 0;
    return g;
}
// rows 0 .. ncy+2 (+ 512 doubles of tail: row-segment bulk copies of the last CTA may run past
// the last row); the Carver places one more row (row -1) in front of every field.  Rows -1
// and ncy+2 are the second halo ring of decomposed tiles (width-2 halos).
size_t field_doubles(const GridL &g) { return (size_t)(g.ncy + 3) * (size_t)g.P + 512; }
int n_unknowns(const GridL &g) { return g.ncy * (g.ncx - 1) + (g.ncy - 1) * g.ncx; }

// hierarchy (reading R8): factor 2 while both even and min/2 >= coarse_min
int build_levels(int nx, int ny, double Lx, double Ly, const int bc[4], const stokes_opts &o, GridL *gs, int *nus) {
    int cx = nx, cy = ny, l = 0;
    for (;;) {
        gs[l] = make_grid(cx, cy, Lx, Ly, bc);
        nus[l] = (int)floor(o.nu1 * pow(o.nu_growth, (double)l) + 0.5);
        ++l;
        if (l >= MAXLEV) break;
        if ((cx % 2) || (cy % 2)) break;
        const int m = cx < cy ? cx : cy;
        if (m / 2 < o.coarse_min) break;
        cx /= 2;
        cy /= 2;
    }
    return l;
}

int check_opts(const stokes_opts &o) {
    if (o.smoother < 0 || o.smoother > 3) return STOKES_EINVAL;
    if (o.ras_tile < 2 || o.ras_tile > ras_max_tile() || o.ras_inner < 1) return STOKES_EINVAL;
    if (!(o.omega_v > 0) || !(o.alpha_p > 0) || o.nu1 < 0 || !(o.nu_growth > 0) || o.coarse_min < 2) return STOKES_EINVAL;
    if (o.coarse_direct != 0 && o.coarse_direct != 1) return STOKES_EINVAL;
    if (o.vcycles_per_iter < 1 || o.accel < 0 || o.accel > 2) return STOKES_EINVAL;
    if (o.aa_depth < 0 || o.aa_depth >= AA_MAXS || !(o.aa_beta > 0.0 && o.aa_beta <= 1.0)) return STOKES_EINVAL;
    if (o.gcr_restart < 1 || o.gcr_restart > MAXM || o.max_iter < 0) return STOKES_EINVAL;
    if (o.gcr_true_restart != 0 && o.gcr_true_restart != 1) return STOKES_EINVAL;
    if (o.pressure_sign != 1 && o.pressure_sign != -1) return STOKES_EINVAL;
    if (!(o.theta_step >= 0.0 && o.theta_step <= 1.0) || o.theta_every < 1) return STOKES_EINVAL;
    return STOKES_OK;
}

// lay out (or size) the workspace
size_t carve(stokes_s *h, Carver &cv) {
    for (int l = 0; l < h->nlev; ++l) {
        Level &L = h->lev[l];
        L.etab = cv.field(L.g);
        L.etap = cv.field(L.g);
        for (int k = 0; k < 2; ++k) {
            L.vx[k] = cv.field(L.g);
            L.vy[k] = cv.field(L.g);
        }
        L.bx = cv.field(L.g);
        L.by = cv.field(L.g);
        L.rx = cv.field(L.g);
        L.ry = cv.field(L.g);
    }
    const GridL &g0 = h->lev[0].g;
    h->pbuf[0] = cv.field(g0);
    h->pbuf[1] = cv.field(g0);
    h->rho = cv.field(g0);
    if (h->o.theta_step > 0.0) {
        h->etab_user = cv.field(g0);
        h->etap_user = cv.field(g0);
    } else {
        h->etab_user = h->etap_user = nullptr;
    }
    h->npart = (size_t)energy_blocks(g0) * 12 + 3 * 4096 + 64;
    if (h->o.accel == STOKES_ACCEL_ANDERSON) {  // k_aa_push: AA_MAXS partials per block
        const size_t na = (size_t)aa_blocks(g0) * AA_MAXS + 64;
        if (na > h->npart) h->npart = na;
    }
    h->partials = cv.take(h->npart);
    h->scal = cv.take(S_NSCAL);
    const GridL &gc = h->lev[h->nlev - 1].g;
    const int n = n_unknowns(gc);
    if (h->o.coarse_direct && n <= MAX_DIRECT) {
        h->nc = n;
        h->Minv = cv.take((size_t)n * n);
        h->Mwork = cv.take((size_t)n * 2 * n);
    } else {
        h->nc = 0;
        h->Minv = h->Mwork = nullptr;
    }
    h->dflag = (int *)cv.take(4);
    if (h->o.accel == STOKES_ACCEL_ANDERSON) {
        for (int i = 0; i <= h->o.aa_depth; ++i)
            for (int f = 0; f < 3; ++f) {
                h->aah.G[i].f[f] = cv.field(g0);
                h->aah.R[i].f[f] = cv.field(g0);
            }
        for (int f = 0; f < 3; ++f) h->aat.f[f] = cv.field(g0);
        h->aaH = cv.take(AA_MAXS * AA_MAXS);
        h->aacg = cv.take(AA_MAXS);
        h->aacr = cv.take(AA_MAXS);
    }
    if (h->o.accel == STOKES_ACCEL_GCR) {
        for (int i = 0; i < h->o.gcr_restart; ++i)
            for (int f = 0; f < 3; ++f) {
                h->gz[i][f] = cv.field(g0);
                h->gw[i][f] = cv.field(g0);
            }
        for (int f = 0; f < 3; ++f) h->gr[f] = cv.field(g0);
        h->gtmp[0] = cv.field(g0);
        h->gtmp[1] = cv.field(g0);
        for (int f = 0; f < 3; ++f) h->gew[f] = cv.field(g0);
    }
    return round_up(cv.off, 256);
}

LaunchCtx ctx(stokes_s *h) { return LaunchCtx{h->stream, &h->launches}; }

RhsArgs rhs_arrays(const double *bx, const double *by) {
    RhsArgs r;
    r.mode = RHS_ARRAYS;
    r.bx = bx;
    r.by = by;
    r.p = r.rho = nullptr;
    r.gx = r.gy = 0.0;
    return r;
}
RhsArgs rhs_fine(stokes_s *h) {
    RhsArgs r;
    r.mode = RHS_FINE;
    r.bx = r.by = nullptr;
    r.p = h->pbuf[h->pcur];
    r.rho = h->rho;
    r.gx = h->gx;
    r.gy = h->gy;
    return r;
}

// nsweeps of the smoother on level l for L v = b.  (cur) holds v; Jacobi ping-pongs
// between cur and the other buffer: on return cur points at the result.
// Pairs of sweeps run as one two-sweep pass (launch_jacobi2) where the level allows it, at
// most max_pairs of them (each pair saves one buffer swap: vcycle keeps its count even).
int level_smoother(const stokes_s *h, int l) {
    if (h->o.smoother == STOKES_SMOOTH_MIXED) return l == 0 ? STOKES_SMOOTH_JACOBI : STOKES_SMOOTH_RAS;
    return h->o.smoother;
}
bool uses_ras(const stokes_s *h) {
    return h->o.smoother == STOKES_SMOOTH_RAS || (h->o.smoother == STOKES_SMOOTH_MIXED && h->nlev > 1);
}
void ras_iteration_start(stokes_s *h) { h->ras_c = 0; }
void ras_reset(stokes_s *h) {  // iteration index 0: start of a solve / stand-alone V-cycle or smoothing
    h->ras_c = 0;
    if (uses_ras(h)) cudaMemsetAsync(h->scal + S_ITER, 0, sizeof(double), h->stream);
}
void ras_iteration_end(stokes_s *h) {
    if (uses_ras(h)) launch_iter_inc(ctx(h), h->scal + S_ITER);
}
int jacobi_pairs(stokes_s *h, int l, int n, bool zero_in) {
    if (level_smoother(h, l) != STOKES_SMOOTH_JACOBI || !jacobi2_ok(h->lev[l].g)) return 0;
    return (n - (zero_in ? 1 : 0)) / 2 > 0 ? (n - (zero_in ? 1 : 0)) / 2 : 0;
}
// Small single-domain levels (<= STOKES_TILE_CELLS cells, default 256^2; 0 = off) smooth all n
// sweeps of a pre- / post-smoothing in one launch (k_jacobi_tile): their per-sweep kernels are
// launch- and pipeline-latency bound.  Pre- and post-smoothing of a level decide alike (same n),
// so a V-cycle still swaps its buffers an even number of times.  Layered 4096^2 solve (CUDA
// events): off 549 ms, <= 128^2 541, <= 256^2 538, <= 512^2 541, <= 1024^2 571 ms (the 3.4x
// staging redundancy of an 8 x 32 tile loses to the streamed pairs from 512^2 up).
static long long tile_cells() {  // (read per call: tests force either path)
    const char *e = getenv("STOKES_TILE_CELLS");
    return e ? atoll(e) : 256LL * 256LL;
}
static bool post_fused_prolong() {  // STOKES_TILE_PROLONG=0: separate prolongation launch (diagnostics)
    const char *e = getenv("STOKES_TILE_PROLONG");
    return !(e && e[0] == '0');
}
static bool tile_level(stokes_s *h, int l) {
    const GridL &g = h->lev[l].g;
    return (long long)g.ncx * g.ncy <= tile_cells();
}
void smooth(stokes_s *h, int l, double *&cx, double *&cy, double *&ox, double *&oy, const RhsArgs &rhs, int n,
            bool zero_in, int max_pairs) {
    Level &L = h->lev[l];
    const LaunchCtx c = ctx(h);
    if (n <= 0) {
        if (zero_in) {
            cudaMemsetAsync(cx - COL_OFF, 0, field_doubles(L.g) * sizeof(double), h->stream);
            cudaMemsetAsync(cy - COL_OFF, 0, field_doubles(L.g) * sizeof(double), h->stream);
        }
        return;
    }
    const int lsm = level_smoother(h, l);
    if (lsm == STOKES_SMOOTH_RAS) {  // Alg. 3: N_outer = ceil(n / T_inner), made even
        if (zero_in) {
            cudaMemsetAsync(cx - COL_OFF, 0, field_doubles(L.g) * sizeof(double), h->stream);
            cudaMemsetAsync(cy - COL_OFF, 0, field_doubles(L.g) * sizeof(double), h->stream);
        }
        int nout = (n + h->o.ras_inner - 1) / h->o.ras_inner;
        nout += nout % 2;
        const bool fine = rhs.mode == RHS_FINE;
        for (int t = 0; t < nout; ++t) {
            RasArgs a;
            a.vx = cx;
            a.vy = cy;
            a.etap = L.etap;
            a.etab = L.etab;
            a.f4 = fine ? rhs.p : rhs.bx;
            a.f5 = fine ? rhs.rho : rhs.by;
            a.vxo = ox;
            a.vyo = oy;
            a.omega = h->o.omega_v;
            a.gx = fine ? rhs.gx : 0.0;
            a.gy = fine ? rhs.gy : 0.0;
            a.T = h->o.ras_tile;
            a.Tin = h->o.ras_inner;
            a.seed = h->o.ras_seed;
            launch_ras_outer(c, L.g, a, h->scal + S_ITER, h->ras_c++, fine);
            double *tt = cx; cx = ox; ox = tt;
            tt = cy; cy = oy; oy = tt;
        }
    } else if (lsm == STOKES_SMOOTH_JACOBI && tile_level(h, l) &&
               launch_jacobi_tile(c, L.g, L.etab, L.etap, cx, cy, ox, oy, rhs, h->o.omega_v, n, zero_in)) {
        double *t = cx; cx = ox; ox = t;  // all n sweeps in one launch: one buffer swap
        t = cy; cy = oy; oy = t;
    } else if (lsm == STOKES_SMOOTH_JACOBI) {
        int pairs = jacobi_pairs(h, l, n, zero_in);
        if (pairs > max_pairs) pairs = max_pairs;
        for (int s = 0; s < n;) {
            if (pairs > 0 && !(zero_in && s == 0)) {
                launch_jacobi2(c, L.g, L.etab, L.etap, cx, cy, ox, oy, rhs, h->o.omega_v);
                --pairs;
                s += 2;
            } else {
                launch_jacobi(c, L.g, L.etab, L.etap, cx, cy, ox, oy, rhs, h->o.omega_v, zero_in && s == 0);
                s += 1;
            }
            double *t = cx; cx = ox; ox = t;
            t = cy; cy = oy; oy = t;
        }
    } else {
        if (zero_in) {
            cudaMemsetAsync(cx - COL_OFF, 0, field_doubles(L.g) * sizeof(double), h->stream);
            cudaMemsetAsync(cy - COL_OFF, 0, field_doubles(L.g) * sizeof(double), h->stream);
        }
        if (jacobi2_ok(L.g)) {  // streamed two-pass sweeps, out of place (ping-pong like Jacobi)
            for (int s = 0; s < n; ++s) {
                launch_rbgs_stream(c, L.g, L.etab, L.etap, cx, cy, ox, oy, rhs, h->o.omega_v);
                double *t = cx; cx = ox; ox = t;
                t = cy; cy = oy; oy = t;
            }
        } else {
            for (int s = 0; s < n; ++s) launch_rbgs(c, L.g, L.etab, L.etap, cx, cy, rhs, h->o.omega_v);
        }
    }
}

// One V-cycle (Eq. multigrid_levels) on level l for L v = b, v in
// (ax, ay) with scratch (bx_, by_); the result is left in (ax, ay) (the sweep count per
// cycle, 2 nu, is even).  zero_in: the initial guess is 0 (coarse corrections).
// Coarse tail in one CTA (kernels.cu k_vtail): from level l down, when every remaining level
// is a small single-domain damped-Jacobi level and the coarsest is solved directly.
// STOKES_VTAIL=0 disables it; STOKES_VTAIL_CELLS sets the largest level (cells) it starts at.
static int vtail_cells() {
    static const int v = [] {
        const char *e = getenv("STOKES_VTAIL");
        if (e && e[0] == '0') return 0;
        const char *c = getenv("STOKES_VTAIL_CELLS");
        return c ? atoi(c) : 1024;
    }();
    return v;
}
static bool vtail_ok(stokes_s *h, int l) {
    if (!h->o.coarse_direct || h->nc <= 0 || h->nlev - l > TAIL_MAXL || h->nlev - l < 2) return false;
    const GridL &g0 = h->lev[l].g;
    if ((long long)g0.ncx * g0.ncy > vtail_cells()) return false;
    for (int k = l; k < h->nlev; ++k) {
        const GridL &g = h->lev[k].g;
        if (!(g.bN && g.bS && g.bW && g.bE) || jacobi2_ok(g)) return false;
        if (k < h->nlev - 1 && level_smoother(h, k) != STOKES_SMOOTH_JACOBI) return false;
    }
    return true;
}
// Cooperative coarse cycle (kernels.cu k_vtail<true>): the same stages on a grid of one
// CTA per SM with grid-wide barriers, from the first level of <= STOKES_COOP_CELLS cells
// down.  Off by default: measured slower (layered 4096^2 bench: 551 ms per solve with the
// per-level kernels, 578 / 580 / 605 ms with the cooperative cycle from 256^2 / 512^2 /
// 1024^2 -- ~13 grid-wide barriers per level at ~3 us each cost more than the launches
// they replace; parity-green, kept as an option).
static int coop_cells() {
    static const int v = [] {
        const char *c = getenv("STOKES_COOP_CELLS");
        return c ? atoi(c) : 0;
    }();
    return v;
}
static bool coop_ok(stokes_s *h, int l) {
    if (!h->o.coarse_direct || h->nc <= 0 || h->nlev - l > TAIL_MAXL || h->nlev - l < 2) return false;
    const GridL &g0 = h->lev[l].g;
    if ((long long)g0.ncx * g0.ncy > coop_cells() || (long long)g0.ncx * g0.ncy <= vtail_cells()) return false;
    for (int k = l; k < h->nlev; ++k) {
        const GridL &g = h->lev[k].g;
        if (!(g.bN && g.bS && g.bW && g.bE)) return false;
        if (k < h->nlev - 1 && level_smoother(h, k) != STOKES_SMOOTH_JACOBI) return false;
    }
    return true;
}
void vcycle(stokes_s *h, int l, double *ax, double *ay, double *sx, double *sy, const RhsArgs &rhs, bool zero_in,
            int done_pre, int leave_last, double **lx, double **ly) {
    Level &L = h->lev[l];
    const LaunchCtx c = ctx(h);
    const bool coop = zero_in && !done_pre && rhs.mode == RHS_ARRAYS && coop_ok(h, l);
    if (coop || (zero_in && !done_pre && rhs.mode == RHS_ARRAYS && vtail_ok(h, l))) {
        TailArgs a;
        a.nl = h->nlev - l;
        for (int k = 0; k < a.nl; ++k) {
            Level &T = h->lev[l + k];
            TailLevel &t = a.lev[k];
            t.g = T.g;
            t.etab = T.etab;
            t.etap = T.etap;
            t.bx = k == 0 ? const_cast<double *>(rhs.bx) : T.bx;
            t.by = k == 0 ? const_cast<double *>(rhs.by) : T.by;
            t.ax = k == 0 ? ax : T.vx[0];
            t.ay = k == 0 ? ay : T.vy[0];
            t.sx = k == 0 ? sx : T.vx[1];
            t.sy = k == 0 ? sy : T.vy[1];
            t.rx = T.rx;
            t.ry = T.ry;
            t.nu = T.nu;
        }
        if (coop) launch_vtail_coop(c, a, h->Minv, h->nc, h->o.omega_v);
        else launch_vtail(c, a, h->Minv, h->nc, h->o.omega_v);
        return;
    }
    double *cx = ax, *cy = ay, *ox = sx, *oy = sy;
    if (done_pre) {  // the first pre-smoothing sweep was done by a fused kernel into (sx, sy)
        cx = sx; cy = sy; ox = ax; oy = ay;
    }
    if (l == h->nlev - 1) {  // coarsest (a8)
        if (h->nc > 0) {
            const double *bx = rhs.bx, *by = rhs.by;
            if (rhs.mode != RHS_ARRAYS) {
                launch_make_rhs(c, L.g, rhs, L.bx, L.by);
                bx = L.bx;
                by = L.by;
            }
            launch_coarse_solve(c, L.g, h->Minv, bx, by, ax, ay);
        } else {
            smooth(h, l, cx, cy, ox, oy, rhs, 2 * L.nu, zero_in, jacobi_pairs(h, l, 2 * L.nu, zero_in) & ~1);
            if (cx != ax) {  // an even number of buffer swaps (2 nu sweeps, even pair count)
                cudaMemcpyAsync(ax - COL_OFF, cx - COL_OFF, field_doubles(L.g) * 8, cudaMemcpyDeviceToDevice, h->stream);
                cudaMemcpyAsync(ay - COL_OFF, cy - COL_OFF, field_doubles(L.g) * 8, cudaMemcpyDeviceToDevice, h->stream);
            }
        }
        return;
    }
    Level &C = h->lev[l + 1];
    // each two-sweep pass saves one buffer swap: keep the pair count even so that the
    // 2 nu sweeps of the cycle end in (ax, ay) without a copy
    const int pre_n = L.nu - done_pre, post_n = L.nu - leave_last;
    int pre_pairs = jacobi_pairs(h, l, pre_n, zero_in && !done_pre);
    int post_pairs = jacobi_pairs(h, l, post_n, false);
    if (!leave_last && ((pre_pairs + post_pairs) & 1)) {
        if (post_pairs > 0) --post_pairs;
        else --pre_pairs;
    }
    // the last pre-smoothing pair fused with (2) + (3) when the level allows it (k_j2rr)
    const bool fuse_rr = pre_pairs >= 1 && pre_n >= 2 && level_smoother(h, l) == STOKES_SMOOTH_JACOBI && j2rr_ok(L.g) &&
                         !tile_level(h, l);  // (tile-smoothed levels: one launch per smoothing)
    if (fuse_rr) {
        smooth(h, l, cx, cy, ox, oy, rhs, pre_n - 2, zero_in && !done_pre, pre_pairs - 1);  // (1)
        launch_j2rr(c, L.g, C.g, L.etab, L.etap, cx, cy, ox, oy, rhs, h->o.omega_v, C.bx, C.by);
        double *tt = cx; cx = ox; ox = tt;
        tt = cy; cy = oy; oy = tt;
    } else {
        smooth(h, l, cx, cy, ox, oy, rhs, pre_n, zero_in && !done_pre, pre_pairs);  // (1) pre-smoothing
    }
    if (fuse_rr) {
    } else if (jacobi2_ok(L.g)) {  // (2) residual + (3) restriction in one pass
        launch_residual_restrict(c, L.g, C.g, L.etab, L.etap, cx, cy, rhs, C.bx, C.by);
    } else {
        launch_residual(c, L.g, L.etab, L.etap, cx, cy, rhs, L.rx, L.ry);      // (2) residual
        launch_restrict_vel(c, L.g, C.g, L.rx, L.ry, C.bx, C.by);             // (3) restriction
    }
    vcycle(h, l + 1, C.vx[0], C.vy[0], C.vx[1], C.vy[1], rhs_arrays(C.bx, C.by), true);  // (4)
    if (!leave_last && level_smoother(h, l) == STOKES_SMOOTH_JACOBI && tile_level(h, l) && post_fused_prolong() &&
        launch_jacobi_tile(c, L.g, L.etab, L.etap, cx, cy, ox, oy, rhs, h->o.omega_v, post_n, false, &C.g, C.vx[0],
                           C.vy[0])) {  // (5) + (6): the correction applied while the tile smoother stages v
        double *t = cx; cx = ox; ox = t;
        t = cy; cy = oy; oy = t;
    } else {
        launch_prolong(c, L.g, C.g, C.vx[0], C.vy[0], cx, cy);                // (5) correction
        smooth(h, l, cx, cy, ox, oy, rhs, post_n, false, post_pairs);        // (6) post-smoothing
    }
    if (leave_last) {
        *lx = cx;
        *ly = cy;
        return;
    }
    if (cx != ax) {
        cudaMemcpyAsync(ax - COL_OFF, cx - COL_OFF, field_doubles(L.g) * 8, cudaMemcpyDeviceToDevice, h->stream);
        cudaMemcpyAsync(ay - COL_OFF, cy - COL_OFF, field_doubles(L.g) * 8, cudaMemcpyDeviceToDevice, h->stream);
    }
}

// E of the current state (v, pbuf[pcur]) -> scal[S_E]; mean of the stored p -> scal[S_MSHIFT];
// optional residual arrays (padded).  Fused single pass where the level allows it.
void state_energy(stokes_s *h, double *rx, double *ry, double *rp) {
    Level &F = h->lev[0];
    const LaunchCtx c = ctx(h);
    const double inv_np = 1.0 / ((double)F.g.ncx * F.g.ncy);
    double *p = h->pbuf[h->pcur];
    if (stream_ok(F.g)) {
        launch_uzawa_energy(c, F.g, F.etab, F.etap, F.vx[0], F.vy[0], p, nullptr, h->rho, h->gx, h->gy, 0.0,
                            h->scal + S_ZERO, rx, ry, rp, h->partials);
        launch_uzawa_final(c, h->partials, stream_blocks(F.g), h->scal + S_SF, inv_np, h->scal + S_E,
                           h->scal + S_MSHIFT);
    } else {
        launch_energy(c, F.g, F.etab, F.etap, F.vx[0], F.vy[0], p, h->rho, h->gx, h->gy, rx, ry, rp, h->partials, false);
        launch_energy_final(c, h->partials, energy_blocks(F.g), h->scal + S_SF, h->scal + S_E);
        launch_pupdate(c, F.g, F.etap, F.vx[0], F.vy[0], p, nullptr, 0.0, h->scal + S_ZERO,
                       h->partials);  // sum of the stored p (its mean)
        launch_finalize(c, h->partials, pupdate_blocks(F.g), 1, inv_np, h->scal + S_MSHIFT);
    }
}

// the body of one Uzawa iteration (a12, mode UZAWA) reading pbuf[pcur]: V-cycle(s) on
// L v = f - G p^k, pressure update into pbuf[1-pcur] + mean, energy residual of the new
// (v, p), E -> pinned host.
void uzawa_body(stokes_s *h) {
    Level &F = h->lev[0];
    const LaunchCtx c = ctx(h);
    ras_iteration_start(h);
    for (int k = 0; k < h->o.vcycles_per_iter; ++k)
        vcycle(h, 0, F.vx[0], F.vy[0], F.vx[1], F.vy[1], rhs_fine(h), false);
    ras_iteration_end(h);
    const double a_s = h->o.pressure_sign * h->o.alpha_p;
    const double inv_np = 1.0 / ((double)F.g.ncx * F.g.ncy);
    const double *pin = h->pbuf[h->pcur];
    double *pout = h->pbuf[1 - h->pcur];
    if (stream_ok(F.g)) {
        launch_uzawa_energy(c, F.g, F.etab, F.etap, F.vx[0], F.vy[0], pin, pout, h->rho, h->gx, h->gy, a_s,
                            h->scal + S_MSHIFT, nullptr, nullptr, nullptr, h->partials);
        launch_uzawa_final(c, h->partials, stream_blocks(F.g), h->scal + S_SF, inv_np, h->scal + S_E,
                           h->scal + S_MSHIFT);
    } else {
        launch_pupdate(c, F.g, F.etap, F.vx[0], F.vy[0], pin, pout, a_s, h->scal + S_MSHIFT, h->partials);
        launch_finalize(c, h->partials, pupdate_blocks(F.g), 1, inv_np, h->scal + S_MSHIFT);
        launch_energy(c, F.g, F.etab, F.etap, F.vx[0], F.vy[0], pout, h->rho, h->gx, h->gy, nullptr, nullptr,
                      nullptr, h->partials, false);
        launch_energy_final(c, h->partials, energy_blocks(F.g), h->scal + S_SF, h->scal + S_E);
    }
    cudaMemcpyAsync(h->hscal, h->scal, 8 * sizeof(double), cudaMemcpyDeviceToHost, h->stream);
}

int sync(stokes_s *h) {
    CK(cudaStreamSynchronize(h->stream));
    CKL();
    return STOKES_OK;
}

// Sf = sum f^2 / d_v (the normaliser of E) -> scal[S_SF]
void force_energy(stokes_s *h) {
    Level &F = h->lev[0];
    const LaunchCtx c = ctx(h);
    launch_energy(c, F.g, F.etab, F.etap, F.vx[0], F.vy[0], h->pbuf[0], h->rho, h->gx, h->gy, nullptr, nullptr,
                  nullptr, h->partials, true);
    launch_energy_final(c, h->partials, energy_blocks(F.g), h->scal + S_ZERO, h->scal + S_SFPART);
    // S_SFPART+1 holds the sum Sv of f -> copy into S_SF
    cudaMemcpyAsync(h->scal + S_SF, h->scal + S_SFPART + 1, sizeof(double), cudaMemcpyDeviceToDevice, h->stream);
}

// copy the E that state_energy left in scal[S_E] to the host
int read_energy(stokes_s *h, double *E) {
    CK(cudaMemcpyAsync(h->hscal, h->scal, 8 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    int st = sync(h);
    if (st) return st;
    *E = h->hscal[S_E];
    return STOKES_OK;
}
int energy_now(stokes_s *h, double *E) {
    state_energy(h, nullptr, nullptr, nullptr);
    cudaMemcpyAsync(h->hscal, h->scal, 8 * sizeof(double), cudaMemcpyDeviceToHost, h->stream);
    int st = sync(h);
    if (st) return st;
    *E = h->hscal[S_E];
    return STOKES_OK;
}

void drop_graphs(stokes_s *h) {
    for (int k = 0; k < 2; ++k)
        if (h->uzawa_exec[k]) {
            cudaGraphExecDestroy(h->uzawa_exec[k]);
            h->uzawa_exec[k] = nullptr;
        }
    for (int k = 0; k < 4; ++k)
        if (h->loop_exec[k]) {
            cudaGraphExecDestroy(h->loop_exec[k]);
            h->loop_exec[k] = nullptr;
        }
    for (int k = 0; k < 4; ++k)
        if (h->fused_exec[k]) {
            cudaGraphExecDestroy(h->fused_exec[k]);
            h->fused_exec[k] = nullptr;
        }
    for (int k = 0; k < MAXM; ++k)
        if (h->gcr_exec[k]) {
            cudaGraphExecDestroy(h->gcr_exec[k]);
            h->gcr_exec[k] = nullptr;
        }
}

int ensure_uzawa_graphs(stokes_s *h) {
    // capture one iteration per pressure buffer into CUDA graphs (the coarse levels are
    // launch-bound), replay them alternately
    const int keep = h->pcur;
    for (int k = 0; k < 2; ++k) {
        if (h->uzawa_exec[k]) continue;
        cudaGraph_t graph;
        const long long before = h->launches;
        h->pcur = k;
        CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        uzawa_body(h);
        cudaError_t e = cudaStreamEndCapture(h->stream, &graph);
        h->pcur = keep;
        if (e != cudaSuccess) return fail_cuda(e, "graph capture");
        h->uzawa_kernels = h->launches - before;
        h->launches = before;
        e = cudaGraphInstantiate(&h->uzawa_exec[k], graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            h->uzawa_exec[k] = nullptr;
            return fail_cuda(e, "graph instantiate");
        }
    }
    return STOKES_OK;
}

int solve_uzawa(stokes_s *h, double rtol, double E0, int *iters, double *Eout) {
    ras_reset(h);
    int st = ensure_uzawa_graphs(h);
    if (st) return st;
    double E = E0;
    int k;
    int status = STOKES_NOT_CONVERGED;
    for (k = 1; k <= h->o.max_iter; ++k) {
        CK(cudaGraphLaunch(h->uzawa_exec[h->pcur], h->stream));
        h->pcur ^= 1;
        h->launches += h->uzawa_kernels;
        st = sync(h);
        if (st) return st;
        E = h->hscal[S_E];
        record_E(h, k - 1, E);
        if (!(E == E) || isinf(E) || E > 1e6 * E0) { status = STOKES_EDIVERGED; break; }
        if (E <= rtol) { status = STOKES_OK; break; }
    }
    if (k > h->o.max_iter) k = h->o.max_iter;
    *iters = k;
    *Eout = E;
    return status;
}

// ---- Uzawa with the a12 fusion: the pressure update and the energy residual of iterate k
// ride on the first pre-smoothing sweep of V-cycle k+1 (one HBM pass instead of two).
bool fused_ok(stokes_s *h) {
    return h->o.smoother == STOKES_SMOOTH_JACOBI && h->o.vcycles_per_iter == 1 && h->nlev > 1 && h->o.max_iter >= 1 &&
           h->lev[0].nu >= 1 && stream_ok(h->lev[0].g);
}
// from v^k (buf 0) and p^(k-1) = pbuf[pcur]: p^k -> pbuf[1-pcur], E(v^k, p^k), v' -> buf 1
void fused_tail(stokes_s *h) {
    Level &F = h->lev[0];
    const LaunchCtx c = ctx(h);
    launch_jacobi_uzawa(c, F.g, F.etab, F.etap, F.vx[0], F.vy[0], F.vx[1], F.vy[1], h->pbuf[h->pcur],
                        h->pbuf[1 - h->pcur], h->rho, h->gx, h->gy, h->o.pressure_sign * h->o.alpha_p,
                        h->scal + S_MSHIFT, h->o.omega_v, h->partials);
    launch_uzawa_final(c, h->partials, stream_blocks(F.g), h->scal + S_SF, 1.0 / ((double)F.g.ncx * F.g.ncy),
                       h->scal + S_E, h->scal + S_MSHIFT);
    cudaMemcpyAsync(h->hscal, h->scal, 8 * sizeof(double), cudaMemcpyDeviceToHost, h->stream);
}
// k_jju variant of the tail: the last post-smoothing sweep of the V-cycle rides along.
// v^(k-1/2) in buffer b (the V-cycle left it there), p^(k-1) = pbuf[pcur]: p^k ->
// pbuf[1-pcur], E(v^k, p^k), v' -> buffer 1-b.  Returns 1-b (where the next V-cycle starts).
int fused_tail_jju(stokes_s *h, int b, bool to_host = true) {
    Level &F = h->lev[0];
    const LaunchCtx c = ctx(h);
    launch_jacobi_jju(c, F.g, F.etab, F.etap, F.vx[b], F.vy[b], F.vx[1 - b], F.vy[1 - b], h->pbuf[h->pcur],
                      h->pbuf[1 - h->pcur], h->rho, h->gx, h->gy, h->o.pressure_sign * h->o.alpha_p,
                      h->scal + S_MSHIFT, h->o.omega_v, h->partials);
    launch_uzawa_final(c, h->partials, jju_blocks(F.g), h->scal + S_SF, 1.0 / ((double)F.g.ncx * F.g.ncy),
                       h->scal + S_E, h->scal + S_MSHIFT);
    if (to_host) cudaMemcpyAsync(h->hscal, h->scal, 8 * sizeof(double), cudaMemcpyDeviceToHost, h->stream);
    return 1 - b;
}
// graph body: rest of V-cycle k+1 (its first sweep already in buffer q) on L v = f - G
// pbuf[pcur], then the fused tail of iterate k+1.  Returns the buffer of the next first sweep.
int fused_body(stokes_s *h, int q, bool to_host = true) {
    Level &F = h->lev[0];
    ras_iteration_start(h);
    int nq = 1;
    if (jju_ok(F.g)) {
        double *lx = nullptr, *ly = nullptr;
        vcycle(h, 0, F.vx[1 - q], F.vy[1 - q], F.vx[q], F.vy[q], rhs_fine(h), false, 1, 1, &lx, &ly);
        ras_iteration_end(h);
        nq = fused_tail_jju(h, lx == F.vx[0] ? 0 : 1, to_host);
    } else {
        vcycle(h, 0, F.vx[0], F.vy[0], F.vx[1], F.vy[1], rhs_fine(h), false, 1);
        ras_iteration_end(h);
        fused_tail(h);
    }
    return nq;
}
// ---- device-side Uzawa loop (a12 stopping test on the GPU) -------------------------------
// After iteration 1 the rest of the solve is ONE graph launch: a conditional WHILE node whose
// body runs two fused iterations (the two parities of the pressure / sweep buffers), each
// followed by k_loop_check (E history, divergence guard, E <= rtol, max_iter -- the host
// loop's tests, on the device); the second half sits in a conditional IF node so the loop
// can stop after either.  The host synchronises once per solve instead of once per
// iteration.  STOKES_DEVICE_LOOP=0 keeps the host loop.
constexpr int LOOP_RUNNING = 100;
__global__ void k_loop_check(double *scal, double *dhist, cudaGraphConditionalHandle hnext,
                             cudaGraphConditionalHandle hstop, int has_stop) {
    double *L = scal + S_LOOP;
    const double E = scal[S_E];
    const int k = (int)L[3] + 1;
    L[3] = k;
    L[5] = E;
    if (k - 1 < LOOP_HCAP) dhist[k - 1] = E;
    int st = LOOP_RUNNING;
    if (!(E == E) || isinf(E) || E > 1e6 * L[1]) st = STOKES_EDIVERGED;
    else if (E <= L[0]) st = STOKES_OK;
    else if (k >= (int)L[2]) st = STOKES_NOT_CONVERGED;
    L[4] = st;
    cudaGraphSetConditional(hnext, st == LOOP_RUNNING ? 1u : 0u);
    if (has_stop && st != LOOP_RUNNING) cudaGraphSetConditional(hstop, 0u);
}
static bool device_loop_env() {
    static const bool v = [] {
        const char *e = getenv("STOKES_DEVICE_LOOP");
        return !(e && e[0] == '0');
    }();
    return v;
}
// capture the loop graph entered in state (q, pcur); leaves h->pcur unchanged
static int build_loop(stokes_s *h, int q, int *nq_out) {
    const int keep = h->pcur;
    cudaGraph_t G = nullptr;
    cudaGraphExec_t ex = nullptr;
    cudaError_t e = cudaGraphCreate(&G, 0);
    if (e != cudaSuccess) return fail_cuda(e, "loop graph");
    cudaGraphConditionalHandle hw, hi;
    cudaGraphNodeParams wp = {};
    cudaGraphNode_t wn, in;
    cudaGraph_t BW = nullptr, BI = nullptr;
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    cudaGraph_t cg = nullptr;
    const long long before = h->launches;
    long long nk = 0;
    int q1 = q, q2 = q;
    e = cudaGraphConditionalHandleCreate(&hw, G, 1, cudaGraphCondAssignDefault);
    if (e == cudaSuccess) {
        wp.type = cudaGraphNodeTypeConditional;
        wp.conditional.handle = hw;
        wp.conditional.type = cudaGraphCondTypeWhile;
        wp.conditional.size = 1;
        e = cudaGraphAddNode(&wn, G, nullptr, 0, &wp);
    }
    if (e == cudaSuccess) {
        BW = wp.conditional.phGraph_out[0];
        e = cudaGraphConditionalHandleCreate(&hi, BW, 0, cudaGraphCondAssignDefault);
    }
    if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(h->stream, BW, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {  // half A: iteration in state (q, pcur), then the check (IF <- continue)
        q1 = fused_body(h, q, false);
        nk = h->launches - before;
        k_loop_check<<<1, 1, 0, h->stream>>>(h->scal, h->dhist, hi, hw, 1);
        e = cudaStreamGetCaptureInfo(h->stream, &cs, nullptr, &cg, &deps, &nd);
        if (e == cudaSuccess) {
            cudaGraphNodeParams ip = {};
            ip.type = cudaGraphNodeTypeConditional;
            ip.conditional.handle = hi;
            ip.conditional.type = cudaGraphCondTypeIf;
            ip.conditional.size = 1;
            e = cudaGraphAddNode(&in, cg, deps, nd, &ip);
            if (e == cudaSuccess) {
                BI = ip.conditional.phGraph_out[0];
                e = cudaStreamUpdateCaptureDependencies(h->stream, &in, 1, cudaStreamSetCaptureDependencies);
            }
        }
        cudaGraph_t out = nullptr;
        const cudaError_t e2 = cudaStreamEndCapture(h->stream, &out);
        if (e == cudaSuccess) e = e2;
    }
    if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(h->stream, BI, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {  // half B: the other parity, then the check (WHILE <- continue)
        h->pcur = 1 - keep;
        q2 = fused_body(h, q1, false);
        k_loop_check<<<1, 1, 0, h->stream>>>(h->scal, h->dhist, hw, hw, 0);
        cudaGraph_t out = nullptr;
        e = cudaStreamEndCapture(h->stream, &out);
    }
    h->pcur = keep;
    h->launches = before;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&ex, G, 0);
    cudaGraphDestroy(G);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail_cuda(e, "device loop graph");
    }
    if (q2 != q) {  // the state after two iterations must be the entry state
        cudaGraphExecDestroy(ex);
        g_last_error = "device loop: buffer parity not periodic";
        return STOKES_ECUDA;
    }
    h->loop_exec[(q << 1) | keep] = ex;
    // the host replays the buffer sequence from these (also what the host-loop graphs record)
    h->fused_nq[(q << 1) | keep] = q1;
    h->fused_nq[(q1 << 1) | (1 - keep)] = q2;
    h->fused_kernels = nk;
    *nq_out = q1;
    return STOKES_OK;
}

int solve_uzawa_fused(stokes_s *h, double rtol, double E0, int *iters, double *Eout) {
    ras_reset(h);
    Level &F = h->lev[0];
    const bool jju = jju_ok(F.g);
    int *next_q = h->fused_nq;  // buffer of the first sweep after a body of slot k (set at capture)
    auto slot_of = [&](int q) { return (q << 1) | h->pcur; };
    auto ensure = [&](int q) -> int {  // capture the body for (pbuf[pcur], first sweep in buffer q)
        const int k = slot_of(q);
        if (h->fused_exec[k]) return STOKES_OK;
        cudaGraph_t graph;
        const long long before = h->launches;
        CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        next_q[k] = fused_body(h, q);
        cudaError_t e = cudaStreamEndCapture(h->stream, &graph);
        if (e != cudaSuccess) return fail_cuda(e, "graph capture");
        h->fused_kernels = h->launches - before;
        h->launches = before;
        e = cudaGraphInstantiate(&h->fused_exec[k], graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            h->fused_exec[k] = nullptr;
            return fail_cuda(e, "graph instantiate");
        }
        return STOKES_OK;
    };
    double E = E0;
    int k = 1, status = STOKES_NOT_CONVERGED;
    // iteration 1: a full V-cycle from (v^0, p^0), then the fused tail of iterate 1
    int q = 1, b = 0;  // q: buffer of the next first sweep; b: buffer of v^(k-1/2) (k_jju path)
    nvtxRangePushA("uzawa: iteration 1");
    ras_iteration_start(h);
    if (jju) {
        double *lx = nullptr, *ly = nullptr;
        vcycle(h, 0, F.vx[0], F.vy[0], F.vx[1], F.vy[1], rhs_fine(h), false, 0, 1, &lx, &ly);
        ras_iteration_end(h);
        b = lx == F.vx[0] ? 0 : 1;
        q = fused_tail_jju(h, b);
    } else {
        vcycle(h, 0, F.vx[0], F.vy[0], F.vx[1], F.vy[1], rhs_fine(h), false);
        ras_iteration_end(h);
        fused_tail(h);
    }
    nvtxRangePop();
    NVTX_RANGE("uzawa: iterations 2..k (device loop or graph replays)");
    for (;;) {
        h->pcur ^= 1;  // pbuf[pcur] = p^k
        int st = sync(h);
        if (st) return st;
        E = h->hscal[S_E];
        record_E(h, k - 1, E);
        if (!(E == E) || isinf(E) || E > 1e6 * E0) { status = STOKES_EDIVERGED; break; }
        if (E <= rtol) { status = STOKES_OK; break; }
        if (k >= h->o.max_iter) break;
        if (jju && k == 1 && device_loop_env() && !h->loop_off) {  // the rest on the device
            int nq1 = 0;
            const int li = (q << 1) | h->pcur;
            if (!h->dhist) {
                if (cudaMalloc(&h->dhist, LOOP_HCAP * sizeof(double)) != cudaSuccess) {
                    cudaGetLastError();
                    h->dhist = nullptr;
                    h->loop_off = true;
                }
            }
            if (!h->loop_off && !h->loop_exec[li] && build_loop(h, q, &nq1)) h->loop_off = true;
            if (!h->loop_off) {
                const double L0[6] = {rtol, E0, (double)h->o.max_iter, 1.0, (double)LOOP_RUNNING, E};
                memcpy(h->hscal + S_LOOP, L0, sizeof L0);
                CK(cudaMemcpyAsync(h->scal + S_LOOP, h->hscal + S_LOOP, sizeof L0, cudaMemcpyHostToDevice, h->stream));
                CK(cudaGraphLaunch(h->loop_exec[li], h->stream));
                CK(cudaMemcpyAsync(h->hscal + S_LOOP, h->scal + S_LOOP, sizeof L0, cudaMemcpyDeviceToHost, h->stream));
                if ((st = sync(h))) return st;
                const int kf = (int)h->hscal[S_LOOP + 3];
                const int stf = (int)h->hscal[S_LOOP + 4];
                E = h->hscal[S_LOOP + 5];
                if (h->hist && kf > 1) {  // E of iterations 2..kf (device history)
                    const int n = (kf < LOOP_HCAP ? kf : LOOP_HCAP) - 1;
                    double *tmp = (double *)malloc(n * sizeof(double));
                    if (!tmp) return STOKES_ENOMEM;
                    CK(cudaMemcpyAsync(tmp, h->dhist + 1, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
                    if ((st = sync(h))) { free(tmp); return st; }
                    for (int i = 0; i < n; ++i) record_E(h, i + 1, tmp[i]);
                    free(tmp);
                }
                // replay the state sequence of iterations 2..kf on the host (buffers, pcur)
                for (int it = 2; it <= kf; ++it) {
                    const int slot = slot_of(q);
                    h->launches += h->fused_kernels + 1;  // + k_loop_check
                    q = next_q[slot];
                    b = 1 - q;
                    h->pcur ^= 1;
                }
                k = kf;
                status = stf == LOOP_RUNNING ? STOKES_NOT_CONVERGED : stf;
                break;
            }
        }
        ++k;
        const int slot = slot_of(q);
        if ((st = ensure(q))) return st;
        CK(cudaGraphLaunch(h->fused_exec[slot], h->stream));
        h->launches += h->fused_kernels;
        q = next_q[slot];
        b = 1 - q;  // k_jju path: v^(k-1/2) stayed in the buffer the pass read
    }
    if (jju) {  // v^k was never stored: one JacobiOp sweep from v^(k-1/2) (buffer b, untouched)
        RhsArgs r = rhs_fine(h);
        r.p = h->pbuf[1 - h->pcur];  // p^(k-1)
        const LaunchCtx c = ctx(h);
        launch_jacobi(c, F.g, F.etab, F.etap, F.vx[b], F.vy[b], F.vx[1 - b], F.vy[1 - b], r, h->o.omega_v, false);
        if (b == 0) {  // v^k is now in buffer 1 -> buffer 0
            cudaMemcpyAsync(F.vx[0] - COL_OFF, F.vx[1] - COL_OFF, field_doubles(F.g) * 8, cudaMemcpyDeviceToDevice, h->stream);
            cudaMemcpyAsync(F.vy[0] - COL_OFF, F.vy[1] - COL_OFF, field_doubles(F.g) * 8, cudaMemcpyDeviceToDevice, h->stream);
        }
    }
    *iters = k;
    *Eout = E;
    return status;  // (v^k in buf 0, p^k in pbuf[pcur], its mean in S_MSHIFT)
}

// One fused GCR step i (Alg. 4 inner loop body) on the stream:
// V-cycle (z_v = V(0; r_v)); z_p + w = A z + first dot (one streaming pass); i fused MGS
// steps (axpy + next dot per HBM pass); normalise + update x, r + energy of r (one pass);
// E, nu^2, <r,r> -> pinned host.  The stored z_p is not de-meaned (inert, reading R14).
static bool gcr_defer_z() {  // STOKES_GCR_DEFER_Z=0: the z update inside every MGS step (diagnostics)
    const char *e = getenv("STOKES_GCR_DEFER_Z");
    return !(e && e[0] == '0');
}
void gcr_step_body(stokes_s *h, int i) {
    Level &F = h->lev[0];
    const GridL &g = F.g;
    const LaunchCtx c = ctx(h);
    double **z = h->gz[i], **w = h->gw[i], **r = h->gr;
    double *x[3] = {F.vx[0], F.vy[0], h->pbuf[h->pcur]};
    const size_t nf = field_doubles(g);
    double *PA = h->partials, *PB = h->partials + 4096, *PC = h->partials + 8192;
    ras_iteration_start(h);
    for (int q = 0; q < h->o.vcycles_per_iter; ++q)
        vcycle(h, 0, z[0], z[1], h->gtmp[0], h->gtmp[1], rhs_arrays(r[0], r[1]), q == 0);
    ras_iteration_end(h);
    launch_precond_apply(c, g, F.etab, F.etap, z[0], z[1], r[2], h->o.alpha_p, z[2], w[0], w[1], w[2],
                         i > 0 ? (const double *const *)h->gw[0] : nullptr, r[0], r[1], PA);
    int nb = stream_blocks(g);
    double *pin = PA, *pout = PB;
    const bool defer = gcr_defer_z();  // z -= gamma_j z_j for all j in the update pass (same arithmetic)
    for (int j = 0; j < i; ++j) {
        const double *const *nxt = (j + 1 < i) ? (const double *const *)h->gw[j + 1] : nullptr;
        launch_mgs_step(c, pin, nb, 2, 0, w, defer ? nullptr : z, (const double *const *)h->gw[j],
                        (const double *const *)h->gz[j], nxt, (const double *const *)r, nf, pout,
                        defer ? h->scal + S_GAMS + j : nullptr);
        nb = gcr_flat_blocks(nf);
        double *t = pin;
        pin = pout;
        pout = t;
    }
    launch_gcr_update(c, pin, nb, w, z, x, r, (const double *const *)h->gew, nf, PC, h->scal + S_GAMS, defer ? i : 0,
                      h->gz);
    launch_gcr_final(c, PC, gcr_flat_blocks(nf), pin, nb, h->scal + S_SF, h->scal + S_E, h->scal + S_NU2,
                     h->scal + S_RR);
    cudaMemcpyAsync(h->hscal, h->scal, 16 * sizeof(double), cudaMemcpyDeviceToHost, h->stream);
}

int solve_gcr_fused(stokes_s *h, double rtol, double E0, int *iters, double *Eout) {
    ras_reset(h);
    const int m = h->o.gcr_restart;
    double **r = h->gr;
    state_energy(h, r[0], r[1], r[2]);  // r0 = b - A x0
    int k = 0, status = STOKES_NOT_CONVERGED, fresh = 1;
    double E = E0;
    while (k < h->o.max_iter && status == STOKES_NOT_CONVERGED) {
        if (!fresh && h->o.gcr_true_restart) state_energy(h, r[0], r[1], r[2]);  // restart (R13)
        fresh = 0;
        for (int i = 0; i < m && k < h->o.max_iter; ++i) {
            if (!h->gcr_exec[i]) {  // capture step i once (pcur is fixed during GCR)
                cudaGraph_t graph;
                const long long before = h->launches;
                CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
                gcr_step_body(h, i);
                cudaError_t e = cudaStreamEndCapture(h->stream, &graph);
                if (e != cudaSuccess) return fail_cuda(e, "graph capture");
                h->gcr_kernels[i] = h->launches - before;
                h->launches = before;
                e = cudaGraphInstantiate(&h->gcr_exec[i], graph, 0);
                cudaGraphDestroy(graph);
                if (e != cudaSuccess) {
                    h->gcr_exec[i] = nullptr;
                    return fail_cuda(e, "graph instantiate");
                }
            }
            CK(cudaGraphLaunch(h->gcr_exec[i], h->stream));
            h->launches += h->gcr_kernels[i];
            int st = sync(h);
            if (st) return st;
            ++k;
            const double nu2 = h->hscal[S_NU2], rr = h->hscal[S_RR];
            E = h->hscal[S_E];
            record_E(h, k - 1, E);
            if (!(nu2 > 1e-28 * rr)) { status = STOKES_EDIVERGED; break; }  // breakdown (R13)
            if (!(E == E) || isinf(E) || E > 1e6 * E0) { status = STOKES_EDIVERGED; break; }
            if (E <= rtol) {  // exit test on the true residual (R13): else restart from it
                double Et;
                state_energy(h, r[0], r[1], r[2]);
                if ((st = read_energy(h, &Et))) return st;
                fresh = 1;
                if (Et <= rtol) status = STOKES_OK;
                break;
            }
        }
    }
    *iters = k;
    // the true E of x and the mean of x_p for the output de-mean
    int st = energy_now(h, &E);
    if (st) return st;
    *Eout = E;
    return status;
}

// Flexible GCR(m) with modified Gram-Schmidt, Alg. 4, readings R13/R14.
int solve_gcr(stokes_s *h, double rtol, double E0, int *iters, double *Eout) {
    ras_reset(h);
    Level &F = h->lev[0];
    const GridL &g = F.g;
    const LaunchCtx c = ctx(h);
    const int m = h->o.gcr_restart;
    const int nb = energy_blocks(g);
    double *x[3] = {F.vx[0], F.vy[0], h->pbuf[h->pcur]};
    double **r = h->gr;
    // r0 = b - A x0 (recursive residual)
    state_energy(h, r[0], r[1], r[2]);
    int k = 0, status = STOKES_NOT_CONVERGED, fresh = 1;
    double E = E0;
    const double inv_np = 1.0 / ((double)g.ncx * g.ncy);
    while (k < h->o.max_iter && status == STOKES_NOT_CONVERGED) {
        if (!fresh && h->o.gcr_true_restart) state_energy(h, r[0], r[1], r[2]);  // restart (R13)
        fresh = 0;
        for (int i = 0; i < m && k < h->o.max_iter; ++i) {
            double **z = h->gz[i], **w = h->gw[i];
            // z = M^-1 r: dv = Vcycle(0; r_v); dp = alpha eta_P (r_p - D dv); de-mean dp
            ras_iteration_start(h);
            for (int q = 0; q < h->o.vcycles_per_iter; ++q)
                vcycle(h, 0, z[0], z[1], h->gtmp[0], h->gtmp[1], rhs_arrays(r[0], r[1]), q == 0);
            ras_iteration_end(h);
            launch_precond_p(c, g, F.etap, z[0], z[1], r[2], h->o.alpha_p, z[2], h->partials);
            launch_finalize(c, h->partials, nb, 1, inv_np, h->scal + S_ZMEAN);
            launch_sub_mean(c, g, h->scal + S_ZMEAN, z[2]);
            // w = A z
            launch_apply_padded(c, g, F.etab, F.etap, z[0], z[1], z[2], w[0], w[1], w[2]);
            for (int j = 0; j < i; ++j) {  // modified Gram-Schmidt
                const double *a[3] = {w[0], w[1], w[2]};
                const double *b[3] = {h->gw[j][0], h->gw[j][1], h->gw[j][2]};
                launch_dots(c, g, a, b, 1, h->partials);
                launch_finalize(c, h->partials, nb, 1, 1.0, h->scal + S_GAMMA);
                launch_axpy3(c, g, h->scal, S_GAMMA, -1.0, h->gw[j][0], h->gw[j][1], h->gw[j][2], w[0], w[1], w[2]);
                launch_axpy3(c, g, h->scal, S_GAMMA, -1.0, h->gz[j][0], h->gz[j][1], h->gz[j][2], z[0], z[1], z[2]);
            }
            {
                const double *a[6] = {w[0], w[1], w[2], r[0], r[1], r[2]};
                launch_dots(c, g, a, a, 2, h->partials);
                launch_finalize(c, h->partials, nb, 2, 1.0, h->scal + S_NU2);
            }
            launch_scale3(c, g, h->scal + S_NU2, 1, w[0], w[1], w[2]);
            launch_scale3(c, g, h->scal + S_NU2, 1, z[0], z[1], z[2]);
            {
                const double *a[3] = {r[0], r[1], r[2]};
                const double *b[3] = {w[0], w[1], w[2]};
                launch_dots(c, g, a, b, 1, h->partials);
                launch_finalize(c, h->partials, nb, 1, 1.0, h->scal + S_BETA);
            }
            launch_axpy3(c, g, h->scal, S_BETA, 1.0, z[0], z[1], z[2], x[0], x[1], x[2]);
            launch_axpy3(c, g, h->scal, S_BETA, -1.0, w[0], w[1], w[2], r[0], r[1], r[2]);
            launch_energy_vec(c, g, F.etab, F.etap, r[0], r[1], r[2], h->partials);
            launch_energy_final(c, h->partials, nb, h->scal + S_SF, h->scal + S_E);
            cudaMemcpyAsync(h->hscal, h->scal, 16 * sizeof(double), cudaMemcpyDeviceToHost, h->stream);
            int st = sync(h);
            if (st) return st;
            ++k;
            const double nu2 = h->hscal[S_NU2], rr = h->hscal[S_RR];
            E = h->hscal[S_E];
            record_E(h, k - 1, E);
            if (!(nu2 > 1e-28 * rr)) { status = STOKES_EDIVERGED; break; }  // breakdown (R13)
            if (!(E == E) || isinf(E) || E > 1e6 * E0) { status = STOKES_EDIVERGED; break; }
            if (E <= rtol) {  // exit test on the true residual (R13): else restart from it
                double Et;
                state_energy(h, r[0], r[1], r[2]);
                if ((st = read_energy(h, &Et))) return st;
                fresh = 1;
                if (Et <= rtol) status = STOKES_OK;
                break;
            }
        }
    }
    *iters = k;
    // the true E of x; the pressure mean of x (inert) is removed at output
    // through S_MSHIFT
    int st = energy_now(h, &E);
    if (st) return st;
    *Eout = E;
    return status;
}

bool valid_level(stokes_s *h, int l) { return h && !h->dist && l >= 0 && l < h->nlev; }
int build_hierarchy(stokes_s *h);

}  // namespace sk

// ===================================================================== C ABI
using namespace sk;
extern "C" {

int stokes_opts_default(stokes_opts *o) {
    if (!o) return STOKES_EINVAL;
    o->smoother = STOKES_SMOOTH_JACOBI;
    o->omega_v = 0.3;
    o->alpha_p = 0.6;
    o->nu1 = 5;
    o->nu_growth = 1.0;
    o->coarse_min = 8;
    o->coarse_direct = 1;
    o->vcycles_per_iter = 1;
    o->accel = STOKES_ACCEL_NONE;
    o->gcr_restart = 10;
    o->max_iter = 10000;
    o->pressure_sign = 1;
    o->theta_step = 0.0;
    o->theta_every = 25;
    o->aa_depth = 5;
    o->aa_beta = 0.7;
    o->ras_tile = 32;
    o->ras_inner = 4;
    o->ras_seed = 2603;
    o->gcr_true_restart = 1;
    return STOKES_OK;
}

static int prepare(stokes_s *h, int nx, int ny, double Lx, double Ly, const int bc[4], const stokes_opts *opts) {
    if (nx < 2 || ny < 2 || !(Lx > 0) || !(Ly > 0) || !bc) return STOKES_EINVAL;
    for (int k = 0; k < 4; ++k)
        if (bc[k] != 0 && bc[k] != 1) return STOKES_EINVAL;
    h->nx = nx;
    h->ny = ny;
    h->Lx = Lx;
    h->Ly = Ly;
    memcpy(h->bc, bc, sizeof(h->bc));
    if (opts) h->o = *opts;
    else stokes_opts_default(&h->o);
    if (check_opts(h->o)) return STOKES_EINVAL;
    GridL gs[MAXLEV];
    int nus[MAXLEV];
    h->nlev = build_levels(nx, ny, Lx, Ly, bc, h->o, gs, nus);
    for (int l = 0; l < h->nlev; ++l) {
        h->lev[l].g = gs[l];
        h->lev[l].nu = nus[l];
    }
    return STOKES_OK;
}

int stokes_workspace_bytes(int nx, int ny, const stokes_opts *opts, size_t *bytes) {
    if (!bytes) return STOKES_EINVAL;
    stokes_s h;
    memset(&h, 0, sizeof h);
    const int bc[4] = {0, 0, 0, 0};
    int st = prepare(&h, nx, ny, 1.0, 1.0, bc, opts);
    if (st) return st;
    Carver cv{nullptr, 0, 0, true};
    *bytes = carve(&h, cv);
    return STOKES_OK;
}

int stokes_create(int nx, int ny, double Lx, double Ly, const int bc[4], const stokes_opts *opts, void *cuda_stream,
                  void *workspace, size_t workspace_bytes, stokes_t *out) {
    if (!out) return STOKES_EINVAL;
    stokes_s *h = (stokes_s *)calloc(1, sizeof(stokes_s));
    if (!h) return STOKES_ENOMEM;
    int st = prepare(h, nx, ny, Lx, Ly, bc, opts);
    if (st) { free(h); return st; }
    cudaGetDevice(&h->device);
    h->stream = (cudaStream_t)cuda_stream;
    if (!h->stream) {  // the legacy default stream cannot be graph-captured: use our own
        cudaError_t e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) { free(h); return fail_cuda(e, "cudaStreamCreate"); }
        h->own_stream = true;
    }
    Carver dry{nullptr, 0, 0, true};
    const size_t need = carve(h, dry);
    if (workspace) {
        if (workspace_bytes < need || ((uintptr_t)workspace & 255)) { free(h); return STOKES_ENOMEM; }
        h->ws = workspace;
        h->own_ws = false;
    } else {
        cudaError_t e = cudaMalloc(&h->ws, need);
        if (e != cudaSuccess) { free(h); fail_cuda(e, "cudaMalloc workspace"); return STOKES_ENOMEM; }
        h->own_ws = true;
    }
    h->ws_bytes = need;
    Carver cv{(char *)h->ws, 0, need, false};
    carve(h, cv);
    cudaError_t e = cudaMallocHost(&h->hscal, S_NSCAL * sizeof(double));
    if (e != cudaSuccess) { if (h->own_ws) cudaFree(h->ws); free(h); fail_cuda(e, "cudaMallocHost"); return STOKES_ECUDA; }
    memset(h->hscal, 0, S_NSCAL * sizeof(double));
    // zero everything once: walls / ghosts of every buffer stay 0 (reading R1, R5)
    e = cudaMemsetAsync(h->ws, 0, need, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) {
        cudaFreeHost(h->hscal);
        if (h->own_ws) cudaFree(h->ws);
        free(h);
        return fail_cuda(e, "workspace init");
    }
    *out = h;
    return STOKES_OK;
}

int stokes_destroy(stokes_t h) {
    DEVICE_GUARD(h);
    if (!h) return STOKES_EINVAL;
    if (h->dist) {
        dist_destroy(h->dist);
        free(h);
        return STOKES_OK;
    }
    drop_graphs(h);
    if (h->mk_ws) cudaFree(h->mk_ws);
    if (h->dhist) cudaFree(h->dhist);
    if (h->hscal) cudaFreeHost(h->hscal);
    if (h->own_ws && h->ws) cudaFree(h->ws);
    if (h->own_stream) cudaStreamDestroy(h->stream);
    free(h);
    return STOKES_OK;
}

int stokes_num_levels(stokes_t h, int *nlev) {
    DEVICE_GUARD(h);
    if (!h || !nlev) return STOKES_EINVAL;
    if (h->dist) {
        *nlev = dist_num_levels(h->dist);
        return STOKES_OK;
    }
    *nlev = h->nlev;
    return STOKES_OK;
}
int stokes_level_shape(stokes_t h, int level, int *nx, int *ny, int *nu) {
    DEVICE_GUARD(h);
    if (!valid_level(h, level) || !nx || !ny || !nu) return STOKES_EINVAL;
    *nx = h->lev[level].g.ncx;
    *ny = h->lev[level].g.ncy;
    *nu = h->lev[level].nu;
    return STOKES_OK;
}

int stokes_set_viscosity(stokes_t h, const double *eta_b, const double *eta_p) {
    DEVICE_GUARD(h);
    NVTX_RANGE("stokes_set_viscosity");
    if (!h || !eta_b || !eta_p) return STOKES_EINVAL;
    if (h->dist) return dist_set_viscosity(h->dist, eta_b, eta_p);
    const LaunchCtx c = ctx(h);
    CK(cudaMemsetAsync(h->dflag, 0, sizeof(int), h->stream));
    launch_count_nonpos(c, eta_b, (size_t)(h->ny + 1) * (h->nx + 1), h->dflag);
    launch_count_nonpos(c, eta_p, (size_t)h->ny * h->nx, h->dflag);
    int bad = 0;
    CK(cudaMemcpyAsync(&h->hscal[S_NSCAL - 1], h->dflag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    int st = sync(h);
    if (st) return st;
    memcpy(&bad, &h->hscal[S_NSCAL - 1], sizeof(int));
    if (bad) return STOKES_EINVAL;
    Level &F = h->lev[0];
    launch_in_b(c, F.g, eta_b, F.etab);
    launch_in_p(c, F.g, eta_p, F.etap);
    if (h->etab_user) {  // kept for viscosity rescaling
        CK(cudaMemcpyAsync(h->etab_user - COL_OFF, F.etab - COL_OFF, field_doubles(F.g) * 8, cudaMemcpyDeviceToDevice,
                           h->stream));
        CK(cudaMemcpyAsync(h->etap_user - COL_OFF, F.etap - COL_OFF, field_doubles(F.g) * 8, cudaMemcpyDeviceToDevice,
                           h->stream));
    }
    return build_hierarchy(h);
}

int stokes_lithostatic(stokes_t h, double *p) {
    DEVICE_GUARD(h);
    if (!h || !p || h->dist) return STOKES_EINVAL;
    if (!h->have_rho) return STOKES_ESTATE;
    launch_lithostatic(ctx(h), h->lev[0].g, h->rho, h->gy, p);
    return sync(h);
}

}  // extern "C"
namespace sk {
// coarse viscosities (a7) and the coarsest inverse (a8) from the level-0 viscosities
int build_hierarchy(stokes_s *h) {
    const LaunchCtx c = ctx(h);
    Level &F = h->lev[0];
    int bad = 0, st;
    for (int l = 0; l + 1 < h->nlev; ++l) {  // a7: coarse viscosities by restriction
        launch_restrict_b(c, h->lev[l].g, h->lev[l + 1].g, h->lev[l].etab, h->lev[l + 1].etab);
        launch_restrict_p(c, h->lev[l].g, h->lev[l + 1].g, h->lev[l].etap, h->lev[l + 1].etap);
    }
    if (h->o.coarse_direct) {  // a8: explicit inverse of -L_c
        if (h->nc == 0) return STOKES_EINVAL;  // coarsest too large for the direct solve
        Level &C = h->lev[h->nlev - 1];
        CK(cudaMemsetAsync(h->dflag, 0, sizeof(int), h->stream));
        launch_coarse_assemble(c, C.g, C.etab, C.etap, h->Minv);
        launch_coarse_invert(c, h->Mwork, h->Minv, h->nc, h->dflag);
        CK(cudaMemcpyAsync(&h->hscal[S_NSCAL - 1], h->dflag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        st = sync(h);
        if (st) return st;
        memcpy(&bad, &h->hscal[S_NSCAL - 1], sizeof(int));
        if (bad) return STOKES_EINVAL;
    }
    if (h->o.accel == STOKES_ACCEL_GCR) launch_energy_weights(c, F.g, F.etab, F.etap, h->gew[0], h->gew[1], h->gew[2]);
    h->have_eta = true;
    if (h->have_rho) force_energy(h);
    return sync(h);
}
}  // namespace sk
extern "C" {

int stokes_set_density(stokes_t h, const double *rho_b) {
    DEVICE_GUARD(h);
    if (!h || !rho_b) return STOKES_EINVAL;
    if (h->dist) return dist_set_density(h->dist, rho_b);
    launch_in_b(ctx(h), h->lev[0].g, rho_b, h->rho);
    h->have_rho = true;
    if (h->have_eta) force_energy(h);
    return sync(h);
}

int stokes_set_gravity(stokes_t h, double gx, double gy) {
    DEVICE_GUARD(h);
    if (!h || !(gx == gx) || !(gy == gy)) return STOKES_EINVAL;
    if (h->dist) return dist_set_gravity(h->dist, gx, gy);
    h->gx = gx;
    h->gy = gy;
    drop_graphs(h);  // gravity is baked into the captured graphs
    if (h->have_eta && h->have_rho) force_energy(h);
    return sync(h);
}

int stokes_apply_operator(stokes_t h, const double *vx, const double *vy, const double *p, double *ax, double *ay,
                          double *ap) {
    DEVICE_GUARD(h);
    if (!h || h->dist || !vx || !vy || !p || !ax || !ay || !ap) return STOKES_EINVAL;
    if (!h->have_eta) return STOKES_ESTATE;
    Level &F = h->lev[0];
    const LaunchCtx c = ctx(h);
    launch_in_velocity(c, F.g, vx, vy, F.rx, F.ry);  // scratch: rx/ry hold the padded v
    launch_in_p(c, F.g, p, F.bx);
    launch_apply(c, F.g, F.etab, F.etap, F.rx, F.ry, F.bx, ax, ay, ap);
    return sync(h);
}

int stokes_residual(stokes_t h, const double *vx, const double *vy, const double *p, double *rx, double *ry,
                    double *rp, double *rel_energy) {
    DEVICE_GUARD(h);
    if (!h || !vx || !vy || !p) return STOKES_EINVAL;
    if (h->dist) {  // decomposed handles: E only
        if (rx || ry || rp || !rel_energy) return STOKES_EINVAL;
        return dist_residual_energy(h->dist, vx, vy, p, rel_energy);
    }
    if (!h->have_eta || !h->have_rho) return STOKES_ESTATE;
    Level &F = h->lev[0];
    const LaunchCtx c = ctx(h);
    launch_in_velocity(c, F.g, vx, vy, F.vx[0], F.vy[0]);
    h->pcur = 0;
    launch_in_p(c, F.g, p, h->pbuf[0]);
    state_energy(h, F.rx, F.ry, F.bx);
    if (rx) launch_out_vx(c, F.g, F.rx, rx);
    if (ry) launch_out_vy(c, F.g, F.ry, ry);
    if (rp) launch_out_p(c, F.g, F.bx, rp, nullptr);
    CK(cudaMemcpyAsync(h->hscal, h->scal, 8 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    int st = sync(h);
    if (st) return st;
    if (rel_energy) *rel_energy = h->hscal[S_E];
    return STOKES_OK;
}

int stokes_vcycle(stokes_t h, const double *bx, const double *by, double *vx, double *vy) {
    DEVICE_GUARD(h);
    NVTX_RANGE("stokes_vcycle");
    if (!h || h->dist || !bx || !by || !vx || !vy) return STOKES_EINVAL;
    if (!h->have_eta) return STOKES_ESTATE;
    Level &F = h->lev[0];
    const LaunchCtx c = ctx(h);
    launch_in_vx_raw(c, F.g, bx, F.bx);
    launch_in_vy_raw(c, F.g, by, F.by);
    launch_in_velocity(c, F.g, vx, vy, F.vx[0], F.vy[0]);
    ras_reset(h);
    vcycle(h, 0, F.vx[0], F.vy[0], F.vx[1], F.vy[1], rhs_arrays(F.bx, F.by), false);
    launch_out_vx(c, F.g, F.vx[0], vx);
    launch_out_vy(c, F.g, F.vy[0], vy);
    return sync(h);
}

int stokes_solve_hist(stokes_t h, double rtol, double *vx, double *vy, double *p, int *iters, double *rel_energy,
                      double *hist, int hist_len) {
    DEVICE_GUARD(h);
    if (!h || hist_len < 0 || (hist_len > 0 && !hist) || h->dist) return STOKES_EINVAL;
    h->hist = hist_len > 0 ? hist : nullptr;
    h->hist_len = hist_len;
    h->hist_off = 0;
    const int st = stokes_solve(h, rtol, vx, vy, p, iters, rel_energy);
    h->hist = nullptr;
    h->hist_len = 0;
    return st;
}

int stokes_solve(stokes_t h, double rtol, double *vx, double *vy, double *p, int *iters, double *rel_energy) {
    DEVICE_GUARD(h);
    NVTX_RANGE("stokes_solve");
    if (!h || !vx || !vy || !p || !iters || !rel_energy || !(rtol >= 0)) return STOKES_EINVAL;
    if (h->dist) return dist_solve(h->dist, rtol, vx, vy, p, iters, rel_energy);
    if (!h->have_eta || !h->have_rho) return STOKES_ESTATE;
    Level &F = h->lev[0];
    const LaunchCtx c = ctx(h);
    // load the initial guess
    launch_in_velocity(c, F.g, vx, vy, F.vx[0], F.vy[0]);
    h->pcur = 0;
    launch_in_p(c, F.g, p, h->pbuf[0]);
    CK(cudaMemsetAsync(h->scal + S_MSHIFT, 0, sizeof(double), h->stream));
    CK(cudaMemcpyAsync(h->hscal + 32, h->scal + S_SF, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    int st = sync(h);
    if (st) return st;
    const double Sf = h->hscal[32];
    int status;
    if (!(Sf > 0)) {  // f == 0: zero solution, 0 iterations
        CK(cudaMemsetAsync(vx, 0, (size_t)h->ny * (h->nx + 1) * 8, h->stream));
        CK(cudaMemsetAsync(vy, 0, (size_t)(h->ny + 1) * h->nx * 8, h->stream));
        CK(cudaMemsetAsync(p, 0, (size_t)h->ny * h->nx * 8, h->stream));
        *iters = 0;
        *rel_energy = 0.0;
        return sync(h);
    }
    double E0;
    st = energy_now(h, &E0);
    if (st) return st;
    if (E0 <= rtol) {
        *iters = 0;
        *rel_energy = E0;
        status = STOKES_OK;  // energy_now left the mean of the stored p in S_MSHIFT
    } else if (h->o.theta_step > 0.0) {
        status = solve_staged(h, rtol, iters, rel_energy);
    } else {
        status = solve_inner(h, rtol, E0, iters, rel_energy);
    }
    if (status < 0 && status != STOKES_EDIVERGED) return status;
    launch_out_vx(c, F.g, F.vx[0], vx);
    launch_out_vy(c, F.g, F.vy[0], vy);
    launch_out_p(c, F.g, h->pbuf[h->pcur], p, h->scal + S_MSHIFT);
    st = sync(h);
    if (st) return st;
    return status;
}

}  // extern "C"
namespace sk {
int solve_inner(stokes_s *h, double rtol, double E0, int *iters, double *E) {
    if (h->o.accel == STOKES_ACCEL_ANDERSON) return solve_anderson(h, rtol, E0, iters, E);
    if (h->o.accel == STOKES_ACCEL_GCR)
        return stream_ok(h->lev[0].g) ? solve_gcr_fused(h, rtol, E0, iters, E) : solve_gcr(h, rtol, E0, iters, E);
    return fused_ok(h) ? solve_uzawa_fused(h, rtol, E0, iters, E) : solve_uzawa(h, rtol, E0, iters, E);
}
// Anderson acceleration AA(m, beta) over the Uzawa map G (Alg. 5, PAPER.md:1502-1588,
// reading R26; the oracle's solve_anderson): per iteration one graph-replayed Uzawa step
// x^k -> G(x^k) with its energy residual (the stopping test, G(x^k) returned), then
// push (G_k, R_k, Gram row), the tiny constrained least squares, and the mixed update.
int solve_anderson(stokes_s *h, double rtol, double E0, int *iters, double *Eout) {
    ras_reset(h);
    int st = ensure_uzawa_graphs(h);
    if (st) return st;
    Level &F = h->lev[0];
    const LaunchCtx c = ctx(h);
    const int m = h->o.aa_depth, ns = m + 1;
    const size_t fb = field_doubles(F.g) * 8;
    // T = x^0 (its pressure mean = S_MSHIFT, from energy_now)
    CK(cudaMemcpyAsync(h->aat.f[0] - COL_OFF, F.vx[0] - COL_OFF, fb, cudaMemcpyDeviceToDevice, h->stream));
    CK(cudaMemcpyAsync(h->aat.f[1] - COL_OFF, F.vy[0] - COL_OFF, fb, cudaMemcpyDeviceToDevice, h->stream));
    CK(cudaMemcpyAsync(h->aat.f[2] - COL_OFF, h->pbuf[h->pcur] - COL_OFF, fb, cudaMemcpyDeviceToDevice, h->stream));
    CK(cudaMemcpyAsync(h->scal + S_AAMT, h->scal + S_MSHIFT, 8, cudaMemcpyDeviceToDevice, h->stream));
    const int nb = aa_blocks(F.g);
    const double inv_np = 1.0 / ((double)F.g.ncx * F.g.ncy);
    double E = E0;
    int k, status = STOKES_NOT_CONVERGED;
    for (k = 0; k < h->o.max_iter; ++k) {
        CK(cudaGraphLaunch(h->uzawa_exec[h->pcur], h->stream));  // G(x^k), E of it
        h->pcur ^= 1;
        h->launches += h->uzawa_kernels;
        if ((st = sync(h))) return st;
        E = h->hscal[S_E];
        record_E(h, k, E);
        if (!(E == E) || isinf(E) || E > 1e6 * E0) { status = STOKES_EDIVERGED; break; }
        if (E <= rtol) { status = STOKES_OK; break; }
        const int slot = k % ns, mk = k < m ? k : m;
        AAWin win;
        win.n = mk + 1;
        win.self = mk;
        for (int a = 0; a <= mk; ++a) {
            win.slot[a] = (k - mk + a) % ns;
            win.r[a] = h->aah.R[win.slot[a]];
        }
        const AAVec work{{F.vx[0], F.vy[0], h->pbuf[h->pcur]}};
        launch_aa_push(c, F.g, work, h->scal + S_MSHIFT, h->aat, h->scal + S_AAMT, h->aah.G[slot], h->aah.R[slot],
                       win, h->partials);
        launch_aa_solve(c, h->partials, nb, win, h->o.aa_beta, h->aaH, h->aacg, h->aacr);
        launch_aa_update(c, F.g, h->aah, ns, h->aacg, h->aacr, work, h->aat, h->partials);
        launch_finalize(c, h->partials, nb, 1, inv_np, h->scal + S_MSHIFT);  // lazy de-mean of x^{k+1}
        CK(cudaMemcpyAsync(h->scal + S_AAMT, h->scal + S_MSHIFT, 8, cudaMemcpyDeviceToDevice, h->stream));
    }
    if (k >= h->o.max_iter) k = h->o.max_iter - 1;
    *iters = k + 1;
    *Eout = E;
    return status;
}
// computational viscosity (1 - theta) eta_min + theta eta and its hierarchy
int set_theta(stokes_s *h, double theta) {
    Level &F = h->lev[0];
    const LaunchCtx c = ctx(h);
    launch_eta_blend(c, F.g, h->etab_user, h->etap_user, F.etab, F.etap,
                     reinterpret_cast<const unsigned long long *>(h->scal + S_ETAMIN), theta);
    return build_hierarchy(h);
}
// Viscosity rescaling: stages theta = 0, step, .. < 1 of theta_every
// iterations each (no stopping test: the staged systems are not the problem), warm-started
// from the previous stage; then theta = 1 (the caller's viscosity, restored exactly) to
// E <= rtol with the remaining iteration budget.  Same schedule as the oracle.
int solve_staged(stokes_s *h, double rtol, int *iters, double *Eout) {
    Level &F = h->lev[0];
    const LaunchCtx c = ctx(h);
    const int budget = h->o.max_iter;
    int used = 0, it = 0, st = 0, status = STOKES_OK;
    double E = 0.0, E0 = 0.0;
    const unsigned long long big = 0x7ff0000000000000ull;  // +inf
    CK(cudaMemcpyAsync(h->scal + S_ETAMIN, &big, 8, cudaMemcpyHostToDevice, h->stream));
    launch_eta_min(c, F.g, h->etab_user, h->etap_user, reinterpret_cast<unsigned long long *>(h->scal + S_ETAMIN));
    for (int k = 0;; ++k) {
        const double theta = k * h->o.theta_step;
        if (theta >= 1.0 || used >= budget) break;
        if ((st = set_theta(h, theta))) return st;
        if ((st = energy_now(h, &E0))) return st;
        h->o.max_iter = budget - used < h->o.theta_every ? budget - used : h->o.theta_every;
        h->hist_off = used;
        status = solve_inner(h, -1.0, E0, &it, &E);
        h->o.max_iter = budget;
        if (status < 0 && status != STOKES_EDIVERGED) return status;
        used += it;
        if (status == STOKES_EDIVERGED) break;
    }
    if ((st = set_theta(h, 1.0))) return st;
    if (status != STOKES_EDIVERGED && used < budget) {
        if ((st = energy_now(h, &E0))) return st;
        if (E0 <= rtol) {
            E = E0;
            status = STOKES_OK;
        } else {
            h->o.max_iter = budget - used;
            h->hist_off = used;
            status = solve_inner(h, rtol, E0, &it, &E);
            h->o.max_iter = budget;
            if (status < 0 && status != STOKES_EDIVERGED) return status;
            used += it;
        }
    } else if (status != STOKES_EDIVERGED) {
        status = STOKES_NOT_CONVERGED;
    }
    *iters = used;
    *Eout = E;
    return status;
}
}  // namespace sk
extern "C" {

// ---------------------------------------------------------------- per-step entry points
int stokes_smooth(stokes_t h, int level, const double *bx, const double *by, double *vx, double *vy, int nsweeps) {
    DEVICE_GUARD(h);
    if (!valid_level(h, level) || !bx || !by || !vx || !vy || nsweeps < 0) return STOKES_EINVAL;
    if (!h->have_eta) return STOKES_ESTATE;
    Level &L = h->lev[level];
    const LaunchCtx c = ctx(h);
    launch_in_vx_raw(c, L.g, bx, L.bx);
    launch_in_vy_raw(c, L.g, by, L.by);
    launch_in_velocity(c, L.g, vx, vy, L.vx[0], L.vy[0]);
    double *cx = L.vx[0], *cy = L.vy[0], *ox = L.vx[1], *oy = L.vy[1];
    ras_reset(h);
    smooth(h, level, cx, cy, ox, oy, rhs_arrays(L.bx, L.by), nsweeps, false, nsweeps);
    launch_out_vx(c, L.g, cx, vx);
    launch_out_vy(c, L.g, cy, vy);
    return sync(h);
}

int stokes_level_residual(stokes_t h, int level, const double *bx, const double *by, const double *vx,
                          const double *vy, double *rx, double *ry) {
    DEVICE_GUARD(h);
    if (!valid_level(h, level) || !bx || !by || !vx || !vy || !rx || !ry) return STOKES_EINVAL;
    if (!h->have_eta) return STOKES_ESTATE;
    Level &L = h->lev[level];
    const LaunchCtx c = ctx(h);
    launch_in_vx_raw(c, L.g, bx, L.bx);
    launch_in_vy_raw(c, L.g, by, L.by);
    launch_in_velocity(c, L.g, vx, vy, L.vx[0], L.vy[0]);
    launch_residual(c, L.g, L.etab, L.etap, L.vx[0], L.vy[0], rhs_arrays(L.bx, L.by), L.rx, L.ry);
    launch_out_vx(c, L.g, L.rx, rx);
    launch_out_vy(c, L.g, L.ry, ry);
    return sync(h);
}

int stokes_restrict(stokes_t h, int level, int kind, const double *fine, double *coarse) {
    DEVICE_GUARD(h);
    if (!valid_level(h, level) || level + 1 >= h->nlev || kind < 0 || kind > 3 || !fine || !coarse) return STOKES_EINVAL;
    Level &L = h->lev[level], &C = h->lev[level + 1];
    const LaunchCtx c = ctx(h);
    switch (kind) {
    case 0:
        launch_in_vx_raw(c, L.g, fine, L.rx);
        launch_restrict_vx(c, L.g, C.g, L.rx, C.rx);
        launch_out_vx(c, C.g, C.rx, coarse);
        break;
    case 1:
        launch_in_vy_raw(c, L.g, fine, L.ry);
        launch_restrict_vy(c, L.g, C.g, L.ry, C.ry);
        launch_out_vy(c, C.g, C.ry, coarse);
        break;
    case 2:
        launch_in_p(c, L.g, fine, L.rx);
        launch_restrict_p(c, L.g, C.g, L.rx, C.rx);
        launch_out_p(c, C.g, C.rx, coarse, nullptr);
        break;
    default:
        launch_in_b(c, L.g, fine, L.rx);
        launch_restrict_b(c, L.g, C.g, L.rx, C.rx);
        launch_out_b(c, C.g, C.rx, coarse);
        break;
    }
    return sync(h);
}

int stokes_prolong(stokes_t h, int level, const double *ex, const double *ey, double *vx, double *vy) {
    DEVICE_GUARD(h);
    if (!valid_level(h, level) || level + 1 >= h->nlev || !ex || !ey || !vx || !vy) return STOKES_EINVAL;
    Level &L = h->lev[level], &C = h->lev[level + 1];
    const LaunchCtx c = ctx(h);
    launch_in_velocity(c, C.g, ex, ey, C.vx[0], C.vy[0]);
    launch_in_velocity(c, L.g, vx, vy, L.vx[0], L.vy[0]);
    launch_prolong(c, L.g, C.g, C.vx[0], C.vy[0], L.vx[0], L.vy[0]);
    launch_out_vx(c, L.g, L.vx[0], vx);
    launch_out_vy(c, L.g, L.vy[0], vy);
    return sync(h);
}

int stokes_get_viscosity(stokes_t h, int level, double *eta_b, double *eta_p) {
    DEVICE_GUARD(h);
    if (!valid_level(h, level) || !eta_b || !eta_p) return STOKES_EINVAL;
    if (!h->have_eta) return STOKES_ESTATE;
    Level &L = h->lev[level];
    const LaunchCtx c = ctx(h);
    launch_out_b(c, L.g, L.etab, eta_b);
    launch_out_p(c, L.g, L.etap, eta_p, nullptr);
    return sync(h);
}

int stokes_coarse_solve(stokes_t h, const double *bx, const double *by, double *vx, double *vy) {
    DEVICE_GUARD(h);
    if (!h || h->dist || !bx || !by || !vx || !vy) return STOKES_EINVAL;
    if (!h->have_eta) return STOKES_ESTATE;
    if (h->nc == 0) return STOKES_EINVAL;
    Level &C = h->lev[h->nlev - 1];
    const LaunchCtx c = ctx(h);
    launch_in_vx_raw(c, C.g, bx, C.bx);
    launch_in_vy_raw(c, C.g, by, C.by);
    launch_coarse_solve(c, C.g, h->Minv, C.bx, C.by, C.vx[0], C.vy[0]);
    launch_out_vx(c, C.g, C.vx[0], vx);
    launch_out_vy(c, C.g, C.vy[0], vy);
    return sync(h);
}

int stokes_launch_count(stokes_t h, long long *count, int reset) {
    DEVICE_GUARD(h);
    if (!h || !count) return STOKES_EINVAL;
    if (h->dist) {
        *count = dist_launches(h->dist, reset);
        return STOKES_OK;
    }
    *count = h->launches;
    if (reset) h->launches = 0;
    return STOKES_OK;
}

int stokes_time_kernel(stokes_t h, int kernel, int reps, double *avg_ms, double *bytes) {
    DEVICE_GUARD(h);
    if (!h || h->dist || !avg_ms || !bytes || reps < 1) return STOKES_EINVAL;
    if (!h->have_eta || !h->have_rho) return STOKES_ESTATE;
    Level &F = h->lev[0];
    const GridL &g = F.g;
    const LaunchCtx c = ctx(h);
    const double cells = (double)g.ncx * g.ncy;
    auto run = [&](void) {
        switch (kernel) {
        case 0: launch_jacobi(c, g, F.etab, F.etap, F.vx[0], F.vy[0], F.vx[1], F.vy[1], rhs_fine(h), h->o.omega_v, false); break;
        case 1: state_energy(h, nullptr, nullptr, nullptr); break;
        case 2:
            if (h->nlev > 1 && jacobi2_ok(g)) {
                launch_residual_restrict(c, g, h->lev[1].g, F.etab, F.etap, F.vx[0], F.vy[0], rhs_fine(h),
                                         h->lev[1].bx, h->lev[1].by);
            } else {
                launch_residual(c, g, F.etab, F.etap, F.vx[0], F.vy[0], rhs_fine(h), F.rx, F.ry);
                if (h->nlev > 1) launch_restrict_vel(c, g, h->lev[1].g, F.rx, F.ry, h->lev[1].bx, h->lev[1].by);
            }
            break;
        case 3: if (h->nlev > 1) launch_prolong(c, g, h->lev[1].g, h->lev[1].vx[0], h->lev[1].vy[0], F.vx[1], F.vy[1]); break;
        case 4:
            if (stream_ok(g))
                launch_uzawa_energy(c, g, F.etab, F.etap, F.vx[0], F.vy[0], h->pbuf[h->pcur], h->pbuf[1 - h->pcur],
                                    h->rho, h->gx, h->gy, h->o.alpha_p, h->scal + S_ZERO, nullptr, nullptr, nullptr,
                                    h->partials);
            else
                launch_pupdate(c, g, F.etap, F.vx[0], F.vy[0], h->pbuf[h->pcur], h->pbuf[1 - h->pcur], h->o.alpha_p,
                               h->scal + S_ZERO, h->partials);
            break;
        case 5:
            if (jacobi2_ok(g)) launch_rbgs_stream(c, g, F.etab, F.etap, F.vx[0], F.vy[0], F.vx[1], F.vy[1], rhs_fine(h), h->o.omega_v);
            else launch_rbgs(c, g, F.etab, F.etap, F.vx[1], F.vy[1], rhs_fine(h), h->o.omega_v);
            break;
        case 7: launch_jacobi2(c, g, F.etab, F.etap, F.vx[0], F.vy[0], F.vx[1], F.vy[1], rhs_fine(h), h->o.omega_v); break;
        case 8: {
            RasArgs a;
            const RhsArgs r = rhs_fine(h);
            a.vx = F.vx[0];
            a.vy = F.vy[0];
            a.etap = F.etap;
            a.etab = F.etab;
            a.f4 = r.p;
            a.f5 = r.rho;
            a.vxo = F.vx[1];
            a.vyo = F.vy[1];
            a.omega = h->o.omega_v;
            a.gx = r.gx;
            a.gy = r.gy;
            a.T = h->o.ras_tile;
            a.Tin = h->o.ras_inner;
            a.seed = h->o.ras_seed;
            launch_ras_outer(c, g, a, h->scal + S_ITER, 0, true);
            break;
        }
        case 9:
            launch_jacobi_jju(c, g, F.etab, F.etap, F.vx[0], F.vy[0], F.vx[1], F.vy[1], h->pbuf[h->pcur],
                              h->pbuf[1 - h->pcur], h->rho, h->gx, h->gy, h->o.alpha_p, h->scal + S_ZERO,
                              h->o.omega_v, h->partials);
            break;
        default:
            launch_jacobi_uzawa(c, g, F.etab, F.etap, F.vx[0], F.vy[0], F.vx[1], F.vy[1], h->pbuf[h->pcur],
                                h->pbuf[1 - h->pcur], h->rho, h->gx, h->gy, h->o.alpha_p, h->scal + S_ZERO,
                                h->o.omega_v, h->partials);
            break;
        }
    };
    // algorithmic bytes per launch: 8 B per value read or written
    // 0 Jacobi: read vx,vy,eta_p,eta_b,p,rho + write vx,vy; 1 energy: read 6; 2 residual (read 6,
    // write 2) + restriction (read 2 fine, write 1/2); 3 prolongation (read/write 2 + 1/2 coarse);
    // 4 fused Uzawa pressure step + energy: read 6, write p; 5 RBGS (4 phases, fused bytes);
    // 6 Uzawa step + energy + first Jacobi sweep of the next V-cycle: read 6, write p, vx, vy;
    // 7 two Jacobi sweeps in one pass: read 6, write 2; 8 one RAS outer iteration (T_inner
    // sweeps in shared memory): read 6, write 2; 9 the last post-smoothing sweep + Uzawa step +
    // energy + first sweep of the next V-cycle (k_jju): read 6, write p, vx, vy
    double per_cell[10] = {64.0, 48.0, 64.0 + 16.0 + 4.0, 32.0 + 4.0, 56.0, 64.0, 72.0, 64.0, 64.0, 72.0};
    if (h->nlev > 1 && jacobi2_ok(g)) per_cell[2] = 48.0 + 4.0;  // fused: the residual stays on chip
    // RBGS: one streamed pass on a single domain (read 6 + write 2), else two passes (read 6 + write 1 each)
    if (jacobi2_ok(g) && !(g.bN && g.bS && g.bW && g.bE && rbgs1_enabled())) per_cell[5] = 2 * 56.0;
    if (kernel < 0 || kernel > 9) return STOKES_EINVAL;
    if ((kernel == 6 && !stream_ok(g)) || (kernel == 7 && !jacobi2_ok(g)) || (kernel == 9 && !jju_ok(g)))
        return STOKES_EINVAL;
    *bytes = per_cell[kernel] * cells;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    run();
    run();
    CK(cudaEventRecord(e0, h->stream));
    for (int r = 0; r < reps; ++r) run();
    CK(cudaEventRecord(e1, h->stream));
    CK(cudaEventSynchronize(e1));
    CKL();
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *avg_ms = ms / reps;
    return STOKES_OK;
}

const char *stokes_strerror(int s) {
    switch (s) {
    case STOKES_OK: return "ok";
    case STOKES_NOT_CONVERGED: return "not converged (max_iter reached)";
    case STOKES_EINVAL: return "invalid argument";
    case STOKES_ENOMEM: return "out of device memory / workspace too small";
    case STOKES_ECUDA: return "CUDA error";
    case STOKES_ENCCL: return "NCCL error";
    case STOKES_EDIVERGED: return "diverged";
    case STOKES_ESTATE: return "call order: set_viscosity / set_density first";
    default: return "unknown status";
    }
}
const char *stokes_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
