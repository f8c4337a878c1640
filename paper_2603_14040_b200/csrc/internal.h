// Internal declarations of libstokes_b200 (not part of the ABI).
//
// Data layout in HBM: every staggered field of a level is one FP64 array
// on the paper's padded index space (ncy+2) x (ncx+2) (basic / boundary
// B / ghost G nodes), row pitch P doubles (multiple of 32 = 256 B), element (i, j) at
// base[i * P + j].  base = allocation + P + COL_OFF so that interior column 1 is 256-B
// aligned: a warp reading columns 1..32 of a row touches exactly two 128-B lines.  Rows -1
// and ncy+2 and columns -1 and ncx+2 also exist: the second halo ring of decomposed tiles.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/stokes.h"

#define COL_OFF 31

struct GridL {          // one multigrid level, passed by value to kernels
    int ncx, ncy, P;    // cells in x / y, row pitch (doubles)
    double dx, dy;
    double idx, idy;    // 1/dx, 1/dy
    double idx2, idy2;  // 1/dx^2, 1/dy^2
    double idxdy;       // 1/(dx dy)
    double idx2x2, idy2x2;  // 2/dx^2, 2/dy^2
    double sW, sE, sN, sS;  // mirror signs: +1 free slip, -1 no slip
    // 2D domain decomposition: a level may be one tile of the global grid.
    // bX = 1: side X is a global boundary (mirrors / walls); 0: a halo filled
    // from the neighbouring tile.  Single-domain levels have all four set.
    int bN, bS, bW, bE;
    int nvxj;  // last vx unknown column: ncx-1 if bE (east wall) else ncx (the tile's east faces)
    int nvyi;  // last vy unknown row:    ncy-1 if bS else ncy
    int par;   // (global row + column offset of the tile) & 1: red-black colour parity (R11)
};

// first call on the current device (per-device one-time setup, e.g. cudaFuncSetAttribute of
// the > 48 KB dynamic shared memory kernels: the attribute is per device); thread-safe
bool first_on_device(unsigned long long *mask);

__host__ __device__ inline size_t at(const GridL &g, int i, int j) { return (size_t)i * (size_t)g.P + (size_t)j; }

// launch bookkeeping shared by all launchers
struct LaunchCtx {
    cudaStream_t stream;
    long long *counter;  // incremented per kernel launch (host side)
};

// ---------------------------------------------------------------- kernels.cu launchers
// RHS modes of the smoother / residual kernels
enum { RHS_ARRAYS = 0, RHS_FINE = 1 };  // b from arrays (bx, by) / b = f - G p from (rho, p)

struct RhsArgs {
    int mode;
    const double *bx, *by;          // RHS_ARRAYS
    const double *p, *rho;          // RHS_FINE
    double gx, gy;
};

void launch_jacobi(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, const double *vxi,
                   const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs, double omega, bool zero_in);
// n (<= 8) damped-Jacobi sweeps of a single-domain level with array right-hand sides in ONE
// launch (tiles staged in shared memory; k_jacobi's arithmetic); false: not applicable
// ex / ey (coarse level gc): the post-smoothing's input is v + P e (the prolongation applied
// while staging) -- prolongation and post-smoothing in one launch
bool launch_jacobi_tile(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                        const double *vxi, const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs,
                        double omega, int n, bool zero_in, const GridL *gc = nullptr, const double *ex = nullptr,
                        const double *ey = nullptr);
void launch_rbgs(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, double *vx, double *vy,
                 const RhsArgs &rhs, double omega);
void launch_residual(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, const double *vx,
                     const double *vy, const RhsArgs &rhs, double *rx, double *ry);
void launch_restrict_vel(const LaunchCtx &c, const GridL &gf, const GridL &gc, const double *rx, const double *ry,
                         double *bxc, double *byc);
void launch_restrict_b(const LaunchCtx &c, const GridL &gf, const GridL &gc, const double *f, double *cc);
void launch_restrict_p(const LaunchCtx &c, const GridL &gf, const GridL &gc, const double *f, double *cc);
void launch_restrict_vx(const LaunchCtx &c, const GridL &gf, const GridL &gc, const double *f, double *cc);
void launch_restrict_vy(const LaunchCtx &c, const GridL &gf, const GridL &gc, const double *f, double *cc);
void launch_prolong(const LaunchCtx &c, const GridL &gf, const GridL &gc, const double *exc, const double *eyc,
                    double *vx, double *vy);
// coarse tail of the V-cycle in one CTA (levels 0..nl-1 of the tail, the last one solved by
// the explicit inverse): lev[l].(ax, ay) = V-cycle result with zero initial guess on
// L v = (bx, by); (sx, sy, rx, ry) scratch.  Single-domain Jacobi levels only.
#define TAIL_MAXL 12
struct TailLevel {
    GridL g;
    const double *etab, *etap;
    double *bx, *by;  // level 0: the caller's right-hand side (read only); below: restricted residuals
    double *ax, *ay, *sx, *sy, *rx, *ry;
    int nu;
};
struct TailArgs {
    TailLevel lev[TAIL_MAXL];
    int nl;
};
void launch_vtail(const LaunchCtx &c, const TailArgs &a, const double *Minv, int n, double omega);
// the same stages over a cooperative grid (one CTA per SM, grid-wide barriers); -1 if the launch failed
int launch_vtail_coop(const LaunchCtx &c, const TailArgs &a, const double *Minv, int n, double omega);
// full saddle residual + energy partial sums (Sv, Sp) per block; writes r arrays if non-null.
// force_only: Sv of f (the normaliser Sf).  Returns the number of partial blocks.
int energy_blocks(const GridL &g);
void launch_energy(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, const double *vx,
                   const double *vy, const double *p, const double *rho, double gx, double gy, double *rx,
                   double *ry, double *rp, double *partials, bool force_only);
void launch_energy_vec(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, const double *rx,
                       const double *ry, const double *rp, double *partials);
void launch_make_rhs(const LaunchCtx &c, const GridL &g, const RhsArgs &rhs, double *bx, double *by);
// p <- (p - *mshift) + sign * alpha * eta_p * (-D v); partial sums of the new p per block
int pupdate_blocks(const GridL &g);
void launch_pupdate(const LaunchCtx &c, const GridL &g, const double *etap, const double *vx, const double *vy,
                    const double *pin, double *pout, double alpha_signed, const double *mshift, double *partials);
void launch_uzawa_final(const LaunchCtx &c, const double *partials, int nblocks, const double *Sf, double inv_np,
                        double *out, double *mean);

// ---------------------------------------------------------------- stream.cu (TMA row streaming)
bool stream_ok(const GridL &g);   // level wide enough for the 256-column streaming CTAs
int stream_blocks(const GridL &g);
void launch_jacobi_stream(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                          const double *vxi, const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs,
                          double omega);
void launch_residual_stream(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                            const double *vx, const double *vy, const RhsArgs &rhs, double *rx, double *ry);
// fused Uzawa pressure step + energy residual; partials = 3 per CTA (Sv, Sp, sum p')
// two Jacobi sweeps in one pass (single-domain levels with jacobi2_ok)
bool jacobi2_ok(const GridL &g);
bool rbgs1_enabled();  // one-pass RBGS on single domains (STOKES_RBGS1=0 disables it)
// the last post-smoothing Jacobi sweep + the fused Uzawa step (JacobiUzawaOp) in one pass
// (k_jju, single domains; STOKES_JJU=0 disables it); partials: 3 per block, jju_blocks(g)
bool jju_ok(const GridL &g);
// the last pre-smoothing two-sweep pass fused with the residual and its restriction (k_j2rr;
// single domains; STOKES_J2RR=0 disables it): vxo, vyo = the pair's output, bxc, byc = b^H
bool j2rr_ok(const GridL &g);
void launch_j2rr(const LaunchCtx &c, const GridL &g, const GridL &gc, const double *etab, const double *etap,
                 const double *vxi, const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs, double omega,
                 double *bxc, double *byc);
int jju_blocks(const GridL &g);
void launch_jacobi_jju(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                       const double *vxi, const double *vyi, double *vxo, double *vyo, const double *pin, double *pout,
                       const double *rho, double gx, double gy, double alpha_signed, const double *mshift,
                       double omega, double *partials);
void launch_jacobi2(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, const double *vxi,
                    const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs, double omega);
// split passes of decomposed tiles (halo exchange overlapped with the interior): part 0 = the
// two layers of unknowns next to every non-global side, part 1 = the rest of the level
void launch_jacobi2_part(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                         const double *vxi, const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs,
                         double omega, int part);
void launch_jacobi_stream_part(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                               const double *vxi, const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs,
                               double omega, int part);
// Anderson acceleration (aa.cu): ring of AA_MAXS history slots of three padded fields
constexpr int AA_MAXS = 16;
struct AAVec {
    double *f[3];
};
struct AAWin {  // the history window, oldest -> newest; member `self` is the new slot
    int n, self;
    int slot[AA_MAXS];
    AAVec r[AA_MAXS];
};
struct AAHist {
    AAVec G[AA_MAXS], R[AA_MAXS];
};
int aa_blocks(const GridL &g);
void launch_aa_push(const LaunchCtx &c, const GridL &g, const AAVec &work, const double *ms_g, const AAVec &T,
                    const double *ms_t, const AAVec &Gk, const AAVec &Rk, const AAWin &win, double *partials);
void launch_aa_solve(const LaunchCtx &c, const double *partials, int nblocks, const AAWin &win, double beta,
                     double *H, double *cg, double *cr);
void launch_aa_update(const LaunchCtx &c, const GridL &g, const AAHist &hist, int ns, const double *cg,
                      const double *cr, const AAVec &work, const AAVec &T, double *partials);
// RAS-type temporal blocking (ras.cu): one outer iteration, (vx, vy) -> (vxo, vyo)
struct RasArgs {
    const double *vx, *vy, *etap, *etab, *f4, *f5;  // f4, f5 = p, rho (fine) | bx, by
    double *vxo, *vyo;
    double omega, gx, gy;
    int T, Tin;
    uint64_t seed;
};
void launch_ras_outer(const LaunchCtx &c, const GridL &g, const RasArgs &a, const double *iter, int c_draw,
                      bool fine);
void launch_iter_inc(const LaunchCtx &c, double *k);
int ras_max_tile();
// viscosity rescaling: min over the valid nodes of both caller fields
// into *emin (as the bit pattern of a positive double, atomicMin), then the blend
void launch_eta_min(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                    unsigned long long *emin);
void launch_eta_blend(const LaunchCtx &c, const GridL &g, const double *ebu, const double *epu, double *etab,
                      double *etap, const unsigned long long *emin, double theta);
// lithostatic pressure, user P layout
void launch_lithostatic(const LaunchCtx &c, const GridL &g, const double *rho, double gy, double *p);
// RBGS sweep as two streamed passes, out of place (jacobi2_ok levels): (vxi, vyi) -> (vxo, vyo)
void launch_rbgs_stream(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                        const double *vxi, const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs,
                        double omega);
// fine residual fused with the velocity restriction to the next level (jacobi2_ok levels)
void launch_residual_restrict(const LaunchCtx &c, const GridL &g, const GridL &gc, const double *etab,
                              const double *etap, const double *vx, const double *vy, const RhsArgs &rhs, double *bxc,
                              double *byc);
// last Uzawa step fused into the next V-cycle's first Jacobi sweep (3 partials per CTA)
void launch_jacobi_uzawa(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                         const double *vxi, const double *vyi, double *vxo, double *vyo, const double *pin,
                         double *pout, const double *rho, double gx, double gy, double alpha_signed,
                         const double *mshift, double omega, double *partials);
// pout == nullptr: energy only (p' = pin - *mshift is not stored)
void launch_uzawa_energy(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                         const double *vx, const double *vy, const double *pin, double *pout, const double *rho,
                         double gx, double gy, double alpha_signed, const double *mshift, double *rx, double *ry,
                         double *rp, double *partials);
// out[k] = scale * sum_b partials[b * ncomp + k], deterministic fixed-order tree
void launch_finalize(const LaunchCtx &c, const double *partials, int nblocks, int ncomp, double scale, double *out);
// energy: E = sqrt((S[0] + S[1]) / Sf[0]) -> out[0]; also copies S to out[1..2]
void launch_energy_final(const LaunchCtx &c, const double *partials, int nblocks, const double *Sf, double *out);

// layout conversion (user <-> padded)
void launch_in_velocity(const LaunchCtx &c, const GridL &g, const double *ux, const double *uy, double *vx,
                        double *vy);
void launch_in_p(const LaunchCtx &c, const GridL &g, const double *u, double *a);
void launch_in_b(const LaunchCtx &c, const GridL &g, const double *u, double *a);
void launch_in_vx_raw(const LaunchCtx &c, const GridL &g, const double *u, double *a);
void launch_in_vy_raw(const LaunchCtx &c, const GridL &g, const double *u, double *a);
void launch_out_vx(const LaunchCtx &c, const GridL &g, const double *a, double *u);
void launch_out_vy(const LaunchCtx &c, const GridL &g, const double *a, double *u);
void launch_out_p(const LaunchCtx &c, const GridL &g, const double *a, double *u, const double *shift);
void launch_out_b(const LaunchCtx &c, const GridL &g, const double *a, double *u);
void launch_apply(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, const double *vx,
                  const double *vy, const double *p, double *ax, double *ay, double *ap);
void launch_count_nonpos(const LaunchCtx &c, const double *a, size_t n, int *count);

// coarsest level: assemble -L_c (n x n, mirror relations folded), invert, apply
void launch_coarse_assemble(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, double *M);
// Minv holds -L_c on entry and its inverse on exit; work must hold n x 2n doubles
void launch_coarse_invert(const LaunchCtx &c, double *work, double *Minv, int n, int *fail);
void launch_coarse_solve(const LaunchCtx &c, const GridL &g, const double *Minv, const double *bx,
                         const double *by, double *vx, double *vy);

// GCR vector kernels (vectors = (x, y, p) padded triples on the fine level)
int dot_blocks(const GridL &g);
void launch_dots(const LaunchCtx &c, const GridL &g, const double *const *a, const double *const *b, int nd,
                 double *partials);
void launch_axpy3(const LaunchCtx &c, const GridL &g, const double *coef, int coef_index, double coef_sign,
                  const double *xx, const double *xy, const double *xp, double *yx, double *yy, double *yp);
void launch_scale3(const LaunchCtx &c, const GridL &g, const double *coef, int invert_sqrt, double *x,
                   double *y, double *p);
void launch_precond_p(const LaunchCtx &c, const GridL &g, const double *etap, const double *zx, const double *zy,
                      const double *rp, double alpha, double *zp, double *partials);
void launch_sub_mean(const LaunchCtx &c, const GridL &g, const double *mean, double *p);
void launch_apply_padded(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                         const double *vx, const double *vy, const double *p, double *ax, double *ay, double *ap);
void launch_refresh_mirrors(const LaunchCtx &c, const GridL &g, double *vx, double *vy);
void launch_energy_weights(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, double *ewx,
                           double *ewy, double *ewp);

// fused GCR kernels (stream.cu: preconditioner + apply; gcr.cu: flat MGS / update)
void launch_precond_apply(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                          const double *zx, const double *zy, const double *rp, double alpha, double *zp, double *wx,
                          double *wy, double *wp, const double *const *w0, const double *rx, const double *ry,
                          double *partials);
int gcr_flat_blocks(size_t nfield);  // CTAs (= partials) of the flat GCR kernels for fields of nfield doubles
// z == nullptr: the MGS z update is deferred (gamma stored to *gout) and done by launch_gcr_update
// (z -= gamma_j z_j for j = 0 .. nz-1, the same operations in the same order)
void launch_mgs_step(const LaunchCtx &c, const double *pin, int nbin, int ncin, int kin, double *const *w,
                     double *const *z, const double *const *wj, const double *const *zj, const double *const *nxt,
                     const double *const *r, size_t nfield, double *pout, double *gout = nullptr);
void launch_gcr_update(const LaunchCtx &c, const double *pin, int nbin, double *const *w, double *const *z,
                       double *const *x, double *const *r, const double *const *ew, size_t nfield, double *pout,
                       const double *gammas = nullptr, int nz = 0, double *const (*zj)[3] = nullptr);
void launch_gcr_final(const LaunchCtx &c, const double *pupd, int nbu, const double *pnorm, int nbn,
                      const double *Sf, double *E, double *nu2, double *rr);

// ---------------------------------------------------------------- decomposition helpers
struct StripList {  // host-side list of strided strip copies (any length)
    double *dst[512];
    const double *src[512];
    int n[512], dstride[512], sstride[512];
    int count;
};
void launch_strips(const LaunchCtx &c, const StripList &l);
void launch_rbgs_phase(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, double *vx,
                       double *vy, const RhsArgs &rhs, double omega, int comp, int colour);
// out = (E, Sv, Sp) from the tiles' local (Sv, Sp, sum p); mean written to each mshift
void launch_dist_mean(const LaunchCtx &c, const double *base, int nseg, int nb, size_t stride, double inv_np,
                      double *out);
void launch_dist_final(const LaunchCtx &c, const double *const *loc, int nloc, const double *Sf, double inv_np,
                       double *out, double *const *mshift, int nm);
