// Hand-written FP64 CUDA kernels of the matrix-free multigrid Stokes solve (sm_100a).
//
// Every kernel cites the passage of PAPER.md it implements; the readings R1..R23 are
// listed in DESIGN.md §3.  No tensor cores: nothing here is a dense contraction
// (DESIGN.md §6); every hot kernel is HBM-bandwidth bound and is measured against the
// measured copy bandwidth (MEASURED_PEAKS.json).
//
// Index space of a level: padded (ncy+2) x (ncx+2), row pitch g.P (internal.h).
//   vx unknowns i in [1,ncy], j in [1,ncx-1]; walls j = 0, ncx; mirrors i = 0, ncy+1
//   vy unknowns i in [1,ncy-1], j in [1,ncx]; walls i = 0, ncy; mirrors j = 0, ncx+1
//   P  unknowns i in [1,ncy], j in [1,ncx];  basic nodes i in [0,ncy], j in [0,ncx]
// (Listing loop bounds PAPER.md:2352-2353, reading R1.)  Wall entries are zero in every
// velocity buffer from allocation on and are never written; every kernel that writes a
// velocity unknown next to a boundary also writes its mirror (reading R5: "refresh the
// mirrors after every update" == "mirror = partner's current value").
#include <math.h>

#include <cooperative_groups.h>

#include "internal.h"

namespace {

constexpr int BX = 32, BY = 8;  // 256-thread tiles: one warp spans 32 consecutive columns

inline dim3 cell_grid(const GridL &g) { return dim3((g.ncx + BX - 1) / BX, (g.ncy + BY - 1) / BY); }

// ------------------------------------------------------------------ stencil pieces
struct ArrayAcc {  // plain global loads
    const double *__restrict__ a;
    size_t P;
    __device__ __forceinline__ double operator()(int i, int j) const { return a[(size_t)i * P + j]; }
};

// x-momentum row at vx(i,j): Listing vx_op_point -- coefficients verbatim.
template <class VX, class VY>
__device__ __forceinline__ double lx_row(const GridL &g, const double *__restrict__ etab,
                                         const double *__restrict__ etap, const VX &vx, const VY &vy, int i, int j) {
    const double etaA = etap[at(g, i, j)], etaB = etap[at(g, i, j + 1)];
    const double eta1 = etab[at(g, i - 1, j)], eta2 = etab[at(g, i, j)];
    const double vx3 = -(eta1 + eta2) * g.idy2 - 2.0 * (etaA + etaB) * g.idx2;
    return 2.0 * etaA * g.idx2 * vx(i, j - 1) + eta1 * g.idy2 * vx(i - 1, j) + vx3 * vx(i, j) +
           eta2 * g.idy2 * vx(i + 1, j) + 2.0 * etaB * g.idx2 * vx(i, j + 1) +
           g.idxdy * (eta1 * (vy(i - 1, j) - vy(i - 1, j + 1)) + eta2 * (vy(i, j + 1) - vy(i, j)));
}
// y-momentum row at vy(i,j) (reading R2, "the same procedure"): the mirror of
// the Listing, from sigma'_yy at P nodes and sigma'_xy at basic nodes.
template <class VX, class VY>
__device__ __forceinline__ double ly_row(const GridL &g, const double *__restrict__ etab,
                                         const double *__restrict__ etap, const VX &vx, const VY &vy, int i, int j) {
    const double etaN = etap[at(g, i, j)], etaS = etap[at(g, i + 1, j)];
    const double etaW = etab[at(g, i, j - 1)], etaE = etab[at(g, i, j)];
    const double vy3 = -2.0 * (etaN + etaS) * g.idy2 - (etaW + etaE) * g.idx2;
    return 2.0 * etaS * g.idy2 * vy(i + 1, j) + 2.0 * etaN * g.idy2 * vy(i - 1, j) + etaE * g.idx2 * vy(i, j + 1) +
           etaW * g.idx2 * vy(i, j - 1) + vy3 * vy(i, j) +
           g.idxdy * (etaE * (vx(i + 1, j) - vx(i, j)) - etaW * (vx(i + 1, j - 1) - vx(i, j - 1)));
}
// a_ii of the BC-folded operator (reading R5; Eq. jacobi_update, diag(-L) PAPER.md:1615)
__device__ __forceinline__ double lx_diag(const GridL &g, const double *__restrict__ etab,
                                          const double *__restrict__ etap, int i, int j) {
    const double eta1 = etab[at(g, i - 1, j)], eta2 = etab[at(g, i, j)];
    double a = -(eta1 + eta2) * g.idy2 - 2.0 * (etap[at(g, i, j)] + etap[at(g, i, j + 1)]) * g.idx2;
    if (i == 1 && g.bN) a += g.sN * eta1 * g.idy2;
    if (i == g.ncy && g.bS) a += g.sS * eta2 * g.idy2;
    return a;
}
__device__ __forceinline__ double ly_diag(const GridL &g, const double *__restrict__ etab,
                                          const double *__restrict__ etap, int i, int j) {
    const double etaW = etab[at(g, i, j - 1)], etaE = etab[at(g, i, j)];
    double a = -2.0 * (etap[at(g, i, j)] + etap[at(g, i + 1, j)]) * g.idy2 - (etaW + etaE) * g.idx2;
    if (j == 1 && g.bW) a += g.sW * etaW * g.idx2;
    if (j == g.ncx && g.bE) a += g.sE * etaE * g.idx2;
    return a;
}
// right-hand side of the velocity equation at a vx / vy node:
//   RHS_ARRAYS: b;  RHS_FINE: f - G p with f = -g rho (reading R4/R23), G p = -grad_h p
__device__ __forceinline__ double rhs_x(const GridL &g, const RhsArgs &r, int i, int j) {
    if (r.mode == RHS_ARRAYS) return r.bx[at(g, i, j)];
    double f = 0.0;
    if (r.gx != 0.0) f = -r.gx * (0.5 * (r.rho[at(g, i - 1, j)] + r.rho[at(g, i, j)]));
    return f - (r.p[at(g, i, j)] - r.p[at(g, i, j + 1)]) * g.idx;
}
__device__ __forceinline__ double rhs_y(const GridL &g, const RhsArgs &r, int i, int j) {
    if (r.mode == RHS_ARRAYS) return r.by[at(g, i, j)];
    double f = 0.0;
    if (r.gy != 0.0) f = -r.gy * (0.5 * (r.rho[at(g, i, j - 1)] + r.rho[at(g, i, j)]));
    return f - (r.p[at(g, i, j)] - r.p[at(g, i + 1, j)]) * g.idy;
}

// deterministic block sum (fixed xor-shuffle tree + fixed warp order); result valid in thread 0
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *sh) {
    const int t = threadIdx.x + threadIdx.y * blockDim.x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((t & 31) == 0) sh[t >> 5] = v;
    __syncthreads();
    if (t < 32) {
        v = (t < NT / 32) ? sh[t] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    __syncthreads();
    return v;
}

// ------------------------------------------------------------------ smoother (a4)
// Damped Jacobi, Eq. damped_jacobi: v <- v + omega (b - L v)_i / a_ii,
// reads only the old iterate (ping-pong buffers).  zero_in: the old iterate is 0 (first
// sweep of a coarse correction), so v_in is not read.
// 1/a by the FP64 MUFU seed and two Newton steps (<= 1 ulp; as the streamed kernels' rcp)
__device__ __forceinline__ double rcp_nr(double a) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    r = r * fma(-a, r, 2.0);
    return r * fma(-a, r, 2.0);
}
template <bool ZERO, bool RCP = false>  // RCP: multiply by rcp_nr(a_ii) instead of dividing
__device__ __forceinline__ void jacobi_pt(const GridL &g, const double *__restrict__ etab,
                                          const double *__restrict__ etap, const double *__restrict__ vxi,
                                          const double *__restrict__ vyi, double *__restrict__ vxo,
                                          double *__restrict__ vyo, const RhsArgs &rhs, double omega, int i, int j) {
    const ArrayAcc ax{vxi, (size_t)g.P}, ay{vyi, (size_t)g.P};
    if (j <= g.nvxj) {
        const double a = lx_diag(g, etab, etap, i, j);
        const double b = rhs_x(g, rhs, i, j);
        double vn;
        if (RCP) vn = ZERO ? omega * b * rcp_nr(a) : ax(i, j) + omega * (b - lx_row(g, etab, etap, ax, ay, i, j)) * rcp_nr(a);
        else if (ZERO) vn = omega * b / a;
        else vn = ax(i, j) + omega * (b - lx_row(g, etab, etap, ax, ay, i, j)) / a;
        vxo[at(g, i, j)] = vn;
        if (i == 1 && g.bN) vxo[at(g, 0, j)] = g.sN * vn;
        if (i == g.ncy && g.bS) vxo[at(g, g.ncy + 1, j)] = g.sS * vn;
    }
    if (i <= g.nvyi) {
        const double a = ly_diag(g, etab, etap, i, j);
        const double b = rhs_y(g, rhs, i, j);
        double vn;
        if (RCP) vn = ZERO ? omega * b * rcp_nr(a) : ay(i, j) + omega * (b - ly_row(g, etab, etap, ax, ay, i, j)) * rcp_nr(a);
        else if (ZERO) vn = omega * b / a;
        else vn = ay(i, j) + omega * (b - ly_row(g, etab, etap, ax, ay, i, j)) / a;
        vyo[at(g, i, j)] = vn;
        if (j == 1 && g.bW) vyo[at(g, i, 0)] = g.sW * vn;
        if (j == g.ncx && g.bE) vyo[at(g, i, g.ncx + 1)] = g.sE * vn;
    }
}
template <bool ZERO>
__global__ void __launch_bounds__(BX *BY) k_jacobi(GridL g, const double *__restrict__ etab,
                                                   const double *__restrict__ etap, const double *__restrict__ vxi,
                                                   const double *__restrict__ vyi, double *__restrict__ vxo,
                                                   double *__restrict__ vyo, RhsArgs rhs, double omega) {
    const int j = blockIdx.x * BX + threadIdx.x + 1;
    const int i = blockIdx.y * BY + threadIdx.y + 1;
    if (i > g.ncy || j > g.ncx) return;
    jacobi_pt<ZERO>(g, etab, etap, vxi, vyi, vxo, vyo, rhs, omega, i, j);
}

// ---- n damped-Jacobi sweeps of a small level in ONE launch (temporal blocking in shared memory)
// The coarse levels between the one-CTA tail and the streamed levels are latency-bound: a sweep
// there is a few microseconds of launch and pipeline fill for little work.  Here a CTA owns a
// TTR x TTC tile of cells, stages the tile plus an (n+1)-cell frame of vx, vy, eta_b, eta_p, b_x,
// b_y in shared memory (global indices clipped to the array's nodes 0..ncy+1 x 0..ncx+1), and
// runs the n sweeps in place there: sweep k updates the unknowns within n-1-k cells of the tile
// (the region sweep k+1 reads), ping-ponging two shared buffers per component, with the SAME
// point function as k_jacobi (jacobi_pt on a GridL whose pitch is the shared tile's: global
// indices, the global boundary logic and mirrors unchanged; 1/a_ii by the MUFU seed + Newton
// steps of the streamed kernels unless TT_RCP = 0, which equals n launches of k_jacobi bit for
// bit).  Then the tile's unknowns (and its mirror nodes) are stored.
// The bilinear coarse-grid correction of prolong_pt at one fine vx / vy
// unknown, as a value (the same expressions, so v + corr rounds as prolong_pt's update).
__device__ __forceinline__ double corr_x(const GridL &gc, const double *__restrict__ ex, int i, int j) {
    const int J0 = j >> 1;
    int I0;
    double wy0, wy1;
    if (i & 1) { I0 = (i + 1) / 2 - 1; wy0 = 0.25; wy1 = 0.75; }
    else { I0 = i / 2; wy0 = 0.75; wy1 = 0.25; }
    if (j & 1)
        return wy0 * 0.5 * (ex[at(gc, I0, J0)] + ex[at(gc, I0, J0 + 1)]) +
               wy1 * 0.5 * (ex[at(gc, I0 + 1, J0)] + ex[at(gc, I0 + 1, J0 + 1)]);
    return wy0 * ex[at(gc, I0, J0)] + wy1 * ex[at(gc, I0 + 1, J0)];
}
__device__ __forceinline__ double corr_y(const GridL &gc, const double *__restrict__ ey, int i, int j) {
    const int I0 = i >> 1;
    int J0;
    double wx0, wx1;
    if (j & 1) { J0 = (j + 1) / 2 - 1; wx0 = 0.25; wx1 = 0.75; }
    else { J0 = j / 2; wx0 = 0.75; wx1 = 0.25; }
    if (i & 1)
        return wx0 * 0.5 * (ey[at(gc, I0, J0)] + ey[at(gc, I0 + 1, J0)]) +
               wx1 * 0.5 * (ey[at(gc, I0, J0 + 1)] + ey[at(gc, I0 + 1, J0 + 1)]);
    return wx0 * ey[at(gc, I0, J0)] + wx1 * ey[at(gc, I0, J0 + 1)];
}
#ifndef TT_ROWS
#define TT_ROWS 8
#endif
#ifndef TT_RCP
#define TT_RCP 1  // 1/a_ii by MUFU seed + Newton (as the streamed kernels) instead of the IEEE division
#endif
#ifndef TT_THREADS
#define TT_THREADS 512  // 2 threads per tile cell: the sweeps are latency-bound (256 threads: +4 ms per solve)
#endif
constexpr int TTR = TT_ROWS, TTC = 32, TT_MAXN = 8;  // tile rows / columns, most sweeps per launch
constexpr int TTN = TT_THREADS;                      // threads per tile CTA
__host__ __device__ constexpr int tt_rows(int n) { return TTR + 2 * (n + 1); }
__host__ __device__ constexpr int tt_cols(int n) { return TTC + 2 * (n + 1); }
template <bool ZERO>
__global__ void __launch_bounds__(TTN) k_jacobi_tile(GridL g, const double *__restrict__ etab,
                                                          const double *__restrict__ etap, const double *__restrict__ vxi,
                                                          const double *__restrict__ vyi, double *__restrict__ vxo,
                                                          double *__restrict__ vyo, const double *__restrict__ bx,
                                                          const double *__restrict__ by, double omega, int n, GridL gc,
                                                          const double *__restrict__ ex, const double *__restrict__ ey) {
    extern __shared__ __align__(16) double tsm[];
    const int R = tt_rows(n), C = tt_cols(n), A = R * C;
    double *s_eb = tsm, *s_ep = tsm + A, *s_bx = tsm + 2 * A, *s_by = tsm + 3 * A;
    double *s_v = tsm + 4 * A;  // buffer b: vx at s_v + 2 b A, vy at s_v + (2 b + 1) A
    const int t = threadIdx.x, nt = TTN;
    const int I0 = 1 + blockIdx.y * TTR, J0 = 1 + blockIdx.x * TTC;  // first cell of the tile
    const int ib = I0 - (n + 1), jb = J0 - (n + 1);                    // global index of tile entry (0, 0)
    // stage: every array entry of the frame that exists (nodes 0..ncy+1 x 0..ncx+1), 0 elsewhere
    for (int e = t; e < A; e += nt) {
        const int i = ib + e / C, j = jb + e % C;
        const bool in = i >= 0 && i <= g.ncy + 1 && j >= 0 && j <= g.ncx + 1;
        const size_t q = at(g, i, j);
        s_eb[e] = in ? etab[q] : 0.0;
        s_ep[e] = in ? etap[q] : 0.0;
        s_bx[e] = in ? bx[q] : 0.0;
        s_by[e] = in ? by[q] : 0.0;
        double x = (!ZERO && in) ? vxi[q] : 0.0, y = (!ZERO && in) ? vyi[q] : 0.0;
        if (!ZERO && ex && in) {  // post-smoothing: the coarse-grid correction added while staging
            // (unknowns, and the mirror nodes as the mirror of their partner's correction)
            if (j >= 1 && j <= g.nvxj) {
                if (i >= 1 && i <= g.ncy) x += corr_x(gc, ex, i, j);
                else if (i == 0 && g.bN) x += g.sN * corr_x(gc, ex, 1, j);
                else if (i == g.ncy + 1 && g.bS) x += g.sS * corr_x(gc, ex, g.ncy, j);
            }
            if (i >= 1 && i <= g.nvyi) {
                if (j >= 1 && j <= g.ncx) y += corr_y(gc, ey, i, j);
                else if (j == 0 && g.bW) y += g.sW * corr_y(gc, ey, i, 1);
                else if (j == g.ncx + 1 && g.bE) y += g.sE * corr_y(gc, ey, i, g.ncx);
            }
        }
        s_v[e] = x;
        s_v[A + e] = y;
        s_v[2 * A + e] = x;  // entries no sweep writes (walls, the frame) read the same in both buffers
        s_v[3 * A + e] = y;
    }
    __syncthreads();
    GridL gt = g;  // global indices on the shared tile: at(gt, i, j) = i C + j, arrays shifted by (ib, jb)
    gt.P = C;
    const ptrdiff_t sh = (ptrdiff_t)ib * C + jb;
    RhsArgs rhs;
    rhs.mode = RHS_ARRAYS;
    rhs.bx = s_bx - sh;
    rhs.by = s_by - sh;
    rhs.p = rhs.rho = nullptr;
    rhs.gx = rhs.gy = 0.0;
    for (int k = 0; k < n; ++k) {
        const int m = n - 1 - k;  // sweep k: the unknowns within m cells of the tile
        const int i_lo = max(I0 - m, 1), i_hi = min(I0 + TTR - 1 + m, g.ncy);
        const int j_lo = max(J0 - m, 1), j_hi = min(J0 + TTC - 1 + m, g.ncx);
        const int w = j_hi - j_lo + 1, cnt = (i_hi - i_lo + 1) * w;
        const double *vix = s_v + 2 * (k & 1) * A - sh, *viy = vix + A;
        double *vox = s_v + 2 * ((k + 1) & 1) * A - sh, *voy = vox + A;
        for (int e = t; e < cnt; e += nt) {
            const int i = i_lo + e / w, j = j_lo + e % w;
            if (ZERO && k == 0) jacobi_pt<true, TT_RCP>(gt, s_eb - sh, s_ep - sh, vix, viy, vox, voy, rhs, omega, i, j);
            else jacobi_pt<false, TT_RCP>(gt, s_eb - sh, s_ep - sh, vix, viy, vox, voy, rhs, omega, i, j);
        }
        __syncthreads();
    }
    // store the tile's unknowns and the mirror nodes its boundary rows / columns own
    const double *fx = s_v + 2 * (n & 1) * A - sh, *fy = fx + A;
    const int i1 = min(I0 + TTR - 1, g.ncy), j1 = min(J0 + TTC - 1, g.ncx);
    const int ilo = (I0 == 1) ? 0 : I0, ihi = (i1 == g.ncy) ? g.ncy + 1 : i1;
    const int jlo = (J0 == 1) ? 0 : J0, jhi = (j1 == g.ncx) ? g.ncx + 1 : j1;
    const int w = jhi - jlo + 1, cnt = (ihi - ilo + 1) * w;
    for (int e = t; e < cnt; e += nt) {
        const int i = ilo + e / w, j = jlo + e % w;
        const size_t q = at(g, i, j), s = at(gt, i, j);
        const bool xin = j >= 1 && j <= g.nvxj, yin = i >= 1 && i <= g.nvyi;
        const bool xrow = i >= 1 && i <= g.ncy;  // vx rows of unknowns; rows 0 / ncy+1: mirrors
        if (xin && (xrow || (i == 0 && g.bN) || (i == g.ncy + 1 && g.bS))) vxo[q] = fx[s];
        const bool ycol = j >= 1 && j <= g.ncx;
        if (yin && (ycol || (j == 0 && g.bW) || (j == g.ncx + 1 && g.bE))) vyo[q] = fy[s];
    }
}

// Damped red-black Gauss-Seidel (Eq. sor_update), one of the four phases
// (reading R11): component comp (0 vx, 1 vy), colour = (i+j) mod 2 on level indices.
// Unknowns of one phase never read each other, so the phase is parallel and in place.
__global__ void __launch_bounds__(BX *BY) k_rbgs_phase(GridL g, const double *__restrict__ etab,
                                                       const double *__restrict__ etap, double *vx, double *vy,
                                                       RhsArgs rhs, double omega, int comp, int colour) {
    const int i = blockIdx.y * BY + threadIdx.y + 1;
    const int j = 2 * (blockIdx.x * BX + threadIdx.x) + 1 + ((i + 1 + colour + g.par) & 1);
    const ArrayAcc ax{vx, (size_t)g.P}, ay{vy, (size_t)g.P};
    if (comp == 0) {
        if (i > g.ncy || j > g.nvxj) return;
        const double a = lx_diag(g, etab, etap, i, j);
        const double vn = ax(i, j) + omega * (rhs_x(g, rhs, i, j) - lx_row(g, etab, etap, ax, ay, i, j)) / a;
        vx[at(g, i, j)] = vn;
        if (i == 1 && g.bN) vx[at(g, 0, j)] = g.sN * vn;
        if (i == g.ncy && g.bS) vx[at(g, g.ncy + 1, j)] = g.sS * vn;
    } else {
        if (i > g.nvyi || j > g.ncx) return;
        const double a = ly_diag(g, etab, etap, i, j);
        const double vn = ay(i, j) + omega * (rhs_y(g, rhs, i, j) - ly_row(g, etab, etap, ax, ay, i, j)) / a;
        vy[at(g, i, j)] = vn;
        if (j == 1 && g.bW) vy[at(g, i, 0)] = g.sW * vn;
        if (j == g.ncx && g.bE) vy[at(g, i, g.ncx + 1)] = g.sE * vn;
    }
}

// r = b - L v (Eq. mg_residual) at the unknowns of a level.
__device__ __forceinline__ void residual_pt(const GridL &g, const double *__restrict__ etab,
                                            const double *__restrict__ etap, const double *__restrict__ vx,
                                            const double *__restrict__ vy, const RhsArgs &rhs,
                                            double *__restrict__ rx, double *__restrict__ ry, int i, int j) {
    const ArrayAcc ax{vx, (size_t)g.P}, ay{vy, (size_t)g.P};
    if (j <= g.nvxj) rx[at(g, i, j)] = rhs_x(g, rhs, i, j) - lx_row(g, etab, etap, ax, ay, i, j);
    if (i <= g.nvyi) ry[at(g, i, j)] = rhs_y(g, rhs, i, j) - ly_row(g, etab, etap, ax, ay, i, j);
}
__global__ void __launch_bounds__(BX *BY) k_residual(GridL g, const double *__restrict__ etab,
                                                     const double *__restrict__ etap, const double *__restrict__ vx,
                                                     const double *__restrict__ vy, RhsArgs rhs,
                                                     double *__restrict__ rx, double *__restrict__ ry) {
    const int j = blockIdx.x * BX + threadIdx.x + 1;
    const int i = blockIdx.y * BY + threadIdx.y + 1;
    if (i > g.ncy || j > g.ncx) return;
    residual_pt(g, etab, etap, vx, vy, rhs, rx, ry, i, j);
}


// ------------------------------------------------ viscosity rescaling / lithostatic (NEXT-1)
// eta_min over the basic nodes [0,ncy]x[0,ncx] and P nodes [1,ncy]x[1,ncx]: positive
// doubles order like their bit patterns, so an unsigned atomicMin is exact.
__global__ void k_eta_min(GridL g, const double *__restrict__ eb, const double *__restrict__ ep,
                          unsigned long long *emin) {
    const int j = blockIdx.x * BX + threadIdx.x;
    const int i = blockIdx.y * BY + threadIdx.y;
    double m = INFINITY;
    if (i <= g.ncy && j <= g.ncx) {
        m = eb[at(g, i, j)];
        if (i >= 1 && j >= 1) m = fmin(m, ep[at(g, i, j)]);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m < INFINITY) atomicMin(emin, (unsigned long long)__double_as_longlong(m));
}
// eta_comp = (1 - theta) eta_min + theta eta on the same nodes
__global__ void k_eta_blend(GridL g, const double *__restrict__ ebu, const double *__restrict__ epu,
                            double *__restrict__ eb, double *__restrict__ ep, const unsigned long long *emin,
                            double theta) {
    const int j = blockIdx.x * BX + threadIdx.x;
    const int i = blockIdx.y * BY + threadIdx.y;
    if (i > g.ncy || j > g.ncx) return;
    const double m = __longlong_as_double((long long)*emin);
    eb[at(g, i, j)] = (1.0 - theta) * m + theta * ebu[at(g, i, j)];
    if (i >= 1 && j >= 1) ep[at(g, i, j)] = (1.0 - theta) * m + theta * epu[at(g, i, j)];
}
// column prefix sums in row order (deterministic): one thread per P column
__global__ void k_lithostatic(GridL g, const double *__restrict__ rb, double gy, double *__restrict__ p) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (j > g.ncx) return;
    double acc = gy * (0.5 * g.dy) * (0.5 * (rb[at(g, 0, j - 1)] + rb[at(g, 0, j)]));
    p[j - 1] = acc;
    for (int i = 1; i < g.ncy; ++i) {
        acc = acc + gy * g.dy * (0.5 * (rb[at(g, i, j - 1)] + rb[at(g, i, j)]));
        p[(size_t)i * g.ncx + (j - 1)] = acc;
    }
}

// ------------------------------------------------------------------ transfers (a5, a6, a7)
// Normalised bilinear restriction (Alg. 2 weights; reading R6) in
// gather form: each coarse node sums its own fine contributors, so neither the 4-colour
// schedule of Alg. 2 nor atomics are needed.  For factor 2 the hat weights are
// [1/2, 1, 1/2] along a vertex-centred axis and [1/4, 3/4, 3/4, 1/4] along a cell-centred
// axis; contributors outside the closed domain (mirror / ghost nodes) are dropped and the
// sum of the remaining weights renormalises.
__device__ __forceinline__ double W4(int d) { return (d == 0 || d == 3) ? 0.25 : 0.75; }

__device__ __forceinline__ void restrict_vel_pt(const GridL &gf, const GridL &gc, const double *__restrict__ rx,
                                                const double *__restrict__ ry, double *__restrict__ bxc,
                                                double *__restrict__ byc, int I, int J) {
    if (bxc && J <= gc.nvxj) {  // vx: x vertex-centred, y cell-centred
        double s = 0.0, w = 0.0;
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const int i = 2 * I - 2 + d;
            if ((i < 1 && gf.bN) || (i > gf.ncy && gf.bS)) continue;
            const double row = 0.5 * rx[at(gf, i, 2 * J - 1)] + rx[at(gf, i, 2 * J)] + 0.5 * rx[at(gf, i, 2 * J + 1)];
            s += W4(d) * row;
            w += W4(d);
        }
        bxc[at(gc, I, J)] = s / (2.0 * w);
    }
    if (byc && I <= gc.nvyi) {  // vy: x cell-centred, y vertex-centred
        double s = 0.0, w = 0.0;
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const int j = 2 * J - 2 + d;
            if ((j < 1 && gf.bW) || (j > gf.ncx && gf.bE)) continue;
            const double col = 0.5 * ry[at(gf, 2 * I - 1, j)] + ry[at(gf, 2 * I, j)] + 0.5 * ry[at(gf, 2 * I + 1, j)];
            s += W4(d) * col;
            w += W4(d);
        }
        byc[at(gc, I, J)] = s / (2.0 * w);
    }
}
__global__ void k_restrict_vel(GridL gf, GridL gc, const double *__restrict__ rx, const double *__restrict__ ry,
                               double *__restrict__ bxc, double *__restrict__ byc) {
    const int J = blockIdx.x * BX + threadIdx.x + 1;
    const int I = blockIdx.y * BY + threadIdx.y + 1;
    if (I > gc.ncy || J > gc.ncx) return;
    restrict_vel_pt(gf, gc, rx, ry, bxc, byc, I, J);
}
// basic-node field (eta_b): [1/2,1,1/2] x [1/2,1,1/2] over fine basic nodes in [0,ncy]x[0,ncx]
__global__ void k_restrict_b(GridL gf, GridL gc, const double *__restrict__ f, double *__restrict__ c) {
    // owned coarse basic nodes: rows [1 - bN, ncy], cols [1 - bW, ncx] (row/col 0 of an
    // interior tile is a halo owned by the neighbour); fine halo rows/cols are valid data,
    // only nodes outside the GLOBAL domain are dropped (reading R6)
    const int J = blockIdx.x * BX + threadIdx.x + (gc.bW ? 0 : 1);
    const int I = blockIdx.y * BY + threadIdx.y + (gc.bN ? 0 : 1);
    if (I > gc.ncy || J > gc.ncx) return;
    const double w3[3] = {0.5, 1.0, 0.5};
    double s = 0.0, wy = 0.0, wx = 0.0;
    for (int dj = 0; dj < 3; ++dj) {
        const int j = 2 * J - 1 + dj;
        if (j >= 0 && (j <= gf.ncx || !gf.bE)) wx += w3[dj];
    }
    for (int di = 0; di < 3; ++di) {
        const int i = 2 * I - 1 + di;
        if (i < 0 || (i > gf.ncy && gf.bS)) continue;
        wy += w3[di];
        double row = 0.0;
        for (int dj = 0; dj < 3; ++dj) {
            const int j = 2 * J - 1 + dj;
            if (j < 0 || (j > gf.ncx && gf.bE)) continue;
            row += w3[dj] * f[at(gf, i, j)];
        }
        s += w3[di] * row;
    }
    c[at(gc, I, J)] = s / (wy * wx);
}
// P-node field (eta_p): [1,3,3,1]/8 per axis over fine P nodes in [1,ncy]x[1,ncx]
__global__ void k_restrict_p(GridL gf, GridL gc, const double *__restrict__ f, double *__restrict__ c) {
    const int J = blockIdx.x * BX + threadIdx.x + 1;
    const int I = blockIdx.y * BY + threadIdx.y + 1;
    if (I > gc.ncy || J > gc.ncx) return;
    double s = 0.0, wy = 0.0, wx = 0.0;
    for (int dj = 0; dj < 4; ++dj) {
        const int j = 2 * J - 2 + dj;
        if ((j >= 1 || !gf.bW) && (j <= gf.ncx || !gf.bE)) wx += W4(dj);
    }
    for (int di = 0; di < 4; ++di) {
        const int i = 2 * I - 2 + di;
        if ((i < 1 && gf.bN) || (i > gf.ncy && gf.bS)) continue;
        wy += W4(di);
        double row = 0.0;
        for (int dj = 0; dj < 4; ++dj) {
            const int j = 2 * J - 2 + dj;
            if ((j < 1 && gf.bW) || (j > gf.ncx && gf.bE)) continue;
            row += W4(dj) * f[at(gf, i, j)];
        }
        s += W4(di) * row;
    }
    c[at(gc, I, J)] = s / (wy * wx);
}

// Bilinear prolongation + correction: each fine unknown adds the
// hat-weighted coarse correction of its (up to) four surrounding coarse nodes; coarse
// mirror nodes hold the homogeneous-BC image, coarse walls are 0 (Appendix B).
__device__ __forceinline__ void prolong_pt(const GridL &gf, const GridL &gc, const double *__restrict__ ex,
                                           const double *__restrict__ ey, double *__restrict__ vx,
                                           double *__restrict__ vy, int i, int j) {
    if (j <= gf.nvxj) {  // vx: x vertex-centred, y cell-centred
        const int J0 = j >> 1;
        int I0;
        double wy0, wy1;
        if (i & 1) { I0 = (i + 1) / 2 - 1; wy0 = 0.25; wy1 = 0.75; }
        else { I0 = i / 2; wy0 = 0.75; wy1 = 0.25; }
        double s;
        if (j & 1)
            s = wy0 * 0.5 * (ex[at(gc, I0, J0)] + ex[at(gc, I0, J0 + 1)]) +
                wy1 * 0.5 * (ex[at(gc, I0 + 1, J0)] + ex[at(gc, I0 + 1, J0 + 1)]);
        else
            s = wy0 * ex[at(gc, I0, J0)] + wy1 * ex[at(gc, I0 + 1, J0)];
        const double vn = vx[at(gf, i, j)] + s;
        vx[at(gf, i, j)] = vn;
        if (i == 1 && gf.bN) vx[at(gf, 0, j)] = gf.sN * vn;
        if (i == gf.ncy && gf.bS) vx[at(gf, gf.ncy + 1, j)] = gf.sS * vn;
    }
    if (i <= gf.nvyi) {  // vy: y vertex-centred, x cell-centred
        const int I0 = i >> 1;
        int J0;
        double wx0, wx1;
        if (j & 1) { J0 = (j + 1) / 2 - 1; wx0 = 0.25; wx1 = 0.75; }
        else { J0 = j / 2; wx0 = 0.75; wx1 = 0.25; }
        double s;
        if (i & 1)
            s = wx0 * 0.5 * (ey[at(gc, I0, J0)] + ey[at(gc, I0 + 1, J0)]) +
                wx1 * 0.5 * (ey[at(gc, I0, J0 + 1)] + ey[at(gc, I0 + 1, J0 + 1)]);
        else
            s = wx0 * ey[at(gc, I0, J0)] + wx1 * ey[at(gc, I0, J0 + 1)];
        const double vn = vy[at(gf, i, j)] + s;
        vy[at(gf, i, j)] = vn;
        if (j == 1 && gf.bW) vy[at(gf, i, 0)] = gf.sW * vn;
        if (j == gf.ncx && gf.bE) vy[at(gf, i, gf.ncx + 1)] = gf.sE * vn;
    }
}
__global__ void __launch_bounds__(BX *BY) k_prolong(GridL gf, GridL gc, const double *__restrict__ ex,
                                                    const double *__restrict__ ey, double *__restrict__ vx,
                                                    double *__restrict__ vy) {
    const int j = blockIdx.x * BX + threadIdx.x + 1;
    const int i = blockIdx.y * BY + threadIdx.y + 1;
    if (i > gf.ncy || j > gf.ncx) return;
    prolong_pt(gf, gc, ex, ey, vx, vy, i, j);
}

// Same prolongation, one thread per aligned pair of fine columns (2J-1, 2J) of one row:
// 16-B loads / stores of the fine velocities (column 2J-1 is 16-B aligned by the layout)
// and the coarse values shared by the pair; identical arithmetic to k_prolong.
__global__ void __launch_bounds__(BX *BY) k_prolong2(GridL gf, GridL gc, const double *__restrict__ ex,
                                                     const double *__restrict__ ey, double *__restrict__ vx,
                                                     double *__restrict__ vy) {
    const int J = blockIdx.x * BX + threadIdx.x + 1;  // fine columns 2J-1, 2J
    const int i = blockIdx.y * BY + threadIdx.y + 1;
    if (i > gf.ncy || 2 * J > gf.ncx) return;
    const int j = 2 * J - 1;
    {  // vx: x vertex-centred, y cell-centred
        int I0;
        double wy0, wy1;
        if (i & 1) { I0 = (i + 1) / 2 - 1; wy0 = 0.25; wy1 = 0.75; }
        else { I0 = i / 2; wy0 = 0.75; wy1 = 0.25; }
        const double a0 = ex[at(gc, I0, J - 1)], a1 = ex[at(gc, I0, J)];
        const double b0 = ex[at(gc, I0 + 1, J - 1)], b1 = ex[at(gc, I0 + 1, J)];
        const double s_odd = wy0 * 0.5 * (a0 + a1) + wy1 * 0.5 * (b0 + b1);  // column 2J-1
        const double s_even = wy0 * a1 + wy1 * b1;                            // column 2J
        double2 *p = reinterpret_cast<double2 *>(vx + at(gf, i, j));
        double2 v = *p;
        v.x += s_odd;
        const bool wall = 2 * J > gf.nvxj;  // column 2J = ncx is the east wall
        if (!wall) v.y += s_even;
        *p = v;
        if (i == 1 && gf.bN) *reinterpret_cast<double2 *>(vx + at(gf, 0, j)) = make_double2(gf.sN * v.x, wall ? 0.0 : gf.sN * v.y);
        if (i == gf.ncy && gf.bS)
            *reinterpret_cast<double2 *>(vx + at(gf, gf.ncy + 1, j)) = make_double2(gf.sS * v.x, wall ? 0.0 : gf.sS * v.y);
    }
    if (i <= gf.nvyi) {  // vy: y vertex-centred, x cell-centred
        const int I0 = i >> 1;
        const double c0 = ey[at(gc, I0, J - 1)], c1 = ey[at(gc, I0, J)], c2 = ey[at(gc, I0, J + 1)];
        double s_odd, s_even;  // columns 2J-1 (J0 = J-1; 1/4, 3/4) and 2J (J0 = J; 3/4, 1/4)
        if (i & 1) {
            const double d0 = ey[at(gc, I0 + 1, J - 1)], d1 = ey[at(gc, I0 + 1, J)], d2 = ey[at(gc, I0 + 1, J + 1)];
            s_odd = 0.25 * 0.5 * (c0 + d0) + 0.75 * 0.5 * (c1 + d1);
            s_even = 0.75 * 0.5 * (c1 + d1) + 0.25 * 0.5 * (c2 + d2);
        } else {
            s_odd = 0.25 * c0 + 0.75 * c1;
            s_even = 0.75 * c1 + 0.25 * c2;
        }
        double2 *p = reinterpret_cast<double2 *>(vy + at(gf, i, j));
        double2 v = *p;
        v.x += s_odd;
        v.y += s_even;
        *p = v;
        if (J == 1 && gf.bW) vy[at(gf, i, 0)] = gf.sW * v.x;
        if (2 * J == gf.ncx && gf.bE) vy[at(gf, i, gf.ncx + 1)] = gf.sE * v.y;
    }
}

// ------------------------------------------------------------------ residual + energy (a3)
// Full saddle residual r_v = f - L v - G p, r_p = -D v and the
// per-block partial sums Sv = sum r_v^2 / (-a_ii), Sp = sum r_p^2 eta_p / (2/dx^2+2/dy^2).
__global__ void __launch_bounds__(BX *BY) k_energy(GridL g, const double *__restrict__ etab,
                                                   const double *__restrict__ etap, const double *__restrict__ vx,
                                                   const double *__restrict__ vy, const double *__restrict__ p,
                                                   const double *__restrict__ rho, double gx, double gy,
                                                   double *__restrict__ rxo, double *__restrict__ ryo,
                                                   double *__restrict__ rpo, double *__restrict__ partials,
                                                   int force_only) {
    __shared__ double sh[BX * BY / 32];
    const int j = blockIdx.x * BX + threadIdx.x + 1;
    const int i = blockIdx.y * BY + threadIdx.y + 1;
    double sv = 0.0, sp = 0.0;
    if (i <= g.ncy && j <= g.ncx) {
        const ArrayAcc ax{vx, (size_t)g.P}, ay{vy, (size_t)g.P};
        RhsArgs rhs;
        rhs.mode = RHS_FINE;
        rhs.p = p;
        rhs.rho = rho;
        rhs.gx = gx;
        rhs.gy = gy;
        rhs.bx = rhs.by = nullptr;
        if (j <= g.nvxj) {
            const double a = lx_diag(g, etab, etap, i, j);
            double r;
            if (force_only) r = (gx != 0.0) ? -gx * (0.5 * (rho[at(g, i - 1, j)] + rho[at(g, i, j)])) : 0.0;
            else r = rhs_x(g, rhs, i, j) - lx_row(g, etab, etap, ax, ay, i, j);
            sv += r * r / (-a);
            if (rxo) rxo[at(g, i, j)] = r;
        }
        if (i <= g.nvyi) {
            const double a = ly_diag(g, etab, etap, i, j);
            double r;
            if (force_only) r = (gy != 0.0) ? -gy * (0.5 * (rho[at(g, i, j - 1)] + rho[at(g, i, j)])) : 0.0;
            else r = rhs_y(g, rhs, i, j) - ly_row(g, etab, etap, ax, ay, i, j);
            sv += r * r / (-a);
            if (ryo) ryo[at(g, i, j)] = r;
        }
        if (!force_only) {
            const double rp = -((vx[at(g, i, j)] - vx[at(g, i, j - 1)]) * g.idx + (vy[at(g, i, j)] - vy[at(g, i - 1, j)]) * g.idy);
            sp = rp * rp * (etap[at(g, i, j)] / (2.0 * g.idx2 + 2.0 * g.idy2));
            if (rpo) rpo[at(g, i, j)] = rp;
        }
    }
    sv = block_sum<BX * BY>(sv, sh);
    sp = block_sum<BX * BY>(sp, sh);
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        const size_t b = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
        partials[2 * b] = sv;
        partials[2 * b + 1] = sp;
    }
}
// energy of a given residual vector (GCR recursive residual)
__global__ void __launch_bounds__(BX *BY) k_energy_vec(GridL g, const double *__restrict__ etab,
                                                       const double *__restrict__ etap, const double *__restrict__ rx,
                                                       const double *__restrict__ ry, const double *__restrict__ rp,
                                                       double *__restrict__ partials) {
    __shared__ double sh[BX * BY / 32];
    const int j = blockIdx.x * BX + threadIdx.x + 1;
    const int i = blockIdx.y * BY + threadIdx.y + 1;
    double sv = 0.0, sp = 0.0;
    if (i <= g.ncy && j <= g.ncx) {
        if (j <= g.nvxj) { const double r = rx[at(g, i, j)]; sv += r * r / (-lx_diag(g, etab, etap, i, j)); }
        if (i <= g.nvyi) { const double r = ry[at(g, i, j)]; sv += r * r / (-ly_diag(g, etab, etap, i, j)); }
        const double r = rp[at(g, i, j)];
        sp = r * r * (etap[at(g, i, j)] / (2.0 * g.idx2 + 2.0 * g.idy2));
    }
    sv = block_sum<BX * BY>(sv, sh);
    sp = block_sum<BX * BY>(sp, sh);
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        const size_t b = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
        partials[2 * b] = sv;
        partials[2 * b + 1] = sp;
    }
}

// ------------------------------------------------------------------ pressure update (a10)
// Uzawa pressure step, reading R3: p <- p + alpha eta_P r_p with r_p = -D v (PAPER.md:824
// with the physical sign), applied to the stored p minus the previous mean: the zero-mean
// projection is inert for v and E (G 1 = 0), so it is applied one step
// late and at the output; per-block partial sums of the new p give the next mean.
__global__ void __launch_bounds__(BX *BY) k_pupdate(GridL g, const double *__restrict__ etap,
                                                    const double *__restrict__ vx, const double *__restrict__ vy,
                                                    const double *pin, double *pout, double alpha_signed,
                                                    const double *__restrict__ mshift, double *__restrict__ partials) {
    __shared__ double sh[BX * BY / 32];
    const int j = blockIdx.x * BX + threadIdx.x + 1;
    const int i = blockIdx.y * BY + threadIdx.y + 1;
    double s = 0.0;
    if (i <= g.ncy && j <= g.ncx) {
        const double dv = (vx[at(g, i, j)] - vx[at(g, i, j - 1)]) * g.idx + (vy[at(g, i, j)] - vy[at(g, i - 1, j)]) * g.idy;
        const double pn = (pin[at(g, i, j)] - *mshift) + alpha_signed * etap[at(g, i, j)] * (-dv);
        if (pout) pout[at(g, i, j)] = pn;
        s = pn;
    }
    s = block_sum<BX * BY>(s, sh);
    if (threadIdx.x == 0 && threadIdx.y == 0) partials[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
}

// ------------------------------------------------------------------ deterministic finalisation
__global__ void __launch_bounds__(1024) k_finalize(const double *__restrict__ partials, int nblocks, int ncomp,
                                                   double scale, double *__restrict__ out) {
    __shared__ double sh[32];
    for (int c = 0; c < ncomp; ++c) {
        double s = 0.0;
        for (int b = threadIdx.x; b < nblocks; b += 1024) s += partials[(size_t)b * ncomp + c];
        s = block_sum<1024>(s, sh);
        if (threadIdx.x == 0) out[c] = scale * s;
    }
}
__global__ void __launch_bounds__(1024) k_energy_final(const double *__restrict__ partials, int nblocks,
                                                       const double *__restrict__ Sf, double *__restrict__ out) {
    __shared__ double sh[32];
    double s0 = 0.0, s1 = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += 1024) {
        s0 += partials[2 * (size_t)b];
        s1 += partials[2 * (size_t)b + 1];
    }
    s0 = block_sum<1024>(s0, sh);
    s1 = block_sum<1024>(s1, sh);
    if (threadIdx.x == 0) {
        out[1] = s0;
        out[2] = s1;
        out[0] = (Sf[0] > 0.0) ? sqrt((s0 + s1) / Sf[0]) : 0.0;
    }
}

// Uzawa step finalisation from the fused pass (Sv, Sp, sum p' per block):
// out[0] = E = sqrt((Sv + Sp) / Sf), out[1] = Sv, out[2] = Sp; *mean = inv_np * sum p'
__global__ void __launch_bounds__(1024) k_uzawa_final(const double *__restrict__ partials, int nblocks,
                                                      const double *__restrict__ Sf, double inv_np,
                                                      double *__restrict__ out, double *__restrict__ mean) {
    __shared__ double sh[32];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += 1024) {
        s0 += partials[3 * (size_t)b];
        s1 += partials[3 * (size_t)b + 1];
        s2 += partials[3 * (size_t)b + 2];
    }
    s0 = block_sum<1024>(s0, sh);
    s1 = block_sum<1024>(s1, sh);
    s2 = block_sum<1024>(s2, sh);
    if (threadIdx.x == 0) {
        out[1] = s0;
        out[2] = s1;
        out[0] = (Sf[0] > 0.0) ? sqrt((s0 + s1) / Sf[0]) : 0.0;
        *mean = s2 * inv_np;
    }
}

// ------------------------------------------------------------------ layout conversion
// user -> padded velocity: unknowns copied, walls 0, mirrors from partners
__global__ void k_in_velocity(GridL g, const double *__restrict__ ux, const double *__restrict__ uy,
                              double *__restrict__ vx, double *__restrict__ vy) {
    const int j = blockIdx.x * BX + threadIdx.x;  // 0..ncx+1
    const int i = blockIdx.y * BY + threadIdx.y;  // 0..ncy+1
    if (i > g.ncy + 1 || j > g.ncx + 1) return;
    // vx: walls (global W/E sides) 0; mirrors (global N/S) from partners; tile halos 0
    // (a decomposed level fills them by a halo exchange right after)
    if (j <= g.ncx) {
        double v = 0.0;
        if (!((j == 0 && g.bW) || (j == g.ncx && g.bE))) {
            if (i >= 1 && i <= g.ncy) v = ux[(size_t)(i - 1) * (g.ncx + 1) + j];
            else if (i == 0) v = g.bN ? g.sN * ux[j] : 0.0;
            else v = g.bS ? g.sS * ux[(size_t)(g.ncy - 1) * (g.ncx + 1) + j] : 0.0;
        }
        vx[at(g, i, j)] = v;
    }
    if (i <= g.ncy) {
        double v = 0.0;
        if (!((i == 0 && g.bN) || (i == g.ncy && g.bS))) {
            if (j >= 1 && j <= g.ncx) v = uy[(size_t)i * g.ncx + (j - 1)];
            else if (j == 0) v = g.bW ? g.sW * uy[(size_t)i * g.ncx] : 0.0;
            else v = g.bE ? g.sE * uy[(size_t)i * g.ncx + (g.ncx - 1)] : 0.0;
        }
        vy[at(g, i, j)] = v;
    }
}
__global__ void k_in_p(GridL g, const double *__restrict__ u, double *__restrict__ a) {
    const int j = blockIdx.x * BX + threadIdx.x + 1, i = blockIdx.y * BY + threadIdx.y + 1;
    if (i <= g.ncy && j <= g.ncx) a[at(g, i, j)] = u[(size_t)(i - 1) * g.ncx + (j - 1)];
}
__global__ void k_in_b(GridL g, const double *__restrict__ u, double *__restrict__ a) {
    const int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y;
    if (i <= g.ncy && j <= g.ncx) a[at(g, i, j)] = u[(size_t)i * (g.ncx + 1) + j];
}
__global__ void k_in_vx_raw(GridL g, const double *__restrict__ u, double *__restrict__ a) {
    const int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y + 1;
    if (i <= g.ncy && j <= g.ncx)
        a[at(g, i, j)] = ((j == 0 && g.bW) || (j == g.ncx && g.bE)) ? 0.0 : u[(size_t)(i - 1) * (g.ncx + 1) + j];
}
__global__ void k_in_vy_raw(GridL g, const double *__restrict__ u, double *__restrict__ a) {
    const int j = blockIdx.x * BX + threadIdx.x + 1, i = blockIdx.y * BY + threadIdx.y;
    if (i <= g.ncy && j <= g.ncx)
        a[at(g, i, j)] = ((i == 0 && g.bN) || (i == g.ncy && g.bS)) ? 0.0 : u[(size_t)i * g.ncx + (j - 1)];
}
__global__ void k_out_vx(GridL g, const double *__restrict__ a, double *__restrict__ u) {
    const int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y + 1;
    if (i <= g.ncy && j <= g.ncx)
        u[(size_t)(i - 1) * (g.ncx + 1) + j] = ((j == 0 && g.bW) || (j == g.ncx && g.bE)) ? 0.0 : a[at(g, i, j)];
}
__global__ void k_out_vy(GridL g, const double *__restrict__ a, double *__restrict__ u) {
    const int j = blockIdx.x * BX + threadIdx.x + 1, i = blockIdx.y * BY + threadIdx.y;
    if (i <= g.ncy && j <= g.ncx)
        u[(size_t)i * g.ncx + (j - 1)] = ((i == 0 && g.bN) || (i == g.ncy && g.bS)) ? 0.0 : a[at(g, i, j)];
}
__global__ void k_out_p(GridL g, const double *__restrict__ a, double *__restrict__ u, const double *shift) {
    const int j = blockIdx.x * BX + threadIdx.x + 1, i = blockIdx.y * BY + threadIdx.y + 1;
    if (i <= g.ncy && j <= g.ncx) u[(size_t)(i - 1) * g.ncx + (j - 1)] = a[at(g, i, j)] - (shift ? *shift : 0.0);
}
__global__ void k_out_b(GridL g, const double *__restrict__ a, double *__restrict__ u) {
    const int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y;
    if (i <= g.ncy && j <= g.ncx) u[(size_t)i * (g.ncx + 1) + j] = a[at(g, i, j)];
}
// A x in user layout: ax, ay = L v + G p (walls 0), ap = D v  (a2)
__global__ void __launch_bounds__(BX *BY) k_apply(GridL g, const double *__restrict__ etab,
                                                  const double *__restrict__ etap, const double *__restrict__ vx,
                                                  const double *__restrict__ vy, const double *__restrict__ p,
                                                  double *__restrict__ ax, double *__restrict__ ay,
                                                  double *__restrict__ ap) {
    const int j = blockIdx.x * BX + threadIdx.x + 1;
    const int i = blockIdx.y * BY + threadIdx.y + 1;
    if (i > g.ncy || j > g.ncx) return;
    const ArrayAcc axx{vx, (size_t)g.P}, ayy{vy, (size_t)g.P};
    const size_t wx = g.ncx + 1, wy = g.ncx;
    if (j < g.ncx)
        ax[(size_t)(i - 1) * wx + j] = lx_row(g, etab, etap, axx, ayy, i, j) + (p[at(g, i, j)] - p[at(g, i, j + 1)]) * g.idx;
    else
        ax[(size_t)(i - 1) * wx + g.ncx] = 0.0;
    if (j == 1 && g.bW) ax[(size_t)(i - 1) * wx] = 0.0;
    if (i < g.ncy)
        ay[(size_t)i * wy + (j - 1)] = ly_row(g, etab, etap, axx, ayy, i, j) + (p[at(g, i, j)] - p[at(g, i + 1, j)]) * g.idy;
    else
        ay[(size_t)g.ncy * wy + (j - 1)] = 0.0;
    if (i == 1 && g.bN) ay[(size_t)(j - 1)] = 0.0;
    ap[(size_t)(i - 1) * g.ncx + (j - 1)] =
        (vx[at(g, i, j)] - vx[at(g, i, j - 1)]) * g.idx + (vy[at(g, i, j)] - vy[at(g, i - 1, j)]) * g.idy;
}
// same, padded outputs (GCR: w = A z)
__global__ void __launch_bounds__(BX *BY) k_apply_padded(GridL g, const double *__restrict__ etab,
                                                         const double *__restrict__ etap, const double *__restrict__ vx,
                                                         const double *__restrict__ vy, const double *__restrict__ p,
                                                         double *__restrict__ ax, double *__restrict__ ay,
                                                         double *__restrict__ ap) {
    const int j = blockIdx.x * BX + threadIdx.x + 1;
    const int i = blockIdx.y * BY + threadIdx.y + 1;
    if (i > g.ncy || j > g.ncx) return;
    const ArrayAcc axx{vx, (size_t)g.P}, ayy{vy, (size_t)g.P};
    if (j <= g.nvxj) ax[at(g, i, j)] = lx_row(g, etab, etap, axx, ayy, i, j) + (p[at(g, i, j)] - p[at(g, i, j + 1)]) * g.idx;
    if (i <= g.nvyi) ay[at(g, i, j)] = ly_row(g, etab, etap, axx, ayy, i, j) + (p[at(g, i, j)] - p[at(g, i + 1, j)]) * g.idy;
    ap[at(g, i, j)] = (vx[at(g, i, j)] - vx[at(g, i, j - 1)]) * g.idx + (vy[at(g, i, j)] - vy[at(g, i - 1, j)]) * g.idy;
}
// energy weights of the GCR residual: ewx = 1/(-a_ii) at vx unknowns, ewy at vy unknowns,
// ewp = eta_P/(2/dx^2+2/dy^2) at P nodes, so that
// E^2 Sf = sum r^2 ew over the padded arrays (zeros elsewhere)
__global__ void k_energy_weights(GridL g, const double *__restrict__ etab, const double *__restrict__ etap,
                                 double *__restrict__ ewx, double *__restrict__ ewy, double *__restrict__ ewp) {
    const int j = blockIdx.x * BX + threadIdx.x + 1, i = blockIdx.y * BY + threadIdx.y + 1;
    if (i > g.ncy || j > g.ncx) return;
    if (j <= g.nvxj) ewx[at(g, i, j)] = 1.0 / (-lx_diag(g, etab, etap, i, j));
    if (i <= g.nvyi) ewy[at(g, i, j)] = 1.0 / (-ly_diag(g, etab, etap, i, j));
    ewp[at(g, i, j)] = etap[at(g, i, j)] / (2.0 * g.idx2 + 2.0 * g.idy2);
}
// materialise b = f - G p (RHS_FINE) or copy b (RHS_ARRAYS) at the unknowns
__global__ void k_make_rhs(GridL g, RhsArgs rhs, double *__restrict__ bx, double *__restrict__ by) {
    const int j = blockIdx.x * BX + threadIdx.x + 1, i = blockIdx.y * BY + threadIdx.y + 1;
    if (i > g.ncy || j > g.ncx) return;
    if (j <= g.nvxj) bx[at(g, i, j)] = rhs_x(g, rhs, i, j);
    if (i <= g.nvyi) by[at(g, i, j)] = rhs_y(g, rhs, i, j);
}
__global__ void k_refresh_mirrors(GridL g, double *__restrict__ vx, double *__restrict__ vy) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 1 && t <= g.ncx - 1) {
        vx[at(g, 0, t)] = g.sN * vx[at(g, 1, t)];
        vx[at(g, g.ncy + 1, t)] = g.sS * vx[at(g, g.ncy, t)];
    }
    if (t >= 1 && t <= g.ncy - 1) {
        vy[at(g, t, 0)] = g.sW * vy[at(g, t, 1)];
        vy[at(g, t, g.ncx + 1)] = g.sE * vy[at(g, t, g.ncx)];
    }
}
__global__ void k_count_nonpos(const double *__restrict__ a, size_t n, int *count) {
    int c = 0;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x)
        c += !(a[k] > 0.0);
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// ------------------------------------------------------------------ coarsest level (a8)
// value of the unit vector e_c at padded node (i, j), mirror relations and walls folded
__device__ __forceinline__ int vx_unknown(const GridL &g, int i, int j) { return (i - 1) * (g.ncx - 1) + (j - 1); }
__device__ __forceinline__ int vy_unknown(const GridL &g, int i, int j) {
    return g.ncy * (g.ncx - 1) + (i - 1) * g.ncx + (j - 1);
}
struct UnitVX {
    GridL g;
    int c;
    __device__ double operator()(int i, int j) const {
        if (j <= 0 || j >= g.ncx) return 0.0;
        double s = 1.0;
        if (i == 0) { i = 1; s = g.sN; }
        else if (i == g.ncy + 1) { i = g.ncy; s = g.sS; }
        return vx_unknown(g, i, j) == c ? s : 0.0;
    }
};
struct UnitVY {
    GridL g;
    int c;
    __device__ double operator()(int i, int j) const {
        if (i <= 0 || i >= g.ncy) return 0.0;
        double s = 1.0;
        if (j == 0) { j = 1; s = g.sW; }
        else if (j == g.ncx + 1) { j = g.ncx; s = g.sE; }
        return vy_unknown(g, i, j) == c ? s : 0.0;
    }
};
__global__ void k_coarse_assemble(GridL g, const double *__restrict__ etab, const double *__restrict__ etap,
                                  double *__restrict__ M, int n) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;  // column (unit vector)
    const int r = blockIdx.y;                              // row
    if (c >= n) return;
    const UnitVX ux{g, c};
    const UnitVY uy{g, c};
    const int nvx = g.ncy * (g.ncx - 1);
    double v;
    if (r < nvx) {
        const int i = r / (g.ncx - 1) + 1, j = r % (g.ncx - 1) + 1;
        v = lx_row(g, etab, etap, ux, uy, i, j);
    } else {
        const int rr = r - nvx;
        const int i = rr / g.ncx + 1, j = rr % g.ncx + 1;
        v = ly_row(g, etab, etap, ux, uy, i, j);
    }
    M[(size_t)r * n + c] = -v;  // -L_c (SPD)
}
// Gauss-Jordan inverse of the SPD matrix M (n x n, row-major), one CTA; no pivoting needed
// for SPD.  A = [M | I] in `work` (n x 2n).  Setup-time only.
__global__ void __launch_bounds__(1024) k_coarse_invert(double *__restrict__ work, double *__restrict__ Minv, int n,
                                                        int *fail) {
    extern __shared__ double sm[];
    double *colk = sm;       // n
    double *rowk = sm + n;   // 2n
    const int n2 = 2 * n;
    for (int k = 0; k < n; ++k) {
        const double piv = work[(size_t)k * n2 + k];
        if (!(piv > 0.0)) {
            if (threadIdx.x == 0) *fail = 1;
            return;
        }
        for (int t = threadIdx.x; t < n; t += blockDim.x) colk[t] = work[(size_t)t * n2 + k];
        for (int t = threadIdx.x; t < n2; t += blockDim.x) rowk[t] = work[(size_t)k * n2 + t] / piv;
        __syncthreads();
        for (size_t e = threadIdx.x; e < (size_t)n * n2; e += blockDim.x) {
            const int r = (int)(e / n2), cc = (int)(e % n2);
            if (r == k) work[e] = rowk[cc];
            else work[e] -= colk[r] * rowk[cc];
        }
        __syncthreads();
    }
    for (size_t e = threadIdx.x; e < (size_t)n * n; e += blockDim.x) {
        const int r = (int)(e / n), cc = (int)(e % n);
        Minv[e] = work[(size_t)r * n2 + n + cc];
    }
}
// v = L_c^-1 b = -(-L_c)^-1 b on the coarsest unknowns; mirrors written.
__device__ __forceinline__ void coarse_solve_cta(const GridL &g, const double *__restrict__ Minv, int n,
                                                 const double *__restrict__ bx, const double *__restrict__ by,
                                                 double *__restrict__ vx, double *__restrict__ vy, double *u) {
    const int nvx = g.ncy * (g.ncx - 1);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        if (k < nvx) u[k] = bx[at(g, k / (g.ncx - 1) + 1, k % (g.ncx - 1) + 1)];
        else u[k] = by[at(g, (k - nvx) / g.ncx + 1, (k - nvx) % g.ncx + 1)];
    }
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        double s = 0.0;
        for (int c = 0; c < n; ++c) s += Minv[(size_t)r * n + c] * u[c];
        const double v = -s;
        if (r < nvx) {
            const int i = r / (g.ncx - 1) + 1, j = r % (g.ncx - 1) + 1;
            vx[at(g, i, j)] = v;
            if (i == 1 && g.bN) vx[at(g, 0, j)] = g.sN * v;
            if (i == g.ncy && g.bS) vx[at(g, g.ncy + 1, j)] = g.sS * v;
        } else {
            const int i = (r - nvx) / g.ncx + 1, j = (r - nvx) % g.ncx + 1;
            vy[at(g, i, j)] = v;
            if (j == 1 && g.bW) vy[at(g, i, 0)] = g.sW * v;
            if (j == g.ncx && g.bE) vy[at(g, i, g.ncx + 1)] = g.sE * v;
        }
    }
}
__global__ void __launch_bounds__(256) k_coarse_solve(GridL g, const double *__restrict__ Minv, int n,
                                                      const double *__restrict__ bx, const double *__restrict__ by,
                                                      double *__restrict__ vx, double *__restrict__ vy) {
    extern __shared__ double u[];
    coarse_solve_cta(g, Minv, n, bx, by, vx, vy, u);
}

// ------------------------------------------------------------------ coarse tail (a9)
// The V-cycle from a small level down to the coarsest and back in ONE CTA: the same point
// operations as the per-level kernels (damped Jacobi with a zero first iterate, residual,
// velocity restriction, direct coarsest solve, prolongation + correction) in the host
// V-cycle's order, with a CTA barrier between stages instead of a kernel boundary.  Below
// ~32^2 cells a level's kernels are launch-latency bound (~2.5 us each, 12-13 per level);
// here a sweep of a 32^2 level is one point per thread.
__device__ __forceinline__ RhsArgs make_rhs_arrays(const double *bx, const double *by) {
    RhsArgs r;
    r.mode = RHS_ARRAYS;
    r.bx = bx;
    r.by = by;
    r.p = nullptr;
    r.rho = nullptr;
    r.gx = r.gy = 0.0;
    return r;
}
// COOP = false: the whole tail in ONE CTA (levels <= 32^2, k_vtail).  COOP = true: the same
// stages over a cooperative grid of one 1024-thread CTA per SM with a grid-wide barrier
// between stages (levels <= STOKES_COOP_CELLS, default 512^2): a level's ~13 kernels of a
// few microseconds of work each, which the per-level kernels spend mostly on launch and
// pipeline fill, become stages separated by grid syncs.
template <bool COOP>
__device__ __forceinline__ void tsync() {
    if (COOP) cooperative_groups::this_grid().sync();
    else __syncthreads();
}
__device__ __forceinline__ void tail_copy(const GridL &g, const double *src, double *dst, int t0, int nt) {
    const int n = (g.ncy + 2) * g.P;  // padded rows (mirrors included)
    for (int e = t0; e < n; e += nt) dst[e - COL_OFF] = src[e - COL_OFF];
}
template <bool COOP>
__global__ void __launch_bounds__(1024) k_vtail(TailArgs a, const double *__restrict__ Minv, int n, double omega) {
    extern __shared__ double u[];
    double *cx[TAIL_MAXL], *cy[TAIL_MAXL], *ox[TAIL_MAXL], *oy[TAIL_MAXL];
    const int t0 = COOP ? blockIdx.x * blockDim.x + threadIdx.x : threadIdx.x;
    const int nt = COOP ? gridDim.x * blockDim.x : blockDim.x;
    auto sweeps = [&](int l, int nsw, bool zero_first) {
        const TailLevel &L = a.lev[l];
        const RhsArgs rhs = make_rhs_arrays(L.bx, L.by);
        const int np = L.g.ncx * L.g.ncy;
        for (int s = 0; s < nsw; ++s) {
            for (int q = t0; q < np; q += nt) {
                const int i = q / L.g.ncx + 1, j = q % L.g.ncx + 1;
                if (zero_first && s == 0) jacobi_pt<true>(L.g, L.etab, L.etap, cx[l], cy[l], ox[l], oy[l], rhs, omega, i, j);
                else jacobi_pt<false>(L.g, L.etab, L.etap, cx[l], cy[l], ox[l], oy[l], rhs, omega, i, j);
            }
            tsync<COOP>();
            double *t = cx[l]; cx[l] = ox[l]; ox[l] = t;
            t = cy[l]; cy[l] = oy[l]; oy[l] = t;
        }
    };
    const int last = a.nl - 1;
    for (int l = 0; l < last; ++l) {  // down: pre-smoothing, residual, restriction
        const TailLevel &L = a.lev[l], &C = a.lev[l + 1];
        cx[l] = L.ax; cy[l] = L.ay; ox[l] = L.sx; oy[l] = L.sy;
        sweeps(l, L.nu, true);
        const RhsArgs rhs = make_rhs_arrays(L.bx, L.by);
        const int np = L.g.ncx * L.g.ncy;
        for (int q = t0; q < np; q += nt)
            residual_pt(L.g, L.etab, L.etap, cx[l], cy[l], rhs, L.rx, L.ry, q / L.g.ncx + 1, q % L.g.ncx + 1);
        tsync<COOP>();
        const int nc = C.g.ncx * C.g.ncy;
        for (int q = t0; q < nc; q += nt)
            restrict_vel_pt(L.g, C.g, L.rx, L.ry, C.bx, C.by, q / C.g.ncx + 1, q % C.g.ncx + 1);
        tsync<COOP>();
    }
    {  // coarsest: direct solve into its (ax, ay) (one CTA)
        const TailLevel &L = a.lev[last];
        if (!COOP || blockIdx.x == 0) coarse_solve_cta(L.g, Minv, n, L.bx, L.by, L.ax, L.ay, u);
        tsync<COOP>();
    }
    for (int l = last - 1; l >= 0; --l) {  // up: prolongation + correction, post-smoothing
        const TailLevel &L = a.lev[l], &C = a.lev[l + 1];
        const int np = L.g.ncx * L.g.ncy;
        for (int q = t0; q < np; q += nt)
            prolong_pt(L.g, C.g, C.ax, C.ay, cx[l], cy[l], q / L.g.ncx + 1, q % L.g.ncx + 1);
        tsync<COOP>();
        sweeps(l, L.nu, false);
        if (cx[l] != L.ax) {  // an odd number of buffer swaps: result back to (ax, ay)
            tail_copy(L.g, cx[l], L.ax, t0, nt);
            tail_copy(L.g, cy[l], L.ay, t0, nt);
            tsync<COOP>();
        }
    }
}

// ------------------------------------------------------------------ GCR vector kernels (a11)
// Euclidean inner products over the unknowns (vx, vy, p) (reading R13), nd pairs at once.
constexpr int MAXD = 12;
struct DotArgs {
    const double *a[MAXD][3];
    const double *b[MAXD][3];
    int nd;
};
__global__ void __launch_bounds__(BX *BY) k_dots(GridL g, DotArgs d, double *__restrict__ partials) {
    __shared__ double sh[BX * BY / 32];
    const int j = blockIdx.x * BX + threadIdx.x + 1;
    const int i = blockIdx.y * BY + threadIdx.y + 1;
    const bool in = (i <= g.ncy && j <= g.ncx);
    const size_t q = in ? at(g, i, j) : 0;
    const size_t blk = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
    for (int k = 0; k < d.nd; ++k) {
        double s = 0.0;
        if (in) {
            if (j < g.ncx) s += d.a[k][0][q] * d.b[k][0][q];
            if (i < g.ncy) s += d.a[k][1][q] * d.b[k][1][q];
            s += d.a[k][2][q] * d.b[k][2][q];
        }
        s = block_sum<BX * BY>(s, sh);
        if (threadIdx.x == 0 && threadIdx.y == 0) partials[blk * d.nd + k] = s;
    }
}
// y += sign * coef[idx] * x over unknowns (+ mirrors of velocity, linear)
__global__ void __launch_bounds__(BX *BY) k_axpy3(GridL g, const double *__restrict__ coef, int idx, double sgn,
                                                  const double *__restrict__ xx, const double *__restrict__ xy,
                                                  const double *__restrict__ xp, double *__restrict__ yx,
                                                  double *__restrict__ yy, double *__restrict__ yp) {
    const int j = blockIdx.x * BX + threadIdx.x;  // include mirrors: 0..ncx+1
    const int i = blockIdx.y * BY + threadIdx.y;
    if (i > g.ncy + 1 || j > g.ncx + 1) return;
    const double a = sgn * coef[idx];
    const size_t q = at(g, i, j);
    if (j >= 1 && j <= g.ncx - 1) yx[q] += a * xx[q];                    // vx unknowns + mirror rows
    if (i >= 1 && i <= g.ncy - 1) yy[q] += a * xy[q];                    // vy unknowns + mirror cols
    if (i >= 1 && i <= g.ncy && j >= 1 && j <= g.ncx) yp[q] += a * xp[q];  // P
}
__global__ void __launch_bounds__(BX *BY) k_scale3(GridL g, const double *__restrict__ coef, int invert_sqrt,
                                                   double *__restrict__ x, double *__restrict__ y,
                                                   double *__restrict__ p) {
    const int j = blockIdx.x * BX + threadIdx.x;
    const int i = blockIdx.y * BY + threadIdx.y;
    if (i > g.ncy + 1 || j > g.ncx + 1) return;
    const double a = invert_sqrt ? 1.0 / sqrt(coef[0]) : coef[0];
    const size_t q = at(g, i, j);
    if (j >= 1 && j <= g.ncx - 1) x[q] *= a;
    if (i >= 1 && i <= g.ncy - 1) y[q] *= a;
    if (i >= 1 && i <= g.ncy && j >= 1 && j <= g.ncx) p[q] *= a;
}
// z_p = alpha eta_P (r_p - D z_v) (preconditioner M^-1, reading R3/R14) + partial sums
__global__ void __launch_bounds__(BX *BY) k_precond_p(GridL g, const double *__restrict__ etap,
                                                      const double *__restrict__ zx, const double *__restrict__ zy,
                                                      const double *__restrict__ rp, double alpha,
                                                      double *__restrict__ zp, double *__restrict__ partials) {
    __shared__ double sh[BX * BY / 32];
    const int j = blockIdx.x * BX + threadIdx.x + 1;
    const int i = blockIdx.y * BY + threadIdx.y + 1;
    double s = 0.0;
    if (i <= g.ncy && j <= g.ncx) {
        const double dz = (zx[at(g, i, j)] - zx[at(g, i, j - 1)]) * g.idx + (zy[at(g, i, j)] - zy[at(g, i - 1, j)]) * g.idy;
        const double v = alpha * etap[at(g, i, j)] * (rp[at(g, i, j)] - dz);
        zp[at(g, i, j)] = v;
        s = v;
    }
    s = block_sum<BX * BY>(s, sh);
    if (threadIdx.x == 0 && threadIdx.y == 0) partials[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
}
__global__ void k_sub_mean(GridL g, const double *__restrict__ mean, double *__restrict__ p) {
    const int j = blockIdx.x * BX + threadIdx.x + 1, i = blockIdx.y * BY + threadIdx.y + 1;
    if (i <= g.ncy && j <= g.ncx) p[at(g, i, j)] -= *mean;
}


// ------------------------------------------------------------------ 2D decomposition helpers (§8(e))
// strided strip copies (halo columns / rows, packing for the transports): one CTA per strip
constexpr int MAXSTRIP = 48;
struct Strips {
    double *dst[MAXSTRIP];
    const double *src[MAXSTRIP];
    int n[MAXSTRIP];
    int dstride[MAXSTRIP], sstride[MAXSTRIP];
    int count;
};
__global__ void k_strip_copy(Strips s) {
    const int k = blockIdx.y;
    if (k >= s.count) return;
    double *d = s.dst[k];
    const double *a = s.src[k];
    const int ds = s.dstride[k], ss = s.sstride[k];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < s.n[k]; e += gridDim.x * blockDim.x)
        d[(size_t)e * ds] = a[(size_t)e * ss];
}
// sum of the tiles' local (Sv, Sp, sum p) triples in tile order (deterministic)
struct Ptrs {
    const double *p[64];
    double *q[64];
    int n;
};
__global__ void k_dist_final(Ptrs loc, const double *__restrict__ Sf, double inv_np, double *__restrict__ out,
                             Ptrs mshift, int write_mean) {
    if (threadIdx.x != 0) return;
    double sv = 0.0, sp = 0.0, ps = 0.0;
    for (int t = 0; t < loc.n; ++t) {
        sv += loc.p[t][0];
        sp += loc.p[t][1];
        ps += loc.p[t][2];
    }
    out[0] = (Sf[0] > 0.0) ? sqrt((sv + sp) / Sf[0]) : 0.0;
    out[1] = sv;
    out[2] = sp;
    if (write_mean)
        for (int t = 0; t < mshift.n; ++t) *mshift.q[t] = ps * inv_np;
}

}  // namespace

// ====================================================================== launchers
#define LAUNCH_BOOK(c) (++*(c).counter)
static inline dim3 tpb() { return dim3(BX, BY); }

void launch_jacobi(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, const double *vxi,
                   const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs, double omega, bool zero_in) {
    if (!zero_in && stream_ok(g)) {
        launch_jacobi_stream(c, g, etab, etap, vxi, vyi, vxo, vyo, rhs, omega);
        return;
    }
    if (zero_in) k_jacobi<true><<<cell_grid(g), tpb(), 0, c.stream>>>(g, etab, etap, vxi, vyi, vxo, vyo, rhs, omega);
    else k_jacobi<false><<<cell_grid(g), tpb(), 0, c.stream>>>(g, etab, etap, vxi, vyi, vxo, vyo, rhs, omega);
    LAUNCH_BOOK(c);
}
bool launch_jacobi_tile(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                        const double *vxi, const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs,
                        double omega, int n, bool zero_in, const GridL *gc, const double *ex, const double *ey) {
    if (ex && (zero_in || !gc)) return false;
    if (rhs.mode != RHS_ARRAYS || n < 1 || n > TT_MAXN || !(g.bN && g.bS && g.bW && g.bE)) return false;
    static unsigned long long done = 0;
    if (first_on_device(&done)) {
        const int most = 8 * tt_rows(TT_MAXN) * tt_cols(TT_MAXN) * 8;
        cudaFuncSetAttribute(k_jacobi_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, most);
        cudaFuncSetAttribute(k_jacobi_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, most);
    }
    const int smem = 8 * tt_rows(n) * tt_cols(n) * 8;
    const dim3 grid((g.ncx + TTC - 1) / TTC, (g.ncy + TTR - 1) / TTR);
    if (zero_in)
        k_jacobi_tile<true><<<grid, TTN, smem, c.stream>>>(g, etab, etap, vxi, vyi, vxo, vyo, rhs.bx, rhs.by,
                                                           omega, n, g, nullptr, nullptr);
    else
        k_jacobi_tile<false><<<grid, TTN, smem, c.stream>>>(g, etab, etap, vxi, vyi, vxo, vyo, rhs.bx, rhs.by,
                                                            omega, n, gc ? *gc : g, ex, ey);
    LAUNCH_BOOK(c);
    return true;
}
void launch_rbgs(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, double *vx, double *vy,
                 const RhsArgs &rhs, double omega) {
    const dim3 grid((g.ncx / 2 + 1 + BX - 1) / BX, (g.ncy + BY - 1) / BY);
    for (int comp = 0; comp < 2; ++comp)
        for (int colour = 0; colour < 2; ++colour) {
            k_rbgs_phase<<<grid, tpb(), 0, c.stream>>>(g, etab, etap, vx, vy, rhs, omega, comp, colour);
            LAUNCH_BOOK(c);
        }
}
void launch_residual(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, const double *vx,
                     const double *vy, const RhsArgs &rhs, double *rx, double *ry) {
    if (stream_ok(g)) {
        launch_residual_stream(c, g, etab, etap, vx, vy, rhs, rx, ry);
        return;
    }
    k_residual<<<cell_grid(g), tpb(), 0, c.stream>>>(g, etab, etap, vx, vy, rhs, rx, ry);
    LAUNCH_BOOK(c);
}
void launch_restrict_vel(const LaunchCtx &c, const GridL &gf, const GridL &gc, const double *rx, const double *ry,
                         double *bxc, double *byc) {
    k_restrict_vel<<<cell_grid(gc), tpb(), 0, c.stream>>>(gf, gc, rx, ry, bxc, byc);
    LAUNCH_BOOK(c);
}
void launch_restrict_vx(const LaunchCtx &c, const GridL &gf, const GridL &gc, const double *f, double *cc) {
    launch_restrict_vel(c, gf, gc, f, nullptr, cc, nullptr);
}
void launch_restrict_vy(const LaunchCtx &c, const GridL &gf, const GridL &gc, const double *f, double *cc) {
    launch_restrict_vel(c, gf, gc, nullptr, f, nullptr, cc);
}
void launch_restrict_b(const LaunchCtx &c, const GridL &gf, const GridL &gc, const double *f, double *cc) {
    const dim3 grid((gc.ncx + 1 + BX - 1) / BX, (gc.ncy + 1 + BY - 1) / BY);
    k_restrict_b<<<grid, tpb(), 0, c.stream>>>(gf, gc, f, cc);
    LAUNCH_BOOK(c);
}
void launch_restrict_p(const LaunchCtx &c, const GridL &gf, const GridL &gc, const double *f, double *cc) {
    k_restrict_p<<<cell_grid(gc), tpb(), 0, c.stream>>>(gf, gc, f, cc);
    LAUNCH_BOOK(c);
}
void launch_prolong(const LaunchCtx &c, const GridL &gf, const GridL &gc, const double *exc, const double *eyc,
                    double *vx, double *vy) {
    if (gf.ncx % 2 == 0) {  // paired columns (single domain and decomposed tiles)
        const dim3 grid((gf.ncx / 2 + BX - 1) / BX, (gf.ncy + BY - 1) / BY);
        k_prolong2<<<grid, tpb(), 0, c.stream>>>(gf, gc, exc, eyc, vx, vy);
    } else {
        k_prolong<<<cell_grid(gf), tpb(), 0, c.stream>>>(gf, gc, exc, eyc, vx, vy);
    }
    LAUNCH_BOOK(c);
}
int energy_blocks(const GridL &g) {
    const dim3 gr = cell_grid(g);
    return (int)(gr.x * gr.y);
}
void launch_energy(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, const double *vx,
                   const double *vy, const double *p, const double *rho, double gx, double gy, double *rx,
                   double *ry, double *rp, double *partials, bool force_only) {
    k_energy<<<cell_grid(g), tpb(), 0, c.stream>>>(g, etab, etap, vx, vy, p, rho, gx, gy, rx, ry, rp, partials,
                                                   force_only ? 1 : 0);
    LAUNCH_BOOK(c);
}
void launch_energy_vec(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, const double *rx,
                       const double *ry, const double *rp, double *partials) {
    k_energy_vec<<<cell_grid(g), tpb(), 0, c.stream>>>(g, etab, etap, rx, ry, rp, partials);
    LAUNCH_BOOK(c);
}
int pupdate_blocks(const GridL &g) { return energy_blocks(g); }
void launch_pupdate(const LaunchCtx &c, const GridL &g, const double *etap, const double *vx, const double *vy,
                    const double *pin, double *pout, double alpha_signed, const double *mshift, double *partials) {
    k_pupdate<<<cell_grid(g), tpb(), 0, c.stream>>>(g, etap, vx, vy, pin, pout, alpha_signed, mshift, partials);
    LAUNCH_BOOK(c);
}
void launch_finalize(const LaunchCtx &c, const double *partials, int nblocks, int ncomp, double scale, double *out) {
    k_finalize<<<1, 1024, 0, c.stream>>>(partials, nblocks, ncomp, scale, out);
    LAUNCH_BOOK(c);
}
void launch_energy_final(const LaunchCtx &c, const double *partials, int nblocks, const double *Sf, double *out) {
    k_energy_final<<<1, 1024, 0, c.stream>>>(partials, nblocks, Sf, out);
    LAUNCH_BOOK(c);
}
void launch_uzawa_final(const LaunchCtx &c, const double *partials, int nblocks, const double *Sf, double inv_np,
                        double *out, double *mean) {
    k_uzawa_final<<<1, 1024, 0, c.stream>>>(partials, nblocks, Sf, inv_np, out, mean);
    LAUNCH_BOOK(c);
}
void launch_in_velocity(const LaunchCtx &c, const GridL &g, const double *ux, const double *uy, double *vx,
                        double *vy) {
    const dim3 grid((g.ncx + 2 + BX - 1) / BX, (g.ncy + 2 + BY - 1) / BY);
    k_in_velocity<<<grid, tpb(), 0, c.stream>>>(g, ux, uy, vx, vy);
    LAUNCH_BOOK(c);
}
void launch_in_p(const LaunchCtx &c, const GridL &g, const double *u, double *a) {
    k_in_p<<<cell_grid(g), tpb(), 0, c.stream>>>(g, u, a);
    LAUNCH_BOOK(c);
}
static inline dim3 node_grid(const GridL &g) { return dim3((g.ncx + 1 + BX - 1) / BX, (g.ncy + 1 + BY - 1) / BY); }
void launch_in_b(const LaunchCtx &c, const GridL &g, const double *u, double *a) {
    k_in_b<<<node_grid(g), tpb(), 0, c.stream>>>(g, u, a);
    LAUNCH_BOOK(c);
}
void launch_in_vx_raw(const LaunchCtx &c, const GridL &g, const double *u, double *a) {
    k_in_vx_raw<<<node_grid(g), tpb(), 0, c.stream>>>(g, u, a);
    LAUNCH_BOOK(c);
}
void launch_in_vy_raw(const LaunchCtx &c, const GridL &g, const double *u, double *a) {
    k_in_vy_raw<<<node_grid(g), tpb(), 0, c.stream>>>(g, u, a);
    LAUNCH_BOOK(c);
}
void launch_out_vx(const LaunchCtx &c, const GridL &g, const double *a, double *u) {
    k_out_vx<<<node_grid(g), tpb(), 0, c.stream>>>(g, a, u);
    LAUNCH_BOOK(c);
}
void launch_out_vy(const LaunchCtx &c, const GridL &g, const double *a, double *u) {
    k_out_vy<<<node_grid(g), tpb(), 0, c.stream>>>(g, a, u);
    LAUNCH_BOOK(c);
}
void launch_out_p(const LaunchCtx &c, const GridL &g, const double *a, double *u, const double *shift) {
    k_out_p<<<cell_grid(g), tpb(), 0, c.stream>>>(g, a, u, shift);
    LAUNCH_BOOK(c);
}
void launch_out_b(const LaunchCtx &c, const GridL &g, const double *a, double *u) {
    k_out_b<<<node_grid(g), tpb(), 0, c.stream>>>(g, a, u);
    LAUNCH_BOOK(c);
}
void launch_apply(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, const double *vx,
                  const double *vy, const double *p, double *ax, double *ay, double *ap) {
    k_apply<<<cell_grid(g), tpb(), 0, c.stream>>>(g, etab, etap, vx, vy, p, ax, ay, ap);
    LAUNCH_BOOK(c);
}
void launch_apply_padded(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                         const double *vx, const double *vy, const double *p, double *ax, double *ay, double *ap) {
    k_apply_padded<<<cell_grid(g), tpb(), 0, c.stream>>>(g, etab, etap, vx, vy, p, ax, ay, ap);
    LAUNCH_BOOK(c);
}
void launch_refresh_mirrors(const LaunchCtx &c, const GridL &g, double *vx, double *vy) {
    const int n = (g.ncx > g.ncy ? g.ncx : g.ncy) + 1;
    k_refresh_mirrors<<<(n + 255) / 256, 256, 0, c.stream>>>(g, vx, vy);
    LAUNCH_BOOK(c);
}
void launch_energy_weights(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, double *ewx,
                           double *ewy, double *ewp) {
    k_energy_weights<<<cell_grid(g), tpb(), 0, c.stream>>>(g, etab, etap, ewx, ewy, ewp);
    LAUNCH_BOOK(c);
}
void launch_make_rhs(const LaunchCtx &c, const GridL &g, const RhsArgs &rhs, double *bx, double *by) {
    k_make_rhs<<<cell_grid(g), tpb(), 0, c.stream>>>(g, rhs, bx, by);
    LAUNCH_BOOK(c);
}
void launch_count_nonpos(const LaunchCtx &c, const double *a, size_t n, int *count) {
    int blocks = (int)((n + 255) / 256);
    if (blocks > 4096) blocks = 4096;
    if (blocks < 1) blocks = 1;
    k_count_nonpos<<<blocks, 256, 0, c.stream>>>(a, n, count);
    LAUNCH_BOOK(c);
}
void launch_coarse_assemble(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, double *M) {
    const int n = g.ncy * (g.ncx - 1) + (g.ncy - 1) * g.ncx;
    k_coarse_assemble<<<dim3((n + 127) / 128, n), 128, 0, c.stream>>>(g, etab, etap, M, n);
    LAUNCH_BOOK(c);
}
__global__ void k_aug(const double *__restrict__ M, double *__restrict__ work, int n) {
    const size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (e >= (size_t)n * 2 * n) return;
    const int r = (int)(e / (2 * n)), cc = (int)(e % (2 * n));
    work[e] = cc < n ? M[(size_t)r * n + cc] : (cc - n == r ? 1.0 : 0.0);
}
void launch_coarse_invert(const LaunchCtx &c, double *work, double *Minv, int n, int *fail) {
    const size_t tot = (size_t)n * 2 * n;
    k_aug<<<(unsigned)((tot + 255) / 256), 256, 0, c.stream>>>(Minv, work, n);
    LAUNCH_BOOK(c);
    k_coarse_invert<<<1, 1024, 3 * n * sizeof(double), c.stream>>>(work, Minv, n, fail);
    LAUNCH_BOOK(c);
}
void launch_coarse_solve(const LaunchCtx &c, const GridL &g, const double *Minv, const double *bx,
                         const double *by, double *vx, double *vy) {
    const int n = g.ncy * (g.ncx - 1) + (g.ncy - 1) * g.ncx;
    k_coarse_solve<<<1, 256, n * sizeof(double), c.stream>>>(g, Minv, n, bx, by, vx, vy);
    LAUNCH_BOOK(c);
}
void launch_vtail(const LaunchCtx &c, const TailArgs &a, const double *Minv, int n, double omega) {
    k_vtail<false><<<1, 1024, n * sizeof(double), c.stream>>>(a, Minv, n, omega);
    LAUNCH_BOOK(c);
}
int launch_vtail_coop(const LaunchCtx &c, const TailArgs &a, const double *Minv, int n, double omega) {
    static int grid[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!grid[dev & 63]) {  // one wave of co-resident CTAs
        int nb = 0, nsm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_vtail<true>, 1024, n * sizeof(double));
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        grid[dev & 63] = (nb > 0 ? nb : 1) * nsm;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid[dev & 63]);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = n * sizeof(double);
    cfg.stream = c.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_vtail<true>, a, Minv, n, omega);
    LAUNCH_BOOK(c);
    return e == cudaSuccess ? 0 : -1;
}
int dot_blocks(const GridL &g) { return energy_blocks(g); }
void launch_dots(const LaunchCtx &c, const GridL &g, const double *const *a, const double *const *b, int nd,
                 double *partials) {
    DotArgs d;
    d.nd = nd;
    for (int k = 0; k < nd; ++k)
        for (int f = 0; f < 3; ++f) {
            d.a[k][f] = a[3 * k + f];
            d.b[k][f] = b[3 * k + f];
        }
    k_dots<<<cell_grid(g), tpb(), 0, c.stream>>>(g, d, partials);
    LAUNCH_BOOK(c);
}
void launch_axpy3(const LaunchCtx &c, const GridL &g, const double *coef, int coef_index, double coef_sign,
                  const double *xx, const double *xy, const double *xp, double *yx, double *yy, double *yp) {
    k_axpy3<<<dim3((g.ncx + 2 + BX - 1) / BX, (g.ncy + 2 + BY - 1) / BY), tpb(), 0, c.stream>>>(
        g, coef, coef_index, coef_sign, xx, xy, xp, yx, yy, yp);
    LAUNCH_BOOK(c);
}
void launch_scale3(const LaunchCtx &c, const GridL &g, const double *coef, int invert_sqrt, double *x, double *y,
                   double *p) {
    k_scale3<<<dim3((g.ncx + 2 + BX - 1) / BX, (g.ncy + 2 + BY - 1) / BY), tpb(), 0, c.stream>>>(g, coef, invert_sqrt,
                                                                                                x, y, p);
    LAUNCH_BOOK(c);
}
void launch_precond_p(const LaunchCtx &c, const GridL &g, const double *etap, const double *zx, const double *zy,
                      const double *rp, double alpha, double *zp, double *partials) {
    k_precond_p<<<cell_grid(g), tpb(), 0, c.stream>>>(g, etap, zx, zy, rp, alpha, zp, partials);
    LAUNCH_BOOK(c);
}
void launch_sub_mean(const LaunchCtx &c, const GridL &g, const double *mean, double *p) {
    k_sub_mean<<<cell_grid(g), tpb(), 0, c.stream>>>(g, mean, p);
    LAUNCH_BOOK(c);
}

void launch_eta_min(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                    unsigned long long *emin) {
    const dim3 grid((g.ncx + 1 + BX - 1) / BX, (g.ncy + 1 + BY - 1) / BY);
    k_eta_min<<<grid, tpb(), 0, c.stream>>>(g, etab, etap, emin);
    LAUNCH_BOOK(c);
}
void launch_eta_blend(const LaunchCtx &c, const GridL &g, const double *ebu, const double *epu, double *etab,
                      double *etap, const unsigned long long *emin, double theta) {
    const dim3 grid((g.ncx + 1 + BX - 1) / BX, (g.ncy + 1 + BY - 1) / BY);
    k_eta_blend<<<grid, tpb(), 0, c.stream>>>(g, ebu, epu, etab, etap, emin, theta);
    LAUNCH_BOOK(c);
}
void launch_lithostatic(const LaunchCtx &c, const GridL &g, const double *rho, double gy, double *p) {
    k_lithostatic<<<(g.ncx + 127) / 128, 128, 0, c.stream>>>(g, rho, gy, p);
    LAUNCH_BOOK(c);
}
void launch_rbgs_phase(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, double *vx,
                       double *vy, const RhsArgs &rhs, double omega, int comp, int colour) {
    const dim3 grid((g.ncx / 2 + 1 + BX - 1) / BX, (g.ncy + BY - 1) / BY);
    k_rbgs_phase<<<grid, tpb(), 0, c.stream>>>(g, etab, etap, vx, vy, rhs, omega, comp, colour);
    LAUNCH_BOOK(c);
}
void launch_strips(const LaunchCtx &c, const StripList &l) {
    for (int base = 0; base < l.count; base += MAXSTRIP) {
        Strips s;
        s.count = 0;
        int nmax = 1;
        for (int k = base; k < l.count && s.count < MAXSTRIP; ++k, ++s.count) {
            s.dst[s.count] = l.dst[k];
            s.src[s.count] = l.src[k];
            s.n[s.count] = l.n[k];
            s.dstride[s.count] = l.dstride[k];
            s.sstride[s.count] = l.sstride[k];
            if (l.n[k] > nmax) nmax = l.n[k];
        }
        int bx = (nmax + 255) / 256;
        if (bx > 16) bx = 16;
        k_strip_copy<<<dim3(bx, s.count), 256, 0, c.stream>>>(s);
        LAUNCH_BOOK(c);
    }
}
// the mean of nseg segments of nb per-CTA partial sums (segment s at base + s * stride):
// one CTA, a fixed order (lane-strided per segment, then the fixed shuffle tree), so every
// tile that reduces the same buffer gets the same value (decomposed Anderson, dist.cu)
__global__ void __launch_bounds__(256) k_dist_mean(const double *__restrict__ base, int nseg, int nb, size_t stride,
                                                   double inv_np, double *__restrict__ out) {
    __shared__ double sh[8];
    double v = 0.0;
    for (int sg = 0; sg < nseg; ++sg)
        for (int b = threadIdx.x; b < nb; b += 256) v += base[(size_t)sg * stride + b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += sh[w];
        *out = t * inv_np;
    }
}
void launch_dist_mean(const LaunchCtx &c, const double *base, int nseg, int nb, size_t stride, double inv_np,
                      double *out) {
    k_dist_mean<<<1, 256, 0, c.stream>>>(base, nseg, nb, stride, inv_np, out);
    LAUNCH_BOOK(c);
}
void launch_dist_final(const LaunchCtx &c, const double *const *loc, int nloc, const double *Sf, double inv_np,
                       double *out, double *const *mshift, int nm) {
    Ptrs a, b;
    a.n = nloc;
    for (int t = 0; t < nloc; ++t) a.p[t] = loc[t];
    b.n = nm;
    for (int t = 0; t < nm; ++t) b.q[t] = mshift[t];
    k_dist_final<<<1, 32, 0, c.stream>>>(a, Sf, inv_np, out, b, nm > 0);
    LAUNCH_BOOK(c);
}
