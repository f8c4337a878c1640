// Marker-in-cell transfers and marker advection, FP64, sm_100a.
//
//   stokes_markers_to_grid  PAPER.md:467-495 (§4.2 "Marker-to-grid interpolation"): eta_b,
//                           rho_b on basic nodes and eta_p on pressure nodes as weighted
//                           averages of the marker values with the bilinear weights of
//                           PAPER.md:480-484 (reading R28).
//   stokes_grid_to_markers  PAPER.md:497-511: velocity at the markers (R29).
//   stokes_advect_markers   PAPER.md:560-600: Euler / Heun / RK4 (Listing rk4_agnostic order,
//                           PAPER.md:2226-2254), locally polynomial order 2 / 3 (R32),
//                           closed-box clamping (R30).
//   stokes_marker_timestep  PAPER.md:526-532 CFL-like step (R31).
//
// Determinism (the paper's scatter-add with atomics, is order-dependent):
// the marker -> grid sums are GATHERS.  Markers are binned by the reference cell of each
// target grid (integer-atomic counting sort: histogram -> exclusive scan -> scatter), each
// bin's index list is sorted ascending, and every node merges the (up to) four bins that
// touch it in ascending MARKER INDEX -- exactly the order in which the paper's serial loop
// over markers adds into that node.  Products and sums use explicitly rounded intrinsics
// (no FMA contraction), so the result is bit-identical to the plain CPU loop.
//
// Data in HBM per call (n markers, user layouts of include/stokes.h): x, y, eta, rho read;
// per target grid a sorted index list + a 32-B record (t_x, t_y, eta, rho) -- t = offset of
// the marker from its reference node / spacing, computed once -- then a gather per node.
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "handle.h"

namespace {

struct MkGrid {
    int nx, ny;
    double Lx, Ly, dx, dy, hx, hy;  // hx = 0.5 dx, hy = 0.5 dy: offsets of the staggered grids
    double rdx, rdy;                // RN(1/dx), RN(1/dy): floor of the quotient without a division
    double sW, sE, sN, sS;          // mirror signs (free slip +1, no slip -1)
};

constexpr int TPB = 256;
constexpr int SCAN_T = 1024;          // threads of the scan kernels
constexpr int SCAN_TILE = 4 * SCAN_T;  // elements per scan tile

__device__ __forceinline__ double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

// floor(RN(a / h)) -- the oracle's floor of the correctly rounded quotient -- from the product
// q = RN(a * RN(1/h)): |q - a/h| <= |a/h| (2^-52 + 2^-106), so floor(q) can differ from
// floor(RN(a/h)) only when a/h lies within ~3.4e-16 |a/h| of an integer; any q within
// 1e-9 max(1, |q|) of an integer takes the IEEE division instead (rare), so the result is
// always identical to the division's.
__device__ __forceinline__ int floor_quot(double a, double h, double rh) {
    const double q = __dmul_rn(a, rh);
    const double n = rint(q);
    if (fabs(q - n) <= 1e-9 * fmax(1.0, fabs(q))) return (int)floor(__ddiv_rn(a, h));
    return (int)floor(q);
}
// Reference node of a grid whose node k sits at k h + o (R28): k = floor((x - o)/h) clamped to
// [kmin, kmax]; t = (x - (k h + o)) / h.  The exact operation sequence of the oracle.
__device__ __forceinline__ int ref_node(double x, double h, double rh, double o, int kmin, int kmax, double &t) {
    int k = floor_quot(__dsub_rn(x, o), h, rh);
    k = k < kmin ? kmin : (k > kmax ? kmax : k);
    double xn = __dadd_rn(__dmul_rn((double)k, h), o);
    t = __ddiv_rn(__dsub_rn(x, xn), h);
    return k;
}
__device__ __forceinline__ int ref_only(double x, double h, double rh, double o, int kmin, int kmax) {
    int k = floor_quot(__dsub_rn(x, o), h, rh);
    return k < kmin ? kmin : (k > kmax ? kmax : k);
}

// bins: basic grid -> reference cell (ir, jr) in [0,ny) x [0,nx), index ir*nx + jr;
//       P grid     -> reference P node (ir, jr) in [-1,ny) x [-1,nx), index (ir+1)*(nx+1) + jr+1
__device__ __forceinline__ void marker_bins(const MkGrid &G, double x, double y, int &bb, int &bp) {
    x = clampd(x, 0.0, G.Lx);
    y = clampd(y, 0.0, G.Ly);
    int jb = ref_only(x, G.dx, G.rdx, 0.0, 0, G.nx - 1), ib = ref_only(y, G.dy, G.rdy, 0.0, 0, G.ny - 1);
    int jp = ref_only(x, G.dx, G.rdx, G.hx, -1, G.nx - 1), ip = ref_only(y, G.dy, G.rdy, G.hy, -1, G.ny - 1);
    bb = ib * G.nx + jb;
    bp = (ip + 1) * (G.nx + 1) + (jp + 1);
}

// warp-aggregated integer atomicAdd: lanes with equal address share one atomic; each lane gets
// base + (number of lower lanes with the same address).
__device__ __forceinline__ int agg_add(int *addr, unsigned active) {
    unsigned peers = __match_any_sync(active, (unsigned long long)addr);
    int leader = __ffs(peers) - 1;
    int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == leader) base = atomicAdd(addr, __popc(peers));
    base = __shfl_sync(peers, base, leader);
    return base + __popc(peers & ((1u << lane) - 1));
}

__global__ void k_mk_count(long long n, const double *__restrict__ x, const double *__restrict__ y, MkGrid G,
                           int *__restrict__ cntB, int *__restrict__ cntP) {
    long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned active = __ballot_sync(~0u, m < n);
    if (m >= n) return;
    int bb, bp;
    marker_bins(G, x[m], y[m], bb, bp);
    agg_add(cntB + bb, active);
    agg_add(cntP + bp, active);
}

__global__ void k_mk_scatter(long long n, const double *__restrict__ x, const double *__restrict__ y, MkGrid G,
                             int *__restrict__ fillB, int *__restrict__ fillP, int *__restrict__ sidxB,
                             int *__restrict__ sidxP) {
    long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned active = __ballot_sync(~0u, m < n);
    if (m >= n) return;
    int bb, bp;
    marker_bins(G, x[m], y[m], bb, bp);
    sidxB[agg_add(fillB + bb, active)] = (int)m;
    sidxP[agg_add(fillP + bp, active)] = (int)m;
}

// ---- exclusive scan of the bin counts (3 kernels, 1024-thread blocks)
__device__ int block_excl_scan(int v, int &total) {
    __shared__ int ws[32];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int s = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int t = __shfl_up_sync(~0u, s, d);
        if (lane >= d) s += t;
    }
    if (lane == 31) ws[wid] = s;
    __syncthreads();
    if (wid == 0) {
        int w = ws[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int t = __shfl_up_sync(~0u, w, d);
            if (lane >= d) w += t;
        }
        ws[lane] = w;
    }
    __syncthreads();
    int pre = (wid ? ws[wid - 1] : 0) + s - v;
    total = ws[31];
    __syncthreads();
    return pre;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_reduce(const int *__restrict__ cnt, int nb, int *__restrict__ tsum) {
    long long base = (long long)blockIdx.x * SCAN_TILE + threadIdx.x * 4;
    int s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (base + k < nb) s += cnt[base + k];
    int tot;
    block_excl_scan(s, tot);
    if (threadIdx.x == 0) tsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_top(int *__restrict__ tsum, int nt, int *__restrict__ off, int nb) {
    int chunk = (nt + SCAN_T - 1) / SCAN_T;
    int b0 = threadIdx.x * chunk;
    int s = 0;
    for (int k = 0; k < chunk; ++k)
        if (b0 + k < nt) s += tsum[b0 + k];
    int tot;
    int run = block_excl_scan(s, tot);
    for (int k = 0; k < chunk; ++k)
        if (b0 + k < nt) {
            int v = tsum[b0 + k];
            tsum[b0 + k] = run;
            run += v;
        }
    if (threadIdx.x == 0) off[nb] = tot;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_apply(const int *__restrict__ cnt, int nb, const int *__restrict__ tpre,
                                                       int *__restrict__ off, int *__restrict__ fill) {
    long long base = (long long)blockIdx.x * SCAN_TILE + threadIdx.x * 4;
    int v[4], s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = base + k < nb ? cnt[base + k] : 0;
        s += v[k];
    }
    int tot;
    int run = block_excl_scan(s, tot) + tpre[blockIdx.x];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (base + k < nb) {
            off[base + k] = run;
            fill[base + k] = run;
            run += v[k];
        }
}

// ---- per-bin ascending index order + sorted records.  One warp owns 32 consecutive bins:
// each lane insertion-sorts its bin's (short) index list, then the warp writes the records of
// the 32 bins' contiguous range coalesced.
template <bool BASIC>
__global__ void k_mk_records(int nbins, const int *__restrict__ off, int *__restrict__ sidx,
                             const double *__restrict__ x, const double *__restrict__ y,
                             const double *__restrict__ eta, const double *__restrict__ rho, MkGrid G,
                             double4 *__restrict__ rec) {
    int warp = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    int lane = threadIdx.x & 31;
    int b0 = warp * 32;
    if (b0 >= nbins) return;
    int b = b0 + lane;
    if (b < nbins) {
        int s = off[b], e = off[b + 1];
        for (int k = s + 1; k < e; ++k) {  // insertion sort (bins hold ~4-16 markers)
            int v = sidx[k];
            int q = k - 1;
            while (q >= s && sidx[q] > v) {
                sidx[q + 1] = sidx[q];
                --q;
            }
            sidx[q + 1] = v;
        }
    }
    __syncwarp();
    // RU records per lane per step, every load before the stores (the output may alias the
    // inputs as far as the compiler knows: loads after a store would wait for it)
    constexpr int RU = 4;
    const int r0 = off[b0], r1 = off[min(b0 + 32, nbins)];
    for (int k0 = r0 + lane; k0 < r1; k0 += 32 * RU) {
        int m[RU];
        double xv[RU], yv[RU], ev[RU], rv[RU];
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            const int k = k0 + 32 * u;
            m[u] = k < r1 ? sidx[k] : -1;
        }
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            if (m[u] < 0) continue;
            xv[u] = x[m[u]];
            yv[u] = y[m[u]];
            ev[u] = eta[m[u]];
            rv[u] = BASIC ? rho[m[u]] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            if (m[u] < 0) continue;
            const double xm = clampd(xv[u], 0.0, G.Lx), ym = clampd(yv[u], 0.0, G.Ly);
            double tx, ty;
            if (BASIC) {
                ref_node(xm, G.dx, G.rdx, 0.0, 0, G.nx - 1, tx);
                ref_node(ym, G.dy, G.rdy, 0.0, 0, G.ny - 1, ty);
            } else {
                ref_node(xm, G.dx, G.rdx, G.hx, -1, G.nx - 1, tx);
                ref_node(ym, G.dy, G.rdy, G.hy, -1, G.ny - 1, ty);
            }
            rec[k0 + 32 * u] = make_double4(tx, ty, ev[u], rv[u]);
        }
    }
}

// ---- gather: node (i, j) merges the four bins (ir, jr) = (i-1, j-1), (i-1, j), (i, j-1), (i, j)
// in ascending marker index; the node is corner (1,1), (1,0), (0,1), (0,0) of those bins and
// takes the weight x-factor * y-factor with factor t (corner 1) or 1 - t (corner 0), as
// w00..w11 of PAPER.md:480-484.  A CTA covers 32 x 8 nodes, each warp an 8 x 4 patch, so the
// four lanes that share a bin read its records together (L1 reuse instead of HBM re-reads).
constexpr int GX = 32, GY = 8;
template <bool BASIC>
__global__ void __launch_bounds__(256) k_mk_gather(MkGrid G, const int *__restrict__ off,
                                                   const int *__restrict__ sidx, const double4 *__restrict__ rec,
                                                   double *__restrict__ out_eta, double *__restrict__ out_rho,
                                                   unsigned long long *__restrict__ n_empty) {
    // basic: nodes (ny+1) x (nx+1), bins ny x nx (index ir*nx + jr)
    // P    : nodes ny x nx,         bins (ny+1) x (nx+1) (index (ir+1)*(nx+1) + jr+1)
    const int NW = BASIC ? G.nx + 1 : G.nx, NH = BASIC ? G.ny + 1 : G.ny;
    const int BW = BASIC ? G.nx : G.nx + 1, BH = BASIC ? G.ny : G.ny + 1;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int j = blockIdx.x * GX + (w & 3) * 8 + (lane & 7);
    const int i = blockIdx.y * GY + (w >> 2) * 4 + (lane >> 3);
    const bool live = i < NH && j < NW;
    // bin coordinates in the bin array (P bins are shifted by +1)
    const int bi = BASIC ? i : i + 1, bj = BASIC ? j : j + 1;
    int h0 = 0, e0 = 0, h1 = 0, e1 = 0, h2 = 0, e2 = 0, h3 = 0, e3 = 0;
    if (live) {
        if (bi - 1 >= 0 && bj - 1 >= 0) { int b = (bi - 1) * BW + bj - 1; h0 = off[b]; e0 = off[b + 1]; }
        if (bi - 1 >= 0 && bj < BW)     { int b = (bi - 1) * BW + bj;     h1 = off[b]; e1 = off[b + 1]; }
        if (bi < BH && bj - 1 >= 0)     { int b = bi * BW + bj - 1;       h2 = off[b]; e2 = off[b + 1]; }
        if (bi < BH && bj < BW)         { int b = bi * BW + bj;           h3 = off[b]; e3 = off[b + 1]; }
    }
    int c0 = h0 < e0 ? sidx[h0] : INT_MAX, c1 = h1 < e1 ? sidx[h1] : INT_MAX;
    int c2 = h2 < e2 ? sidx[h2] : INT_MAX, c3 = h3 < e3 ? sidx[h3] : INT_MAX;
    double sw = 0.0, se = 0.0, sr = 0.0;
    while (true) {
        int best = c0, sel = 0;
        if (c1 < best) { best = c1; sel = 1; }
        if (c2 < best) { best = c2; sel = 2; }
        if (c3 < best) { best = c3; sel = 3; }
        if (best == INT_MAX) break;
        int k = sel == 0 ? h0 : sel == 1 ? h1 : sel == 2 ? h2 : h3;
        const double4 r = rec[k];
        double fx = (sel == 0 || sel == 2) ? r.x : __dsub_rn(1.0, r.x);
        double fy = (sel <= 1) ? r.y : __dsub_rn(1.0, r.y);
        double wgt = __dmul_rn(fx, fy);
        sw = __dadd_rn(sw, wgt);
        se = __dadd_rn(se, __dmul_rn(wgt, r.z));
        if (BASIC) sr = __dadd_rn(sr, __dmul_rn(wgt, r.w));
        ++k;
        if (sel == 0) { h0 = k; c0 = k < e0 ? sidx[k] : INT_MAX; }
        else if (sel == 1) { h1 = k; c1 = k < e1 ? sidx[k] : INT_MAX; }
        else if (sel == 2) { h2 = k; c2 = k < e2 ? sidx[k] : INT_MAX; }
        else { h3 = k; c3 = k < e3 ? sidx[k] : INT_MAX; }
    }
    bool empty = live && sw == 0.0;
    unsigned ball = __ballot_sync(~0u, empty);
    if (lane == 0 && ball) atomicAdd(n_empty, (unsigned long long)__popc(ball));
    if (!live) return;
    const size_t q = (size_t)i * NW + j;
    if (out_eta) out_eta[q] = empty ? 0.0 : __ddiv_rn(se, sw);
    if (BASIC && out_rho) out_rho[q] = empty ? 0.0 : __ddiv_rn(sr, sw);
}

// ---- grid -> marker (R29): velocity nodes with wall zeros and BC mirrors from user layouts
__device__ __forceinline__ double vx_node(const MkGrid &G, const double *__restrict__ vx, int i, int j) {
    if (j <= 0 || j >= G.nx) return 0.0;
    if (i < 0) return G.sN * vx[(size_t)j];
    if (i >= G.ny) return G.sS * vx[(size_t)(G.ny - 1) * (G.nx + 1) + j];
    return vx[(size_t)i * (G.nx + 1) + j];
}
__device__ __forceinline__ double vy_node(const MkGrid &G, const double *__restrict__ vy, int i, int j) {
    if (i <= 0 || i >= G.ny) return 0.0;
    if (j < 0) return G.sW * vy[(size_t)i * G.nx];
    if (j >= G.nx) return G.sE * vy[(size_t)i * G.nx + (G.nx - 1)];
    return vy[(size_t)i * G.nx + j];
}
__device__ __forceinline__ double interp4(double tx, double ty, double v00, double v01, double v10, double v11) {
    double ux = __dsub_rn(1.0, tx), uy = __dsub_rn(1.0, ty);
    double s = __dmul_rn(__dmul_rn(ux, uy), v00);
    s = __dadd_rn(s, __dmul_rn(__dmul_rn(tx, uy), v01));
    s = __dadd_rn(s, __dmul_rn(__dmul_rn(ux, ty), v10));
    return __dadd_rn(s, __dmul_rn(__dmul_rn(tx, ty), v11));
}
__device__ __forceinline__ void velocity_at(const MkGrid &G, const double *__restrict__ vx,
                                            const double *__restrict__ vy, double x, double y, double &u,
                                            double &v) {
    x = clampd(x, 0.0, G.Lx);
    y = clampd(y, 0.0, G.Ly);
    double tx, ty;
    int jr = ref_node(x, G.dx, G.rdx, 0.0, 0, G.nx - 1, tx);
    int ir = ref_node(y, G.dy, G.rdy, G.hy, -1, G.ny - 1, ty);
    u = interp4(tx, ty, vx_node(G, vx, ir, jr), vx_node(G, vx, ir, jr + 1), vx_node(G, vx, ir + 1, jr),
                vx_node(G, vx, ir + 1, jr + 1));
    jr = ref_node(x, G.dx, G.rdx, G.hx, -1, G.nx - 1, tx);
    ir = ref_node(y, G.dy, G.rdy, 0.0, 0, G.ny - 1, ty);
    v = interp4(tx, ty, vy_node(G, vy, ir, jr), vy_node(G, vy, ir, jr + 1), vy_node(G, vy, ir + 1, jr),
                vy_node(G, vy, ir + 1, jr + 1));
}

// LPI (R32): value, gradient and mixed second derivative of the same bilinear interpolant
__device__ __forceinline__ void jet4(double tx, double ty, const MkGrid &G, double v00, double v01, double v10,
                                     double v11, double &val, double &gx, double &gy, double &gxy) {
    val = interp4(tx, ty, v00, v01, v10, v11);
    gx = __ddiv_rn(__dadd_rn(__dmul_rn(__dsub_rn(1.0, ty), __dsub_rn(v01, v00)), __dmul_rn(ty, __dsub_rn(v11, v10))),
                   G.dx);
    gy = __ddiv_rn(__dadd_rn(__dmul_rn(__dsub_rn(1.0, tx), __dsub_rn(v10, v00)), __dmul_rn(tx, __dsub_rn(v11, v01))),
                   G.dy);
    gxy = __ddiv_rn(__dadd_rn(__dsub_rn(__dsub_rn(v11, v10), v01), v00), __dmul_rn(G.dx, G.dy));
}
__device__ __forceinline__ void velocity_jet(const MkGrid &G, const double *__restrict__ vx,
                                             const double *__restrict__ vy, double x, double y, double &u,
                                             double &v, double J[4], double &Hu, double &Hv) {
    x = clampd(x, 0.0, G.Lx);
    y = clampd(y, 0.0, G.Ly);
    double tx, ty;
    int jr = ref_node(x, G.dx, G.rdx, 0.0, 0, G.nx - 1, tx);
    int ir = ref_node(y, G.dy, G.rdy, G.hy, -1, G.ny - 1, ty);
    jet4(tx, ty, G, vx_node(G, vx, ir, jr), vx_node(G, vx, ir, jr + 1), vx_node(G, vx, ir + 1, jr),
         vx_node(G, vx, ir + 1, jr + 1), u, J[0], J[1], Hu);
    jr = ref_node(x, G.dx, G.rdx, G.hx, -1, G.nx - 1, tx);
    ir = ref_node(y, G.dy, G.rdy, 0.0, 0, G.ny - 1, ty);
    jet4(tx, ty, G, vy_node(G, vy, ir, jr), vy_node(G, vy, ir, jr + 1), vy_node(G, vy, ir + 1, jr),
         vy_node(G, vy, ir + 1, jr + 1), v, J[2], J[3], Hv);
}

__global__ void k_mk_g2m(long long n, const double *__restrict__ x, const double *__restrict__ y, MkGrid G,
                         const double *__restrict__ vx, const double *__restrict__ vy, double *__restrict__ um,
                         double *__restrict__ vm) {
    long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= n) return;
    double u, v;
    velocity_at(G, vx, vy, x[m], y[m], u, v);
    um[m] = u;
    vm[m] = v;
}

// ---- advection (R30): x + dt * combination of stage velocities, stages and result clamped
template <int SCHEME>
__global__ void k_mk_advect(long long n, double *__restrict__ x, double *__restrict__ y, MkGrid G,
                            const double *__restrict__ vx, const double *__restrict__ vy, double dt,
                            unsigned long long *__restrict__ n_clamped) {
    long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool out = false;
    if (m < n) {
        double xA = x[m], yA = y[m], xn, yn, u1, v1;
        if (SCHEME >= 3) {  // Eq. lpi_update, order 2 (3) or 3 (4): x + dt v0 + dt^2/2 J v0 (+ dt^3/6 H:v0v0)
            double J[4], Hu, Hv;
            velocity_jet(G, vx, vy, xA, yA, u1, v1, J, Hu, Hv);
            const double c2 = __dmul_rn(__dmul_rn(0.5, dt), dt);
            const double jx = __dadd_rn(__dmul_rn(J[0], u1), __dmul_rn(J[1], v1));
            const double jy = __dadd_rn(__dmul_rn(J[2], u1), __dmul_rn(J[3], v1));
            xn = __dadd_rn(__dadd_rn(xA, __dmul_rn(dt, u1)), __dmul_rn(c2, jx));
            yn = __dadd_rn(__dadd_rn(yA, __dmul_rn(dt, v1)), __dmul_rn(c2, jy));
            if (SCHEME == 4) {  // (H : v0 v0)_i = 2 d2v_i/dxdy v0x v0y
                const double c3 = __dmul_rn(__dmul_rn(__dmul_rn(1.0 / 6.0, dt), dt), dt);
                xn = __dadd_rn(xn, __dmul_rn(c3, __dmul_rn(__dmul_rn(__dmul_rn(2.0, Hu), u1), v1)));
                yn = __dadd_rn(yn, __dmul_rn(c3, __dmul_rn(__dmul_rn(__dmul_rn(2.0, Hv), u1), v1)));
            }
        } else {
        velocity_at(G, vx, vy, xA, yA, u1, v1);
        if (SCHEME == 0) {  // Eq. euler_advection
            xn = __dadd_rn(xA, __dmul_rn(dt, u1));
            yn = __dadd_rn(yA, __dmul_rn(dt, v1));
        } else if (SCHEME == 1) {  // Eq. heun_method
            double u2, v2;
            double xs = clampd(__dadd_rn(xA, __dmul_rn(dt, u1)), 0.0, G.Lx);
            double ys = clampd(__dadd_rn(yA, __dmul_rn(dt, v1)), 0.0, G.Ly);
            velocity_at(G, vx, vy, xs, ys, u2, v2);
            double hdt = __dmul_rn(0.5, dt);
            xn = __dadd_rn(xA, __dmul_rn(hdt, __dadd_rn(u1, u2)));
            yn = __dadd_rn(yA, __dmul_rn(hdt, __dadd_rn(v1, v2)));
        } else {  // Eq. rk4_method, combination order of Listing rk4_agnostic
            double hdt = __dmul_rn(0.5, dt), u2, v2, u3, v3, u4, v4;
            velocity_at(G, vx, vy, clampd(__dadd_rn(xA, __dmul_rn(hdt, u1)), 0.0, G.Lx),
                        clampd(__dadd_rn(yA, __dmul_rn(hdt, v1)), 0.0, G.Ly), u2, v2);
            velocity_at(G, vx, vy, clampd(__dadd_rn(xA, __dmul_rn(hdt, u2)), 0.0, G.Lx),
                        clampd(__dadd_rn(yA, __dmul_rn(hdt, v2)), 0.0, G.Ly), u3, v3);
            velocity_at(G, vx, vy, clampd(__dadd_rn(xA, __dmul_rn(dt, u3)), 0.0, G.Lx),
                        clampd(__dadd_rn(yA, __dmul_rn(dt, v3)), 0.0, G.Ly), u4, v4);
            const double sixth = 1.0 / 6.0;
            double ue = __dmul_rn(sixth, __dadd_rn(__dadd_rn(__dadd_rn(u1, __dmul_rn(2.0, u2)), __dmul_rn(2.0, u3)), u4));
            double ve = __dmul_rn(sixth, __dadd_rn(__dadd_rn(__dadd_rn(v1, __dmul_rn(2.0, v2)), __dmul_rn(2.0, v3)), v4));
            xn = __dadd_rn(xA, __dmul_rn(dt, ue));
            yn = __dadd_rn(yA, __dmul_rn(dt, ve));
        }
        }
        out = xn < 0.0 || xn > G.Lx || yn < 0.0 || yn > G.Ly;
        x[m] = clampd(xn, 0.0, G.Lx);
        y[m] = clampd(yn, 0.0, G.Ly);
    }
    unsigned ball = __ballot_sync(~0u, out);
    if ((threadIdx.x & 31) == 0 && ball) atomicAdd(n_clamped, (unsigned long long)__popc(ball));
}

// ---- max |v| over the velocity unknowns (R31); non-negative doubles order like their bits
__global__ void k_mk_vmax(MkGrid G, const double *__restrict__ vx, const double *__restrict__ vy,
                          unsigned long long *__restrict__ mx2) {
    long long nvx = (long long)G.ny * (G.nx + 1), nvy = (long long)(G.ny + 1) * G.nx;
    double ax = 0.0, ay = 0.0;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < nvx + nvy;
         q += (long long)gridDim.x * blockDim.x) {
        if (q < nvx) {
            int j = (int)(q % (G.nx + 1));
            if (j > 0 && j < G.nx) ax = fmax(ax, fabs(vx[q]));
        } else {
            long long r = q - nvx;
            int i = (int)(r / G.nx);
            if (i > 0 && i < G.ny) ay = fmax(ay, fabs(vy[r]));
        }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        ax = fmax(ax, __shfl_xor_sync(~0u, ax, d));
        ay = fmax(ay, __shfl_xor_sync(~0u, ay, d));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(mx2, (unsigned long long)__double_as_longlong(ax));
        atomicMax(mx2 + 1, (unsigned long long)__double_as_longlong(ay));
    }
}

MkGrid mk_grid(const stokes_s *h) {
    MkGrid G;
    G.nx = h->nx;
    G.ny = h->ny;
    G.Lx = h->Lx;
    G.Ly = h->Ly;
    G.dx = h->Lx / h->nx;
    G.dy = h->Ly / h->ny;
    G.hx = 0.5 * G.dx;
    G.hy = 0.5 * G.dy;
    G.rdx = 1.0 / G.dx;
    G.rdy = 1.0 / G.dy;
    G.sW = h->bc[0] ? -1.0 : 1.0;
    G.sE = h->bc[1] ? -1.0 : 1.0;
    G.sN = h->bc[2] ? -1.0 : 1.0;
    G.sS = h->bc[3] ? -1.0 : 1.0;
    return G;
}

unsigned blocks_for(long long n, int tpb) { return (unsigned)((n + tpb - 1) / tpb); }

// marker scratch, grown on demand (cudaMalloc; freed by stokes_destroy)
int mk_reserve(stokes_s *h, size_t bytes) {
    if (h->mk_bytes >= bytes) return STOKES_OK;
    if (h->mk_ws) {
        cudaError_t e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) return sk::fail_cuda(e, "marker scratch");
        cudaFree(h->mk_ws);
        h->mk_ws = nullptr;
        h->mk_bytes = 0;
    }
    cudaError_t e = cudaMalloc(&h->mk_ws, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        h->mk_ws = nullptr;
        sk::g_last_error = "marker scratch: cudaMalloc failed";
        return STOKES_ENOMEM;
    }
    h->mk_bytes = bytes;
    return STOKES_OK;
}

struct MkCarve {
    char *base;
    size_t off;
    template <class T>
    T *take(size_t count) {
        off = (off + 255) & ~(size_t)255;
        T *p = base ? (T *)(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
};

int check_single(const stokes_s *h) { return (!h || h->dist) ? STOKES_EINVAL : STOKES_OK; }

// one counting sort of the markers into the bins of one target grid
void sort_bins(stokes_s *h, const LaunchCtx &c, int nb, int *cnt, int *off, int *fill, int *tsum) {
    int nt = (nb + SCAN_TILE - 1) / SCAN_TILE;
    k_scan_reduce<<<nt, SCAN_T, 0, c.stream>>>(cnt, nb, tsum);
    ++*c.counter;
    k_scan_top<<<1, SCAN_T, 0, c.stream>>>(tsum, nt, off, nb);
    ++*c.counter;
    k_scan_apply<<<nt, SCAN_T, 0, c.stream>>>(cnt, nb, tsum, off, fill);
    ++*c.counter;
}

}  // namespace

extern "C" {

int stokes_markers_to_grid(stokes_t h, long long n, const double *xm, const double *ym, const double *eta_m,
                           const double *rho_m, double *eta_b, double *eta_p, double *rho_b, long long *n_empty) {
    DEVICE_GUARD(h);
    if (check_single(h)) return STOKES_EINVAL;
    if (n < 0 || n >= INT_MAX) return STOKES_EINVAL;
    if (n > 0 && (!xm || !ym || !eta_m || (!rho_m && rho_b))) return STOKES_EINVAL;
    const MkGrid G = mk_grid(h);
    const int nbB = G.nx * G.ny, nbP = (G.nx + 1) * (G.ny + 1);
    const int ntB = (nbB + SCAN_TILE - 1) / SCAN_TILE, ntP = (nbP + SCAN_TILE - 1) / SCAN_TILE;
    MkCarve cv{nullptr, 0};
    for (int pass = 0; pass < 2; ++pass) {  // pass 0 sizes, pass 1 carves
        if (pass == 1) {
            int st = mk_reserve(h, cv.off + 256);
            if (st) return st;
            cv = MkCarve{(char *)h->mk_ws, 0};
        }
        cv.take<unsigned long long>(4);
        cv.take<int>(nbB + 1); cv.take<int>(nbB + 1); cv.take<int>(nbB); cv.take<int>(ntB);
        cv.take<int>(nbP + 1); cv.take<int>(nbP + 1); cv.take<int>(nbP); cv.take<int>(ntP);
        cv.take<int>(n); cv.take<int>(n);
        cv.take<double4>(n); cv.take<double4>(n);
    }
    cv = MkCarve{(char *)h->mk_ws, 0};
    auto *scal = cv.take<unsigned long long>(4);
    int *cntB = cv.take<int>(nbB + 1), *offB = cv.take<int>(nbB + 1), *fillB = cv.take<int>(nbB), *tsB = cv.take<int>(ntB);
    int *cntP = cv.take<int>(nbP + 1), *offP = cv.take<int>(nbP + 1), *fillP = cv.take<int>(nbP), *tsP = cv.take<int>(ntP);
    int *sidxB = cv.take<int>(n), *sidxP = cv.take<int>(n);
    double4 *recB = cv.take<double4>(n), *recP = cv.take<double4>(n);
    const LaunchCtx c = sk::ctx(h);
    CK(cudaMemsetAsync(scal, 0, 4 * sizeof(unsigned long long), c.stream));
    CK(cudaMemsetAsync(cntB, 0, (nbB + 1) * sizeof(int), c.stream));
    CK(cudaMemsetAsync(cntP, 0, (nbP + 1) * sizeof(int), c.stream));
    if (n > 0) {
        k_mk_count<<<blocks_for(n, TPB), TPB, 0, c.stream>>>(n, xm, ym, G, cntB, cntP);
        ++*c.counter;
    }
    sort_bins(h, c, nbB, cntB, offB, fillB, tsB);
    sort_bins(h, c, nbP, cntP, offP, fillP, tsP);
    if (n > 0) {
        k_mk_scatter<<<blocks_for(n, TPB), TPB, 0, c.stream>>>(n, xm, ym, G, fillB, fillP, sidxB, sidxP);
        ++*c.counter;
    }
    const double *rho_src = rho_m ? rho_m : eta_m;  // rho records unused when rho_b is NULL
    k_mk_records<true><<<blocks_for((long long)(nbB + 31) / 32 * 32, TPB), TPB, 0, c.stream>>>(
        nbB, offB, sidxB, xm, ym, eta_m, rho_src, G, recB);
    ++*c.counter;
    k_mk_records<false><<<blocks_for((long long)(nbP + 31) / 32 * 32, TPB), TPB, 0, c.stream>>>(
        nbP, offP, sidxP, xm, ym, eta_m, rho_src, G, recP);
    ++*c.counter;
    const dim3 gB((G.nx + 1 + GX - 1) / GX, (G.ny + 1 + GY - 1) / GY), gP((G.nx + GX - 1) / GX, (G.ny + GY - 1) / GY);
    k_mk_gather<true><<<gB, 256, 0, c.stream>>>(G, offB, sidxB, recB, eta_b, rho_b, scal);
    ++*c.counter;
    k_mk_gather<false><<<gP, 256, 0, c.stream>>>(G, offP, sidxP, recP, eta_p, nullptr, scal);
    ++*c.counter;
    CKL();
    if (n_empty) {
        CK(cudaMemcpyAsync(&h->hscal[sk::S_NSCAL - 2], scal, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           c.stream));
        int st = sk::sync(h);
        if (st) return st;
        unsigned long long v;
        memcpy(&v, &h->hscal[sk::S_NSCAL - 2], sizeof v);
        *n_empty = (long long)v;
        return STOKES_OK;
    }
    return STOKES_OK;
}

int stokes_grid_to_markers(stokes_t h, long long n, const double *xm, const double *ym, const double *vx,
                           const double *vy, double *vxm, double *vym) {
    DEVICE_GUARD(h);
    if (check_single(h)) return STOKES_EINVAL;
    if (n < 0 || (n > 0 && (!xm || !ym || !vx || !vy || !vxm || !vym))) return STOKES_EINVAL;
    if (n == 0) return STOKES_OK;
    const LaunchCtx c = sk::ctx(h);
    k_mk_g2m<<<blocks_for(n, TPB), TPB, 0, c.stream>>>(n, xm, ym, mk_grid(h), vx, vy, vxm, vym);
    ++*c.counter;
    CKL();
    return STOKES_OK;
}

int stokes_advect_markers(stokes_t h, long long n, double *xm, double *ym, const double *vx, const double *vy,
                          double dt, int scheme, long long *n_clamped) {
    DEVICE_GUARD(h);
    if (check_single(h)) return STOKES_EINVAL;
    if (n < 0 || (n > 0 && (!xm || !ym || !vx || !vy)) || scheme < 0 || scheme > 4 || !isfinite(dt))
        return STOKES_EINVAL;
    int st = mk_reserve(h, 256);
    if (st) return st;
    auto *cl = (unsigned long long *)h->mk_ws;
    const LaunchCtx c = sk::ctx(h);
    if (n_clamped) CK(cudaMemsetAsync(cl, 0, sizeof(unsigned long long), c.stream));
    if (n > 0) {
        const MkGrid G = mk_grid(h);
        unsigned nb = blocks_for(n, TPB);
        if (scheme == 0) k_mk_advect<0><<<nb, TPB, 0, c.stream>>>(n, xm, ym, G, vx, vy, dt, cl);
        else if (scheme == 1) k_mk_advect<1><<<nb, TPB, 0, c.stream>>>(n, xm, ym, G, vx, vy, dt, cl);
        else if (scheme == 2) k_mk_advect<2><<<nb, TPB, 0, c.stream>>>(n, xm, ym, G, vx, vy, dt, cl);
        else if (scheme == 3) k_mk_advect<3><<<nb, TPB, 0, c.stream>>>(n, xm, ym, G, vx, vy, dt, cl);
        else k_mk_advect<4><<<nb, TPB, 0, c.stream>>>(n, xm, ym, G, vx, vy, dt, cl);
        ++*c.counter;
        CKL();
    }
    if (n_clamped) {
        CK(cudaMemcpyAsync(&h->hscal[sk::S_NSCAL - 2], cl, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           c.stream));
        st = sk::sync(h);
        if (st) return st;
        unsigned long long v;
        memcpy(&v, &h->hscal[sk::S_NSCAL - 2], sizeof v);
        *n_clamped = (long long)v;
    }
    return STOKES_OK;
}

int stokes_marker_timestep(stokes_t h, const double *vx, const double *vy, double cfl, double max_dt, double *dt) {
    DEVICE_GUARD(h);
    if (check_single(h)) return STOKES_EINVAL;
    if (!vx || !vy || !dt || !(cfl > 0) || !(max_dt > 0)) return STOKES_EINVAL;
    int st = mk_reserve(h, 256);
    if (st) return st;
    auto *mx2 = (unsigned long long *)h->mk_ws;
    const LaunchCtx c = sk::ctx(h);
    const MkGrid G = mk_grid(h);
    CK(cudaMemsetAsync(mx2, 0, 2 * sizeof(unsigned long long), c.stream));
    k_mk_vmax<<<2 * 148, TPB, 0, c.stream>>>(G, vx, vy, mx2);
    ++*c.counter;
    CKL();
    CK(cudaMemcpyAsync(&h->hscal[sk::S_NSCAL - 4], mx2, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       c.stream));
    st = sk::sync(h);
    if (st) return st;
    double mx, my;
    memcpy(&mx, &h->hscal[sk::S_NSCAL - 4], sizeof mx);
    memcpy(&my, &h->hscal[sk::S_NSCAL - 3], sizeof my);
    double d = max_dt;  // R31: min(max_dt, cfl min(dx/max|vx|, dy/max|vy|))
    if (mx > 0.0) d = fmin(d, cfl * (G.dx / mx));
    if (my > 0.0) d = fmin(d, cfl * (G.dy / my));
    *dt = d;
    return STOKES_OK;
}

}  // extern "C"
