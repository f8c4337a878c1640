// TMA-staged row-streaming engine for the bandwidth-bound hot loops (sm_100a).
//
// A CTA of TW = 256 threads owns 256 consecutive columns j0..j0+255 of a level and a
// strip of rows [i0, i1].  One elected thread streams the rows i0-1 .. i1+1 of the NF
// input fields into an NS-deep shared-memory ring: each field row segment
// [j0-2, j0+258) (2080 B, 16-B aligned by the layout of internal.h) is ONE bulk-async
// copy (cp.async.bulk, executed by the TMA engine) completing on the slot's mbarrier.
// All 256 threads then evaluate their column on the three staged rows i-1, i, i+1 and
// store results straight to HBM.  Every input element is read from HBM once per strip
// and up to NS-3 rows per CTA are in flight without costing registers; the grid is
// sized so that one wave of CTAs covers the level (strip height from the occupancy), so
// there is no tail wave.  The operators (Op) are:
//   JacobiOp      damped Jacobi sweep, Eq. damped_jacobi       [a4]
//   ResidualOp    r = b - L v, Eq. mg_residual                   [a3/a5]
//   UzawaOp       pressure update p += alpha eta_P (-D v) (reading R3)
//                 fused with the energy residual of the new (v, p) [a10+a3]
// Stencil coefficients are those of kernels.cu (Listing vx_op_point).
#include <math.h>
#include <stdlib.h>

#include <type_traits>

#include "internal.h"

namespace {

#ifndef WS_PROXY_FENCE
#define WS_PROXY_FENCE 1
#endif
constexpr int TW = 256;          // columns per CTA
constexpr int RW = TW + 4;       // staged row width (doubles): [j0-2, j0+TW+2)
constexpr int NS = 8;            // landing ring depth (rows): NS-1 rows in flight per CTA
constexpr int NF = 6;            // staged fields
constexpr int SMEM = NS * NF * RW * 8 + 2 * NS * 8;
constexpr int MINB = 2;          // CTAs per SM (shared memory: 2 x 97.5 KB)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// Register window of the three rows i-1 (A), i (B), i+1 (C) of every field for this
// thread's column: value and its left / right neighbours.  Each staged row is read from
// its shared-memory landing slot exactly once, when it becomes row C; components an
// operator never reads are dead code and cost neither loads nor registers.
struct R3 {
    double l, c, r;
};
struct Fld {
    R3 A, B, C;
};
struct Win {
    Fld f[NF];
    __device__ __forceinline__ double A(int k, int dc = 0) const { return dc < 0 ? f[k].A.l : (dc > 0 ? f[k].A.r : f[k].A.c); }
    __device__ __forceinline__ double B(int k, int dc = 0) const { return dc < 0 ? f[k].B.l : (dc > 0 ? f[k].B.r : f[k].B.c); }
    __device__ __forceinline__ double C(int k, int dc = 0) const { return dc < 0 ? f[k].C.l : (dc > 0 ? f[k].C.r : f[k].C.c); }
    template <int NFU>
    __device__ __forceinline__ void shift() {  // advance one row with no new data (C stale)
#pragma unroll
        for (int k = 0; k < NFU; ++k) {
            f[k].A = f[k].B;
            f[k].B = f[k].C;
        }
    }
    template <int NFU, int ROW = RW>
    __device__ __forceinline__ void push(const double *slot, int t) {  // t = column offset in the segment
#pragma unroll
        for (int k = 0; k < NFU; ++k) {
            f[k].A = f[k].B;
            f[k].B = f[k].C;
            const double *s = slot + k * ROW + t;
            f[k].C.l = s[-1];
            f[k].C.c = s[0];
            f[k].C.r = s[1];
        }
    }
};
enum { F_VX = 0, F_VY = 1, F_EP = 2, F_EB = 3, F_4 = 4, F_5 = 5 };  // F_4: p | bx, F_5: rho | by

// Row / column ranges of a launch, one per blockIdx.z (two at most: the split passes of a
// decomposed tile run the boundary strips N + S or W + E in one launch).  Default: the level.
struct Reg2 {
    int i_lo[2], i_hi[2], j_lo[2], j_hi[2];
};
__device__ __forceinline__ int zsel(const int (&a)[2], int z) { return z ? a[1] : a[0]; }  // no local copy
Reg2 full_region(const GridL &g) {
    Reg2 r;
    r.i_lo[0] = r.i_lo[1] = 1;
    r.i_hi[0] = r.i_hi[1] = g.ncy;
    r.j_lo[0] = r.j_lo[1] = 1;
    r.j_hi[0] = r.j_hi[1] = g.ncx;
    return r;
}

// reciprocal without the IEEE-division subroutine: MUFU seed + two Newton steps.
// RCP_SEED 1 (default): the FP64 MUFU seed rcp.approx.ftz.f64 (~20 bits, one instruction,
// no conversions); 0: the IEEE-rounded float reciprocal of the rounded argument (~24 bits,
// F2F + MUFU + fix-up + F2F).  Either way two Newton steps reach full precision (<= 1 ulp;
// |a| is far inside the normal range on every level here).
#ifndef RCP_SEED
#define RCP_SEED 1
#endif
__device__ __forceinline__ double rcp(double a) {
#if RCP_SEED
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
#else
    double r = (double)__frcp_rn((float)a);
#endif
    r = r * fma(-a, r, 2.0);
    r = r * fma(-a, r, 2.0);
    return r;
}

// ---- stencil rows on the window (coefficients of Listing vx_op_point / reading R2)
struct RowX {
    double L, a;  // (L v) at the node and a_ii
};
// Written as coefficient x (neighbour - centre) differences (the stress form of
// PAPER.md:643-661): the same operator as the Listing's coefficients with ~20% fewer
// FP64 operations and shorter dependency chains; a_ii is formed separately.
template <bool EDGE = true, class W>  // EDGE = false: row i is no N/S boundary row
__device__ __forceinline__ RowX lx_win(const GridL &g, const W &w, int i) {
    const double eta1 = w.A(F_EB), eta2 = w.B(F_EB), etaA = w.B(F_EP), etaB = w.B(F_EP, 1);
    const double vc = w.B(F_VX);
    RowX r;
    r.L = g.idx2x2 * (etaA * (w.B(F_VX, -1) - vc) + etaB * (w.B(F_VX, 1) - vc)) +
          g.idy2 * (eta1 * (w.A(F_VX) - vc) + eta2 * (w.C(F_VX) - vc)) +
          g.idxdy * (eta1 * (w.A(F_VY) - w.A(F_VY, 1)) + eta2 * (w.B(F_VY, 1) - w.B(F_VY)));
    r.a = -(eta1 + eta2) * g.idy2 - (etaA + etaB) * g.idx2x2;
    if (EDGE && i == 1 && g.bN) r.a += g.sN * eta1 * g.idy2;
    if (EDGE && i == g.ncy && g.bS) r.a += g.sS * eta2 * g.idy2;
    return r;
}
template <bool EDGE = true, class W>  // EDGE = false: column j is no W/E boundary column
__device__ __forceinline__ RowX ly_win(const GridL &g, const W &w, int j) {
    const double etaN = w.B(F_EP), etaS = w.C(F_EP), etaW = w.B(F_EB, -1), etaE = w.B(F_EB);
    const double vc = w.B(F_VY);
    RowX r;
    r.L = g.idy2x2 * (etaS * (w.C(F_VY) - vc) + etaN * (w.A(F_VY) - vc)) +
          g.idx2 * (etaE * (w.B(F_VY, 1) - vc) + etaW * (w.B(F_VY, -1) - vc)) +
          g.idxdy * (etaE * (w.C(F_VX) - w.B(F_VX)) - etaW * (w.C(F_VX, -1) - w.B(F_VX, -1)));
    r.a = -(etaN + etaS) * g.idy2x2 - (etaW + etaE) * g.idx2;
    if (EDGE && j == 1 && g.bW) r.a += g.sW * etaW * g.idx2;
    if (EDGE && j == g.ncx && g.bE) r.a += g.sE * etaE * g.idx2;
    return r;
}
// The same rows split as L v = S + a v_c: S = the weighted sum of the neighbours only (the
// mirror ghost of a global wall left out: its coefficient is folded into a, exactly as in
// lx_win), a = the BC-folded centre coefficient.  A damped Jacobi update then reads
//   v' = v + w (b - L v) / a = (1 - w) v + (w / a) (b - S)
// -- 11 FP64 operations for S instead of 15 for L, and the update no longer needs L.
struct RowS {
    double S, a;
};
template <bool EDGE = true, class W>
__device__ __forceinline__ RowS lxs_win(const GridL &g, const W &w, int i) {
    const double eta1 = w.A(F_EB), eta2 = w.B(F_EB), etaA = w.B(F_EP), etaB = w.B(F_EP, 1);
    double vN = w.A(F_VX), vS = w.C(F_VX);
    RowS r;
    r.a = -(eta1 + eta2) * g.idy2 - (etaA + etaB) * g.idx2x2;
    if (EDGE && i == 1 && g.bN) {
        r.a += g.sN * eta1 * g.idy2;
        vN = 0.0;
    }
    if (EDGE && i == g.ncy && g.bS) {
        r.a += g.sS * eta2 * g.idy2;
        vS = 0.0;
    }
    r.S = g.idx2x2 * (etaA * w.B(F_VX, -1) + etaB * w.B(F_VX, 1)) + g.idy2 * (eta1 * vN + eta2 * vS) +
          g.idxdy * (eta1 * (w.A(F_VY) - w.A(F_VY, 1)) + eta2 * (w.B(F_VY, 1) - w.B(F_VY)));
    return r;
}
template <bool EDGE = true, class W>
__device__ __forceinline__ RowS lys_win(const GridL &g, const W &w, int j) {
    const double etaN = w.B(F_EP), etaS = w.C(F_EP), etaW = w.B(F_EB, -1), etaE = w.B(F_EB);
    double vW = w.B(F_VY, -1), vE = w.B(F_VY, 1);
    RowS r;
    r.a = -(etaN + etaS) * g.idy2x2 - (etaW + etaE) * g.idx2;
    if (EDGE && j == 1 && g.bW) {
        r.a += g.sW * etaW * g.idx2;
        vW = 0.0;
    }
    if (EDGE && j == g.ncx && g.bE) {
        r.a += g.sE * etaE * g.idx2;
        vE = 0.0;
    }
    r.S = g.idy2x2 * (etaS * w.C(F_VY) + etaN * w.A(F_VY)) + g.idx2 * (etaE * vE + etaW * vW) +
          g.idxdy * (etaE * (w.C(F_VX) - w.B(F_VX)) - etaW * (w.C(F_VX, -1) - w.B(F_VX, -1)));
    return r;
}
// body force (reading R4/R23) at vx / vy nodes from the staged rho rows
template <class W>
__device__ __forceinline__ double fx_win(const W &w, double gx) {
    return gx != 0.0 ? -gx * (0.5 * (w.A(F_5) + w.B(F_5))) : 0.0;
}
template <class W>
__device__ __forceinline__ double fy_win(const W &w, double gy) {
    return gy != 0.0 ? -gy * (0.5 * (w.B(F_5, -1) + w.B(F_5))) : 0.0;
}

template <int MODE>
struct JacobiOp {
    static constexpr bool WS = true;  // warp-specialised engine
    static constexpr int NF = 6;
    static constexpr int NRED = 0;
    const double *src[NF];
    double *vxo, *vyo;
    double omega, gx, gy;
    __device__ __forceinline__ void row(const GridL &g, const Win &w, int i, int j, double *) const {
        const size_t P = g.P;
        if (j <= g.nvxj) {
            const RowX x = lx_win(g, w, i);
            const double b = (MODE == RHS_FINE) ? fx_win(w, gx) - (w.B(F_4) - w.B(F_4, 1)) * g.idx : w.B(F_4);
            const double vn = w.B(F_VX) + omega * (b - x.L) * rcp(x.a);
            vxo[(size_t)i * P + j] = vn;
            if (i == 1 && g.bN) vxo[j] = g.sN * vn;
            if (i == g.ncy && g.bS) vxo[(size_t)(g.ncy + 1) * P + j] = g.sS * vn;
        }
        if (i <= g.nvyi) {
            const RowX y = ly_win(g, w, j);
            const double b = (MODE == RHS_FINE) ? fy_win(w, gy) - (w.B(F_4) - w.C(F_4)) * g.idy : w.B(F_5);
            const double vn = w.B(F_VY) + omega * (b - y.L) * rcp(y.a);
            vyo[(size_t)i * P + j] = vn;
            if (j == 1 && g.bW) vyo[(size_t)i * P] = g.sW * vn;
            if (j == g.ncx && g.bE) vyo[(size_t)i * P + g.ncx + 1] = g.sE * vn;
        }
    }
};

template <int MODE>
struct ResidualOp {
    static constexpr bool WS = true;  // warp-specialised engine
    static constexpr int NF = 6;
    static constexpr int NRED = 0;
    const double *src[NF];
    double *rx, *ry;
    double gx, gy;
    __device__ __forceinline__ void row(const GridL &g, const Win &w, int i, int j, double *) const {
        const size_t P = g.P;
        if (j <= g.nvxj) {
            const double b = (MODE == RHS_FINE) ? fx_win(w, gx) - (w.B(F_4) - w.B(F_4, 1)) * g.idx : w.B(F_4);
            rx[(size_t)i * P + j] = b - lx_win(g, w, i).L;
        }
        if (i <= g.nvyi) {
            const double b = (MODE == RHS_FINE) ? fy_win(w, gy) - (w.B(F_4) - w.C(F_4)) * g.idy : w.B(F_5);
            ry[(size_t)i * P + j] = b - ly_win(g, w, j).L;
        }
    }
};

// Uzawa pressure step fused with the energy residual of the new iterate:
//   p' = (p - mshift) + alpha_s eta_P (-D v)     (reading R3; de-mean R10)
//   r_v = f - L v - G p',  r_p = -D v,  Sv += r_v^2/(-a_ii), Sp += r_p^2 eta_P/(2/dx^2+2/dy^2)
// p' at the east / south neighbours is recomputed from v on the window, so one pass reads
// (vx, vy, eta_p, eta_b, p, rho) and writes p'.  Partial sums per CTA: (Sv, Sp, sum p').
struct UzawaOp {
    static constexpr bool WS = false;  // warp-specialised engine
    static constexpr int NF = 6;
    static constexpr int NRED = 3;
    const double *src[NF];
    double *po;             // p' output: a DIFFERENT buffer from src[F_4] (neighbouring CTAs stage
                            // rows / halo columns of p that this CTA would otherwise overwrite)
    const double *mshift;
    double alpha_s, gx, gy;
    double *rxo, *ryo, *rpo;  // optional residual outputs
    int write_p;
    __device__ __forceinline__ double divB(const GridL &g, const Win &w, int dc) const {  // (D v)(i, j+dc)
        return (w.B(F_VX, dc) - w.B(F_VX, dc - 1)) * g.idx + (w.B(F_VY, dc) - w.A(F_VY, dc)) * g.idy;
    }
    __device__ __forceinline__ double divC(const GridL &g, const Win &w) const {  // (D v)(i+1, j)
        return (w.C(F_VX) - w.C(F_VX, -1)) * g.idx + (w.C(F_VY) - w.B(F_VY)) * g.idy;
    }
    __device__ __forceinline__ void row(const GridL &g, const Win &w, int i, int j, double *acc) const {
        const double ms = *mshift;
        const double dv = divB(g, w, 0);
        const double pn = (w.B(F_4) - ms) + alpha_s * w.B(F_EP) * (-dv);
        if (write_p) po[(size_t)i * g.P + j] = pn;
        const double rp = -dv;
        acc[1] += rp * rp * (w.B(F_EP) / (2.0 * g.idx2 + 2.0 * g.idy2));
        acc[2] += pn;
        if (rpo) rpo[(size_t)i * g.P + j] = rp;
        if (j <= g.nvxj) {
            const double pe = (w.B(F_4, 1) - ms) + alpha_s * w.B(F_EP, 1) * (-divB(g, w, 1));
            const RowX x = lx_win(g, w, i);
            const double r = fx_win(w, gx) - (pn - pe) * g.idx - x.L;
            acc[0] -= r * r * rcp(x.a);
            if (rxo) rxo[(size_t)i * g.P + j] = r;
        }
        if (i <= g.nvyi) {
            const double ps = (w.C(F_4) - ms) + alpha_s * w.C(F_EP) * (-divC(g, w));
            const RowX y = ly_win(g, w, j);
            const double r = fy_win(w, gy) - (pn - ps) * g.idy - y.L;
            acc[0] -= r * r * rcp(y.a);
            if (ryo) ryo[(size_t)i * g.P + j] = r;
        }
    }
};

// GCR preconditioner pressure part fused with the operator apply (a11):
//   z_p = alpha eta_P (r_p - D z_v)            (M^-1 of the Uzawa splitting, R3)
//   w = A z = [L z_v + G z_p ; D z_v]
// z_p at the east / south neighbours is recomputed on the window.  Partial dots for the
// first Gram-Schmidt coefficient: <w, w0> (first == 0) or <w, w>, <r, w> (first step).
struct PrecondApplyOp {
    static constexpr bool WS = false;  // warp-specialised engine
    static constexpr int NF = 5;
    static constexpr int NRED = 2;
    const double *src[6];        // zx, zy, eta_p, eta_b, r_p
    double *zp, *wx, *wy, *wp;
    const double *w0x, *w0y, *w0p;  // previous basis vector (null on the first step)
    const double *rx, *ry;           // residual velocity parts (first step: <r, w>)
    double alpha;
    __device__ __forceinline__ double divB(const GridL &g, const Win &w, int dc) const {
        return (w.B(F_VX, dc) - w.B(F_VX, dc - 1)) * g.idx + (w.B(F_VY, dc) - w.A(F_VY, dc)) * g.idy;
    }
    __device__ __forceinline__ void row(const GridL &g, const Win &w, int i, int j, double *acc) const {
        const size_t q = (size_t)i * g.P + j;
        const double dz = divB(g, w, 0);
        const double zc = alpha * w.B(F_EP) * (w.B(F_4) - dz);
        zp[q] = zc;
        wp[q] = dz;
        if (w0x) acc[0] += dz * w0p[q];
        else { acc[0] += dz * dz; acc[1] += w.B(F_4) * dz; }
        if (j <= g.nvxj) {
            const double ze = alpha * w.B(F_EP, 1) * (w.B(F_4, 1) - divB(g, w, 1));
            const double v = lx_win(g, w, i).L + (zc - ze) * g.idx;
            wx[q] = v;
            if (w0x) acc[0] += v * w0x[q];
            else { acc[0] += v * v; acc[1] += rx[q] * v; }
        }
        if (i <= g.nvyi) {
            const double ds = (w.C(F_VX) - w.C(F_VX, -1)) * g.idx + (w.C(F_VY) - w.B(F_VY)) * g.idy;
            const double zs = alpha * w.C(F_EP) * (w.C(F_4) - ds);
            const double v = ly_win(g, w, j).L + (zc - zs) * g.idy;
            wy[q] = v;
            if (w0x) acc[0] += v * w0y[q];
            else { acc[0] += v * v; acc[1] += ry[q] * v; }
        }
    }
};

// The last Uzawa step fused into the first pre-smoothing sweep of the next V-cycle
// (SURVEY §8(a) a12): from v^k and p^(k-1) one pass computes
//   p^k = (p^(k-1) - mshift) + alpha_s eta_P (-D v^k)                 (a10, reading R3)
//   r_v = f - L v^k - G p^k,  r_p = -D v^k -> partial sums of E(v^k, p^k) (a3)
//   v' = v^k + omega r_v / a_ii                                          (a4, first sweep)
// (p^k at the east / south neighbours recomputed on the window).  If E(v^k, p^k) <= rtol
// the sweep's output is discarded and (v^k, p^k) returned: the iterates are unchanged.
struct JacobiUzawaOp {
    static constexpr bool WS = false;
    static constexpr int NF = 6;
    static constexpr int NRED = 3;
    const double *src[6];  // vx, vy, eta_p, eta_b, p^(k-1), rho
    double *vxo, *vyo, *po;
    const double *mshift;
    double alpha_s, omega, gx, gy;
    __device__ __forceinline__ double divB(const GridL &g, const Win &w, int dc) const {
        return (w.B(F_VX, dc) - w.B(F_VX, dc - 1)) * g.idx + (w.B(F_VY, dc) - w.A(F_VY, dc)) * g.idy;
    }
    __device__ __forceinline__ void row(const GridL &g, const Win &w, int i, int j, double *acc) const {
        const size_t P = g.P;
        const double ms = *mshift;
        const double dv = divB(g, w, 0);
        const double pn = (w.B(F_4) - ms) + alpha_s * w.B(F_EP) * (-dv);
        po[(size_t)i * P + j] = pn;
        acc[1] += dv * dv * (w.B(F_EP) / (2.0 * g.idx2 + 2.0 * g.idy2));
        acc[2] += pn;
        if (j <= g.nvxj) {
            const double pe = (w.B(F_4, 1) - ms) + alpha_s * w.B(F_EP, 1) * (-divB(g, w, 1));
            const RowX x = lx_win(g, w, i);
            const double r = fx_win(w, gx) - (pn - pe) * g.idx - x.L;
            const double ia = rcp(x.a);
            acc[0] -= r * r * ia;
            const double vn = w.B(F_VX) + omega * r * ia;
            vxo[(size_t)i * P + j] = vn;
            if (i == 1 && g.bN) vxo[j] = g.sN * vn;
            if (i == g.ncy && g.bS) vxo[(size_t)(g.ncy + 1) * P + j] = g.sS * vn;
        }
        if (i <= g.nvyi) {
            const double ds = (w.C(F_VX) - w.C(F_VX, -1)) * g.idx + (w.C(F_VY) - w.B(F_VY)) * g.idy;
            const double ps = (w.C(F_4) - ms) + alpha_s * w.C(F_EP) * (-ds);
            const RowX y = ly_win(g, w, j);
            const double r = fy_win(w, gy) - (pn - ps) * g.idy - y.L;
            const double ia = rcp(y.a);
            acc[0] -= r * r * ia;
            const double vn = w.B(F_VY) + omega * r * ia;
            vyo[(size_t)i * P + j] = vn;
            if (j == 1 && g.bW) vyo[(size_t)i * P] = g.sW * vn;
            if (j == g.ncx && g.bE) vyo[(size_t)i * P + g.ncx + 1] = g.sE * vn;
        }
    }
};

// Warp-specialised engine: warps 0..7 compute (one column per thread), warp 8 is the TMA
// producer.  Slot s has a FULL mbarrier (producer arrive.expect_tx + TMA complete_tx) and
// an EMPTY mbarrier (one arrive per compute warp once it has pulled the row into its
// registers), so no CTA-wide barrier is needed per row and the compute warps may drift.
constexpr int NTHR = TW + 32;
template <class Op>
__global__ void __maxnreg__(112) k_stream(GridL g, Op op, int H, double *__restrict__ partials, Reg2 R, int seg) {
    extern __shared__ __align__(128) double sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + NS * NF * RW);
    uint64_t *empty = full + NS;
    __shared__ double red[NTHR / 32];
    const int t = threadIdx.x;
    const int warp = t >> 5;
    const int z = blockIdx.z;
    const int j0 = zsel(R.j_lo, z) + TW * blockIdx.x;
    const int i0 = zsel(R.i_lo, z) + blockIdx.y * H;
    const int i1 = min(i0 + H - 1, zsel(R.i_hi, z));
    const int jhi = zsel(R.j_hi, z);
    const int rbase = i0 - 1;  // first staged row
    const int rlast = i1 + 1;  // last staged row
    if (t == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, TW / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    double acc[Op::NRED > 0 ? Op::NRED : 1];
#pragma unroll
    for (int k = 0; k < (Op::NRED > 0 ? Op::NRED : 1); ++k) acc[k] = 0.0;
    if (warp == TW / 32) {  // ---------------- producer warp
        if ((t & 31) == 0) {
            const size_t P = g.P;
            for (int r = rbase; r <= rlast; ++r) {
                const int rel = r - rbase, slot = rel % NS;
                if (rel >= NS) mbar_wait(empty + slot, ((rel / NS) - 1) & 1);  // consumers done with r-NS
                mbar_expect_tx(full + slot, Op::NF * seg * 8);
#pragma unroll
                for (int f = 0; f < Op::NF; ++f)
                    bulk_g2s(sm + (slot * NF + f) * RW, op.src[f] + (size_t)r * P + (j0 - 2), seg * 8, full + slot);
            }
        }
    } else {  // ---------------------------- compute warps
        const int j = j0 + t;
        auto consume = [&](Win &w, int r) {  // wait for row r, pull it into the window, free the slot
            const int rel = r - rbase, slot = rel % NS;
            mbar_wait(full + slot, (rel / NS) & 1);
            w.template push<Op::NF>(sm + slot * NF * RW, t + 2);
#if WS_PROXY_FENCE
            // the slot's generic-proxy reads must be ordered before the producer's next
            // async-proxy (TMA) write into it.  Without this fence a slot was occasionally
            // refilled under a slow reader: whole rows of a CTA strip came out wrong when the
            // halo exchange ran concurrently on another stream (tools/overlap_where.py)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
            __syncwarp();
            if ((t & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + slot)) : "memory");
        };
        Win w;
        consume(w, rbase);
        consume(w, rbase + 1);
        for (int i = i0; i <= i1; ++i) {
            consume(w, i + 1);  // window: A = i-1, B = i, C = i+1
            if (j <= jhi) op.row(g, w, i, j, acc);
        }
    }
    if (Op::NRED > 0) {  // deterministic CTA reduction over the compute warps
        const size_t b = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#pragma unroll
        for (int k = 0; k < Op::NRED; ++k) {
            double v = warp < TW / 32 ? acc[k] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            __syncthreads();
            if ((t & 31) == 0) red[warp] = v;
            __syncthreads();
            if (t < 32) {
                v = (t < TW / 32) ? red[t] : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (t == 0) partials[b * Op::NRED + k] = v;
            }
        }
    }
}

// CTA-barrier engine (register-heavy operators: 256 threads, up to 128 registers, 2 CTAs/SM):
// thread 0 issues the bulk copies; one __syncthreads per row frees the row's slot.
template <class Op>
__global__ void __launch_bounds__(TW, MINB) k_stream_bar(GridL g, Op op, int H, double *__restrict__ partials, Reg2 R,
                                                          int seg) {
    extern __shared__ __align__(128) double sm[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + NS * NF * RW);
    __shared__ double red[TW / 32];
    const int t = threadIdx.x;
    const int z = blockIdx.z;
    const int j0 = zsel(R.j_lo, z) + TW * blockIdx.x;
    const int j = j0 + t;
    const int i0 = zsel(R.i_lo, z) + blockIdx.y * H;
    const int i1 = min(i0 + H - 1, zsel(R.i_hi, z));
    const int jhi = zsel(R.j_hi, z);
    const int rbase = i0 - 1;
    const int rlast = i1 + 1;
    const size_t P = g.P;
    auto issue = [&](int r) {
        const int slot = (r - rbase) % NS;
        uint64_t *bar = bars + slot;
        mbar_expect_tx(bar, Op::NF * seg * 8);
#pragma unroll
        for (int f = 0; f < Op::NF; ++f)
            bulk_g2s(sm + (slot * NF + f) * RW, op.src[f] + (size_t)r * P + (j0 - 2), seg * 8, bar);
    };
    if (t == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(bars + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0)
        for (int r = rbase; r < rbase + NS && r <= rlast; ++r) issue(r);
    auto consume = [&](Win &w, int r) {
        const int rel = r - rbase;
        mbar_wait(bars + rel % NS, (rel / NS) & 1);
        w.template push<Op::NF>(sm + (rel % NS) * NF * RW, t + 2);
    };
    auto refill = [&](int r) {
        if (t == 0 && r + NS <= rlast) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(r + NS);
        }
    };
    double acc[Op::NRED > 0 ? Op::NRED : 1];
#pragma unroll
    for (int k = 0; k < (Op::NRED > 0 ? Op::NRED : 1); ++k) acc[k] = 0.0;
    Win w;
    consume(w, rbase);
    consume(w, rbase + 1);
    __syncthreads();
    refill(rbase);
    refill(rbase + 1);
    for (int i = i0; i <= i1; ++i) {
        consume(w, i + 1);
        if (j <= jhi) op.row(g, w, i, j, acc);
        __syncthreads();
        refill(i + 1);
    }
    if (Op::NRED > 0) {
        const size_t b = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#pragma unroll
        for (int k = 0; k < Op::NRED; ++k) {
            double v = acc[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            __syncthreads();
            if ((t & 31) == 0) red[t >> 5] = v;
            __syncthreads();
            if (t < 32) {
                v = (t < TW / 32) ? red[t] : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (t == 0) partials[b * Op::NRED + k] = v;
            }
        }
    }
}

int g_slots = 0;  // resident CTAs of k_stream on the device (SMs x MINB)
template <class Op>
void prepare_kernel() {
    static unsigned long long done = 0;
    if (first_on_device(&done)) {
        cudaFuncSetAttribute(k_stream<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        cudaFuncSetAttribute(k_stream_bar<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    }
}
int slots() {
    if (!g_slots) {
        int dev = 0, nsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        g_slots = (nsm > 0 ? nsm : 148) * MINB;
    }
    return g_slots;
}
// strip height: one wave of CTAs covers the level
int strip_h(const GridL &g) {
    const int ncb = (g.ncx + TW - 1) / TW;
    int strips = slots() / ncb;
    if (strips < 1) strips = 1;
    int H = (g.ncy + strips - 1) / strips;
    return H < 4 ? 4 : H;
}
dim3 stream_grid(const GridL &g) {
    const int H = strip_h(g);
    return dim3((g.ncx + TW - 1) / TW, (g.ncy + H - 1) / H);
}
template <class Op>
void run(const LaunchCtx &c, const GridL &g, const Op &op, double *partials) {
    prepare_kernel<Op>();
    if (Op::WS) k_stream<Op><<<stream_grid(g), NTHR, SMEM, c.stream>>>(g, op, strip_h(g), partials, full_region(g), RW);
    else k_stream_bar<Op><<<stream_grid(g), TW, SMEM, c.stream>>>(g, op, strip_h(g), partials, full_region(g), RW);
    ++*c.counter;
}
// The split pass of a decomposed tile (halo overlap): part 0 = the HW = 2
// layers of unknowns next to every non-global side (what the neighbours' halos need), part 1
// = the rest.  Part 0 runs first; the halo exchange of its output overlaps part 1, which
// leaves `reserve` SMs free for the exchange kernels.
struct Split {
    Reg2 ns, we, in;
    int nns, nwe, we_rows;
};
Split split_regions(const GridL &g) {
    Split s;
    const int lo_i = g.bN ? 1 : 3, hi_i = g.bS ? g.ncy : g.ncy - 2, lo_j = g.bW ? 1 : 3, hi_j = g.bE ? g.ncx : g.ncx - 2;
    s.nns = s.nwe = 0;
    if (!g.bN) { s.ns.i_lo[s.nns] = 1; s.ns.i_hi[s.nns] = 2; s.ns.j_lo[s.nns] = 1; s.ns.j_hi[s.nns] = g.ncx; ++s.nns; }
    if (!g.bS) { s.ns.i_lo[s.nns] = g.ncy - 1; s.ns.i_hi[s.nns] = g.ncy; s.ns.j_lo[s.nns] = 1; s.ns.j_hi[s.nns] = g.ncx; ++s.nns; }
    if (!g.bW) { s.we.i_lo[s.nwe] = lo_i; s.we.i_hi[s.nwe] = hi_i; s.we.j_lo[s.nwe] = 1; s.we.j_hi[s.nwe] = 2; ++s.nwe; }
    if (!g.bE) { s.we.i_lo[s.nwe] = lo_i; s.we.i_hi[s.nwe] = hi_i; s.we.j_lo[s.nwe] = g.ncx - 1; s.we.j_hi[s.nwe] = g.ncx; ++s.nwe; }
    s.we_rows = hi_i - lo_i + 1;
    s.in.i_lo[0] = s.in.i_lo[1] = lo_i;
    s.in.i_hi[0] = s.in.i_hi[1] = hi_i;
    s.in.j_lo[0] = s.in.j_lo[1] = lo_j;
    s.in.j_hi[0] = s.in.j_hi[1] = hi_j;
    return s;
}
int reserve_sms() {  // SMs left to the halo exchange while the interior part runs
    static const int v = [] {
        const char *e = getenv("STOKES_COMM_SMS");
        return e ? atoi(e) : 4;
    }();
    return v;
}
template <class Op>
void run_part(const LaunchCtx &c, const GridL &g, const Op &op, int part) {
    static_assert(Op::NRED == 0, "split passes carry no reductions");
    prepare_kernel<Op>();
    const Split sp = split_regions(g);
    auto go = [&](dim3 grid, int H, const Reg2 &R, int seg) {
        if (Op::WS) k_stream<Op><<<grid, NTHR, SMEM, c.stream>>>(g, op, H, nullptr, R, seg);
        else k_stream_bar<Op><<<grid, TW, SMEM, c.stream>>>(g, op, H, nullptr, R, seg);
        ++*c.counter;
    };
    if (part == 0) {
        if (sp.nns) go(dim3((g.ncx + TW - 1) / TW, 1, sp.nns), 2, sp.ns, RW);
        if (sp.nwe) {
            int H = (sp.we_rows + slots() - 1) / slots();
            if (H < 4) H = 4;
            go(dim3(1, (sp.we_rows + H - 1) / H, sp.nwe), H, sp.we, 6);  // 2 columns: 6-double segments
        }
        return;
    }
    const int rows = sp.in.i_hi[0] - sp.in.i_lo[0] + 1, cols = sp.in.j_hi[0] - sp.in.j_lo[0] + 1;
    const int ncb = (cols + TW - 1) / TW;
    int sl = slots() - MINB * reserve_sms();
    int strips = sl / ncb;
    if (strips < 1) strips = 1;
    int H = (rows + strips - 1) / strips;
    if (H < 4) H = 4;
    go(dim3(ncb, (rows + H - 1) / H, 1), H, sp.in, RW);
}
void fill_src(const double **src, const double *vx, const double *vy, const double *etap, const double *etab,
              const double *f4, const double *f5) {
    src[0] = vx;
    src[1] = vy;
    src[2] = etap;
    src[3] = etab;
    src[4] = f4;
    src[5] = f5;
}

// ---- two damped-Jacobi sweeps in one HBM pass (temporal blocking of a4) -----------------
// Sweep 1 runs one row ahead of sweep 2 on a CTA that owns tw (<= TW - 2) output columns
// j0 .. j0+tw-1: thread t evaluates sweep 1 at column j0-1+t (one redundant column on each
// side), parks (vx', vy') of the last four rows in shared memory, and sweep 2 of row i-1
// reads them back with its column neighbours (one CTA barrier per row).  Strips overlap
// by one sweep-1 row.  The fields are read once and written once per two sweeps: the same
// 64 B/cell as one sweep.  Mirror ghosts of the intermediate iterate are applied when
// sweep 2 reads them, walls are copied through: exactly the arithmetic of two JacobiOp
// sweeps.  On decomposed tiles sweep 1 also updates the first halo ring from the second
// (width-2 halos exchanged once per pass).  (A warp-specialised variant exchanging the intermediate iterate by warp
// shuffles, without CTA barriers, measured 435 us vs 340 us for this one at 4096^2.)
// the two-sweep pass runs 160-thread CTAs (5 warps; 4 CTAs = 20 warps per SM at 96
// registers) with a 5-row ring of 164-wide rows (48.5 KB per CTA): fewer warps wait at each
// row barrier than with r01's 320-thread CTAs (277 vs 294 us at 4096^2)
#ifndef J2_NSJ
#define J2_NSJ 5  // 5-deep landing ring at 160-wide CTAs (r02: 6 rows at 320 threads 293.7 us)
#endif
#ifndef J2_HMIN
#define J2_HMIN 4  // minimum strip height of the two-sweep pass
#endif
#ifndef J2_LATE
#define J2_LATE 0
#endif
#ifndef J2_JT
#define J2_JT 160  // r02: 160 threads x 4 CTAs per SM 277 us; 320 x 2 (r01) 293.7, 192 x 3 314, 128 x 5 283
#endif
#ifndef J2_MINB
#define J2_MINB 4
#endif
constexpr int JT = J2_JT, JRW = JT + 4, NSJ = J2_NSJ;
constexpr int SMEMJ = NSJ * NF * JRW * 8 + 4 * 2 * JT * 8 + NSJ * 8;

struct J2Args {
    const double *src[6];  // vx, vy, eta_p, eta_b, p | bx, rho | by
    double *vxo, *vyo;
    double omega, gx, gy;
    int tw;   // output columns per CTA (even, <= TW - 2)
    int seg;  // doubles staged per row and field (<= the ring row width; 16-B multiple)
    Reg2 R;   // row / column ranges (per blockIdx.z)
};

// Register window with a static rotation: row r of the strip lives in slot (r - sfirst) % 3
// and the row loop is unrolled by three, so advancing the window moves no registers.
struct RowV {
    R3 f[NF];
};
__device__ __forceinline__ double pick(const R3 &x, int dc) { return dc < 0 ? x.l : (dc > 0 ? x.r : x.c); }
template <int KA, int KB, int KC>
struct WinV {  // sweep-1 view: A, B, C = slots KA, KB, KC
    const RowV *r;
    __device__ __forceinline__ double A(int k, int dc = 0) const { return pick(r[KA].f[k], dc); }
    __device__ __forceinline__ double B(int k, int dc = 0) const { return pick(r[KB].f[k], dc); }
    __device__ __forceinline__ double C(int k, int dc = 0) const { return pick(r[KC].f[k], dc); }
};
template <int KB, int KC>
struct WinS2 {  // sweep-2 view: velocities from the intermediate rows, the rest one row back
    const RowV *r;
    R3 vx[3], vy[3];
    double lag_eb, lag_5;  // eta_b, f5 of the row above B (already overwritten in the slots)
    __device__ __forceinline__ double A(int k, int dc = 0) const {
        return k == F_VX ? pick(vx[0], dc) : k == F_VY ? pick(vy[0], dc) : k == F_EB ? lag_eb : lag_5;
    }
    __device__ __forceinline__ double B(int k, int dc = 0) const {
        return k == F_VX ? pick(vx[1], dc) : k == F_VY ? pick(vy[1], dc) : pick(r[KB].f[k], dc);
    }
    __device__ __forceinline__ double C(int k, int dc = 0) const {
        return k == F_VX ? pick(vx[2], dc) : k == F_VY ? pick(vy[2], dc) : pick(r[KC].f[k], dc);
    }
};
template <int K>
struct Slot {
    static constexpr int v = K;
};
// Lazy register window: only the components each role reads are held.  Row s is pulled
// from its landing slot twice: the 5 values sweep 1 reads as row C (step s-1) and the 14 it
// reads as row B (step s); the 8 still needed as row A (step s+1) are carried over.  The slot
// is released after its B pull, so rows s and s+1 stay resident.
struct V3 {
    R3 A[NF], B[NF], C[NF];
};
struct W1 {  // sweep-1 view
    const V3 *v;
    __device__ __forceinline__ double A(int k, int dc = 0) const { return pick(v->A[k], dc); }
    __device__ __forceinline__ double B(int k, int dc = 0) const { return pick(v->B[k], dc); }
    __device__ __forceinline__ double C(int k, int dc = 0) const { return pick(v->C[k], dc); }
};
struct W2 {  // sweep-2 view of row s-1: velocities from the intermediate rows, eta from A/B
    const V3 *v;
    R3 vx[3], vy[3];
    double lag_eb;  // eta_b of row s-2
    __device__ __forceinline__ double A(int k, int dc = 0) const {
        return k == F_VX ? pick(vx[0], dc) : k == F_VY ? pick(vy[0], dc) : lag_eb;
    }
    __device__ __forceinline__ double B(int k, int dc = 0) const {
        return k == F_VX ? pick(vx[1], dc) : k == F_VY ? pick(vy[1], dc) : pick(v->A[k], dc);
    }
    __device__ __forceinline__ double C(int k, int dc = 0) const {
        return k == F_VX ? pick(vx[2], dc) : k == F_VY ? pick(vy[2], dc) : pick(v->B[k], dc);
    }
};
template <int MODE, bool TILE>  // TILE = false: a single domain (every side global), no halo-ring logic
__global__ void __launch_bounds__(JT, J2_MINB) k_jacobi2(GridL g, J2Args a, int H) {
    extern __shared__ __align__(128) double sm[];
    double *s1 = sm + NSJ * NF * JRW;  // [4 rows][vx', vy'][JT]
    uint64_t *bars = reinterpret_cast<uint64_t *>(s1 + 4 * 2 * JT);
    const int t = threadIdx.x;
    const int z = blockIdx.z;
    const int j0 = zsel(a.R.j_lo, z) + a.tw * blockIdx.x;
    const int c = j0 - 1 + t;  // sweep-1 column of this thread (= sweep-2 column for 1 <= t <= tw)
    const int i0 = zsel(a.R.i_lo, z) + blockIdx.y * H;
    const int i1 = min(i0 + H - 1, zsel(a.R.i_hi, z));
    const int jhi = zsel(a.R.j_hi, z);
    // decomposed tiles: on a side that is no global boundary the first halo
    // ring holds the neighbour's unknowns; sweep 1 updates it too (from the second ring),
    // so that sweep 2 of the tile's own unknowns is exact.  Global sides: mirrors / walls.
    const int hN = TILE && !g.bN, hS = TILE && !g.bS, hW = TILE && !g.bW, hE = TILE && !g.bE;
    const int rlo = max(i0 - 2, -hN), rhi = min(i1 + 2, g.ncy + 1 + hS);
    const int sfirst = max(i0 - 1, 0), slast = min(i1 + 1, g.ncy + 1);
    const size_t P = g.P;
    auto issue_at = [&](int r, int slot) {  // row r into ring slot `slot` (= (r - rlo) % NSJ)
        uint64_t *bar = bars + slot;
        mbar_expect_tx(bar, NF * a.seg * 8);
#pragma unroll
        for (int f = 0; f < NF; ++f)
            bulk_g2s(sm + (slot * NF + f) * JRW, a.src[f] + (size_t)r * P + (j0 - 2), a.seg * 8, bar);
    };
    if (t == 0) {
        for (int k = 0; k < NSJ; ++k) mbar_init(bars + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0)
        for (int r = rlo; r < rlo + NSJ && r <= rhi; ++r) issue_at(r, r - rlo);
    // rows are waited for strictly in order rlo, rlo+1, ...: the next one's ring slot and
    // mbarrier phase advance incrementally (no division per row)
    int wslot = 0;
    uint32_t wphase = 0;
    auto wait_next = [&](int &slot) {  // wait for the next staged row; this thread's column in it
        slot = wslot;
        mbar_wait(bars + wslot, wphase);
        const double *q = sm + wslot * (NF * JRW) + t + 1;
        if (++wslot == NSJ) {
            wslot = 0;
            wphase ^= 1u;
        }
        return q;
    };
    V3 v;
    auto pullB = [&](const double *q) {
        v.B[F_VX] = R3{q[-1], q[0], q[1]};
        v.B[F_VY] = R3{q[JRW - 1], q[JRW], q[JRW + 1]};
        v.B[F_EP].c = q[F_EP * JRW];
        v.B[F_EP].r = q[F_EP * JRW + 1];
        v.B[F_EB].l = q[F_EB * JRW - 1];
        v.B[F_EB].c = q[F_EB * JRW];
        v.B[F_4].c = q[F_4 * JRW];
        v.B[F_4].r = q[F_4 * JRW + 1];
        v.B[F_5].l = q[F_5 * JRW - 1];
        v.B[F_5].c = q[F_5 * JRW];
    };
    auto pullC = [&](const double *q) {
        v.C[F_VX].l = q[-1];
        v.C[F_VX].c = q[0];
        v.C[F_VY].c = q[JRW];
        v.C[F_EP].c = q[F_EP * JRW];
        v.C[F_4].c = q[F_4 * JRW];
    };
    auto toA = [&]() {  // row B becomes row A
        v.A[F_EB].l = v.B[F_EB].l;
        v.A[F_EB].c = v.B[F_EB].c;
        v.A[F_EP].c = v.B[F_EP].c;
        v.A[F_EP].r = v.B[F_EP].r;
        v.A[F_VX].c = v.B[F_VX].c;
        v.A[F_VY].c = v.B[F_VY].c;
        v.A[F_VY].r = v.B[F_VY].r;
        v.A[F_5].c = v.B[F_5].c;
    };
    auto refill = [&](int r, int slot) {  // every thread has pulled row r as row B: its slot takes row r + NSJ
        if (t == 0 && r + NSJ <= rhi) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_at(r + NSJ, slot);
        }
    };
    if (rlo < sfirst) {
        int sl;
        pullB(wait_next(sl));
        toA();
        __syncthreads();
        refill(rlo, sl);
    }
    int slotB;
    const double *qB = wait_next(slotB);  // row sfirst
    const bool own_col = t >= 1 && t <= a.tw && c <= jhi;
    const bool cx_in = c >= 1 - hW && c <= g.nvxj + hE, cy_in = c >= 1 - hW && c <= g.ncx + hE;
    const double omc = 1.0 - a.omega;
    // w/a_ii and right-hand side of sweep-1 row s-1 (= the sweep-2 row): equal in both sweeps
    double iax = 0.0, iay = 0.0, bxp = 0.0, byp = 0.0, lag_eb = 0.0;
    // one row step s: sweep 1 of row s, sweep 2 of row s-1.  EDGE = false (CTAs whose rows
    // and columns all stay off the boundary): no boundary logic at all.
    // ER: row-boundary logic (rows 0, 1 / ncy, ncy+1 of sweep 1, rows 1 / ncy of sweep 2);
    // EC: column-boundary logic (CTAs whose columns reach a W / E wall).  A single domain
    // takes the row logic per row step and the column logic per CTA, so the CTAs along the
    // walls run the plain interior code on almost every row (tiles: both on edge CTAs).
    auto step = [&](auto er, auto ec, int s) {
        constexpr bool ER = decltype(er)::value, EC = decltype(ec)::value;
        pullB(qB);
        int slotC = 0;
        const double *qC = qB;
        if (s + 1 <= rhi) {
            qC = wait_next(slotC);
            pullC(qC);
        }
        const W1 w{&v};
        // ---- sweep 1, row s
        double vx1 = v.B[F_VX].c, vy1 = v.B[F_VY].c, iax_n = 0.0, iay_n = 0.0, bx_n = 0.0, by_n = 0.0;
        // (iax / iay hold w / a_ii: the S form of the update, lxs_win)
        if ((!ER || (s >= 1 - hN && s <= g.ncy + hS)) && (!EC || cx_in)) {
            const RowS x = lxs_win<ER>(g, w, s);
            bx_n = (MODE == RHS_FINE) ? fx_win(w, a.gx) - (w.B(F_4) - w.B(F_4, 1)) * g.idx : w.B(F_4);
            iax_n = a.omega * rcp(x.a);
            vx1 = fma(iax_n, bx_n - x.S, omc * w.B(F_VX));
        }
        if ((!ER || (s >= 1 - hN && s <= g.nvyi + hS)) && (!EC || cy_in)) {
            const RowS y = lys_win<EC>(g, w, c);
            by_n = (MODE == RHS_FINE) ? fy_win(w, a.gy) - (w.B(F_4) - w.C(F_4)) * g.idy : w.B(F_5);
            iay_n = a.omega * rcp(y.a);
            vy1 = fma(iay_n, by_n - y.S, omc * w.B(F_VY));
        }
        s1[((s & 3) * 2 + 0) * JT + t] = vx1;
        s1[((s & 3) * 2 + 1) * JT + t] = vy1;
        __syncthreads();
        if (!J2_LATE) refill(s, slotB);
        // ---- sweep 2, row i = s-1 on the intermediate iterate
        const int i = s - 1;
        if (own_col && i >= i0 && i <= i1) {
            const double *qa = s1 + (((s - 2) & 3) * 2) * JT + t, *qb = s1 + (((s - 1) & 3) * 2) * JT + t,
                         *qc = s1 + ((s & 3) * 2) * JT + t;
            W2 u;
            u.v = &v;
            u.lag_eb = lag_eb;
            u.vx[0] = R3{0.0, qa[0], 0.0};
            u.vx[1] = R3{qb[-1], qb[0], qb[1]};
            u.vx[2] = R3{qc[-1], qc[0], 0.0};
            u.vy[0] = R3{0.0, qa[JT], qa[JT + 1]};
            u.vy[1] = R3{qb[JT - 1], qb[JT], qb[JT + 1]};
            u.vy[2] = R3{0.0, qc[JT], 0.0};
            // (the wall mirrors of the intermediate iterate are folded into w / a_ii: lxs_win /
            // lys_win leave the ghosts out on global sides)
            if (!EC || c <= g.nvxj) {
                const RowS x = lxs_win<ER>(g, u, i);
                const double vn = fma(iax, bxp - x.S, omc * u.B(F_VX));
                a.vxo[(size_t)i * P + c] = vn;
                if (ER && i == 1 && g.bN) a.vxo[c] = g.sN * vn;
                if (ER && i == g.ncy && g.bS) a.vxo[(size_t)(g.ncy + 1) * P + c] = g.sS * vn;
            }
            if (!ER || i <= g.nvyi) {
                const RowS y = lys_win<EC>(g, u, c);
                const double vn = fma(iay, byp - y.S, omc * u.B(F_VY));
                a.vyo[(size_t)i * P + c] = vn;
                if (EC && c == 1 && g.bW) a.vyo[(size_t)i * P] = g.sW * vn;
                if (EC && c == g.ncx && g.bE) a.vyo[(size_t)i * P + g.ncx + 1] = g.sE * vn;
            }
        }
        if (J2_LATE) refill(s, slotB);
        qB = qC;
        slotB = slotC;
        lag_eb = v.A[F_EB].c;
        toA();
        iax = iax_n;
        iay = iay_n;
        bxp = bx_n;
        byp = by_n;
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    if (TILE) {  // decomposed tiles: all boundary / halo-ring logic on the edge CTAs
        const bool interior = i0 >= 2 && i1 + 1 <= g.ncy - 1 && j0 >= 2 && j0 + JT - 2 <= g.ncx - 1;
        if (interior)
            for (int s = sfirst; s <= slast; ++s) step(F_(), F_(), s);
        else
            for (int s = sfirst; s <= slast; ++s) step(T_(), T_(), s);
    } else {  // rows 0..2 and ncy..ncy+1 take the row logic (sweep 1 rows 0, 1, ncy, ncy+1; sweep 2 rows 1, ncy)
        const bool col_edge = !(j0 >= 2 && j0 + JT - 2 <= g.ncx - 1);
        for (int s = sfirst; s <= slast; ++s) {
            const bool row_edge = s <= 2 || s >= g.ncy;
            if (col_edge) {
                if (row_edge) step(T_(), T_(), s);
                else step(F_(), T_(), s);
            } else {
                if (row_edge) step(T_(), F_(), s);
                else step(F_(), F_(), s);
            }
        }
    }
}

// ---- the last post-smoothing sweep of V-cycle k fused with the Uzawa step of iterate k and
// the first pre-smoothing sweep of V-cycle k+1 (a4 + a10 + a3 + a4) ------
// Stage 1 (row s) is the Jacobi sweep of JacobiOp on L v = f - G p^(k-1) from v^(k-1/2) (the
// last post-smoothing sweep: its output is v^k); stage 2 (row s-1) is JacobiUzawaOp on v^k
// held in shared memory like sweep 2 of k_jacobi2: p^k = (p^(k-1) - mshift) + alpha eta_P
// (-D v^k), the partial sums of E(v^k, p^k) and v' = v^k + omega (f - L v^k - G p^k)/a_ii.
// One HBM pass instead of two (JacobiOp + JacobiUzawaOp).  v^k itself is not written: when
// E(v^k, p^k) <= rtol the solver recomputes it with one JacobiOp sweep from v^(k-1/2), which
// this pass leaves untouched (driver.cu solve_uzawa_fused).  Single domains.
#ifndef JJ_T
#define JJ_T 160  // r02: 160 x 3 CTAs per SM 350.8 us, 256 x 2 356.4, 192 x 2 379.2 (128 registers)
#endif
#ifndef JJ_MINB
#define JJ_MINB 3
#endif
constexpr int JJT = JJ_T, JJRW = JJT + 4;
constexpr int SMEMJJ = NSJ * NF * JJRW * 8 + 4 * 2 * JJT * 8 + NSJ * 8;

struct JJArgs {
    const double *src[6];  // v^(k-1/2) x, y, eta_p, eta_b, p^(k-1), rho
    double *vxo, *vyo, *po;
    const double *mshift;
    double omega, alpha_s, gx, gy;
    int tw;
};
struct W2J {  // stage-2 view of row s-1: v^k from the intermediate rows, the rest one row back
    const V3 *v;
    R3 vx[3], vy[3];
    double lag_eb, lag_5;  // eta_b, rho of row s-2
    __device__ __forceinline__ double A(int k, int dc = 0) const {
        return k == F_VX ? pick(vx[0], dc) : k == F_VY ? pick(vy[0], dc) : k == F_EB ? lag_eb : lag_5;
    }
    __device__ __forceinline__ double B(int k, int dc = 0) const {
        return k == F_VX ? pick(vx[1], dc) : k == F_VY ? pick(vy[1], dc) : pick(v->A[k], dc);
    }
    __device__ __forceinline__ double C(int k, int dc = 0) const {
        return k == F_VX ? pick(vx[2], dc) : k == F_VY ? pick(vy[2], dc) : pick(v->B[k], dc);
    }
};

__global__ void __launch_bounds__(JJT, JJ_MINB) k_jju(GridL g, JJArgs a, int H, double *__restrict__ partials) {
    extern __shared__ __align__(128) double sm[];
    double *s1 = sm + NSJ * NF * JJRW;  // [4 rows][vx^k, vy^k][JJT]
    uint64_t *bars = reinterpret_cast<uint64_t *>(s1 + 4 * 2 * JJT);
    __shared__ double red[JJT / 32];
    const int t = threadIdx.x;
    const int j0 = 1 + a.tw * blockIdx.x;
    const int c = j0 - 1 + t;
    const int i0 = 1 + blockIdx.y * H;
    const int i1 = min(i0 + H - 1, g.ncy);
    const int rlo = max(i0 - 2, 0), rhi = min(i1 + 2, g.ncy + 1);
    const int sfirst = max(i0 - 1, 0), slast = min(i1 + 1, g.ncy + 1);
    const size_t P = g.P;
    auto issue = [&](int r) {
        const int slot = (r - rlo) % NSJ;
        uint64_t *bar = bars + slot;
        mbar_expect_tx(bar, NF * JJRW * 8);
#pragma unroll
        for (int f = 0; f < NF; ++f)
            bulk_g2s(sm + (slot * NF + f) * JJRW, a.src[f] + (size_t)r * P + (j0 - 2), JJRW * 8, bar);
    };
    if (t == 0) {
        for (int k = 0; k < NSJ; ++k) mbar_init(bars + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0)
        for (int r = rlo; r < rlo + NSJ && r <= rhi; ++r) issue(r);
    auto row_at = [&](int r) {
        const int rel = r - rlo;
        mbar_wait(bars + rel % NSJ, (rel / NSJ) & 1);
        return sm + (rel % NSJ) * NF * JJRW + t + 1;
    };
    V3 v;
    auto pullB = [&](const double *q) {
        v.B[F_VX] = R3{q[-1], q[0], q[1]};
        v.B[F_VY] = R3{q[JJRW - 1], q[JJRW], q[JJRW + 1]};
        v.B[F_EP].c = q[F_EP * JJRW];
        v.B[F_EP].r = q[F_EP * JJRW + 1];
        v.B[F_EB].l = q[F_EB * JJRW - 1];
        v.B[F_EB].c = q[F_EB * JJRW];
        v.B[F_4].c = q[F_4 * JJRW];
        v.B[F_4].r = q[F_4 * JJRW + 1];
        v.B[F_5].l = q[F_5 * JJRW - 1];
        v.B[F_5].c = q[F_5 * JJRW];
    };
    auto pullC = [&](const double *q) {
        v.C[F_VX].l = q[-1];
        v.C[F_VX].c = q[0];
        v.C[F_VY].c = q[JJRW];
        v.C[F_EP].c = q[F_EP * JJRW];
        v.C[F_4].c = q[F_4 * JJRW];
    };
    auto toA = [&]() {  // row B becomes row A (stage 2 also reads p and rho of it)
        v.A[F_EB].l = v.B[F_EB].l;
        v.A[F_EB].c = v.B[F_EB].c;
        v.A[F_EP].c = v.B[F_EP].c;
        v.A[F_EP].r = v.B[F_EP].r;
        v.A[F_VX].c = v.B[F_VX].c;
        v.A[F_VY].c = v.B[F_VY].c;
        v.A[F_VY].r = v.B[F_VY].r;
        v.A[F_4].c = v.B[F_4].c;
        v.A[F_4].r = v.B[F_4].r;
        v.A[F_5].l = v.B[F_5].l;
        v.A[F_5].c = v.B[F_5].c;
    };
    auto refill = [&](int r) {
        if (t == 0 && r + NSJ <= rhi) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(r + NSJ);
        }
    };
    if (rlo < sfirst) {
        pullB(row_at(rlo));
        toA();
        __syncthreads();
        refill(rlo);
    }
    const bool cx_in = c >= 1 && c <= g.nvxj, cy_in = c >= 1 && c <= g.ncx;
    double iax = 0.0, iay = 0.0, lag_eb = 0.0, lag_5 = 0.0;
    double acc[3] = {0.0, 0.0, 0.0};
    const double ms = *a.mshift;
    const double cp = 1.0 / (2.0 * g.idx2 + 2.0 * g.idy2);
    auto step = [&](auto er, auto ec, int s) {  // ER / EC: row / column boundary logic (as k_jacobi2)
        constexpr bool ER = decltype(er)::value, EC = decltype(ec)::value;
        pullB(row_at(s));
        if (s + 1 <= rhi) pullC(row_at(s + 1));
        const W1 w{&v};
        // ---- stage 1, row s: the last post-smoothing sweep (RHS f - G p^(k-1))
        double vx1 = v.B[F_VX].c, vy1 = v.B[F_VY].c, iax_n = 0.0, iay_n = 0.0;
        if ((!ER || (s >= 1 && s <= g.ncy)) && (!EC || cx_in)) {
            const RowX x = lx_win<ER>(g, w, s);
            const double b = fx_win(w, a.gx) - (w.B(F_4) - w.B(F_4, 1)) * g.idx;
            iax_n = rcp(x.a);
            vx1 = w.B(F_VX) + a.omega * (b - x.L) * iax_n;
        }
        if ((!ER || (s >= 1 && s <= g.nvyi)) && (!EC || cy_in)) {
            const RowX y = ly_win<EC>(g, w, c);
            const double b = fy_win(w, a.gy) - (w.B(F_4) - w.C(F_4)) * g.idy;
            iay_n = rcp(y.a);
            vy1 = w.B(F_VY) + a.omega * (b - y.L) * iay_n;
        }
        s1[((s & 3) * 2 + 0) * JJT + t] = vx1;
        s1[((s & 3) * 2 + 1) * JJT + t] = vy1;
        __syncthreads();
        refill(s);
        // ---- stage 2, row i = s-1: Uzawa step + energy + first sweep on v^k
        const int i = s - 1;
        if (i >= i0 && i <= i1 && t >= 1 && t <= a.tw && c <= g.ncx) {
            const double *qa = s1 + (((s - 2) & 3) * 2) * JJT + t, *qb = s1 + (((s - 1) & 3) * 2) * JJT + t,
                         *qc = s1 + ((s & 3) * 2) * JJT + t;
            W2J u;
            u.v = &v;
            u.lag_eb = lag_eb;
            u.lag_5 = lag_5;
            u.vx[0] = R3{0.0, qa[0], 0.0};
            u.vx[1] = R3{qb[-1], qb[0], qb[1]};
            u.vx[2] = R3{qc[-1], qc[0], 0.0};
            u.vy[0] = R3{0.0, qa[JJT], qa[JJT + 1]};
            u.vy[1] = R3{qb[JJT - 1], qb[JJT], qb[JJT + 1]};
            u.vy[2] = R3{0.0, qc[JJT], 0.0};
            if (ER && i == 1) u.vx[0].c = g.sN * u.vx[1].c;
            if (ER && i == g.ncy) u.vx[2].c = g.sS * u.vx[1].c;
            if (EC && c == 1) u.vy[1].l = g.sW * u.vy[1].c;
            if (EC && c == g.ncx) u.vy[1].r = g.sE * u.vy[1].c;
            const double dv = (u.B(F_VX) - u.B(F_VX, -1)) * g.idx + (u.B(F_VY) - u.A(F_VY)) * g.idy;
            const double pn = (u.B(F_4) - ms) + a.alpha_s * u.B(F_EP) * (-dv);
            a.po[(size_t)i * P + c] = pn;
            acc[1] += dv * dv * (u.B(F_EP) * cp);
            acc[2] += pn;
            if (!EC || c <= g.nvxj) {
                const double de = (u.B(F_VX, 1) - u.B(F_VX)) * g.idx + (u.B(F_VY, 1) - u.A(F_VY, 1)) * g.idy;
                const double pe = (u.B(F_4, 1) - ms) + a.alpha_s * u.B(F_EP, 1) * (-de);
                const RowX x = lx_win<ER>(g, u, i);
                const double r = fx_win(u, a.gx) - (pn - pe) * g.idx - x.L;
                acc[0] -= r * r * iax;
                const double vn = u.B(F_VX) + a.omega * r * iax;
                a.vxo[(size_t)i * P + c] = vn;
                if (ER && i == 1) a.vxo[c] = g.sN * vn;
                if (ER && i == g.ncy) a.vxo[(size_t)(g.ncy + 1) * P + c] = g.sS * vn;
            }
            if (!ER || i <= g.nvyi) {
                const double ds = (u.C(F_VX) - u.C(F_VX, -1)) * g.idx + (u.C(F_VY) - u.B(F_VY)) * g.idy;
                const double ps = (u.C(F_4) - ms) + a.alpha_s * u.C(F_EP) * (-ds);
                const RowX y = ly_win<EC>(g, u, c);
                const double r = fy_win(u, a.gy) - (pn - ps) * g.idy - y.L;
                acc[0] -= r * r * iay;
                const double vn = u.B(F_VY) + a.omega * r * iay;
                a.vyo[(size_t)i * P + c] = vn;
                if (EC && c == 1) a.vyo[(size_t)i * P] = g.sW * vn;
                if (EC && c == g.ncx) a.vyo[(size_t)i * P + g.ncx + 1] = g.sE * vn;
            }
        }
        lag_eb = v.A[F_EB].c;
        lag_5 = v.A[F_5].c;
        toA();
        iax = iax_n;
        iay = iay_n;
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    const bool col_edge = !(j0 >= 2 && j0 + JJT - 2 <= g.ncx - 1);
    for (int s = sfirst; s <= slast; ++s) {
        const bool row_edge = s <= 2 || s >= g.ncy;
        if (col_edge) {
            if (row_edge) step(T_(), T_(), s);
            else step(F_(), T_(), s);
        } else {
            if (row_edge) step(T_(), F_(), s);
            else step(F_(), F_(), s);
        }
    }
    // deterministic CTA reduction of (Sv, Sp, sum p^k): fixed xor tree per warp, warps in order
    const size_t b = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double x = acc[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        __syncthreads();
        if ((t & 31) == 0) red[t >> 5] = x;
        __syncthreads();
        if (t < 32) {
            x = (t < JJT / 32) ? red[t] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if (t == 0) partials[b * 3 + k] = x;
        }
    }
}


// ---- fine residual fused with its restriction (a3 + a5) --------------------------------
// A CTA streams fine rows through the TMA landing ring (columns j0-1 .. j0+tw, tw <= TW-2:
// one redundant column each side), evaluates r = b - L v on each row into an 8-row shared
// ring, and every time a coarse row I is complete (fine row min(2I+1, ncy) done) emits
// b^H(I, .) for the tw/2 coarse columns it owns with the normalised weights of
// k_restrict_vel (Appendix B; rows / columns outside the domain dropped and renormalised).
// The fine residual never reaches HBM: 48 B/fine cell read + 4 B written instead of 84.
#ifndef RR_NS
#define RR_NS 4  // 3 CTAs per SM (24 warps): 203 -> 184 us at 4096^2 (tools/variants.py, r02)
#endif
#ifndef RR_ROWS
#define RR_ROWS 5
#endif
#ifndef RR_MINB
#define RR_MINB 3
#endif
#ifndef RR_TW
#define RR_TW TW
#endif
constexpr int NSRR = RR_NS;      // landing ring depth of the residual+restriction pass
constexpr int RRR = RR_ROWS;     // residual rows kept for the restriction (>= 5: rows 2I-2..2I+1 + the next)
constexpr int RTW = RR_TW, RRW = RTW + 4;  // CTA width (threads = columns) and staged row width
constexpr int SMEMRR = NSRR * NF * RRW * 8 + RRR * 2 * RTW * 8 + NSRR * 8;

struct RRArgs {
    const double *src[6];  // vx, vy, eta_p, eta_b, p | bx, rho | by
    double *bxc, *byc;     // coarse right-hand sides
    double gx, gy;
    int tw;
};

template <int MODE>
__global__ void __launch_bounds__(RTW, RR_MINB) k_resrestrict(GridL g, GridL gc, RRArgs a, int HC) {
    extern __shared__ __align__(128) double sm[];
    double *rr = sm + NSRR * NF * RRW;  // [RRR rows][rx, ry][RTW]
    uint64_t *bars = reinterpret_cast<uint64_t *>(rr + RRR * 2 * RTW);
    const int t = threadIdx.x;
    const int j0 = 1 + a.tw * blockIdx.x;  // odd: coarse columns (j0+1)/2 ..
    const int c = j0 - 1 + t;
    const int I0 = 1 + blockIdx.y * HC;
    const int I1 = min(I0 + HC - 1, gc.ncy);
    // decomposed tiles: the residual is also evaluated on the first halo ring of non-global
    // sides (from the second ring), where the restriction weights reach
    const int hN = !g.bN, hS = !g.bS, hW = !g.bW, hE = !g.bE;
    const int ilo = max(2 * I0 - 2, 1 - hN), ihi = min(2 * I1 + 1, g.ncy + hS);
    const int rlo = ilo - 1, rhi = ihi + 1;
    const size_t P = g.P;
    auto issue_at = [&](int r, int slot) {
        uint64_t *bar = bars + slot;
        mbar_expect_tx(bar, NF * RRW * 8);
#pragma unroll
        for (int f = 0; f < NF; ++f)
            bulk_g2s(sm + (slot * NF + f) * RRW, a.src[f] + (size_t)r * P + (j0 - 2), RRW * 8, bar);
    };
    if (t == 0) {
        for (int k = 0; k < NSRR; ++k) mbar_init(bars + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0)
        for (int r = rlo; r < rlo + NSRR && r <= rhi; ++r) issue_at(r, r - rlo);
    // lazy register window (as k_jacobi2): row i pulled as row C at step i-1 (5 values) and as
    // row B at step i (14); only the 8 values row A still needs are carried
    int wslot = 0;
    uint32_t wphase = 0;
    auto wait_next = [&](int &slot) {  // rows are waited for in order rlo, rlo+1, ...
        slot = wslot;
        mbar_wait(bars + wslot, wphase);
        const double *q = sm + wslot * (NF * RRW) + t + 1;
        if (++wslot == NSRR) {
            wslot = 0;
            wphase ^= 1u;
        }
        return q;
    };
    V3 v;
#pragma unroll
    for (int f = 0; f < NF; ++f) v.A[f] = v.B[f] = v.C[f] = R3{0.0, 0.0, 0.0};
    auto pullB = [&](const double *q) {
        v.B[F_VX] = R3{q[-1], q[0], q[1]};
        v.B[F_VY] = R3{q[RRW - 1], q[RRW], q[RRW + 1]};
        v.B[F_EP].c = q[F_EP * RRW];
        v.B[F_EP].r = q[F_EP * RRW + 1];
        v.B[F_EB].l = q[F_EB * RRW - 1];
        v.B[F_EB].c = q[F_EB * RRW];
        v.B[F_4].c = q[F_4 * RRW];
        v.B[F_4].r = q[F_4 * RRW + 1];
        v.B[F_5].l = q[F_5 * RRW - 1];
        v.B[F_5].c = q[F_5 * RRW];
    };
    auto pullC = [&](const double *q) {
        v.C[F_VX].l = q[-1];
        v.C[F_VX].c = q[0];
        v.C[F_VY].c = q[RRW];
        v.C[F_EP].c = q[F_EP * RRW];
        v.C[F_4].c = q[F_4 * RRW];
    };
    auto toA = [&]() {
        v.A[F_EB].l = v.B[F_EB].l;
        v.A[F_EB].c = v.B[F_EB].c;
        v.A[F_EP].c = v.B[F_EP].c;
        v.A[F_EP].r = v.B[F_EP].r;
        v.A[F_VX].c = v.B[F_VX].c;
        v.A[F_VY].c = v.B[F_VY].c;
        v.A[F_VY].r = v.B[F_VY].r;
        v.A[F_5].c = v.B[F_5].c;
    };
    auto refill = [&](int r, int slot) {  // row r pulled as row B by every thread: its slot takes r + NSRR
        if (t == 0 && r + NSRR <= rhi) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_at(r + NSRR, slot);
        }
    };
    int slotA;
    pullB(wait_next(slotA));  // row rlo = the first step's row A
    toA();
    int slotB;
    const double *qB = wait_next(slotB);  // row ilo
    __syncthreads();
    refill(rlo, slotA);
    const bool cx_in = c >= 1 - hW && c <= g.nvxj + hE, cy_in = c >= 1 - hW && c <= g.ncx + hE;
    // emit phase: threads [0, tw/2) restrict vx, threads [tw/2, tw) restrict vy (one coarse
    // value each, so no half of the CTA idles at the next barrier)
    const int half = a.tw / 2;
    const int J = (j0 + 1) / 2 + (t < half ? t : t - half);  // coarse column of this thread
    const bool emit_x = t < half && J <= gc.nvxj, emit_y = t >= half && t < 2 * half && J <= gc.ncx;
    for (int i = ilo; i <= ihi; ++i) {
        pullB(qB);  // A = i-1, B = i, C = i+1 (rhi = ihi + 1: row i+1 always staged)
        int slotC;
        const double *qC = wait_next(slotC);
        pullC(qC);
        const W1 w{&v};
        double rx = 0.0, ry = 0.0;
        if (cx_in) {
            const double b = (MODE == RHS_FINE) ? fx_win(w, a.gx) - (w.B(F_4) - w.B(F_4, 1)) * g.idx : w.B(F_4);
            rx = b - lx_win(g, w, i).L;
        }
        if (cy_in && i <= g.nvyi + hS) {
            const double b = (MODE == RHS_FINE) ? fy_win(w, a.gy) - (w.B(F_4) - w.C(F_4)) * g.idy : w.B(F_5);
            ry = b - ly_win(g, w, c).L;
        }
        rr[((i % RRR) * 2 + 0) * RTW + t] = rx;
        rr[((i % RRR) * 2 + 1) * RTW + t] = ry;
        __syncthreads();
        refill(i, slotB);
        // coarse row completed by fine row i (global S side: row ncy + 1 is dropped)
        const int I = (i & 1) ? (i - 1) / 2 : ((i == g.ncy && g.bS) ? i / 2 : 0);
        if (I >= I0 && I <= I1) {
            if (emit_x) {  // vx: x vertex-centred [1/2, 1, 1/2], y cell-centred [1/4, 3/4, 3/4, 1/4]
                const int q = 2 * J - (j0 - 1);  // ring column of fine column 2J
                double sx = 0.0, wsum = 0.0;
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    const int fi = 2 * I - 2 + d;
                    if ((fi < 1 && g.bN) || (fi > g.ncy && g.bS)) continue;
                    const double *row = rr + ((fi % RRR) * 2 + 0) * RTW;
                    const double h = 0.5 * row[q - 1] + row[q] + 0.5 * row[q + 1];
                    const double wd = (d == 0 || d == 3) ? 0.25 : 0.75;
                    sx += wd * h;
                    wsum += wd;
                }
                a.bxc[at(gc, I, J)] = sx * (wsum == 2.0 ? 0.25 : 1.0 / (2.0 * wsum));
            }
            if (emit_y && I <= gc.nvyi) {  // vy: x cell-centred, y vertex-centred
                const int q = 2 * J - 2 - (j0 - 1);  // ring column of fine column 2J-2
                double sy = 0.0, wsum = 0.0;
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    const int fj = 2 * J - 2 + d;
                    if ((fj < 1 && g.bW) || (fj > g.ncx && g.bE)) continue;
                    const double col = 0.5 * rr[(((2 * I - 1) % RRR) * 2 + 1) * RTW + q + d] +
                                       rr[(((2 * I) % RRR) * 2 + 1) * RTW + q + d] +
                                       0.5 * rr[(((2 * I + 1) % RRR) * 2 + 1) * RTW + q + d];
                    const double wd = (d == 0 || d == 3) ? 0.25 : 0.75;
                    sy += wd * col;
                    wsum += wd;
                }
                a.byc[at(gc, I, J)] = sy * (wsum == 2.0 ? 0.25 : 1.0 / (2.0 * wsum));
            }
        }
        toA();
        qB = qC;
        slotB = slotC;
    }
}


// ---- the last pre-smoothing pair fused with the residual and its restriction ------------
// (a4 + a3 + a5; single domains).  One row step s: sweep 1 of row s (-> s1 ring), CTA
// barrier, sweep 2 of row s-1 (-> HBM for the owned cells and -> s2 ring), the residual
// r = b - L v2 of row s-3 on the s2 ring (-> rr ring), and the restriction of the coarse row
// whose last fine row is s-4 (as k_resrestrict).  Every ring row a stage reads was written
// at an earlier step, so ONE barrier per step orders all of them.  The CTA owns tw = JT2 - 6
// columns (column c = j0 - 3 + t: sweep 1 valid on every lane, sweep 2 on lanes 1..JT2-2,
// the residual on 2..JT2-3, which covers the restriction's reach) and a strip of coarse rows.
// The residual's viscosities and right-hand side of rows s-2..s-4 ride in registers (the
// lazy window's row-A values carried two more steps).  One HBM pass instead of two: reads 6 +
// writes 2 fields + b^H (1/4): 64 + 4 B per fine cell instead of 64 + 52.  Off by default
// (slower than the two passes it replaces, see j2rr_ok).
#ifndef J2R_T
#define J2R_T 160
#endif
#ifndef J2R_MINB
#define J2R_MINB 3
#endif
constexpr int JT2 = J2R_T, JRW2 = JT2 + 4;
constexpr int SMEMJ2R = NSJ * NF * JRW2 * 8 + (4 + 4 + RRR) * 2 * JT2 * 8 + NSJ * 8;

struct J2RArgs {
    const double *src[6];  // vx, vy, eta_p, eta_b, p | bx, rho | by
    double *vxo, *vyo;     // the pair's output (the smoothed iterate)
    double *bxc, *byc;     // coarse right-hand sides
    double omega, gx, gy;
    int tw;
};
struct E4 {  // viscosities of a carried row: eta_b (l, c), eta_p (c, r)
    double ebl, ebc, epc, epr;
};
struct W3 {  // residual view of row s-3: velocities from the s2 ring, viscosities carried
    R3 vx[3], vy[3];
    E4 eb, ec;       // rows s-3 (B) and s-2 (C)
    double lag4_eb;  // eta_b (c) of row s-4 (A)
    __device__ __forceinline__ double A(int k, int dc = 0) const {
        return k == F_VX ? pick(vx[0], dc) : k == F_VY ? pick(vy[0], dc) : lag4_eb;
    }
    __device__ __forceinline__ double B(int k, int dc = 0) const {
        return k == F_VX ? pick(vx[1], dc) : k == F_VY ? pick(vy[1], dc) : k == F_EB ? (dc < 0 ? eb.ebl : eb.ebc)
                                                                                     : (dc > 0 ? eb.epr : eb.epc);
    }
    __device__ __forceinline__ double C(int k, int dc = 0) const {
        return k == F_VX ? pick(vx[2], dc) : k == F_VY ? pick(vy[2], dc) : ec.epc;
    }
};

template <int MODE>
__global__ void __launch_bounds__(JT2, J2R_MINB) k_j2rr(GridL g, GridL gc, J2RArgs a, int HC) {
    extern __shared__ __align__(128) double sm[];
    double *s1 = sm + NSJ * NF * JRW2;  // [4 rows][vx1, vy1][JT2]
    double *s2 = s1 + 4 * 2 * JT2;      // [4 rows][vx2, vy2][JT2]
    double *rr = s2 + 4 * 2 * JT2;      // [RRR rows][rx, ry][JT2]
    uint64_t *bars = reinterpret_cast<uint64_t *>(rr + RRR * 2 * JT2);
    const int t = threadIdx.x;
    const int j0 = 1 + a.tw * blockIdx.x;  // odd: the staged segment starts at j0 - 4
    const int c = j0 - 3 + t;
    const int I0 = 1 + blockIdx.y * HC, I1 = min(I0 + HC - 1, gc.ncy);
    const int o_lo = 2 * I0 - 1, o_hi = min(2 * I1, g.ncy);         // owned fine rows (pair output)
    const int r_lo = max(2 * I0 - 2, 1), r_hi = min(2 * I1 + 1, g.ncy);  // residual rows
    const int w_lo = 2 * I0 - 3, w_hi = 2 * I1 + 2;                 // sweep-2 rows (clipped to 1..ncy)
    const int rlo = max(2 * I0 - 5, 0), rhi = min(2 * I1 + 4, g.ncy + 1);
    const size_t P = g.P;
    auto issue_at = [&](int r, int slot) {
        uint64_t *bar = bars + slot;
        mbar_expect_tx(bar, NF * JRW2 * 8);
#pragma unroll
        for (int f = 0; f < NF; ++f)
            bulk_g2s(sm + (slot * NF + f) * JRW2, a.src[f] + (size_t)r * P + (j0 - 4), JRW2 * 8, bar);
    };
    if (t == 0) {
        for (int k = 0; k < NSJ; ++k) mbar_init(bars + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int e = t; e < 8 * 2 * JT2; e += JT2) s1[e] = 0.0;  // s1 and s2: rows never swept read as walls (0)
    __syncthreads();
    if (t == 0)
        for (int r = rlo; r < rlo + NSJ && r <= rhi; ++r) issue_at(r, r - rlo);
    int wslot = 0;
    uint32_t wphase = 0;
    auto wait_next = [&](int &slot) {
        slot = wslot;
        mbar_wait(bars + wslot, wphase);
        const double *q = sm + wslot * (NF * JRW2) + t + 1;
        if (++wslot == NSJ) {
            wslot = 0;
            wphase ^= 1u;
        }
        return q;
    };
    V3 v;
#pragma unroll
    for (int f = 0; f < NF; ++f) v.A[f] = v.B[f] = v.C[f] = R3{0.0, 0.0, 0.0};
    auto pullB = [&](const double *q) {
        v.B[F_VX] = R3{q[-1], q[0], q[1]};
        v.B[F_VY] = R3{q[JRW2 - 1], q[JRW2], q[JRW2 + 1]};
        v.B[F_EP].c = q[F_EP * JRW2];
        v.B[F_EP].r = q[F_EP * JRW2 + 1];
        v.B[F_EB].l = q[F_EB * JRW2 - 1];
        v.B[F_EB].c = q[F_EB * JRW2];
        v.B[F_4].c = q[F_4 * JRW2];
        v.B[F_4].r = q[F_4 * JRW2 + 1];
        v.B[F_5].l = q[F_5 * JRW2 - 1];
        v.B[F_5].c = q[F_5 * JRW2];
    };
    auto pullC = [&](const double *q) {
        v.C[F_VX].l = q[-1];
        v.C[F_VX].c = q[0];
        v.C[F_VY].c = q[JRW2];
        v.C[F_EP].c = q[F_EP * JRW2];
        v.C[F_4].c = q[F_4 * JRW2];
    };
    auto toA = [&]() {
        v.A[F_EB].l = v.B[F_EB].l;
        v.A[F_EB].c = v.B[F_EB].c;
        v.A[F_EP].c = v.B[F_EP].c;
        v.A[F_EP].r = v.B[F_EP].r;
        v.A[F_VX].c = v.B[F_VX].c;
        v.A[F_VY].c = v.B[F_VY].c;
        v.A[F_VY].r = v.B[F_VY].r;
        v.A[F_5].c = v.B[F_5].c;
    };
    auto refill = [&](int r, int slot) {
        if (t == 0 && r + NSJ <= rhi) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_at(r + NSJ, slot);
        }
    };
    int slotA;
    pullB(wait_next(slotA));  // row rlo: row A of the first step
    toA();
    int slotB = 0;
    const double *qB = rlo + 1 <= rhi ? wait_next(slotB) : nullptr;
    __syncthreads();
    refill(rlo, slotA);
    const bool cx_in = c >= 1 && c <= g.nvxj, cy_in = c >= 1 && c <= g.ncx;
    const bool lane2 = t >= 1 && t <= JT2 - 2, lane3 = t >= 2 && t <= JT2 - 3;
    const bool own_col = t >= 3 && t < 3 + a.tw && c <= g.ncx;
    // carried state: b and 1/a_ii of sweep-1 rows s-1 (p), s-2 (2), s-3 (3); viscosities of
    // rows s-2, s-3 and eta_b of row s-4 for the residual
    double iax = 0.0, iay = 0.0, bxp = 0.0, byp = 0.0, bx2 = 0.0, by2 = 0.0, bx3 = 0.0, by3 = 0.0;
    E4 e2{0.0, 0.0, 0.0, 0.0}, e3{0.0, 0.0, 0.0, 0.0};
    double lag4_eb = 0.0;
    // emission lanes (as k_resrestrict): [0, tw/2) vx, [tw/2, tw) vy, one coarse column each
    const int half = a.tw / 2;
    const int J = (j0 + 1) / 2 + (t < half ? t : t - half);
    const bool emit_x = t < half && J <= gc.nvxj, emit_y = t >= half && t < 2 * half && J <= gc.ncx;
    // the last step restricts coarse row I1, completed by fine row 2 I1 + 1 (row ncy on the
    // last strip: row ncy + 1 lies outside the domain)
    const int s_lo = rlo + 1, s_hi = (2 * I1 >= g.ncy ? g.ncy : 2 * I1 + 1) + 4;
    for (int s = s_lo; s <= s_hi; ++s) {
        const bool haveB = s <= rhi, haveC = s + 1 <= rhi;
        int slotC = 0;
        const double *qC = nullptr;
        if (haveB) pullB(qB);
        if (haveC) {
            qC = wait_next(slotC);
            pullC(qC);
        }
        const W1 w{&v};
        // ---- sweep 1, row s
        double vx1 = v.B[F_VX].c, vy1 = v.B[F_VY].c, iax_n = 0.0, iay_n = 0.0, bx_n = 0.0, by_n = 0.0;
        if (haveB && s >= 1 && s <= g.ncy && cx_in) {
            const RowX x = lx_win<true>(g, w, s);
            bx_n = (MODE == RHS_FINE) ? fx_win(w, a.gx) - (w.B(F_4) - w.B(F_4, 1)) * g.idx : w.B(F_4);
            iax_n = rcp(x.a);
            vx1 = w.B(F_VX) + a.omega * (bx_n - x.L) * iax_n;
        }
        if (haveB && s >= 1 && s <= g.nvyi && cy_in) {
            const RowX y = ly_win<true>(g, w, c);
            by_n = (MODE == RHS_FINE) ? fy_win(w, a.gy) - (w.B(F_4) - w.C(F_4)) * g.idy : w.B(F_5);
            iay_n = rcp(y.a);
            vy1 = w.B(F_VY) + a.omega * (by_n - y.L) * iay_n;
        }
        s1[((s & 3) * 2 + 0) * JT2 + t] = vx1;
        s1[((s & 3) * 2 + 1) * JT2 + t] = vy1;
        __syncthreads();
        if (haveB) refill(s, slotB);
        // ---- sweep 2, row i = s-1 on the intermediate iterate -> HBM (owned) and the s2 ring
        {
            const int i = s - 1;
            double vx2 = 0.0, vy2 = 0.0;
            if (lane2 && i >= max(w_lo, 0) && i <= min(w_hi, g.ncy + 1)) {
                const double *qa = s1 + (((s - 2) & 3) * 2) * JT2 + t, *qb = s1 + (((s - 1) & 3) * 2) * JT2 + t,
                             *qc = s1 + ((s & 3) * 2) * JT2 + t;
                W2 u;
                u.v = &v;
                u.lag_eb = e2.ebc;
                u.vx[0] = R3{0.0, qa[0], 0.0};
                u.vx[1] = R3{qb[-1], qb[0], qb[1]};
                u.vx[2] = R3{qc[-1], qc[0], 0.0};
                u.vy[0] = R3{0.0, qa[JT2], qa[JT2 + 1]};
                u.vy[1] = R3{qb[JT2 - 1], qb[JT2], qb[JT2 + 1]};
                u.vy[2] = R3{0.0, qc[JT2], 0.0};
                if (i == 1) u.vx[0].c = g.sN * u.vx[1].c;
                if (i == g.ncy) u.vx[2].c = g.sS * u.vx[1].c;
                if (c == 1) u.vy[1].l = g.sW * u.vy[1].c;
                if (c == g.ncx) u.vy[1].r = g.sE * u.vy[1].c;
                vx2 = u.B(F_VX);  // walls / rows outside the unknowns keep the intermediate value
                vy2 = u.B(F_VY);
                if (i >= 1 && i <= g.ncy && cx_in) {
                    const RowX x = lx_win<true>(g, u, i);
                    vx2 = u.B(F_VX) + a.omega * (bxp - x.L) * iax;
                }
                if (i >= 1 && i <= g.nvyi && cy_in) {
                    const RowX y = ly_win<true>(g, u, c);
                    vy2 = u.B(F_VY) + a.omega * (byp - y.L) * iay;
                }
                if (own_col && i >= o_lo && i <= o_hi) {
                    if (cx_in) {
                        a.vxo[(size_t)i * P + c] = vx2;
                        if (i == 1) a.vxo[c] = g.sN * vx2;
                        if (i == g.ncy) a.vxo[(size_t)(g.ncy + 1) * P + c] = g.sS * vx2;
                    }
                    if (i <= g.nvyi) {
                        a.vyo[(size_t)i * P + c] = vy2;
                        if (c == 1) a.vyo[(size_t)i * P] = g.sW * vy2;
                        if (c == g.ncx) a.vyo[(size_t)i * P + g.ncx + 1] = g.sE * vy2;
                    }
                }
            }
            s2[(((s - 1) & 3) * 2 + 0) * JT2 + t] = vx2;
            s2[(((s - 1) & 3) * 2 + 1) * JT2 + t] = vy2;
        }
        // ---- residual r = b - L v2, row ir = s-3 (s2 rows s-4 .. s-2, written at earlier steps)
        {
            const int ir = s - 3;
            double rx = 0.0, ry = 0.0;
            if (lane3 && ir >= r_lo && ir <= r_hi) {
                const double *qa = s2 + (((s - 4) & 3) * 2) * JT2 + t, *qb = s2 + (((s - 3) & 3) * 2) * JT2 + t,
                             *qc = s2 + (((s - 2) & 3) * 2) * JT2 + t;
                W3 u;
                u.eb = e3;
                u.ec = e2;
                u.lag4_eb = lag4_eb;
                u.vx[0] = R3{0.0, qa[0], 0.0};
                u.vx[1] = R3{qb[-1], qb[0], qb[1]};
                u.vx[2] = R3{qc[-1], qc[0], 0.0};
                u.vy[0] = R3{0.0, qa[JT2], qa[JT2 + 1]};
                u.vy[1] = R3{qb[JT2 - 1], qb[JT2], qb[JT2 + 1]};
                u.vy[2] = R3{0.0, qc[JT2], 0.0};
                if (ir == 1) u.vx[0].c = g.sN * u.vx[1].c;
                if (ir == g.ncy) u.vx[2].c = g.sS * u.vx[1].c;
                if (c == 1) u.vy[1].l = g.sW * u.vy[1].c;
                if (c == g.ncx) u.vy[1].r = g.sE * u.vy[1].c;
                if (cx_in) rx = bx3 - lx_win<true>(g, u, ir).L;
                if (cy_in && ir <= g.nvyi) ry = by3 - ly_win<true>(g, u, c).L;
            }
            rr[(((ir % RRR) + RRR) % RRR * 2 + 0) * JT2 + t] = rx;
            rr[(((ir % RRR) + RRR) % RRR * 2 + 1) * JT2 + t] = ry;
        }
        // ---- restriction of the coarse row completed by fine row s-4 (rr rows <= s-4)
        {
            const int i = s - 4;
            const int I = (i & 1) ? (i - 1) / 2 : ((i == g.ncy) ? i / 2 : 0);
            if (i >= 1 && I >= I0 && I <= I1) {
                if (emit_x) {
                    const int q = 2 * J - (j0 - 3);  // rr column of fine column 2J
                    double sx = 0.0, wsum = 0.0;
#pragma unroll
                    for (int d = 0; d < 4; ++d) {
                        const int fi = 2 * I - 2 + d;
                        if (fi < 1 || fi > g.ncy) continue;
                        const double *row = rr + ((fi % RRR) * 2 + 0) * JT2;
                        const double h = 0.5 * row[q - 1] + row[q] + 0.5 * row[q + 1];
                        const double wd = (d == 0 || d == 3) ? 0.25 : 0.75;
                        sx += wd * h;
                        wsum += wd;
                    }
                    a.bxc[at(gc, I, J)] = sx * (wsum == 2.0 ? 0.25 : 1.0 / (2.0 * wsum));
                }
                if (emit_y && I <= gc.nvyi) {
                    const int q = 2 * J - 2 - (j0 - 3);  // rr column of fine column 2J-2
                    double sy = 0.0, wsum = 0.0;
#pragma unroll
                    for (int d = 0; d < 4; ++d) {
                        const int fj = 2 * J - 2 + d;
                        if (fj < 1 || fj > g.ncx) continue;
                        const double col = 0.5 * rr[(((2 * I - 1) % RRR) * 2 + 1) * JT2 + q + d] +
                                           rr[(((2 * I) % RRR) * 2 + 1) * JT2 + q + d] +
                                           0.5 * rr[(((2 * I + 1) % RRR) * 2 + 1) * JT2 + q + d];
                        const double wd = (d == 0 || d == 3) ? 0.25 : 0.75;
                        sy += wd * col;
                        wsum += wd;
                    }
                    a.byc[at(gc, I, J)] = sy * (wsum == 2.0 ? 0.25 : 1.0 / (2.0 * wsum));
                }
            }
        }
        // ---- carry: rows shift down by one
        lag4_eb = e3.ebc;
        e3 = e2;
        e2 = E4{v.A[F_EB].l, v.A[F_EB].c, v.A[F_EP].c, v.A[F_EP].r};
        bx3 = bx2;
        by3 = by2;
        bx2 = bxp;
        by2 = byp;
        toA();
        iax = iax_n;
        iay = iay_n;
        bxp = bx_n;
        byp = by_n;
        qB = qC;
        slotB = slotC;
    }
}

// ---- damped red-black Gauss-Seidel in two streamed passes (a4, reading R11) -------------
// The four phases (vx red, vx black, vy red, vy black; red = (i + j + par) even) as two
// passes, one per component: pass COMP updates that component's red nodes of row s and
// its black nodes of row s-2 in the same row step (one CTA barrier per step), reading the
// other component read-only.  Red values go back into the landing slot (black neighbours
// two rows later read them); every final value is written to the OUTPUT buffer, so the
// input stays the old iterate for the neighbouring CTAs' halos (pass 0: vx in -> vx out,
// pass 1 reads the new vx: vy in -> vy out).  Halo columns j0-1 / j0+tw and rows i0-1 /
// i1+1 get their red update redundantly.  Lane parity picks red (row s) or black (row
// s-2): every thread does one update per step with no divergent paths.  Exactly the
// arithmetic of the four phase kernels.  2 x 56 B/cell per sweep instead of 4 x 64.
struct SmV {  // stencil view straight on three landing slots (values change in place)
    const double *a, *b, *c;
    __device__ __forceinline__ double A(int k, int dc = 0) const { return a[k * RW + dc]; }
    __device__ __forceinline__ double B(int k, int dc = 0) const { return b[k * RW + dc]; }
    __device__ __forceinline__ double C(int k, int dc = 0) const { return c[k * RW + dc]; }
};
constexpr int NSR = 8;  // landing ring: rows s-3 .. s+1 resident, 3 in flight

template <int COMP, int MODE>
__global__ void __launch_bounds__(TW, MINB) k_rbgs_pass(GridL g, J2Args a, int H) {
    extern __shared__ __align__(128) double sm[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + NSR * NF * RW);
    const int t = threadIdx.x;
    const int j0 = 1 + a.tw * blockIdx.x;
    const int c = j0 - 1 + t;
    const int i0 = 1 + blockIdx.y * H;
    const int i1 = min(i0 + H - 1, g.ncy);
    const int rlo = max(i0 - 2, 0), rhi = min(i1 + 2, g.ncy + 1);
    const size_t P = g.P;
    const int nrow = COMP == 0 ? g.ncy : g.nvyi, ncol = COMP == 0 ? g.nvxj : g.ncx;  // unknown range
    auto issue = [&](int r) {
        const int slot = (r - rlo) % NSR;
        uint64_t *bar = bars + slot;
        mbar_expect_tx(bar, NF * RW * 8);
#pragma unroll
        for (int f = 0; f < NF; ++f)
            bulk_g2s(sm + (slot * NF + f) * RW, a.src[f] + (size_t)r * P + (j0 - 2), RW * 8, bar);
    };
    if (t == 0) {
        for (int k = 0; k < NSR; ++k) mbar_init(bars + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0)
        for (int r = rlo; r < rlo + NSR && r <= rhi; ++r) issue(r);
    int landed = rlo - 1;  // rows waited for so far
    auto slot_of = [&](int r) { return sm + ((r - rlo) % NSR) * NF * RW + t + 1; };
    auto wait_to = [&](int r) {
        for (; landed < r; ++landed) {
            const int rel = landed + 1 - rlo;
            mbar_wait(bars + rel % NSR, (rel / NSR) & 1);
        }
    };
    const int s_lo = max(i0 - 1, 1), s_hi = i1 + 2;
    double *out = COMP == 0 ? a.vxo : a.vyo;
    for (int s = s_lo; s <= s_hi; ++s) {
        wait_to(min(s + 1, rhi));
        const bool red = ((s + c + g.par) & 1) == 0;
        const int r = red ? s : s - 2;  // red node of row s, or black node of row s-2
        const bool act = red ? (r <= min(i1 + 1, nrow) && c >= 1 && c <= min(ncol, j0 + a.tw))
                             : (r >= i0 && r <= min(i1, nrow) && t >= 1 && t <= a.tw && c <= ncol);
        if (act) {
            double *sb = slot_of(r);
            const SmV w{slot_of(r - 1), sb, slot_of(r + 1)};
            double vn;
            if (COMP == 0) {
                const RowX x = lx_win(g, w, r);
                const double b = (MODE == RHS_FINE) ? fx_win(w, a.gx) - (w.B(F_4) - w.B(F_4, 1)) * g.idx : w.B(F_4);
                vn = w.B(F_VX) + a.omega * (b - x.L) * rcp(x.a);
            } else {
                const RowX y = ly_win(g, w, c);
                const double b = (MODE == RHS_FINE) ? fy_win(w, a.gy) - (w.B(F_4) - w.C(F_4)) * g.idy : w.B(F_5);
                vn = w.B(F_VY) + a.omega * (b - y.L) * rcp(y.a);
            }
            if (red) sb[COMP * RW] = vn;  // black neighbours of rows r +- 1 read it two steps later
            if (r >= i0 && r <= i1 && t >= 1 && t <= a.tw) {
                out[(size_t)r * P + c] = vn;
                if (COMP == 0) {
                    if (r == 1 && g.bN) out[c] = g.sN * vn;
                    if (r == g.ncy && g.bS) out[(size_t)(g.ncy + 1) * P + c] = g.sS * vn;
                } else {
                    if (c == 1 && g.bW) out[(size_t)r * P] = g.sW * vn;
                    if (c == g.ncx && g.bE) out[(size_t)r * P + g.ncx + 1] = g.sE * vn;
                }
            }
        }
        __syncthreads();
        // row s-3 is done (last read by the black update of row s-2): its slot takes s-3+NSR
        if (t == 0 && s - 3 >= rlo && s - 3 + NSR <= rhi) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(s - 3 + NSR);
        }
    }
}

// ---- damped red-black Gauss-Seidel in ONE streamed pass (a4, reading R11) ---------------
// All four phases of a sweep as a wavefront over the rows of a strip, one CTA barrier per
// row step s:
//   (vx, red)   row s          (vx, black) row s-2
//   (vy, red)   row s-4        (vy, black) row s-6
// A red node's neighbours in its own component are black and vice versa, so at step s the
// lanes with (s + c + par) even do the two red updates and the others the two black ones:
// every lane does one vx and one vy update per step (no idle lanes).  Each update reads
// exactly the values the serial phase order gives it (old black vx for vx red, vx red of
// rows s-3..s-1 for vx black, final vx and old black vy for vy red, vy red of rows s-7..s-5
// for vy black; DESIGN.md §6 lists the check), in place in the shared-memory landing ring,
// which keeps rows s-7 .. s+1 resident plus the rows in flight.  The dependency cone is
// three columns wide on the west and two on the east, so a CTA of TWR lanes (column
// c = j0 - 3 + t; RB1_SPLIT: one warp set for the vx and one for the vy updates, which are
// independent within a step) owns tw = TWR - 6 output columns and the strip recomputes rows i0-2 ..
// i1+3 redundantly.  Fields read once and written once per sweep: 64 B/cell per sweep
// instead of 2 x 56 for the two component passes.  Single domains only
// (the cone is wider than the decomposed tiles' two halo rings).
#ifndef RB1_TW
#define RB1_TW 128
#endif
#ifndef RB1_NS
#define RB1_NS 11
#endif
#ifndef RB1_SPLIT  // 1: separate warps for the vx and the vy update of a column (2 x TWR threads)
#define RB1_SPLIT 1
#endif
constexpr int TWR = RB1_TW, RWR = TWR + 4, NSB = RB1_NS;  // ring: rows s-7 .. s+1 resident
constexpr int NTB = RB1_SPLIT ? 2 * TWR : TWR;
constexpr int SMEMB = NSB * NF * RWR * 8 + NSB * 8;
static_assert(NSB >= 10, "the one-pass RBGS keeps 9 rows resident");

struct SmB {  // stencil view straight on three landing slots of the one-pass ring
    const double *a, *b, *c;
    __device__ __forceinline__ double A(int k, int dc = 0) const { return a[k * RWR + dc]; }
    __device__ __forceinline__ double B(int k, int dc = 0) const { return b[k * RWR + dc]; }
    __device__ __forceinline__ double C(int k, int dc = 0) const { return c[k * RWR + dc]; }
};

template <int MODE>
__global__ void __launch_bounds__(NTB) k_rbgs1(GridL g, J2Args a, int H) {
    extern __shared__ __align__(128) double sm[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + NSB * NF * RWR);
    const int tt = threadIdx.x;
    const int t = RB1_SPLIT ? tt % TWR : tt;        // lane of the column
    const int role = RB1_SPLIT ? tt / TWR : 2;      // 0: vx updates, 1: vy updates, 2: both (warp-uniform)
    const int j0 = 1 + a.tw * blockIdx.x;  // odd: the staged segment starts at j0 - 4 (16-B aligned)
    const int c = j0 - 3 + t;
    const int i0 = 1 + blockIdx.y * H;
    const int i1 = min(i0 + H - 1, g.ncy);
    const int rlo = max(i0 - 3, 0), rhi = min(i1 + 4, g.ncy + 1);
    const size_t P = g.P;
    auto issue = [&](int r) {
        const int slot = (r - rlo) % NSB;
        uint64_t *bar = bars + slot;
        mbar_expect_tx(bar, NF * RWR * 8);
#pragma unroll
        for (int f = 0; f < NF; ++f)
            bulk_g2s(sm + (slot * NF + f) * RWR, a.src[f] + (size_t)r * P + (j0 - 4), RWR * 8, bar);
    };
    if (tt == 0) {
        for (int k = 0; k < NSB; ++k) mbar_init(bars + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tt == 0)
        for (int r = rlo; r < rlo + NSB && r <= rhi; ++r) issue(r);
    // rows are waited for in order; the ring slot / mbarrier phase of the next row to wait for
    // and the slot of row s advance incrementally (no division per access)
    int landed = rlo - 1, wslot = 0;
    uint32_t wphase = 0;
    auto wait_to = [&](int r) {
        for (; landed < r; ++landed) {
            mbar_wait(bars + wslot, wphase);
            if (++wslot == NSB) {
                wslot = 0;
                wphase ^= 1u;
            }
        }
    };
    const double *sm_t = sm + t + 1;
    int sbase = 0;  // ring slot of row s
    auto slot_back = [&](int d) {  // this thread's column in the slot of row s - d (-1 <= d <= NSB - 1)
        int q = sbase - d;
        q += q < 0 ? NSB : 0;
        q -= q >= NSB ? NSB : 0;
        return const_cast<double *>(sm_t + q * (NF * RWR));
    };
    // valid lanes of each phase (the cone) and the output columns of this CTA
    const bool own = t >= 3 && t < 3 + a.tw;
    const bool vx_red_ok = c >= 1 && c <= g.nvxj;
    const bool vx_blk_ok = vx_red_ok && t >= 1 && t <= TWR - 2;
    const bool vy_red_ok = c >= 1 && c <= g.ncx && t >= 2 && t <= TWR - 2;
    const bool vy_blk_ok = c >= 1 && c <= g.ncx && t >= 3 && t <= TWR - 3;
    const int s_lo = max(i0 - 2, 1), s_hi = i1 + 6;
    sbase = (s_lo - rlo) % NSB;
    for (int s = s_lo; s <= s_hi; ++s, sbase = sbase + 1 == NSB ? 0 : sbase + 1) {
        wait_to(min(s + 1, rhi));
        const bool red = ((s + c + g.par) & 1) == 0;
        // ---- vx: red node of row s or black node of row s-2
        if (role != 1) {
            const int d = red ? 0 : 2, r = s - d;
            const bool act = red ? (vx_red_ok && r <= min(i1 + 3, g.ncy))
                                 : (vx_blk_ok && r >= max(i0 - 1, 1) && r <= min(i1 + 2, g.ncy));
            if (act) {
                double *sb = slot_back(d);
                const SmB w{slot_back(d + 1), sb, slot_back(d - 1)};
                const RowX x = lx_win(g, w, r);
                const double b = (MODE == RHS_FINE) ? fx_win(w, a.gx) - (w.B(F_4) - w.B(F_4, 1)) * g.idx : w.B(F_4);
                const double vn = w.B(F_VX) + a.omega * (b - x.L) * rcp(x.a);
                sb[F_VX * RWR] = vn;
                if (own && r >= i0 && r <= i1) {
                    a.vxo[(size_t)r * P + c] = vn;
                    if (r == 1 && g.bN) a.vxo[c] = g.sN * vn;
                    if (r == g.ncy && g.bS) a.vxo[(size_t)(g.ncy + 1) * P + c] = g.sS * vn;
                }
            }
        }
        // ---- vy: red node of row s-4 or black node of row s-6
        if (role != 0) {
            const int d = red ? 4 : 6, r = s - d;
            const bool act = red ? (vy_red_ok && r >= max(i0 - 1, 1) && r <= min(i1 + 1, g.nvyi))
                                 : (vy_blk_ok && r >= i0 && r <= min(i1, g.nvyi));
            if (act) {
                double *sb = slot_back(d);
                const SmB w{slot_back(d + 1), sb, slot_back(d - 1)};
                const RowX y = ly_win(g, w, c);
                const double b = (MODE == RHS_FINE) ? fy_win(w, a.gy) - (w.B(F_4) - w.C(F_4)) * g.idy : w.B(F_5);
                const double vn = w.B(F_VY) + a.omega * (b - y.L) * rcp(y.a);
                sb[F_VY * RWR] = vn;
                if (own && r >= i0 && r <= i1) {
                    a.vyo[(size_t)r * P + c] = vn;
                    if (c == 1 && g.bW) a.vyo[(size_t)r * P] = g.sW * vn;
                    if (c == g.ncx && g.bE) a.vyo[(size_t)r * P + g.ncx + 1] = g.sE * vn;
                }
            }
        }
        __syncthreads();
        // row s-7 was last read by the vy black update of row s-6: its slot takes s-7+NSB
        if (tt == 0 && s - 7 >= rlo && s - 7 + NSB <= rhi) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(s - 7 + NSB);
        }
    }
}

int jt_tw(const GridL &g) {  // two-sweep pass: output columns per CTA (even, <= JT - 2)
    const int ncb = (g.ncx + JT - 3) / (JT - 2);
    int tw = (g.ncx + ncb - 1) / ncb;
    return tw + (tw & 1);
}
dim3 jt_grid(const GridL &g, int *H) {
    const int tw = jt_tw(g);
    const int ncb = (g.ncx + tw - 1) / tw;
    int strips = slots() / MINB * J2_MINB / ncb;  // resident two-sweep CTAs: SMs x J2_MINB
    if (strips < 1) strips = 1;
    int h = (g.ncy + strips - 1) / strips;
    if (h < J2_HMIN) h = J2_HMIN;  // (taller minimum strips: fewer CTAs on the coarse levels)
    *H = h;
    return dim3(ncb, (g.ncy + h - 1) / h);
}
int j2_tw(const GridL &g) {  // output columns per CTA: even, <= TW - 2, balanced over the blocks
    const int ncb = (g.ncx + TW - 3) / (TW - 2);
    int tw = (g.ncx + ncb - 1) / ncb;
    return tw + (tw & 1);
}
dim3 j2_grid(const GridL &g, int *H) {
    const int tw = j2_tw(g);
    const int ncb = (g.ncx + tw - 1) / tw;
    int strips = slots() / ncb;
    if (strips < 1) strips = 1;
    int h = (g.ncy + strips - 1) / strips;
    if (h < 4) h = 4;
    *H = h;
    return dim3(ncb, (g.ncy + h - 1) / h);
}

}  // namespace

bool stream_ok(const GridL &g) { return g.ncx >= TW / 2 && g.ncy >= 8; }
int stream_blocks(const GridL &g) {
    const dim3 gr = stream_grid(g);
    return (int)(gr.x * gr.y);
}

// two-sweep pass / fused residual+restriction: single domains and decomposed tiles whose
// width-2 halos are current (dist.cu exchanges them after every pass)
bool jacobi2_ok(const GridL &g) { return stream_ok(g); }

template <int MODE, bool TILE>
void j2_go_t(const LaunchCtx &c, dim3 grid, int H, const GridL &g, const J2Args &a) {
    static unsigned long long done = 0;
    if (first_on_device(&done))
        cudaFuncSetAttribute(k_jacobi2<MODE, TILE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEMJ);
    k_jacobi2<MODE, TILE><<<grid, JT, SMEMJ, c.stream>>>(g, a, H);
    ++*c.counter;
}
template <int MODE>
void j2_go(const LaunchCtx &c, dim3 grid, int H, const GridL &g, const J2Args &a) {
    if (g.bN && g.bS && g.bW && g.bE) j2_go_t<MODE, false>(c, grid, H, g, a);  // single domain
    else j2_go_t<MODE, true>(c, grid, H, g, a);
}
// one part of the split two-sweep pass (see run_part): part 0 the boundary strips, part 1 the rest
void launch_jacobi2_part(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                         const double *vxi, const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs,
                         double omega, int part) {
    J2Args a;
    a.vxo = vxo;
    a.vyo = vyo;
    a.omega = omega;
    const bool fine = rhs.mode == RHS_FINE;
    fill_src(a.src, vxi, vyi, etap, etab, fine ? rhs.p : rhs.bx, fine ? rhs.rho : rhs.by);
    a.gx = fine ? rhs.gx : 0.0;
    a.gy = fine ? rhs.gy : 0.0;
    const Split sp = split_regions(g);
    auto go = [&](dim3 grid, int H) {
        if (fine) j2_go<RHS_FINE>(c, grid, H, g, a);
        else j2_go<RHS_ARRAYS>(c, grid, H, g, a);
    };
    if (part == 0) {
        if (sp.nns) {
            a.R = sp.ns;
            a.tw = jt_tw(g);
            a.seg = JRW;
            go(dim3((g.ncx + a.tw - 1) / a.tw, 1, sp.nns), 2);
        }
        if (sp.nwe) {
            a.R = sp.we;
            a.tw = 2;
            a.seg = 6;
            int H = (sp.we_rows + slots() - 1) / slots();
            if (H < 4) H = 4;
            go(dim3(1, (sp.we_rows + H - 1) / H, sp.nwe), H);
        }
        return;
    }
    a.R = sp.in;
    a.seg = JRW;
    const int rows = sp.in.i_hi[0] - sp.in.i_lo[0] + 1, cols = sp.in.j_hi[0] - sp.in.j_lo[0] + 1;
    int ncb = (cols + JT - 3) / (JT - 2);
    a.tw = (cols + ncb - 1) / ncb;
    a.tw += a.tw & 1;
    ncb = (cols + a.tw - 1) / a.tw;
    int strips = (slots() / MINB - reserve_sms()) * J2_MINB / ncb;
    if (strips < 1) strips = 1;
    int H = (rows + strips - 1) / strips;
    if (H < 4) H = 4;
    go(dim3(ncb, (rows + H - 1) / H, 1), H);
}

void launch_jacobi2(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap, const double *vxi,
                    const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs, double omega) {
    J2Args a;
    a.vxo = vxo;
    a.vyo = vyo;
    a.omega = omega;
    a.tw = jt_tw(g);
    a.seg = JRW;
    a.R = full_region(g);
    int H = 0;
    const dim3 grid = jt_grid(g, &H);
    if (rhs.mode == RHS_FINE) {
        fill_src(a.src, vxi, vyi, etap, etab, rhs.p, rhs.rho);
        a.gx = rhs.gx;
        a.gy = rhs.gy;
        j2_go<RHS_FINE>(c, grid, H, g, a);
    } else {
        fill_src(a.src, vxi, vyi, etap, etab, rhs.bx, rhs.by);
        a.gx = a.gy = 0.0;
        j2_go<RHS_ARRAYS>(c, grid, H, g, a);
    }
}

void launch_jacobi_stream(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                          const double *vxi, const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs,
                          double omega) {
    if (rhs.mode == RHS_FINE) {
        JacobiOp<RHS_FINE> op;
        fill_src(op.src, vxi, vyi, etap, etab, rhs.p, rhs.rho);
        op.vxo = vxo;
        op.vyo = vyo;
        op.omega = omega;
        op.gx = rhs.gx;
        op.gy = rhs.gy;
        run(c, g, op, nullptr);
    } else {
        JacobiOp<RHS_ARRAYS> op;
        fill_src(op.src, vxi, vyi, etap, etab, rhs.bx, rhs.by);
        op.vxo = vxo;
        op.vyo = vyo;
        op.omega = omega;
        op.gx = op.gy = 0.0;
        run(c, g, op, nullptr);
    }
}

void launch_jacobi_stream_part(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                               const double *vxi, const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs,
                               double omega, int part) {
    if (rhs.mode == RHS_FINE) {
        JacobiOp<RHS_FINE> op;
        fill_src(op.src, vxi, vyi, etap, etab, rhs.p, rhs.rho);
        op.vxo = vxo;
        op.vyo = vyo;
        op.omega = omega;
        op.gx = rhs.gx;
        op.gy = rhs.gy;
        run_part(c, g, op, part);
    } else {
        JacobiOp<RHS_ARRAYS> op;
        fill_src(op.src, vxi, vyi, etap, etab, rhs.bx, rhs.by);
        op.vxo = vxo;
        op.vyo = vyo;
        op.omega = omega;
        op.gx = op.gy = 0.0;
        run_part(c, g, op, part);
    }
}

// the last pre-smoothing pair fused with the residual and its restriction (k_j2rr):
// single-domain levels whose pairs stream; OFF by default (STOKES_J2RR=1 enables it):
// measured slower -- 537 us per fine launch against 245 + 193 us for the pair and the
// residual+restriction pass, layered solve 546 -> 588 ms (r02): the three stencil stages per
// row step at 128 registers (3 CTAs per SM) cost more issue time than the HBM pass they save
bool j2rr_ok(const GridL &g) {
    static const bool on = [] {
        const char *e = getenv("STOKES_J2RR");
        return e && e[0] == '1';
    }();
    return on && g.bN && g.bS && g.bW && g.bE && jacobi2_ok(g);
}
void launch_j2rr(const LaunchCtx &c, const GridL &g, const GridL &gc, const double *etab, const double *etap,
                 const double *vxi, const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs, double omega,
                 double *bxc, double *byc) {
    J2RArgs a;
    const bool fine = rhs.mode == RHS_FINE;
    fill_src(a.src, vxi, vyi, etap, etab, fine ? rhs.p : rhs.bx, fine ? rhs.rho : rhs.by);
    a.vxo = vxo;
    a.vyo = vyo;
    a.bxc = bxc;
    a.byc = byc;
    a.omega = omega;
    a.gx = fine ? rhs.gx : 0.0;
    a.gy = fine ? rhs.gy : 0.0;
    a.tw = JT2 - 6;
    const int ncb = (g.ncx + a.tw - 1) / a.tw;
    int strips = slots() / MINB * J2R_MINB / ncb;  // one wave at J2R_MINB CTAs per SM
    if (strips < 1) strips = 1;
    int HC = (gc.ncy + strips - 1) / strips;
    if (HC < 2) HC = 2;
    const dim3 grid(ncb, (gc.ncy + HC - 1) / HC);
    static unsigned long long done = 0;
    if (first_on_device(&done)) {
        cudaFuncSetAttribute(k_j2rr<RHS_FINE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEMJ2R);
        cudaFuncSetAttribute(k_j2rr<RHS_ARRAYS>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEMJ2R);
    }
    if (fine) k_j2rr<RHS_FINE><<<grid, JT2, SMEMJ2R, c.stream>>>(g, gc, a, HC);
    else k_j2rr<RHS_ARRAYS><<<grid, JT2, SMEMJ2R, c.stream>>>(g, gc, a, HC);
    ++*c.counter;
}

void launch_residual_restrict(const LaunchCtx &c, const GridL &g, const GridL &gc, const double *etab,
                              const double *etap, const double *vx, const double *vy, const RhsArgs &rhs, double *bxc,
                              double *byc) {
    RRArgs a;
    a.bxc = bxc;
    a.byc = byc;
    {  // output columns per CTA: even, <= RTW - 2, balanced over the column blocks
        const int nb = (g.ncx + RTW - 3) / (RTW - 2);
        a.tw = (g.ncx + nb - 1) / nb;
        a.tw += a.tw & 1;
    }
    const int ncb = (g.ncx + a.tw - 1) / a.tw;
    int strips = slots() / MINB * RR_MINB / ncb;  // one wave at RR_MINB CTAs per SM
    if (strips < 1) strips = 1;
    int HC = (gc.ncy + strips - 1) / strips;
    if (HC < 2) HC = 2;
    const dim3 grid(ncb, (gc.ncy + HC - 1) / HC);
    if (rhs.mode == RHS_FINE) {
        fill_src(a.src, vx, vy, etap, etab, rhs.p, rhs.rho);
        a.gx = rhs.gx;
        a.gy = rhs.gy;
        static unsigned long long done = 0;
        if (first_on_device(&done)) {
            cudaFuncSetAttribute(k_resrestrict<RHS_FINE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEMRR);
        }
        k_resrestrict<RHS_FINE><<<grid, RTW, SMEMRR, c.stream>>>(g, gc, a, HC);
    } else {
        fill_src(a.src, vx, vy, etap, etab, rhs.bx, rhs.by);
        a.gx = a.gy = 0.0;
        static unsigned long long done = 0;
        if (first_on_device(&done)) {
            cudaFuncSetAttribute(k_resrestrict<RHS_ARRAYS>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEMRR);
        }
        k_resrestrict<RHS_ARRAYS><<<grid, RTW, SMEMRR, c.stream>>>(g, gc, a, HC);
    }
    ++*c.counter;
}

template <int COMP, int MODE>
void rbgs_pass(const LaunchCtx &c, const GridL &g, const J2Args &a) {
    constexpr int SM = NSR * NF * RW * 8 + NSR * 8;
    static unsigned long long done = 0;
    if (first_on_device(&done)) {
        cudaFuncSetAttribute(k_rbgs_pass<COMP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
    }
    int H = 0;
    const dim3 grid = j2_grid(g, &H);
    k_rbgs_pass<COMP, MODE><<<grid, TW, SM, c.stream>>>(g, a, H);
    ++*c.counter;
}

// one wave of one-pass CTAs over the level; false (use the two component passes) when the
// strips would be shorter than RB1_HMIN rows: each strip recomputes 7 rows and runs H + 8
// barrier steps, which the smaller levels do not amortise (layered 4096^2 RBGS solve with
// the one-pass kernel on every level >= 128^2: 1521 ms vs 1331 ms with two passes, r02)
#ifndef RB1_HMIN
#define RB1_HMIN 32
#endif
int rbgs1_mode();
template <int MODE>
bool rbgs1(const LaunchCtx &c, const GridL &g, const J2Args &a0) {
    static unsigned long long done = 0;
    static int per_sm[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (first_on_device(&done)) {
        cudaFuncSetAttribute(k_rbgs1<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEMB);
        int nb = 0, nsm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_rbgs1<MODE>, NTB, SMEMB);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        per_sm[dev & 63] = (nb > 0 ? nb : 1) * nsm;
    }
    J2Args a = a0;
    a.tw = TWR - 6;
    a.tw -= a.tw & 1;
    const int ncb = (g.ncx + a.tw - 1) / a.tw;
    int strips = per_sm[dev & 63] / ncb;  // one wave of CTAs covers the level
    if (strips < 1) strips = 1;
    int H = (g.ncy + strips - 1) / strips;
    if (rbgs1_mode() != 2 && H < RB1_HMIN) return false;
    if (H < 8) H = 8;
    k_rbgs1<MODE><<<dim3(ncb, (g.ncy + H - 1) / H), NTB, SMEMB, c.stream>>>(g, a, H);
    ++*c.counter;
    return true;
}
// STOKES_RBGS1=0: the two component passes also on single domains (comparison); =2: the
// one-pass kernel on every streamed single-domain level (strips >= 8 rows; parity tests)
int rbgs1_mode() {
    static const int v = [] {
        const char *e = getenv("STOKES_RBGS1");
        return e ? atoi(e) : 1;
    }();
    return v;
}
bool rbgs1_enabled() { return rbgs1_mode() != 0; }

void launch_rbgs_stream(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                        const double *vxi, const double *vyi, double *vxo, double *vyo, const RhsArgs &rhs,
                        double omega) {
    J2Args a;
    a.omega = omega;
    a.tw = j2_tw(g);
    a.vxo = vxo;
    a.vyo = vyo;
    const bool fine = rhs.mode == RHS_FINE;
    a.gx = fine ? rhs.gx : 0.0;
    a.gy = fine ? rhs.gy : 0.0;
    if (g.bN && g.bS && g.bW && g.bE && rbgs1_enabled()) {  // single domain: all four phases in one pass
        fill_src(a.src, vxi, vyi, etap, etab, fine ? rhs.p : rhs.bx, fine ? rhs.rho : rhs.by);
        if (fine ? rbgs1<RHS_FINE>(c, g, a) : rbgs1<RHS_ARRAYS>(c, g, a)) return;
    }
    // pass 0: vx (reads vy old), pass 1: vy (reads the new vx)
    fill_src(a.src, vxi, vyi, etap, etab, fine ? rhs.p : rhs.bx, fine ? rhs.rho : rhs.by);
    if (fine) rbgs_pass<0, RHS_FINE>(c, g, a);
    else rbgs_pass<0, RHS_ARRAYS>(c, g, a);
    a.src[0] = vxo;
    if (fine) rbgs_pass<1, RHS_FINE>(c, g, a);
    else rbgs_pass<1, RHS_ARRAYS>(c, g, a);
}

void launch_residual_stream(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                            const double *vx, const double *vy, const RhsArgs &rhs, double *rx, double *ry) {
    if (rhs.mode == RHS_FINE) {
        ResidualOp<RHS_FINE> op;
        fill_src(op.src, vx, vy, etap, etab, rhs.p, rhs.rho);
        op.rx = rx;
        op.ry = ry;
        op.gx = rhs.gx;
        op.gy = rhs.gy;
        run(c, g, op, nullptr);
    } else {
        ResidualOp<RHS_ARRAYS> op;
        fill_src(op.src, vx, vy, etap, etab, rhs.bx, rhs.by);
        op.rx = rx;
        op.ry = ry;
        op.gx = op.gy = 0.0;
        run(c, g, op, nullptr);
    }
}

void launch_precond_apply(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                          const double *zx, const double *zy, const double *rp, double alpha, double *zp, double *wx,
                          double *wy, double *wp, const double *const *w0, const double *rx, const double *ry,
                          double *partials) {
    PrecondApplyOp op;
    op.src[0] = zx;
    op.src[1] = zy;
    op.src[2] = etap;
    op.src[3] = etab;
    op.src[4] = rp;
    op.src[5] = nullptr;
    op.zp = zp;
    op.wx = wx;
    op.wy = wy;
    op.wp = wp;
    op.w0x = w0 ? w0[0] : nullptr;
    op.w0y = w0 ? w0[1] : nullptr;
    op.w0p = w0 ? w0[2] : nullptr;
    op.rx = rx;
    op.ry = ry;
    op.alpha = alpha;
    run(c, g, op, partials);
}

void launch_jacobi_uzawa(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                         const double *vxi, const double *vyi, double *vxo, double *vyo, const double *pin,
                         double *pout, const double *rho, double gx, double gy, double alpha_signed,
                         const double *mshift, double omega, double *partials) {
    JacobiUzawaOp op;
    fill_src(op.src, vxi, vyi, etap, etab, pin, rho);
    op.vxo = vxo;
    op.vyo = vyo;
    op.po = pout;
    op.mshift = mshift;
    op.alpha_s = alpha_signed;
    op.omega = omega;
    op.gx = gx;
    op.gy = gy;
    run(c, g, op, partials);
}

// single domains whose levels stream (jacobi2_ok); grid = one wave, blocks returned
static dim3 jju_grid(const GridL &g, int *H, int *tw) {
    const int nb = (g.ncx + JJT - 3) / (JJT - 2);
    int w = (g.ncx + nb - 1) / nb;
    w += w & 1;
    const int ncb = (g.ncx + w - 1) / w;
    int strips = slots() / MINB * JJ_MINB / ncb;
    if (strips < 1) strips = 1;
    int h = (g.ncy + strips - 1) / strips;
    if (h < 4) h = 4;
    *H = h;
    *tw = w;
    return dim3(ncb, (g.ncy + h - 1) / h);
}
bool jju_ok(const GridL &g) {
    static const bool on = [] {
        const char *e = getenv("STOKES_JJU");
        return !(e && e[0] == '0');
    }();
    return on && g.bN && g.bS && g.bW && g.bE && jacobi2_ok(g);
}
int jju_blocks(const GridL &g) {
    int H, tw;
    const dim3 gr = jju_grid(g, &H, &tw);
    return (int)(gr.x * gr.y);
}
void launch_jacobi_jju(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                       const double *vxi, const double *vyi, double *vxo, double *vyo, const double *pin, double *pout,
                       const double *rho, double gx, double gy, double alpha_signed, const double *mshift,
                       double omega, double *partials) {
    static unsigned long long done = 0;
    if (first_on_device(&done)) cudaFuncSetAttribute(k_jju, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEMJJ);
    JJArgs a;
    fill_src(a.src, vxi, vyi, etap, etab, pin, rho);
    a.vxo = vxo;
    a.vyo = vyo;
    a.po = pout;
    a.mshift = mshift;
    a.omega = omega;
    a.alpha_s = alpha_signed;
    a.gx = gx;
    a.gy = gy;
    int H = 0;
    const dim3 grid = jju_grid(g, &H, &a.tw);
    k_jju<<<grid, JJT, SMEMJJ, c.stream>>>(g, a, H, partials);
    ++*c.counter;
}

void launch_uzawa_energy(const LaunchCtx &c, const GridL &g, const double *etab, const double *etap,
                         const double *vx, const double *vy, const double *pin, double *pout, const double *rho,
                         double gx, double gy, double alpha_signed, const double *mshift, double *rx, double *ry,
                         double *rp, double *partials) {
    UzawaOp op;
    fill_src(op.src, vx, vy, etap, etab, pin, rho);
    op.po = pout;
    op.mshift = mshift;
    op.alpha_s = alpha_signed;
    op.gx = gx;
    op.gy = gy;
    op.rxo = rx;
    op.ryo = ry;
    op.rpo = rp;
    op.write_p = pout != nullptr;
    run(c, g, op, partials);
}
