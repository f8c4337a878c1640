// Flat (layout-agnostic) vector kernels of the flexible GCR(m) accelerator (a11),
// Alg. 4, readings R13 / R14.
//
// A GCR vector is three padded fields (vx, vy, p) of the fine level.  Every entry that
// is not an unknown is 0 in w-, r- and residual-type vectors (written only at unknowns;
// zeroed at allocation), so inner products may run over the whole padded arrays; z-type
// vectors carry their velocity mirrors, which the axpys keep consistent (linear).
// Each kernel first reduces the previous kernel's per-CTA partials into its scalar
// coefficient (every CTA, same fixed order: deterministic), then streams the vectors with
// 16-B loads and leaves its own per-CTA partials -- one HBM pass per MGS step (fused
// axpy + next dot, 168 B/cell) instead of dot / finalize / axpy / axpy.
#include <math.h>

#include "internal.h"

namespace {

constexpr int FT = 256;  // threads per CTA
#ifndef MGS_UNROLL
#define MGS_UNROLL 2  // elements per thread in flight in the MGS / update streams (SolCx 2048^2 GCR(30): 117.8 -> 117.0 ms)
#endif
constexpr int MGS_U = MGS_UNROLL;
#ifndef FLAT_PER_SM_LONG
#define FLAT_PER_SM_LONG 6
#endif

// sum of partials[b * ncomp + k] over b, fixed order, every CTA identical; result to all threads
__device__ double coef(const double *__restrict__ partials, int nb, int ncomp, int k, double *sh) {
    if (threadIdx.x < 32) {
        double s = 0.0;
        for (int b = threadIdx.x; b < nb; b += 32) s += partials[(size_t)b * ncomp + k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) sh[0] = s;
    }
    __syncthreads();
    const double v = sh[0];
    __syncthreads();
    return v;
}
__device__ double block_sum_ft(double v, double *sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = (threadIdx.x < FT / 32) ? sh[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;
}

struct V3 {
    double *f[3];
};
struct C3 {
    const double *f[3];
};
constexpr int ZT = 32;  // = MAXM (handle.h)
struct ZTab {           // the z_j of the deferred z update, j = 0 .. nz-1
    const double *f[ZT][3];
};

// MGS step j: gamma = <w, w_j> (from the previous partials);
// w -= gamma w_j; z -= gamma z_j; then partial dots for the next coefficient:
// <w, w_{j+1}> if nxt is given, else <w, w> and <r, w> (normalisation + beta).
// z.f[0] == nullptr: the z update is deferred -- gamma is stored to gout and k_gcr_update
// applies z -= gamma_j z_j for every j in the same order (the same operations per element,
// so the same z, for 72 of the 168 B/cell of a step).
__global__ void __launch_bounds__(FT) k_mgs_step(const double *__restrict__ pin, int nbin, int ncin, int kin,
                                                 V3 w, V3 z, C3 wj, C3 zj, C3 nxt, C3 r, size_t n2,
                                                 double *__restrict__ pout, double *__restrict__ gout) {
    __shared__ double sh[32];
    const double gam = coef(pin, nbin, ncin, kin, sh);
    if (gout && blockIdx.x == 0 && threadIdx.x == 0) *gout = gam;
    const bool upd_z = z.f[0] != nullptr;
    double a0 = 0.0, a1 = 0.0;
    const size_t stride = (size_t)gridDim.x * FT;
#pragma unroll
    for (int f = 0; f < 3; ++f) {
        double2 *W = reinterpret_cast<double2 *>(w.f[f]);
        double2 *Z = reinterpret_cast<double2 *>(z.f[f]);
        const double2 *WJ = reinterpret_cast<const double2 *>(wj.f[f]);
        const double2 *ZJ = reinterpret_cast<const double2 *>(zj.f[f]);
        const double2 *N = reinterpret_cast<const double2 *>(nxt.f[f]);
        const double2 *R = reinterpret_cast<const double2 *>(r.f[f]);
#pragma unroll MGS_U
        for (size_t e = blockIdx.x * (size_t)FT + threadIdx.x; e < n2; e += stride) {
            double2 a = W[e], b = WJ[e];
            a.x -= gam * b.x;
            a.y -= gam * b.y;
            W[e] = a;
            if (upd_z) {
                double2 c = Z[e];
                const double2 d = ZJ[e];
                c.x -= gam * d.x;
                c.y -= gam * d.y;
                Z[e] = c;
            }
            if (N) {
                const double2 q = N[e];
                a0 += a.x * q.x + a.y * q.y;
            } else {
                const double2 q = R[e];
                a0 += a.x * a.x + a.y * a.y;
                a1 += q.x * a.x + q.y * a.y;
            }
        }
    }
    a0 = block_sum_ft(a0, sh);
    a1 = block_sum_ft(a1, sh);
    if (threadIdx.x == 0) {
        pout[2 * (size_t)blockIdx.x] = a0;
        pout[2 * (size_t)blockIdx.x + 1] = a1;
    }
}

// normalise + update: nu^2 = <w,w>, beta' = <r,w> (previous partials);
// w /= nu, z /= nu, beta = beta'/nu = <r, w/nu>; x += beta z; r -= beta w; partials of the
// energy of the new r (sum r^2 * ew) and of <r_old, r_old> (breakdown test).
// nz > 0: first the deferred MGS updates of z, z -= gamma_j z_j for j = 0 .. nz-1 in order
// (gammas[j] from the MGS steps), then as before.
__global__ void __launch_bounds__(FT) k_gcr_update(const double *__restrict__ pin, int nbin, V3 w, V3 z, V3 x, V3 r,
                                                   C3 ew, size_t n2, double *__restrict__ pout,
                                                   const double *__restrict__ gammas, int nz, ZTab zt) {
    __shared__ double sh[32];
    __shared__ double gs[ZT];
    if (threadIdx.x < nz) gs[threadIdx.x] = gammas[threadIdx.x];  // (ordered before use by coef's barriers)
    const double nu2 = coef(pin, nbin, 2, 0, sh);
    const double bp = coef(pin, nbin, 2, 1, sh);
    const double s = 1.0 / sqrt(nu2);
    const double beta = bp * s;
    double a0 = 0.0, a1 = 0.0;
    const size_t stride = (size_t)gridDim.x * FT;
#pragma unroll
    for (int f = 0; f < 3; ++f) {
        double2 *W = reinterpret_cast<double2 *>(w.f[f]);
        double2 *Z = reinterpret_cast<double2 *>(z.f[f]);
        double2 *X = reinterpret_cast<double2 *>(x.f[f]);
        double2 *R = reinterpret_cast<double2 *>(r.f[f]);
        const double2 *EW = reinterpret_cast<const double2 *>(ew.f[f]);
#pragma unroll MGS_U
        for (size_t e = blockIdx.x * (size_t)FT + threadIdx.x; e < n2; e += stride) {
            double2 wv = W[e], zv = Z[e], xv = X[e], rv = R[e];
            for (int j = 0; j < nz; ++j) {  // deferred MGS z updates, in step order
                const double2 d = reinterpret_cast<const double2 *>(zt.f[j][f])[e];
                const double gam = gs[j];
                zv.x -= gam * d.x;
                zv.y -= gam * d.y;
            }
            const double2 q = EW[e];
            a1 += rv.x * rv.x + rv.y * rv.y;
            wv.x *= s;
            wv.y *= s;
            zv.x *= s;
            zv.y *= s;
            xv.x += beta * zv.x;
            xv.y += beta * zv.y;
            rv.x -= beta * wv.x;
            rv.y -= beta * wv.y;
            W[e] = wv;
            Z[e] = zv;
            X[e] = xv;
            R[e] = rv;
            a0 += rv.x * rv.x * q.x + rv.y * rv.y * q.y;
        }
    }
    a0 = block_sum_ft(a0, sh);
    a1 = block_sum_ft(a1, sh);
    if (threadIdx.x == 0) {
        pout[2 * (size_t)blockIdx.x] = a0;
        pout[2 * (size_t)blockIdx.x + 1] = a1;
    }
}

// E = sqrt(sum r^2 ew / Sf), nu^2 and <r,r> for the host-side tests -> out[S_E], out[nu2], out[rr]
__global__ void __launch_bounds__(FT) k_gcr_final(const double *__restrict__ pupd, int nbu,
                                                  const double *__restrict__ pnorm, int nbn,
                                                  const double *__restrict__ Sf, double *__restrict__ E,
                                                  double *__restrict__ nu2, double *__restrict__ rr) {
    __shared__ double sh[32];
    const double se = coef(pupd, nbu, 2, 0, sh);
    const double r2 = coef(pupd, nbu, 2, 1, sh);
    const double n2 = coef(pnorm, nbn, 2, 0, sh);
    if (threadIdx.x == 0) {
        *E = Sf[0] > 0.0 ? sqrt(se / Sf[0]) : 0.0;
        *nu2 = n2;
        *rr = r2;
    }
}

// CTAs of the flat GCR kernels for vectors of n2 double2 per field: 4 per SM, 6 for long
// vectors (>= 2^20 double2 per field: 48 warps per SM keep more loads in flight; SolCx 2048^2
// GCR(30): 116.9 -> 106.6 ms; 5 / 7 / 8 per SM 110.2 / 119.7 / 114.7 ms -- 7 and 8 spill into a
// second wave).  Short vectors keep 4 (block 512^2: 27.1 ms vs 28.3 at 6): every CTA also
// reduces all of the previous kernel's partials.
int flat_blocks(size_t n2) {
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (nsm <= 0) nsm = 148;
    }
    return nsm * (n2 >= ((size_t)1 << 20) ? FLAT_PER_SM_LONG : 4);
}

}  // namespace

int gcr_flat_blocks(size_t nfield) { return flat_blocks(nfield / 2); }

void launch_mgs_step(const LaunchCtx &c, const double *pin, int nbin, int ncin, int kin, double *const *w,
                     double *const *z, const double *const *wj, const double *const *zj, const double *const *nxt,
                     const double *const *r, size_t nfield, double *pout, double *gout) {
    V3 W{{w[0] - COL_OFF, w[1] - COL_OFF, w[2] - COL_OFF}};
    V3 Z{{nullptr, nullptr, nullptr}};
    C3 ZJ{{nullptr, nullptr, nullptr}};
    if (z) {  // (z == nullptr: the z update deferred to launch_gcr_update)
        Z = V3{{z[0] - COL_OFF, z[1] - COL_OFF, z[2] - COL_OFF}};
        ZJ = C3{{zj[0] - COL_OFF, zj[1] - COL_OFF, zj[2] - COL_OFF}};
    }
    C3 WJ{{wj[0] - COL_OFF, wj[1] - COL_OFF, wj[2] - COL_OFF}};
    C3 N{{nullptr, nullptr, nullptr}}, R{{nullptr, nullptr, nullptr}};
    if (nxt) N = C3{{nxt[0] - COL_OFF, nxt[1] - COL_OFF, nxt[2] - COL_OFF}};
    else R = C3{{r[0] - COL_OFF, r[1] - COL_OFF, r[2] - COL_OFF}};
    k_mgs_step<<<flat_blocks(nfield / 2), FT, 0, c.stream>>>(pin, nbin, ncin, kin, W, Z, WJ, ZJ, N, R, nfield / 2, pout, gout);
    ++*c.counter;
}

void launch_gcr_update(const LaunchCtx &c, const double *pin, int nbin, double *const *w, double *const *z,
                       double *const *x, double *const *r, const double *const *ew, size_t nfield, double *pout,
                       const double *gammas, int nz, double *const (*zj)[3]) {
    ZTab zt;
    for (int j = 0; j < nz && j < ZT; ++j)
        for (int f = 0; f < 3; ++f) zt.f[j][f] = zj[j][f] - COL_OFF;
    V3 W{{w[0] - COL_OFF, w[1] - COL_OFF, w[2] - COL_OFF}};
    V3 Z{{z[0] - COL_OFF, z[1] - COL_OFF, z[2] - COL_OFF}};
    V3 X{{x[0] - COL_OFF, x[1] - COL_OFF, x[2] - COL_OFF}};
    V3 R{{r[0] - COL_OFF, r[1] - COL_OFF, r[2] - COL_OFF}};
    C3 EW{{ew[0] - COL_OFF, ew[1] - COL_OFF, ew[2] - COL_OFF}};
    k_gcr_update<<<flat_blocks(nfield / 2), FT, 0, c.stream>>>(pin, nbin, W, Z, X, R, EW, nfield / 2, pout, gammas,
                                                     nz < ZT ? nz : ZT, zt);
    ++*c.counter;
}

void launch_gcr_final(const LaunchCtx &c, const double *pupd, int nbu, const double *pnorm, int nbn,
                      const double *Sf, double *E, double *nu2, double *rr) {
    k_gcr_final<<<1, FT, 0, c.stream>>>(pupd, nbu, pnorm, nbn, Sf, E, nu2, rr);
    ++*c.counter;
}
