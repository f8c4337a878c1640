// Anderson acceleration AA(m) with mixing beta over the Uzawa fixed point (SURVEY §8(f)
// NEXT-2): Alg. 5, reading R26.
//
// x = (vx, vy, p) on the padded fine fields.  The history keeps, per ring slot i,
// G_i = G(x^i) and R_i = G(x^i) - x^i (pressures de-meaned: the working pressure is stored
// with a lazy mean, R10), so the mixed update of Alg. 5 is
//   x^{k+1} = (1 - beta) sum a_i x^i + beta sum a_i G_i = sum a_i G_i - (1 - beta) sum a_i R_i.
// Linear combinations keep the velocity mirrors consistent (mirror = +-partner, exact) and
// the walls zero, so the kernels run over whole padded rows; inner products count only
// the unknowns (Euclidean, reading R13).  Three kernels per iteration after the Uzawa step:
//   k_aa_push   G_k, R_k from the working state and T = x^k; partial dots <R_k, R_i>
//   k_aa_solve  one thread: the Gram row, (H + lambda I) z = 1, a = z / sum z (the oracle's
//               elimination, same order), coefficients of G_i and R_i
//   k_aa_update x^{k+1} -> working fields and T, partial sums of p (its lazy mean)
#include <math.h>

#include "internal.h"

namespace {

constexpr int AT = 256;  // threads per CTA (grid-stride over padded elements)


__device__ double block_sum_at(double v, double *sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = (threadIdx.x < AT / 32) ? sh[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;
}

// is padded element (i, j) an unknown of field f (0 vx, 1 vy, 2 p)
__device__ __forceinline__ bool unknown(const GridL &g, int f, int i, int j) {
    if (f == 0) return i >= 1 && i <= g.ncy && j >= 1 && j <= g.nvxj;
    if (f == 1) return i >= 1 && i <= g.nvyi && j >= 1 && j <= g.ncx;
    return i >= 1 && i <= g.ncy && j >= 1 && j <= g.ncx;
}

// NW: compile-time bound on the window (accumulators in registers: fewer for short windows,
// so more CTAs fit per SM)
template <int NW>
__global__ void __launch_bounds__(AT) k_aa_push(GridL g, AAVec work, const double *ms_g, AAVec T, const double *ms_t,
                                                AAVec Gk, AAVec Rk, AAWin win, double *__restrict__ partials) {
    __shared__ double sh[32];
    __shared__ const double *rw[3][AA_MAXS];  // window pointers (no dynamic indexing of the parameters)
    if (threadIdx.x < 3 * AA_MAXS) {
        const int f = threadIdx.x / AA_MAXS, w = threadIdx.x % AA_MAXS;
        rw[f][w] = win.r[w].f[f];
    }
    __syncthreads();
    double acc[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) acc[w] = 0.0;
    const double mg = *ms_g, mt = *ms_t;
    const int rows = g.ncy + 2, cols = g.ncx + 2, nw = win.n, self = win.self;
    // rows over CTAs, columns over threads: coalesced, no per-element index division
#pragma unroll
    for (int f = 0; f < 3; ++f) {
        const double *X = work.f[f], *TT = T.f[f];
        double *GG = Gk.f[f], *RR = Rk.f[f];
        const double sg = f == 2 ? mg : 0.0, st = f == 2 ? mt : 0.0;
        for (int i = blockIdx.x; i < rows; i += gridDim.x) {
            for (int j = threadIdx.x; j < cols; j += AT) {
                const size_t e = (size_t)i * g.P + j;
                // every load of the element before its stores: the window arrays may alias
                // G_k / R_k as far as the compiler knows, so loads after the stores would wait
                const double xv = X[e], tv = TT[e];
                double rv[NW];
#pragma unroll
                for (int w = 0; w < NW; ++w) rv[w] = (w < nw && w != self) ? rw[f][w][e] : 0.0;
                const double gv = xv - sg;
                const double r = gv - (tv - st);
                GG[e] = gv;
                RR[e] = r;
                if (unknown(g, f, i, j)) {
#pragma unroll
                    for (int w = 0; w < NW; ++w)
                        if (w < nw) acc[w] += r * (w == self ? r : rv[w]);
                }
            }
        }
    }
    const size_t b = blockIdx.x;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        if (w >= nw) break;
        const double v = block_sum_at(acc[w], sh);
        if (threadIdx.x == 0) partials[b * AA_MAXS + w] = v;
    }
}

// one thread: reduce the partials (fixed order) into Gram row `self`, solve, coefficients
__global__ void __launch_bounds__(AT) k_aa_solve(const double *__restrict__ partials, int nblocks, AAWin win,
                                                 double beta, double *H, double *cg, double *cr) {
    __shared__ double sh[32];
    // new row / column of the (slot-indexed) Gram matrix: the block partials of each entry
    // summed by the CTA in a fixed order (strided per thread, then the fixed shuffle tree)
    for (int w = 0; w < win.n; ++w) {
        double s = 0.0;
        for (int b = threadIdx.x; b < nblocks; b += AT) s += partials[(size_t)b * AA_MAXS + w];
        s = block_sum_at(s, sh);
        if (threadIdx.x == 0) {
            H[win.slot[win.self] * AA_MAXS + win.slot[w]] = s;
            H[win.slot[w] * AA_MAXS + win.slot[win.self]] = s;
        }
    }
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    __threadfence_block();
    const int nn = win.n;
    const int *order = win.slot;  // window oldest -> newest (the oracle's order)
    for (int s = 0; s < AA_MAXS; ++s) cg[s] = cr[s] = 0.0;
    if (nn < 2) {  // x^1 = G(x^0)
        cg[win.slot[win.self]] = 1.0;
        return;
    }
    double A[AA_MAXS][AA_MAXS + 1];
    double dmax = 0.0;
    for (int a = 0; a < nn; ++a) dmax = fmax(dmax, H[order[a] * AA_MAXS + order[a]]);
    const double lam = 1e-10 * dmax;
    for (int a = 0; a < nn; ++a) {
        for (int c = 0; c < nn; ++c) A[a][c] = H[order[a] * AA_MAXS + order[c]] + (a == c ? lam : 0.0);
        A[a][nn] = 1.0;
    }
    bool ok = true;
    for (int c = 0; c < nn && ok; ++c) {
        int piv = c;
        for (int r = c + 1; r < nn; ++r)
            if (fabs(A[r][c]) > fabs(A[piv][c])) piv = r;
        if (!(fabs(A[piv][c]) > 0.0)) {
            ok = false;
            break;
        }
        if (piv != c)
            for (int j = 0; j <= nn; ++j) {
                const double t = A[c][j];
                A[c][j] = A[piv][j];
                A[piv][j] = t;
            }
        for (int r = c + 1; r < nn; ++r) {
            const double f = A[r][c] / A[c][c];
            for (int j = c; j <= nn; ++j) A[r][j] -= f * A[c][j];
        }
    }
    double z[AA_MAXS], sz = 0.0;
    if (ok) {
        for (int i = nn - 1; i >= 0; --i) {
            double t = A[i][nn];
            for (int j = i + 1; j < nn; ++j) t -= A[i][j] * z[j];
            z[i] = t / A[i][i];
        }
        for (int i = 0; i < nn; ++i) sz += z[i];
        ok = fabs(sz) > 0.0;
    }
    if (!ok) {  // degenerate history: the plain step x^{k+1} = G(x^k)
        cg[win.slot[win.self]] = 1.0;
        return;
    }
    for (int a = 0; a < nn; ++a) {
        const double al = z[a] / sz;
        cg[order[a]] = al;
        cr[order[a]] = -(1.0 - beta) * al;
    }
}

__global__ void __launch_bounds__(AT) k_aa_update(GridL g, AAHist hist, int ns, const double *__restrict__ cg,
                                                  const double *__restrict__ cr, AAVec work, AAVec T,
                                                  double *__restrict__ partials) {
    __shared__ double sh[32];
    // the nonzero terms of x = sum c_k v_k as a compact list (coefficient, pointer per field):
    // no dynamic indexing of the parameter structs, no zero-coefficient branches in the loop
    __shared__ double cf[2 * AA_MAXS];
    __shared__ const double *vp[3][2 * AA_MAXS];
    __shared__ int nt;
    if (threadIdx.x == 0) {
        int k = 0;
        for (int q = 0; q < ns; ++q) {  // the order of the previous loop: G_q then R_q
            if (cg[q] != 0.0) {
                cf[k] = cg[q];
                for (int f = 0; f < 3; ++f) vp[f][k] = hist.G[q].f[f];
                ++k;
            }
            if (cr[q] != 0.0) {
                cf[k] = cr[q];
                for (int f = 0; f < 3; ++f) vp[f][k] = hist.R[q].f[f];
                ++k;
            }
        }
        nt = k;
    }
    __syncthreads();
    double psum = 0.0;
    const int rows = g.ncy + 2, cols = g.ncx + 2, nterm = nt;
#pragma unroll
    for (int f = 0; f < 3; ++f) {
        double *W = work.f[f], *TT = T.f[f];
        for (int i = blockIdx.x; i < rows; i += gridDim.x) {
            for (int j = threadIdx.x; j < cols; j += AT) {
                const size_t e = (size_t)i * g.P + j;
                double x = 0.0;
                for (int k = 0; k < nterm; ++k) x += cf[k] * vp[f][k][e];
                W[e] = x;
                TT[e] = x;
                if (f == 2 && unknown(g, 2, i, j)) psum += x;
            }
        }
    }
    psum = block_sum_at(psum, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = psum;
}

}  // namespace

int aa_blocks(const GridL &g) {
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const size_t b = (size_t)g.ncy + 2;  // one CTA per padded row, capped at 8 per SM (grid-stride)
    const size_t cap = (size_t)(nsm > 0 ? nsm : 148) * 8;
    return (int)(b < cap ? b : cap);
}
void launch_aa_push(const LaunchCtx &c, const GridL &g, const AAVec &work, const double *ms_g, const AAVec &T,
                    const double *ms_t, const AAVec &Gk, const AAVec &Rk, const AAWin &win, double *partials) {
    const int nb = aa_blocks(g);
    if (win.n <= 4) k_aa_push<4><<<nb, AT, 0, c.stream>>>(g, work, ms_g, T, ms_t, Gk, Rk, win, partials);
    else if (win.n <= 8) k_aa_push<8><<<nb, AT, 0, c.stream>>>(g, work, ms_g, T, ms_t, Gk, Rk, win, partials);
    else if (win.n <= 12) k_aa_push<12><<<nb, AT, 0, c.stream>>>(g, work, ms_g, T, ms_t, Gk, Rk, win, partials);
    else k_aa_push<AA_MAXS><<<nb, AT, 0, c.stream>>>(g, work, ms_g, T, ms_t, Gk, Rk, win, partials);
    ++*c.counter;
}
void launch_aa_solve(const LaunchCtx &c, const double *partials, int nblocks, const AAWin &win, double beta,
                     double *H, double *cg, double *cr) {
    k_aa_solve<<<1, AT, 0, c.stream>>>(partials, nblocks, win, beta, H, cg, cr);
    ++*c.counter;
}
void launch_aa_update(const LaunchCtx &c, const GridL &g, const AAHist &hist, int ns, const double *cg,
                      const double *cr, const AAVec &work, const AAVec &T, double *partials) {
    k_aa_update<<<aa_blocks(g), AT, 0, c.stream>>>(g, hist, ns, cg, cr, work, T, partials);
    ++*c.counter;
}
