// RAS-type temporally blocked Jacobi smoother: Alg. 3, PAPER.md:
// 1175-1210, reading R27.  One launch = one outer iteration: every CTA owns
// one tile of the shifted T x T tiling (T <= 32), stages the tile and a one-cell frame of
// all six input fields in shared memory, runs T_inner damped-Jacobi sweeps there with the
// frame frozen (the values of the outer iteration's input: the buffer is not written by
// this launch), and writes its unknowns -- and their wall mirrors -- to the OUTPUT buffer
// (single writer, out of place, so no "benign races").  The shift comes from the
// counter-based generator of R27, draw q = k * 65536 + c with k the solve's iteration
// index (device scalar, so CUDA-graph replays draw new shifts) and c the static index of
// the outer iteration within the V-cycle.  HBM traffic per outer iteration: the 64 B/cell
// of ONE Jacobi sweep (+ the frame, ~13 % at T = 32) for T_inner sweeps.
#include <math.h>

#include "internal.h"

namespace {

constexpr int RT = 256;        // threads per CTA
constexpr int RMAX = 32;       // tile edge limit
constexpr int RW2 = RMAX + 2;  // staged edge (tile + frame)
constexpr int RN = RW2 * RW2;

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// stencil view on the staged region: (i, j) are LEVEL indices, (i0 - 1, j0 - 1) is smem (0, 0)
struct RasView {
    const double *f[6];  // vx, vy, eta_p, eta_b, f4, f5 (vx / vy = the current sweep's input)
    int i0, j0;
    int r, c;  // node (level indices)
    __device__ __forceinline__ double at(int k, int i, int j) const { return f[k][(i - i0 + 1) * RW2 + (j - j0 + 1)]; }
    __device__ __forceinline__ double A(int k, int dc = 0) const { return at(k, r - 1, c + dc); }
    __device__ __forceinline__ double B(int k, int dc = 0) const { return at(k, r, c + dc); }
    __device__ __forceinline__ double C(int k, int dc = 0) const { return at(k, r + 1, c + dc); }
};

// the stencil rows of stream.cu (Listing vx_op_point, reading R2), on the view
__device__ __forceinline__ double lx_L(const GridL &g, const RasView &w, double &a) {
    const double eta1 = w.A(3), eta2 = w.B(3), etaA = w.B(2), etaB = w.B(2, 1);
    const double vc = w.B(0);
    a = -(eta1 + eta2) * g.idy2 - (etaA + etaB) * g.idx2x2;
    if (w.r == 1 && g.bN) a += g.sN * eta1 * g.idy2;
    if (w.r == g.ncy && g.bS) a += g.sS * eta2 * g.idy2;
    return g.idx2x2 * (etaA * (w.B(0, -1) - vc) + etaB * (w.B(0, 1) - vc)) +
           g.idy2 * (eta1 * (w.A(0) - vc) + eta2 * (w.C(0) - vc)) +
           g.idxdy * (eta1 * (w.A(1) - w.A(1, 1)) + eta2 * (w.B(1, 1) - w.B(1)));
}
__device__ __forceinline__ double ly_L(const GridL &g, const RasView &w, double &a) {
    const double etaN = w.B(2), etaS = w.C(2), etaW = w.B(3, -1), etaE = w.B(3);
    const double vc = w.B(1);
    a = -(etaN + etaS) * g.idy2x2 - (etaW + etaE) * g.idx2;
    if (w.c == 1 && g.bW) a += g.sW * etaW * g.idx2;
    if (w.c == g.ncx && g.bE) a += g.sE * etaE * g.idx2;
    return g.idy2x2 * (etaS * (w.C(1) - vc) + etaN * (w.A(1) - vc)) +
           g.idx2 * (etaE * (w.B(1, 1) - vc) + etaW * (w.B(1, -1) - vc)) +
           g.idxdy * (etaE * (w.C(0) - w.B(0)) - etaW * (w.C(0, -1) - w.B(0, -1)));
}

template <int MODE>
__global__ void __launch_bounds__(RT) k_ras(GridL g, RasArgs a, const double *__restrict__ iter, int c_draw) {
    extern __shared__ __align__(16) double sm[];
    // smem: vx[2], vy[2] (ping-pong), eta_p, eta_b, f4, f5
    // (ping-pong by offset arithmetic on `sm`, no pointer arrays: keeps the accesses LDS/STS)
    double *sep = sm + 4 * RN, *seb = sm + 5 * RN, *s4 = sm + 6 * RN, *s5 = sm + 7 * RN;
    const int T = a.T;
    const uint64_t q = (uint64_t)(long long)iter[0] * 65536ull + (uint64_t)c_draw;
    const uint64_t u = splitmix64(a.seed ^ (q * 0x9E3779B97F4A7C15ull));
    const int si = (int)((u & 0xffffffffull) % (uint64_t)T), sj = (int)((u >> 32) % (uint64_t)T);
    const int ti = blockIdx.y, tj = blockIdx.x;
    const int i0 = max(1, ti * T - si + 1), i1 = min(g.ncy, (ti + 1) * T - si);
    const int j0 = max(1, tj * T - sj + 1), j1 = min(g.ncx, (tj + 1) * T - sj);
    if (i0 > i1 || j0 > j1) return;
    const int ni = i1 - i0 + 3, nj = j1 - j0 + 3;  // staged rows / columns (with the frame)
    const size_t P = g.P;
    // staging: U elements x 6 fields of independent loads in flight per thread (memory-level
    // parallelism: one CTA holds only 8 warps)
    constexpr int U = 5;
    const int ne = ni * nj;
    for (int e0 = threadIdx.x; e0 < ne; e0 += RT * U) {
        double v[U][6];
        int sidx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * RT;
            sidx[u] = -1;
            if (e < ne) {
                const int ii = e / nj, jj = e - (e / nj) * nj;
                const size_t gi = (size_t)(i0 - 1 + ii) * P + (j0 - 1 + jj);
                sidx[u] = ii * RW2 + jj;
                v[u][0] = __ldg(a.vx + gi);
                v[u][1] = __ldg(a.vy + gi);
                v[u][2] = __ldg(a.etap + gi);
                v[u][3] = __ldg(a.etab + gi);
                v[u][4] = __ldg(a.f4 + gi);
                v[u][5] = __ldg(a.f5 + gi);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int s = sidx[u];
            if (s < 0) continue;
            sm[s] = v[u][0];
            sm[RN + s] = v[u][0];
            sm[2 * RN + s] = v[u][1];
            sm[3 * RN + s] = v[u][1];
            sep[s] = v[u][2];
            seb[s] = v[u][3];
            s4[s] = v[u][4];
            s5[s] = v[u][5];
        }
    }
    __syncthreads();
    const int xj1 = min(j1, g.nvxj), yi1 = min(i1, g.nvyi);
    const int tw = j1 - j0 + 1, th = i1 - i0 + 1;
    // this thread's cells (fixed for the whole launch): smem index, and -- constant over the
    // inner sweeps -- the right-hand side b and 1/a_ii of its vx and vy unknowns
    constexpr int CPT = (RMAX * RMAX + RT - 1) / RT;
    int cs[CPT];
    double bxv[CPT], byv[CPT], iax[CPT], iay[CPT];
    unsigned ux = 0, uy = 0;  // bit c: cell c carries a vx / vy unknown
    RasView w;
    w.f[2] = sep;
    w.f[3] = seb;
    w.f[4] = s4;
    w.f[5] = s5;
    w.i0 = i0;
    w.j0 = j0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int e = threadIdx.x + k * RT;
        cs[k] = 0;
        bxv[k] = byv[k] = iax[k] = iay[k] = 0.0;
        if (e >= tw * th) continue;
        const int i = i0 + e / tw, j = j0 + e % tw;
        cs[k] = (i - i0 + 1) * RW2 + (j - j0 + 1);
        w.f[0] = sm;
        w.f[1] = sm + 2 * RN;
        w.r = i;
        w.c = j;
        if (j <= xj1) {
            ux |= 1u << k;
            double ad;
            lx_L(g, w, ad);
            iax[k] = 1.0 / ad;
            bxv[k] = (MODE == RHS_FINE) ? (a.gx != 0.0 ? -a.gx * (0.5 * (w.A(5) + w.B(5))) : 0.0) -
                                              (w.B(4) - w.B(4, 1)) * g.idx
                                        : w.B(4);
        }
        if (i <= yi1) {
            uy |= 1u << k;
            double ad;
            ly_L(g, w, ad);
            iay[k] = 1.0 / ad;
            byv[k] = (MODE == RHS_FINE) ? (a.gy != 0.0 ? -a.gy * (0.5 * (w.B(5, -1) + w.B(5))) : 0.0) -
                                              (w.B(4) - w.C(4)) * g.idy
                                        : w.B(5);
        }
    }
    const double ix2 = g.idx2x2, iy2 = g.idy2, ixy = g.idxdy, yy2 = g.idy2x2, xx2 = g.idx2;
    int cur = 0;
    for (int tau = 0; tau < a.Tin; ++tau) {
        const double *X = sm + cur * RN, *Y = sm + (2 + cur) * RN;
        double *NX = sm + (cur ^ 1) * RN, *NY = sm + (2 + (cur ^ 1)) * RN;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int q = cs[k];
            if (ux & (1u << k)) {  // vx row in stress-difference form (= lx_L)
                const double eta1 = seb[q - RW2], eta2 = seb[q], etaA = sep[q], etaB = sep[q + 1];
                const double vc = X[q];
                const double L = ix2 * (etaA * (X[q - 1] - vc) + etaB * (X[q + 1] - vc)) +
                                 iy2 * (eta1 * (X[q - RW2] - vc) + eta2 * (X[q + RW2] - vc)) +
                                 ixy * (eta1 * (Y[q - RW2] - Y[q - RW2 + 1]) + eta2 * (Y[q + 1] - Y[q]));
                const double vn = vc + a.omega * (bxv[k] - L) * iax[k];
                NX[q] = vn;
                if (g.bN && q < 2 * RW2 && i0 == 1) NX[q - RW2] = g.sN * vn;  // the tile's own mirror
                if (g.bS && i1 == g.ncy && q >= (th)*RW2 && q < (th + 1) * RW2) NX[q + RW2] = g.sS * vn;
            }
            if (uy & (1u << k)) {  // vy row (= ly_L)
                const double etaN = sep[q], etaS = sep[q + RW2], etaW = seb[q - 1], etaE = seb[q];
                const double vc = Y[q];
                const double L = yy2 * (etaS * (Y[q + RW2] - vc) + etaN * (Y[q - RW2] - vc)) +
                                 xx2 * (etaE * (Y[q + 1] - vc) + etaW * (Y[q - 1] - vc)) +
                                 ixy * (etaE * (X[q + RW2] - X[q]) - etaW * (X[q + RW2 - 1] - X[q - 1]));
                const double vn = vc + a.omega * (byv[k] - L) * iay[k];
                NY[q] = vn;
                const int jj = q % RW2;
                if (g.bW && j0 == 1 && jj == 1) NY[q - 1] = g.sW * vn;
                if (g.bE && j1 == g.ncx && jj == tw) NY[q + 1] = g.sE * vn;
            }
        }
        __syncthreads();
        cur ^= 1;
    }
    // single writer: the tile's unknowns and their wall mirrors to the output buffer
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int e = threadIdx.x + k * RT;
        if (e >= tw * th) continue;
        const int i = i0 + e / tw, j = j0 + e % tw;
        const int q = cs[k];
        const size_t gi = (size_t)i * P + j;
        if (ux & (1u << k)) {
            const double v = sm[cur * RN + q];
            a.vxo[gi] = v;
            if (i == 1 && g.bN) a.vxo[j] = g.sN * v;
            if (i == g.ncy && g.bS) a.vxo[(size_t)(g.ncy + 1) * P + j] = g.sS * v;
        }
        if (uy & (1u << k)) {
            const double v = sm[(2 + cur) * RN + q];
            a.vyo[gi] = v;
            if (j == 1 && g.bW) a.vyo[(size_t)i * P] = g.sW * v;
            if (j == g.ncx && g.bE) a.vyo[(size_t)i * P + g.ncx + 1] = g.sE * v;
        }
    }
}

__global__ void k_iter_inc(double *k) { k[0] += 1.0; }

}  // namespace

void launch_ras_outer(const LaunchCtx &c, const GridL &g, const RasArgs &a, const double *iter, int c_draw,
                      bool fine) {
    const int T = a.T;
    const dim3 grid((g.ncx + T - 1) / T + 1, (g.ncy + T - 1) / T + 1);  // any shift in [0, T)
    const int smem = 8 * RN * (int)sizeof(double);
    static unsigned long long done = 0;
    if (first_on_device(&done)) {
        cudaFuncSetAttribute(k_ras<RHS_FINE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_ras<RHS_ARRAYS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    }
    if (fine) k_ras<RHS_FINE><<<grid, RT, smem, c.stream>>>(g, a, iter, c_draw);
    else k_ras<RHS_ARRAYS><<<grid, RT, smem, c.stream>>>(g, a, iter, c_draw);
    ++*c.counter;
}
void launch_iter_inc(const LaunchCtx &c, double *k) {
    k_iter_inc<<<1, 1, 0, c.stream>>>(k);
    ++*c.counter;
}
int ras_max_tile() { return RMAX; }
