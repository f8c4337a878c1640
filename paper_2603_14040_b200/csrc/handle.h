// Handle structure and host-runtime helpers shared by driver.cu (single domain) and
// dist.cu (2D domain decomposition).  Internal; not part of the ABI.
#pragma once
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "internal.h"

#define MAXLEV 24
#define MAXM 32
#define MAX_DIRECT 1024  // largest coarsest system solved by the explicit inverse (a8)

namespace sk {

extern thread_local std::string g_last_error;

// device scalar slots
enum { S_MSHIFT = 0, S_E = 1, S_SV = 2, S_SP = 3, S_SF = 4, S_SFPART = 5, S_ZMEAN = 8, S_GAMMA = 9, S_NU2 = 10, S_LOC = 16,
       S_RR = 11, S_BETA = 12, S_ZERO = 13, S_E0 = 14, S_ETAMIN = 24, S_AAMT = 25, S_ITER = 26,
       S_LOOP = 40,  // device-side Uzawa loop: [0] rtol [1] E0 [2] max_iter [3] k [4] status [5] E
       S_GAMS = 64,  // GCR: the MGS coefficients gamma_j of the current step (MAXM slots)
       S_NSCAL = 128 };
constexpr int LOOP_HCAP = 16384;  // device history of E (stokes_solve_hist) in device-loop solves

struct Level {
    GridL g;
    double *etab, *etap;
    double *vx[2], *vy[2];  // level 0: solution ping-pong; coarse: correction ping-pong
    double *bx, *by;        // right-hand side
    double *rx, *ry;        // residual scratch
    int nu;
};

}  // namespace sk

struct stokes_s {
    int device;  // the CUDA device the handle was created on (every ABI call runs there)
    int nx, ny;
    double Lx, Ly;
    int bc[4];
    stokes_opts o;
    cudaStream_t stream;
    bool own_stream;
    void *ws;
    size_t ws_bytes;
    bool own_ws;
    int nlev;
    sk::Level lev[MAXLEV];
    double *pbuf[2], *rho;  // pressure ping-pong (the fused Uzawa pass reads one, writes the other)
    double *etab_user, *etap_user;  // the caller's fine viscosities (theta_step > 0: rescaling)
    AAHist aah;                     // Anderson history slots (accel = ANDERSON)
    AAVec aat;                      // Anderson: x^k (de-meaned pressure at mean S_AAMT)
    double *aaH, *aacg, *aacr;      // Gram matrix (slot-indexed), mixing coefficients
    int ras_c;                      // RAS draw index within the current V-cycle (reading R27)
    int pcur;
    double *partials;
    size_t npart;
    double *scal;       // device scalars
    double *hscal;      // pinned host mirror
    double *Minv, *Mwork;
    int nc;
    int *dflag;
    // GCR vectors (fine level, padded): z_i, w_i, r, V-cycle scratch
    double *gz[MAXM][3], *gw[MAXM][3], *gr[3], *gtmp[2], *gew[3];
    cudaGraphExec_t gcr_exec[MAXM];  // GCR step i (i MGS steps) captured
    long long gcr_kernels[MAXM];
    bool have_eta, have_rho;
    double gx, gy;
    long long launches;
    cudaGraphExec_t uzawa_exec[2];  // iteration reading pbuf[k]
    cudaGraphExec_t fused_exec[4];  // fused-tail iteration reading pbuf[k & 1], first sweep in buffer k >> 1 (a12 fusion)
    int fused_nq[4];                // buffer of the next first sweep after graph k
    cudaGraphExec_t loop_exec[4];   // device-side Uzawa loop entered in state (q, pcur) = (k >> 1, k & 1)
    double *dhist;                  // device E history of the device loop (LOOP_HCAP doubles)
    bool loop_off;                  // device loop unavailable (capture / instantiate failed): host loop
    long long fused_kernels;
    long long uzawa_kernels;
    void *mk_ws;        // marker-in-cell scratch (markers.cu), grown on demand
    size_t mk_bytes;
    struct Dist *dist;  // non-null: a 2D-decomposed handle (all calls dispatch to dist_*)
    double *hist;       // stokes_solve_hist: host buffer of E after every iteration (or null)
    int hist_len, hist_off;
};


namespace sk {
using ::stokes_s;
// Every ABI entry point runs on the handle's device and restores the caller's current device.
struct DevGuard {
    int prev = -1, want;
    explicit DevGuard(int d) : want(d) {
        if (d >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != d) cudaSetDevice(d);
    }
    ~DevGuard() {
        if (want >= 0 && prev >= 0 && prev != want) cudaSetDevice(prev);
    }
};

int fail_cuda(cudaError_t e, const char *what);
size_t round_up(size_t v, size_t a);
GridL make_grid(int ncx, int ncy, double Lx, double Ly, const int bc[4]);
size_t field_doubles(const GridL &g);
int n_unknowns(const GridL &g);
int build_levels(int nx, int ny, double Lx, double Ly, const int bc[4], const stokes_opts &o, GridL *gs, int *nus);
struct Carver {  // bump allocator over the workspace (256-B granules)
    char *base;
    size_t off, cap;
    bool dry;
    double *take(size_t ndoubles) {
        off = round_up(off, 256);
        double *p = dry ? nullptr : (double *)(base + off);
        off += ndoubles * sizeof(double);
        return p;
    }
    double *field(const GridL &g) {  // row -1 .. ncy+2 + tail; returns &(0, 0)
        double *a = take(field_doubles(g) + g.P);
        return dry ? nullptr : a + g.P + COL_OFF;
    }
};
int check_opts(const stokes_opts &o);
size_t carve(stokes_s *h, Carver &cv);
LaunchCtx ctx(stokes_s *h);
RhsArgs rhs_arrays(const double *bx, const double *by);
RhsArgs rhs_fine(stokes_s *h);
void smooth(stokes_s *h, int l, double *&cx, double *&cy, double *&ox, double *&oy, const RhsArgs &rhs, int n,
            bool zero_in, int max_pairs = 0);
int jacobi_pairs(stokes_s *h, int l, int n, bool zero_in);
int level_smoother(const stokes_s *h, int l);
bool uses_ras(const stokes_s *h);
void ras_iteration_start(stokes_s *h);  // before the V-cycle(s) of one iteration
void ras_reset(stokes_s *h);            // iteration index 0
void ras_iteration_end(stokes_s *h);    // after them (advances the device iteration index)
// leave_last (level l only): the post-smoothing stops one sweep early (the fused k_jju pass
// does the last one); no final copy, *lx / *ly = the buffer holding that iterate
void vcycle(stokes_s *h, int l, double *ax, double *ay, double *sx, double *sy, const RhsArgs &rhs, bool zero_in,
            int done_pre = 0, int leave_last = 0, double **lx = nullptr, double **ly = nullptr);
int sync(stokes_s *h);
inline void record_E(stokes_s *h, int k, double E) {  // E after iteration k + 1 of the current solve stage
    const int q = h->hist_off + k;
    if (h->hist && q >= 0 && q < h->hist_len) h->hist[q] = E;
}
int build_hierarchy(stokes_s *h);
int solve_inner(stokes_s *h, double rtol, double E0, int *iters, double *E);
int solve_anderson(stokes_s *h, double rtol, double E0, int *iters, double *E);
int solve_staged(stokes_s *h, double rtol, int *iters, double *E);
void drop_graphs(stokes_s *h);
void force_energy(stokes_s *h);
}  // namespace sk

#define DEVICE_GUARD(h) sk::DevGuard dev_guard_((h) ? (h)->device : -1)
// NVTX ranges (header-only NVTX3: free unless a profiler is attached) around the ABI calls
// and the solve phases, so nsys / ncu timelines show where a solve spends its time
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
#define NVTX_RANGE(name) NvtxRange nvtx_range_(name)
#define CK(call)                                                  \
    do {                                                          \
        cudaError_t e_ = (call);                                  \
        if (e_ != cudaSuccess) return sk::fail_cuda(e_, #call);   \
    } while (0)
#define CKL()                                                               \
    do {                                                                    \
        cudaError_t e_ = cudaGetLastError();                                \
        if (e_ != cudaSuccess) return sk::fail_cuda(e_, "kernel launch");   \
    } while (0)

// ---- 2D decomposition (dist.cu): dispatch targets of the ABI for decomposed handles
int dist_destroy(struct Dist *D);
int dist_set_viscosity(struct Dist *D, const double *eta_b, const double *eta_p);
int dist_set_density(struct Dist *D, const double *rho_b);
int dist_set_gravity(struct Dist *D, double gx, double gy);
int dist_residual_energy(struct Dist *D, const double *vx, const double *vy, const double *p, double *E);
int dist_solve(struct Dist *D, double rtol, double *vx, double *vy, double *p, int *iters, double *E);
int dist_num_levels(struct Dist *D);
long long dist_launches(struct Dist *D, int reset);
