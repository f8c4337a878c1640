// 2D domain decomposition of the multigrid Stokes solve.
//
// The global nx x ny grid is split into px x py tiles of (nx/px) x (ny/py) cells, the
// paper's Cartesian decomposition (interior + 1-cell halo, boundary
// ranks' halos repurposed as boundary nodes).  It is EXACT: every
// stencil of a tile reads the same values the single-domain solve reads (halos refreshed
// after every write of a velocity / residual / correction / pressure field), so the
// iterates equal the single-GPU ones up to the order of the global sums.
//
//   distributed levels 0..La-1  each tile runs the same kernels with per-side global-
//                               boundary flags (GridL.bN/bS/bW/bE, mirrors and walls only on
//                               global sides); two-phase halo exchange (W/E columns over all
//                               rows, then N/S rows over all columns: corners included)
//   agglomeration level La      the tiles' restricted residuals are gathered into the GLOBAL
//                               level-La grid, held by every process (the B200 analogue of the
//                               paper's CPU-side coarse levels); the coarse
//                               tail of the V-cycle runs there redundantly and every tile takes
//                               its window of the correction (no scatter message)
//   global sums                 (Sv, Sp, sum p) per tile -> fixed-order combine / ncclAllReduce
//
// Transports: VIRTUAL (rank < 0): all tiles in this process on one GPU, halos copied by
// strip-copy kernels -- the exactness test of the decomposition on one B200.  NCCL (rank >=
// 0): one tile per process/GPU, ncclSend/ncclRecv of packed halo columns and contiguous rows
// over NVLink, ncclAllGather for the agglomeration, ncclAllReduce for the sums; all
// graph-capturable.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <nccl.h>

#include "handle.h"

using namespace sk;

#define MAXT 64

struct Dist {
    int NX, NY, px, py, nxt, nyt;
    double Lx, Ly;
    int bc[4];
    stokes_opts o;
    int rank;  // -1 virtual, -2 loopback (packed transport in one process), >= 0 NCCL
    int mode;  // M_VIRTUAL, M_LOOPBACK, M_NCCL
    int nt;
    stokes_s *tile[MAXT];
    int tx[MAXT], ty[MAXT];
    int La;          // distributed levels
    int L;           // total levels (global hierarchy)
    stokes_s *tail;  // global level La and below
    cudaStream_t stream;
    bool own_stream;
    cudaStream_t cstream;  // halo exchanges overlapped with the interior part of a pass
    cudaStream_t xs;       // the stream exchange() enqueues on (stream, or cstream while overlapping)
    cudaEvent_t ev[2];
    bool overlap;
    int overlap_min;    // split / overlap only levels whose tile is >= this many cells wide
    bool serial_split;  // diagnostics (STOKES_DIST_OVERLAP=2): split passes, exchange not overlapped
    double *dscal;   // [0] E [1] Sv [2] Sp [3] Sf [4] zero
    double *hsc;
    ncclComm_t comm;
    double *sb[MAXT], *rb[MAXT];  // per local tile: packed halo columns / agglomeration blocks
    size_t nbuf;
    long long launches;
    cudaGraphExec_t exec[2];
    long long body_kernels;
    // GCR(m) on the tiles: partial-sum buffers holding every tile's per-CTA
    // partials back to back (NCCL: all-gathered), so each tile's next fused kernel reduces
    // the GLOBAL sum in one fixed order; one graph per inner step i
    double *gpart[3];
    size_t gseg;  // doubles per tile segment
    // Anderson AA(m, beta) on the tiles: the same scheme for the Gram row and the pressure mean
    double *apart[2];
    cudaGraphExec_t aexec[2];  // the plain (unfused) Uzawa iteration G(x) per pressure parity
    long long akernels;
    cudaGraphExec_t gexec[MAXM];
    long long gkernels[MAXM];
    int pcur;
    bool have_eta, have_rho;
    double gx, gy;
    // schedule-recording dry run of the NCCL transport (rank >= 0, no unique id): the NCCL
    // calls are recorded here (NC_REC long longs per call) instead of issued
    bool halo2;  // packed transports: the two-round halo exchange (STOKES_HALO_2PHASE=1) instead of one round
    bool dry;
    long long *nlog;
    int nlog_n, nlog_cap;
};

int dist_eta_hierarchy(Dist *D);

namespace {

enum { FX_V = 0, FX_R = 1, FX_P = 2, FX_ETA = 3, FX_RHO = 4, FX_B = 5, FX_VP = 6, FX_GR = 7 };
enum { M_VIRTUAL = 0, M_LOOPBACK = 1, M_NCCL = 2, M_NCCL_SELF = 3 };
constexpr int HW = 2;  // halo width: the two-sweep pass and the fused residual+restriction read two rings

LaunchCtx dctx(Dist &D) { return LaunchCtx{D.xs, &D.launches}; }
bool packed(const Dist &D) { return D.mode != M_VIRTUAL; }
bool self_nccl(const Dist &D) { return D.mode == M_NCCL_SELF; }

// ---- the NCCL calls of the multi-process transport (M_NCCL).  In the dry run (stokes_create_dist
// with rank >= 0 and no unique id: no communicator) each call is RECORDED -- (op, peer, count,
// datatype, reduction) -- instead of issued, and the collectives keep their local part, so
// every rank's schedule can be built in one process on one GPU, one rank after another (no
// kernel ever waits on another rank), and checked against NCCL's matching rules
// (tests/test_gpu_nccl_schedule.py; stokes_dist_schedule).
constexpr int NC_REC = 5;
enum { NC_GSTART = 1, NC_GEND = 2, NC_SEND = 3, NC_RECV = 4, NC_ALLGATHER = 5, NC_ALLREDUCE = 6, NC_BODY = 7,
       NC_BODY_END = 8 };  // (7 / 8: begin / end of the capture of one Uzawa iteration's graph)
int nc_log(Dist &D, int op, int peer, size_t count, int dtype, int redop) {
    if (D.nlog_n == D.nlog_cap) {
        const int cap = D.nlog_cap ? 2 * D.nlog_cap : 1024;
        long long *p = (long long *)realloc(D.nlog, (size_t)cap * NC_REC * sizeof(long long));
        if (!p) return STOKES_ENOMEM;
        D.nlog = p;
        D.nlog_cap = cap;
    }
    long long *r = D.nlog + (size_t)D.nlog_n++ * NC_REC;
    r[0] = op;
    r[1] = peer;
    r[2] = (long long)count;
    r[3] = dtype;
    r[4] = redop;
    return STOKES_OK;
}
// ncclSend of n doubles to `peer` and ncclRecv of n doubles from it (inside a group).  Dry run:
// both recorded, and the receive buffer gets what this rank sends (valid values, e.g. positive
// viscosities in the halos, instead of uninitialised memory)
int nc_sendrecv(Dist &D, const double *sbuf, double *rbuf, size_t n, int peer, cudaStream_t s) {
    if (D.dry) {
        CK(cudaMemcpyAsync(rbuf, sbuf, n * 8, cudaMemcpyDeviceToDevice, s));
        int st = nc_log(D, NC_SEND, peer, n, (int)ncclDouble, -1);
        return st ? st : nc_log(D, NC_RECV, peer, n, (int)ncclDouble, -1);
    }
    if (ncclSend(sbuf, n, ncclDouble, peer, D.comm, s) != ncclSuccess) return STOKES_ENCCL;
    return ncclRecv(rbuf, n, ncclDouble, peer, D.comm, s) == ncclSuccess ? STOKES_OK : STOKES_ENCCL;
}
// all-gather of n doubles per rank (in place when send == recv + rank * n).  Dry run: every
// rank's slot gets this rank's block (valid values -- e.g. positive viscosities for the
// agglomerated tail's checks -- not the other ranks' data)
int nc_allgather(Dist &D, const double *send, double *recv, size_t n, cudaStream_t s) {
    if (D.dry) {
        for (int r = 0; r < D.px * D.py; ++r)
            if (send != recv + (size_t)r * n)
                CK(cudaMemcpyAsync(recv + (size_t)r * n, send, n * 8, cudaMemcpyDeviceToDevice, s));
        return nc_log(D, NC_ALLGATHER, -1, n, (int)ncclDouble, -1);
    }
    return ncclAllGather(send, recv, n, ncclDouble, D.comm, s) == ncclSuccess ? STOKES_OK : STOKES_ENCCL;
}
int nc_allreduce(Dist &D, void *buf, size_t n, ncclDataType_t t, ncclRedOp_t op, cudaStream_t s) {  // in place
    if (D.dry) return nc_log(D, NC_ALLREDUCE, -1, n, (int)t, (int)op);
    return ncclAllReduce(buf, buf, n, t, op, D.comm, s) == ncclSuccess ? STOKES_OK : STOKES_ENCCL;
}

// the fields of a halo exchange: FX_VP = velocity buffer idx and pressure buffer pidx
int nfields(Dist &D, stokes_s *h, int l, int which, int idx, double **f) {
    Level &L = h->lev[l];
    switch (which) {
    case FX_V: f[0] = L.vx[idx]; f[1] = L.vy[idx]; return 2;
    case FX_VP: f[0] = L.vx[idx & 1]; f[1] = L.vy[idx & 1]; f[2] = h->pbuf[idx >> 1]; return 3;
    case FX_R: f[0] = L.rx; f[1] = L.ry; return 2;
    case FX_B: f[0] = L.bx; f[1] = L.by; return 2;
    case FX_P: f[0] = h->pbuf[idx]; return 1;
    case FX_ETA: f[0] = L.etab; f[1] = L.etap; return 2;
    case FX_GR: f[0] = h->gr[0]; f[1] = h->gr[1]; f[2] = h->gr[2]; return 3;  // GCR residual (level 0)
    default: (void)D; f[0] = h->rho; return 1;
    }
}
int tile_at(Dist &D, int tx, int ty) { return D.mode != M_NCCL ? ty * D.px + tx : -1; }

void add_strip(StripList &s, double *dst, const double *src, int n, int ds, int ss) {
    s.dst[s.count] = dst;
    s.src[s.count] = src;
    s.n[s.count] = n;
    s.dstride[s.count] = ds;
    s.sstride[s.count] = ss;
    ++s.count;
}
// a whole field incl. its row -1 (copies / clears that must not leave a stale second ring)
double *fstart(const GridL &g, double *p) { return p - COL_OFF - g.P; }
size_t fsize(const GridL &g) { return field_doubles(g) + g.P; }

// point-to-point transfer of n doubles between local buffers: device copy (LOOPBACK) or a
// real ncclSend / ncclRecv pair on the one-rank communicator (NCCL_SELF; caller groups)
int p2p_local(Dist &D, double *dst, const double *src, size_t n) {
    if (self_nccl(D)) {
        if (ncclSend(src, n, ncclDouble, 0, D.comm, D.xs) != ncclSuccess) return STOKES_ENCCL;
        if (ncclRecv(dst, n, ncclDouble, 0, D.comm, D.xs) != ncclSuccess) return STOKES_ENCCL;
        return STOKES_OK;
    }
    CK(cudaMemcpyAsync(dst, src, n * 8, cudaMemcpyDeviceToDevice, D.xs));
    return STOKES_OK;
}
int group_start(Dist &D) {
    if (D.dry) return nc_log(D, NC_GSTART, -1, 0, -1, -1);
    if (D.mode == M_NCCL || self_nccl(D)) return ncclGroupStart() == ncclSuccess ? STOKES_OK : STOKES_ENCCL;
    return STOKES_OK;
}
int group_end(Dist &D) {
    if (D.dry) return nc_log(D, NC_GEND, -1, 0, -1, -1);
    if (D.mode == M_NCCL || self_nccl(D)) return ncclGroupEnd() == ncclSuccess ? STOKES_OK : STOKES_ENCCL;
    return STOKES_OK;
}

// ---- one-round packed halo exchange (default for the packed transports).  Every neighbour
// of a tile -- the four sides, and the four diagonal tiles where both adjacent sides are
// tiles -- receives its strips in ONE grouped round (the two-round scheme below sends the W/E
// columns first and the N/S rows, corners included, second: two NCCL latencies per exchange).
// Direction (dx, dy): the block this tile sends spans
//   rows  dy < 0: 1 .. HW,  dy > 0: ncy-HW+1 .. ncy,  dy = 0: r_lo .. r_hi
//   cols  dx < 0: 1 .. HW,  dx > 0: ncx-HW+1 .. ncx,  dx = 0: c_lo .. c_hi
// and the block it receives from there spans rows 1-HW .. 0 / ncy+1 .. ncy+HW / r_lo .. r_hi
// and the same for columns, where [r_lo, r_hi] = the tile's rows plus the HW halo rows on a
// GLOBAL N / S side (mirror rows, held alike by the side neighbour), [c_lo, c_hi] likewise:
// every halo cell is written by exactly one message and the corners come straight from the
// diagonal tile's own cells.  A block is packed as strips along its long dimension (per
// field: one strip per column for dy = 0, one per row otherwise), in ascending order on both
// sides, so the sender's and the receiver's packings agree element by element.
struct HaloDir {
    int dx, dy;
};
constexpr HaloDir HDIR[8] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}, {-1, -1}, {1, -1}, {-1, 1}, {1, 1}};
int opposite(int d) {
    for (int e = 0; e < 8; ++e)
        if (HDIR[e].dx == -HDIR[d].dx && HDIR[e].dy == -HDIR[d].dy) return e;
    return -1;
}
bool has_nb(const Dist &D, int tx, int ty, int d) {
    const int x = tx + HDIR[d].dx, y = ty + HDIR[d].dy;
    return x >= 0 && x < D.px && y >= 0 && y < D.py;
}
// rows [*a, *b] of the block sent (recv = false) to / received (recv = true) from direction d
void dir_rows(const Dist &D, const GridL &g, int ty, int d, bool recv, int *a, int *b) {
    const int dy = HDIR[d].dy;
    if (dy < 0) { *a = recv ? 1 - HW : 1; *b = recv ? 0 : HW; }
    else if (dy > 0) { *a = recv ? g.ncy + 1 : g.ncy - HW + 1; *b = recv ? g.ncy + HW : g.ncy; }
    else { *a = ty > 0 ? 1 : 1 - HW; *b = ty + 1 < D.py ? g.ncy : g.ncy + HW; }
}
void dir_cols(const Dist &D, const GridL &g, int tx, int d, bool recv, int *a, int *b) {
    const int dx = HDIR[d].dx;
    if (dx < 0) { *a = recv ? 1 - HW : 1; *b = recv ? 0 : HW; }
    else if (dx > 0) { *a = recv ? g.ncx + 1 : g.ncx - HW + 1; *b = recv ? g.ncx + HW : g.ncx; }
    else { *a = tx > 0 ? 1 : 1 - HW; *b = tx + 1 < D.px ? g.ncx : g.ncx + HW; }
}
// segment offsets / lengths (doubles) of the 8 directions in a tile's send (= receive) buffer
void seg_layout(const Dist &D, const GridL &g, int tx, int ty, int nf, size_t *off, size_t *len) {
    size_t o = 0;
    for (int d = 0; d < 8; ++d) {
        int r0, r1, c0, c1;
        dir_rows(D, g, ty, d, false, &r0, &r1);
        dir_cols(D, g, tx, d, false, &c0, &c1);
        off[d] = o;
        len[d] = has_nb(D, tx, ty, d) ? (size_t)nf * (r1 - r0 + 1) * (c1 - c0 + 1) : 0;
        o += len[d];
    }
}
// the strips that pack (recv = false: field -> buffer) or unpack (recv = true: buffer ->
// field) direction d of one tile
void dir_strips(const Dist &D, const GridL &g, int tx, int ty, int d, bool recv, double *const *f, int nf,
                double *buf, StripList &s) {
    int r0, r1, c0, c1;
    dir_rows(D, g, ty, d, recv, &r0, &r1);
    dir_cols(D, g, tx, d, recv, &c0, &c1);
    const int nr = r1 - r0 + 1, nc = c1 - c0 + 1;
    const bool by_col = HDIR[d].dy == 0;  // long dimension: rows (W / E blocks)
    size_t e = 0;
    for (int q = 0; q < nf; ++q) {
        if (by_col) {
            for (int j = c0; j <= c1; ++j, e += nr) {
                if (recv) add_strip(s, f[q] + at(g, r0, j), buf + e, nr, g.P, 1);
                else add_strip(s, buf + e, f[q] + at(g, r0, j), nr, 1, g.P);
            }
        } else {
            for (int i = r0; i <= r1; ++i, e += nc) {
                if (recv) add_strip(s, f[q] + at(g, i, c0), buf + e, nc, 1, 1);
                else add_strip(s, buf + e, f[q] + at(g, i, c0), nc, 1, 1);
            }
        }
    }
}
int exchange_one_round(Dist &D, int l, int which, int idx) {
    const LaunchCtx c = dctx(D);
    double *f[3];
    size_t off[MAXT][8], len[MAXT][8];
    StripList s;
    s.count = 0;
    for (int k = 0; k < D.nt; ++k) {  // pack every direction of every local tile
        const GridL &g = D.tile[k]->lev[l].g;
        const int nf = nfields(D, D.tile[k], l, which, idx, f);
        seg_layout(D, g, D.tx[k], D.ty[k], nf, off[k], len[k]);
        if (off[k][7] + len[k][7] > D.nbuf) return fail_cuda(cudaErrorInvalidValue, "halo buffer too small");
        for (int d = 0; d < 8; ++d)
            if (len[k][d]) {
                if (s.count + 3 * HW > 512) { launch_strips(c, s); s.count = 0; }
                dir_strips(D, g, D.tx[k], D.ty[k], d, false, f, nf, D.sb[k] + off[k][d], s);
            }
    }
    if (s.count) launch_strips(c, s);
    int st = group_start(D);
    if (st) return st;
    for (int k = 0; k < D.nt; ++k)
        for (int d = 0; d < 8; ++d) {
            if (!len[k][d]) continue;
            if (D.mode == M_NCCL) {
                const int peer = D.rank + HDIR[d].dy * D.px + HDIR[d].dx;
                st = nc_sendrecv(D, D.sb[0] + off[0][d], D.rb[0] + off[0][d], len[0][d], peer, D.xs);
            } else {  // my segment d <- the neighbour's segment towards me
                const int nb = tile_at(D, D.tx[k] + HDIR[d].dx, D.ty[k] + HDIR[d].dy), o = opposite(d);
                st = p2p_local(D, D.rb[k] + off[k][d], D.sb[nb] + off[nb][o], len[k][d]);
            }
            if (st) return st;
        }
    if ((st = group_end(D))) return st;
    s.count = 0;
    for (int k = 0; k < D.nt; ++k) {  // unpack into the halos
        const GridL &g = D.tile[k]->lev[l].g;
        const int nf = nfields(D, D.tile[k], l, which, idx, f);
        for (int d = 0; d < 8; ++d)
            if (len[k][d]) {
                if (s.count + 3 * HW > 512) { launch_strips(c, s); s.count = 0; }
                dir_strips(D, g, D.tx[k], D.ty[k], d, true, f, nf, D.rb[k] + off[k][d], s);
            }
    }
    if (s.count) launch_strips(c, s);
    return STOKES_OK;
}

// Halo exchange of the selected fields of level l: HW = 2 rings, two phases (W/E columns
// over rows -1 .. ncy+2, then N/S rows over columns -1 .. ncx+2: corners included).
//   my column ncx + h <- E neighbour's column h,   my column 1 - h <- W neighbour's ncx + 1 - h
//   my row    ncy + h <- S neighbour's row h,      my row    1 - h <- N neighbour's ncy + 1 - h
// (h = 1, 2; the same map for every node type, since tiles own the east vx faces, the south
// vy faces and the south-east basic nodes of their cells).
int exchange(Dist &D, int l, int which, int idx) {
    const LaunchCtx c = dctx(D);
    double *f[3], *fu[3];
    const int rows = D.tile[0]->lev[l].g.ncy + 2 * HW, cols = D.tile[0]->lev[l].g.ncx + 2 * HW;
    if (!packed(D)) {  // ---- virtual: strip-copy kernels between the tiles' buffers
        StripList s;
        s.count = 0;
        for (int k = 0; k < D.nt; ++k) {
            const GridL &g = D.tile[k]->lev[l].g;
            const int nf = nfields(D, D.tile[k], l, which, idx, f);
            for (int side = 0; side < 2; ++side) {
                const int nb = side ? (D.tx[k] + 1 < D.px ? tile_at(D, D.tx[k] + 1, D.ty[k]) : -1)
                                    : (D.tx[k] > 0 ? tile_at(D, D.tx[k] - 1, D.ty[k]) : -1);
                if (nb < 0) continue;
                nfields(D, D.tile[nb], l, which, idx, fu);
                for (int q = 0; q < nf; ++q)
                    for (int hh = 1; hh <= HW; ++hh) {
                        const int jd = side ? g.ncx + hh : 1 - hh, js = side ? hh : g.ncx + 1 - hh;
                        add_strip(s, f[q] + at(g, -1, jd), fu[q] + at(g, -1, js), rows, g.P, g.P);
                    }
            }
        }
        if (s.count) launch_strips(c, s);
        s.count = 0;
        for (int k = 0; k < D.nt; ++k) {
            const GridL &g = D.tile[k]->lev[l].g;
            const int nf = nfields(D, D.tile[k], l, which, idx, f);
            for (int side = 0; side < 2; ++side) {
                const int nb = side ? (D.ty[k] + 1 < D.py ? tile_at(D, D.tx[k], D.ty[k] + 1) : -1)
                                    : (D.ty[k] > 0 ? tile_at(D, D.tx[k], D.ty[k] - 1) : -1);
                if (nb < 0) continue;
                nfields(D, D.tile[nb], l, which, idx, fu);
                for (int q = 0; q < nf; ++q)
                    for (int hh = 1; hh <= HW; ++hh) {
                        const int id = side ? g.ncy + hh : 1 - hh, is = side ? hh : g.ncy + 1 - hh;
                        add_strip(s, f[q] + at(g, id, -1), fu[q] + at(g, is, -1), cols, 1, 1);
                    }
            }
        }
        if (s.count) launch_strips(c, s);
        return STOKES_OK;
    }
    if (!D.halo2) return exchange_one_round(D, l, which, idx);
    // ---- packed transports, two rounds (STOKES_HALO_2PHASE=1): NCCL (one tile per process),
    // NCCL_SELF (every tile here, real ncclSend / ncclRecv on a one-rank communicator),
    // LOOPBACK (every tile here, device copies)
    int nf = 0, st;
    {  // phase 1: W/E columns packed into sb = [W part | E part], nf x HW x rows each
        StripList s;
        s.count = 0;
        for (int k = 0; k < D.nt; ++k) {
            const GridL &g = D.tile[k]->lev[l].g;
            nf = nfields(D, D.tile[k], l, which, idx, f);
            const bool W = D.tx[k] > 0, E = D.tx[k] + 1 < D.px;
            for (int q = 0; q < nf; ++q)
                for (int hh = 1; hh <= HW; ++hh) {
                    const size_t e = (size_t)(q * HW + hh - 1) * rows;
                    if (W) add_strip(s, D.sb[k] + e, f[q] + at(g, -1, hh), rows, 1, g.P);
                    if (E) add_strip(s, D.sb[k] + (size_t)nf * HW * rows + e, f[q] + at(g, -1, g.ncx + 1 - hh), rows, 1, g.P);
                }
        }
        if (s.count) launch_strips(c, s);
        const size_t part = (size_t)nf * HW * rows;
        if ((st = group_start(D))) return st;
        if (D.mode == M_NCCL) {
            const int W = D.tx[0] > 0 ? D.rank - 1 : -1, E = D.tx[0] + 1 < D.px ? D.rank + 1 : -1;
            if (W >= 0 && (st = nc_sendrecv(D, D.sb[0], D.rb[0], part, W, D.xs))) return st;
            if (E >= 0 && (st = nc_sendrecv(D, D.sb[0] + part, D.rb[0] + part, part, E, D.xs))) return st;
        } else {  // my W part <- W neighbour's E part, my E part <- E neighbour's W part
            for (int k = 0; k < D.nt; ++k) {
                if (D.tx[k] > 0 && (st = p2p_local(D, D.rb[k], D.sb[tile_at(D, D.tx[k] - 1, D.ty[k])] + part, part)))
                    return st;
                if (D.tx[k] + 1 < D.px && (st = p2p_local(D, D.rb[k] + part, D.sb[tile_at(D, D.tx[k] + 1, D.ty[k])], part)))
                    return st;
            }
        }
        if ((st = group_end(D))) return st;
        s.count = 0;
        for (int k = 0; k < D.nt; ++k) {
            const GridL &g = D.tile[k]->lev[l].g;
            nfields(D, D.tile[k], l, which, idx, f);
            for (int q = 0; q < nf; ++q)
                for (int hh = 1; hh <= HW; ++hh) {
                    const size_t e = (size_t)(q * HW + hh - 1) * rows;
                    if (D.tx[k] > 0) add_strip(s, f[q] + at(g, -1, 1 - hh), D.rb[k] + e, rows, g.P, 1);
                    if (D.tx[k] + 1 < D.px) add_strip(s, f[q] + at(g, -1, g.ncx + hh), D.rb[k] + part + e, rows, g.P, 1);
                }
        }
        if (s.count) launch_strips(c, s);
    }
    // phase 2: the HW halo rows of a side are one contiguous block (rows r .. r+HW-1, columns
    // -1 .. ncx+2): sent straight from / received straight into the field
    if ((st = group_start(D))) return st;
    for (int k = 0; k < D.nt; ++k) {
        const GridL &g = D.tile[k]->lev[l].g;
        const size_t blk = (size_t)(HW - 1) * g.P + cols;
        nfields(D, D.tile[k], l, which, idx, f);
        if (D.mode == M_NCCL) {
            const int N = D.ty[0] > 0 ? D.rank - D.px : -1, S = D.ty[0] + 1 < D.py ? D.rank + D.px : -1;
            for (int q = 0; q < nf; ++q) {
                if (N >= 0 && (st = nc_sendrecv(D, f[q] + at(g, 1, -1), f[q] + at(g, 1 - HW, -1), blk, N, D.xs)))
                    return st;
                if (S >= 0 &&
                    (st = nc_sendrecv(D, f[q] + at(g, g.ncy + 1 - HW, -1), f[q] + at(g, g.ncy + 1, -1), blk, S, D.xs)))
                    return st;
            }
        } else {
            for (int q = 0; q < nf; ++q) {
                if (D.ty[k] > 0) {
                    nfields(D, D.tile[tile_at(D, D.tx[k], D.ty[k] - 1)], l, which, idx, fu);
                    if ((st = p2p_local(D, f[q] + at(g, 1 - HW, -1), fu[q] + at(g, g.ncy + 1 - HW, -1), blk))) return st;
                }
                if (D.ty[k] + 1 < D.py) {
                    nfields(D, D.tile[tile_at(D, D.tx[k], D.ty[k] + 1)], l, which, idx, fu);
                    if ((st = p2p_local(D, f[q] + at(g, g.ncy + 1, -1), fu[q] + at(g, 1, -1), blk))) return st;
                }
            }
        }
    }
    return group_end(D);
}

// tile rectangle [r0, r0+nr) x [c0, c0+nc) of a level-La field -> global tail level 0 at
// the tile's offset (NCCL: all-gathered first).  `which`: 0 velocity rhs (bx, by), 1 eta.
int gather_to_tail(Dist &D, int which) {
    Level &T0 = D.tail->lev[0];
    const int La = D.La;
    auto rect = [&](int k, int f, int &r0, int &c0, int &nr, int &nc) {
        const GridL &gc = D.tile[0]->lev[La].g;  // all tiles share sizes
        (void)k;
        if (which == 0) { r0 = 1; c0 = 1; nr = gc.ncy; nc = gc.ncx; }  // owned unknowns (+ global walls, 0)
        else if (f == 0) { r0 = 0; c0 = 0; nr = gc.ncy + 1; nc = gc.ncx + 1; }  // basic nodes (halo-consistent)
        else { r0 = 1; c0 = 1; nr = gc.ncy; nc = gc.ncx; }  // P nodes
    };
    const GridL &gc = D.tile[0]->lev[La].g;
    if (D.mode == M_VIRTUAL) {
        for (int k = 0; k < D.nt; ++k) {
            Level &C = D.tile[k]->lev[La];
            double *src[2] = {which == 0 ? C.bx : C.etab, which == 0 ? C.by : C.etap};
            double *dst[2] = {which == 0 ? T0.bx : T0.etab, which == 0 ? T0.by : T0.etap};
            const int gi = D.ty[k] * gc.ncy, gj = D.tx[k] * gc.ncx;
            for (int f = 0; f < 2; ++f) {
                int r0, c0, nr, nc;
                rect(k, f, r0, c0, nr, nc);
                CK(cudaMemcpy2DAsync(dst[f] + at(T0.g, gi + r0, gj + c0), T0.g.P * 8, src[f] + at(gc, r0, c0), gc.P * 8,
                                     (size_t)nc * 8, nr, cudaMemcpyDeviceToDevice, D.stream));
            }
        }
        return STOKES_OK;
    }
    // packed: every tile packs its rectangles into a block of its sb; the blocks of all ranks
    // are all-gathered (NCCL) or concatenated (loopback) into rb[0] and unpacked in rank order
    const size_t blk = (size_t)2 * (gc.ncy + 1) * (gc.ncx + 1);
    double *dst[2] = {which == 0 ? T0.bx : T0.etab, which == 0 ? T0.by : T0.etap};
    for (int k = 0; k < D.nt; ++k) {
        Level &C = D.tile[k]->lev[La];
        double *src[2] = {which == 0 ? C.bx : C.etab, which == 0 ? C.by : C.etap};
        for (int f = 0; f < 2; ++f) {
            int r0, c0, nr, nc;
            rect(k, f, r0, c0, nr, nc);
            CK(cudaMemcpy2DAsync(D.sb[k] + f * (blk / 2), (size_t)nc * 8, src[f] + at(gc, r0, c0), gc.P * 8,
                                 (size_t)nc * 8, nr, cudaMemcpyDeviceToDevice, D.stream));
        }
    }
    if (D.mode == M_NCCL) {
        if (int st = nc_allgather(D, D.sb[0], D.rb[0], blk, D.stream)) return st;
    } else {
        int st = group_start(D);
        for (int k = 0; k < D.nt && !st; ++k) st = p2p_local(D, D.rb[0] + (size_t)k * blk, D.sb[k], blk);
        if (st || (st = group_end(D))) return st;
    }
    for (int r = 0; r < D.px * D.py; ++r) {
        const int gi = (r / D.px) * gc.ncy, gj = (r % D.px) * gc.ncx;
        for (int f = 0; f < 2; ++f) {
            int r0, c0, nr, nc;
            rect(r, f, r0, c0, nr, nc);
            CK(cudaMemcpy2DAsync(dst[f] + at(T0.g, gi + r0, gj + c0), T0.g.P * 8, D.rb[0] + r * blk + f * (blk / 2),
                                 (size_t)nc * 8, (size_t)nc * 8, nr, cudaMemcpyDeviceToDevice, D.stream));
        }
    }
    return STOKES_OK;
}

// every tile takes its window (halos included) of the tail's level-0 correction
int scatter_from_tail(Dist &D) {
    Level &T0 = D.tail->lev[0];
    for (int k = 0; k < D.nt; ++k) {
        Level &C = D.tile[k]->lev[D.La];
        const GridL &gc = C.g;
        const int gi = D.ty[k] * gc.ncy, gj = D.tx[k] * gc.ncx;
        CK(cudaMemcpy2DAsync(C.vx[0] + at(gc, 0, 0), gc.P * 8, T0.vx[0] + at(T0.g, gi, gj), T0.g.P * 8,
                             (size_t)(gc.ncx + 2) * 8, gc.ncy + 2, cudaMemcpyDeviceToDevice, D.stream));
        CK(cudaMemcpy2DAsync(C.vy[0] + at(gc, 0, 0), gc.P * 8, T0.vy[0] + at(T0.g, gi, gj), T0.g.P * 8,
                             (size_t)(gc.ncx + 2) * 8, gc.ncy + 2, cudaMemcpyDeviceToDevice, D.stream));
    }
    return STOKES_OK;
}

RhsArgs tile_rhs(stokes_s *t, int l, bool fine) {
    return fine ? rhs_fine(t) : rhs_arrays(t->lev[l].bx, t->lev[l].by);
}

// n smoother sweeps on distributed level l; cur = index of the buffer holding v.  Damped
// Jacobi runs the single-domain kernels: pairs of sweeps as ONE two-sweep pass (k_jacobi2,
// which also updates the first halo ring) where the level allows, at most max_pairs of them;
// the width-2 halos are exchanged once per pass.  RBGS: the four phase kernels with an
// exchange after each phase.
int dsmooth(Dist &D, int l, int &cur, int n, bool zero_in, bool fine, int max_pairs) {
    if (n <= 0 && zero_in) {
        for (int k = 0; k < D.nt; ++k) {
            Level &L = D.tile[k]->lev[l];
            CK(cudaMemsetAsync(fstart(L.g, L.vx[cur]), 0, fsize(L.g) * 8, D.stream));
            CK(cudaMemsetAsync(fstart(L.g, L.vy[cur]), 0, fsize(L.g) * 8, D.stream));
        }
        return STOKES_OK;
    }
    int st;
    if (D.o.smoother == STOKES_SMOOTH_JACOBI) {
        const GridL &g0 = D.tile[0]->lev[l].g;
        int pairs = jacobi2_ok(g0) ? (n - (zero_in ? 1 : 0)) / 2 : 0;
        if (pairs > max_pairs) pairs = max_pairs;
        for (int s = 0; s < n;) {
            const bool two = pairs > 0 && !(zero_in && s == 0);
            if (D.overlap && stream_ok(g0) && g0.ncx >= D.overlap_min && !(zero_in && s == 0)) {
                // boundary layers first, then their halo exchange on the comm stream while the
                // interior of the tiles is swept
                for (int pp = 0; pp < 2; ++pp) {
                    const int part = pp;
                    for (int k = 0; k < D.nt; ++k) {
                        stokes_s *t = D.tile[k];
                        Level &L = t->lev[l];
                        if (two)
                            launch_jacobi2_part(ctx(t), L.g, L.etab, L.etap, L.vx[cur], L.vy[cur], L.vx[1 - cur],
                                                L.vy[1 - cur], tile_rhs(t, l, fine), D.o.omega_v, part);
                        else
                            launch_jacobi_stream_part(ctx(t), L.g, L.etab, L.etap, L.vx[cur], L.vy[cur],
                                                      L.vx[1 - cur], L.vy[1 - cur], tile_rhs(t, l, fine), D.o.omega_v,
                                                      part);
                    }
                    if (pp == 0) {
                        CK(cudaEventRecord(D.ev[0], D.stream));
                        CK(cudaStreamWaitEvent(D.cstream, D.ev[0], 0));
                        D.xs = D.serial_split ? D.stream : D.cstream;
                        st = exchange(D, l, FX_V, 1 - cur);
                        D.xs = D.stream;
                        if (st) return st;
                        CK(cudaEventRecord(D.ev[1], D.cstream));
                    }
                }
                CK(cudaStreamWaitEvent(D.stream, D.ev[1], 0));
                if (two) { --pairs; s += 2; }
                else s += 1;
                cur ^= 1;
                continue;
            }
            for (int k = 0; k < D.nt; ++k) {
                stokes_s *t = D.tile[k];
                Level &L = t->lev[l];
                if (two)
                    launch_jacobi2(ctx(t), L.g, L.etab, L.etap, L.vx[cur], L.vy[cur], L.vx[1 - cur], L.vy[1 - cur],
                                   tile_rhs(t, l, fine), D.o.omega_v);
                else
                    launch_jacobi(ctx(t), L.g, L.etab, L.etap, L.vx[cur], L.vy[cur], L.vx[1 - cur], L.vy[1 - cur],
                                  tile_rhs(t, l, fine), D.o.omega_v, zero_in && s == 0);
            }
            if (two) { --pairs; s += 2; }
            else s += 1;
            cur ^= 1;
            if ((st = exchange(D, l, FX_V, cur))) return st;
        }
        return STOKES_OK;
    }
    for (int s = 0; s < n; ++s) {
        if (zero_in && s == 0)
            for (int k = 0; k < D.nt; ++k) {
                Level &L = D.tile[k]->lev[l];
                CK(cudaMemsetAsync(fstart(L.g, L.vx[cur]), 0, fsize(L.g) * 8, D.stream));
                CK(cudaMemsetAsync(fstart(L.g, L.vy[cur]), 0, fsize(L.g) * 8, D.stream));
            }
        for (int comp = 0; comp < 2; ++comp)
            for (int colour = 0; colour < 2; ++colour) {
                for (int k = 0; k < D.nt; ++k) {
                    stokes_s *t = D.tile[k];
                    Level &L = t->lev[l];
                    launch_rbgs_phase(ctx(t), L.g, L.etab, L.etap, L.vx[cur], L.vy[cur], tile_rhs(t, l, fine),
                                      D.o.omega_v, comp, colour);
                }
                if ((st = exchange(D, l, FX_V, cur))) return st;
            }
    }
    return STOKES_OK;
}

// distributed V-cycle on level l (Eq. multigrid_levels); v in buffer 0.
// done_pre = 1: the first pre-smoothing sweep was done by the fused Uzawa pass into buffer 1.
// The same launch sequence as the single-domain vcycle (driver.cu): an even pair count so the
// 2 nu sweeps end in buffer 0, the residual fused with its restriction where the level streams.
int dvcycle(Dist &D, int l, bool fine, bool zero_in, int done_pre = 0) {
    int cur = done_pre ? 1 : 0, st;
    const int nu = D.tile[0]->lev[l].nu;
    const GridL &g0 = D.tile[0]->lev[l].g;
    const bool j2 = D.o.smoother == STOKES_SMOOTH_JACOBI && jacobi2_ok(g0);
    const int pre_n = nu - done_pre;
    int pre_pairs = j2 ? (pre_n - (zero_in && !done_pre ? 1 : 0)) / 2 : 0, post_pairs = j2 ? nu / 2 : 0;
    if (pre_pairs < 0) pre_pairs = 0;
    if ((pre_pairs + post_pairs) & 1) {
        if (post_pairs > 0) --post_pairs;
        else --pre_pairs;
    }
    if ((st = dsmooth(D, l, cur, pre_n, zero_in && !done_pre, fine, pre_pairs))) return st;  // (1)
    if (jacobi2_ok(g0)) {  // (2) + (3): residual and restriction in one pass, then the coarse halos
        for (int k = 0; k < D.nt; ++k) {
            stokes_s *t = D.tile[k];
            Level &L = t->lev[l], &C = t->lev[l + 1];
            launch_residual_restrict(ctx(t), L.g, C.g, L.etab, L.etap, L.vx[cur], L.vy[cur], tile_rhs(t, l, fine), C.bx,
                                     C.by);
        }
    } else {
        for (int k = 0; k < D.nt; ++k) {
            stokes_s *t = D.tile[k];
            Level &L = t->lev[l];
            launch_residual(ctx(t), L.g, L.etab, L.etap, L.vx[cur], L.vy[cur], tile_rhs(t, l, fine), L.rx, L.ry);
        }
        if ((st = exchange(D, l, FX_R, 0))) return st;
        for (int k = 0; k < D.nt; ++k) {
            stokes_s *t = D.tile[k];
            launch_restrict_vel(ctx(t), t->lev[l].g, t->lev[l + 1].g, t->lev[l].rx, t->lev[l].ry, t->lev[l + 1].bx,
                                t->lev[l + 1].by);
        }
    }
    if (l + 1 < D.La) {                                                         // (4)
        if ((st = exchange(D, l + 1, FX_B, 0))) return st;  // the coarse right-hand side's halos
        if ((st = dvcycle(D, l + 1, false, true))) return st;
    } else {  // agglomerated coarse tail, redundant on every process
        if ((st = gather_to_tail(D, 0))) return st;
        Level &T0 = D.tail->lev[0];
        vcycle(D.tail, 0, T0.vx[0], T0.vy[0], T0.vx[1], T0.vy[1], rhs_arrays(T0.bx, T0.by), true);
        if ((st = scatter_from_tail(D))) return st;
    }
    for (int k = 0; k < D.nt; ++k) {                                            // (5)
        stokes_s *t = D.tile[k];
        Level &L = t->lev[l], &C = t->lev[l + 1];
        launch_prolong(ctx(t), L.g, C.g, C.vx[0], C.vy[0], L.vx[cur], L.vy[cur]);
    }
    if ((st = exchange(D, l, FX_V, cur))) return st;
    if ((st = dsmooth(D, l, cur, nu, false, fine, post_pairs))) return st;      // (6)
    if (cur != 0) {
        for (int k = 0; k < D.nt; ++k) {
            Level &L = D.tile[k]->lev[l];
            CK(cudaMemcpyAsync(fstart(L.g, L.vx[0]), fstart(L.g, L.vx[cur]), fsize(L.g) * 8, cudaMemcpyDeviceToDevice, D.stream));
            CK(cudaMemcpyAsync(fstart(L.g, L.vy[0]), fstart(L.g, L.vy[cur]), fsize(L.g) * 8, cudaMemcpyDeviceToDevice, D.stream));
        }
    }
    return STOKES_OK;
}

// combine the tiles' local (Sv, Sp, sum p) at t->scal[S_LOC..] into E (dscal[0]) and the
// global pressure mean (each tile's scal[S_MSHIFT] when write_mean)
int combine(Dist &D, bool write_mean) {
    const LaunchCtx c = dctx(D);
    const double *loc[MAXT];
    double *ms[MAXT];
    for (int k = 0; k < D.nt; ++k) {
        loc[k] = D.tile[k]->scal + S_LOC;
        ms[k] = D.tile[k]->scal + S_MSHIFT;
    }
    if (D.mode == M_NCCL)
        if (int st = nc_allreduce(D, D.tile[0]->scal + S_LOC, 3, ncclDouble, ncclSum, D.stream)) return st;
    if (self_nccl(D))  // (one rank: the sum over the tiles follows on the device)
        for (int k = 0; k < D.nt; ++k)
            if (ncclAllReduce(D.tile[k]->scal + S_LOC, D.tile[k]->scal + S_LOC, 3, ncclDouble, ncclSum, D.comm,
                              D.stream) != ncclSuccess)
                return STOKES_ENCCL;
    launch_dist_final(c, loc, D.nt, D.dscal + 3, 1.0 / ((double)D.NX * D.NY), D.dscal, ms, write_mean ? D.nt : 0);
    return STOKES_OK;
}

// local sums of the fused Uzawa pass (pout_idx >= 0: p' -> pbuf[pout_idx]) or of the energy
// of the current state only (pout_idx < 0) -> each tile's scal[S_LOC..S_LOC+2]
int tiles_uzawa(Dist &D, int pin_idx, int pout_idx, double alpha_s) {
    const bool fused = stream_ok(D.tile[0]->lev[0].g);
    for (int k = 0; k < D.nt; ++k) {
        stokes_s *t = D.tile[k];
        Level &F = t->lev[0];
        const LaunchCtx c = ctx(t);
        const double *pin = t->pbuf[pin_idx];
        double *pout = pout_idx >= 0 ? t->pbuf[pout_idx] : nullptr;
        const double *ms = t->scal + (pout ? S_MSHIFT : S_ZERO);
        if (fused) {  // p' at the east / south neighbours recomputed from v: no p halo needed
            launch_uzawa_energy(c, F.g, F.etab, F.etap, F.vx[0], F.vy[0], pin, pout, t->rho, D.gx, D.gy, alpha_s, ms,
                                nullptr, nullptr, nullptr, t->partials);
            launch_finalize(c, t->partials, stream_blocks(F.g), 3, 1.0, t->scal + S_LOC);
        } else {
            double *pp = t->partials + 8192;
            launch_pupdate(c, F.g, F.etap, F.vx[0], F.vy[0], pin, pout, alpha_s, ms, pp);
            launch_finalize(c, pp, pupdate_blocks(F.g), 1, 1.0, t->scal + S_LOC + 2);
        }
    }
    if (fused) return STOKES_OK;
    if (pout_idx >= 0) {  // the energy stencil reads p' at the east / south halo
        int st = exchange(D, 0, FX_P, pout_idx);
        if (st) return st;
    }
    for (int k = 0; k < D.nt; ++k) {
        stokes_s *t = D.tile[k];
        Level &F = t->lev[0];
        const LaunchCtx c = ctx(t);
        launch_energy(c, F.g, F.etab, F.etap, F.vx[0], F.vy[0], t->pbuf[pout_idx >= 0 ? pout_idx : pin_idx], t->rho,
                      D.gx, D.gy, nullptr, nullptr, nullptr, t->partials, false);
        launch_finalize(c, t->partials, energy_blocks(F.g), 2, 1.0, t->scal + S_LOC);
    }
    return STOKES_OK;
}

int dist_body(Dist &D) {  // one Uzawa iteration reading pbuf[pcur]
    int st;
    if ((st = dvcycle(D, 0, true, false))) return st;
    const double a_s = D.o.pressure_sign * D.o.alpha_p;
    if ((st = tiles_uzawa(D, D.pcur, 1 - D.pcur, a_s))) return st;
    if ((st = combine(D, true))) return st;
    if ((st = exchange(D, 0, FX_P, 1 - D.pcur))) return st;
    CK(cudaMemcpyAsync(D.hsc, D.dscal, 8 * sizeof(double), cudaMemcpyDeviceToHost, D.stream));
    return STOKES_OK;
}

// a12 fusion on the tiles (as solve_uzawa_fused, driver.cu): from v^k (buffer 0) and
// p^(k-1) = pbuf[pcur] one pass per tile computes p^k -> pbuf[1-pcur], the local sums of
// E(v^k, p^k) and the first pre-smoothing sweep of V-cycle k+1 -> buffer 1; then the global
// sums and the halos of (v', p^k)
bool dist_fused_ok(const Dist &D) {
    return D.o.smoother == STOKES_SMOOTH_JACOBI && D.o.vcycles_per_iter == 1 && D.tile[0]->lev[0].nu >= 1 &&
           stream_ok(D.tile[0]->lev[0].g);
}
int dist_fused_tail(Dist &D) {
    const double a_s = D.o.pressure_sign * D.o.alpha_p;
    for (int k = 0; k < D.nt; ++k) {
        stokes_s *t = D.tile[k];
        Level &F = t->lev[0];
        const LaunchCtx c = ctx(t);
        launch_jacobi_uzawa(c, F.g, F.etab, F.etap, F.vx[0], F.vy[0], F.vx[1], F.vy[1], t->pbuf[D.pcur],
                            t->pbuf[1 - D.pcur], t->rho, D.gx, D.gy, a_s, t->scal + S_MSHIFT, D.o.omega_v, t->partials);
        launch_finalize(c, t->partials, stream_blocks(F.g), 3, 1.0, t->scal + S_LOC);
    }
    int st;
    if ((st = combine(D, true))) return st;
    if ((st = exchange(D, 0, FX_VP, 1 | ((1 - D.pcur) << 1)))) return st;
    CK(cudaMemcpyAsync(D.hsc, D.dscal, 8 * sizeof(double), cudaMemcpyDeviceToHost, D.stream));
    return STOKES_OK;
}
int dist_fused_body(Dist &D) {  // the rest of V-cycle k+1 (first sweep in buffer 1), then the fused tail
    int st;
    if ((st = dvcycle(D, 0, true, false, 1))) return st;
    return dist_fused_tail(D);
}

int dsync(Dist &D) {
    CK(cudaStreamSynchronize(D.stream));
    CKL();
    return STOKES_OK;
}

int state_E(Dist &D, double *E) {  // E of (v, pbuf[pcur]); mean of p -> mshift
    int st = tiles_uzawa(D, D.pcur, -1, 0.0);
    if (st) return st;
    st = combine(D, true);
    if (st) return st;
    CK(cudaMemcpyAsync(D.hsc, D.dscal, 8 * sizeof(double), cudaMemcpyDeviceToHost, D.stream));
    if ((st = dsync(D))) return st;
    *E = D.hsc[0];
    return STOKES_OK;
}

int force_E(Dist &D) {  // Sf -> dscal[3]
    for (int k = 0; k < D.nt; ++k) {
        stokes_s *t = D.tile[k];
        Level &F = t->lev[0];
        const LaunchCtx c = ctx(t);
        launch_energy(c, F.g, F.etab, F.etap, F.vx[0], F.vy[0], t->pbuf[0], t->rho, D.gx, D.gy, nullptr, nullptr,
                      nullptr, t->partials, true);
        launch_finalize(c, t->partials, energy_blocks(F.g), 2, 1.0, t->scal + S_LOC);
        CK(cudaMemsetAsync(t->scal + S_LOC + 2, 0, 8, D.stream));
    }
    CK(cudaMemsetAsync(D.dscal + 3, 0, 8, D.stream));  // Sf slot = 0 while combining
    int st = combine(D, false);
    if (st) return st;
    CK(cudaMemcpyAsync(D.dscal + 3, D.dscal + 1, 8, cudaMemcpyDeviceToDevice, D.stream));
    return dsync(D);
}

// ---- flexible GCR(m) with MGS (Alg. 4; readings R13 / R14) on the tiles
// The single-domain fused kernels run per tile.  Every GCR vector lives at the tile's owned
// unknowns (w-type vectors are written only there, so their halos stay 0 and the per-tile
// dot products sum each unknown once); z comes out of the distributed V-cycle with valid
// halos, x keeps consistent halos through the axpys with global coefficients, and r's halos
// (the V-cycle's right-hand side, the z_p recomputation of PrecondApplyOp) are exchanged
// after every update.  A kernel's per-CTA partials go to the tile's segment of one buffer
// (NCCL: all-gathered across the ranks), and the next kernel of EVERY tile reduces the
// whole buffer in the same fixed order: the global inner products, identical everywhere.
static int gather_segments(Dist &D, double *base, size_t seg) {  // every rank's segment of `base` everywhere
    if (D.mode == M_NCCL_SELF) {  // the same call on the one-rank communicator (in place, per tile)
        if (ncclGroupStart() != ncclSuccess) return STOKES_ENCCL;
        for (int k = 0; k < D.nt; ++k)
            if (ncclAllGather(base + (size_t)k * seg, base + (size_t)k * seg, seg, ncclDouble, D.comm, D.stream) !=
                ncclSuccess)
                return STOKES_ENCCL;
        return ncclGroupEnd() == ncclSuccess ? STOKES_OK : STOKES_ENCCL;
    }
    if (D.mode != M_NCCL) return STOKES_OK;
    return nc_allgather(D, base + (size_t)D.rank * seg, base, seg, D.stream);
}
static int tiles_sum(Dist &D, int buf, int nb) {  // NCCL: all-gather rank segments of gpart[buf]
    return gather_segments(D, D.gpart[buf], (size_t)nb * 2);
}
static double *seg_of(Dist &D, int buf, int k, int nb) {  // tile k's partials (NCCL: this rank's)
    const int r = D.mode == M_NCCL ? D.rank : k;
    return D.gpart[buf] + (size_t)r * nb * 2;
}
static int nranks(const Dist &D) { return D.mode == M_NCCL ? D.px * D.py : D.nt; }

// r = b - A x (true residual) on every tile + its E -> dscal[0]; x halos refreshed first
static int dist_gcr_residual(Dist &D) {
    int st;
    if ((st = exchange(D, 0, FX_VP, 0 | (D.pcur << 1)))) return st;
    for (int k = 0; k < D.nt; ++k) {
        stokes_s *t = D.tile[k];
        Level &F = t->lev[0];
        const LaunchCtx c = ctx(t);
        launch_uzawa_energy(c, F.g, F.etab, F.etap, F.vx[0], F.vy[0], t->pbuf[D.pcur], nullptr, t->rho, D.gx, D.gy,
                            0.0, t->scal + S_ZERO, t->gr[0], t->gr[1], t->gr[2], t->partials);
        launch_finalize(c, t->partials, stream_blocks(F.g), 3, 1.0, t->scal + S_LOC);
    }
    if ((st = combine(D, false))) return st;
    return exchange(D, 0, FX_GR, 0);
}

// one GCR step i on the tiles (as gcr_step_body, driver.cu): z_i = V-cycle(0; r_v) (the
// distributed V-cycle), z_p + w = A z + first dot, i MGS steps, normalise + update x, r + the
// energy of r; E, nu^2, <r,r> -> dscal[0..2] -> host
static int dist_gcr_step_body(Dist &D, int i) {
    int st;
    const int NR = nranks(D);
    // the distributed V-cycle reads its right-hand side from lev[0].(bx, by) and leaves the
    // result in lev[0].(vx[0], vy[0]): point them at r, z_i and the scratch for the capture
    double *keep[MAXT][6];
    for (int k = 0; k < D.nt; ++k) {
        stokes_s *t = D.tile[k];
        Level &F = t->lev[0];
        double *kk[6] = {F.bx, F.by, F.vx[0], F.vy[0], F.vx[1], F.vy[1]};
        memcpy(keep[k], kk, sizeof kk);
        F.bx = t->gr[0];
        F.by = t->gr[1];
        F.vx[0] = t->gz[i][0];
        F.vy[0] = t->gz[i][1];
        F.vx[1] = t->gtmp[0];
        F.vy[1] = t->gtmp[1];
    }
    st = dvcycle(D, 0, false, true);
    for (int k = 0; k < D.nt; ++k) {  // restore
        Level &F = D.tile[k]->lev[0];
        F.bx = keep[k][0];
        F.by = keep[k][1];
        F.vx[0] = keep[k][2];
        F.vy[0] = keep[k][3];
        F.vx[1] = keep[k][4];
        F.vy[1] = keep[k][5];
    }
    if (st) return st;
    const int nbs = stream_blocks(D.tile[0]->lev[0].g), nbf = gcr_flat_blocks(field_doubles(D.tile[0]->lev[0].g));
    for (int k = 0; k < D.nt; ++k) {
        stokes_s *t = D.tile[k];
        Level &F = t->lev[0];
        double **z = t->gz[i], **w = t->gw[i], **r = t->gr;
        launch_precond_apply(ctx(t), F.g, F.etab, F.etap, z[0], z[1], r[2], D.o.alpha_p, z[2], w[0], w[1], w[2],
                             i > 0 ? (const double *const *)t->gw[0] : nullptr, r[0], r[1], seg_of(D, 0, k, nbs));
    }
    if ((st = tiles_sum(D, 0, nbs))) return st;
    int pin = 0, nbin = nbs * NR;
    for (int j = 0; j < i; ++j) {
        const int pout = 1 + (j & 1);
        for (int k = 0; k < D.nt; ++k) {
            stokes_s *t = D.tile[k];
            const size_t nf = field_doubles(t->lev[0].g);
            const double *const *nxt = (j + 1 < i) ? (const double *const *)t->gw[j + 1] : nullptr;
            launch_mgs_step(ctx(t), D.gpart[pin], nbin, 2, 0, t->gw[i], nullptr, (const double *const *)t->gw[j],
                            (const double *const *)t->gz[j], nxt, (const double *const *)t->gr, nf, seg_of(D, pout, k, nbf),
                            t->scal + S_GAMS + j);  // (z update deferred to the update pass, as on one domain)
        }
        if ((st = tiles_sum(D, pout, nbf))) return st;
        pin = pout;
        nbin = nbf * NR;
    }
    const int pu = pin == 1 ? 2 : 1;  // the update's partials: the buffer pin is not
    for (int k = 0; k < D.nt; ++k) {
        stokes_s *t = D.tile[k];
        Level &F = t->lev[0];
        double *x[3] = {F.vx[0], F.vy[0], t->pbuf[D.pcur]};
        launch_gcr_update(ctx(t), D.gpart[pin], nbin, t->gw[i], t->gz[i], x, t->gr, (const double *const *)t->gew,
                          field_doubles(F.g), seg_of(D, pu, k, nbf), t->scal + S_GAMS, i, t->gz);
    }
    if ((st = tiles_sum(D, pu, nbf))) return st;
    launch_gcr_final(dctx(D), D.gpart[pu], nbf * NR, D.gpart[pin], nbin, D.dscal + 3, D.dscal + 0, D.dscal + 1,
                     D.dscal + 2);
    if ((st = exchange(D, 0, FX_GR, 0))) return st;  // r's halos for the next V-cycle
    CK(cudaMemcpyAsync(D.hsc, D.dscal, 8 * sizeof(double), cudaMemcpyDeviceToHost, D.stream));
    return STOKES_OK;
}

static int dist_solve_gcr(Dist &D, double rtol, double E0, int *iters, double *Eout) {
    int st;
    const int m = D.o.gcr_restart;
    if (!D.gpart[0]) {  // partial buffers: every rank / tile, the larger of the two kernels' block counts
        const int nbs = stream_blocks(D.tile[0]->lev[0].g), nbf = gcr_flat_blocks(field_doubles(D.tile[0]->lev[0].g));
        D.gseg = (size_t)2 * (nbs > nbf ? nbs : nbf);
        for (int b = 0; b < 3; ++b)
            if (cudaMalloc(&D.gpart[b], D.gseg * nranks(D) * sizeof(double)) != cudaSuccess) return STOKES_ENOMEM;
    }
    if ((st = dist_gcr_residual(D))) return st;  // r0 = b - A x0
    int k = 0, status = STOKES_NOT_CONVERGED, fresh = 1;
    double E = E0;
    while (k < D.o.max_iter && status == STOKES_NOT_CONVERGED) {
        if (!fresh && D.o.gcr_true_restart && (st = dist_gcr_residual(D))) return st;  // restart (R13)
        fresh = 0;
        for (int i = 0; i < m && k < D.o.max_iter; ++i) {
            if (!D.gexec[i]) {
                cudaGraph_t graph;
                const long long before = dist_launches(&D, 0);
                CK(cudaStreamBeginCapture(D.stream, cudaStreamCaptureModeThreadLocal));
                const int bst = dist_gcr_step_body(D, i);
                cudaError_t e = cudaStreamEndCapture(D.stream, &graph);
                if (bst) return bst;
                if (e != cudaSuccess) return fail_cuda(e, "dist GCR graph capture");
                D.gkernels[i] = dist_launches(&D, 0) - before;
                D.launches -= D.gkernels[i];
                e = cudaGraphInstantiate(&D.gexec[i], graph, 0);
                cudaGraphDestroy(graph);
                if (e != cudaSuccess) { D.gexec[i] = nullptr; return fail_cuda(e, "dist GCR graph instantiate"); }
            }
            CK(cudaGraphLaunch(D.gexec[i], D.stream));
            D.launches += D.gkernels[i];
            if ((st = dsync(D))) return st;
            ++k;
            E = D.hsc[0];
            const double nu2 = D.hsc[1], rr = D.hsc[2];
            if (!(nu2 > 1e-28 * rr)) { status = STOKES_EDIVERGED; break; }  // breakdown (R13)
            if (!(E == E) || isinf(E) || E > 1e6 * E0) { status = STOKES_EDIVERGED; break; }
            if (E <= rtol) {  // exit test on the true residual (R13): else restart from it
                if ((st = dist_gcr_residual(D))) return st;
                CK(cudaMemcpyAsync(D.hsc, D.dscal, 8 * sizeof(double), cudaMemcpyDeviceToHost, D.stream));
                if ((st = dsync(D))) return st;
                fresh = 1;
                if (D.hsc[0] <= rtol) status = STOKES_OK;
                break;
            }
        }
    }
    *iters = k;
    // the true E of x and the mean of x_p for the output de-mean (x halos first)
    if ((st = exchange(D, 0, FX_VP, 0 | (D.pcur << 1)))) return st;
    if ((st = state_E(D, &E))) return st;
    *Eout = E;
    return status;
}

// ---- Anderson acceleration AA(m, beta) (Alg. 5; reading R26) on the tiles
// G = one plain Uzawa iteration of the decomposed solve (its own graph per pressure parity);
// per tile the fused k_aa_push / k_aa_update kernels, their per-CTA partials (the Gram row,
// the sum of the new pressure) in one buffer across the tiles (NCCL: all-gathered), so every
// tile solves the same small system from the same global sums in the same order, and the
// pressure's lazy mean is the global one.  The working state's halos are exchanged after
// every update (the update writes the first ring; the V-cycle reads two).
static int dist_solve_anderson(Dist &D, double rtol, double E0, int *iters, double *Eout) {
    int st;
    const int NR = nranks(D), nbA = aa_blocks(D.tile[0]->lev[0].g);
    const int m = D.o.aa_depth, ns = m + 1;
    if (!D.apart[0])
        for (int b = 0; b < 2; ++b)
            if (cudaMalloc(&D.apart[b], (size_t)nbA * AA_MAXS * NR * sizeof(double)) != cudaSuccess) return STOKES_ENOMEM;
    const int keep = D.pcur;
    for (int q = 0; q < 2; ++q) {  // G(x): the plain Uzawa iteration, one graph per pressure parity
        if (D.aexec[q]) continue;
        D.pcur = q;
        for (int t = 0; t < D.nt; ++t) D.tile[t]->pcur = q;
        cudaGraph_t graph;
        const long long before = dist_launches(&D, 0);
        CK(cudaStreamBeginCapture(D.stream, cudaStreamCaptureModeThreadLocal));
        const int bst = dist_body(D);
        cudaError_t e = cudaStreamEndCapture(D.stream, &graph);
        D.pcur = keep;
        for (int t = 0; t < D.nt; ++t) D.tile[t]->pcur = keep;
        if (bst) return bst;
        if (e != cudaSuccess) return fail_cuda(e, "dist AA graph capture");
        D.akernels = dist_launches(&D, 0) - before;
        D.launches -= D.akernels;
        e = cudaGraphInstantiate(&D.aexec[q], graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) { D.aexec[q] = nullptr; return fail_cuda(e, "dist AA graph instantiate"); }
    }
    // T = x^0 (its pressure mean: S_MSHIFT, set by state_E)
    for (int k = 0; k < D.nt; ++k) {
        stokes_s *t = D.tile[k];
        Level &F = t->lev[0];
        const size_t fb = field_doubles(F.g) * 8;
        CK(cudaMemcpyAsync(t->aat.f[0] - COL_OFF, F.vx[0] - COL_OFF, fb, cudaMemcpyDeviceToDevice, D.stream));
        CK(cudaMemcpyAsync(t->aat.f[1] - COL_OFF, F.vy[0] - COL_OFF, fb, cudaMemcpyDeviceToDevice, D.stream));
        CK(cudaMemcpyAsync(t->aat.f[2] - COL_OFF, t->pbuf[D.pcur] - COL_OFF, fb, cudaMemcpyDeviceToDevice, D.stream));
        CK(cudaMemcpyAsync(t->scal + S_AAMT, t->scal + S_MSHIFT, 8, cudaMemcpyDeviceToDevice, D.stream));
    }
    const double inv_np = 1.0 / ((double)D.NX * D.NY);
    double E = E0;
    int k, status = STOKES_NOT_CONVERGED;
    for (k = 0; k < D.o.max_iter; ++k) {
        CK(cudaGraphLaunch(D.aexec[D.pcur], D.stream));  // G(x^k) and E of it
        D.pcur ^= 1;
        for (int t = 0; t < D.nt; ++t) D.tile[t]->pcur = D.pcur;
        D.launches += D.akernels;
        if ((st = dsync(D))) return st;
        E = D.hsc[0];
        if (!(E == E) || isinf(E) || E > 1e6 * E0) { status = STOKES_EDIVERGED; break; }
        if (E <= rtol) { status = STOKES_OK; break; }
        const int slot = k % ns, mk = k < m ? k : m;
        for (int q = 0; q < D.nt; ++q) {
            stokes_s *t = D.tile[q];
            Level &F = t->lev[0];
            AAWin win;
            win.n = mk + 1;
            win.self = mk;
            for (int a = 0; a <= mk; ++a) {
                win.slot[a] = (k - mk + a) % ns;
                win.r[a] = t->aah.R[win.slot[a]];
            }
            const AAVec work{{F.vx[0], F.vy[0], t->pbuf[D.pcur]}};
            launch_aa_push(ctx(t), F.g, work, t->scal + S_MSHIFT, t->aat, t->scal + S_AAMT, t->aah.G[slot],
                           t->aah.R[slot], win, D.apart[0] + (size_t)(D.mode == M_NCCL ? D.rank : q) * nbA * AA_MAXS);
        }
        if ((st = gather_segments(D, D.apart[0], (size_t)nbA * AA_MAXS))) return st;
        for (int q = 0; q < D.nt; ++q) {
            stokes_s *t = D.tile[q];
            Level &F = t->lev[0];
            AAWin win;
            win.n = mk + 1;
            win.self = mk;
            for (int a = 0; a <= mk; ++a) {
                win.slot[a] = (k - mk + a) % ns;
                win.r[a] = t->aah.R[win.slot[a]];
            }
            const AAVec work{{F.vx[0], F.vy[0], t->pbuf[D.pcur]}};
            launch_aa_solve(ctx(t), D.apart[0], nbA * NR, win, D.o.aa_beta, t->aaH, t->aacg, t->aacr);
            launch_aa_update(ctx(t), F.g, t->aah, ns, t->aacg, t->aacr, work, t->aat,
                             D.apart[1] + (size_t)(D.mode == M_NCCL ? D.rank : q) * nbA * AA_MAXS);
        }
        // the update's partial sums of the new pressure: nbA per tile, gathered densely
        if (D.mode == M_NCCL || D.mode == M_NCCL_SELF) {
            // (segments are nbA * AA_MAXS apart; the first nbA doubles of each hold the sums)
            if ((st = gather_segments(D, D.apart[1], (size_t)nbA * AA_MAXS))) return st;
        }
        for (int q = 0; q < D.nt; ++q) {
            stokes_s *t = D.tile[q];
            launch_dist_mean(ctx(t), D.apart[1], NR, nbA, (size_t)nbA * AA_MAXS, inv_np, t->scal + S_MSHIFT);
            CK(cudaMemcpyAsync(t->scal + S_AAMT, t->scal + S_MSHIFT, 8, cudaMemcpyDeviceToDevice, D.stream));
        }
        if ((st = exchange(D, 0, FX_VP, 0 | (D.pcur << 1)))) return st;  // both halo rings of x^{k+1}
    }
    if (k >= D.o.max_iter) k = D.o.max_iter - 1;
    *iters = k + 1;
    *Eout = E;
    return status;
}

void drop(Dist &D) {
    for (int k = 0; k < 2; ++k)
        if (D.exec[k]) {
            cudaGraphExecDestroy(D.exec[k]);
            D.exec[k] = nullptr;
        }
    for (int k = 0; k < MAXM; ++k)
        if (D.gexec[k]) {
            cudaGraphExecDestroy(D.gexec[k]);
            D.gexec[k] = nullptr;
        }
    for (int k = 0; k < 2; ++k)
        if (D.aexec[k]) {
            cudaGraphExecDestroy(D.aexec[k]);
            D.aexec[k] = nullptr;
        }
}

// a tile handle: levels 0..La (La = agglomeration staging) with per-side flags
int make_tile(Dist &D, int tx, int ty, stokes_s **out) {
    stokes_s *h = (stokes_s *)calloc(1, sizeof(stokes_s));
    if (!h) return STOKES_ENOMEM;
    h->o = D.o;
    h->o.coarse_direct = 0;
    h->o.accel = D.o.accel;  // GCR / Anderson vectors per tile (carve)
    h->nx = D.nxt;
    h->ny = D.nyt;
    h->Lx = D.Lx * D.nxt / D.NX;
    h->Ly = D.Ly * D.nyt / D.NY;
    memcpy(h->bc, D.bc, sizeof(h->bc));
    h->stream = D.stream;
    h->nlev = D.La + 1;
    for (int l = 0; l <= D.La; ++l) {
        GridL g = make_grid(D.nxt >> l, D.nyt >> l, h->Lx, h->Ly, D.bc);
        g.bN = ty == 0;
        g.bS = ty == D.py - 1;
        g.bW = tx == 0;
        g.bE = tx == D.px - 1;
        g.nvxj = g.bE ? g.ncx - 1 : g.ncx;
        g.nvyi = g.bS ? g.ncy - 1 : g.ncy;
        g.par = (((ty * D.nyt) >> l) + ((tx * D.nxt) >> l)) & 1;
        h->lev[l].g = g;
        h->lev[l].nu = (int)floor(D.o.nu1 * pow(D.o.nu_growth, (double)l) + 0.5);
    }
    Carver dry{nullptr, 0, 0, true};
    const size_t need = carve(h, dry);
    cudaError_t e = cudaMalloc(&h->ws, need);
    if (e != cudaSuccess) { free(h); fail_cuda(e, "cudaMalloc tile"); return STOKES_ENOMEM; }
    h->own_ws = true;
    h->ws_bytes = need;
    Carver cv{(char *)h->ws, 0, need, false};
    carve(h, cv);
    e = cudaMallocHost(&h->hscal, S_NSCAL * sizeof(double));
    if (e == cudaSuccess) e = cudaMemsetAsync(h->ws, 0, need, D.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(D.stream);
    if (e != cudaSuccess) { cudaFree(h->ws); free(h); return fail_cuda(e, "tile init"); }
    *out = h;
    return STOKES_OK;
}
void free_handle(stokes_s *h) {
    if (!h) return;
    drop_graphs(h);
    if (h->hscal) cudaFreeHost(h->hscal);
    if (h->own_ws && h->ws) cudaFree(h->ws);
    free(h);
}

// tile window of a global user-layout array (virtual mode) <-> contiguous tile array
// kind: 0 vx ny x (nx+1), 1 vy (ny+1) x nx, 2 P ny x nx, 3 basic (ny+1) x (nx+1)
void tile_window(Dist &D, int k, int kind, int &off, int &rows, int &cols, int &gpitch) {
    const int i0 = D.ty[k] * D.nyt, j0 = D.tx[k] * D.nxt;
    switch (kind) {
    case 0: rows = D.nyt; cols = D.nxt + 1; gpitch = D.NX + 1; break;
    case 1: rows = D.nyt + 1; cols = D.nxt; gpitch = D.NX; break;
    case 2: rows = D.nyt; cols = D.nxt; gpitch = D.NX; break;
    default: rows = D.nyt + 1; cols = D.nxt + 1; gpitch = D.NX + 1; break;
    }
    off = i0 * gpitch + j0;
}
// copy the tile-k window of a user array into tmp (virtual) or pass the rank's array through
const double *window_in(Dist &D, int k, int kind, const double *u, double *tmp) {
    if (D.mode == M_NCCL) return u;
    int off, rows, cols, gp;
    tile_window(D, k, kind, off, rows, cols, gp);
    cudaMemcpy2DAsync(tmp, (size_t)cols * 8, u + off, (size_t)gp * 8, (size_t)cols * 8, rows, cudaMemcpyDeviceToDevice,
                      D.stream);
    return tmp;
}
void window_out(Dist &D, int k, int kind, const double *tmp, double *u) {
    int off, rows, cols, gp;
    tile_window(D, k, kind, off, rows, cols, gp);
    cudaMemcpy2DAsync(u + off, (size_t)gp * 8, tmp, (size_t)cols * 8, (size_t)cols * 8, rows, cudaMemcpyDeviceToDevice,
                      D.stream);
}
// scratch for windows: a tile's level-0 GCR-free buffers large enough for a user array
double *tmp_of(stokes_s *t, int which) { return which == 0 ? t->lev[0].bx - COL_OFF : t->lev[0].by - COL_OFF; }

}  // namespace

// ====================================================================== dist entry points
int dist_num_levels(Dist *D) { return D->L; }
long long dist_launches(Dist *D, int reset) {
    long long n = D->launches + D->tail->launches;
    for (int k = 0; k < D->nt; ++k) n += D->tile[k]->launches;
    if (reset) {
        D->launches = 0;
        D->tail->launches = 0;
        for (int k = 0; k < D->nt; ++k) D->tile[k]->launches = 0;
    }
    return n;
}

int dist_destroy(Dist *D) {
    drop(*D);
    for (int k = 0; k < D->nt; ++k) free_handle(D->tile[k]);
    free_handle(D->tail);
    if ((D->mode == M_NCCL || D->mode == M_NCCL_SELF) && D->comm) ncclCommDestroy(D->comm);
    free(D->nlog);
    for (int k = 0; k < MAXT; ++k) {
        if (D->sb[k]) cudaFree(D->sb[k]);
        if (D->rb[k]) cudaFree(D->rb[k]);
    }
    if (D->dscal) cudaFree(D->dscal);
    if (D->hsc) cudaFreeHost(D->hsc);
    for (int k = 0; k < 3; ++k)
        if (D->gpart[k]) cudaFree(D->gpart[k]);
    for (int k = 0; k < 2; ++k)
        if (D->apart[k]) cudaFree(D->apart[k]);
    if (D->own_stream) cudaStreamDestroy(D->stream);
    if (D->cstream) cudaStreamDestroy(D->cstream);
    for (int k = 0; k < 2; ++k)
        if (D->ev[k]) cudaEventDestroy(D->ev[k]);
    free(D);
    return STOKES_OK;
}

int dist_set_viscosity(Dist *D, const double *eta_b, const double *eta_p) {
    for (int k = 0; k < D->nt; ++k) {
        stokes_s *t = D->tile[k];
        Level &F = t->lev[0];
        const LaunchCtx c = ctx(t);
        launch_in_b(c, F.g, window_in(*D, k, 3, eta_b, tmp_of(t, 0)), F.etab);
        launch_in_p(c, F.g, window_in(*D, k, 2, eta_p, tmp_of(t, 1)), F.etap);
    }
    int st;
    if ((st = exchange(*D, 0, FX_ETA, 0))) return st;
    if (D->o.theta_step > 0.0)  // the caller's field (halos included) for the rescaling stages
        for (int k = 0; k < D->nt; ++k) {
            stokes_s *t = D->tile[k];
            Level &F = t->lev[0];
            CK(cudaMemcpyAsync(fstart(F.g, t->etab_user), fstart(F.g, F.etab), fsize(F.g) * 8, cudaMemcpyDeviceToDevice,
                               D->stream));
            CK(cudaMemcpyAsync(fstart(F.g, t->etap_user), fstart(F.g, F.etap), fsize(F.g) * 8, cudaMemcpyDeviceToDevice,
                               D->stream));
        }
    if ((st = dist_eta_hierarchy(D))) return st;
    if ((st = dsync(*D))) return st;
    D->have_eta = true;
    drop(*D);
    if (D->have_rho) return force_E(*D);
    return STOKES_OK;
}
// coarse viscosities of the tiles (halos per level), the agglomerated tail's hierarchy and
// coarsest inverse, GCR energy weights -- from the tiles' current level-0 eta (halos valid)
int dist_eta_hierarchy(Dist *D) {
    int st;
    for (int l = 0; l < D->La; ++l) {  // a7 on the tiles, halos refreshed per level
        for (int k = 0; k < D->nt; ++k) {
            stokes_s *t = D->tile[k];
            launch_restrict_b(ctx(t), t->lev[l].g, t->lev[l + 1].g, t->lev[l].etab, t->lev[l + 1].etab);
            launch_restrict_p(ctx(t), t->lev[l].g, t->lev[l + 1].g, t->lev[l].etap, t->lev[l + 1].etap);
        }
        if ((st = exchange(*D, l + 1, FX_ETA, 0))) return st;
    }
    if ((st = gather_to_tail(*D, 1))) return st;
    if ((st = build_hierarchy(D->tail))) return st;  // tail: coarse eta + coarsest inverse
    if (D->o.accel == STOKES_ACCEL_GCR)  // GCR energy weights at each tile's unknowns
        for (int k = 0; k < D->nt; ++k) {
            stokes_s *t = D->tile[k];
            Level &F = t->lev[0];
            launch_energy_weights(ctx(t), F.g, F.etab, F.etap, t->gew[0], t->gew[1], t->gew[2]);
        }
    return STOKES_OK;
}

int dist_set_density(Dist *D, const double *rho_b) {
    for (int k = 0; k < D->nt; ++k) {
        stokes_s *t = D->tile[k];
        launch_in_b(ctx(t), t->lev[0].g, window_in(*D, k, 3, rho_b, tmp_of(t, 0)), t->rho);
    }
    int st;
    if ((st = exchange(*D, 0, FX_RHO, 0))) return st;
    D->have_rho = true;
    drop(*D);
    if (D->have_eta) return force_E(*D);
    return dsync(*D);
}

int dist_set_gravity(Dist *D, double gx, double gy) {
    D->gx = gx;
    D->gy = gy;
    for (int k = 0; k < D->nt; ++k) {
        D->tile[k]->gx = gx;
        D->tile[k]->gy = gy;
    }
    drop(*D);
    if (D->have_eta && D->have_rho) return force_E(*D);
    return STOKES_OK;
}

static int load_state(Dist *D, const double *vx, const double *vy, const double *p) {
    for (int k = 0; k < D->nt; ++k) {
        stokes_s *t = D->tile[k];
        Level &F = t->lev[0];
        const LaunchCtx c = ctx(t);
        launch_in_velocity(c, F.g, window_in(*D, k, 0, vx, tmp_of(t, 0)), window_in(*D, k, 1, vy, tmp_of(t, 1)),
                           F.vx[0], F.vy[0]);
        launch_in_p(c, F.g, window_in(*D, k, 2, p, F.rx - COL_OFF), t->pbuf[0]);
        CK(cudaMemsetAsync(t->scal + S_MSHIFT, 0, 8, D->stream));
    }
    D->pcur = 0;
    for (int k = 0; k < D->nt; ++k) D->tile[k]->pcur = 0;
    int st;
    if ((st = exchange(*D, 0, FX_V, 0))) return st;
    return exchange(*D, 0, FX_P, 0);
}

int dist_residual_energy(Dist *D, const double *vx, const double *vy, const double *p, double *E) {
    if (!D->have_eta || !D->have_rho) return STOKES_ESTATE;
    int st = load_state(D, vx, vy, p);
    if (st) return st;
    return state_E(*D, E);
}

static int dist_core(Dist *D, double rtol, double E0, int *kout, double *Eout) {
    int st, k = 0, status = STOKES_OK;
    double E = E0;
    if (E0 > rtol && D->o.accel == STOKES_ACCEL_GCR) {
        status = dist_solve_gcr(*D, rtol, E0, &k, &E);
        if (status < 0 && status != STOKES_EDIVERGED) return status;
    } else if (E0 > rtol && D->o.accel == STOKES_ACCEL_ANDERSON) {
        status = dist_solve_anderson(*D, rtol, E0, &k, &E);
        if (status < 0 && status != STOKES_EDIVERGED) return status;
    } else if (E0 > rtol) {
        status = STOKES_NOT_CONVERGED;
        const int keep = D->pcur;
        const bool fused = dist_fused_ok(*D);
        for (int q = 0; q < 2; ++q) {  // capture one iteration per pressure parity
            if (D->exec[q]) continue;
            D->pcur = q;
            for (int t = 0; t < D->nt; ++t) D->tile[t]->pcur = q;
            cudaGraph_t graph;
            const long long before = dist_launches(D, 0);
            if (D->dry && (st = nc_log(*D, NC_BODY, q, 0, -1, -1))) return st;
            CK(cudaStreamBeginCapture(D->stream, cudaStreamCaptureModeThreadLocal));
            int bst = fused ? dist_fused_body(*D) : dist_body(*D);
            cudaError_t e = cudaStreamEndCapture(D->stream, &graph);
            if (D->dry && !bst && (st = nc_log(*D, NC_BODY_END, q, 0, -1, -1))) return st;
            D->pcur = keep;
            for (int t = 0; t < D->nt; ++t) D->tile[t]->pcur = keep;
            if (bst) return bst;
            if (e != cudaSuccess) return fail_cuda(e, "dist graph capture");
            D->body_kernels = dist_launches(D, 0) - before;
            D->launches -= D->body_kernels;  // captured, not executed
            e = cudaGraphInstantiate(&D->exec[q], graph, 0);
            cudaGraphDestroy(graph);
            if (e != cudaSuccess) { D->exec[q] = nullptr; return fail_cuda(e, "dist graph instantiate"); }
        }
        if (fused && D->o.max_iter >= 1) {
            // iteration 1: a full V-cycle from (v^0, p^0), then the fused tail of iterate 1;
            // iteration k+1: the captured rest of V-cycle k+1 + the fused tail
            if ((st = dvcycle(*D, 0, true, false))) return st;
            if ((st = dist_fused_tail(*D))) return st;
            for (k = 1;; ) {
                D->pcur ^= 1;  // pbuf[pcur] = p^k
                for (int t = 0; t < D->nt; ++t) D->tile[t]->pcur = D->pcur;
                if ((st = dsync(*D))) return st;
                E = D->hsc[0];
                if (!(E == E) || isinf(E) || E > 1e6 * E0) { status = STOKES_EDIVERGED; break; }
                if (E <= rtol) { status = STOKES_OK; break; }
                if (k >= D->o.max_iter) break;
                ++k;
                CK(cudaGraphLaunch(D->exec[D->pcur], D->stream));
                D->launches += D->body_kernels;
            }
        } else {
            for (k = 1; k <= D->o.max_iter; ++k) {
                CK(cudaGraphLaunch(D->exec[D->pcur], D->stream));
                D->pcur ^= 1;
                for (int t = 0; t < D->nt; ++t) D->tile[t]->pcur = D->pcur;
                D->launches += D->body_kernels;
                if ((st = dsync(*D))) return st;
                E = D->hsc[0];
                if (!(E == E) || isinf(E) || E > 1e6 * E0) { status = STOKES_EDIVERGED; break; }
                if (E <= rtol) { status = STOKES_OK; break; }
            }
            if (k > D->o.max_iter) k = D->o.max_iter;
        }
    }
    *kout = k;
    *Eout = E;
    return status;
}

// eta_min over both caller fields of every tile (reading R24) -> each tile's S_ETAMIN
// (positive doubles order as their bit patterns: atomicMin / ncclMin on uint64)
static int dist_eta_min(Dist &D) {
    const unsigned long long big = 0x7ff0000000000000ull;  // +inf
    unsigned long long *m0 = reinterpret_cast<unsigned long long *>(D.tile[0]->scal + S_ETAMIN);
    CK(cudaMemcpyAsync(m0, &big, 8, cudaMemcpyHostToDevice, D.stream));
    for (int k = 0; k < D.nt; ++k) {
        stokes_s *t = D.tile[k];
        launch_eta_min(ctx(t), t->lev[0].g, t->etab_user, t->etap_user, m0);
    }
    if (D.mode == M_NCCL)
        if (int st = nc_allreduce(D, m0, 1, ncclUint64, ncclMin, D.stream)) return st;
    if (D.mode == M_NCCL_SELF)
        if (ncclAllReduce(m0, m0, 1, ncclUint64, ncclMin, D.comm, D.stream) != ncclSuccess) return STOKES_ENCCL;
    for (int k = 1; k < D.nt; ++k)
        CK(cudaMemcpyAsync(D.tile[k]->scal + S_ETAMIN, m0, 8, cudaMemcpyDeviceToDevice, D.stream));
    CK(cudaStreamSynchronize(D.stream));  // (the host constant `big` is stack memory)
    return STOKES_OK;
}
static int dist_set_theta(Dist &D, double theta) {  // eta = (1 - theta) eta_min + theta eta_user
    for (int k = 0; k < D.nt; ++k) {
        stokes_s *t = D.tile[k];
        Level &F = t->lev[0];
        launch_eta_blend(ctx(t), F.g, t->etab_user, t->etap_user, F.etab, F.etap,
                         reinterpret_cast<const unsigned long long *>(t->scal + S_ETAMIN), theta);
    }
    int st = exchange(D, 0, FX_ETA, 0);
    if (st) return st;
    return dist_eta_hierarchy(&D);
}
// the staged solve of solve_staged (driver.cu) on the tiles: stages theta = 0, step, ... < 1 of
// theta_every iterations each (no stopping test), then theta = 1 to E <= rtol
static int dist_solve_staged(Dist *D, double rtol, int *iters, double *Eout) {
    const int budget = D->o.max_iter;
    int used = 0, it = 0, st = 0, status = STOKES_OK;
    double E = 0.0, E0 = 0.0;
    if ((st = dist_eta_min(*D))) return st;
    for (int k = 0;; ++k) {
        const double theta = k * D->o.theta_step;
        if (theta >= 1.0 || used >= budget) break;
        if ((st = dist_set_theta(*D, theta))) return st;
        if ((st = force_E(*D))) return st;
        if ((st = state_E(*D, &E0))) return st;
        D->o.max_iter = budget - used < D->o.theta_every ? budget - used : D->o.theta_every;
        status = dist_core(D, -1.0, E0, &it, &E);
        D->o.max_iter = budget;
        if (status < 0 && status != STOKES_EDIVERGED) return status;
        used += it;
        if (status == STOKES_EDIVERGED) break;
    }
    if ((st = dist_set_theta(*D, 1.0))) return st;
    if ((st = force_E(*D))) return st;
    if (status != STOKES_EDIVERGED && used < budget) {
        if ((st = state_E(*D, &E0))) return st;
        if (E0 <= rtol) {
            E = E0;
            status = STOKES_OK;
        } else {
            D->o.max_iter = budget - used;
            status = dist_core(D, rtol, E0, &it, &E);
            D->o.max_iter = budget;
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

int dist_solve(Dist *D, double rtol, double *vx, double *vy, double *p, int *iters, double *Eout) {
    NVTX_RANGE("dist_solve");
    if (!D->have_eta || !D->have_rho) return STOKES_ESTATE;
    int st = load_state(D, vx, vy, p);
    if (st) return st;
    CK(cudaMemcpyAsync(D->hsc + 8, D->dscal + 3, 8, cudaMemcpyDeviceToHost, D->stream));
    if ((st = dsync(*D))) return st;
    int status = STOKES_OK;
    double E0 = 0.0, E = 0.0;
    int k = 0;
    if (!(D->hsc[8] > 0)) {  // f == 0
        *iters = 0;
        *Eout = 0.0;
        for (int q = 0; q < D->nt; ++q) {
            stokes_s *t = D->tile[q];
            CK(cudaMemsetAsync(fstart(t->lev[0].g, t->lev[0].vx[0]), 0, fsize(t->lev[0].g) * 8, D->stream));
            CK(cudaMemsetAsync(fstart(t->lev[0].g, t->lev[0].vy[0]), 0, fsize(t->lev[0].g) * 8, D->stream));
            CK(cudaMemsetAsync(fstart(t->lev[0].g, t->pbuf[0]), 0, fsize(t->lev[0].g) * 8, D->stream));
            CK(cudaMemsetAsync(t->scal + S_MSHIFT, 0, 8, D->stream));
        }
    } else {
        if (D->o.theta_step > 0.0) {  // viscosity-rescaling stages (reading R24)
            status = dist_solve_staged(D, rtol, &k, &E);
            if (status < 0 && status != STOKES_EDIVERGED) return status;
        } else {
            if ((st = state_E(*D, &E0))) return st;
            E = E0;
            if (E0 > rtol) {
                status = dist_core(D, rtol, E0, &k, &E);
                if (status < 0 && status != STOKES_EDIVERGED) return status;
            }
        }
        *iters = k;
        *Eout = E;
    }
    for (int q = 0; q < D->nt; ++q) {  // outputs (zero-mean p through each tile's mshift)
        stokes_s *t = D->tile[q];
        Level &F = t->lev[0];
        const LaunchCtx c = ctx(t);
        if (D->mode == M_NCCL) {
            launch_out_vx(c, F.g, F.vx[0], vx);
            launch_out_vy(c, F.g, F.vy[0], vy);
            launch_out_p(c, F.g, t->pbuf[D->pcur], p, t->scal + S_MSHIFT);
        } else {
            launch_out_vx(c, F.g, F.vx[0], tmp_of(t, 0));
            window_out(*D, q, 0, tmp_of(t, 0), vx);
            launch_out_vy(c, F.g, F.vy[0], tmp_of(t, 1));
            window_out(*D, q, 1, tmp_of(t, 1), vy);
            launch_out_p(c, F.g, t->pbuf[D->pcur], F.rx - COL_OFF, t->scal + S_MSHIFT);
            window_out(*D, q, 2, F.rx - COL_OFF, p);
        }
    }
    if ((st = dsync(*D))) return st;
    return status;
}

extern "C" {

int stokes_dist_schedule(stokes_t h, long long *rec, int cap, int *n) {
    if (!h || !h->dist || !h->dist->dry || !n || cap < 0 || (cap > 0 && !rec)) return STOKES_EINVAL;
    const Dist &D = *h->dist;
    *n = D.nlog_n;
    const int m = D.nlog_n < cap ? D.nlog_n : cap;
    if (m) memcpy(rec, D.nlog, (size_t)m * NC_REC * sizeof(long long));
    return STOKES_OK;
}

int stokes_nccl_unique_id(void *id128) {
    if (!id128) return STOKES_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return STOKES_ENCCL;
    memcpy(id128, &id, sizeof(id) < 128 ? sizeof(id) : 128);
    return STOKES_OK;
}

int stokes_create_dist(int nx, int ny, double Lx, double Ly, const int bc[4], int px, int py, int rank,
                       const void *nccl_unique_id, const stokes_opts *opts, void *cuda_stream, stokes_t *out) {
    if (!out || px < 1 || py < 1 || px * py > MAXT || nx % px || ny % py || !bc) return STOKES_EINVAL;
    if (rank >= px * py || rank < -3) return STOKES_EINVAL;
    if (opts && opts->smoother >= 2) return STOKES_EINVAL;  // RAS / Mixed: single domain only
    Dist *D = (Dist *)calloc(1, sizeof(Dist));
    if (!D) return STOKES_ENOMEM;
    D->NX = nx;
    D->NY = ny;
    D->px = px;
    D->py = py;
    D->nxt = nx / px;
    D->nyt = ny / py;
    D->Lx = Lx;
    D->Ly = Ly;
    memcpy(D->bc, bc, sizeof(D->bc));
    if (opts) D->o = *opts;
    else stokes_opts_default(&D->o);
    if (check_opts(D->o) || !(Lx > 0) || !(Ly > 0)) { free(D); return STOKES_EINVAL; }
    for (int k = 0; k < 4; ++k)
        if (bc[k] != 0 && bc[k] != 1) { free(D); return STOKES_EINVAL; }
    D->rank = rank;
    D->mode = rank >= 0 ? M_NCCL : (rank == -2 ? M_LOOPBACK : (rank == -3 ? M_NCCL_SELF : M_VIRTUAL));
    {
        const char *e = getenv("STOKES_HALO_2PHASE");
        D->halo2 = e && e[0] == '1';
    }
    // global hierarchy and the agglomeration level (tile levels while the tile is >= dmin)
    GridL gs[MAXLEV];
    int nus[MAXLEV];
    D->L = build_levels(nx, ny, Lx, Ly, bc, D->o, gs, nus);
    // distribute while tiles are >= dmin cells: NCCL exchanges cost ~10-30 us each, so the
    // multi-GPU default agglomerates at 512-cell tiles (the redundant global tail is then a
    // ~1024 x 512 grid at 8 GPUs); in-process transports keep more levels distributed
    int dmin = D->mode == M_NCCL ? 512 : 64;
    if (const char *e = getenv("STOKES_DIST_DMIN")) dmin = atoi(e) > 2 ? atoi(e) : 2;
    int La = 0;
    while (La + 1 <= D->L - 1) {
        const int cx = D->nxt >> La, cy = D->nyt >> La;
        if ((cx % 2) || (cy % 2) || (cx < dmin) || (cy < dmin)) break;
        ++La;
    }
    if (La < 1) { free(D); return STOKES_EINVAL; }  // tiles too small / not coarsenable
    D->La = La;
    D->stream = (cudaStream_t)cuda_stream;
    if (!D->stream) {
        if (cudaStreamCreateWithFlags(&D->stream, cudaStreamNonBlocking) != cudaSuccess) { free(D); return STOKES_ECUDA; }
        D->own_stream = true;
    }
    D->xs = D->stream;
    if (cudaStreamCreateWithFlags(&D->cstream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&D->ev[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&D->ev[1], cudaEventDisableTiming) != cudaSuccess) {
        free(D);
        return STOKES_ECUDA;
    }
    {   // overlap the halo exchange with the interior: on by default with one tile per GPU
        // (NCCL transport: the exchange latency is what it hides); off for the in-process
        // transports, whose tiles share one GPU (nothing to hide, the split only adds launches).
        // STOKES_DIST_OVERLAP = 0 off, 1 on, 2 split passes with the exchange not overlapped
        const char *e = getenv("STOKES_DIST_OVERLAP");
        D->overlap = e ? e[0] != '0' : D->mode == M_NCCL;
        // a split pass costs ~12 us (boundary-strip launches, the interior on 4 fewer SMs;
        // measured on one B200) against the ~30 us of the two NCCL rounds it
        // hides: worth it only where the interior part outlasts the exchange -- tile levels
        // >= 1024 cells wide (pass >= 72 us).  STOKES_OVERLAP_MIN overrides.
        const char *m = getenv("STOKES_OVERLAP_MIN");
        D->overlap_min = m ? atoi(m) : (e ? 0 : 1024);
        D->serial_split = e && e[0] == '2';
    }
    int st;
    if (D->mode != M_NCCL) {
        D->nt = px * py;
        for (int k = 0; k < D->nt; ++k) {
            D->tx[k] = k % px;
            D->ty[k] = k / px;
        }
    } else {
        D->nt = 1;
        D->tx[0] = rank % px;
        D->ty[0] = rank / px;
        D->dry = !nccl_unique_id;  // schedule-recording dry run: no communicator
        if (!D->dry) {
            ncclUniqueId id;
            memcpy(&id, nccl_unique_id, sizeof(id));
            if (ncclCommInitRank(&D->comm, px * py, id, rank) != ncclSuccess) { free(D); return STOKES_ENCCL; }
        }
    }
    if (D->mode == M_NCCL_SELF) {  // a one-rank communicator: every halo goes through ncclSend / ncclRecv to self
        ncclUniqueId id;
        if (ncclGetUniqueId(&id) != ncclSuccess || ncclCommInitRank(&D->comm, 1, id, 0) != ncclSuccess) {
            free(D);
            return STOKES_ENCCL;
        }
    }
    for (int k = 0; k < D->nt; ++k)
        if ((st = make_tile(*D, D->tx[k], D->ty[k], &D->tile[k]))) { dist_destroy(D); return st; }
    // the coarse tail: global level La
    stokes_opts ot = D->o;
    stokes_t tail = nullptr;
    st = stokes_create(nx >> La, ny >> La, Lx, Ly, bc, &ot, D->stream, nullptr, 0, &tail);
    if (st) { dist_destroy(D); return st; }
    D->tail = tail;
    for (int l = 0; l < tail->nlev; ++l) tail->lev[l].nu = (int)floor(D->o.nu1 * pow(D->o.nu_growth, (double)(La + l)) + 0.5);
    if (D->tail->nlev + La != D->L) { dist_destroy(D); return STOKES_EINVAL; }
    const GridL &gf = D->tile[0]->lev[0].g, &gc = D->tile[0]->lev[La].g;
    // packed halos: 3 fields x HW x (the W / E columns over ncy + 2 HW rows, the N / S rows over
    // ncx + 2 HW columns, the four HW x HW corners); agglomeration blocks
    const size_t nhalo = 3 * HW * (2 * (size_t)(gf.ncy + 2 * HW) + 2 * (size_t)(gf.ncx + 2 * HW) + 4 * HW);
    const size_t nagg = 2 * (size_t)(gc.ncy + 1) * (gc.ncx + 1) * (size_t)(px * py);
    D->nbuf = (nhalo > nagg ? nhalo : nagg) + 64;
    bool okm = cudaMalloc(&D->dscal, 64 * 8) == cudaSuccess && cudaMallocHost(&D->hsc, 64 * 8) == cudaSuccess;
    const int nbufs = (D->mode == M_LOOPBACK || D->mode == M_NCCL_SELF) ? D->nt : 1;
    for (int k = 0; k < nbufs && okm; ++k)
        okm = cudaMalloc(&D->sb[k], D->nbuf * 8) == cudaSuccess && cudaMalloc(&D->rb[k], D->nbuf * 8) == cudaSuccess;
    if (!okm) {
        dist_destroy(D);
        return STOKES_ENOMEM;
    }
    cudaMemsetAsync(D->dscal, 0, 64 * 8, D->stream);
    if ((st = dsync(*D))) { dist_destroy(D); return st; }
    stokes_s *h = (stokes_s *)calloc(1, sizeof(stokes_s));
    h->dist = D;
    cudaGetDevice(&h->device);
    h->nx = nx;
    h->ny = ny;
    h->stream = D->stream;
    *out = h;
    return STOKES_OK;
}

}  // extern "C"
