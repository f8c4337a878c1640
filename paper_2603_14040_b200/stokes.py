"""Thin Python binding of libstokes_b200.so (include/stokes.h): argument marshalling only.

Every step of the solve runs in the library's CUDA kernels; PyTorch provides the device
memory (the workspace and the user arrays), the stream and, for distributed runs, the
process group.  There is no CPU fallback: constructing a Stokes object without the CUDA
library or without a GPU raises.

Arrays: torch.float64 CUDA tensors (contiguous) in the user layout of include/stokes.h:
    vx (ny, nx+1), vy (ny+1, nx), p / eta_p (ny, nx), eta_b / rho_b (ny+1, nx+1).
`solve`, `residual`, `vcycle` and `apply_operator` also accept CPU tensors (e.g. pinned):
they are copied to the device on the handle's stream and the results copied back
(marshalling for the end-to-end path).
"""
import ctypes
import os

import torch

from . import build as _build

FREE_SLIP, NO_SLIP = 0, 1
STATUS = {0: "ok", 1: "not converged", -1: "invalid argument", -2: "out of memory", -3: "CUDA error",
          -4: "NCCL error", -5: "diverged", -6: "call order"}
OK, NOT_CONVERGED, EINVAL, ENOMEM, ECUDA, ENCCL, EDIVERGED, ESTATE = 0, 1, -1, -2, -3, -4, -5, -6

_lib = None


class StokesError(RuntimeError):
    def __init__(self, status, what):
        extra = ""
        if _lib is not None:
            extra = _lib.stokes_last_error().decode()
        super().__init__(f"{what}: {STATUS.get(status, status)} ({status}) {extra}".strip())
        self.status = status


class Opts(ctypes.Structure):
    """stokes_opts (field order = ABI)."""
    _fields_ = [
        ("smoother", ctypes.c_int),
        ("omega_v", ctypes.c_double),
        ("alpha_p", ctypes.c_double),
        ("nu1", ctypes.c_int),
        ("nu_growth", ctypes.c_double),
        ("coarse_min", ctypes.c_int),
        ("coarse_direct", ctypes.c_int),
        ("vcycles_per_iter", ctypes.c_int),
        ("accel", ctypes.c_int),
        ("gcr_restart", ctypes.c_int),
        ("max_iter", ctypes.c_int),
        ("pressure_sign", ctypes.c_int),
        ("theta_step", ctypes.c_double),
        ("theta_every", ctypes.c_int),
        ("aa_depth", ctypes.c_int),
        ("aa_beta", ctypes.c_double),
        ("ras_tile", ctypes.c_int),
        ("ras_inner", ctypes.c_int),
        ("ras_seed", ctypes.c_uint64),
        ("gcr_true_restart", ctypes.c_int),
    ]


def lib(build_if_missing=True):
    """Load libstokes_b200.so (in-tree).  Raises if it cannot be loaded."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("STOKES_LIB", _build.LIB)  # experiments: an alternative build of the library
    if not os.path.exists(path):
        if not build_if_missing:
            raise RuntimeError(f"{path} missing: run paper_2603_14040_b200/build.py (nvcc, sm_100a)")
        _build.build()
    L = ctypes.CDLL(path)
    P, I, D, S = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
    pi, pd = ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)
    sig = {
        "stokes_opts_default": [ctypes.POINTER(Opts)],
        "stokes_workspace_bytes": [I, I, ctypes.POINTER(Opts), ctypes.POINTER(S)],
        "stokes_create": [I, I, D, D, pi, ctypes.POINTER(Opts), P, P, S, ctypes.POINTER(P)],
        "stokes_destroy": [P],
        "stokes_num_levels": [P, pi],
        "stokes_level_shape": [P, I, pi, pi, pi],
        "stokes_set_viscosity": [P, P, P],
        "stokes_set_density": [P, P],
        "stokes_set_gravity": [P, D, D],
        "stokes_apply_operator": [P, P, P, P, P, P, P],
        "stokes_residual": [P, P, P, P, P, P, P, pd],
        "stokes_vcycle": [P, P, P, P, P],
        "stokes_solve": [P, D, P, P, P, pi, pd],
        "stokes_solve_hist": [P, D, P, P, P, pi, pd, pd, I],
        "stokes_smooth": [P, I, P, P, P, P, I],
        "stokes_level_residual": [P, I, P, P, P, P, P, P],
        "stokes_restrict": [P, I, I, P, P],
        "stokes_prolong": [P, I, P, P, P, P],
        "stokes_get_viscosity": [P, I, P, P],
        "stokes_coarse_solve": [P, P, P, P, P],
        "stokes_launch_count": [P, ctypes.POINTER(ctypes.c_longlong), I],
        "stokes_time_kernel": [P, I, I, pd, pd],
        "stokes_strerror": [I],
        "stokes_last_error": [],
        "stokes_create_dist": [I, I, D, D, pi, I, I, I, P, ctypes.POINTER(Opts), P, ctypes.POINTER(P)],
        "stokes_nccl_unique_id": [P],
        "stokes_dist_schedule": [P, ctypes.POINTER(ctypes.c_longlong), I, ctypes.POINTER(I)],
        "stokes_lithostatic": [P, P],
        "stokes_markers_to_grid": [P, ctypes.c_longlong, P, P, P, P, P, P, P, ctypes.POINTER(ctypes.c_longlong)],
        "stokes_grid_to_markers": [P, ctypes.c_longlong, P, P, P, P, P, P],
        "stokes_advect_markers": [P, ctypes.c_longlong, P, P, P, P, D, I, ctypes.POINTER(ctypes.c_longlong)],
        "stokes_marker_timestep": [P, P, P, D, D, pd],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.stokes_strerror.restype = ctypes.c_char_p
    L.stokes_last_error.restype = ctypes.c_char_p
    _lib = L
    return L


EXPORTED = ["stokes_opts_default", "stokes_workspace_bytes", "stokes_create", "stokes_destroy",
            "stokes_num_levels", "stokes_level_shape", "stokes_set_viscosity", "stokes_set_density",
            "stokes_set_gravity", "stokes_apply_operator", "stokes_residual", "stokes_vcycle", "stokes_solve", "stokes_solve_hist",
            "stokes_smooth", "stokes_level_residual", "stokes_restrict", "stokes_prolong",
            "stokes_get_viscosity", "stokes_coarse_solve", "stokes_launch_count", "stokes_time_kernel",
            "stokes_strerror", "stokes_last_error", "stokes_create_dist", "stokes_nccl_unique_id",
            "stokes_dist_schedule", "stokes_lithostatic", "stokes_markers_to_grid", "stokes_grid_to_markers", "stokes_advect_markers",
            "stokes_marker_timestep"]


def default_opts(**kw):
    o = Opts()
    lib().stokes_opts_default(ctypes.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise TypeError(f"unknown option {k!r}")
        setattr(o, k, v)
    return o


def _check(st, what):
    if st < 0:
        raise StokesError(st, what)
    return st


def shapes(nx, ny):
    return {"vx": (ny, nx + 1), "vy": (ny + 1, nx), "p": (ny, nx), "b": (ny + 1, nx + 1)}


class Stokes:
    """One single-GPU solver handle (stokes_create).  Methods mirror the C ABI names."""

    def __init__(self, nx, ny, Lx=1.0, Ly=1.0, bc=(FREE_SLIP,) * 4, device=None, stream=None, **opts):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2603_14040_b200 needs a CUDA GPU (B200, sm_100a); no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.nx, self.ny, self.Lx, self.Ly, self.bc = nx, ny, Lx, Ly, tuple(bc)
        self.opts = default_opts(**opts)
        L = lib()
        nbytes = ctypes.c_size_t()
        _check(L.stokes_workspace_bytes(nx, ny, ctypes.byref(self.opts), ctypes.byref(nbytes)), "workspace_bytes")
        with torch.cuda.device(self.device):
            # a dedicated stream: CUDA graphs cannot be captured on the legacy default stream
            self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
            # torch owns the device memory of the handle (north_star: torch for memory)
            self._ws = torch.empty(nbytes.value + 256, dtype=torch.uint8, device=self.device)
            base = self._ws.data_ptr()
            aligned = (base + 255) // 256 * 256
            self._h = ctypes.c_void_p()
            bcs = (ctypes.c_int * 4)(*self.bc)
            _check(L.stokes_create(nx, ny, float(Lx), float(Ly), bcs, ctypes.byref(self.opts),
                                   ctypes.c_void_p(self.stream.cuda_stream), ctypes.c_void_p(aligned),
                                   nbytes.value, ctypes.byref(self._h)), "create")

    def close(self):
        if getattr(self, "_h", None):
            lib().stokes_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ helpers
    def _dev(self, t, shape=None):
        if t is None:
            return None
        if not torch.is_tensor(t):
            t = torch.as_tensor(t)
        if shape is not None and tuple(t.shape) != tuple(shape):
            raise ValueError(f"expected shape {shape}, got {tuple(t.shape)}")
        if t.dtype != torch.float64:
            raise TypeError("arrays must be torch.float64")
        if t.device != self.device:
            # host (pinned) input: copied on torch's current stream, so every later use on that
            # stream is ordered after it; _sync_inputs() orders the handle's stream after it too
            with torch.cuda.device(self.device):
                t = t.to(self.device, non_blocking=True)
        return t.contiguous()

    def _empty(self, kind, level=0):
        nx, ny, _ = self.level_shape(level)
        return torch.empty(shapes(nx, ny)[kind], dtype=torch.float64, device=self.device)

    @staticmethod
    def _p(t):
        return ctypes.c_void_p(t.data_ptr()) if t is not None else None

    def _sync_outputs(self):
        # results written on the handle's stream must be visible on torch's current stream
        if self.stream != torch.cuda.current_stream(self.device):
            torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def _sync_inputs(self):
        # inputs produced on torch's current stream must be visible on the handle's stream
        if self.stream != torch.cuda.current_stream(self.device):
            self.stream.wait_stream(torch.cuda.current_stream(self.device))

    # ------------------------------------------------------------ shape queries
    @property
    def num_levels(self):
        n = ctypes.c_int()
        _check(lib().stokes_num_levels(self._h, ctypes.byref(n)), "num_levels")
        return n.value

    def level_shape(self, level):
        a, b, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(lib().stokes_level_shape(self._h, level, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)),
               "level_shape")
        return a.value, b.value, c.value

    # ------------------------------------------------------------ setup
    def set_viscosity(self, eta_b, eta_p):
        sh = shapes(self.nx, self.ny)
        eb, ep = self._dev(eta_b, sh["b"]), self._dev(eta_p, sh["p"])
        self._sync_inputs()
        _check(lib().stokes_set_viscosity(self._h, self._p(eb), self._p(ep)), "set_viscosity")

    def set_density(self, rho_b):
        r = self._dev(rho_b, shapes(self.nx, self.ny)["b"])
        self._sync_inputs()
        _check(lib().stokes_set_density(self._h, self._p(r)), "set_density")

    def set_gravity(self, gx, gy):
        _check(lib().stokes_set_gravity(self._h, float(gx), float(gy)), "set_gravity")

    # ------------------------------------------------------------ hot path
    def apply_operator(self, vx, vy, p):
        sh = shapes(self.nx, self.ny)
        vx, vy, p = self._dev(vx, sh["vx"]), self._dev(vy, sh["vy"]), self._dev(p, sh["p"])
        ax, ay, ap = self._empty("vx"), self._empty("vy"), self._empty("p")
        self._sync_inputs()
        _check(lib().stokes_apply_operator(self._h, *map(self._p, (vx, vy, p, ax, ay, ap))), "apply_operator")
        return ax, ay, ap

    def residual(self, vx, vy, p, want_arrays=True):
        sh = shapes(self.nx, self.ny)
        vx, vy, p = self._dev(vx, sh["vx"]), self._dev(vy, sh["vy"]), self._dev(p, sh["p"])
        rx = self._empty("vx") if want_arrays else None
        ry = self._empty("vy") if want_arrays else None
        rp = self._empty("p") if want_arrays else None
        e = ctypes.c_double()
        self._sync_inputs()
        _check(lib().stokes_residual(self._h, *map(self._p, (vx, vy, p, rx, ry, rp)), ctypes.byref(e)), "residual")
        return rx, ry, rp, e.value

    def vcycle(self, bx, by, vx, vy):
        sh = shapes(self.nx, self.ny)
        bx, by = self._dev(bx, sh["vx"]), self._dev(by, sh["vy"])
        vx = self._dev(vx, sh["vx"]).clone()
        vy = self._dev(vy, sh["vy"]).clone()
        self._sync_inputs()
        _check(lib().stokes_vcycle(self._h, *map(self._p, (bx, by, vx, vy))), "vcycle")
        return vx, vy

    def solve(self, rtol, vx=None, vy=None, p=None, out=None, hist_len=0):
        """Solve to E <= rtol.  Returns dict(vx, vy, p, iters, E, status[, hist]).  If the
        initial guess tensors are on the CPU (e.g. pinned), they are copied in and the solution
        is copied back to CPU tensors (`out` may supply pinned output buffers).  hist_len > 0:
        also the energy residual after every iteration (stokes_solve_hist)."""
        sh = shapes(self.nx, self.ny)
        given = [t for t in (vx, vy, p) if t is not None]
        host = bool(given) and not (torch.is_tensor(given[0]) and given[0].is_cuda)
        z = lambda k: torch.zeros(sh[k], dtype=torch.float64, device=self.device)

        def guess(t, k):  # the solve overwrites its initial guess: never the caller's tensor
            if t is None:
                return z(k)
            d = self._dev(t, sh[k])
            return d.clone() if (torch.is_tensor(t) and d.data_ptr() == t.data_ptr()) else d
        with torch.cuda.device(self.device):
            dvx, dvy, dp = guess(vx, "vx"), guess(vy, "vy"), guess(p, "p")
        it, e = ctypes.c_int(), ctypes.c_double()
        self._sync_inputs()
        if hist_len:
            hbuf = (ctypes.c_double * hist_len)()
            st = lib().stokes_solve_hist(self._h, float(rtol), *map(self._p, (dvx, dvy, dp)), ctypes.byref(it),
                                         ctypes.byref(e), hbuf, hist_len)
        else:
            st = lib().stokes_solve(self._h, float(rtol), *map(self._p, (dvx, dvy, dp)), ctypes.byref(it),
                                    ctypes.byref(e))
        if st < 0 and st != EDIVERGED:
            _check(st, "solve")
        res = {"vx": dvx, "vy": dvy, "p": dp, "iters": it.value, "E": e.value, "status": st}
        if hist_len:
            res["hist"] = list(hbuf)[: min(it.value, hist_len)]
        if host:
            with torch.cuda.stream(self.stream):
                for k in ("vx", "vy", "p"):
                    dst = out[k] if out is not None else torch.empty(sh[k], dtype=torch.float64, pin_memory=True)
                    dst.copy_(res[k], non_blocking=True)
                    res[k] = dst
            self.stream.synchronize()
        return res

    # ------------------------------------------------------------ per-step entry points
    def smooth(self, level, bx, by, vx, vy, nsweeps):
        nx, ny, _ = self.level_shape(level)
        sh = shapes(nx, ny)
        bx, by = self._dev(bx, sh["vx"]), self._dev(by, sh["vy"])
        vx, vy = self._dev(vx, sh["vx"]).clone(), self._dev(vy, sh["vy"]).clone()
        self._sync_inputs()
        _check(lib().stokes_smooth(self._h, level, *map(self._p, (bx, by, vx, vy)), nsweeps), "smooth")
        return vx, vy

    def level_residual(self, level, bx, by, vx, vy):
        nx, ny, _ = self.level_shape(level)
        sh = shapes(nx, ny)
        args = [self._dev(a, sh[k]) for a, k in ((bx, "vx"), (by, "vy"), (vx, "vx"), (vy, "vy"))]
        rx, ry = self._empty("vx", level), self._empty("vy", level)
        self._sync_inputs()
        _check(lib().stokes_level_residual(self._h, level, *map(self._p, args), self._p(rx), self._p(ry)),
               "level_residual")
        return rx, ry

    KINDS = {"vx": 0, "vy": 1, "p": 2, "b": 3}

    def restrict(self, level, kind, fine):
        nx, ny, _ = self.level_shape(level)
        fine = self._dev(fine, shapes(nx, ny)[kind])
        coarse = self._empty(kind, level + 1)
        self._sync_inputs()
        _check(lib().stokes_restrict(self._h, level, self.KINDS[kind], self._p(fine), self._p(coarse)), "restrict")
        return coarse

    def prolong(self, level, ex, ey, vx, vy):
        nx, ny, _ = self.level_shape(level)
        cx, cy, _ = self.level_shape(level + 1)
        ex, ey = self._dev(ex, shapes(cx, cy)["vx"]), self._dev(ey, shapes(cx, cy)["vy"])
        vx = self._dev(vx, shapes(nx, ny)["vx"]).clone()
        vy = self._dev(vy, shapes(nx, ny)["vy"]).clone()
        self._sync_inputs()
        _check(lib().stokes_prolong(self._h, level, *map(self._p, (ex, ey, vx, vy))), "prolong")
        return vx, vy

    def get_viscosity(self, level):
        eb, ep = self._empty("b", level), self._empty("p", level)
        _check(lib().stokes_get_viscosity(self._h, level, self._p(eb), self._p(ep)), "get_viscosity")
        return eb, ep

    def coarse_solve(self, bx, by):
        l = self.num_levels - 1
        nx, ny, _ = self.level_shape(l)
        sh = shapes(nx, ny)
        bx, by = self._dev(bx, sh["vx"]), self._dev(by, sh["vy"])
        vx, vy = self._empty("vx", l), self._empty("vy", l)
        self._sync_inputs()
        _check(lib().stokes_coarse_solve(self._h, *map(self._p, (bx, by, vx, vy))), "coarse_solve")
        return vx, vy

    # ------------------------------------------------------------ marker-in-cell (NEXT-4)
    ADVECT = {"euler": 0, "heun": 1, "rk4": 2, "lpi2": 3, "lpi3": 4}

    def _marker(self, t, n=None):
        t = self._dev(t)
        if t.dim() != 1 or (n is not None and t.numel() != n):
            raise ValueError("marker arrays must be 1-D of equal length")
        return t

    def markers_to_grid(self, xm, ym, eta_m, rho_m, count_empty=True):
        """(eta_b, eta_p, rho_b, n_empty) from marker values (R28)."""
        xm = self._marker(xm)
        n = xm.numel()
        ym, eta_m, rho_m = self._marker(ym, n), self._marker(eta_m, n), self._marker(rho_m, n)
        eb, ep, rb = self._empty("b"), self._empty("p"), self._empty("b")
        ne = ctypes.c_longlong(-1)
        self._sync_inputs()
        _check(lib().stokes_markers_to_grid(self._h, n, *map(self._p, (xm, ym, eta_m, rho_m, eb, ep, rb)),
                                            ctypes.byref(ne) if count_empty else None), "markers_to_grid")
        self._sync_outputs()
        return eb, ep, rb, ne.value

    def grid_to_markers(self, xm, ym, vx, vy):
        """velocity at the markers (R29)."""
        sh = shapes(self.nx, self.ny)
        xm = self._marker(xm)
        ym = self._marker(ym, xm.numel())
        vx, vy = self._dev(vx, sh["vx"]), self._dev(vy, sh["vy"])
        um, vm = torch.empty_like(xm), torch.empty_like(xm)
        self._sync_inputs()
        _check(lib().stokes_grid_to_markers(self._h, xm.numel(), *map(self._p, (xm, ym, vx, vy, um, vm))),
               "grid_to_markers")
        self._sync_outputs()
        return um, vm

    def advect_markers(self, xm, ym, vx, vy, dt, scheme="rk4", count_clamped=True):
        """one advection step IN PLACE on (xm, ym) (CUDA float64 tensors of the
        handle's device); returns the number of clamped markers (R30), or -1 if not counted."""
        sh = shapes(self.nx, self.ny)
        for t in (xm, ym):
            if not (torch.is_tensor(t) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
                raise TypeError("advect_markers updates in place: xm, ym must be contiguous CUDA float64 tensors")
        if xm.numel() != ym.numel():
            raise ValueError("xm, ym differ in length")
        vx, vy = self._dev(vx, sh["vx"]), self._dev(vy, sh["vy"])
        nc = ctypes.c_longlong(-1)
        self._sync_inputs()
        _check(lib().stokes_advect_markers(self._h, xm.numel(), *map(self._p, (xm, ym, vx, vy)), float(dt),
                                           self.ADVECT[scheme], ctypes.byref(nc) if count_clamped else None),
               "advect_markers")
        self._sync_outputs()
        return nc.value

    def marker_timestep(self, vx, vy, cfl, max_dt):
        """R31: min(max_dt, cfl min(dx/max|vx|, dy/max|vy|))."""
        sh = shapes(self.nx, self.ny)
        vx, vy = self._dev(vx, sh["vx"]), self._dev(vy, sh["vy"])
        dt = ctypes.c_double()
        self._sync_inputs()
        _check(lib().stokes_marker_timestep(self._h, self._p(vx), self._p(vy), float(cfl), float(max_dt),
                                            ctypes.byref(dt)), "marker_timestep")
        return dt.value

    # ------------------------------------------------------------ instrumentation
    def lithostatic(self):
        """lithostatic pressure p = int_0^y rho g_y dy', the paper's initial
        guess with gravity: pass it as solve(p=...)"""
        p = self._empty("p", 0)
        _check(lib().stokes_lithostatic(self._h, self._p(p)), "lithostatic")
        return p

    def launch_count(self, reset=False):
        c = ctypes.c_longlong()
        _check(lib().stokes_launch_count(self._h, ctypes.byref(c), int(reset)), "launch_count")
        return c.value

    KERNELS = {"jacobi": 0, "energy": 1, "residual_restrict": 2, "prolong": 3, "pupdate": 4, "rbgs": 5,
               "jacobi_uzawa": 6, "jacobi2": 7,
               "ras": 8, "jju": 9}

    def time_kernel(self, kernel, reps=20):
        ms, nb = ctypes.c_double(), ctypes.c_double()
        _check(lib().stokes_time_kernel(self._h, self.KERNELS[kernel], reps, ctypes.byref(ms), ctypes.byref(nb)),
               "time_kernel")
        return ms.value, nb.value


from .decomp import tile_windows  # noqa: E402,F401


def nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    _check(lib().stokes_nccl_unique_id(buf), "nccl_unique_id")
    return buf.raw


class StokesDist(Stokes):
    """2D-decomposed handle (stokes_create_dist).

    rank=None: all px*py tiles in this process on one GPU, arrays are the GLOBAL user-layout
    arrays; transport="virtual" copies halo strips between the tiles directly,
    transport="loopback" runs the NCCL code path's packing / unpacking with device copies
    in place of ncclSend/Recv/AllGather; transport="nccl_self" sends every packed halo through
    real ncclSend / ncclRecv on a one-rank communicator (tests of the multi-GPU path on one B200).
    rank=r (with torch.distributed initialised): NCCL decomposition, one tile per process;
    arrays are the tile windows (`tile_windows`).  The NCCL unique id is created on rank 0
    and broadcast with torch.distributed (the process group is plumbing only).
    rank=r with transport="nccl_dry": the same rank-r handle as a schedule-recording dry run
    (no communicator, no torch.distributed): `schedule()` returns the NCCL calls it would have
    issued (stokes_dist_schedule); the numerical results are meaningless."""

    def __init__(self, nx, ny, Lx=1.0, Ly=1.0, bc=(FREE_SLIP,) * 4, px=1, py=1, rank=None, device=None,
                 stream=None, transport="virtual", **opts):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2603_14040_b200 needs a CUDA GPU (B200, sm_100a); no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.gnx, self.gny, self.px, self.py, self.rank = nx, ny, px, py, rank
        self.nx, self.ny = (nx, ny) if rank is None else (nx // px, ny // py)
        self.Lx, self.Ly, self.bc = Lx, Ly, tuple(bc)
        self.opts = default_opts(**opts)
        uid = None
        if rank is not None and transport != "nccl_dry":
            import torch.distributed as dist
            obj = [nccl_unique_id() if dist.get_rank() == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = ctypes.create_string_buffer(obj[0], 128)
        with torch.cuda.device(self.device):
            self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
            self._h = ctypes.c_void_p()
            bcs = (ctypes.c_int * 4)(*self.bc)
            code = rank if rank is not None else {"virtual": -1, "loopback": -2, "nccl_self": -3}[transport]
            _check(lib().stokes_create_dist(nx, ny, float(Lx), float(Ly), bcs, px, py, code,
                                            uid, ctypes.byref(self.opts), ctypes.c_void_p(self.stream.cuda_stream),
                                            ctypes.byref(self._h)), "create_dist")

    def level_shape(self, level):
        raise NotImplementedError("per-level queries are not available on decomposed handles")

    def schedule(self):
        """Dry-run handles: the recorded NCCL calls, a list of (op, peer, count, dtype, redop)."""
        n = ctypes.c_int()
        _check(lib().stokes_dist_schedule(self._h, None, 0, ctypes.byref(n)), "dist_schedule")
        buf = (ctypes.c_longlong * (5 * max(n.value, 1)))()
        _check(lib().stokes_dist_schedule(self._h, buf, n.value, ctypes.byref(n)), "dist_schedule")
        return [tuple(buf[5 * i:5 * i + 5]) for i in range(n.value)]

    def residual(self, vx, vy, p, want_arrays=False):
        sh = shapes(self.nx, self.ny)
        vx, vy, p = self._dev(vx, sh["vx"]), self._dev(vy, sh["vy"]), self._dev(p, sh["p"])
        e = ctypes.c_double()
        self._sync_inputs()
        _check(lib().stokes_residual(self._h, self._p(vx), self._p(vy), self._p(p), None, None, None,
                                     ctypes.byref(e)), "residual")
        return None, None, None, e.value
