"""Dense assembly of the discrete Stokes saddle operator, written independently of the
oracle (numpy only), directly from the STRESS formulas of PAPER.md:637-661 (stress-
conservative FD, §4.4.2), Eqs. gradient/divergence_discrete and the
ghost-mirror boundary rule.  Used as the pin of the oracle's operator (P1),
of its fixed point (P4, bordered zero-mean LU) and of the smoother algebra (P7).

Unknown ordering: vx (i=1..ny, j=1..nx-1), vy (i=1..ny-1, j=1..nx), p (i=1..ny, j=1..nx),
all row-major on the padded (ny+2) x (nx+2) index space of the paper's arrays.
"""
import numpy as np


class Dense:
    def __init__(self, nx, ny, Lx, Ly, bc, eta_b, eta_p, fold_mirrors=True):
        self.nx, self.ny = nx, ny
        self.dx, self.dy = Lx / nx, Ly / ny
        s = [1.0 if b == 0 else -1.0 for b in bc]  # free slip mirror +, no slip mirror -
        sW, sE, sN, sS = s
        W = nx + 2
        npad = (ny + 2) * W
        self.vx_idx = [(i, j) for i in range(1, ny + 1) for j in range(1, nx)]
        self.vy_idx = [(i, j) for i in range(1, ny) for j in range(1, nx + 1)]
        self.p_idx = [(i, j) for i in range(1, ny + 1) for j in range(1, nx + 1)]
        self.nvx, self.nvy, self.np_ = len(self.vx_idx), len(self.vy_idx), len(self.p_idx)
        n = self.n = self.nvx + self.nvy + self.np_
        Evx = np.zeros((ny + 2, W, n))
        Evy = np.zeros((ny + 2, W, n))
        Ep = np.zeros((ny + 2, W, n))
        for k, (i, j) in enumerate(self.vx_idx):
            Evx[i, j, k] = 1.0
        for k, (i, j) in enumerate(self.vy_idx):
            Evy[i, j, self.nvx + k] = 1.0
        for k, (i, j) in enumerate(self.p_idx):
            Ep[i, j, self.nvx + self.nvy + k] = 1.0
        if fold_mirrors:
            Evx[0, 1:nx] = sN * Evx[1, 1:nx]
            Evx[ny + 1, 1:nx] = sS * Evx[ny, 1:nx]
            Evy[1:ny, 0] = sW * Evy[1:ny, 1]
            Evy[1:ny, nx + 1] = sE * Evy[1:ny, nx]
        dx, dy = self.dx, self.dy
        etaB = np.zeros((ny + 2, W))
        etaB[: ny + 1, : nx + 1] = eta_b
        etaP = np.zeros((ny + 2, W))
        etaP[1 : ny + 1, 1 : nx + 1] = eta_p
        # deviatoric stresses: sxx, syy at P nodes; sxy at basic nodes
        Sxx = np.zeros((ny + 2, W, n))
        Syy = np.zeros((ny + 2, W, n))
        Sxy = np.zeros((ny + 2, W, n))
        for i in range(1, ny + 1):
            for j in range(1, nx + 1):
                Sxx[i, j] = 2 * etaP[i, j] * (Evx[i, j] - Evx[i, j - 1]) / dx
                Syy[i, j] = 2 * etaP[i, j] * (Evy[i, j] - Evy[i - 1, j]) / dy
        for i in range(0, ny + 1):
            for j in range(0, nx + 1):
                Sxy[i, j] = etaB[i, j] * ((Evx[i + 1, j] - Evx[i, j]) / dy + (Evy[i, j + 1] - Evy[i, j]) / dx)
        A = np.zeros((n, n))
        for k, (i, j) in enumerate(self.vx_idx):  # Eq. xmom
            A[k] = ((Sxx[i, j + 1] - Sxx[i, j]) / dx + (Sxy[i, j] - Sxy[i - 1, j]) / dy
                    - (Ep[i, j + 1] - Ep[i, j]) / dx)
        for k, (i, j) in enumerate(self.vy_idx):  # Eq. ymom
            A[self.nvx + k] = ((Syy[i + 1, j] - Syy[i, j]) / dy + (Sxy[i, j] - Sxy[i, j - 1]) / dx
                               - (Ep[i + 1, j] - Ep[i, j]) / dy)
        for k, (i, j) in enumerate(self.p_idx):  # Eq. mass
            A[self.nvx + self.nvy + k] = (Evx[i, j] - Evx[i, j - 1]) / dx + (Evy[i, j] - Evy[i - 1, j]) / dy
        self.A = A
        nv = self.nvx + self.nvy
        self.L = A[:nv, :nv]
        self.G = A[:nv, nv:]
        self.D = A[nv:, :nv]

    # user layout <-> unknown vector ----------------------------------------
    def pack(self, vx, vy, p):
        u = np.zeros(self.n)
        u[: self.nvx] = [vx[i - 1, j] for (i, j) in self.vx_idx]
        u[self.nvx : self.nvx + self.nvy] = [vy[i, j - 1] for (i, j) in self.vy_idx]
        u[self.nvx + self.nvy :] = [p[i - 1, j - 1] for (i, j) in self.p_idx]
        return u

    def pack_v(self, vx, vy):
        return self.pack(vx, vy, np.zeros((self.ny, self.nx)))[: self.nvx + self.nvy]

    def unpack(self, u):
        nx, ny = self.nx, self.ny
        vx = np.zeros((ny, nx + 1))
        vy = np.zeros((ny + 1, nx))
        p = np.zeros((ny, nx))
        for k, (i, j) in enumerate(self.vx_idx):
            vx[i - 1, j] = u[k]
        for k, (i, j) in enumerate(self.vy_idx):
            vy[i, j - 1] = u[self.nvx + k]
        if u.size > self.nvx + self.nvy:
            for k, (i, j) in enumerate(self.p_idx):
                p[i - 1, j - 1] = u[self.nvx + self.nvy + k]
        return vx, vy, p

    def force(self, rho_b, gx, gy):
        """f = -g rho averaged to the velocity node (reading R4/R23)."""
        f = np.zeros(self.n)
        for k, (i, j) in enumerate(self.vx_idx):
            f[k] = -gx * (rho_b[i - 1, j] + rho_b[i, j]) / 2
        for k, (i, j) in enumerate(self.vy_idx):
            f[self.nvx + k] = -gy * (rho_b[i, j - 1] + rho_b[i, j]) / 2
        return f

    def solve_bordered(self, f_full):
        """Exact zero-mean solution of [L G; D 0][v;p] = [f;0]: bordered LU with 1^T p = 0."""
        n = self.n
        B = np.zeros((n + 1, n + 1))
        B[:n, :n] = self.A
        nv = self.nvx + self.nvy
        B[nv:n, n] = 1.0
        B[n, nv:n] = 1.0
        rhs = np.zeros(n + 1)
        rhs[:n] = f_full
        sol = np.linalg.solve(B, rhs)
        return sol[:n]
