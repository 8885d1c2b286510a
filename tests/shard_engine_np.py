"""TEST-ONLY numpy stand-in for a ShardPlan (paper_1811_05571_b200.distributed).

Implements the same phase semantics and exchange-buffer layouts as the CUDA shard plan
(admm_plan.cu enqueue_phase / DESIGN.md §6) with plain numpy, so the production
orchestrator (run_iterations + TorchComm over gloo) can be exercised with world size > 1
on a machine without GPUs.  It is the checker's model of one rank, never product code.
"""
from __future__ import annotations

import numpy as np
import torch

X_GHAT, X_OUTBOX, X_SCAL = 0, 1, 2


def soft(a, kappa):
    mag = np.abs(a)
    out = np.zeros_like(a)
    nz = mag > kappa
    out[nz] = a[nz] * (1.0 - kappa / mag[nz])
    return out


class NumpyShard:
    """One rank: phases 1-4 of admm_plan.cu enqueue_phase including the per-iteration
    objective of a sharded plan (recurrence a_b = (w' + h_b + ghat_b)/2 into the A region,
    rows |sum_q a_iq - g_i|^2 after the gather; two-pass closes iteration k-1's objective in
    iteration k, the sweep closes iteration k's)."""

    def __init__(self, h, g, rho, lam, method, M, N, grid, coords):
        self.Pr, self.Pc = grid
        self.pr, self.pc = coords
        self.rank = self.pr * self.Pc + self.pc
        self.M, self.N = M, N
        self.Mr, self.Nc = M // self.Pr, N // self.Pc
        self.i0, self.j0 = self.pr * self.Mr, self.pc * self.Nc
        m, n = h.shape
        self.mb, self.nb = m // M, n // N
        self.rho, self.lam = rho, lam
        self.kappa = lam / rho if method in ("sectioning", "reference") else lam / (M * rho)
        self.schedule = "sweep" if self.Pr == 1 else "twopass"
        self.g = g
        self.col_bounds = [k * self.nb for k in range(N + 1)]
        self.n_pix = n
        # own blocks and their Woodbury inverses K = (rho I + H H^H)^-1
        self.H, self.K = {}, {}
        for il in range(self.Mr):
            for jl in range(self.Nc):
                i, j = self.i0 + il, self.j0 + jl
                hb = h[i * self.mb:(i + 1) * self.mb, j * self.nb:(j + 1) * self.nb]
                self.H[il, jl] = hb
                self.K[il, jl] = np.linalg.inv(rho * np.eye(self.mb) + hb @ hb.conj().T)
        # exchange buffers (float64 views of complex arrays), slots in rank order.  A ghat
        # slot is [ghat | A region (a_b = H_b v) | fused scalars]; column sharding (Pr == 1)
        # on the sweep schedule carries each rank's 8 scalars in 4 extra complex elements
        # after its slot: one all-gather per iteration (admm_plan.cu).
        self.fused_scal = self.Pr == 1 and self.Pc > 1
        nmv = self.Mr * self.Nc * self.mb
        gslot = 2 * nmv + (4 if self.fused_scal else 0)
        gbuf = np.zeros((self.Pc, gslot), np.complex128)
        self.ghat = gbuf[:, :nmv].reshape(self.Pc, self.Mr, self.Nc, self.mb)
        self.A = gbuf[:, nmv:2 * nmv].reshape(self.Pc, self.Mr, self.Nc, self.mb)
        assert np.shares_memory(self.ghat, gbuf) and np.shares_memory(self.A, gbuf)
        self.outbox = np.zeros((M, self.Nc, self.nb), np.complex128)
        if self.fused_scal:
            self.scal = gbuf[:, 2 * nmv:].view(np.float64)  # [rank == pc][8]
        else:
            self.scal = np.zeros((self.Pr * self.Pc, 8))
        self.buffers = {X_GHAT: torch.from_numpy(gbuf.view(np.float64).reshape(-1)),
                        X_OUTBOX: torch.from_numpy(self.outbox.view(np.float64).reshape(-1))}
        sz = {X_GHAT: gslot * 2, X_OUTBOX: self.Mr * self.Nc * self.nb * 2}
        off = {X_GHAT: self.pc * sz[X_GHAT], X_OUTBOX: self.pr * sz[X_OUTBOX]}
        if not self.fused_scal:
            self.buffers[X_SCAL] = torch.from_numpy(self.scal.reshape(-1))
            sz[X_SCAL], off[X_SCAL] = 8, self.rank * 8
        self.slots = {w: (off[w], sz[w]) for w in sz}
        self.reset()

    def buffer(self, which):
        full = self.buffers[which]
        off, n = self.slots[which]
        return full, full[off:off + n]

    def ghat_of(self, il, q):
        return self.ghat[q // self.Nc, il, q % self.Nc]

    def g_ij(self, il, jl):
        i, j = self.i0 + il, self.j0 + jl
        gij = self.g[i * self.mb:(i + 1) * self.mb].copy()
        for q in range(self.N):
            if q != j:
                gij = gij - self.ghat_of(il, q)
        return gij

    def reset(self):
        z = lambda k: np.zeros(k, np.complex128)  # noqa: E731
        self.u = {b: z(self.nb) for b in self.H}
        self.s = {b: z(self.nb) for b in self.H}
        self.c = {b: z(self.nb) for b in self.H}
        self.q = {b: z(self.mb) for b in self.H}
        self.v = {jl: z(self.nb) for jl in range(self.Nc)}
        self.hs = {b: z(self.mb) for b in self.H}
        self.ghat[...] = 0
        self.A[...] = 0
        self.outbox[:] = 0
        self.trace_rows = []
        self.iter = 0
        self.l1prev = 0.0
        self.objrows = 0.0
        if self.schedule == "sweep":  # prologue: w = H c^0 = 0
            self._k_apply({b: np.zeros(self.mb, np.complex128) for b in self.H})

    def _k_apply(self, w):
        gij = {b: self.g_ij(*b) for b in self.H}  # all from the previous ghat (Jacobi)
        for (il, jl) in self.H:
            q = self.K[il, jl] @ (gij[il, jl] - w[il, jl])
            self.q[il, jl] = q
            self.ghat[self.pc, il, jl] = gij[il, jl] - self.rho * q

    def _column_update(self, count_v):
        rp2 = rd2 = l1 = 0.0
        for jl in range(self.Nc):
            mean = self.outbox[:, jl].sum(axis=0) / self.M
            vn = soft(mean, self.kappa)
            if count_v:
                rd2 += float(np.sum(np.abs(vn - self.v[jl]) ** 2))
                l1 += float(np.sum(np.abs(vn)))
            self.v[jl] = vn
            for il in range(self.Mr):
                u = self.u[il, jl]
                rp2 += float(np.sum(np.abs(u - vn) ** 2))
                self.s[il, jl] = (self.s[il, jl] + u) - vn
                self.c[il, jl] = vn - self.s[il, jl]
        self.scal[self.rank, :4] = [rp2, rd2, l1, 0.0]
        self.scal[self.rank, 4] = 0.0

    def _arec(self, w):
        """a_b = (w' + h_b + ghat_b) / 2, h_b = a_b - w' (ghat_b before this K apply)."""
        for (il, jl) in self.H:
            a = 0.5 * ((w[il, jl] + self.hs[il, jl]) + self.ghat[self.pc, il, jl])
            self.hs[il, jl] = a - w[il, jl]
            self.A[self.pc, il, jl] = a

    def _rows(self):
        """sum over this rank's row blocks of |sum_q a_iq - g_i|^2 (ascending q)."""
        tot = 0.0
        for il in range(self.Mr):
            i = self.i0 + il
            hv = np.zeros(self.mb, np.complex128)
            for q in range(self.N):
                hv = hv + self.A[q // self.Nc, il, q % self.Nc]
            tot += float(np.sum(np.abs(hv - self.g[i * self.mb:(i + 1) * self.mb]) ** 2))
        return tot

    def phase(self, k):
        if k == 1 and self.schedule == "sweep":
            for (il, jl), hb in self.H.items():
                self.u[il, jl] = self.c[il, jl] + hb.conj().T @ self.q[il, jl]
                self.outbox[self.i0 + il, jl] = self.u[il, jl] + self.s[il, jl]
            self._column_update(True)
            w = {b: self.H[b] @ self.c[b] for b in self.H}
            self._arec(w)
            self._k_apply(w)
        elif k == 1:
            w = {b: self.H[b] @ self.c[b] for b in self.H}
            if self.iter >= 1:
                self._arec(w)
            self._k_apply(w)
        elif k == 2:
            for (il, jl), hb in self.H.items():
                self.u[il, jl] = self.c[il, jl] + hb.conj().T @ self.q[il, jl]
                self.outbox[self.i0 + il, jl] = self.u[il, jl] + self.s[il, jl]
        elif k == 3 and self.schedule == "sweep":
            self.objrows = self._rows()  # every rank holds all rows after the gather
        elif k == 3:
            self._column_update(self.pr == 0)
            self.scal[self.rank, 4] = self._rows() if (self.iter >= 1 and self.pc == 0) else 0.0
        elif k == 4:
            a, d, l1 = self.scal[:, 0].sum(), self.scal[:, 1].sum(), self.scal[:, 2].sum()
            row = [np.sqrt(a), np.sqrt(self.rho * self.rho * self.M * d), float("nan")]
            if self.schedule == "sweep":
                row[2] = 0.5 * self.objrows + self.lam * l1
            elif self.iter >= 1:
                self.trace_rows[-1][2] = 0.5 * self.scal[:, 4].sum() + self.lam * self.l1prev
            if self.schedule != "sweep":
                self.l1prev = l1
            self.trace_rows.append(row)
            self.iter += 1

    def segment_v(self):
        return {self.j0 + jl: self.v[jl].copy() for jl in range(self.Nc)}
