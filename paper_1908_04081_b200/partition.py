"""Row-slab partition with matrix-powers ghost zones.

Host-side setup of a row-partitioned solve (once per matrix and world size):
rank r owns the contiguous global rows [bounds[r], bounds[r+1]).  To run the
s-level matrix-powers recurrence without communication between levels
(communication-avoiding MPK, the [dhmy08] kernel the paper defers to,
PAPER.md:89,131), a rank also holds the ghost rows within graph distance
`depth` of its slab, ordered by distance:

    local rows = [owned | ghost depth 1 | ... | ghost depth D]   (each in global order)

so the rows a level must (redundantly) compute are a prefix of the local rows:
level l produces P_{l+1} on depth <= D-1-l and R_{l+1} on depth <= D-2-l.
Once per outer loop the owners send each neighbour the p, r and x values of the
ghost rows it holds (one grouped exchange), and the only global reduction is
the Gram allreduce.  For 7-point stencils on z-slabs the ghost levels are whole
planes.

`RankPartition` carries exactly what `sscg_plan_create_part` (include/sscg.h)
consumes.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class CsrRows:
    """Row access to a global CSR matrix (a SparseMatrix or the arrays)."""

    def __init__(self, n, row_ptr, col_idx, values):
        self.n = int(n)
        self.row_ptr = np.asarray(row_ptr, dtype=np.int64)
        self.col_idx = np.asarray(col_idx)
        self.values = np.asarray(values, dtype=np.float64)

    @classmethod
    def of(cls, a):
        return cls(a.n, a.row_ptr, a.col_idx, a.values)

    def rows(self, idx):
        """(indptr, global cols, vals) of the rows idx, in the order given."""
        idx = np.asarray(idx, dtype=np.int64)
        starts = self.row_ptr[idx]
        lens = self.row_ptr[idx + 1] - starts
        indptr = np.zeros(len(idx) + 1, dtype=np.int64)
        np.cumsum(lens, out=indptr[1:])
        flat = np.repeat(starts - indptr[:-1], lens) + np.arange(indptr[-1], dtype=np.int64)
        return indptr, self.col_idx[flat].astype(np.int64), self.values[flat]


class Stencil7Rows:
    """Rows of the 7-point Dirichlet Laplacian on nx*ny*nz (x fastest) generated
    on demand: the same values and column order as problems.stencil7, without
    ever materialising the global matrix (for large weak-scaled slabs)."""

    def __init__(self, nx, ny, nz):
        self.nx, self.ny, self.nz = nx, ny, nz
        self.n = nx * ny * nz

    def rows(self, idx):
        idx = np.asarray(idx, dtype=np.int64)
        nx, ny, nz = self.nx, self.ny, self.nz
        ix, iy, iz = idx % nx, (idx // nx) % ny, idx // (nx * ny)
        offs = [(-nx * ny, iz > 0), (-nx, iy > 0), (-1, ix > 0), (0, None),
                (1, ix < nx - 1), (nx, iy < ny - 1), (nx * ny, iz < nz - 1)]
        counts = np.ones(len(idx), dtype=np.int64)
        for _, m in offs:
            if m is not None:
                counts += m
        indptr = np.zeros(len(idx) + 1, dtype=np.int64)
        np.cumsum(counts, out=indptr[1:])
        cols = np.empty(indptr[-1], dtype=np.int64)
        vals = np.empty(indptr[-1], dtype=np.float64)
        pos = indptr[:-1].copy()
        for off, m in offs:
            if m is None:
                cols[pos] = idx
                vals[pos] = 6.0
                pos += 1
            else:
                sel = np.nonzero(m)[0]
                cols[pos[sel]] = idx[sel] + off
                vals[pos[sel]] = -1.0
                pos[sel] += 1
        return indptr, cols, vals


class Varcoef27Rows:
    """Rows of the c4 operator (problems.varcoef27: 27-point variable-coefficient
    diffusion on n^3, lognormal cells, harmonic-mean face weights / |o|^2,
    Dirichlet) generated on demand with the same values, column order and
    rounding, so a rank builds only its slab + ghost planes.  The cell field k
    and the diagonal are global (n^3 doubles each: 57 MB at 192^3); the
    right-hand side is the generator's (`rhs()`).  jacobi=True gives the
    two-sided Jacobi-scaled operator of problems.varcoef27_jacobi."""

    OFFS = [(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]

    def __init__(self, n, sigma_ln=1.5, seed=0, jacobi=False):
        self.m, self.n = n, n ** 3
        rng = np.random.default_rng(seed)
        k = np.exp(rng.normal(0.0, sigma_ln, (n, n, n)))
        b = rng.standard_normal(self.n)
        self._b = b / np.linalg.norm(b)
        self.k = k.ravel()
        self.jacobi = jacobi
        # the diagonal in the generator's accumulation order (offsets in
        # lexicographic order, in-domain w h, out-of-domain w k_i)
        idx = np.arange(n)
        diag = np.zeros((n, n, n))
        for (dz, dy, dx) in self.OFFS:
            if (dz, dy, dx) == (0, 0, 0):
                continue
            m = self._mask3(idx, dz, dy, dx)
            w0 = 1.0 / (dz * dz + dy * dy + dx * dx)
            shifted = np.zeros_like(k)
            sz, sy, sx = (slice(max(0, -d), n - max(0, d)) for d in (dz, dy, dx))
            tz, ty, tx = (slice(max(0, d), n - max(0, -d)) for d in (dz, dy, dx))
            shifted[sz, sy, sx] = k[tz, ty, tx]
            h = np.where(m, 2.0 * k * shifted / np.where(m, k + shifted, 1.0), 0.0)
            diag += np.where(m, w0 * h, w0 * k)
        self.diag = diag.ravel()
        self.root = np.sqrt(self.diag) if jacobi else None

    @staticmethod
    def _mask3(idx, dz, dy, dx):
        n = len(idx)
        mz = (idx + dz >= 0) & (idx + dz < n)
        my = (idx + dy >= 0) & (idx + dy < n)
        mx = (idx + dx >= 0) & (idx + dx < n)
        return mz[:, None, None] & my[None, :, None] & mx[None, None, :]

    def rhs(self):
        return self._b

    def rows(self, idx):
        idx = np.asarray(idx, dtype=np.int64)
        n = self.m
        ix, iy, iz = idx % n, (idx // n) % n, idx // (n * n)
        masks = []
        counts = np.zeros(len(idx), dtype=np.int64)
        for (dz, dy, dx) in self.OFFS:
            m = ((iz + dz >= 0) & (iz + dz < n) & (iy + dy >= 0) & (iy + dy < n) &
                 (ix + dx >= 0) & (ix + dx < n))
            masks.append(m)
            counts += m
        indptr = np.zeros(len(idx) + 1, dtype=np.int64)
        np.cumsum(counts, out=indptr[1:])
        cols = np.empty(indptr[-1], dtype=np.int64)
        vals = np.empty(indptr[-1], dtype=np.float64)
        pos = indptr[:-1].copy()
        for (dz, dy, dx), m in zip(self.OFFS, masks):
            sel = np.nonzero(m)[0]
            rows = idx[sel]
            if (dz, dy, dx) == (0, 0, 0):
                c, v = rows, self.diag[rows]
            else:
                c = rows + (dz * n * n + dy * n + dx)
                w0 = 1.0 / (dz * dz + dy * dy + dx * dx)
                ki, kc = self.k[rows], self.k[c]
                v = -(w0 * (2.0 * ki * kc / (ki + kc)))
            if self.jacobi:  # matio.jacobi_precondition: / (root[min] * root[max])
                v = v / (self.root[np.minimum(rows, c)] * self.root[np.maximum(rows, c)])
            cols[pos[sel]] = c
            vals[pos[sel]] = v
            pos[sel] += 1
        return indptr, cols, vals


def slab_bounds(n, world, align=1):
    """Contiguous row ranges, as equal as possible (multiples of `align`)."""
    units = n // align
    b = [(units * r // world) * align for r in range(world)] + [n]
    return np.array(b, dtype=np.int64)


@dataclass
class RankPartition:
    rank: int
    world: int
    depth: int
    row_lo: int
    row_hi: int
    global_rows: np.ndarray          # local -> global row index
    lvl_rows: np.ndarray             # [depth + 1]
    row_ptr: np.ndarray              # [n_rows + 1] int64
    col_idx: np.ndarray              # [nnz] int32, local
    values: np.ndarray               # [nnz]
    peers: list = field(default_factory=list)
    send_off: np.ndarray = None      # [n_peers + 1]
    recv_off: np.ndarray = None
    send_idx: np.ndarray = None      # local owned rows, grouped by peer
    recv_idx: np.ndarray = None      # local ghost rows, grouped by peer
    requests: dict = field(default_factory=dict)  # owner -> sorted global ghost rows

    @property
    def n_own(self):
        return int(self.lvl_rows[0])

    @property
    def n_rows(self):
        return int(self.lvl_rows[self.depth - 1])

    @property
    def n_local(self):
        return int(self.lvl_rows[self.depth])


def build_local(rows, bounds, rank, depth):
    """Ghost levels (BFS by graph distance), local ordering and local CSR of one
    rank; halo send lists are filled in by `link_halos`."""
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    levels = [np.arange(lo, hi, dtype=np.int64)]
    known = levels[0]
    csr_parts = []
    frontier = levels[0]
    for d in range(1, depth + 1):
        ip, cols, vals = rows.rows(frontier)
        csr_parts.append((ip, cols, vals))
        nxt = np.setdiff1d(np.unique(cols), known, assume_unique=True)
        levels.append(nxt)
        known = np.union1d(known, nxt)
        frontier = nxt
    order = np.concatenate(levels)
    lvl = np.cumsum([len(v) for v in levels]).astype(np.int64)
    # global -> local for every referenced column (all lie in levels 0..depth)
    perm = np.argsort(order, kind="stable")
    sorted_g = order[perm]

    def g2l(g):
        pos = np.searchsorted(sorted_g, g)
        if np.any(pos >= len(sorted_g)) or np.any(sorted_g[np.minimum(pos, len(sorted_g) - 1)] != g):
            raise ValueError("column outside the ghost zone (depth too small?)")
        return perm[pos]

    ptrs, cols_l, vals_l = [np.zeros(1, dtype=np.int64)], [], []
    base = 0
    for ip, cols, vals in csr_parts:  # rows of levels 0 .. depth-1, in local order
        ptrs.append(ip[1:] + base)
        base += ip[-1]
        cols_l.append(g2l(cols).astype(np.int32))
        vals_l.append(vals)
    row_ptr = np.concatenate(ptrs)
    part = RankPartition(
        rank=rank, world=len(bounds) - 1, depth=depth, row_lo=lo, row_hi=hi,
        global_rows=order, lvl_rows=lvl, row_ptr=row_ptr,
        col_idx=np.concatenate(cols_l) if cols_l else np.zeros(0, np.int32),
        values=np.concatenate(vals_l) if vals_l else np.zeros(0))
    # ghost rows grouped by owner, global order inside each group
    ghosts = order[lvl[0]:]
    owners = np.searchsorted(bounds, ghosts, side="right") - 1
    for q in np.unique(owners):
        g = np.sort(ghosts[owners == q])
        part.requests[int(q)] = g
    return part


def link_halos(parts_requests, part):
    """Fill send/recv lists of `part` given every rank's ghost requests
    (parts_requests[r] = {owner: sorted global rows r needs from owner})."""
    me = part.rank
    recv_from = sorted(part.requests)
    send_to = sorted(r for r, req in enumerate(parts_requests) if r != me and me in req)
    peers = sorted(set(recv_from) | set(send_to))
    order = part.global_rows
    perm = np.argsort(order, kind="stable")
    sorted_g = order[perm]
    send_idx, recv_idx, so, ro = [], [], [0], [0]
    for q in peers:
        want = parts_requests[q].get(me, np.zeros(0, np.int64)) if q != me else np.zeros(0, np.int64)
        send_idx.append((np.asarray(want) - part.row_lo).astype(np.int32))
        so.append(so[-1] + len(want))
        got = part.requests.get(q, np.zeros(0, np.int64))
        recv_idx.append(perm[np.searchsorted(sorted_g, got)].astype(np.int32))
        ro.append(ro[-1] + len(got))
    part.peers = peers
    part.send_off = np.array(so, dtype=np.int64)
    part.recv_off = np.array(ro, dtype=np.int64)
    part.send_idx = np.concatenate(send_idx) if send_idx else np.zeros(0, np.int32)
    part.recv_idx = np.concatenate(recv_idx) if recv_idx else np.zeros(0, np.int32)
    return part


def partition_all(rows, world, depth, align=1):
    """Every rank's partition in one process (virtual groups, tests)."""
    bounds = slab_bounds(rows.n, world, align)
    parts = [build_local(rows, bounds, r, depth) for r in range(world)]
    reqs = [p.requests for p in parts]
    return [link_halos(reqs, p) for p in parts]


def partition_rank(rows, rank, world, depth, exchange, align=1):
    """This rank's partition in a multi-process job: `exchange(obj)` must return
    the list of every rank's obj (torch.distributed.all_gather_object)."""
    bounds = slab_bounds(rows.n, world, align)
    part = build_local(rows, bounds, rank, depth)
    reqs = exchange(part.requests)
    return link_halos(reqs, part)
