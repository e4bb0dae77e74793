"""Row-partitioned adaptive s-step CG: host driver.

Three ways to run the partitioned algorithm:

* `solve_partitioned(rows, b, x0, cfg, rank, world, ...)` -- one process per GPU
  (torchrun): this rank builds its slab + ghost zones (partition.py), the
  ranks agree on an NCCL unique id over torch.distributed (plumbing only), and
  the C library runs every outer loop as one CUDA graph containing one grouped
  NCCL halo exchange and one NCCL allreduce.
* `DeviceGroup` -- one process, one rank per listed GPU: the
  communicators come from ncclCommInitAll and one host thread + stream per GPU
  runs that rank's solve; `adaptive_solve(problem, cfg, devices=[...])`.
* `VirtualGroup` -- all ranks' plans in ONE process on one GPU, driven in lock
  step with device copies for the halo and a fixed-order sum for the
  allreduce: the multi-rank kernels and partition exercised on a single GPU.

Every rank computes identical decisions (bitwise-identical reduced Gram), so
the trace returned on each rank is the same.
"""

from __future__ import annotations

import ctypes as C
import hashlib

import numpy as np

from . import _lib as L
from .adaptive import LogBuffers, build_trace, make_config
from .partition import partition_all, partition_rank


def _part_struct(part, rank, world, nccl_id=None, nccl_lib=None):
    keep = dict(
        row_ptr=np.ascontiguousarray(part.row_ptr, dtype=np.int64),
        col_idx=np.ascontiguousarray(part.col_idx, dtype=np.int32),
        values=np.ascontiguousarray(part.values, dtype=np.float64),
        lvl=np.ascontiguousarray(part.lvl_rows, dtype=np.int64),
        peers=np.ascontiguousarray(part.peers, dtype=np.int32),
        so=np.ascontiguousarray(part.send_off, dtype=np.int64),
        ro=np.ascontiguousarray(part.recv_off, dtype=np.int64),
        si=np.ascontiguousarray(part.send_idx, dtype=np.int32),
        ri=np.ascontiguousarray(part.recv_idx, dtype=np.int32),
        gr=np.ascontiguousarray(part.global_rows, dtype=np.int64),
    )
    s = L.SscgPart()
    s.n_own, s.n_rows, s.n_local = part.n_own, part.n_rows, part.n_local
    s.nnz = len(keep["values"])
    s.depth, s.rank, s.world, s.n_peers = part.depth, rank, world, len(part.peers)
    i64 = C.POINTER(C.c_int64)
    s.row_ptr = keep["row_ptr"].ctypes.data_as(i64)
    s.col_idx = L.iptr(keep["col_idx"])
    s.values = L.dptr(keep["values"])
    s.lvl_rows = keep["lvl"].ctypes.data_as(i64)
    s.peer_rank = L.iptr(keep["peers"])
    s.send_off = keep["so"].ctypes.data_as(i64)
    s.recv_off = keep["ro"].ctypes.data_as(i64)
    s.send_idx = L.iptr(keep["si"])
    s.recv_idx = L.iptr(keep["ri"])
    s.global_rows = keep["gr"].ctypes.data_as(i64)
    if nccl_id is not None:
        keep["id"] = C.create_string_buffer(bytes(nccl_id), 128)
        s.nccl_id = C.cast(keep["id"], C.c_void_p)
    s.nccl_lib = nccl_lib.encode() if nccl_lib else None
    return s, keep


class PartPlan:
    """One rank's device plan (owns the sscg_plan handle)."""

    def __init__(self, part, rank, world, device=0, nccl_id=None, nccl_lib=None):
        lib = L.load()
        L.require_device(device)
        s, keep = _part_struct(part, rank, world, nccl_id, nccl_lib)
        h = C.c_void_p()
        L.check(lib.sscg_plan_create_part(C.byref(h), int(device), C.byref(s)))
        self.handle, self.part, self._lib, self._keep = h, part, lib, keep

    def mpk_schedule(self, sigma):
        return L.plan_mpk_schedule(self._lib, self.handle, sigma)

    def collectives(self):
        return L.plan_collectives(self._lib, self.handle)

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self._lib.sscg_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def logs_digest(logs):
    """Hash of everything a rank decided: status, counts, the per-outer
    records (s_bar, s~, s_actual, breaks) and every alpha / beta bit.  Every
    rank of a partitioned solve reduces the same Gram bits and so must take the
    same decisions; a mismatch means the ranks desynchronised."""
    s = logs.s
    h = hashlib.sha256()
    h.update(np.array([s.status, s.total_iters, s.total_outer, s.n_records], np.int64).tobytes())
    nrec = min(int(s.n_records), len(logs.rec_i))
    nit = min(int(s.total_iters), len(logs.iters))
    h.update(np.ascontiguousarray(logs.rec_i[:nrec, :5]).tobytes())
    h.update(np.ascontiguousarray(logs.iters[:nit, :2]).tobytes())
    return h.hexdigest()


class RankMismatch(RuntimeError):
    """The ranks of a partitioned solve did not take identical decisions."""


def check_ranks_agree(digests):
    if len(set(digests)) != 1:
        bad = [r for r, d in enumerate(digests) if d != digests[0]]
        raise RankMismatch(f"ranks {bad} disagree with rank 0 on the solve's decisions "
                           "(s sequence / alphas / counts)")


def _local_vectors(part, b_global, x0_global):
    b = np.ascontiguousarray(b_global[part.row_lo:part.row_hi], dtype=np.float64)
    x0 = np.ascontiguousarray(x0_global[part.global_rows], dtype=np.float64)
    return b, x0


class VirtualGroup:
    """All `world` ranks of a partitioned solve as plans in this process."""

    def __init__(self, rows, world, depth, device=0):
        self.parts = partition_all(rows, world, depth)
        self.plans = [PartPlan(p, r, world, device) for r, p in enumerate(self.parts)]
        self.world = world

    def solve(self, problem, cfg):
        cfg, ccfg = make_config(cfg, problem, "fast")
        bs, xs = zip(*[_local_vectors(p, problem.b, problem.x0) for p in self.parts])
        vp = C.c_void_p * self.world
        handles = vp(*[pl.handle.value for pl in self.plans])
        bp = (L._DP * self.world)(*[L.dptr(v) for v in bs])
        xp = (L._DP * self.world)(*[L.dptr(v) for v in xs])
        logs = LogBuffers(cfg)
        L.check(L.load().sscg_vgroup_run(C.cast(handles, C.POINTER(C.c_void_p)), self.world, ccfg,
                                         bp, xp, logs.s))
        x = np.empty(problem.a.n)
        for pl, part in zip(self.plans, self.parts):
            xo = np.empty(part.n_own)
            L.check(L.load().sscg_fetch(pl.handle, L.dptr(xo), None))
            x[part.row_lo:part.row_hi] = xo
        tr, co = build_trace(cfg, logs, "fast")
        return x, tr, co, logs

    def hscg(self, problem, eps_star, max_iters=None, mode="reference"):
        """Distributed HSCG over the group (classic.py:33-104): per iteration
        one halo exchange of p / x and two reductions (sscg_vgroup_hscg)."""
        from .classic import hscg_logs, hscg_trace
        if max_iters is None:
            max_iters = 100 * problem.a.n
        bs, xs = zip(*[_local_vectors(p, problem.b, problem.x0) for p in self.parts])
        vp = C.c_void_p * self.world
        handles = vp(*[pl.handle.value for pl in self.plans])
        bp = (L._DP * self.world)(*[L.dptr(v) for v in bs])
        xp = (L._DP * self.world)(*[L.dptr(v) for v in xs])
        iters, logs = hscg_logs(max_iters)
        L.check(L.load().sscg_vgroup_hscg(C.cast(handles, C.POINTER(C.c_void_p)), self.world, bp,
                                          xp, float(eps_star), int(max_iters),
                                          L.HSCG_MODES[mode], logs))
        x = np.empty(problem.a.n)
        for pl, part in zip(self.plans, self.parts):
            xo = np.empty(part.n_own)
            L.check(L.load().sscg_fetch(pl.handle, L.dptr(xo), None))
            x[part.row_lo:part.row_hi] = xo
        tr, co = hscg_trace(iters, logs)
        return x, tr, co


def hscg_partitioned(rows, b_global, x0_global, eps_star, rank, world, device, exchange,
                     broadcast_bytes, max_iters=None, mode="production", nccl_lib=None, info=None):
    """This rank's share of a multi-process distributed HSCG (torchrun): a
    depth-1 ghost zone, one NCCL halo exchange and two NCCL allreduces per
    iteration (sscg_hscg_ex on a partitioned plan).  Returns (x_owned, trace,
    coeffs, plan)."""
    from .build import nccl_library
    from .classic import hscg_logs, hscg_trace
    part = partition_rank(rows, rank, world, 1, exchange)
    lib = L.load()
    nccl_lib = nccl_lib or nccl_library()
    uid = None
    if rank == 0:
        buf = C.create_string_buffer(128)
        L.check(lib.sscg_nccl_unique_id(nccl_lib.encode(), buf))
        uid = bytes(buf.raw)
    uid = broadcast_bytes(uid)
    plan = PartPlan(part, rank, world, device, nccl_id=uid, nccl_lib=nccl_lib)
    if max_iters is None:
        max_iters = 100 * rows.n
    b, x0 = _local_vectors(part, b_global, x0_global)
    iters, logs = hscg_logs(max_iters)
    xo = np.empty(part.n_own)
    L.check(lib.sscg_hscg_ex(plan.handle, L.dptr(b), L.dptr(x0), float(eps_star), int(max_iters),
                             L.HSCG_MODES[mode], L.dptr(xo), logs))
    tr, co = hscg_trace(iters, logs)
    if isinstance(info, dict):
        info.update(plan=plan, part=part, logs=logs, iters=iters, b=b, x0=x0,
                    max_iters=int(max_iters), mode=mode)
    return xo, tr, co, plan


class DeviceGroup:
    """A row-partitioned solve over several GPUs from ONE process (SURVEY.md
    5): rank i on devices[i], communicators by ncclCommInitAll, one host
    thread and stream per GPU (sscg_group_create / sscg_group_solve).  The
    plans are built once (cached on the matrix by `adaptive_solve`) and reused
    for every solve with sigma <= depth."""

    def __init__(self, rows, devices, depth, nccl_lib=None):
        from .build import nccl_library
        lib = L.load()
        self.devices = [int(d) for d in devices]
        self.world = len(self.devices)
        if len(set(self.devices)) != self.world:
            raise ValueError("devices must be distinct GPUs")
        for d in self.devices:
            L.require_device(d)
        self.depth = int(depth)
        self.parts = partition_all(rows, self.world, self.depth)
        nccl_lib = nccl_lib or nccl_library()
        structs, self._keep = [], []
        for r, p in enumerate(self.parts):
            st, keep = _part_struct(p, r, self.world, None, nccl_lib)
            structs.append(st)
            self._keep.append(keep)
        arr = (L.SscgPart * self.world)(*structs)
        hs = (C.c_void_p * self.world)()
        devs = np.array(self.devices, dtype=np.int32)
        L.check(lib.sscg_group_create(C.cast(hs, C.POINTER(C.c_void_p)), self.world,
                                      L.iptr(devs), arr))
        self.handles = [C.c_void_p(h) for h in hs]
        self._lib = lib

    def mpk_schedule(self, sigma):
        return [L.plan_mpk_schedule(self._lib, h, sigma) for h in self.handles]

    def collectives(self):
        return [L.plan_collectives(self._lib, h) for h in self.handles]

    def solve(self, problem, cfg, info=None):
        cfg, ccfg = make_config(cfg, problem, "fast")
        if cfg.sigma > self.depth:
            raise ValueError(f"sigma={cfg.sigma} exceeds the group's ghost depth {self.depth}")
        vecs = [_local_vectors(p, problem.b, problem.x0) for p in self.parts]
        xs = [np.empty(p.n_own) for p in self.parts]
        logs = [LogBuffers(cfg) for _ in self.parts]
        w = self.world
        hp = (C.c_void_p * w)(*[h.value for h in self.handles])
        bp = (L._DP * w)(*[L.dptr(v[0]) for v in vecs])
        xp = (L._DP * w)(*[L.dptr(v[1]) for v in vecs])
        op = (L._DP * w)(*[L.dptr(x) for x in xs])
        lp = (C.POINTER(L.SscgLogs) * w)(*[C.pointer(lg.s) for lg in logs])
        L.check(self._lib.sscg_group_solve(C.cast(hp, C.POINTER(C.c_void_p)), w, ccfg, bp, xp,
                                           op, lp))
        check_ranks_agree([logs_digest(lg) for lg in logs])
        x = np.empty(problem.a.n)
        for p, xo in zip(self.parts, xs):
            x[p.row_lo:p.row_hi] = xo
        tr, co = build_trace(cfg, logs[0], "fast")
        if isinstance(info, dict):
            info.update(device_ms=max(lg.s.device_ms for lg in logs), logs=logs[0],
                        outer_launched=logs[0].s.outer_launched, first_gram=logs[0].first_gram)
        return x, tr, co

    def close(self):
        for h in getattr(self, "handles", []):
            if h is not None and h.value:
                self._lib.sscg_plan_destroy(h)
        self.handles = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_partitioned(rows, problem_scalars, b_global, x0_global, cfg, rank, world, device,
                      exchange, broadcast_bytes, nccl_lib=None, info=None):
    """This rank's share of a multi-process partitioned solve (torchrun).

    rows: row access to the global operator (partition.CsrRows / Stencil7Rows);
    exchange(obj) -> list of every rank's obj; broadcast_bytes(b or None) -> the
    128-byte NCCL id from rank 0.  Returns (x_owned, trace, coeffs, plan)."""
    from .build import nccl_library

    depth = cfg.sigma
    part = partition_rank(rows, rank, world, depth, exchange)
    lib = L.load()
    nccl_lib = nccl_lib or nccl_library()
    uid = None
    if rank == 0:
        buf = C.create_string_buffer(128)
        L.check(lib.sscg_nccl_unique_id(nccl_lib.encode(), buf))
        uid = bytes(buf.raw)
    uid = broadcast_bytes(uid)
    plan = PartPlan(part, rank, world, device, nccl_id=uid, nccl_lib=nccl_lib)
    cfg, ccfg = make_config(cfg, problem_scalars, "fast")
    b, x0 = _local_vectors(part, b_global, x0_global)
    logs = LogBuffers(cfg)
    xo = np.empty(part.n_own)
    L.check(lib.sscg_solve(plan.handle, ccfg, L.dptr(b), L.dptr(x0), L.dptr(xo), logs.s))
    # every rank must have taken the same decisions (bitwise-identical reduced
    # Gram); a divergence would desynchronise the halo -- fail loudly
    check_ranks_agree(exchange(logs_digest(logs)))
    tr, co = build_trace(cfg, logs, "fast")
    if isinstance(info, dict):
        info.update(plan=plan, part=part, logs=logs, ccfg=ccfg, b=b, x0=x0)
    return xo, tr, co, plan
