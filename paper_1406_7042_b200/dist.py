"""Multi-GPU plumbing: one process per GPU, torch.distributed
for rendezvous and the timing reductions.  The hot path has no data-path
collective: a reduced-hybrid run does not shard without a halo exchange, so
N GPUs run N independent replicas (weak scaling, "replicas only"); only the
timing (max over ranks) and the unit counts (sum over ranks) are reduced.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_world():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def init(backend=None):
    """Initialise the process group from torchrun's environment (no-op for a
    single process).  Returns (rank, world, local_rank)."""
    world, rank, local = env_world()
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def _device():
    if dist.is_initialized() and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def barrier():
    if dist.is_initialized():
        dist.barrier()


def reduce_max(x: float) -> float:
    """Max over ranks (the step time of the slowest rank)."""
    if not dist.is_initialized():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(x: float) -> float:
    if not dist.is_initialized():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def replica_scale(rank: int) -> float:
    """Each replica runs an independent excitation: the source amplitude of
    replica r is scaled by (1 + r/8) (the work per rank is unchanged)."""
    return 1.0 + rank / 8.0


def finalize():
    if dist.is_initialized():
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# Slab decomposition along z with a halo exchange per step
# ---------------------------------------------------------------------------
# The fused E->H stencil advances a PEC-closed box, so a rank's slab is a box
# of its own: its internal faces are (wrong) PEC walls one ghost cell outside
# the cells it owns.  A wall corrupts only the tangential H of the ghost layer
# next to it (that H reads the wall's E = 0); every other unknown of the slab,
# E of the ghost layer included, is updated from correct neighbours as long as
# that ghost H is replaced after every step by the neighbour's value, which
# the neighbour computes as a regular interior unknown.  Slabs therefore
# overlap by two cells and exchange two planes (Hx, Hy) per face and step:
#
#   rank r-1:  ...  | c-1 | c |  wall at c+1        cells c-1, c: the overlap
#   rank r  :  wall at c-1  | c-1 | c | ...
#   r -> r-1: H(c + 1/2)   (local half-plane 1    -> r-1's ghost, local nz'-1)
#   r-1 -> r: H(c - 1/2)   (local half-plane nz'-2 -> r's ghost,  local 0)
#
# The arithmetic of every owned unknown is the single-domain kernel's on the
# same values: a decomposed run is bit-for-bit the undecomposed one
# (tests/test_gpu_slab.py on one GPU; tests/test_dist_gloo.py drives the same
# plan and exchange over gloo with two processes).


class SlabPlan:
    """Host-side plan of a z-slab decomposition of a pure-stencil 3-D problem
    (DESIGN.md §6 dict): cuts, local boxes, local problem descriptions, the
    planes each face exchanges, ownership for gathering."""

    def __init__(self, problem, n_slabs, cuts=None):
        import numpy as np
        if int(problem["dim"]) != 3:
            raise ValueError("slab decomposition: 3-D problems only")
        if problem.get("blocks") or problem.get("interface") is not None:
            raise NotImplementedError("slab decomposition of problems with reduced blocks (cuts must avoid them)")
        self.problem = problem
        self.N = int(n_slabs)
        nx, ny, nz = (int(v) for v in problem["n"])
        self.n = (nx, ny, nz)
        self.plane = (ny + 1) * (nx + 1)
        self.S = self.plane * (nz + 1)
        # cut planes (global z indices), default: even; explicit cuts keep sources out of the overlaps
        self.cuts = [int(round(r * nz / self.N)) for r in range(self.N + 1)] if cuts is None else [int(c) for c in cuts]
        if len(self.cuts) != self.N + 1 or self.cuts[0] != 0 or self.cuts[-1] != nz:
            raise ValueError("slab decomposition: cuts must run from 0 to nz with one entry per slab boundary")
        for r in range(self.N):
            if self.cuts[r + 1] - self.cuts[r] < 3:
                raise ValueError("slab decomposition: every slab needs at least 3 cells along z")
        self.wall_lo = [0 if r == 0 else self.cuts[r] - 1 for r in range(self.N)]
        self.wall_hi = [nz if r == self.N - 1 else self.cuts[r + 1] + 1 for r in range(self.N)]
        self.own_lo = [0 if r == 0 else self.cuts[r] for r in range(self.N)]
        self.own_hi = [nz + 1 if r == self.N - 1 else self.cuts[r + 1] for r in range(self.N)]
        # explicit work (sources) must stay out of the overlap planes, which two ranks update
        src = problem.get("sources")
        if src is not None and len(src["unknown"]):
            k = (np.asarray(src["unknown"], np.int64) % self.S) // self.plane
            for r in range(1, self.N):
                if np.any((k >= self.cuts[r] - 1) & (k <= self.cuts[r] + 1)):
                    raise ValueError(f"slab decomposition: a source lies in the overlap of cut {self.cuts[r]}")

    def nz_local(self, r):
        return self.wall_hi[r] - self.wall_lo[r]

    def owner_of_plane(self, k):
        for r in range(self.N):
            if self.own_lo[r] <= k < self.own_hi[r]:
                return r
        raise ValueError(k)

    def _local_ids(self, ids, r):
        """global unknown ids -> (mask of those rank r owns, their local ids)"""
        import numpy as np
        ids = np.asarray(ids, np.int64)
        comp, s = ids // self.S, ids % self.S
        k, rest = s // self.plane, s % self.plane
        own = (k >= self.own_lo[r]) & (k < self.own_hi[r])
        Sl = self.plane * (self.nz_local(r) + 1)
        return own, comp * Sl + (k - self.wall_lo[r]) * self.plane + rest

    def local_problem(self, r):
        import numpy as np
        p = self.problem
        lo, hi = self.wall_lo[r], self.wall_hi[r]
        out = {k: p[k] for k in ("name", "dim", "delta", "dt", "batch", "precision", "n_steps") if k in p}
        out["n"] = (self.n[0], self.n[1], hi - lo)
        out["interface"], out["blocks"] = None, []
        sl = slice(lo * self.plane, (hi + 1) * self.plane)
        if p.get("mat_id") is not None:
            out["mat_id"] = np.ascontiguousarray(np.asarray(p["mat_id"]).reshape(-1)[sl])
            for key in ("mat_coef", "mat_ifmask", "mat_ca"):
                if p.get(key) is not None:
                    out[key] = p[key]
        else:
            out["mat_id"] = None
            out["uniform_coef"] = p["uniform_coef"]
        init = {}
        for c, a in (p.get("init") or {}).items():
            a = np.asarray(a, np.float64).reshape(-1, self.S)
            init[c] = np.ascontiguousarray(a[:, sl])
        out["init"] = init
        src = p.get("sources")
        out["sources"] = None
        if src is not None and len(src["unknown"]):
            own, lid = self._local_ids(src["unknown"], r)
            if own.any():
                d = dict(unknown=lid[own], coef=np.asarray(src["coef"])[own], wave=src["wave"])
                ncol = np.asarray(src["wave"]).shape[1]
                col = np.asarray(src["column"]) if src.get("column") is not None else np.arange(len(own))
                d["column"] = col[own].astype(np.int32)
                assert d["column"].max() < ncol
                out["sources"] = d
        out["probes"] = []
        self.probe_owner = getattr(self, "probe_owner", {})
        for q, pr in enumerate(p.get("probes") or []):
            own, lid = self._local_ids(pr["unknowns"], r)
            if own.all():
                out["probes"].append(dict(kind=0, unknowns=[int(v) for v in lid], weights=list(pr["weights"])))
                self.probe_owner[q] = (r, len(out["probes"]) - 1)
            elif own.any():
                raise ValueError("slab decomposition: a probe spans two slabs")
        return out

    def faces(self, r):
        """[(neighbour, local half-plane to send, local ghost half-plane to fill)] of rank r"""
        f = []
        if r > 0:
            f.append((r - 1, 1, 0))
        if r < self.N - 1:
            f.append((r + 1, self.nz_local(r) - 2, self.nz_local(r) - 1))
        return f

    def gather(self, local_states):
        """{rank: [B][S_local]} of one component -> the global [B][S] array (owned planes)."""
        import numpy as np
        B = next(iter(local_states.values())).shape[0]
        out = np.zeros((B, self.S))
        for r, a in local_states.items():
            k0, k1 = self.own_lo[r], self.own_hi[r]
            l0 = (k0 - self.wall_lo[r]) * self.plane
            out[:, k0 * self.plane:k1 * self.plane] = a[:, l0:l0 + (k1 - k0) * self.plane]
        return out


EXCHANGED = (3, 4)          # Hx, Hy: the tangential H of a z face


def halo_exchange(rank, faces, send, recv):
    """Swap the face planes with the neighbours over torch.distributed (NCCL on
    GPUs, gloo in the CPU tests).  ``send`` / ``recv``: {neighbour: tensor}."""
    ops = []
    for nb, _, _ in faces:
        ops.append(dist.P2POp(dist.isend, send[nb], nb))
        ops.append(dist.P2POp(dist.irecv, recv[nb], nb))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


class SlabSim:
    """A 3-D pure-stencil problem advanced as z slabs.  With an initialised
    process group of world size > 1 every rank holds one slab and exchanges its
    face planes after each step (device buffers, NCCL); otherwise all
    ``n_slabs`` slabs live in this process and the planes are copied between
    the handles on the stream (the single-GPU functional check)."""

    def __init__(self, problem, n_slabs=None, precision=None, cuts=None, **sim_kw):
        from .fdtd import Sim
        self.multi = dist.is_initialized() and dist.get_world_size() > 1
        self.N = dist.get_world_size() if self.multi else int(n_slabs)
        self.rank = dist.get_rank() if self.multi else None
        self.plan = SlabPlan(problem, self.N, cuts)
        prec = int(precision or problem.get("precision", 64))
        self.dtype = torch.float32 if prec == 32 else torch.float64
        ranks = [self.rank] if self.multi else list(range(self.N))
        self.sims = {r: Sim(self.plan.local_problem(r), precision=prec, graph_steps=0, **sim_kw) for r in ranks}
        nx, ny, _ = self.plan.n
        B = int(problem.get("batch", 1))
        n = (ny + 1) * (nx + 1) * B * len(EXCHANGED)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.buf = {(r, nb, d): torch.empty(n, dtype=self.dtype, device=dev)
                    for r in ranks for nb, _, _ in self.plan.faces(r) for d in ("send", "recv")}
        self.plane_elems = (ny + 1) * (nx + 1) * B
        for r, s in self.sims.items():
            for c, a in (self.plan.local_problem(r).get("init") or {}).items():
                s.set_state(int(c), a)

    def _pack(self, r, nb, k, to_state):
        key = (r, nb, "recv" if to_state else "send")
        t = self.buf[key]
        esz = t.element_size()
        for q, c in enumerate(EXCHANGED):
            self.sims[r].plane_device(c, k, t.data_ptr() + q * self.plane_elems * esz, to_state)

    def step(self, n):
        for _ in range(int(n)):
            for s in self.sims.values():
                s.step(1)
            for r in self.sims:
                for nb, k_send, _ in self.plan.faces(r):
                    self._pack(r, nb, k_send, False)
            if self.multi:
                r = self.rank
                faces = self.plan.faces(r)
                halo_exchange(r, faces, {nb: self.buf[(r, nb, "send")] for nb, _, _ in faces},
                              {nb: self.buf[(r, nb, "recv")] for nb, _, _ in faces})
            else:
                for r in self.sims:
                    for nb, _, _ in self.plan.faces(r):
                        self.buf[(r, nb, "recv")].copy_(self.buf[(nb, r, "send")])
            for r in self.sims:
                for nb, _, k_ghost in self.plan.faces(r):
                    self._pack(r, nb, k_ghost, True)

    def sync(self):
        for s in self.sims.values():
            s.sync()

    def get_state(self, comp):
        """The global component array [B][S] (single-process mode), or this
        rank's owned planes placed in a zero global array (multi-process)."""
        return self.plan.gather({r: s.get_state(comp) for r, s in self.sims.items()})

    def probe(self):
        """Probe series [steps][n_probe][B]; columns of probes owned elsewhere are zero."""
        import numpy as np
        series = {r: s.probe() for r, s in self.sims.items()}
        nprobe = len(self.plan.problem.get("probes") or [])
        steps = max((v.shape[0] for v in series.values()), default=0)
        B = int(self.plan.problem.get("batch", 1))
        out = np.zeros((steps, nprobe, B))
        for q, (r, lq) in self.plan.probe_owner.items():
            if r in series and series[r].size:
                out[:, q, :] = series[r][:, lq, :]
        return out

    def close(self):
        for s in self.sims.values():
            s.close()
