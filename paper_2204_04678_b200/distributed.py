"""theta-point sharding over the GPUs of one box (one process per GPU).

The reference parallelises a batch of theta points over threads of one
process (`/root/reference/pkg/src/parinla/runtime.py:134-177`).  Here every
batch — FD stencil, line-search candidates, Hessian stencil, grid wave — is
split over ranks by slot: slot s runs on rank s mod world.  Each rank
evaluates its slots as ONE device batch, then the f values (and a per-slot
status) are exchanged with a single ``all_gather``; every rank ends up with
the identical slot-ordered list, so the host optimizer runs redundantly and
in lockstep on all ranks with no further communication.  The theta batch
is broadcast from rank 0 first so that all ranks provably evaluate the
same points.  This is the path's only exchange step (NCCL over NVLink on
the GPU box; gloo in the CPU tests).

Single-point calls (the serial t-hat evaluation of the line search, the
final f) run on every rank redundantly: they are bitwise identical
because the device kernels are deterministic.
"""

from __future__ import annotations

import math

import numpy as np

from .errors import BatchError, ParinlaError


def shard_info(group=None):
    """(rank, world) of an initialized torch.distributed group, else (0, 1)."""
    try:
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return 0, 1
    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def gather_point_vectors(local, k, n, group=None):
    """Per-point (mode, var) pairs computed on their ranks (point s on rank
    s mod world, ``local`` in that order) -> the full slot-ordered list on
    every rank (one all_gather of 2n doubles per point)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    per = math.ceil(k / world)
    dev = (torch.device("cuda", torch.cuda.current_device())
           if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    buf = torch.zeros((per, 2, n), dtype=torch.float64)
    for j, (mode, var) in enumerate(local):
        buf[j, 0] = torch.as_tensor(mode)
        buf[j, 1] = torch.as_tensor(var)
    buf = buf.to(dev)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    G = torch.stack(out).cpu().numpy()  # [world, per, 2, n]
    return [(G[s % world, s // world, 0], G[s % world, s // world, 1]) for s in range(k)]


class RemoteSlotError(ParinlaError):
    """A slot failed on another rank (its exception type is reported)."""


class ThetaSharding:
    """Wrap a batch objective (``eval_batch(points) -> list[float]``)."""

    def __init__(self, objective, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.obj = objective
        self.group = group
        self.dist = dist
        self.torch = torch
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        backend = dist.get_backend(group)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
        self.device = device
        self.n_exchanges = 0

    @property
    def speculate_t_hat(self):
        return getattr(self.obj, "speculate_t_hat", False)

    @property
    def warm(self):
        return getattr(self.obj, "warm", None)

    @warm.setter
    def warm(self, value):
        self.obj.warm = value

    def __call__(self, theta) -> float:
        return float(self.obj.eval_batch([np.asarray(theta, dtype=np.float64)])[0])

    def _broadcast_points(self, points):
        torch = self.torch
        P = torch.as_tensor(np.stack([np.asarray(p, dtype=np.float64) for p in points]),
                            device=self.device)
        self.dist.broadcast(P, src=0, group=self.group)
        return [row for row in P.cpu().numpy()]

    def eval_batch(self, points):
        torch = self.torch
        k = len(points)
        if k == 0:
            return []
        points = self._broadcast_points(points)
        if hasattr(self.obj, "plan"):
            return self._eval_planned(points)
        mine = list(range(self.rank, k, self.world))
        per = math.ceil(k / self.world)
        buf = torch.full((2, per), float("nan"), dtype=torch.float64)
        err = None
        if mine:
            try:
                vals = self.obj.eval_batch([points[i] for i in mine])
                buf[0, : len(mine)] = torch.tensor(vals, dtype=torch.float64)
                buf[1, : len(mine)] = 0.0
            except BatchError as exc:
                err = exc
                buf[1, : len(mine)] = 0.0
                buf[1, exc.slot] = 1.0
        buf = buf.to(self.device)
        gathered = [torch.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(gathered, buf, group=self.group)
        self.n_exchanges += 1
        G = torch.stack(gathered).cpu().numpy()  # [world, 2, per]
        out, failed = [], []
        for s in range(k):
            r, j = s % self.world, s // self.world
            out.append(float(G[r, 0, j]))
            if G[r, 1, j] != 0.0:
                failed.append(s)
        if failed:
            s = min(failed)
            cause = err.task_error if (err is not None and s % self.world == self.rank) else \
                RemoteSlotError(f"slot {s} failed on rank {s % self.world}")
            raise BatchError(s, cause)
        return out

    def _eval_planned(self, points):
        """Objectives with the plan / eval_subset / finish protocol
        (fit.FitObjective): per-point warm starts are planned identically on
        every rank; the slot results (f, log det, iterations) and, when the
        objective keeps them, the conditional modes are all-gathered, so its
        state (mode sensitivity, recent modes) stays identical on every rank
        and results do not depend on the GPU count."""
        torch = self.torch
        k = len(points)
        pts, warm, st = self.obj.plan(points)
        mine = list(range(self.rank, k, self.world))
        per = math.ceil(k / self.world)
        f, aux, modes = self.obj.eval_subset(pts, warm, st, mine) if mine else ([], [], None)
        buf = torch.full((3, per), float("nan"), dtype=torch.float64)
        if mine:
            buf[0, : len(mine)] = torch.tensor(f, dtype=torch.float64)
            buf[1, : len(mine)] = torch.tensor([a[0] for a in aux], dtype=torch.float64)
            buf[2, : len(mine)] = torch.tensor([float(a[1]) for a in aux], dtype=torch.float64)
        buf = buf.to(self.device)
        gathered = [torch.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(gathered, buf, group=self.group)
        self.n_exchanges += 1
        G = torch.stack(gathered).cpu().numpy()  # [world, 3, per]
        out = [float(G[s % self.world, 0, s // self.world]) for s in range(k)]
        aux_all = [(float(G[s % self.world, 1, s // self.world]), int(G[s % self.world, 2, s // self.world]))
                   for s in range(k)]
        full = None
        if self.obj.wants_modes(st):
            n = self.obj.ev.n
            mb = torch.zeros((per, n), dtype=torch.float64)
            if mine:
                mb[: len(mine)] = torch.as_tensor(modes)
            mb = mb.to(self.device)
            gm = [torch.empty_like(mb) for _ in range(self.world)]
            self.dist.all_gather(gm, mb, group=self.group)
            GM = torch.stack(gm).cpu().numpy()  # [world, per, n]
            full = np.stack([GM[s % self.world, s // self.world] for s in range(k)])
        self.obj.finish(pts, warm, st, out, aux_all, full)
        return out
