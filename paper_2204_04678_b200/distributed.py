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

Failures never desynchronise the ranks: every rank takes part in every
collective whatever its local slots did, and the lowest failed slot is
raised as ``BatchError`` on every rank after the gather.
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


def agree_failed_slot(failed, k, group=None):
    """Collective: the lowest slot any rank reports failed (``failed`` = this
    rank's lowest failed slot or None), or None when every slot succeeded."""
    import torch
    import torch.distributed as dist

    dev = (torch.device("cuda", torch.cuda.current_device())
           if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    t = torch.tensor([k if failed is None else int(failed)], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    v = int(t.item())
    return None if v >= k else v


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

    def _gather_rows(self, rows, per):
        """all_gather a [r, per] float64 block per rank -> [world, r, per]."""
        torch = self.torch
        buf = rows.to(self.device)
        gathered = [torch.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(gathered, buf, group=self.group)
        self.n_exchanges += 1
        return torch.stack(gathered).cpu().numpy()

    def _raise_failed(self, k, G_flag, local_err):
        """After the gather: the lowest failed slot (if any) is raised as
        BatchError on EVERY rank (the reference's run_batch contract,
        runtime.py:167-173), with the local exception on the owning rank."""
        failed = [s for s in range(k) if G_flag[s % self.world, s // self.world] != 0.0]
        if not failed:
            return
        s = min(failed)
        if s % self.world == self.rank and local_err is not None:
            cause = local_err.task_error if isinstance(local_err, BatchError) else local_err
        else:
            cause = RemoteSlotError(f"slot {s} failed on rank {s % self.world}")
        raise BatchError(s, cause)

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
        buf[1, : len(mine)] = 0.0
        err = None
        if mine:
            # every rank takes part in the gather whatever happens locally:
            # a rank that skipped it would leave the others blocked
            try:
                vals = self.obj.eval_batch([points[i] for i in mine])
                buf[0, : len(mine)] = torch.tensor(vals, dtype=torch.float64)
            except BatchError as exc:
                err = exc
                buf[1, exc.slot] = 1.0
            except Exception as exc:  # noqa: BLE001 - re-raised after the gather
                err = exc
                buf[1, 0] = 1.0
        G = self._gather_rows(buf, per)  # [world, 2, per]
        self._raise_failed(k, G[:, 1, :], err)
        return [float(G[s % self.world, 0, s // self.world]) for s in range(k)]

    def _broadcast_mode(self, slot, local_modes, mine):
        """The conditional mode of ``slot`` from the rank that evaluated it
        (one broadcast of n doubles; collective: every rank calls it)."""
        torch = self.torch
        owner = slot % self.world
        src = owner if self.group is None else self.dist.get_global_rank(self.group, owner)
        n = self.obj.ev.n
        if owner == self.rank:
            buf = torch.as_tensor(np.ascontiguousarray(local_modes[mine.index(slot)]),
                                  dtype=torch.float64).to(self.device)
        else:
            buf = torch.empty(n, dtype=torch.float64, device=self.device)
        self.dist.broadcast(buf, src=src, group=self.group)
        return buf.cpu().numpy()

    def _eval_planned(self, points):
        """Objectives with the plan / eval_subset / finish protocol
        (fit.FitObjective): per-point warm starts are planned identically on
        every rank; the slot results (f, log det, iterations) are all-gathered.
        Conditional modes cross ranks only where the host state needs them:
        all of an FD stencil's (the mode sensitivity D, identical on every
        rank), and the accepted point's, fetched lazily from its owner when
        the optimizer accepts it (``finish(..., fetch=...)``).  Results do not
        depend on the GPU count."""
        torch = self.torch
        k = len(points)
        pts, warm, st = self.obj.plan(points)
        mine = list(range(self.rank, k, self.world))
        per = math.ceil(k / self.world)
        buf = torch.full((4, per), float("nan"), dtype=torch.float64)
        buf[3, : len(mine)] = 0.0
        err, modes = None, None
        if mine:
            try:
                f, aux, modes = self.obj.eval_subset(pts, warm, st, mine)
                buf[0, : len(mine)] = torch.tensor(f, dtype=torch.float64)
                buf[1, : len(mine)] = torch.tensor([a[0] for a in aux], dtype=torch.float64)
                buf[2, : len(mine)] = torch.tensor([float(a[1]) for a in aux], dtype=torch.float64)
            except Exception as exc:  # noqa: BLE001 - re-raised after the gather
                err = exc
                buf[3, 0] = 1.0
        G = self._gather_rows(buf, per)  # [world, 4, per]
        self._raise_failed(k, G[:, 3, :], err)
        out = [float(G[s % self.world, 0, s // self.world]) for s in range(k)]
        aux_all = [(float(G[s % self.world, 1, s // self.world]), int(G[s % self.world, 2, s // self.world]))
                   for s in range(k)]
        full, fetch = None, None
        if st is not None:
            n = self.obj.ev.n
            mb = torch.zeros((per, n), dtype=torch.float64)
            if mine:
                mb[: len(mine)] = torch.as_tensor(modes)
            GM = self._gather_rows(mb, per)  # [world, per, n]
            full = np.stack([GM[s % self.world, s // self.world] for s in range(k)])
        elif self.obj.wants_modes(st):
            local = modes

            def fetch(slot, _local=local, _mine=mine):
                return self._broadcast_mode(slot, _local, _mine)
        self.obj.finish(pts, warm, st, out, aux_all, full, fetch=fetch)
        return out
