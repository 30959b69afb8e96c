"""theta sharding over ranks (gloo, world_size 2, CPU): slot-ordered
results identical to a single-process batch, lowest failing slot."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class CountingObjective:
    def __init__(self, rank, fail_at=None):
        self.rank = rank
        self.seen = []
        self.fail_at = fail_at

    def eval_batch(self, pts):
        from paper_2204_04678_b200.errors import BatchError

        out = []
        for j, p in enumerate(pts):
            self.seen.append(tuple(np.round(p, 12)))
            if self.fail_at is not None and abs(p[0] - self.fail_at) < 1e-12:
                raise BatchError(j, ValueError("bad point"))
            out.append(float(np.sin(p[0]) + p[1] ** 2))
        return out


class RaisingObjective:
    def __init__(self, rank, crash_rank):
        self.rank = rank
        self.crash_rank = crash_rank

    def eval_batch(self, pts):
        if self.rank == self.crash_rank:
            raise RuntimeError("device failure")
        return [float(p[0]) for p in pts]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_04678_b200.distributed import ThetaSharding
    from paper_2204_04678_b200.errors import BatchError
    from paper_2204_04678_b200.optimizer import FDConfig, fd_gradient

    obj = CountingObjective(rank)
    sh = ThetaSharding(obj)
    pts = [np.array([0.1 * k, 0.2 * k]) for k in range(7)]
    vals = sh.eval_batch(pts)
    grad, f0 = fd_gradient(sh, np.array([0.3, 0.4]), FDConfig(scheme="central"))
    bad = ThetaSharding(CountingObjective(rank, fail_at=0.5))
    try:
        bad.eval_batch([np.array([0.1 * k, 0.0]) for k in range(8)])
        slot = None
    except BatchError as e:
        slot = e.slot
    # a non-BatchError exception on ONE rank (e.g. an engine error): every
    # rank still joins the gather and raises BatchError for that slot
    crash = ThetaSharding(RaisingObjective(rank, crash_rank=1))
    try:
        crash.eval_batch([np.array([0.1 * k, 0.0]) for k in range(6)])
        crash_slot = None
    except BatchError as e:
        crash_slot = (e.slot, type(e.task_error).__name__)
    seen = len(obj.seen)
    after = sh.eval_batch(pts[:3])  # the group is still in step
    q.put((rank, vals, grad.tolist(), f0, seen, slot, crash_slot, after))
    dist.destroy_process_group()


def test_two_rank_sharding_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    single = CountingObjective(0)
    pts = [np.array([0.1 * k, 0.2 * k]) for k in range(7)]
    want = single.eval_batch(pts)
    from paper_2204_04678_b200.optimizer import FDConfig, fd_gradient

    g_want, f_want = fd_gradient(lambda t: single.eval_batch([t])[0], np.array([0.3, 0.4]),
                                 FDConfig(scheme="central"))
    for rank, vals, grad, f0, seen, slot, crash_slot, after in res:
        assert vals == want  # bitwise, slot ordered
        assert grad == g_want.tolist() and f0 == f_want
        assert slot == 5  # lowest failing slot (theta[0] == 0.5)
        # rank 1 owns slots 1, 3, 5: its first slot is reported on both ranks
        assert crash_slot[0] == 1
        assert crash_slot[1] == ("RuntimeError" if rank == 1 else "RemoteSlotError")
        assert after == want[:3]
    # each rank evaluated only its share: 4 + 3 of the 7, plus 5-point stencil split 3 + 2
    assert sorted(r[4] for r in res) == [3 + 2, 4 + 3]


class _FakeEv:
    """Evaluator stand-in: modes and f depend on theta and on the warm start
    (like a Newton loop stopped at its tolerance)."""
    n = 3

    class spec:  # hyper_params(theta).theta, as ModelSpec
        @staticmethod
        def hyper_params(th):
            from types import SimpleNamespace

            return SimpleNamespace(theta=np.asarray(th, dtype=np.float64))

    def eval_values(self, pts, warm, want_modes=False):
        from types import SimpleNamespace

        vals, modes = [], []
        for i, p in enumerate(pts):
            w = np.zeros(3) if warm is None else (warm[i] if np.ndim(warm) == 2 else warm)
            x = np.array([np.sin(p[0]), p[1] ** 2, p[0] * p[1]])
            modes.append(x)
            vals.append(SimpleNamespace(f=float(np.cos(p[0]) + p[1] ** 2 + 1e-3 * np.sum(w * w)),
                                        log_gaussian_approx=float(p[0]), timings={"inner_iterations": 2}))
        return (vals, np.array(modes)) if want_modes else vals


def _planned_run(obj_factory, sharded):
    from paper_2204_04678_b200.optimizer import FDConfig, fd_gradient, parallel_line_search, LineSearchConfig

    obj = obj_factory()
    f = sharded(obj) if sharded else obj
    th = np.array([0.3, 0.4])
    obj.accept(th, np.array([np.sin(0.3), 0.16, 0.12]))
    g1, f1 = fd_gradient(f, th, FDConfig(scheme="central"))
    ls = f.eval_batch([th + t * np.array([0.1, -0.2]) for t in (0.5, 1.0, 2.0)])
    acc = obj.approx_for(th + 1.0 * np.array([0.1, -0.2]))
    ex = getattr(f, "n_exchanges", None)
    return ([float(v) for v in g1], float(f1), [float(v) for v in ls], obj.D.tolist(),
            acc.mode.tolist(), float(acc.factor.log_det)), ex


def _planned_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_04678_b200.distributed import ThetaSharding
    from paper_2204_04678_b200.fit import FitObjective

    q.put((rank, _planned_run(lambda: FitObjective(_FakeEv()), ThetaSharding)))
    dist.destroy_process_group()


def test_planned_batches_sharded_match_single_process():
    """FitObjective's sensitivity warm starts: stencil modes are all-gathered,
    so D and every later warm start (hence f) match a single process."""
    from paper_2204_04678_b200.fit import FitObjective

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_planned_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    want, _ = _planned_run(lambda: FitObjective(_FakeEv()), None)
    assert want[3] is not None
    for _, (got, exchanges) in res:
        assert got == want
        # stencil: results + modes; line search: results only (the accepted
        # point's mode is broadcast from its owner on demand)
        assert exchanges == 3


class _FakeSelinvEv:
    """marginal_variances stand-in: deterministic (var, mode) per theta."""
    n = 4

    class spec:
        @staticmethod
        def latent_labels():
            return ["a", "b", "c", "d"]

    def cache_get(self, theta):
        return None

    def __init__(self, scale=1.0):
        self.scale = scale

    def marginal_variances(self, theta, warm=None):
        t = float(np.sum(theta))
        return (np.array([1.0, 2.0, 3.0, 4.0]) * (1.0 + t * t) * self.scale,
                np.array([t, -t, 2 * t, 0.5]))


def _marg_points():
    from paper_2204_04678_b200.marginals import IntegrationPoint

    return [IntegrationPoint(np.array([0.1 * i, -0.05 * i]), np.zeros(2), 0.0, 1.0 / (i + 1))
            for i in range(5)]


def _marg_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_04678_b200.marginals import latent_marginals

    r = latent_marginals(_FakeSelinvEv(), _marg_points(), shard=True)
    # shard=False (independent fits per rank, different data): no exchange,
    # each rank keeps its own result
    own = latent_marginals(_FakeSelinvEv(scale=1.0 + rank), _marg_points()[: 2 + rank])
    q.put((rank, r.latent_mean.tolist(), r.latent_sd.tolist(), own.latent_sd.tolist()))
    dist.destroy_process_group()


def test_latent_marginals_sharded_match_single_process():
    """Integration points sharded over ranks, (mode, var) all-gathered:
    the fixed-order mixture is bitwise the single-process one."""
    from paper_2204_04678_b200.marginals import latent_marginals

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_marg_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    want = latent_marginals(_FakeSelinvEv(), _marg_points())
    for rank, mean, sd, own in res:
        assert mean == want.latent_mean.tolist() and sd == want.latent_sd.tolist()
        mine = latent_marginals(_FakeSelinvEv(scale=1.0 + rank), _marg_points()[: 2 + rank])
        assert own == mine.latent_sd.tolist()
