"""Level-1 batch dispatch and budgets.

Mirrors the reference runtime surface (`/root/reference/pkg/src/parinla/
runtime.py:22-177`): ``ThreadBudget``, ``SERIAL``, ``parse_budget``,
``default_budget``, ``run_batch`` with slot-ordered results and lowest-slot
error reporting, plus the runtime counters.

On B200 the level-2 (separator-tree task) parallelism of the reference is
replaced by the tile-DAG kernels inside one GPU, and the level-1 parallelism
over theta points is carried by *batched* objective calls: an objective that
exposes ``eval_batch(points) -> list[float]`` receives the whole slot list in
one call (all slots run concurrently on the device, and across ranks when a
:class:`~.distributed.ThetaSharding` is attached).  Plain callables still go
through a thread pool exactly like the reference.
"""

from __future__ import annotations

import os
import threading
import time
from concurrent.futures import FIRST_EXCEPTION, ThreadPoolExecutor, wait
from dataclasses import dataclass
from typing import Callable, Sequence

from .errors import BatchError, BudgetError


@dataclass(frozen=True)
class ThreadBudget:
    """``l1`` concurrent theta slots, ``l2`` inner workers (kept for API parity)."""

    l1: int = 1
    l2: int = 1

    def __post_init__(self):
        if self.l1 < 1 or self.l2 < 1:
            raise BudgetError(f"budget must be at least 1:1, got {self.l1}:{self.l2}")

    def __str__(self) -> str:
        return f"{self.l1}:{self.l2}"


SERIAL = ThreadBudget(1, 1)


def parse_budget(text: str) -> ThreadBudget:
    """``"A:B"`` -> ThreadBudget(A, B) (reference `runtime.py:40-49`)."""
    parts = text.strip().split(":")
    if len(parts) != 2 or not all(parts):
        raise BudgetError(f"expected 'A:B', got {text!r}")
    try:
        return ThreadBudget(int(parts[0]), int(parts[1]))
    except ValueError:
        raise BudgetError(f"expected integer 'A:B', got {text!r}") from None


def physical_cores() -> int:
    try:
        import psutil

        n = psutil.cpu_count(logical=False)
        if n:
            return int(n)
    except Exception:
        pass
    return os.cpu_count() or 1


def default_budget(n_hyper: int, cores: int | None = None) -> ThreadBudget:
    """l1 = min(2d+1, cores), l2 = cores // l1 (reference `runtime.py:64-71`)."""
    cores = physical_cores() if cores is None else cores
    l1 = max(1, min(2 * max(n_hyper, 1) + 1, cores))
    return ThreadBudget(l1, max(1, cores // l1))


class _Stats:
    def __init__(self):
        self._lock = threading.Lock()
        self.reset()

    def reset(self):
        with getattr(self, "_lock", threading.Lock()):
            self.batch_active = 0
            self.batch_peak = 0
            self.tree_peak = 0
            self.n_batches = 0
            self.batch_wall_s = 0.0
            self.device_batches = 0
            self.device_slots = 0

    def enter(self, k: int = 1):
        with self._lock:
            self.batch_active += k
            self.batch_peak = max(self.batch_peak, self.batch_active)

    def leave(self, k: int = 1):
        with self._lock:
            self.batch_active -= k

    def record(self, wall: float, device_slots: int = 0):
        with self._lock:
            self.n_batches += 1
            self.batch_wall_s += wall
            if device_slots:
                self.device_batches += 1
                self.device_slots += device_slots

    def snapshot(self) -> dict:
        with self._lock:
            return {
                "batch_peak": self.batch_peak,
                "tree_peak": self.tree_peak,
                "n_batches": self.n_batches,
                "batch_wall_s": self.batch_wall_s,
                "device_batches": self.device_batches,
                "device_slots": self.device_slots,
            }


_stats = _Stats()


def runtime_stats() -> dict:
    return _stats.snapshot()


def reset_runtime_stats():
    _stats.reset()


def run_batch(tasks: Sequence[Callable[[], object]], budget: ThreadBudget) -> list:
    """Run independent zero-argument tasks; results in slot order.

    At most ``budget.l1`` in flight; the lowest failing slot is reported as
    ``BatchError(slot)`` and unstarted tasks are cancelled.
    """
    t0 = time.perf_counter()
    out = [None] * len(tasks)
    if budget.l1 == 1 or len(tasks) <= 1:
        for slot, task in enumerate(tasks):
            _stats.enter()
            try:
                out[slot] = task()
            except BaseException as exc:
                raise BatchError(slot, exc) from exc
            finally:
                _stats.leave()
        _stats.record(time.perf_counter() - t0)
        return out

    def wrapped(task):
        _stats.enter()
        try:
            return task()
        finally:
            _stats.leave()

    with ThreadPoolExecutor(max_workers=budget.l1) as pool:
        futs = [pool.submit(wrapped, t) for t in tasks]
        done, pending = wait(futs, return_when=FIRST_EXCEPTION)
        bad = [i for i, f in enumerate(futs) if f in done and f.exception() is not None]
        if bad:
            for f in pending:
                f.cancel()
            slot = min(bad)
            raise BatchError(slot, futs[slot].exception()) from futs[slot].exception()
        for slot, f in enumerate(futs):
            out[slot] = f.result()
    _stats.record(time.perf_counter() - t0)
    return out


def eval_points(f, points: Sequence, budget: ThreadBudget) -> list[float]:
    """Evaluate ``f`` at every point, batched on the device when possible.

    ``f.eval_batch`` (the GPU objective) receives all points at once and
    returns slot-ordered floats; otherwise falls back to ``run_batch`` over
    per-point closures, which is the reference behaviour for plain callables.
    Failures surface as ``BatchError(slot)``.
    """
    batch = getattr(f, "eval_batch", None)
    if batch is not None:
        t0 = time.perf_counter()
        _stats.enter(len(points))
        try:
            vals = batch(points)
        finally:
            _stats.leave(len(points))
        _stats.record(time.perf_counter() - t0, device_slots=len(points))
        return [float(v) for v in vals]
    return run_batch([lambda p=p: float(f(p)) for p in points], budget)
