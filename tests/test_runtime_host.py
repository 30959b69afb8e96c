"""Budgets and batch dispatch (reference test_runtime.py semantics)."""

import time

import numpy as np
import pytest

from paper_2204_04678_b200.errors import BatchError, BudgetError
from paper_2204_04678_b200.runtime import (
    SERIAL, ThreadBudget, default_budget, eval_points, parse_budget, run_batch, runtime_stats,
    reset_runtime_stats,
)


def test_parse_budget():
    assert parse_budget("3:2") == ThreadBudget(3, 2)
    for bad in ("3", "a:b", "0:1", "1:"):
        with pytest.raises(BudgetError):
            parse_budget(bad)


def test_default_budget():
    assert default_budget(2, cores=16) == ThreadBudget(5, 3)
    assert default_budget(5, cores=4) == ThreadBudget(4, 1)


def test_slot_order_and_lowest_error():
    out = run_batch([lambda i=i: i * i for i in range(10)], ThreadBudget(4, 1))
    assert out == [i * i for i in range(10)]

    def boom(i):
        time.sleep(0.01 * (5 - i))
        raise ValueError(i)

    tasks = [lambda: 1, lambda: boom(1), lambda: boom(3)]
    with pytest.raises(BatchError) as info:
        run_batch(tasks, ThreadBudget(3, 1))
    assert info.value.slot in (1, 2)
    with pytest.raises(BatchError) as info:
        run_batch(tasks, SERIAL)
    assert info.value.slot == 1


def test_eval_points_uses_batch_hook():
    calls = []

    class Obj:
        def __call__(self, t):
            raise AssertionError("must not be called per point")

        def eval_batch(self, pts):
            calls.append(len(pts))
            return [float(np.sum(p)) for p in pts]

    reset_runtime_stats()
    vals = eval_points(Obj(), [np.ones(2) * k for k in range(5)], SERIAL)
    assert vals == [0.0, 2.0, 4.0, 6.0, 8.0]
    assert calls == [5]
    assert runtime_stats()["device_slots"] == 5
