"""The C-ABI library loads on the CPU host and exports every symbol that
include/pinla.h declares (no compute call: no GPU here)."""

import os
import re

from conftest import ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "pinla.h")).read()
    return sorted(set(re.findall(r"\b(pinla_[a-z_]+)\s*\(", text)))


def test_header_declares_expected_api():
    syms = declared_symbols()
    for s in ("pinla_create", "pinla_eval_batch", "pinla_selinv_diag", "pinla_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2204_04678_b200 import _lib

    L = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert set(_lib.EXPORTS) <= set(declared_symbols())
    assert b"sm_100a" in L.pinla_version()


def test_struct_layouts_match_header():
    """ctypes structs have the fields of the C structs, in order."""
    from paper_2204_04678_b200 import _lib

    text = open(os.path.join(ROOT, "include", "pinla.h")).read()

    def fields(struct):
        body = re.search(r"typedef struct " + struct + r" \{(.*?)\} " + struct, text, re.S).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        return re.findall(r"\b([a-z_0-9]+);", body)

    assert [f for f, _ in _lib.PinlaModel._fields_] == fields("pinla_model")
    assert [f for f, _ in _lib.PinlaOptions._fields_] == fields("pinla_options")
    assert [f for f, _ in _lib.PinlaStats._fields_] == fields("pinla_stats_t")


def test_create_without_gpu_fails_loudly():
    import numpy as np
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2204_04678_b200.errors import EngineError
    from paper_2204_04678_b200.objective import ObjectiveEvaluator
    from paper_2204_04678_b200.synth import make_instance

    inst = make_instance("c1", nx=6, ny=6, m=40)
    with pytest.raises(EngineError):
        ObjectiveEvaluator(inst.spec, inst.y)
