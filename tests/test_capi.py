"""The C-ABI library loads and exports every symbol include/salient_b200.h declares.

Only host-side entry points (plan/layout/key helpers) are called here; device
compute needs a GPU and is covered by the -m gpu suite.
"""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2110_08450_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "salient_b200.h"


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(sal_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    # and the ctypes signature table covers the same set
    assert set(syms) == set(_lib.SIGNATURES)


def test_version_and_error_channel():
    L = _lib.lib()
    assert L.sal_version() >= 100
    plan = _lib.SalMfgPlan()
    rc = L.sal_mfg_plan_init(ctypes.byref(plan), 0, (ctypes.c_int32 * 1)(1), 8, 100)
    assert rc == -1
    assert b"hops" in L.sal_last_error()
    with pytest.raises(_lib.SalError, match="hops"):
        _lib.check(rc, "plan")


def test_plan_capacities_follow_size_hint():
    L = _lib.lib()
    plan = _lib.SalMfgPlan()
    per = (ctypes.c_int32 * 3)(15, 10, 5)
    _lib.check(L.sal_mfg_plan_init(ctypes.byref(plan), 3, per, 1024, 111_059_956))
    assert list(plan.fanout)[:3] == [5, 10, 15]          # expansion order
    assert list(plan.node_cap)[:4] == [1024, 6144, 67584, 1081344]
    assert list(plan.edge_cap)[:3] == [5120, 61440, 1013760]
    assert plan.table_cap == 1 << 22
    lay = _lib.SalMfgLayout()
    _lib.check(L.sal_mfg_layout_init(ctypes.byref(plan), ctypes.byref(lay)))
    offs = [lay.table, lay.globals, lay.sizes, lay.etot] + list(lay.dst_indptr)[:3] + \
        list(lay.src_local)[:3] + [lay.src_glob, lay.slot, lay.rank, lay.scan]
    assert all(o % 256 == 0 for o in offs)
    assert len(set(offs)) == len(offs)
    assert lay.total >= max(offs)


def test_plan_small_graph_caps_clip():
    L = _lib.lib()
    plan = _lib.SalMfgPlan()
    _lib.check(L.sal_mfg_plan_init(ctypes.byref(plan), 2, (ctypes.c_int32 * 2)(3, 2), 64, 100))
    assert list(plan.node_cap)[:3] == [64, 100, 100]
    rc = L.sal_mfg_plan_init(ctypes.byref(plan), 1, (ctypes.c_int32 * 1)(-1), 8, 100)
    assert rc == -1


def test_invalid_arguments_set_the_error_message():
    """Every SAL_EINVAL comes with its own sal_last_error() message (checked on entry
    points that validate before touching the device)."""
    L = _lib.lib()
    cases = [
        (lambda: L.sal_zero_spans(None, None, 9, None), "zero_spans"),
        (lambda: L.sal_argmax_correct(None, 0, 1, 10, _lib.SAL_BF16, None, None, None, None),
         "argmax_correct"),
        (lambda: L.sal_mean_bwd(None, 8, _lib.SAL_BF16, 8, 0, None, None, None, None, None, None,
                                None, None, 0, None, None, 0.0, None, 8, _lib.SAL_BF16, None),
         "mean_bwd"),
        (lambda: L.sal_sample_aggregate(None, None, None, None, None, 0, 0, None, 0, 0, 0, None,
                                        0, 0, 0, None), "sample_aggregate"),
    ]
    for call, name in cases:
        L.sal_zero_spans(None, None, 0, None)   # a successful call in between
        assert call() == -1                     # SAL_EINVAL
        assert name in L.sal_last_error().decode(), name
