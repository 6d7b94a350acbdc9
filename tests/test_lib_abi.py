"""The C-ABI library loads and exports every symbol include/dspmv.h declares
(no compute calls: CPU-only)."""
import ctypes
import os
import re

from paper_2203_02530_b200 import dspmv as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dspmv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dspmv_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("dspmv_plan_create", "dspmv_schedule_create", "dspmv_apply", "dspmv_apply_host",
                 "dspmv_apply_group", "dspmv_partition", "dspmv_comm_create"):
        assert must in names
    assert len(names) >= 30


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(D.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_no_torch_in_the_boundary():
    src = open(os.path.join(ROOT, "include", "dspmv.h")).read()
    assert "torch" not in src.lower().replace("torch.distributed", "")
    assert "at::" not in src and "c10" not in src


def test_version_and_error_plumbing():
    assert D.dspmv_version() == 1
    try:
        D.dspmv_partition(10, 0)
    except D.DspmvError as e:
        assert e.status == D.DSPMV_ERR_ARG
        assert "partition" in D.dspmv_last_error()
    else:
        raise AssertionError("expected DSPMV_ERR_ARG")


def test_binding_marshalling_without_gpu():
    """Every binding marshals its arguments and reaches the library, which
    rejects the NULL handles (ERR_ARG) -- exercises the Python side on CPU."""
    import numpy as np
    import pytest
    rp = np.array([0, 1], np.int64)
    col = np.array([0], np.int32)
    val = np.array([1.0])
    calls = [
        lambda: D.dspmv_plan_create(None, 1, rp, col, val),
        lambda: D.dspmv_plan_create(None, 1, rp, col, val.astype(np.float32), dtype=D.DSPMV_F32),
        lambda: D.dspmv_plan_info_get(None),
        lambda: D.dspmv_plan_destroy(None),
        lambda: D.dspmv_schedule_create(None, [(0, 0, 0, 0)], 1),
        lambda: D.dspmv_schedule_destroy(None),
        lambda: D.dspmv_schedule_set_timing(None, True),
        lambda: D.dspmv_apply(None, 0, 0),
        lambda: D.dspmv_apply_host(None, val, val),
        lambda: D.dspmv_comm_destroy(None),
        lambda: D.dspmv_comm_info(None),
        lambda: D.dspmv_host_plan_destroy(None),
        lambda: D.dspmv_schedule_set_caller_stream0(None, 1),
        lambda: D.dspmv_apply_graph(None, 0, 0, 1),
        lambda: D.dspmv_apply_graph_prepare(None, 0, 0, 1),
        lambda: D.dspmv_apply_graph_group([], [], [], 1),
        lambda: D.dspmv_apply_group([], [], []),
        lambda: D.dspmv_plan_create(None, 1, rp, col, val, pack_mode=D.DSPMV_PACK_ALIAS_IF_CONTIGUOUS,
                                    accumulate_mode=D.DSPMV_ACC_EXPLICIT_IN_END, debug_checks=True),
    ]
    for c in calls:
        with pytest.raises(D.DspmvError) as e:
            c()
        assert e.value.status == D.DSPMV_ERR_ARG
