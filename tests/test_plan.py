"""Host-side program plans, no GPU (pt_create with PT_DEVICE_HOST + pt_plan_stats).

The plan builder is the executor's compiler: it splits every operator apply
into dataflow tasks, stages the operator in ring pieces and sizes the task
slots.  These checks hold for any operator:
- every program kind plans, and its task types add up;
- the operator pieces stream the algorithmic bytes once (each kernel of an
  A-apply once; each D/R kernel of a sweep once per sweep) -- exactly for
  dense kernels, and fewer for PLR kernels whose factor-heavy leaves are
  stored as their product U.Vt;
- per-task metadata stays within the executor's slot limits;
- a plan-only handle refuses device work with PT_EINVAL.
"""

import ctypes as C

import numpy as np
import pytest

from conftest import FIXTURES, case_path, golden_path
from paper_1410_5910_b200 import _native as nat
from paper_1410_5910_b200.operator import DeviceOperator, load_case_arrays


def host_op(name):
    path = golden_path(name) if name.startswith("fx_") else case_path(name)
    if not path.exists():
        pytest.skip(f"{path.name} not built")
    meta, arr = load_case_arrays(path)
    return DeviceOperator.from_arrays(meta, arr, device="host")


@pytest.mark.parametrize("name", FIXTURES)
def test_every_program_plans(name):
    op = host_op(name)
    for kind, n_it in (("A", 0), ("M", 1), ("M", 2), ("AM", 2), ("S", 0)):
        st = op.plan_stats(kind, n_it)
        assert st["tasks"] > 0
        assert st["t_plr"] + st["y_plr"] + st["y_dense"] == st["tasks"]
        assert st["counters"] >= 1
        if op.kernel_format == "dense":
            # dense kernels run as tile-major dense leaves: 16-row Y tasks, no Vt work
            assert st["t_plr"] == 0
        else:
            assert st["t_plr"] > 0 and st["y_plr"] > 0


@pytest.mark.parametrize("name", FIXTURES)
def test_pieces_stream_the_algorithmic_bytes(name):
    op = host_op(name)
    a = op.plan_stats("A")
    if op.kernel_format == "dense":
        assert a["staged_bytes"] == a["algo_bytes"] > 0
    else:
        assert 0 < a["staged_bytes"] <= a["algo_bytes"]
    m1 = op.plan_stats("M", 1)
    m2 = op.plan_stats("M", 2)
    # the second sweep re-reads every D/R kernel once more
    assert m2["staged_bytes"] > m1["staged_bytes"]
    am = op.plan_stats("AM", 2)
    assert am["staged_bytes"] == a["staged_bytes"] + m2["staged_bytes"]


@pytest.mark.parametrize("name", FIXTURES)
def test_task_metadata_within_slot_limits(name):
    op = host_op(name)
    for kind in ("A", "AM"):
        st = op.plan_stats(kind, 2)
        assert st["max_terms"] <= 16
        assert st["max_pieces"] <= 48


def test_dense_leaves_only_remove_bytes(monkeypatch):
    """Storing factor-heavy leaves as U.Vt changes the bytes, not the structure."""
    # a pure PLR fixture (a mixed operator's dense E blocks stream their
    # factor pair U = E, Vt = I when dense leaves are off)
    name = next((f for f in FIXTURES if "plr" in f and "extrap" not in f), None)
    if name is None:
        pytest.skip("no PLR fixture")
    on = host_op(name).plan_stats("A")
    monkeypatch.setenv("PT_DENSE_LEAVES", "0")
    off = host_op(name).plan_stats("A")
    assert off["staged_bytes"] == off["algo_bytes"] == on["algo_bytes"]
    assert on["staged_bytes"] <= off["staged_bytes"]
    assert on["y_plr"] == off["y_plr"] and on["t_plr"] <= off["t_plr"]


@pytest.mark.parametrize("name", FIXTURES)
def test_partial_sum_block_rows_keep_the_bytes(monkeypatch, name):
    """PT_BLOCK_TERMS=2 splits a block row's kernel terms over partial-sum
    tasks: more output tasks, fewer terms each, the same operator bytes."""
    whole = host_op(name).plan_stats("A")
    monkeypatch.setenv("PT_BLOCK_TERMS", "2")
    split = host_op(name).plan_stats("A")
    assert split["staged_bytes"] == whole["staged_bytes"]
    assert split["algo_bytes"] == whole["algo_bytes"]
    assert split["max_terms"] <= 2
    assert split["y_plr"] >= whole["y_plr"]


def test_plan_only_handle_refuses_device_work():
    op = host_op(FIXTURES[0])
    x = np.zeros(op.N * 2)
    rc = nat.lib().pt_apply_A(op._h, x.ctypes.data, x.ctypes.data, None)
    assert rc == nat.PT_EINVAL
    assert b"plan-only" in nat.lib().pt_last_error()
    g, sm, he = C.c_int32(), C.c_int64(), C.c_int64()
    assert nat.lib().pt_exec_info(op._h, C.byref(g), C.byref(sm), C.byref(he)) == 0
    assert g.value % 148 == 0 and 0 < sm.value <= 232448 and he.value > 0


@pytest.mark.parametrize("name", ["c1", "c3r", "c2", "c3"])
def test_large_case_plans(name):
    """Reference-scale operators (when cases/ holds them) plan within limits."""
    op = host_op(name)
    st = op.plan_stats("AM", 2)
    a, m2 = op.plan_stats("A"), op.plan_stats("M", 2)
    assert st["staged_bytes"] == a["staged_bytes"] + m2["staged_bytes"]
    assert st["staged_bytes"] <= a["algo_bytes"] + m2["algo_bytes"]


@pytest.mark.parametrize("stages", [2, 3])
@pytest.mark.parametrize("name", ["fx_plr", "fx_extrap_plr", "fx_extrap", "c3r", "c4"])
def test_long_tasks_plan_beyond_the_ring_window(name, stages, monkeypatch):
    """A task may hold more pieces than the ring's parity window (2 x stages):
    the producer applies the window bound only to a use's first n_stages
    positions, so long tasks (PT_T_PIECES above the window, many dense terms)
    are planned, not rejected (the GPU runs them in
    test_gpu_parity.py::test_scheduling_variants_bitwise_equal)."""
    monkeypatch.setenv("PT_STAGES", str(stages))
    monkeypatch.setenv("PT_T_PIECES", "16")
    monkeypatch.setenv("PT_T_PIECES_CHAIN", "16")
    op = host_op(name)
    for kind, n_it in (("A", 0), ("M", 2), ("AM", 2)):
        st = op.plan_stats(kind, n_it) if n_it else op.plan_stats(kind)
        assert 1 <= st["max_pieces"] <= 48
