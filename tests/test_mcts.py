"""MCTS (NEXT-1, §III-C) on CPU with a deterministic synthetic cost
model (no GPU): closed forms, bijection pruning, coverage, determinism,
range containment ("0 <= V <= 1")."""
import math

import numpy as np
import pytest

from paper_2203_02530_b200 import dspmv as D
from paper_2203_02530_b200 import mcts as M
from paper_2203_02530_b200 import schedules as PS


def cost(ops):
    """Deterministic stand-in for a measurement: depends on order and streams."""
    ops = np.asarray(ops)
    kinds = list(ops[:, 0])
    t = 1.0 + 0.05 * kinds.index(D.DSPMV_OP_SPMV_LOCAL)
    t += 0.03 * sum(1 for k in kinds if k == D.DSPMV_OP_EVENT_SYNC)
    sL = ops[kinds.index(D.DSPMV_OP_SPMV_LOCAL), 1]
    sP = ops[kinds.index(D.DSPMV_OP_PACK), 1]
    return t - (0.2 if sL != sP else 0.0)


def test_explore_exploit_closed_forms():
    assert math.isclose(M.explore_value(2, 1, False), math.sqrt(2) * math.sqrt(math.log(2)))
    assert M.explore_value(1, 1, False) == 0.0
    assert M.explore_value(5, 3, True) == -math.inf

    class N:  # minimal node
        def __init__(self, n, lo, hi):
            self.n, self.t_min, self.t_max = n, lo, hi
    assert M.exploit_value(N(2, 2, 4), N(3, 1, 5)) == 0.5
    assert M.exploit_value(N(1, 2, 4), N(3, 1, 5)) == 1.0
    assert M.exploit_value(N(2, 1, 1), N(2, 1, 1)) == 1.0


def test_bijection_pruning_first_gpu_vertex():
    I = PS.COARSE.index
    start, pack, yl = I[(D.DSPMV_OP_START, 0)], I[(D.DSPMV_OP_PACK, 0)], I[(D.DSPMV_OP_SPMV_LOCAL, 0)]
    mv = M.legal_moves([(start, None)], 2)
    gpu = [m for m in mv if m[0] in PS.COARSE.gpu]
    assert gpu and all(s == 0 for _, s in gpu)
    mv2 = M.legal_moves([(start, None), (pack, 0)], 2)
    assert sorted(s for v, s in mv2 if v == yl) == [0, 1]


def test_full_search_covers_design_space():
    m = M.MCTS(cost, n_streams=2, seed=1).run(100000)
    assert m.root.fully_explored
    keys = set(m.dataset)
    ref = {PS.canonical_key(o) for o in PS.enumerate_derived(2)}
    assert keys == ref and len(keys) == 768
    best_ops, best_t = m.best()
    assert best_t == min(cost(o) for o in PS.enumerate_derived(2))
    for ops, _ in m.records()[:50]:
        D.dspmv_schedule_validate(ops, 2)


def test_seed_determinism_and_containment():
    a = M.MCTS(cost, seed=7).run(200)
    b = M.MCTS(cost, seed=7).run(200)
    assert list(a.dataset) == list(b.dataset)
    stack = [a.root]
    while stack:
        nd = stack.pop()
        for c in nd.children or []:
            if c.n >= 1:
                assert nd.t_min <= c.t_min <= c.t_max <= nd.t_max
                assert 0.0 <= M.exploit_value(c, nd) <= 1.0
            stack.append(c)
    assert a.root.n == 200


@pytest.mark.parametrize("iters", [50, 100, 200, 400])
def test_iterations_bound_dataset(iters):
    m = M.MCTS(cost, seed=3).run(iters)
    assert m.iterations == iters and len(m.dataset) <= iters


def test_mcts_on_the_per_destination_space():
    """The same search over the per-destination DAG of offsets {-1, +1}
    (P:281-284): every benchmarked schedule is valid for that DAG, distinct,
    and the search is seed-deterministic."""
    sp = PS.Space([-1, 1])
    assert len(sp.vertices) == 16

    def cost_f(ops):
        ops = np.asarray(ops)
        k = list(ops[:, 0])
        return 1.0 + 0.01 * k.index(D.DSPMV_OP_SPMV_LOCAL) + 0.001 * len(k)

    a = M.MCTS(cost_f, seed=5, space=sp).run(300)
    b = M.MCTS(cost_f, seed=5, space=sp).run(300)
    assert list(a.dataset) == list(b.dataset)
    assert len(a.dataset) == 300                 # nothing repeats in a space this large
    for ops, _ in a.records():
        D.dspmv_schedule_validate(ops, 2)
        assert PS.Space.of_ops(ops).offsets == [-1, 1]


def test_mcts_with_orderable_syncs_covers_the_4780_space():
    """Syncs as tree moves (R-N5): the exhaustive search visits
    exactly the 4,780 orderable schedules and finds the cost minimum."""
    m = M.MCTS(cost, n_streams=2, seed=11, syncs="orderable").run(10 ** 6)
    assert m.root.fully_explored
    space = PS.enumerate_orderable(2)
    assert set(m.dataset) == {PS.canonical_key(o) for o in space}
    assert m.best()[1] == min(cost(o) for o in space)
