"""Design-rule pipeline (NEXT-2, §IV) on CPU: SPEC.md examples for
the labeler, feature semantics, Algorithm 1, rule recovery on a planted rule."""
import numpy as np
import pytest

from paper_2203_02530_b200 import dspmv as D
from paper_2203_02530_b200 import rules as R
from paper_2203_02530_b200 import schedules as PS


def test_default_radius():
    assert R.default_radius(2036) == 10 and R.default_radius(50) == 1 and R.default_radius(400) == 2


def test_step_convolve_closed_forms():
    c = R.step_convolve(np.ones(20), 3)
    assert np.all(c[~np.isnan(c)] == 0)                         # constant -> 0
    a = np.arange(30, dtype=float) * 0.5                         # ramp slope s -> r^2 s
    c = R.step_convolve(a, 4)
    assert np.allclose(c[~np.isnan(c)], 16 * 0.5)
    a = np.array([0, 0, 0, 0, 10, 10, 10, 10], float)            # jump between 3 and 4
    c = R.step_convolve(a, 2)
    assert np.nanargmax(c) == 3


def test_labels_bimodal_trimodal_and_invariance():
    # deterministic clusters (linear ramps): within a cluster the step
    # convolution is the constant r^2*s, so the only peaks are at the jumps
    ramp = np.linspace(0, 0.01, 1000)
    t = np.concatenate([1 + ramp, 2 + ramp])
    lab, ranges, _ = R.class_labels(t)
    assert len(ranges) == 2 and ranges[1][1] < 1.5 < ranges[2][0]
    assert np.all(lab[:1000] == 1) and np.all(lab[1000:] == 2)
    r7 = np.linspace(0, 0.01, 700)
    t3 = np.concatenate([1 + r7, 2 + r7, 3.5 + r7])
    lab3, ranges3, _ = R.class_labels(t3)
    assert len(ranges3) == 3
    lab3b, _, _ = R.class_labels(5 * t3 + 7)                     # positive affine invariance
    assert np.array_equal(lab3, lab3b)
    lab1, r1, _ = R.class_labels(np.full(100, 3.0))
    assert len(r1) == 1
    order = np.argsort(t3)
    assert np.all(np.diff(lab3[order]) >= 0)                     # monotone in time


def test_feature_semantics_and_names():
    order = [0, 4, 1, 2, 3, 6, 7, 8, 5, 9]      # start PostRecv Pack y_L PostSend ...
    ops = D.dspmv_schedule_derive(order, [0, 0, 0, 1, 0, 0, 0, 0, 0, 0], 2)
    nm = R.op_names(ops)
    assert "CER-after-Pack" in nm and "CES-b4-PostSend" in nm
    X, cols = R.features([ops, D.dspmv_schedule_derive(order, [0] * 10, 2)])
    j = cols.index(("same", "Pack", "y_L"))
    assert X[0, j] == 0 and X[1, j] == 1                          # "y_L, Pack in different streams"
    assert ("before", "Pack", "PostSend") not in cols              # forced by the DAG -> dropped


def test_algorithm1_and_planted_rule_recovery():
    scheds = PS.enumerate_derived(2)
    X, cols = R.features(scheds)

    def t_of(ops):                       # planted: "Pack before y_L" and different streams fast
        nm = R.op_names(ops)
        k = list(np.asarray(ops)[:, 0])
        fast = nm.index("Pack") < nm.index("y_L") and \
            ops[k.index(D.DSPMV_OP_PACK)][1] != ops[k.index(D.DSPMV_OP_SPMV_LOCAL)][1]
        return 1.0 if fast else 2.0
    times = np.array([t_of(o) for o in scheds])
    labels, ranges, _ = R.class_labels(times)
    assert len(ranges) == 2
    clf, mln, hist = R.train_tree(X, labels)
    assert (clf.predict(X) == labels).all()
    errs = [h[1] for h in hist]
    assert errs[-1] <= errs[0]
    rs = R.rulesets(clf, cols)
    top = rs[1][0][1]
    assert "Pack before y_L" in top and "Pack different stream than y_L" in top
    acc = R.class_accuracy(scheds[:200], times[:200], scheds, times)
    assert acc > 0.9


def test_features_on_orderable_schedules():
    """Every op of every orderable-sync schedule (R-N5) gets a distinct name,
    and the feature matrix separates all 4,780 schedules' vertex orders."""
    from paper_2203_02530_b200 import schedules as PS
    space = PS.enumerate_orderable(2)
    for ops in space[::37]:
        nm = R.op_names(ops)
        assert None not in nm and len(set(nm)) == len(nm), nm
    X, cols = R.features(space[:600])
    assert X.shape[0] == 600 and X.shape[1] > 10


def test_labels_many_separated_classes_mad_threshold():
    """Nine classes separated by >= 40 sigma jumps: the percentile readings of
    P:508 keep too few boundaries (R-N2 keeps the 98th percentile of the
    signal, the literal reading 2 % of the peaks); the log-MAD noise floor
    recovers all nine, and stays at 1 / 2 / 5 classes on single-cluster,
    two-cluster and uniform five-cluster data."""
    rng = np.random.default_rng(0)
    sig = 1e-3
    t9 = np.concatenate([1 + k * 40 * sig * (1 + 0.5 * k) + rng.normal(0, sig, 230) for k in range(9)])
    lab, ranges, bounds = R.class_labels(t9, threshold="mad")
    assert len(ranges) == 9
    order = np.argsort(t9)
    assert np.array_equal(lab[order], np.repeat(np.arange(1, 10), 230))
    assert len(R.class_labels(t9, threshold="signal")[1]) < 9
    assert len(R.class_labels(1 + rng.normal(0, sig, 2000), threshold="mad")[1]) == 1
    t2 = np.concatenate([1 + rng.normal(0, sig, 1000), 2 + rng.normal(0, sig, 1000)])
    assert len(R.class_labels(t2, threshold="mad")[1]) == 2
    t5 = np.concatenate([1 + k * 0.05 + rng.uniform(0, 0.01, 400) for k in range(5)])
    assert len(R.class_labels(t5, threshold="mad")[1]) == 5
    with pytest.raises(ValueError):
        R.class_labels(t5, threshold="bogus")
