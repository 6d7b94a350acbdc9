"""Design-rule generation from measured schedules (NEXT-2; §IV,
P:475-628) -- CPU-side analysis of the sweep / MCTS dataset.

* ``class_labels``  sort, convolve with a step kernel of radius r = 0.5 % of
  the measurements (min 1), find peaks, keep peaks whose prominence is >= the
  98th percentile (reading R-N2: percentile of the convolution signal, so
  measurement-noise peaks are screened), use them as class boundaries
  (P:483-512).  The paper's
  kernel indices are inconsistent (k on -r..r-1, sum over -r+1..r); reading
  R-N1: the balanced kernel k_m = -1 for m in [-r+1, 0], +1 for m in [1, r],
  evaluated where it fully overlaps (r < i < len - r).  A peak at sorted
  position i puts the boundary between positions i and i+1.
* ``features``      ordering feature "u before v" for every pair of named
  operations (inserted syncs included, named CER-after-u / CES-b4-v /
  CSWE-b4-v as in P:607), stream feature "u same stream as v" for every pair
  of GPU vertices; constant columns dropped.  A pair involving an
  op that some schedules lack reads "not (u before v)" when 0.
* ``train_tree``    scikit-learn CART, gini, class_weight=balanced,
  max_depth = max_leaf_nodes - 1, hyper-parameters by Algorithm 1
  (tab:tree-params P:542-555, alg:dt-params P:564-583).
* ``rulesets``      every root-to-leaf path ending in a leaf of class c
  (P:597-611), phrased like the paper's tables ("y_L before CES-b4-PostSend",
  "y_L different stream than Pack"), sorted by training samples.
* ``class_accuracy`` Table V protocol: classes from a subset,
  tree from the subset, classify every implementation, report the share whose
  time falls inside its predicted class's [fastest, slowest] range.
"""
from __future__ import annotations

import itertools

import numpy as np

from . import dspmv as D
from .schedules import GPU, Space

NAMES = D.VERTEX_NAMES


# ------------------------------------------------------------------ labels
def default_radius(m: int) -> int:
    """0.5 % (minimum 1) of the number of measurements."""
    return max(1, int(round(0.005 * m)))


def step_convolve(a, r: int) -> np.ndarray:
    """c_i = sum_{m=1..r} a_{i+m} - sum_{m=-r+1..0} a_{i+m}, for r < i < len-r
    (entries outside that range are nan)."""
    a = np.asarray(a, np.float64)
    n = len(a)
    c = np.full(n, np.nan)
    cs = np.concatenate([[0.0], np.cumsum(a)])
    for i in range(r + 1, n - r):
        c[i] = (cs[i + r + 1] - cs[i + 1]) - (cs[i + 1] - cs[i - r + 1])
    return c


def class_labels(times, radius: int | None = None, percentile: float = 98.0, threshold: str = "signal",
                 mad_k: float = 3.0):
    """Labels (1 = fastest) for `times` (any order) and the class ranges.

    threshold -- which peaks of the step convolution become class boundaries:
      "signal" (R-N2, default): prominence >= the `percentile` of the
               convolution signal;
      "peaks"  (the literal P:508 wording): prominence >= the `percentile` of
               the peaks' own prominences;
      "mad"    (noise floor): log prominence >= median + mad_k * 1.4826 * MAD
               of the peaks' log prominences -- robust when many classes
               exist, where the two percentile readings drop real boundaries."""
    if threshold not in ("signal", "peaks", "mad"):
        raise ValueError("threshold must be 'signal', 'peaks' or 'mad'")
    from scipy.signal import find_peaks, peak_prominences
    t = np.asarray(times, np.float64)
    order = np.argsort(t, kind="stable")
    a = t[order]
    n = len(a)
    r = default_radius(n) if radius is None else radius
    bounds = []
    if n > 2 * r + 2:
        c = step_convolve(a, r)
        valid = np.where(np.isnan(c), -np.inf, c)
        peaks, _ = find_peaks(valid)
        peaks = peaks[np.isfinite(valid[peaks])]
        if len(peaks):
            import warnings
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                prom = peak_prominences(np.where(np.isfinite(valid), valid, np.nanmin(c)), peaks)[0]
            if threshold == "signal":
                # R-N2: a peak is kept when its prominence is >= the 98th
                # percentile of the convolution signal (noise peaks stay below it)
                thr = np.percentile(c[~np.isnan(c)], percentile)
            elif threshold == "peaks":
                thr = np.percentile(prom, percentile)
            else:
                # noise floor on a log scale: noise peaks spread over orders of
                # magnitude, class boundaries stand out above them
                lp = np.log(prom[prom > 0]) if np.any(prom > 0) else np.zeros(1)
                med = float(np.median(lp))
                mad = 1.4826 * float(np.median(np.abs(lp - med)))
                thr = float(np.exp(med + mad_k * mad))
            bounds = sorted(int(p) for p, q in zip(peaks, prom) if q >= thr and q > 0)
    lab_sorted = np.ones(n, np.int64)
    for b in bounds:
        lab_sorted[b + 1:] += 1
    labels = np.empty(n, np.int64)
    labels[order] = lab_sorted
    ranges = {int(k): (float(a[lab_sorted == k].min()), float(a[lab_sorted == k].max()))
              for k in np.unique(lab_sorted)}
    return labels, ranges, bounds


# ---------------------------------------------------------------- features
_SPACES = {}


def _space(ops) -> Space:
    sp = Space.of_ops(ops)
    return _SPACES.setdefault(tuple(sp.offsets), sp)


def op_names(ops) -> list:
    """Names of every op: vertices by name (per-destination ones as
    "Pack[+1]"), syncs as CER-after-u / CES-b4-v / CSWE-b4-v (v = the
    vertex after the wait, u = the latest DAG predecessor of v on the recorded
    stream, else its latest GPU vertex; a second wait before the same v gets
    ':u')."""
    ops = np.asarray(ops).tolist()
    sp = _space(ops)
    names = [None] * len(ops)
    where = {}
    for t, (k, s, e, p) in enumerate(ops):
        if k < 10:
            names[t] = sp.names[sp.index[(k, p)]]
            where[sp.index[(k, p)]] = (t, s)
    def next_vertex(t0):
        kv, pv = next((kk, pp) for kk, _, _, pp in ops[t0 + 1:] if kk < 10)
        return sp.index[(kv, pv)]

    for t, (k, s, e, _) in enumerate(ops):
        if k != D.DSPMV_OP_EVENT_RECORD:
            continue
        waits = [tt for tt in range(t + 1, len(ops)) if ops[tt][0] in (11, 12) and ops[tt][2] == e]
        # the event is named after the latest DAG predecessor, on its stream,
        # of the vertex its first wait guards (with derived syncs the CER
        # directly precedes that wait; with orderable syncs (R-N5) it may come
        # earlier), else after the latest GPU vertex on its stream
        v = next_vertex(waits[0]) if waits else next_vertex(t)
        on_s = [i for i in sp.gpu if i in where and where[i][1] == s and where[i][0] < t]
        preds_v = [i for i in on_s if (i, v) in sp.edges]
        u = max(preds_v or on_s, key=lambda i: where[i][0], default=None)
        uname = sp.names[u] if u is not None else "?"
        names[t] = f"CER-after-{uname}"
        for w in waits:
            base = ("CES-b4-" if ops[w][0] == D.DSPMV_OP_EVENT_SYNC else "CSWE-b4-") + sp.names[next_vertex(w)]
            names[w] = base if base not in names else f"{base}:{uname}"
    return names


def features(schedules):
    """Binary feature matrix over a list of ops arrays; returns (X, columns)."""
    rows = []
    vocab, gpu_vocab = set(), set()
    for ops in schedules:
        nm = op_names(ops)
        pos = {n: i for i, n in enumerate(nm)}
        stream = {D.vertex_label(k, p): s for k, s, e, p in np.asarray(ops).tolist() if k in GPU}
        rows.append((pos, stream))
        vocab.update(nm)
        gpu_vocab.update(stream)
    names = sorted(vocab)
    gpu_names = sorted(gpu_vocab)
    cols = [("before", u, v) for u, v in itertools.combinations(names, 2)]
    cols += [("same", u, v) for u, v in itertools.combinations(gpu_names, 2)]
    X = np.zeros((len(rows), len(cols)), np.int8)
    for i, (pos, stream) in enumerate(rows):
        for j, (kind, u, v) in enumerate(cols):
            if kind == "before":
                X[i, j] = 1 if (u in pos and v in pos and pos[u] < pos[v]) else 0
            else:
                X[i, j] = 1 if (u in stream and v in stream and stream[u] == stream[v]) else 0
    keep = [j for j in range(len(cols)) if X[:, j].min() != X[:, j].max()]
    # an ordering feature between ops that some schedules lack (sync ops) is
    # 0 both when v comes first and when either is absent: its negation reads
    # "not (u before v)", marked by the kind "before?"
    always = set.intersection(*(set(pos) for pos, _ in rows)) if rows else set()
    out_cols = []
    for j in keep:
        kind, u, v = cols[j]
        if kind == "before" and not (u in always and v in always):
            kind = "before?"
        out_cols.append((kind, u, v))
    return X[:, keep], out_cols


# -------------------------------------------------------------------- tree
def _train(X, y, mln):
    from sklearn.tree import DecisionTreeClassifier
    clf = DecisionTreeClassifier(criterion="gini", max_leaf_nodes=mln, max_depth=max(1, mln - 1),
                                 class_weight="balanced", random_state=0)
    clf.fit(X, y)
    err = 1.0 - float((clf.predict(X) == y).mean())
    return err, clf


def train_tree(X, y):
    """Algorithm 1: grow max_leaf_nodes from 2, probing +1..+5,
    while the training error shrinks.  Returns (clf, mln, history)."""
    mln = 2
    err = np.inf
    cur, clf = _train(X, y, mln)
    history = [(mln, cur, clf.get_depth())]
    while cur < err:
        err = cur
        for i in range(1, 6):
            c2, n2 = _train(X, y, mln + i)
            history.append((mln + i, c2, n2.get_depth()))
            if c2 < err:
                clf, mln, cur = n2, mln + i, c2
                break
    return clf, mln, history


def rule_text(col, value: int) -> str:
    kind, u, v = col
    if kind == "before":
        return f"{u} before {v}" if value else f"{v} before {u}"
    if kind == "before?":
        return f"{u} before {v}" if value else f"not ({u} before {v})"
    return f"{u} same stream as {v}" if value else f"{u} different stream than {v}"


def rulesets(clf, cols):
    """{class: [(n_samples, [rules])]} -- root-to-leaf paths per class."""
    t = clf.tree_
    out = {}

    def walk(node, path):
        if t.children_left[node] == -1:
            cls = int(clf.classes_[int(np.argmax(t.value[node][0]))])
            out.setdefault(cls, []).append((int(t.n_node_samples[node]), list(path)))
            return
        f = t.feature[node]
        walk(t.children_left[node], path + [rule_text(cols[f], 0)])
        walk(t.children_right[node], path + [rule_text(cols[f], 1)])

    walk(0, [])
    for k in out:
        out[k].sort(key=lambda p: -p[0])
    return out


def class_accuracy(sub_ops, sub_times, all_ops, all_times):
    """Table V protocol: fraction of all implementations whose time lies in
    the [fastest, slowest] range of the class the subset's tree assigns."""
    labels, ranges, _ = class_labels(sub_times)
    X_all, cols = features(list(sub_ops) + list(all_ops))
    Xs, Xa = X_all[:len(sub_ops)], X_all[len(sub_ops):]
    if len(ranges) == 1:
        lo, hi = ranges[1]
        t = np.asarray(all_times)
        return float(((t >= lo) & (t <= hi)).mean())
    clf, _, _ = train_tree(Xs, labels)
    pred = clf.predict(Xa)
    t = np.asarray(all_times)
    ok = [ranges[int(p)][0] <= ti <= ranges[int(p)][1] for p, ti in zip(pred, t)]
    return float(np.mean(ok))
