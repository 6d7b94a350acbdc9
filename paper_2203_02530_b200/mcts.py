"""Monte-Carlo tree search over the SpMV design space (NEXT-1; §III-C,
P:375-472), driving the library's executor.

A tree node is a prefix P_k of a traversal: DAG vertices in order, GPU
vertices bound to a stream (BoundGPU_s, tab:vertices P:250-264).  Children of
a prefix are the frontier vertices ("all vertices v in G_P not in P_k and
where all predecessors are in P_k") times the stream choices of a
GPU vertex, pruned under stream bijection (a GPU vertex may use an
already-used stream or the next unused one).  Synchronisation is derived from
the prefix (tab:sync) by ``dspmv_schedule_derive`` when a complete
traversal is benchmarked.

Phases (SPEC.md S:204-304 semantics):
  selection   argmax over children of explore + exploit, explore =
              c*sqrt(ln N / n) with c = sqrt(2) (-inf if fully explored),
              exploit = (t_max^c - t_min^c)/(t_max^p - t_min^p) when n >= 2
              and N >= 2, else 1; stops at a node having a child
              with no rollouts or no materialised children.
  expansion   a zero-rollout child of the selected node, chosen
              uniformly at random (seeded).
  rollout     random legal completion, benchmarked by the caller's
              ``measure(ops) -> seconds`` (the paper's protocol);
              the rollout path is added to the tree.
  backprop    t_min <- min(t, t_min), t_max <- max(t, t_max) on the path
              (P:469-472); a node is fully explored when its terminal is
              benchmarked / all its children are fully explored.

The tree walks any ``schedules.Space``: the coarse DAG (default) or the
per-destination DAG of a set of peer offsets, whose traversal
space is too large to enumerate.  ``syncs="orderable"`` makes the
synchronisation operations tree moves of their own (DESIGN.md
R-N5: ``dspmv_schedule_moves``) instead of deriving them when a traversal is
complete.
"""
from __future__ import annotations

import math
import random

import numpy as np

from . import dspmv as D
from .schedules import COARSE, Space, canonical_key

C_EXPLORE = math.sqrt(2.0)


def explore_value(parent_n: int, child_n: int, child_fully_explored: bool) -> float:
    """c * sqrt(ln N / n), -inf for a fully explored child."""
    if child_fully_explored:
        return -math.inf
    if child_n <= 0:
        return math.inf
    return C_EXPLORE * math.sqrt(math.log(parent_n) / child_n)


def exploit_value(child, parent) -> float:
    """Range ratio; 1 without a basis for comparison (also for a
    zero-width parent range, SPEC ledger)."""
    if child.n >= 2 and parent.n >= 2:
        den = parent.t_max - parent.t_min
        if den > 0:
            return (child.t_max - child.t_min) / den
    return 1.0


class Node:
    __slots__ = ("move", "parent", "children", "n", "t_min", "t_max", "fully_explored", "depth")

    def __init__(self, move, parent):
        self.move, self.parent = move, parent
        self.children = None            # materialised lazily
        self.n = 0
        self.t_min = math.inf
        self.t_max = -math.inf
        self.fully_explored = False
        self.depth = 0 if parent is None else parent.depth + 1

    def prefix(self):
        out, nd = [], self
        while nd is not None and nd.move is not None:
            out.append(nd.move)
            nd = nd.parent
        return out[::-1]


def legal_moves(prefix, n_streams: int, space: Space = COARSE):
    """Frontier vertices x stream choices under bijection pruning (vertices
    are indices into ``space.vertices``)."""
    done = {v for v, _ in prefix}
    used = len({s for v, s in prefix if v in space.gpu})
    moves = []
    for v in range(len(space.vertices)):
        if v in done or not space.pred[v] <= done:
            continue
        if v in space.gpu:
            for s in range(min(used + 1, n_streams)):
                moves.append((v, s))
        else:
            moves.append((v, None))
    return moves


def ops_of(prefix, n_streams: int, space: Space = COARSE) -> np.ndarray:
    order = [v for v, _ in prefix]
    streams = [s if s is not None else 0 for _, s in prefix]
    return space.derive(order, streams, n_streams)


class MCTS:
    """measure(ops) -> seconds benchmarks one complete schedule."""

    def __init__(self, measure, n_streams: int = 2, seed: int = 2203, space: Space = COARSE,
                 syncs: str = "derived"):
        if syncs not in ("derived", "orderable"):
            raise ValueError("syncs must be 'derived' or 'orderable'")
        self.measure = measure
        self.n_streams = n_streams
        self.space = space
        self.syncs = syncs
        self.rng = random.Random(seed)
        self.root = Node(None, None)
        self.dataset = {}               # canonical key -> {"ops", "times"}
        self.iterations = 0

    # -- tree helpers
    def moves(self, prefix):
        if self.syncs == "derived":
            return legal_moves(prefix, self.n_streams, self.space)
        if prefix and prefix[-1][0] == D.DSPMV_OP_END:
            return []
        return [tuple(m) for m in D.dspmv_schedule_moves(prefix, self.n_streams, self.space.offsets).tolist()]

    def ops(self, prefix) -> np.ndarray:
        if self.syncs == "derived":
            return ops_of(prefix, self.n_streams, self.space)
        return np.array(prefix, np.int32)

    def _materialise(self, node):
        if node.children is None:
            node.children = [Node(m, node) for m in self.moves(node.prefix())]
        return node.children

    def select(self):
        node = self.root
        while True:
            kids = node.children
            if not kids:
                return node
            if any(c.n == 0 and not c.fully_explored for c in kids):
                return node
            best, best_v = None, -math.inf
            for c in kids:
                v = explore_value(node.n, c.n, c.fully_explored) + exploit_value(c, node)
                if v > best_v:
                    best, best_v = c, v
            if best is None:              # every child fully explored
                return node
            node = best

    def expand(self, node):
        kids = self._materialise(node)
        if not kids:
            return node                   # terminal
        fresh = [c for c in kids if c.n == 0 and not c.fully_explored]
        return self.rng.choice(fresh) if fresh else node

    def rollout(self, node):
        path_end = node
        while True:
            kids = self._materialise(path_end)
            if not kids:
                break
            path_end = self.rng.choice(kids)
        prefix = path_end.prefix()
        ops = self.ops(prefix)
        t = float(self.measure(ops))
        rec = self.dataset.setdefault(canonical_key(ops), {"ops": ops, "times": []})
        rec["times"].append(t)
        return path_end, t

    def backpropagate(self, leaf, t):
        nd = leaf
        leaf.fully_explored = True        # its traversal has been benchmarked
        while nd is not None:
            nd.n += 1
            nd.t_min = min(nd.t_min, t)
            nd.t_max = max(nd.t_max, t)
            if nd.children is not None and nd.children and all(c.fully_explored for c in nd.children):
                nd.fully_explored = True
            nd = nd.parent

    def step(self) -> bool:
        """One selection/expansion/rollout/backprop cycle; False when done."""
        if self.root.fully_explored:
            return False
        node = self.select()
        child = self.expand(node)
        leaf, t = self.rollout(child)
        self.backpropagate(leaf, t)
        self.iterations += 1
        return True

    def run(self, iterations: int):
        for _ in range(iterations):
            if not self.step():
                break
        return self

    # -- results
    def best(self):
        k = min(self.dataset, key=lambda k: np.mean(self.dataset[k]["times"]))
        return self.dataset[k]["ops"], float(np.mean(self.dataset[k]["times"]))

    def records(self):
        """[(ops, mean time)] of every distinct schedule benchmarked."""
        return [(r["ops"], float(np.mean(r["times"]))) for r in self.dataset.values()]
