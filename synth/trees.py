"""Seeded draft-tree generators (inputs only).

A tree of N draft nodes (root excluded, SURVEY.md amb. A1) is given by
  parent[i] in {-1} U [0, i)    (-1 = child of the root; "parent index of node i is < i")
  token[i]  in [0, V), distinct among siblings
  logprob[i] = draft log q(token | path) <= 0 (carried but unused by the verifier, SURVEY.md amb. A23)

`pooled_tree` implements the tree-construction rule of PAPER.md:599 (App. A: "each forward pass
of the draft model generates multiple parallel candidate tokens, which are then pruned based on
cumulative log probabilities so that the total number of tokens remains within the tree budget")
in the concrete form of SPEC.md:121-122 (top-`branching` proposals per frontier node, global
top-`budget` by cumulative log-prob with ancestor closure), over a synthetic draft distribution
(sorted Dirichlet(alpha) per node, SURVEY.md §8(d) "Generators").
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Tree:
    parent: np.ndarray   # int32 [N]
    token: np.ndarray    # int32 [N]
    logprob: np.ndarray  # float32 [N]

    @property
    def n(self) -> int:
        return int(self.parent.shape[0])

    def copy(self) -> "Tree":
        return Tree(self.parent.copy(), self.token.copy(), self.logprob.copy())

    def depth(self) -> np.ndarray:
        d = np.zeros(self.n, np.int32)
        for i in range(self.n):
            p = int(self.parent[i])
            d[i] = 1 if p < 0 else d[p] + 1
        return d

    def children(self, node: int) -> list[int]:
        """Children of `node` (-1 = root)."""
        return [i for i in range(self.n) if int(self.parent[i]) == node]


def _distinct_tokens(rng: np.random.Generator, k: int, vocab: int, exclude=()) -> np.ndarray:
    excl = set(int(e) for e in exclude)
    out: list[int] = []
    while len(out) < k:
        t = int(rng.integers(0, vocab))
        if t not in excl:
            excl.add(t)
            out.append(t)
    return np.asarray(out, np.int32)


def random_tree(rng: np.random.Generator, n: int, vocab: int) -> Tree:
    """Uniformly random parent links (parent[i] ~ U{-1..i-1}) with distinct sibling tokens."""
    parent = np.empty(n, np.int32)
    token = np.empty(n, np.int32)
    sib: dict[int, list[int]] = {}
    for i in range(n):
        p = int(rng.integers(-1, i)) if i > 0 else -1
        parent[i] = p
        t = _distinct_tokens(rng, 1, vocab, sib.get(p, []))[0]
        token[i] = t
        sib.setdefault(p, []).append(int(t))
    logprob = -rng.exponential(1.0, n).astype(np.float32)
    return Tree(parent, token, logprob)


def chain_tree(tokens) -> Tree:
    tokens = np.asarray(tokens, np.int32)
    n = tokens.shape[0]
    return Tree(np.arange(-1, n - 1, dtype=np.int32), tokens.copy(), np.zeros(n, np.float32))


def pooled_tree(rng: np.random.Generator, budget: int, depth: int, branching: int, vocab: int,
                alpha: float = 0.1) -> Tree:
    """SPEC.md:121-122 pooled top-budget construction over a sorted-Dirichlet draft."""
    # candidate pool entries: (cum_logprob, depth, insertion id, parent id, token, logprob)
    nodes: list[dict] = []          # kept nodes, insertion order
    frontier = [-1]                 # -1 = root
    for _ in range(depth):
        proposals = []
        for f in frontier:
            probs = np.sort(rng.dirichlet(np.full(8, alpha)))[::-1]
            probs = np.maximum(probs, 1e-30)
            sib_tokens = [nodes[c]["token"] for c in range(len(nodes)) if nodes[c]["parent"] == f]
            toks = _distinct_tokens(rng, branching, vocab, sib_tokens)
            base = 0.0 if f < 0 else nodes[f]["cum"]
            fdepth = 0 if f < 0 else nodes[f]["depth"]
            for j in range(branching):
                lp = float(np.log(probs[j]))
                proposals.append(dict(parent=f, token=int(toks[j]), logprob=lp, cum=base + lp,
                                      depth=fdepth + 1))
        pool = [dict(nd, kept=True, idx=i) for i, nd in enumerate(nodes)] + \
               [dict(pr, kept=False, idx=None) for pr in proposals]
        # global top-`budget` by cumulative log-prob; ties -> shallower first, then older first
        order = sorted(range(len(pool)), key=lambda i: (-pool[i]["cum"], pool[i]["depth"], i))
        chosen = set(order[:budget])
        new_nodes: list[dict] = []
        remap: dict[int, int] = {}
        # keep old nodes that survive (ancestor closure holds: cum is non-increasing along paths
        # and ties prefer the shallower node, so a kept node's parent is always kept)
        for i, e in enumerate(pool):
            if i in chosen and e["kept"]:
                remap[e["idx"]] = len(new_nodes)
                new_nodes.append(dict(parent=-1 if e["parent"] < 0 else remap[e["parent"]],
                                      token=e["token"], logprob=e["logprob"], cum=e["cum"],
                                      depth=e["depth"]))
        frontier = []
        for i, e in enumerate(pool):
            if i in chosen and not e["kept"]:
                if e["parent"] >= 0 and e["parent"] not in remap:
                    continue
                frontier.append(len(new_nodes))
                new_nodes.append(dict(parent=-1 if e["parent"] < 0 else remap[e["parent"]],
                                      token=e["token"], logprob=e["logprob"], cum=e["cum"],
                                      depth=e["depth"]))
        nodes = new_nodes
    parent = np.asarray([n["parent"] for n in nodes], np.int32)
    token = np.asarray([n["token"] for n in nodes], np.int32)
    logprob = np.asarray([n["logprob"] for n in nodes], np.float32)
    assert all(parent[i] < i for i in range(len(nodes)))
    return Tree(parent, token, logprob)


def best_path(tree: Tree, min_depth: int) -> list[int]:
    """Node indices root->leaf of the max-cumulative-logprob path of depth >= min_depth
    (SPEC.md:128-131 best path), used to choose where acceptance is planted."""
    depth = tree.depth()
    cum = np.zeros(tree.n)
    for i in range(tree.n):
        p = int(tree.parent[i])
        cum[i] = tree.logprob[i] + (0.0 if p < 0 else cum[p])
    if min_depth <= 0:
        return []
    # every node deeper than min_depth has an ancestor at exactly min_depth
    cands = [i for i in range(tree.n) if depth[i] == min_depth]
    if not cands:
        return []
    best = max(cands, key=lambda i: (cum[i], -i))
    path = []
    cur = best
    while cur >= 0:
        path.append(cur)
        cur = int(tree.parent[cur])
    path.reverse()
    return path


def pack(trees: list[Tree]):
    """CSR packing over requests: node_offset[B+1], parent, token, logprob (int32/float32)."""
    off = np.zeros(len(trees) + 1, np.int32)
    for i, t in enumerate(trees):
        off[i + 1] = off[i] + t.n
    if trees:
        parent = np.concatenate([t.parent for t in trees]).astype(np.int32)
        token = np.concatenate([t.token for t in trees]).astype(np.int32)
        logprob = np.concatenate([t.logprob for t in trees]).astype(np.float32)
    else:
        parent = token = np.zeros(0, np.int32)
        logprob = np.zeros(0, np.float32)
    return off, parent, token, logprob
