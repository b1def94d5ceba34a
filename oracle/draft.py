"""Oracle for SURVEY §8(f) NEXT-F3: the edge's draft-tree builder (the second workload of the same
kernels).  TEST INFRASTRUCTURE ONLY (oracle/__init__.py); shares nothing with the library.

PAPER.md App. A: "each forward pass of the draft model generates multiple parallel
candidate tokens, which are then pruned based on cumulative log probabilities so that the total
number of tokens remains within the tree budget"; §4.2: the edge drafts from "the
single path with the highest cumulative log probability".  Concrete rules after SPEC.md S:119-136:

  build_draft_tree(lp, budget, depth, branching):
    nodes = [] (insertion order), frontier = [root]
    repeat `depth` passes:
      every frontier node f proposes its top-`branching` next tokens under the draft distribution
        (ties: smaller token id), node (parent f, token t, logprob lp(f)[t], cum = cum(f) + logprob)
      pool = existing nodes (insertion order) ++ proposals (frontier order, then rank)
      keep the first `budget` of pool sorted by (-cum, depth, token) (S:131 tie-break: smaller
        depth first when pruning, then smaller token id); the kept set is ancestor-closed because a
        child never beats its parent in that order; kept nodes stay in pool (insertion) order
      frontier = the proposals of this pass that were kept
  best_path(tree): root-to-leaf path of the leaf with maximal cum; ties -> greater depth, then the
    lexicographically smaller token sequence

`lp(path)` is the draft model's log-softmax at the position after `path` (a tuple of tokens below
the root).  For the model-backed builder it comes from oracle/model.py's tree forward.
"""
from __future__ import annotations

import numpy as np

from .model import lm_logits, tree_forward


def topk_lowest_id(logprobs, k):
    """Indices of the k largest entries, ties -> smaller index (stable descending sort)."""
    order = np.argsort(-np.asarray(logprobs, np.float64), kind="stable")
    return [int(i) for i in order[:k]]


def build_draft_tree(lp, budget, depth, branching, passes_out=None):
    """Returns (parent, token, logprob, cum) lists in insertion order.  lp(path) -> log-probs [V]."""
    nodes = []   # dicts: parent (index into nodes or -1), token, logprob, cum, depth, path
    frontier = [-1]
    for _ in range(depth):
        proposals = []
        for f in frontier:
            path = () if f < 0 else nodes[f]["path"]
            base = 0.0 if f < 0 else nodes[f]["cum"]
            d = 1 if f < 0 else nodes[f]["depth"] + 1
            l = np.asarray(lp(path), np.float64)
            for t in topk_lowest_id(l, branching):
                proposals.append(dict(parent=f, token=t, logprob=float(l[t]), cum=base + float(l[t]), depth=d,
                                      path=path + (t,)))
        pool = nodes + proposals
        order = sorted(range(len(pool)), key=lambda i: (-pool[i]["cum"], pool[i]["depth"], pool[i]["token"], i))
        keep = sorted(order[:budget])
        remap = {old: new for new, old in enumerate(keep)}
        new_nodes = []
        for old in keep:
            n = dict(pool[old])
            n["parent"] = -1 if n["parent"] < 0 else remap[n["parent"]]
            new_nodes.append(n)
        n_old = len(nodes)
        frontier = [remap[i] for i in keep if i >= n_old]
        nodes = new_nodes
        if passes_out is not None:
            passes_out.append([(n["parent"], n["token"]) for n in nodes])
    return ([n["parent"] for n in nodes], [n["token"] for n in nodes], [n["logprob"] for n in nodes],
            [n["cum"] for n in nodes])


def proactive_expand(lp, head_path, budget, passes, branching):
    """§4.2 proactive drafting: `passes` draft passes rooted at the head
    (the leaf of the best path, given as its token path below the root) with the build rule above;
    the subtree's nodes exclude the head path itself.  Returns (parent, token, logprob, cum) of the
    subtree, parents relative to the subtree (-1 = child of the head), cum relative to the head."""
    head_path = tuple(head_path)
    return build_draft_tree(lambda path: lp(head_path + tuple(path)), budget, passes, branching)


def best_path(parent, token, cum):
    """Node indices of the best root-to-leaf path."""
    n = len(parent)
    if n == 0:
        raise ValueError("no draft")
    children = {i: [] for i in range(n)}
    for i, p in enumerate(parent):
        if p >= 0:
            children[p].append(i)
    depth, seq = [], []
    for i in range(n):
        depth.append(1 if parent[i] < 0 else depth[parent[i]] + 1)
        seq.append(((tuple() if parent[i] < 0 else seq[parent[i]]) + (token[i],)))
    leaves = [i for i in range(n) if not children[i]]
    best = min(leaves, key=lambda i: (-cum[i], -depth[i], seq[i]))
    path = []
    i = best
    while i >= 0:
        path.append(i)
        i = parent[i]
    return path[::-1]


def model_lp(W, session, invT=1.0):
    """Draft log-softmax after a path, from the oracle's tree forward over the session's cache
    (the path's tokens as a chain under the root)."""
    def lp(path):
        parent = list(range(-1, len(path) - 1))
        hf, _, _ = tree_forward(W, session.cache, session.last_token, parent, list(path))
        z = lm_logits(W, hf[-1:])[0] * invT
        z = z - z.max()
        return z - np.log(np.exp(z).sum())
    return lp
