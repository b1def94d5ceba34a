// NEXT-F3: the edge's draft-tree builder on the same kernels — the second
// workload.  PAPER.md App. A: "each forward pass of the draft model generates multiple
// parallel candidate tokens, which are then pruned based on cumulative log probabilities so that
// the total number of tokens remains within the tree budget"; §4.2 the best path.
// Rules after SPEC.md S:119-136 (readings in DESIGN.md §9d, R-draft):
//   every pass: each frontier node proposes its top-`branching` tokens (ties: smaller id) with
//   logprob = log-softmax of the draft model; proposals are pooled with the kept nodes and the first
//   `budget` by (-cum_logprob, depth, token, insertion) are kept (ancestor-closed by construction),
//   in insertion order; the kept proposals form the next frontier.
// One pass = the decoder over the current tree (the verify path up to the final norm), the LM head
// with an fp32 store epilogue for the tree's rows, and k_topb over the frontier rows; the pruning is
// host code (a few dozen nodes).
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

namespace se {

namespace {

// One block per requested row: log-sum-exp of the row, then `b` rounds of block argmax excluding
// the ids already taken (ties -> smaller id).  out_tok / out_lp: [nrows][b].
__global__ void k_topb(const float* __restrict__ logits, int V, const int* __restrict__ rows, int b,
                       int* __restrict__ out_tok, float* __restrict__ out_lp) {
  __shared__ float sv[32];
  __shared__ int si[32];
  __shared__ int taken[8];
  const float* l = logits + (size_t)rows[blockIdx.x] * V;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  float m = -INFINITY;
  for (int v = tid; v < V; v += blockDim.x) m = fmaxf(m, l[v]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) sv[wid] = m;
  __syncthreads();
  if (tid < 32) {
    float x = tid < nw ? sv[tid] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
    if (tid == 0) sv[0] = x;
  }
  __syncthreads();
  m = sv[0];
  __syncthreads();
  float sm = 0.f;
  for (int v = tid; v < V; v += blockDim.x) sm += expf(l[v] - m);
  for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
  if (lane == 0) sv[wid] = sm;
  __syncthreads();
  if (tid < 32) {
    float x = tid < nw ? sv[tid] : 0.f;
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (tid == 0) sv[0] = x;
  }
  __syncthreads();
  const float lse = m + logf(sv[0]);
  __syncthreads();
  for (int k = 0; k < b; ++k) {
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int v = tid; v < V; v += blockDim.x) {
      bool skip = false;
      for (int j = 0; j < k; ++j) skip |= taken[j] == v;
      const float x = l[v];
      if (!skip && (x > best || (x == best && v < bi))) { best = x; bi = v; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float x = __shfl_xor_sync(0xffffffffu, best, o);
      const int i = __shfl_xor_sync(0xffffffffu, bi, o);
      if (x > best || (x == best && i < bi)) { best = x; bi = i; }
    }
    if (lane == 0) { sv[wid] = best; si[wid] = bi; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < nw; ++w)
        if (sv[w] > sv[0] || (sv[w] == sv[0] && si[w] < si[0])) { sv[0] = sv[w]; si[0] = si[w]; }
      taken[k] = si[0];
      out_tok[(size_t)blockIdx.x * b + k] = si[0];
      out_lp[(size_t)blockIdx.x * b + k] = sv[0] - lse;
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t topb_launch(const float* logits, int V, const int* rows, int nrows, int b, int* out_tok, float* out_lp,
                        cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  k_topb<<<nrows, 256, 0, st>>>(logits, V, rows, b, out_tok, out_lp);
  return cudaGetLastError();
}

// One pruning step on the host: pool the kept nodes with the frontier's proposals (tok / lp:
// [frontier][branching]) and keep the first `budget` in (-cum, depth, token, insertion) order.
specedge_status draft_prune(std::vector<DraftNode>& nodes, const std::vector<int>& frontier, const std::vector<int>& tok,
                            const std::vector<float>& lp, int branching, int budget, std::vector<int>& next_frontier) {
  // pool = kept nodes ++ proposals (frontier order, then rank)
  std::vector<DraftNode> pool = nodes;
  const int n_old = (int)nodes.size();
  for (size_t fi = 0; fi < frontier.size(); ++fi) {
    const int f = frontier[fi];
    for (int k = 0; k < branching; ++k) {
      DraftNode d;
      d.parent = f;
      d.token = tok[fi * branching + k];
      d.logprob = lp[fi * branching + k];
      d.cum = (f < 0 ? 0.0 : nodes[f].cum) + (double)d.logprob;
      d.depth = f < 0 ? 1 : nodes[f].depth + 1;
      pool.push_back(d);
    }
  }
  std::vector<int> order(pool.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    if (pool[a].cum != pool[b].cum) return pool[a].cum > pool[b].cum;
    if (pool[a].depth != pool[b].depth) return pool[a].depth < pool[b].depth;
    if (pool[a].token != pool[b].token) return pool[a].token < pool[b].token;
    return a < b;
  });
  order.resize(std::min<size_t>(order.size(), (size_t)budget));
  std::sort(order.begin(), order.end());   // insertion order
  std::vector<int> remap(pool.size(), -1);
  for (size_t j = 0; j < order.size(); ++j) remap[order[j]] = (int)j;
  std::vector<DraftNode> kept;
  next_frontier.clear();
  for (int old : order) {
    DraftNode d = pool[old];
    if (d.parent >= 0) {
      if (remap[d.parent] < 0) return SPECEDGE_E_UNSUPPORTED;   // cannot happen: ancestor-closed order
      d.parent = remap[d.parent];
    }
    if (old >= n_old) next_frontier.push_back((int)kept.size());
    kept.push_back(d);
  }
  nodes.swap(kept);
  return SPECEDGE_OK;
}

}  // namespace se
