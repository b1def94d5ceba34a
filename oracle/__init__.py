"""CPU oracle for SpecEdge's server-side batched tree verification (arXiv 2505.17052).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import anything from here.  The product path
(`paper_2505_17052_b200/`) never imports, links or executes this package, and this package
never imports the product.  The two share no code; only `synth/` (seeded input generators,
no method arithmetic) feeds both.

Plain, slow, obviously-correct numpy in float64.  Every function cites the passage it follows:
  P:n  = /root/reference/PAPER.md line n,   S:n = /root/reference/SPEC.md line n,
  SURVEY §8(c) O1..O8 / amb. A1..A24 = the readings adopted for what the paper leaves unstated
  (all listed in DESIGN.md "Readings").

Pins (tests/test_oracle_*.py, `-m "not gpu"`): Philox Random123 known-answer vectors; bf16 RNE
against torch's converter; RMSNorm/RoPE closed forms and invariants; attention against
torch SDPA; tree forward == brute-force per-path causal decoding (P1); chain == dense causal
prefill (P2); root-only == one AR step (P3); greedy losslessness over iterated verify+commit
(P4); planted full acceptance (P5); no-match (P6); stochastic law chi-square against the
closed form O7 (P7) with a power check; Gumbel marginals (P8); O8 rejection form == O7 law
exactly (P9); commit == fresh prefill (P10); batch/solo equality (P11); determinism (P12);
worked example fixture (tests/golden).  No function here is "parity unpinned".
"""
