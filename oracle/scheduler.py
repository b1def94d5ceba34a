"""Oracle for SURVEY §8(f) NEXT-F1: the server's pipeline-aware scheduler and draft-depth calibration
(§4.3, "interleaving verification tasks across multiple requests ... server
verification time ~= edge drafting time + network round-trip time"; §5.2, P:516 worked depths;
SPEC.md scheduler module S:311-383).

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): plain Python, written from the passages above,
shares no code with the library's C++ scheduler (paper_2505_17052_b200/csrc/scheduler.cu).

Readings (R-sched):
* depth = max(1, round_half_away((verify_ms - rtt_ms) / draft_pass_ms)) — S:330-333; nearest
  rounding is forced by the paper's three published depths.
* timing estimates are exponentially weighted means with weight w ("weight 0.2"): est <- (1-w)
  est + w x; the first observation initialises the estimate when no prior is given.
* one outstanding request per session; the queue is FIFO by arrival (ties: admission order);
  a plan takes the oldest min(capacity, queued) requests and never waits when one is ready (S:343-347
  work conservation); padded_len = max member length (reported only: the GPU path is ragged).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field


def round_half_away(x: float) -> int:
    """Nearest integer, halves away from zero, on the exact value of x (x - floor(x) is exact
    in binary floating point, so no x + 0.5 rounding can move a value below a half across it)."""
    a = abs(x)
    q = math.floor(a)
    r = q + 1 if a - q >= 0.5 else q
    return int(r) if x >= 0 else -int(r)


def calibrate_draft_depth(verify_ms: float, draft_pass_ms: float, rtt_ms: float) -> int:
    """S:330-333 / P:306: choose the number of draft passes so that edge drafting + RTT matches the
    server's verification time."""
    return max(1, round_half_away((verify_ms - rtt_ms) / draft_pass_ms))


class Ewma:
    """Exponentially weighted running mean."""

    def __init__(self, weight: float, init: float | None = None):
        self.w = weight
        self.v = init

    def observe(self, x: float):
        self.v = x if self.v is None else (1.0 - self.w) * self.v + self.w * x
        return self.v


@dataclass
class Pending:
    session: int
    handle: int
    length: int
    arrival: float
    seq: int


@dataclass
class Scheduler:
    """VerifyQueue + DepthPolicy + plan_batch."""
    capacity: int
    ewma_weight: float = 0.2
    fixed_depth: int = 0
    verify: Ewma = None
    draft_pass: Ewma = None
    rtt: Ewma = None
    queue: list = field(default_factory=list)
    outstanding: set = field(default_factory=set)
    seq: int = 0

    def __post_init__(self):
        self.verify = self.verify or Ewma(self.ewma_weight)
        self.draft_pass = self.draft_pass or Ewma(self.ewma_weight)
        self.rtt = self.rtt or Ewma(self.ewma_weight)

    def admit(self, session: int, handle: int, length: int, arrival: float) -> bool:
        """enqueue; a second outstanding request of a session is a protocol error."""
        if session in self.outstanding:
            return False
        self.outstanding.add(session)
        self.queue.append(Pending(session, handle, length, arrival, self.seq))
        self.seq += 1
        return True

    def plan(self):
        """the oldest min(capacity, len(queue)) requests (FIFO by arrival, then admission
        order); returns (members, padded_len) or None when the queue is empty."""
        if not self.queue:
            return None
        order = sorted(self.queue, key=lambda p: (p.arrival, p.seq))
        members = order[:self.capacity]
        chosen = {id(m) for m in members}
        self.queue = [p for p in self.queue if id(p) not in chosen]
        return members, max(m.length for m in members)

    def complete(self, sessions, verify_ms: float):
        for s in sessions:
            self.outstanding.discard(s)
        self.verify.observe(verify_ms)

    def depth(self) -> int:
        if self.fixed_depth > 0:
            return self.fixed_depth
        if self.verify.v is None or self.draft_pass.v is None or self.rtt.v is None:
            return 1
        return calibrate_draft_depth(self.verify.v, self.draft_pass.v, self.rtt.v)
