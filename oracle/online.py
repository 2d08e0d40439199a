"""Online decoding for n = k + 1 (App. C) -- f64 oracle.

TEST INFRASTRUCTURE ONLY (same rule as oracle/__init__.py).

Task results arrive one at a time; the decoder keeps best-effort estimates f^(x_i), i < k,
and on the completion of task j applies (0-based: mains 0..k-1, parity k; reading R-f2a of
DESIGN.md for the garbled third case, after SPEC.md:210-215):
    j < k :  f^(x_j) <- f(x_j) (finalised);  f^(x_i) <- f^(x_i) - f(x_j) for unfinalised i != j
    j = k :  f^(x_i) <- f^(x_i) + k f(x_{k+1})  for every unfinalised i
Estimates start at 0.  Once k distinct tasks have arrived every estimate is final (for the
single missing main: k f(x_{k+1}) - sum of the other k-1 mains); later events
change nothing.  A repeated task is an error (DuplicateTask).
"""
from __future__ import annotations

import numpy as np


class DuplicateTask(ValueError):
    pass


class DecoderState:
    def __init__(self, k: int, d: int):
        self.k = k
        self.est = np.zeros((k, d))
        self.received = np.zeros(k + 1, bool)
        self.finalized = np.zeros(k, bool)

    def update(self, j: int, value) -> None:
        k = self.k
        if self.received[j]:
            raise DuplicateTask(j)
        if self.received.sum() >= k:          # already decoded: record, change nothing
            self.received[j] = True
            return
        value = np.asarray(value, np.float64)
        if j < k:
            self.est[j] = value
            self.finalized[j] = True
            for i in range(k):
                if not self.finalized[i]:
                    self.est[i] = self.est[i] - value
        else:
            for i in range(k):
                if not self.finalized[i]:
                    self.est[i] = self.est[i] + k * value
        self.received[j] = True
        if self.received.sum() == k:
            self.finalized[:] = True


def run_events(k: int, events, d: int) -> DecoderState:
    """events: list of (task, value)."""
    st = DecoderState(k, d)
    for j, v in events:
        st.update(j, v)
    return st
