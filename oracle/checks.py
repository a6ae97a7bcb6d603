"""Teacher-forced greedy check of a device token sequence (oracle; test
infrastructure only — imported by tests/, smoke() and nothing on the product
path).

The reference guarantees that speculative output equals plain AR decoding
token for token (engine.py:13-18, generate_ar engine.py:328-360). Given the
device's emitted sequence, one causal oracle forward over prompt + emitted
gives, for every position i, the AR logits conditioned on the device's own
prefix; the sampler (penalty window of the emitted tokens so far, truncation,
position-keyed draw at len(prompt) + i — engine.py:237-245) then names the
token the reference would emit there. Every position is checked
independently, so one near-tie does not end the comparison; a mismatch is
allowed only where the oracle's top-1 margin of the penalised logits is
below the precision tolerance (north star: 1e-2 relative in bf16).
"""

from __future__ import annotations

import numpy as np

from .sampling import PenaltyWindow, penalized_probs_masked, sample_at, scale_logits, truncate


def teacher_forced(om, prompt, emitted, smp):
    """-> list of (i, oracle_token, relative top-1 margin) for every emitted token."""
    P = len(prompt)
    seq = [int(t) for t in prompt] + [int(t) for t in emitted[:-1]]
    rows = list(range(P - 1, len(seq)))
    b, _ = om.forward(seq, list(range(len(seq))), om.new_cache(), heads_needed=1, logit_rows=rows)
    win = PenaltyWindow(smp.window, om.config.vocab_size)
    out = []
    for i, t in enumerate(emitted):
        logits = b[i, 0]
        member = win.member_mask()
        d = penalized_probs_masked(logits, member, smp)
        want = sample_at(truncate(d, smp.truncation), P + i, smp.seed)
        s = scale_logits(logits, member, smp.temperature, smp.theta, smp.ctrl_style)
        top = np.partition(s, -2)[-2:]
        hi, lo = max(top), min(top)
        out.append((i, int(want), float((hi - lo) / max(1e-30, abs(hi)))))
        win.push(int(t))
    return out


def greedy_mismatches(om, prompt, emitted, smp, tol):
    """Positions where the device token differs from the oracle's although the
    oracle margin exceeds `tol` (must be empty), and the count of positions
    whose margin is below `tol` (not decidable at this precision)."""
    bad, undecided = [], 0
    for i, want, margin in teacher_forced(om, prompt, emitted, smp):
        if margin <= tol:
            undecided += 1
        elif want != int(emitted[i]):
            bad.append((i, int(emitted[i]), want, margin))
    return bad, undecided
