"""Adversarial GREEDY rows for the fp32 error band (test input generator, CPU oracle).

The GREEDY kernel decides each comparison of the walk (clipping.py:185 loss_l < loss_r,
:187/:191 candidate < best) on fp32 losses and re-decides in float64 only inside an error
band.  Part of that band is the code-misround term: an element whose code argument lies
within eta of a rounding boundary may take the other code in fp32, moving the loss by up to
2 eta W^2.  The band covers 2 such elements per side; repeated values parked next to a
boundary break that assumption, which the kernel detects by counting (near_escalate).

Each row built here:
  1. k duplicates of one value v (3 <= k <= d/2) inside an N(0,1) row,
  2. v placed on a code boundary of the L candidate the reference visits at a chosen
     iteration t (fixed point: the walk is re-run until that candidate is still visited),
  3. one free element tuned by bisection over float32 values until loss_l - loss_r of
     iteration t crosses a target of 2e-6 .. 5e-5 relative (a tenth of the rows: an exact
     tie) -- outside the 2-element band, inside what k misrounded elements can move,
  4. v moved by a few ulps (inside eta of the boundary, not on it).
So iteration t's decision hinges on k elements the fp32 evaluation can misround together,
with the two losses closer than those misrounds can move them.  The oracle (pinned to the reference by
tests/test_oracle_golden.py) gives the reference's answer.
"""

from __future__ import annotations

import numpy as np

import oracle

B_DEF, R_DEF = 200, 0.16


def _loss_gap(x, t, nl_t, nr_t, b, r):
    """loss_l - loss_r at iteration t if the walk still visits (nl_t, nr_t) there, else None."""
    nl, nr, ll, lr = oracle.greedy_trace(x, b, r)
    if t >= nl.size or nl[t] != nl_t or nr[t] != nr_t:
        return None
    return ll[t] - lr[t]


def adversarial_row(rng, d, k, b=B_DEF, r=R_DEF, tries=12):
    """One adversarial row (float32, length d) or None if the construction did not settle."""
    x = rng.standard_normal(d).astype(np.float32)
    order = np.argsort(x)
    interior = order[1:-1]
    if interior.size < k + 1:
        return None
    pick = rng.choice(interior, k + 1, replace=False)
    dup, free = pick[:k], pick[k]
    for _ in range(tries):
        x0, x1 = float(x.min()), float(x.max())
        nl, nr, ll, lr = oracle.greedy_trace(x, b, r)
        if nl.size == 0:
            return None
        t = int(rng.integers(0, nl.size))
        step = (x1 - x0) / b
        lo, hi = x0 + (nl[t] + 1) * step, x1 - nr[t] * step
        scale = (hi - lo) / 15
        kb = int(rng.integers(1, 15))
        bnd = lo + (kb - 0.5) * scale
        if not (x0 < bnd < x1):
            continue
        xt = x.copy()
        xt[dup] = np.float32(bnd)
        g = _loss_gap(xt, t, nl[t], nr[t], b, r)
        if g is None:
            x = xt
            continue
        # tune the free element until loss_l - loss_r of iteration t crosses a target gap
        # between the 2-element band and the k-element misround reach (relative 2e-6 .. 5e-5,
        # either sign; a tenth of the rows aim at an exact tie)
        rel = 0.0 if rng.random() < 0.1 else float(np.exp(rng.uniform(np.log(2e-6), np.log(5e-5))))
        tgt = rel * max(abs(ll[t]), abs(lr[t])) * (1 if rng.random() < 0.5 else -1)
        us = np.linspace(x0 + 0.02 * (x1 - x0), x1 - 0.02 * (x1 - x0), 48).astype(np.float32)
        vals = []
        for u in us:
            xt[free] = u
            g = _loss_gap(xt, t, nl[t], nr[t], b, r)
            vals.append(None if g is None else g - tgt)
        lo_u = hi_u = None
        for a_, b_, va, vb in zip(us[:-1], us[1:], vals[:-1], vals[1:]):
            if va is not None and vb is not None and np.sign(va) != np.sign(vb) and va != 0:
                lo_u, hi_u, glo = a_, b_, va
                break
        if lo_u is None:
            continue
        # bisection over float32 values (as integers of the ordered bit pattern)
        a, c = np.float32(lo_u), np.float32(hi_u)
        ok = True
        for _ in range(64):
            if np.nextafter(a, c) == c:
                break
            m = np.float32((np.float64(a) + np.float64(c)) / 2)
            if m == a or m == c:
                break
            xt[free] = m
            vm = _loss_gap(xt, t, nl[t], nr[t], b, r)
            if vm is None:
                ok = False
                break
            vm -= tgt
            if np.sign(vm) == np.sign(glo):
                a = m
            else:
                c = m
        if not ok:
            continue
        xt[free] = a if rng.random() < 0.5 else c
        # park the duplicates a few ulps off the boundary (inside eta, not on it)
        v = np.float32(bnd)
        for _ in range(int(rng.integers(1, 6))):
            v = np.nextafter(v, np.float32(np.inf if rng.random() < 0.5 else -np.inf))
        xt[dup] = v
        return xt
    return None


def adversarial_table(rows, d, seed, b=B_DEF, r=R_DEF):
    """rows adversarial rows of width d (duplicate counts 3 .. d/2), deterministic in seed."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < rows:
        k = int(rng.integers(3, max(4, d // 2 + 1)))
        row = adversarial_row(rng, d, k, b, r)
        if row is not None:
            out.append(row)
    return np.stack(out)
