"""Threshold distances of the fallback-ladder decisions of one head-step.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The north star allows device decisions to differ from the reference only
"where a bound lies within that tolerance of its threshold".  This module
measures, for one head-step of the reference (or of the oracle), how far each
deciding quantity sits from the threshold it is compared with:

  coverage  |cumulative mass - tau| at the coverage crossing
            (attention.py:181-185), when moving k_coverage by one can move K*
  cut       relative mass gap between the last promoted and the first tail
            block of the mass order (attention.py:146-159, 192-203): a near
            tie there swaps which block is promoted
  value     min_b |p_b eta_b - v_tol| / v_tol (fallback.py:141-155); greedy
            mode: the residual's distance from the budget at the stop, and the
            contribution gap at the cut (fallback.py:156-161)
  ranking   smallest gap between consecutive entries of the top r+1 of the
            phase-2 and of the phase-1 log-masses over F (fallback.py:164-178)
  boundary  |max tail l' + Delta - l_(r)| (fallback.py:181-187)
  canary    |max |s - s'| - (Delta + eps)| over the tokens of F
            (fallback.py:190-199)

Every value is +inf when the decision does not exist for the head-step (no
tail, ranking checks off, ...).  ``near_threshold`` applies the tolerances the
parity tests state.
"""

import math

import numpy as np

FIELDS = ("coverage", "cut", "value", "ranking", "boundary", "canary")

# tolerances of the device path (fp32 masses / scores against fp64):
# absolute for coverage / ranking / boundary / canary, relative for cut / value
TOL = {"coverage": 1e-5, "cut": 1e-4, "value": 1e-4, "ranking": 1e-4, "boundary": 1e-4,
       "canary": 1e-4}
# against the UNMODIFIED reference the value annotations eta also differ by the
# documented FP16 value-metadata narrowing (up to ~2.5e-3 relative, SURVEY
# "Metadata width"), which moves p * eta
TOL_REFERENCE = dict(TOL, value=5e-3)


def _top_gaps(vals, r):
    """Smallest gap between consecutive entries among the r+1 largest values."""
    v = np.sort(np.asarray(vals, dtype=np.float64))[::-1][:r + 1]
    if v.size < 2:
        return math.inf
    return float(np.min(v[:-1] - v[1:]))


def decision_margins(masses, order, k_star, k_coverage, partial_mass, etas, lm1, lm2_promoted,
                     delta, canary_gap, *, tau_cov, k_min, k_max, v_tol, greedy_value_budget=None,
                     ranking_depth=1, epsilon_guard=1e-6, rung2_enabled=True,
                     ranking_checks_enabled=True, canary_enabled=True):
    """Threshold distances (dict over FIELDS) of one head-step.

    ``masses`` / ``order``: normalized Phase-1 masses and the mass order
    (attention.py:174-184); ``k_star`` after Rung 1; ``lm1`` Phase-1 log-mass
    of every full block; ``lm2_promoted`` {block: Phase-2 log-mass} over F;
    ``canary_gap`` = max |s - s'| over F's tokens.
    """
    inf = math.inf
    out = dict.fromkeys(FIELDS, inf)
    masses = np.asarray(masses, dtype=np.float64)
    nb = masses.shape[0]
    if nb == 0:
        return out
    order = np.asarray(order, dtype=np.int64)
    cum = float(partial_mass) + np.cumsum(masses[order])
    kc = int(k_coverage)
    hi = min(int(k_max), nb)
    # K* = min(max(kc, k_min), hi): kc matters only if kc +- 1 lands in [k_min, hi]
    if kc + 1 >= k_min and kc - 1 <= hi:
        d = []
        if 1 <= kc <= nb and cum[kc - 1] >= tau_cov:
            d.append(cum[kc - 1] - tau_cov)
        if kc >= 2:
            d.append(tau_cov - cum[kc - 2])
        if kc == nb and cum[-1] < tau_cov:
            d.append(tau_cov - cum[-1])
        if d:
            out["coverage"] = float(min(abs(x) for x in d))
    ks = int(k_star)
    if 0 < ks < nb:
        a, b = masses[order[ks - 1]], masses[order[ks]]
        out["cut"] = float((a - b) / a) if a > 0 else inf
    if rung2_enabled:
        c = masses * np.asarray(etas, dtype=np.float64)
        if greedy_value_budget is None:
            out["value"] = float(np.min(np.abs(c - v_tol)) / v_tol)
        else:
            o = np.lexsort((np.arange(nb), -c))
            resid = float(c.sum())
            dist = abs(resid - greedy_value_budget)
            n = 0
            for bk in o:
                if resid <= greedy_value_budget:
                    break
                resid -= float(c[bk])
                n += 1
                dist = min(dist, abs(resid - greedy_value_budget))
            gap = float(c[o[n - 1]] - c[o[n]]) if 0 < n < nb else inf
            scale = max(greedy_value_budget, 1e-300)
            out["value"] = float(min(dist / scale, gap / scale))
    F = sorted(int(b) for b in lm2_promoted)
    r = int(ranking_depth)
    lm1 = np.asarray(lm1, dtype=np.float64)
    if ranking_checks_enabled and F and len(F) >= r:
        l2 = np.asarray([lm2_promoted[b] for b in F], dtype=np.float64)
        out["ranking"] = min(_top_gaps(l2, r), _top_gaps(lm1[F], r))
        tail = np.ones(nb, dtype=bool)
        tail[F] = False
        if tail.any():
            lr = np.sort(l2)[::-1][r - 1]
            out["boundary"] = float(abs(lm1[tail].max() + delta - lr))
    if canary_enabled and F:
        out["canary"] = float(abs(canary_gap - (delta + epsilon_guard)))
    return out


def near_threshold(margins, tol=None):
    """Names of the decisions within tolerance of their thresholds."""
    tol = TOL if tol is None else tol
    return [k for k in FIELDS if margins[k] < tol[k]]


def margins_from_oracle(res, policy):
    """decision_margins of an ``oracle.decode_step`` result."""
    lm2 = {int(b): float(res["log_mass_p2"][b]) for b in res["promoted"]}
    return decision_margins(
        res["masses"], res["order"], res["k_star"], res["k_coverage"], res["partial_mass"],
        res["etas"], res["log_mass_p1"], lm2, res["delta_h"], res["canary_gap"],
        tau_cov=policy.tau_cov, k_min=policy.k_min, k_max=policy.k_max, v_tol=policy.v_tol,
        greedy_value_budget=policy.greedy_value_budget, ranking_depth=policy.ranking_depth,
        epsilon_guard=policy.epsilon_guard, rung2_enabled=policy.rung2_enabled,
        ranking_checks_enabled=policy.ranking_checks_enabled,
        canary_enabled=policy.canary_enabled)


def as_row(m):
    return [m[k] for k in FIELDS]
