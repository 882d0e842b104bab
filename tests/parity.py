"""Parity rules of SURVEY.md App. B.7 / §8 d6 and the north star, shared by the
GPU tests, smoke() and scripts/parity_report.py.

  * packing, masks, cu_seqlens, ids, active rows: bit-exact (compared elsewhere);
  * per-row logp / entropy: |g - o| <= 1e-5 * max(|o|, 1e-3);
  * advantages: |g - o| <= 1e-5 * |o| (floor 0);
  * partial sums (loss, entropy, logp, ratio, KL sums, the per-turn buckets):
    |g - o| <= 1e-5 * |o| (floor 0), plus 1e-12 * sum|terms| — an fp64
    reassociation allowance (the device and the oracle add the same fp64
    terms in different orders) that matters only for a sum that cancels to
    ~0, seven orders of magnitude below the relative bound anywhere else;
  * counts exact, except the clip counters, which may differ by the rows whose
    ratio sits within 1e-5 of a clip bound (counted by the oracle);
  * small randomized batches (the ragged edge-case tests) whose sums cancel
    to ~0 by chance may add a random-walk allowance: 6 eps_row * sum|t| /
    sqrt(n_rows), eps_row = 1e-7 the device's per-row relative accuracy
    (measured 3.3e-8 rms over all 904 452 C2 rows) — the 6-sigma noise of a
    sum of n independent per-row errors. The full-size configurations are
    checked without it;
  * sum(old_lp - logp) (the k1 KL estimate) is linear in logp and, with the
    synthetic plant logp = old_lp + U(-0.25, 0.25), cancels 580-4100-fold at
    full size, so it sees any SYSTEMATIC per-row logp error 580-4100 times
    magnified. Two such sources were found and removed: the MUFU.EX2 bias
    (-5.1e-8 per term; rowmath.cuh kEx2Bias) and the FFMA rounding of the
    logsumexp argument on the bf16 grid (+1.3e-9 per row in K2; rowmath.cuh
    RoundFix). It is checked like every other sum, at floor 0 with no
    allowance;
  * sum(A) is exactly 0 in real arithmetic for every informative group (the
    GRPO advantages are centred), so both sides hold only fp64 rounding
    residue there: |g - o| <= 1e-9 * N_rollouts.
"""
from __future__ import annotations

import numpy as np

from paper_2603_18815_b200 import _native as N

REL = 1e-5
ROW_FLOOR = 1e-3
REASSOC = 1e-12

GLOBAL_NAMES = {N.P_LOSS_SUM: "loss_sum", N.P_N_ACTIVE: "n_active", N.P_ENTROPY_SUM: "entropy_sum",
                N.P_LOGP_SUM: "logp_sum", N.P_RATIO_SUM: "ratio_sum", N.P_CLIP_LO: "clip_lo", N.P_CLIP_HI: "clip_hi",
                N.P_KL1_SUM: "k1_sum", N.P_ADV_SUM: "adv_sum", N.P_N_ROLLOUTS: "n_rollouts", N.P_KL_SUM: "k3_sum",
                N.P_ERR_RANKS: "err_ranks"}
BUCKET_FIELDS = ("n", "loss", "entropy", "logp", "clip")


def kind(i: int) -> tuple[str, str]:
    """(quantity name, rule) of partial i; rule in sum / count / clip / adv_sum."""
    if i < N.N_GLOBAL:
        name = GLOBAL_NAMES[i]
        if i == N.P_ADV_SUM:
            return name, "adv_sum"
        if i in (N.P_CLIP_LO, N.P_CLIP_HI):
            return name, "clip"
        if i in (N.P_N_ACTIVE, N.P_N_ROLLOUTS, N.P_ERR_RANKS):
            return name, "count"
        return name, "sum"
    k, f = divmod(i - N.N_GLOBAL, N.N_PER_TURN)
    field = BUCKET_FIELDS[f]
    return f"turn_{field}", {"n": "count", "clip": "clip"}.get(field, "sum")


ROW_EPS = 1e-7


def partial_ok(i: int, g: float, o: float, q: float, n_border: int, n_rollouts: float,
               rw_rows: int | None = None) -> tuple[bool, float]:
    """(within tolerance, relative error |g - o| / |o| or inf/0)."""
    _, rule = kind(i)
    err = abs(g - o)
    rel = err / abs(o) if o != 0 else (0.0 if err == 0 else float("inf"))
    if rule == "adv_sum":
        return err <= 1e-9 * max(n_rollouts, 1.0), rel
    if rule == "clip":
        return err <= n_border, rel
    if rule == "count":
        return g == o, rel
    allow = REASSOC * q + (6 * ROW_EPS * q / max(rw_rows, 1) ** 0.5 if rw_rows else 0.0)
    return err <= REL * abs(o) + allow, rel


def partials_report(got, P, Q, n_border: int) -> dict:
    """Per quantity: max relative error (floor 0), violations at floor 0 with no
    allowance, the rule."""
    got = np.asarray(got, np.float64)
    out: dict = {}
    for i in range(N.N_PARTIALS):
        name, rule = kind(i)
        ok, rel = partial_ok(i, got[i], P[i], Q[i], n_border, P[N.P_N_ROLLOUTS])
        r = out.setdefault(name, {"rule": rule, "n": 0, "max_rel": 0.0, "violations": 0})
        if rule == "sum":
            r["floor"] = 0.0
        r["n"] += 1
        if np.isfinite(rel):
            r["max_rel"] = max(r["max_rel"], rel)
        if rule in ("adv_sum", "clip"):
            r["max_abs"] = max(r.get("max_abs", 0.0), abs(got[i] - P[i]))
        r["violations"] += 0 if ok else 1
    return out


def assert_partials_close(got, P, Q, n_border, what="", rw_rows: int | None = None):
    got = np.asarray(got, np.float64)
    bad = []
    for i in range(N.N_PARTIALS):
        ok, rel = partial_ok(i, got[i], P[i], Q[i], n_border, P[N.P_N_ROLLOUTS], rw_rows)
        if not ok:
            bad.append((i, kind(i)[0], got[i], P[i], rel))
    assert not bad, f"{what}: {len(bad)} partials out of tolerance (idx, name, got, oracle, rel): {bad[:6]}"


def assert_rows_close(got, want, what, floor=ROW_FLOOR):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    err = np.abs(got - want)
    tol = REL * np.maximum(np.abs(want), floor)
    bad = np.nonzero(~(err <= tol))[0]
    assert bad.size == 0, (f"{what}: {bad.size} rows out of tolerance; worst idx {bad[:5]} "
                           f"got {got[bad[:5]]} want {want[bad[:5]]} "
                           f"maxrel {np.max(err / np.maximum(np.abs(want), floor))}")


def rows_report(got, want, floor=ROW_FLOOR) -> dict:
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    e = got - want
    rel = np.abs(e) / np.maximum(np.abs(want), floor)
    return {"n": int(len(e)), "floor": floor, "max_rel": float(rel.max()) if len(e) else 0.0,
            "violations": int((rel > REL).sum()), "mean_signed": float(e.mean()) if len(e) else 0.0,
            "rms": float(np.sqrt((e * e).mean())) if len(e) else 0.0}
