"""Write the parity report from a device run and the oracle fixtures.

    python scripts/parity_report.py gpurun_out/parity_dev.json > profiles/parity_r02.json

Per configuration and mode (forward: K1, K3, K2+K4; train: K1, K3, K7): for
every partial quantity the max relative error against the fp64 oracle at floor
0, the number of partials outside 1e-5 relative (floor 0, no allowance), and
the rule; per-row logp / entropy statistics over all C2 rows (live oracle).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from tests.parity import REL, partials_report  # noqa: E402


def main(path: str) -> None:
    dev = json.loads(Path(path).read_text())
    fx = json.loads((ROOT / "tests" / "golden" / "full_partials.json").read_text())
    out = {"tolerance": {"sums": f"|g - o| <= {REL} |o| (floor 0)", "per_row": f"|g - o| <= {REL} max(|o|, 1e-3)",
                         "counts": "exact; clip counts within the oracle's borderline rows",
                         "adv_sum": "exactly 0 in real arithmetic: |g - o| <= 1e-9 N_rollouts"},
           "oracle": "oracle/oracle.c oracle_score_batch, fp64 (tests/golden/full_partials.json)",
           "device": "prorl_score_host, fill mode, seed 31, sigma 2.0, 16 576-row micro-batches", "configs": {}}
    for case, d in dev["cases"].items():
        f = fx.get(case)
        if f is None or f["digest"] != d["digest"]:
            continue
        P, Q = np.array(f["partials"]), np.array(f["abs"])
        entry = {"n_active": f["n_active"], "vocab": f["vocab"], "dtype": f["dtype"], "n_border": f["n_border"]}
        for mode in ("forward", "train"):
            rep = partials_report(d[mode], P, Q, f["n_border"])
            g = np.array(d[mode])
            entry[mode] = {"quantities": rep, "violations_floor0": sum(v["violations"] for v in rep.values()),
                           "k1_bias_per_row": float((g[7] - P[7]) / P[1]),
                           "k1_cancellation": float(Q[7] / abs(P[7])) if P[7] else None}
        out["configs"][case] = entry
    if "rows" in dev:
        out["rows_c2_all"] = dev["rows"]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
