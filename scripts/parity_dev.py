"""Device side of the full-size parity report (profiles/parity_r02.json).

On the GPU box: runs prorl_score_host (fill mode, seed 31) on the full C2 / C3
shards and the C4 rank-0-of-8 shard, forward (K2+K4) and training mode (K7),
and writes the 332 partials per case to gpurun_out/parity_dev.json. With
--rows it also scores every active row of C2 through K1 + keyed generator +
K2 and compares per-row logp / entropy with the live CPU oracle (all host
threads), recording error statistics (max relative error, violations, bias).

    python scripts/parity_dev.py [--rows] [--cases c2,c3,c4r0w8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2603_18815_b200 import synth  # noqa: E402
from paper_2603_18815_b200.hotpath import ScoreConfig, Scorer  # noqa: E402

sys.path.insert(0, str(ROOT / "tests" / "golden"))
from make_full_partials import CASES, SEED, SIGMA, batch_digest, case_config, case_opts  # noqa: E402


def rows_vs_oracle(s: Scorer, dev) -> dict:
    from oracle import oracle as O
    sh = synth.make_shard("c2")
    b = sh.batch
    V, n = 151936, sh.n_active
    pk = s.pack(b.turns, torch.from_numpy(b.ids).to(dev), torch.from_numpy(b.lp).to(dev), b.n_rollouts, V, n)
    keys = s.row_keys(pk["act_row"], pk["act_seq"], pk["cu_seqlens"], torch.from_numpy(b.rollout_key).to(dev))
    mb = 16576
    x = torch.empty((mb, V), dtype=torch.bfloat16, device=dev)
    lp_d, ent_d = [], []
    for r0 in range(0, n, mb):
        m = min(mb, n - r0)
        tg, ol = pk["act_target"][r0:r0 + m], pk["act_old_lp"][r0:r0 + m]
        s.gen_logits_keyed(x, keys[r0:r0 + m], tg, ol, seed=SEED, sigma=SIGMA)
        lp, ent = s.logprob_entropy(x[:m], tg)
        lp_d.append(lp.cpu().numpy())
        ent_d.append(ent.cpu().numpy())
    lp_d, ent_d = np.concatenate(lp_d).astype(np.float64), np.concatenate(ent_d).astype(np.float64)
    hb = O.host_batch(b.turns, b.ids, b.lp, b.reward, b.usable, b.group_off, b.rollout_key)
    t0 = time.time()
    ref = O.score_batch(hb, O.score_cfg(V, "bf16"), SEED, SIGMA, nthreads=os.cpu_count() or 1, want_rows=True,
                        n_active_hint=n)
    secs = time.time() - t0
    from tests.parity import rows_report
    out = {"case": "c2", "n_rows": n, "oracle_seconds": round(secs, 1), "oracle_threads": os.cpu_count()}
    for name, g, o in (("logp", lp_d, ref["logp"][:n]), ("entropy", ent_d, ref["entropy"][:n])):
        out[name] = rows_report(g, o)
        out[name]["max_rel_floor_0"] = float((np.abs(g - o) / np.abs(o)).max())
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default=",".join(CASES))
    ap.add_argument("--rows", action="store_true")
    ap.add_argument("--out", default="gpurun_out/parity_dev.json")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    s = Scorer(0)
    res = {"kernel_config": None, "cases": {}}
    for name in a.cases.split(","):
        c = CASES[name]
        sh = synth.make_shard(c["config"], **c["kw"])
        b = sh.batch.pinned()
        cc = case_config(name)
        cfg = ScoreConfig(vocab=cc["vocab"], dtype=cc["dtype"], microbatch_rows=16576, **case_opts(name))
        tdt = torch.bfloat16 if cc["dtype"] == "bf16" else torch.float32
        pool = [torch.empty((cfg.microbatch_rows, cfg.vocab), dtype=tdt, device=dev) for _ in range(2)]
        fwd, tm = s.score_host(b, cfg, pool, fill=True, seed=SEED, sigma=SIGMA)
        trn, _ = s.score_host(b, cfg, pool, fill=True, seed=SEED, sigma=SIGMA, train=True, n_global=float(sh.n_active))
        res["cases"][name] = {"digest": batch_digest(sh.batch), "n_active": sh.n_active,
                              "forward": [float(v) for v in fwd], "train": [float(v) for v in trn],
                              "score_ms": float(tm[2])}
        print(name, sh.n_active, "loss", fwd[0] / fwd[1], flush=True)
        del pool
        torch.cuda.empty_cache()
    if a.rows:
        res["rows"] = rows_vs_oracle(s, dev)
        print(json.dumps(res["rows"]), flush=True)
    Path(a.out).parent.mkdir(exist_ok=True, parents=True)
    Path(a.out).write_text(json.dumps(res, indent=1) + "\n")
    s.close()


if __name__ == "__main__":
    main()
