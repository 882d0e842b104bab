"""Generate tests/golden/full_partials.json: the CPU oracle's whole-step
partials (oracle_score_batch, fp64) on the FULL shards the headline is about.

Cases (SURVEY.md §8 d6 asks for oracle parity on every config):
  * c2      — BASELINE configs[1], the whole Qwen3-4B-shaped batch (904 452 active rows);
  * c3      — configs[2], the whole Qwen3-8B-shaped batch (2 050 676 active rows), the N=1 bench config;
  * c4r0w8  — configs[3], rank 0 of the 8-GPU group-sharded layout (2 053 469 active rows);
  * c1      — configs[0], the CPU-runnable case (fp32 logits, V = 32 000);
  * c5_wide / c5_narrow — configs[4], the stress sweep at V = 262 144 (64
    turns) and V = 32 000 (group 32), log-normal 1K-64K-token trajectories;
  * c5_mid / c5_short — two points inside the sweep: V = 128 256 (group 16,
    16 turns) and V = 65 536 (group 8, 8 turns, short trajectories).

Each case records the 332 partials, the |term| sums, the count of rows whose
clip decision sits within 1e-5 of a bound, and a digest of the host SoA so a
drift in the synthetic generator is caught before any comparison. The GPU
tests (tests/test_gpu_fullsize.py) compare prorl_score_host against these at
the north-star tolerance; the oracle is test infrastructure only.

    python tests/golden/make_full_partials.py [case ...]     # ~40 min on 8 cores
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402

OUT = Path(__file__).resolve().parent / "full_partials.json"
SEED = 31       # synthetic-logits seed (prorl_score_host fill mode)
SIGMA = 2.0

# BASELINE configs[4] ("stress sweep: 1K-64K token trajectories x 1-64 turns,
# group size 4-32, vocab 32000-262144") at its two vocabulary ends
C5_WIDE = dict(index=4, tasks=8, group=4, tokens=16384, turns=64, vocab=262144, dtype="bf16", asst_share=0.3,
               lengths="lognormal", desc="stress: V=262144 bf16, group 4, 64 turns, lognormal 1K-64K tokens")
C5_NARROW = dict(index=4, tasks=16, group=32, tokens=4096, turns=2, vocab=32000, dtype="bf16", asst_share=0.3,
                 lengths="lognormal", desc="stress: V=32000 bf16, group 32, 1 assistant turn, lognormal 1K-64K tokens")

# and two points inside it: a Llama-3-sized vocabulary with group 16 / 16 turns,
# and V = 65 536 with group 8 / 8 turns on short (1K-4K) trajectories
C5_MID = dict(index=4, tasks=8, group=16, tokens=8192, turns=16, vocab=128256, dtype="bf16", asst_share=0.3,
              lengths="lognormal", desc="stress: V=128256 bf16, group 16, 16 turns, lognormal 1K-64K tokens")
C5_SHORT = dict(index=4, tasks=32, group=8, tokens=2048, turns=8, vocab=65536, dtype="bf16", asst_share=0.3,
                lengths="lognormal", desc="stress: V=65536 bf16, group 8, 8 turns, lognormal 1K-64K tokens (mean 2K)")

CASES = {
    "c1": dict(config="c1", kw={}),
    "c2": dict(config="c2", kw={}),
    "c3": dict(config="c3", kw={}),
    "c4r0w8": dict(config="c4", kw={"rank": 0, "world": 8}),
    "c5_wide": dict(config=C5_WIDE, kw={}),
    "c5_narrow": dict(config=C5_NARROW, kw={}),
    "c5_mid": dict(config=C5_MID, kw={}),
    "c5_short": dict(config=C5_SHORT, kw={}),
    # non-default options on the C2 batch: sampling temperature 0.7
    # (inv_temperature, types.hpp:59) and the population std (ddof 0)
    "c2_t07_ddof0": dict(config="c2", kw={}, opts={"inv_temperature": 1 / 0.7, "ddof": 0}),
}


def case_opts(name: str) -> dict:
    """ScoreConfig options of a case beyond vocab / dtype (defaults otherwise)."""
    return dict(CASES[name].get("opts", {}))


def case_config(name: str) -> dict:
    """The config dict of a case (a BASELINE config name or an explicit dict)."""
    from paper_2603_18815_b200 import synth_spec
    c = CASES[name]["config"]
    return dict(synth_spec.CONFIGS[c]) if isinstance(c, str) else dict(c)


def batch_digest(b) -> str:
    h = hashlib.sha256()
    for a in (b.turns, b.ids, b.lp, b.reward, b.usable, b.group_off, b.rollout_key):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def run_case(name: str, nthreads: int) -> dict:
    from paper_2603_18815_b200 import synth
    c = CASES[name]
    sh = synth.make_shard(c["config"], **c["kw"])
    b = sh.batch
    cfg = case_config(name)
    hb = O.host_batch(b.turns, b.ids, b.lp, b.reward, b.usable, b.group_off, b.rollout_key)
    oc = O.score_cfg(cfg["vocab"], cfg["dtype"], **case_opts(name))
    t0 = time.time()
    r = O.score_batch(hb, oc, SEED, SIGMA, nthreads=nthreads)
    assert r["status"] == 0 and r["n_active"] == sh.n_active
    return {"config": c["config"] if isinstance(c["config"], str) else cfg["desc"], "kw": c["kw"], "seed": SEED, "sigma": SIGMA, "vocab": cfg["vocab"],
            "dtype": cfg["dtype"], "n_active": int(r["n_active"]), "n_rollouts": int(b.n_rollouts),
            "digest": batch_digest(b), "partials": [float(x) for x in r["partials"]],
            "abs": [float(x) for x in r["abs"]], "n_border": int(r["n_border"]),
            "oracle_seconds": round(time.time() - t0, 1), "oracle_threads": nthreads, "opts": case_opts(name)}


def main(argv: list[str]) -> None:
    names = argv or list(CASES)
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    data["source"] = ("oracle/oracle.c oracle_score_batch (fp64) on paper_2603_18815_b200.synth shards; "
                      "generated by tests/golden/make_full_partials.py")
    O.build(ref=False)
    for n in names:
        data[n] = run_case(n, os.cpu_count() or 1)
        OUT.write_text(json.dumps(data, indent=1) + "\n")
        print(n, data[n]["n_active"], data[n]["oracle_seconds"], "s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
