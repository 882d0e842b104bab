"""Trajectory ingestion (prorl_ingest_responses): the reference's /process wire
JSON -> host SoA. Pinned to JSON produced by the reference's own
build_process_response (tests/golden/reference_vectors.json) and to the
synthetic shards the rest of the suite uses."""
import json
import time
from pathlib import Path

import numpy as np
import pytest

from paper_2603_18815_b200 import _native as N
from paper_2603_18815_b200 import synth
from paper_2603_18815_b200.hotpath import RolloutError, ingest_responses

GOLD = json.loads((Path(__file__).parent / "golden" / "reference_vectors.json").read_text())


def _expected(cases, group_off, tol=0.0):
    """Python restatement of the participation rules for the expected SoA."""
    turns, ids, lps, reward, usable = [], [], [], [], []
    n_active = 0
    for g in range(len(group_off) - 1):
        members = cases[group_off[g]:group_off[g + 1]]
        u = [c["reward"] for c in members if c["status"] != "FAILED"]
        info = len(u) >= 2 and max(u) - min(u) > tol
        for j, c in enumerate(members):
            slot = group_off[g] + j
            reward.append(c["reward"])
            usable.append(0 if c["status"] == "FAILED" else 1)
            if not info or c["status"] == "FAILED":
                continue
            off, pos = 0, 0
            for r, L in zip(c["roles"], c["lens"]):
                turns.append((len(ids), slot, L, r))
                ids.extend(c["ids"][off:off + L])
                lps.extend(c["logprobs"][off:off + L] if r == 2 else [0.0] * L)
                if r == 2 and L > 0:
                    n_active += L - (1 if pos == 0 else 0)
                pos += L
                off += L
    return turns, ids, lps, reward, usable, n_active


def _check(b, exp):
    turns, ids, lps, reward, usable, _ = exp
    got_t = [(int(t["src_off"]), int(t["traj"]), int(t["len"]), int(t["role"])) for t in b.turns]
    assert got_t == turns
    assert b.ids.tolist() == ids
    assert b.lp.tolist() == lps          # exact: from_chars round-trips the reference's dump
    assert b.reward.tolist() == reward
    assert b.usable.tolist() == usable


@pytest.mark.parametrize("group_size", [1, 2, 3, 4, 24])
def test_reference_wire_json(group_size):
    cases = GOLD["process_response"]
    group_off = list(range(0, len(cases) + 1, group_size))
    if group_off[-1] != len(cases):
        group_off.append(len(cases))
    b, n_active, n_info = ingest_responses([c["json"].encode() for c in cases], group_off)
    exp = _expected(cases, group_off)
    _check(b, exp)
    assert n_active == exp[5]


def test_synthetic_shard_roundtrip():
    """A synthetic shard serialised in the reference's schema ingests back to the same SoA."""
    from tests.wire import to_responses
    sh = synth.make_shard("c1", seed=99)
    b = sh.batch
    resp = to_responses(b)
    got, n_active, n_info = ingest_responses(resp, b.group_off)
    for f in ("ids", "lp", "reward", "usable"):
        assert np.array_equal(getattr(got, f), getattr(b, f)), f
    assert np.array_equal(got.turns[["src_off", "traj", "len", "role"]], b.turns[["src_off", "traj", "len", "role"]])
    assert n_active == sh.n_active


@pytest.mark.parametrize("bad,code", [
    (b'{"status":"DONE","reward":1,"trajectory":[{"role":"assistant","input_ids":[1],"output_ids":[],"logprobs":[]}]}',
     "malformed_turn"),
    (b'{"status":"DONE","reward":1,"trajectory":[{"role":"assistant","input_ids":[],"output_ids":[1,2],"logprobs":[-1]}]}',
     "malformed_turn"),
    (b'{"status":"DONE","reward":1,"trajectory":[{"role":"tool","input_ids":[1],"output_ids":[],"logprobs":[-1]}]}',
     "malformed_turn"),
    (b'{"status":"DONE","reward":1,"trajectory":[{"role":"robot","input_ids":[1]}]}', "malformed_turn"),
    (b'{"status":"DONE","reward":1,"trajectory":[{"role":"user","input_ids":[1,}]}', "malformed_request"),
    (b'{"status":"DONE","reward":1}', "malformed_request"),
    (b'{"status":"DONE","reward":1,"trajectory":[]} trailing', "malformed_request"),
    (b'{"status":"DONE","reward":1,"trajectory":[{"role":"user","input_ids":[1.5]}]}', "malformed_request"),
])
def test_malformed_responses(bad, code):
    ok = b'{"status":"DONE","reward":0,"trajectory":[{"role":"user","input_ids":[1]}]}'
    with pytest.raises(RolloutError) as e:
        ingest_responses([ok, bad], [0, 2])
    assert e.value.code == code
    assert "response 1" in str(e.value)


def test_throughput_c2_sized():
    """~2.3 M tokens of wire JSON (the C2 shard): report the parse rate."""
    sh = synth.make_shard("c2", max_groups=12)
    b = sh.batch
    resp = []
    by = {}
    for k, t in enumerate(b.turns):
        by.setdefault(int(t["traj"]), []).append(k)
    for s in range(b.n_rollouts):
        parts = []
        for k in by.get(s, []):
            t = b.turns[k]
            o, L, r = int(t["src_off"]), int(t["len"]), int(t["role"])
            ids = ",".join(map(str, b.ids[o:o + L].tolist()))
            if r == 2:
                lps = ",".join(repr(x) for x in b.lp[o:o + L].tolist())
                parts.append(f'{{"input_ids":[],"logprobs":[{lps}],"output_ids":[{ids}],"role":"assistant","text":""}}')
            else:
                parts.append(f'{{"input_ids":[{ids}],"logprobs":[],"output_ids":[],"role":"tool","text":""}}')
        resp.append((f'{{"job_id":"j{s}","reward":{float(b.reward[s])},"status":"'
                     f'{"DONE" if b.usable[s] else "FAILED"}","timings":{{}},"trajectory":[' + ",".join(parts)
                     + "]}").encode())
    nbytes = sum(len(r) for r in resp)
    t0 = time.perf_counter()
    got, n_active, _ = ingest_responses(resp, b.group_off)
    dt = time.perf_counter() - t0
    assert n_active == sh.n_active and np.array_equal(got.ids, b.ids)
    print(f"ingest: {nbytes / 1e6:.1f} MB, {len(b.ids) / 1e6:.2f} M tokens in {dt * 1e3:.1f} ms "
          f"({nbytes / dt / 1e9:.2f} GB/s)")
    assert nbytes / dt > 50e6
