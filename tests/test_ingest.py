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
    # the harness never records a CANCELLED response (harness.cpp:264: the slot
    # is re-issued), so a shard never holds one (see test_cancelled_response_...)
    cases = [c for c in GOLD["process_response"] if c["status"] != "CANCELLED"]
    group_off = list(range(0, len(cases) + 1, group_size))
    if group_off[-1] != len(cases):
        group_off.append(len(cases))
    b, n_active, n_info = ingest_responses([c["json"].encode() for c in cases], group_off)
    exp = _expected(cases, group_off)
    _check(b, exp)
    assert n_active == exp[5]


def test_cancelled_response_makes_the_group_incomplete():
    cancelled = [c for c in GOLD["process_response"] if c["status"] == "CANCELLED"]
    done = [c for c in GOLD["process_response"] if c["status"] == "DONE"]
    assert cancelled and done
    with pytest.raises(RolloutError) as e:
        ingest_responses([done[0]["json"].encode(), cancelled[0]["json"].encode()], [0, 2])
    assert e.value.code == "incomplete_group"


def test_missing_status_reads_as_failed():
    """harness.cpp:263: response.value("status", "FAILED")."""
    ok = b'{"status":"DONE","reward":1,"trajectory":[{"role":"user","input_ids":[1]},' \
         b'{"role":"assistant","output_ids":[2,3],"logprobs":[-1.0,-1.1]}]}'
    no_status = b'{"reward":0,"trajectory":[{"role":"user","input_ids":[1]}]}'
    no_status_no_traj = b'{"reward":0.5}'
    b, n_active, n_info = ingest_responses([ok, no_status, no_status_no_traj], [0, 3])
    assert b.usable.tolist() == [1, 0, 0]
    assert n_info == 0 and n_active == 0  # one usable reward: not informative


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


def _turn_json(role, ids, lps_text=None):
    if role == "assistant":
        return (f'{{"input_ids":[],"logprobs":[{",".join(lps_text)}],"output_ids":[{",".join(map(str, ids))}],'
                f'"role":"assistant"}}')
    return f'{{"input_ids":[{", ".join(map(str, ids))}],"logprobs":[],"output_ids":[],"role":"{role}"}}'


def test_logprob_decimal_parsing_is_exact():
    """Every decimal shape a serialiser produces (shortest repr of doubles and of
    float32 values, %.17g, exponents, 19+ digits, -0.0) parses to the double
    Python's float() gives — bit-exact, including the x87 fast path's fallbacks."""
    rng = np.random.default_rng(7)
    vals = np.concatenate([
        -rng.exponential(2.0, 4000),
        -rng.exponential(2.0, 4000).astype(np.float32).astype(np.float64),
        -(10.0 ** rng.uniform(-12, 2, 4000)),
        np.round(-rng.exponential(2.0, 2000), 4),
    ])
    texts = []
    for k, v in enumerate(vals):
        m = k % 5
        texts.append(repr(float(v)) if m < 2 else ("%.17g" % v if m == 2 else
                     ("%.19f" % v if m == 3 else "%.21e" % v)))
    texts += ["-0.0", "0", "-1", "-1e-300", "-2.2250738585072014e-308", "-123456789012345678901234.5",
              "-0.00000000000000000000000000123", "-1.0000000000000002", "-0.99999999999999999999"]
    want = [float(t) for t in texts]
    ids = list(range(1, len(texts) + 1))
    resp = (f'{{"status":"DONE","reward":1,"trajectory":[{_turn_json("user", [5])},'
            f'{_turn_json("assistant", ids, texts)}]}}').encode()
    other = b'{"status":"DONE","reward":0,"trajectory":[{"role":"user","input_ids":[1]}]}'
    b, _, _ = ingest_responses([resp, other], [0, 2])
    got = b.lp[1:1 + len(texts)]
    assert np.array_equal(got.view(np.uint64), np.array(want).view(np.uint64))


def test_failed_members_are_compacted_out():
    """FAILED rollouts inside an informative group are dropped from the token
    stream (harness.cpp:84-90) while the group keeps their reward slots."""
    def resp(status, reward, ids):
        return (f'{{"status":"{status}","reward":{reward},"trajectory":[{_turn_json("user", ids[:2])},'
                f'{_turn_json("assistant", ids[2:], [repr(-0.5 - 0.1 * i) for i in range(len(ids) - 2)])}]}}').encode()
    rs = [resp("FAILED", 1.0, [9, 9, 9, 9]), resp("DONE", 1.0, [1, 2, 3, 4, 5]), resp("FAILED", 0.0, [8, 8, 8]),
          resp("DONE", 0.0, [6, 7, 8]), resp("FAILED", 0.5, [7, 7, 7, 7, 7])]
    b, n_active, n_info = ingest_responses(rs, [0, 5], threads=1)
    assert n_info == 1
    assert b.ids.tolist() == [1, 2, 3, 4, 5, 6, 7, 8]
    assert [(int(t["src_off"]), int(t["traj"]), int(t["len"])) for t in b.turns] == [(0, 1, 2), (2, 1, 3), (5, 3, 2), (7, 3, 1)]
    assert b.usable.tolist() == [0, 1, 0, 1, 0]
    assert n_active == 3 + 1
    assert b.lp.tolist() == [0.0, 0.0, -0.5, -0.6, -0.7, 0.0, 0.0, -0.5]


@pytest.mark.parametrize("n_threads", [1, 2, 3, 8])
def test_thread_split_is_invariant(n_threads):
    from tests.wire import to_responses
    sh = synth.make_shard("c1", seed=11)
    b = sh.batch
    resp = to_responses(b)
    got, n_active, n_info = ingest_responses(resp, b.group_off, threads=n_threads)
    ref, n_active1, n_info1 = ingest_responses(resp, b.group_off, threads=1)
    assert (n_active, n_info) == (n_active1, n_info1)
    for f in ("ids", "lp", "reward", "usable"):
        assert np.array_equal(getattr(got, f), getattr(ref, f)), f
    assert np.array_equal(got.turns, ref.turns)
