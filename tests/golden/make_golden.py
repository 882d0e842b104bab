"""Generate tests/golden/reference_vectors.json from the REFERENCE ITSELF.

Run in the container that has /root/reference (the compiled reference is
oracle/_ref/libref.so, built by oracle/build_ref.sh from the unmodified
sources). The JSON is committed so the GPU box — which has no
/root/reference — can pin the oracle and the product against it.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import random
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402


def main() -> None:
    O.build(ref=True)
    R = O.ref_lib()
    assert R is not None, "reference library not built"
    rng = random.Random(2603)
    out: dict = {"source": "oracle/_ref/libref.so compiled from /root/reference/proj (trajectory.hpp, "
                           "trainer/harness.cpp, trainer/workload.cpp, mock/policy.cpp)"}

    # flatten / flatten_range on random well-formed trajectories (trajectory.hpp:76-87)
    flat = []
    for case in range(40):
        n_turns = rng.randint(0, 9)
        roles = [rng.choice([0, 1, 2, 3]) for _ in range(n_turns)]
        lens = [rng.randint(0, 6) for _ in range(n_turns)]
        ids = [rng.randint(0, 50000) for _ in range(sum(lens))]
        lps = [-(1.0 + (t % 7) / 10.0) for t in ids]
        b = rng.randint(0, max(n_turns, 1))
        e = rng.randint(b, n_turns + 2)
        buf = np.zeros(max(sum(lens), 1), np.int64)
        a = lambda x, dt: np.ascontiguousarray(x, dt)
        r_, l_, i_, p_ = a(roles, np.int32), a(lens, np.int64), a(ids, np.int64), a(lps, np.float64)
        n = R.ref_flatten(n_turns, r_.ctypes.data, l_.ctypes.data, i_.ctypes.data, p_.ctypes.data, b, e,
                          buf.ctypes.data, len(buf))
        full = np.zeros(max(sum(lens), 1), np.int64)
        nf = R.ref_flatten(n_turns, r_.ctypes.data, l_.ctypes.data, i_.ctypes.data, p_.ctypes.data, 0, n_turns,
                           full.ctypes.data, len(full))
        flat.append({"roles": roles, "lens": lens, "ids": ids, "begin": b, "end": e,
                     "flatten_range": buf[:n].tolist(), "flatten": full[:nf].tolist()})
    out["flatten"] = flat

    # validate (trajectory.hpp:89-99)
    val = []
    for role in range(4):
        for ni in (0, 2):
            for no in (0, 2):
                for nl in (0, 1, 2):
                    val.append({"role": role, "n_input": ni, "n_output": no, "n_logprobs": nl,
                                "malformed": R.ref_validate_turn(role, ni, no, nl)})
    out["validate"] = val

    # usable_rewards / is_informative (harness.cpp:84-102)
    inf = []
    for case in range(200):
        n = rng.randint(1, 8)
        has = [1 if rng.random() > 0.08 else 0 for _ in range(n)]
        failed = [1 if rng.random() < 0.2 else 0 for _ in range(n)]
        rew = [rng.choice([0.0, 1.0, 0.5, 0.25]) for _ in range(n)]
        tol = rng.choice([0.0, 0.0, 0.1, 0.5])
        h, f, w = (np.ascontiguousarray(x, dt) for x, dt in ((has, np.int32), (failed, np.int32), (rew, np.float64)))
        ub = np.zeros(n)
        nu = R.ref_usable_rewards(n, h.ctypes.data, f.ctypes.data, w.ctypes.data, ub.ctypes.data)
        inf.append({"has": has, "failed": failed, "rewards": rew, "tol": tol, "usable": ub[:nu].tolist(),
                    "informative": R.ref_is_informative(n, h.ctypes.data, f.ctypes.data, w.ctypes.data, tol)})
    out["informative"] = inf

    # mock policy generators (policy.cpp:10-53)
    fnv = []
    for s in ["", "a", "foobar", "prorl", "rollout-as-a-service"]:
        b = s.encode()
        buf = np.frombuffer(b, np.uint8) if b else np.zeros(1, np.uint8)
        fnv.append({"s": s, "fnv1a64": str(R.ref_fnv1a64(buf.ctypes.data, len(b)))})
    out["fnv1a64"] = fnv
    ht = []
    for case in range(60):
        seed = rng.randint(0, 2**63)
        prompt = [rng.randint(0, 2**40) for _ in range(rng.randint(0, 5))]
        k = rng.randint(0, 10000)
        V = rng.choice([32000, 50000, 151936, 262144, 7])
        p = np.ascontiguousarray(prompt or [0], np.int64)
        ht.append({"seed": str(seed), "prompt": prompt, "k": k, "vocab": V,
                   "token": R.ref_hash_token(seed, p.ctypes.data, len(prompt), k, V)})
    out["hash_token"] = ht
    out["token_logprob"] = [{"t": t, "lp": R.ref_token_logprob(t)} for t in range(0, 30)]

    # workload rewards (workload.cpp:62-107)
    wl = []
    for seed, P, n in [(0, 4, 4), (2603, 4, 4), (2604, 64, 8), (2605, 128, 8), (2606, 16, 16), (7, 9, 1), (11, 5, 32)]:
        buf = np.zeros(P * n)
        R.ref_generate_workload_rewards(P, n, seed, 0.5, buf.ctypes.data)
        wl.append({"seed": seed, "num_prompts": P, "n": n, "rewards": buf.tolist()})
    out["workload"] = wl

    # /process wire JSON produced by the reference's build_process_response (handlers.cpp:57-91)
    import ctypes as C
    resp = []
    for case in range(24):
        n_turns = rng.randint(0, 7)
        roles = [rng.choice([0, 1, 2, 3]) for _ in range(n_turns)]
        lens = [rng.randint(0, 5) for _ in range(n_turns)]
        ids = [rng.randint(0, 151935) for _ in range(sum(lens))]
        lps = [round(-rng.random() * 5, rng.choice([1, 3, 17])) for _ in ids]
        status = rng.choice([0, 0, 0, 1, 2])
        reward = rng.choice([0.0, 1.0, 0.5])
        a = lambda x, dt: np.ascontiguousarray(x or [0], dt)
        r_, l_, i_, p_ = a(roles, np.int32), a(lens, np.int64), a(ids, np.int64), a(lps, np.float64)
        buf = C.create_string_buffer(1 << 16)
        n = R.ref_process_response(f"job-{case}".encode(), n_turns, r_.ctypes.data, l_.ctypes.data, i_.ctypes.data,
                                   p_.ctypes.data, reward, status, b"http://10.0.0.1:8000" if case % 2 else b"",
                                   buf, len(buf))
        resp.append({"roles": roles, "lens": lens, "ids": ids, "logprobs": lps, "reward": reward,
                     "status": ["DONE", "FAILED", "CANCELLED"][status], "json": buf.raw[:n].decode()})
    out["process_response"] = resp

    path = Path(__file__).with_name("reference_vectors.json")
    path.write_text(json.dumps(out, indent=None, separators=(",", ":")))
    print(path, path.stat().st_size)


if __name__ == "__main__":
    main()
