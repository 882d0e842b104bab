"""The synthetic workload built with the REFERENCE's own compiled code — for the
CPU arm of the bench (bench.py --impl reference / cpu_baseline). TEST
INFRASTRUCTURE ONLY; never imported by the product.

Everything the reference owns comes from oracle/_ref/libref.so (compiled in
place from /root/reference by oracle/build_ref.sh, shipped prebuilt to the GPU
box):
  * rewards: trainer::generate_workload (proj/src/trainer/workload.cpp:62-107);
  * token ids / behaviour logprobs: mock::hash_token / token_logprob
    (proj/src/mock/policy.cpp:42-53);
  * each rollout's packed sequence: TokenTrajectory::append (validate) +
    flatten (proj/include/rollout/trajectory.hpp:67-99);
  * FAILED exclusion + zero-variance gate: PromptGroup::usable_rewards /
    is_informative (proj/src/trainer/harness.cpp:84-102).
The synthetic choices the reference does not make (turn structure, the ~2 %
FAILED pattern, config sizes) come from paper_2603_18815_b200/synth_spec.py,
which is pure Python (it loads no native code). The product library is not
loaded on this path. tests/test_oracle_golden.py checks that the batch built
here equals the product's synth.make_shard batch bit for bit.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from oracle import oracle as O
from paper_2603_18815_b200 import synth_spec as S

TURN_DTYPE = np.dtype([("src_off", "<i8"), ("traj", "<i4"), ("len", "<i4"), ("role", "u1"), ("pad", "u1", (7,))])


@dataclass
class RefBatch:
    turns: np.ndarray
    ids: np.ndarray
    lp: np.ndarray
    reward: np.ndarray
    usable: np.ndarray
    group_off: np.ndarray
    rollout_key: np.ndarray
    n_active: int
    groups: list


def _p(a):
    return a.ctypes.data


def build(config: str | dict, seed: int | None = None) -> RefBatch:
    """All informative groups of `config` (the global batch of one step), in
    prompt order, with the reference's generators and rules."""
    R = O.ref_lib()
    if R is None:
        raise RuntimeError("oracle/_ref/libref.so is not built (oracle/build_ref.sh needs /root/reference)")
    cfg = dict(S.CONFIGS[config]) if isinstance(config, str) else dict(config)
    seed = 2603 + cfg.get("index", 0) if seed is None else seed
    G, n, V = cfg["tasks"], cfg["group"], cfg["vocab"]
    rewards = np.zeros(G * n, np.float64)
    assert R.ref_generate_workload_rewards(G, n, seed, 0.5, _p(rewards)) == 0
    rewards = rewards.reshape(G, n)
    failed = S.failed_matrix(seed, G, n)
    turns, ids, lps, reward, usable, goff, rkey, groups = [], [], [], [], [], [0], [], []
    src = seq = n_active = 0
    has = np.ones(n, np.int32)
    for g in range(G):
        fl = failed[g].astype(np.int32)
        rw = np.ascontiguousarray(rewards[g])
        info = R.ref_is_informative(n, _p(has), _p(fl), _p(rw), 0.0)
        if info != 1:
            continue
        groups.append(g)
        for j in range(n):
            key = g * n + j
            reward.append(rw[j])
            rkey.append(key)
            usable.append(0 if fl[j] else 1)
            if not fl[j]:
                roles, lens = S.turn_structure(cfg, seed, key)
                L = int(sum(lens))
                tid = np.zeros(L, np.int64)
                tlp = np.zeros(L, np.float64)
                prompt = np.array([key], np.int64)
                R.ref_hash_tokens(seed, _p(prompt), 1, 0, L, V, _p(tid), _p(tlp))
                lp = np.where(np.repeat(np.array(roles) == S.ROLE_ASSISTANT, lens), tlp, 0.0)
                # the packed sequence is the reference's TokenTrajectory::flatten()
                ro = np.array(roles, np.int32)
                le = np.array(lens, np.int64)
                flat = np.zeros(L, np.int64)
                got = R.ref_flatten(len(roles), _p(ro), _p(le), _p(tid), _p(lp), 0, len(roles), _p(flat), L)
                assert got == L, "reference TokenTrajectory rejected a synthetic turn"
                pos = 0
                for r, ln in zip(roles, lens):
                    turns.append((src, seq, ln, r))
                    src += ln
                    if r == S.ROLE_ASSISTANT and ln > 0:
                        n_active += ln - (1 if pos == 0 else 0)
                    pos += ln
                ids.append(flat)
                lps.append(lp)
            seq += 1
        goff.append(seq)
    t = np.zeros(len(turns), TURN_DTYPE)
    if turns:
        arr = np.array(turns, np.int64)
        t["src_off"], t["traj"], t["len"], t["role"] = arr[:, 0], arr[:, 1], arr[:, 2], arr[:, 3]
    return RefBatch(turns=t, ids=np.concatenate(ids) if ids else np.zeros(0, np.int64),
                    lp=np.concatenate(lps) if lps else np.zeros(0, np.float64),
                    reward=np.array(reward, np.float64), usable=np.array(usable, np.uint8),
                    group_off=np.array(goff, np.int32), rollout_key=np.array(rkey, np.int64), n_active=n_active,
                    groups=groups)


def host_batch(b: RefBatch):
    return O.host_batch(b.turns, b.ids, b.lp, b.reward, b.usable, b.group_off, b.rollout_key)
