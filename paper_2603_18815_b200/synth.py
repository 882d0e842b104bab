"""Synthetic trainer-side batches for the BASELINE.json configs.

What the rollout server would hand the trainer after an iteration
(IterationStats::informative, proj/include/rollout/trainer/harness.hpp:75):
prompt groups whose rollouts carry token-level multi-turn trajectories.

  * rewards: the reference's workload semantics (trainer/workload.cpp:62-107)
    via prorl_synth_rewards (identical values under libstdc++), plus ~2 %
    FAILED rollouts (exercising usable_rewards, harness.cpp:84-90);
  * only informative groups are packed (is_informative, harness.cpp:92-102);
  * turn structure: a user prompt (~10 % of tokens), then alternating
    assistant / tool turns (tool observations appended as in
    handlers.cpp:292-293) with the config's assistant share;
  * token ids: hash_token(seed, [rollout_key], k) mod V (mock/policy.cpp:42-49),
    behaviour logprobs token_logprob(id) (mock/policy.cpp:51-53).

Everything is a deterministic function of (config, seed, rank, world).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .hotpath import HostBatchArrays, shard_lpt, synth_rewards
from .synth_spec import (CONFIGS, _mix, failed_matrix, hash_tokens, is_informative, rollout_lengths,  # noqa: F401
                         token_logprob, turn_structure)


@dataclass
class Shard:
    batch: HostBatchArrays
    groups: list[int]                 # global group (prompt) indices packed on this rank
    n_active: int
    turns_per_rollout: list[int] = field(default_factory=list)


def trajectory(cfg: dict, seed: int, key: int, vocab: int):
    """(roles, lens, ids, lp) of one rollout's token-level trajectory."""
    roles, lens = turn_structure(cfg, seed, key)
    L = int(sum(lens))
    ids = hash_tokens(seed, [key], np.arange(L, dtype=np.uint64), vocab)
    lp = np.zeros(L, dtype=np.float64)
    off = 0
    for r, n in zip(roles, lens):
        if r == N.ROLE_ASSISTANT:
            lp[off:off + n] = token_logprob(ids[off:off + n])
        off += n
    return roles, lens, ids, lp


def make_shard(config: str | dict, rank: int = 0, world: int = 1, seed: int | None = None,
               max_groups: int | None = None, tokens: int | None = None) -> Shard:
    cfg = dict(CONFIGS[config]) if isinstance(config, str) else dict(config)
    if tokens is not None:
        cfg["tokens"] = tokens
    seed = 2603 + cfg.get("index", 0) if seed is None else seed
    G, n, V = cfg["tasks"], cfg["group"], cfg["vocab"]
    rewards = synth_rewards(G, n, seed, 0.5)
    failed = failed_matrix(seed, G, n)
    informative = [g for g in range(G) if is_informative(rewards[g], failed[g])]
    if max_groups is not None:
        informative = informative[:max_groups]
    # LPT over ranks by active-token estimate (deterministic; harness hands
    # groups over in completion order, we sort by prompt index, App. B.1)
    if world > 1:
        load = np.array([sum(rollout_lengths(cfg, seed, g * n + j) for j in range(n) if not failed[g, j])
                         for g in informative], dtype=np.int64)
        owner = shard_lpt(load, world)
        mine = [g for g, o in zip(informative, owner) if o == rank]
    else:
        mine = informative
    turns, ids, lps = [], [], []
    reward, usable, goff, rkey = [], [], [0], []
    src = 0
    seq = 0
    tpr = []
    for g in mine:
        for j in range(n):
            reward.append(rewards[g, j])
            rkey.append(g * n + j)
            usable.append(0 if failed[g, j] else 1)
            if not failed[g, j]:
                roles, lens, tid, tlp = trajectory(cfg, seed, g * n + j, V)
                for r, L in zip(roles, lens):
                    turns.append((src, seq, L, r))
                    src += L
                ids.append(tid)
                lps.append(tlp)
                tpr.append(len(roles))
            seq += 1
        goff.append(seq)
    t = np.zeros(len(turns), dtype=N.TURN_DTYPE)
    if turns:
        arr = np.array(turns, dtype=np.int64)
        t["src_off"], t["traj"], t["len"], t["role"] = arr[:, 0], arr[:, 1], arr[:, 2], arr[:, 3]
    batch = HostBatchArrays(
        turns=t,
        ids=np.concatenate(ids) if ids else np.zeros(0, np.int64),
        lp=np.concatenate(lps) if lps else np.zeros(0, np.float64),
        reward=np.array(reward, dtype=np.float64),
        usable=np.array(usable, dtype=np.uint8),
        group_off=np.array(goff, dtype=np.int32),
        rollout_key=np.array(rkey, dtype=np.int64),
    )
    return Shard(batch=batch, groups=mine, n_active=count_active(t), turns_per_rollout=tpr)


def count_active(turns: np.ndarray) -> int:
    """Active rows (App. B.1): policy tokens at position > 0 of their sequence."""
    n, cur, pos = 0, -1, 0
    for tr, L, r in zip(turns["traj"], turns["len"], turns["role"]):
        if tr != cur:
            cur, pos = tr, 0
        if r == N.ROLE_ASSISTANT and L > 0:
            n += int(L) - (1 if pos == 0 else 0)
        pos += int(L)
    return n
