"""Synthetic workload SPECIFICATION for the BASELINE.json configs — pure
Python/numpy, no native code: the product's synth.py (which builds shards with
the product library) and the reference arm's builder (oracle/ref_workload.py,
which builds the same shards with the reference's own compiled generators)
share these definitions.

  * token ids: hash_token(seed, [rollout_key], k) mod V (mock/policy.cpp:42-49),
    behaviour logprobs token_logprob(id) (mock/policy.cpp:51-53);
  * ~2 % FAILED rollouts (exercising usable_rewards, harness.cpp:84-90);
  * turn structure: a user prompt (~10 % of tokens), then alternating
    assistant / tool turns (tool observations appended as in
    handlers.cpp:292-293) with the config's assistant share.
"""
from __future__ import annotations

import math

import numpy as np

# rollout::Role order (trajectory.hpp:11) == PRORL_ROLE_*
ROLE_SYSTEM, ROLE_USER, ROLE_ASSISTANT, ROLE_TOOL = 0, 1, 2, 3

FNV_OFFSET = np.uint64(14695981039346656037)
FNV_PRIME = np.uint64(1099511628211)

# BASELINE.json configs (index = position in "configs"); seed = 2603 + index.
CONFIGS = {
    "c1": dict(index=0, tasks=4, group=4, tokens=1024, turns=6, vocab=32000, dtype="fp32", asst_share=0.5,
               lengths="fixed", desc="16 trajectories (4 tasks x group 4), ~1K tokens, 6 turns, vocab 32000, fp32"),
    "c2": dict(index=1, tasks=64, group=8, tokens=8192, turns=12, vocab=151936, dtype="bf16", asst_share=0.4,
               lengths="fixed", desc="Qwen3-4B-shaped: 64 tasks x group 8, 8K-token multi-turn SWE trajectories, "
                                     "vocab 151936, bf16 logits"),
    "c3": dict(index=2, tasks=128, group=8, tokens=16384, turns=30, vocab=151936, dtype="bf16", asst_share=0.22,
               lengths="fixed", desc="Qwen3-8B-shaped: 128 tasks x group 8, 16K tokens, ~30 turns, heavy "
                                     "tool-observation masking"),
    "c4": dict(index=3, tasks=256, group=16, tokens=32768, turns=24, vocab=151936, dtype="bf16", asst_share=0.3,
               lengths="lognormal", desc="Qwen3-14B-shaped: 256 tasks x group 16, 32K-token trajectories, skewed "
                                         "lengths, 8-GPU group-sharded"),
}


def _fnv_u64(state, v):
    """FNV-1a over the 8 little-endian bytes of v (policy.cpp:21-25); vectorised."""
    v = np.asarray(v, dtype=np.uint64)
    s = np.asarray(state, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for i in range(8):
            s = (s ^ ((v >> np.uint64(8 * i)) & np.uint64(0xFF))) * FNV_PRIME
    return s


def hash_tokens(seed: int, prompt: list[int], ks: np.ndarray, vocab: int) -> np.ndarray:
    """mock::hash_token(seed, prompt, k, vocab) for a vector of k (policy.cpp:42-49)."""
    s = _fnv_u64(FNV_OFFSET, np.uint64(seed))
    for pid in prompt:
        s = _fnv_u64(s, np.uint64(pid))
    s = _fnv_u64(np.full(len(ks), s, dtype=np.uint64), ks.astype(np.uint64))
    return (s % np.uint64(vocab)).astype(np.int64)


def token_logprob(ids: np.ndarray) -> np.ndarray:
    """mock::token_logprob (policy.cpp:51-53)."""
    return -(1.0 + (ids % 7).astype(np.float64) / 10.0)


def _mix(*xs: int) -> int:
    h = 0x9E3779B97F4A7C15
    for x in xs:
        h ^= (x + 0x9E3779B97F4A7C15 + ((h << 6) & 0xFFFFFFFFFFFFFFFF) + (h >> 2)) & 0xFFFFFFFFFFFFFFFF
        h = (h * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        h ^= h >> 31
    return h


def is_informative(rewards: np.ndarray, failed: np.ndarray, tol: float = 0.0) -> bool:
    """harness.cpp:92-102 over a complete group."""
    u = rewards[~failed]
    return len(u) >= 2 and float(u.max() - u.min()) > tol


def rollout_lengths(cfg: dict, seed: int, key: int) -> int:
    if cfg["lengths"] == "lognormal":
        # skewed: log-normal with mean ~cfg tokens, clamped to [1K, 64K]
        u1 = (_mix(seed, key, 11) >> 11) / float(1 << 53)
        u2 = (_mix(seed, key, 12) >> 11) / float(1 << 53)
        z = math.sqrt(-2.0 * math.log(max(u1, 1e-300))) * math.cos(2 * math.pi * u2)
        sig = 0.6
        mu = math.log(cfg["tokens"]) - 0.5 * sig * sig
        return int(min(max(math.exp(mu + sig * z), 1024), 65536))
    return int(cfg["tokens"])



def turn_structure(cfg: dict, seed: int, key: int) -> tuple[list[int], list[int]]:
    """(roles, lens) of one rollout's trajectory (PRORL_ROLE_* codes)."""
    L = rollout_lengths(cfg, seed, key)
    n_turns = max(2, int(cfg["turns"]))
    prompt = max(1, int(round(0.10 * L)))
    rest = L - prompt
    n_asst = (n_turns - 1 + 1) // 2
    n_tool = (n_turns - 1) - n_asst
    asst_total = int(round(cfg["asst_share"] * L))
    asst_total = min(max(asst_total, n_asst), rest - n_tool) if n_tool > 0 else rest
    tool_total = rest - asst_total

    def split(total, parts, salt):
        if parts <= 0:
            return []
        w = np.array([1.0 + ((_mix(seed, key, salt, i) >> 40) / float(1 << 24)) for i in range(parts)])
        raw = np.floor(w / w.sum() * total).astype(np.int64)
        raw = np.maximum(raw, 1 if total >= parts else 0)
        raw[-1] = total - raw[:-1].sum()
        return list(raw)

    a_lens = split(asst_total, n_asst, 1)
    t_lens = split(tool_total, n_tool, 2)
    roles, lens = [ROLE_USER], [prompt]
    for i in range(n_asst):
        roles.append(ROLE_ASSISTANT)
        lens.append(int(a_lens[i]))
        if i < n_tool:
            roles.append(ROLE_TOOL)
            lens.append(int(t_lens[i]))
    return roles, lens


def failed_matrix(seed: int, G: int, n: int) -> np.ndarray:
    """~2 % FAILED rollouts, deterministic in (seed, group, slot)."""
    return np.array([[(_mix(seed, g, j, 7) % 50) == 0 for j in range(n)] for g in range(G)], dtype=bool)
