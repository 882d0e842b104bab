"""Parity of the sm_100a path (through the C-ABI) against the CPU oracle.

Tolerances (north star; tests/parity.py): packing, masks,
cu_seqlens, turn/seq/pos ids and active-row lists bit-exact; per-row logp /
entropy 1e-5 relative with floor 1e-3; advantages and every partial sum 1e-5
relative with floor 0; counts exact (clip counts up to the oracle's
borderline rows).
"""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2603_18815_b200 import _native as N
from paper_2603_18815_b200 import synth
from paper_2603_18815_b200.hotpath import HostBatchArrays, LossConfig, RolloutError, ScoreConfig
from tests.parity import assert_partials_close, assert_rows_close

pytestmark = pytest.mark.gpu

def dev(a, d):
    return torch.from_numpy(np.ascontiguousarray(a)).to(d)


def device_pack(scorer, b: HostBatchArrays, vocab, n_active, d):
    return scorer.pack(b.turns, dev(b.ids, d), dev(b.lp, d), b.n_rollouts, vocab, n_active)


def compare_pack(gpu, ora):
    for k in ("tokens", "loss_mask", "turn_id", "seq_id", "pos_id", "old_lp", "cu_seqlens", "act_row",
              "act_target", "act_old_lp", "act_seq", "act_turn"):
        g = gpu[k].cpu().numpy()
        o = ora[k]
        assert g.dtype == o.dtype, k
        assert g.shape == o.shape, (k, g.shape, o.shape)
        assert np.array_equal(g.view(np.uint8), o.view(np.uint8)), k  # bitwise (fp32 incl.)
    assert int(gpu["n_active"].item()) == ora["n_active"]


# ---------------------------------------------------------------- K1 pack
@pytest.mark.parametrize("config,kw", [("c1", {}), ("c2", {"max_groups": 3}), ("c3", {"max_groups": 2}),
                                       ("c4", {"max_groups": 1})])
def test_pack_bitexact_configs(scorer, cuda, config, kw):
    sh = synth.make_shard(config, **kw)
    b = sh.batch
    V = synth.CONFIGS[config]["vocab"]
    st, ora = O.pack(b.turns, b.ids, b.lp, b.n_rollouts, V)
    assert st == 0 and ora["n_active"] == sh.n_active
    compare_pack(device_pack(scorer, b, V, sh.n_active, cuda), ora)


def test_pack_bitexact_full_c2(scorer, cuda):
    """Full Qwen3-4B-shaped batch (2.26 M tokens): the packer is cheap on CPU, so bit-exact in full."""
    sh = synth.make_shard("c2")
    b = sh.batch
    st, ora = O.pack(b.turns, b.ids, b.lp, b.n_rollouts, 151936)
    assert st == 0
    compare_pack(device_pack(scorer, b, 151936, sh.n_active, cuda), ora)


def _edge_batch(rng):
    """Ragged edge cases: empty / FAILED (0-turn) slots, zero-length turns,
    assistant-first trajectories, 1-token trajectories, long turns."""
    turns, ids, lps = [], [], []
    src = 0
    n_seq = 9
    specs = {
        0: [(N.ROLE_ASSISTANT, 5), (N.ROLE_TOOL, 3), (N.ROLE_ASSISTANT, 2)],   # assistant first
        1: [],                                                                # FAILED slot
        2: [(N.ROLE_USER, 4), (N.ROLE_ASSISTANT, 0), (N.ROLE_TOOL, 0), (N.ROLE_ASSISTANT, 3)],
        3: [(N.ROLE_USER, 1)],
        4: [(N.ROLE_ASSISTANT, 1)],
        5: [(N.ROLE_SYSTEM, 2), (N.ROLE_USER, 3)] + [(N.ROLE_ASSISTANT, 7), (N.ROLE_TOOL, 11)] * 40,
        6: [],
        7: [(N.ROLE_USER, 5000), (N.ROLE_ASSISTANT, 9000), (N.ROLE_TOOL, 1)],
        8: [(N.ROLE_USER, 2), (N.ROLE_ASSISTANT, 1)],
    }
    for s in range(n_seq):
        for role, L in specs[s]:
            turns.append((src, s, L, role))
            ids.append(rng.integers(0, 32000, L))
            lps.append(-rng.random(L) * 3 if role == N.ROLE_ASSISTANT else np.zeros(L))
            src += L
    t = np.zeros(len(turns), N.TURN_DTYPE)
    arr = np.array(turns, np.int64)
    t["src_off"], t["traj"], t["len"], t["role"] = arr[:, 0], arr[:, 1], arr[:, 2], arr[:, 3]
    return t, np.concatenate(ids).astype(np.int64), np.concatenate(lps), n_seq


def test_pack_edge_cases(scorer, cuda):
    t, ids, lp, n_seq = _edge_batch(np.random.default_rng(3))
    st, ora = O.pack(t, ids, lp, n_seq, 32000)
    assert st == 0
    compare_pack(scorer.pack(t, dev(ids, cuda), dev(lp, cuda), n_seq, 32000, ora["n_active"]), ora)
    # turn ordinals past the 64-bucket range are kept (bucket folding is K4's job)
    assert ora["turn_id"].max() >= 39


def test_pack_empty(scorer, cuda):
    t = np.zeros(0, N.TURN_DTYPE)
    out = scorer.pack(t, torch.zeros(0, dtype=torch.int64, device=cuda), torch.zeros(0, dtype=torch.float64,
                      device=cuda), 3, 100, 0)
    assert out["cu_seqlens"].cpu().tolist() == [0, 0, 0, 0]
    assert int(out["n_active"].item()) == 0


def test_pack_token_out_of_range_fails_loudly(scorer, cuda):
    t, ids, lp, n_seq = _edge_batch(np.random.default_rng(4))
    ids[17] = 32000
    with pytest.raises(RolloutError) as e:
        scorer.pack(t, dev(ids, cuda), dev(lp, cuda), n_seq, 32000, 1)
    assert e.value.code == "shape_mismatch"
    ids[17] = -5
    with pytest.raises(RolloutError):
        scorer.pack(t, dev(ids, cuda), dev(lp, cuda), n_seq, 32000, 1)


def test_pack_unsorted_turns_fail(scorer, cuda):
    t, ids, lp, n_seq = _edge_batch(np.random.default_rng(5))
    t2 = t.copy()
    t2["traj"][0], t2["traj"][-1] = t["traj"][-1], t["traj"][0]
    assert O.pack(t2, ids, lp, n_seq, 32000)[0] == -12  # PRORL_E_SHAPE
    with pytest.raises(RolloutError) as e:
        scorer.pack(t2, dev(ids, cuda), dev(lp, cuda), n_seq, 32000, 1)
    assert e.value.code == "shape_mismatch"


# ---------------------------------------------------------------- K3 grpo
@pytest.mark.parametrize("ddof", [0, 1])
def test_grpo_vs_oracle(scorer, cuda, ddof):
    rng = np.random.default_rng(11 + ddof)
    sizes = rng.integers(1, 40, 300)
    goff = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    R = int(goff[-1])
    reward = rng.choice([0.0, 1.0, 0.5, 0.25, 0.75], R)
    reward[:goff[5]] = 1.0  # a few uniform (non-informative) groups
    usable = (rng.random(R) > 0.1).astype(np.uint8)
    partials = torch.zeros(N.N_PARTIALS, dtype=torch.float64, device=cuda)
    adv, info = scorer.grpo_adv(dev(reward, cuda), dev(usable, cuda), dev(goff, cuda), ddof=ddof, partials=partials)
    oadv, oinfo, asum, nr = O.grpo(reward, usable, goff, ddof=ddof)
    assert info.cpu().numpy().tolist() == oinfo.tolist()
    g = adv.cpu().numpy()
    assert g.dtype == np.float64
    assert np.all(np.abs(g - oadv) <= 1e-5 * np.abs(oadv))  # floor 0 (App. B.7); zeros exact
    p = partials.cpu().numpy()
    assert p[N.P_N_ROLLOUTS] == nr
    assert abs(p[N.P_ADV_SUM] - asum) <= 1e-5 * nr


def test_grpo_reward_gate_matches_reference_semantics(scorer, cuda):
    # test_trainer.cpp:148-166 restated on the device gate
    groups = [([1, 1, 1, 1], [1, 1, 1, 1]), ([1, 0, 1, 1], [1, 1, 1, 1]), ([1, 1, 0, 1], [1, 1, 0, 1]),
              ([1, 0], [1, 0]), ([0.0, 0.1], [1, 1])]
    reward = np.concatenate([g[0] for g in groups]).astype(np.float64)
    usable = np.concatenate([g[1] for g in groups]).astype(np.uint8)
    goff = np.concatenate([[0], np.cumsum([len(g[0]) for g in groups])]).astype(np.int32)
    _, info = scorer.grpo_adv(dev(reward, cuda), dev(usable, cuda), dev(goff, cuda))
    assert info.cpu().tolist() == [0, 1, 0, 0, 1]
    _, info = scorer.grpo_adv(dev(reward, cuda), dev(usable, cuda), dev(goff, cuda), tol=0.1)
    assert info.cpu().tolist() == [0, 1, 0, 0, 0]


# ---------------------------------------------------------------- K2 logprob / entropy
def _logits_pair(n_rows, V, dtype, cuda, scorer, seed=5, stride=None, targets=None, old_lp=None, key0=0):
    stride = stride or V
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    x = torch.empty((n_rows, stride), dtype=tdt, device=cuda)
    tg = None if targets is None else dev(targets.astype(np.int32), cuda)
    ol = None if old_lp is None else dev(old_lp.astype(np.float32), cuda)
    scorer.gen_logits(x, n_rows, key0, tg, ol, seed=seed, sigma=2.0, vocab=V)
    host = O.gen_logits(n_rows, V, key0, targets, old_lp, seed=seed, sigma=2.0, dtype=dtype, row_stride=stride)
    return x, host


@pytest.mark.parametrize("dtype,V,n", [("fp32", 32000, 512), ("bf16", 151936, 384), ("bf16", 32000, 600),
                                       ("bf16", 262144, 64), ("bf16", 1003, 300), ("fp32", 1003, 100),
                                       ("bf16", 7, 50), ("bf16", 4, 33)])
def test_logprob_entropy_vs_oracle(scorer, cuda, dtype, V, n):
    rng = np.random.default_rng(V + n)
    targets = rng.integers(0, V, n).astype(np.int32)
    old = (-0.05 - 2.95 * rng.random(n)).astype(np.float32)
    x, host = _logits_pair(n, V, dtype, cuda, scorer, targets=targets, old_lp=old)
    # generator parity: device logits bit-identical to the oracle's
    xb = x.view(torch.int16 if dtype == "bf16" else torch.int32).cpu().numpy()
    assert np.array_equal(xb.view(np.uint8), host.view(np.uint8))
    lp, ent = scorer.logprob_entropy(x, dev(targets, cuda))
    olp, oent = O.logprob_entropy(host, targets)
    assert_rows_close(lp.cpu().numpy(), olp, "logp")
    assert_rows_close(ent.cpu().numpy(), oent, "entropy")


def test_logprob_padded_stride_rows_and_temperature(scorer, cuda):
    V, stride, n_all = 5001, 5001 + 13, 200
    rng = np.random.default_rng(1)
    x, host = _logits_pair(n_all, V, "bf16", cuda, scorer, stride=stride)
    rows = rng.choice(n_all, 150, replace=False).astype(np.int32)
    targets = rng.integers(0, V, 150).astype(np.int32)
    for it in (1.0, 1.0 / 0.7, 2.5):
        lp, ent = scorer.logprob_entropy(x, dev(targets, cuda), rows=dev(rows, cuda), inv_temp=it, vocab=V)
        olp, oent = O.logprob_entropy(host, targets, rows=rows, inv_temp=it, vocab=V)
        assert_rows_close(lp.cpu().numpy(), olp, f"logp T={it}")
        assert_rows_close(ent.cpu().numpy(), oent, f"entropy T={it}")


def test_logprob_edge_rows(scorer, cuda):
    """all-equal logits (H = ln V), one dominant logit (H ~ 0), -inf (masked
    vocabulary) entries, large-magnitude logits."""
    V = 151936
    rows = []
    rows.append(np.zeros(V, np.float32))                                   # all equal
    r = np.zeros(V, np.float32); r[1234] = 60.0; rows.append(r)           # dominant
    r = np.full(V, -np.inf, np.float32); r[:1000] = np.linspace(-3, 3, 1000); rows.append(r)  # masked tail
    r = np.random.default_rng(0).normal(0, 2, V).astype(np.float32); r[::7] = -np.inf; rows.append(r)
    r = np.random.default_rng(1).normal(0, 30, V).astype(np.float32); rows.append(r)          # wide logits
    r = np.full(V, 1000.0, np.float32); r[5] = 1003.0; rows.append(r)                         # large offset
    host32 = np.stack(rows)
    xb = torch.from_numpy(host32).to(cuda).to(torch.bfloat16)
    hb = xb.view(torch.int16).cpu().numpy().view(np.uint16)
    targets = np.array([7, 1234, 10, 3, 99, 5], np.int32)
    lp, ent = scorer.logprob_entropy(xb, dev(targets, cuda))
    olp, oent = O.logprob_entropy(hb, targets)
    assert_rows_close(lp.cpu().numpy(), olp, "logp")
    assert_rows_close(ent.cpu().numpy(), oent, "entropy")
    assert abs(oent[0] - np.log(V)) < 1e-9
    # fp32 path on the same rows
    xf = torch.from_numpy(host32).to(cuda)
    lp, ent = scorer.logprob_entropy(xf, dev(targets, cuda))
    olp, oent = O.logprob_entropy(host32, targets)
    assert_rows_close(lp.cpu().numpy(), olp, "logp fp32")
    assert_rows_close(ent.cpu().numpy(), oent, "entropy fp32")


def test_logprob_unaligned_base(scorer, cuda):
    """Row starts that are not 16-B aligned (odd element offsets): head/tail lanes."""
    V = 32000
    x, host = _logits_pair(65, V + 3, "bf16", cuda, scorer)  # stride V+3, rows of V+3 logits
    sub = x[:, 3:]            # each row starts 6 bytes after a stride boundary
    targets = np.random.default_rng(2).integers(0, V, 65).astype(np.int32)
    lp, ent = scorer.logprob_entropy(sub, dev(targets, cuda), vocab=V)
    olp, oent = O.logprob_entropy(np.ascontiguousarray(host[:, 3:]), targets)
    assert_rows_close(lp.cpu().numpy(), olp, "logp")
    assert_rows_close(ent.cpu().numpy(), oent, "entropy")


# ---------------------------------------------------------------- K4 loss (+ fused K2+K4)
def _loss_inputs(n, rng, n_seq=37):
    logp = np.log(rng.random(n) * 0.9 + 0.05) - 0.0
    old = (logp + rng.uniform(-0.5, 0.5, n)).astype(np.float32)
    adv = rng.normal(0, 1, n_seq)
    seq = rng.integers(0, n_seq, n).astype(np.int32)
    turn = rng.integers(0, 90, n).astype(np.int16)
    ent = rng.random(n) * 10
    return logp.astype(np.float32), ent.astype(np.float32), old, adv.astype(np.float64), seq, turn


@pytest.mark.parametrize("n", [1, 31, 1000, 70001])
def test_clipped_loss_vs_oracle(scorer, cuda, n):
    rng = np.random.default_rng(n)
    logp, ent, old, adv, seq, turn = _loss_inputs(n, rng)
    p = scorer.clipped_loss(dev(logp, cuda), dev(ent, cuda), dev(old, cuda), dev(adv, cuda), dev(seq, cuda),
                            dev(turn, cuda))
    P, Q, nb = O.loss(logp.astype(np.float64), ent.astype(np.float64), old, adv.astype(np.float64), seq, turn)
    assert_partials_close(p.cpu().numpy(), P, Q, nb, "loss")


@pytest.mark.parametrize("kl_coef", [1e-4, 0.5])
def test_clipped_loss_with_kl_vs_oracle(scorer, cuda, kl_coef):
    """k3 KL penalty vs a reference policy (coefficient 1e-4)."""
    from paper_2603_18815_b200.hotpath import LossConfig
    rng = np.random.default_rng(17)
    logp, ent, old, adv, seq, turn = _loss_inputs(20000, rng)
    ref = (logp + rng.normal(0, 0.3, len(logp)) * (rng.random(len(logp)) < 0.9)).astype(np.float32)
    cfg = LossConfig(kl_coef=kl_coef)
    p = scorer.clipped_loss(dev(logp, cuda), dev(ent, cuda), dev(old, cuda), dev(adv, cuda), dev(seq, cuda),
                            dev(turn, cuda), cfg=cfg, ref_lp=dev(ref, cuda))
    P, Q, nb = O.loss(logp.astype(np.float64), ent.astype(np.float64), old, adv.astype(np.float64), seq, turn,
                      ref_lp=ref, kl_coef=kl_coef)
    assert P[N.P_KL_SUM] > 0
    assert_partials_close(p.cpu().numpy(), P, Q, nb, "loss+kl")


def test_clipped_loss_deterministic(scorer, cuda):
    rng = np.random.default_rng(9)
    args = [dev(a, cuda) for a in _loss_inputs(50000, rng)]
    a = scorer.clipped_loss(*args).cpu().numpy()
    b = scorer.clipped_loss(*args).cpu().numpy()
    assert np.array_equal(a, b)


def test_fused_score_rows_matches_k2_and_oracle(scorer, cuda):
    V, n = 151936, 700
    rng = np.random.default_rng(21)
    targets = rng.integers(0, V, n).astype(np.int32)
    old = (-1.0 - 0.6 * rng.random(n)).astype(np.float32)
    x, host = _logits_pair(n, V, "bf16", cuda, scorer, targets=targets, old_lp=old, seed=77)
    adv = rng.normal(0, 1, 13).astype(np.float64)
    seq = rng.integers(0, 13, n).astype(np.int32)
    turn = rng.integers(0, 70, n).astype(np.int16)
    td = dev(targets, cuda)
    partials, lp, ent = scorer.score_rows(x, td, dev(old, cuda), dev(adv, cuda), dev(seq, cuda), dev(turn, cuda))
    lp2, ent2 = scorer.logprob_entropy(x, td)
    assert torch.equal(lp, lp2) and torch.equal(ent, ent2)       # same arithmetic, bit-identical
    olp, oent = O.logprob_entropy(host, targets)
    assert_rows_close(lp.cpu().numpy(), olp, "logp")
    P, Q, nb = O.loss(olp, oent, old, adv.astype(np.float64), seq, turn)
    assert_partials_close(partials.cpu().numpy(), P, Q, nb, "fused")
    # realistic clipping from the planted targets
    assert 0 < P[N.P_CLIP_LO] + P[N.P_CLIP_HI] < n


# ---------------------------------------------------------------- whole step (C-ABI, host buffers)
def _cfg(config):
    c = synth.CONFIGS[config]
    return ScoreConfig(vocab=c["vocab"], dtype=c["dtype"], microbatch_rows=1000)


def _oracle_step(b: HostBatchArrays, cfg: ScoreConfig, seed, n_active, nthreads=8):
    hb = O.host_batch(b.turns, b.ids, b.lp, b.reward, b.usable, b.group_off, b.rollout_key)
    oc = O.score_cfg(cfg.vocab, cfg.dtype, microbatch_rows=cfg.microbatch_rows)
    return O.score_batch(hb, oc, seed, 2.0, nthreads=nthreads, want_rows=True, n_active_hint=n_active)


@pytest.mark.parametrize("config,kw", [("c1", {}), ("c1", {"seed": 99}), ("c2", {"max_groups": 1, "tokens": 2048}),
                                       ("c3", {"max_groups": 1, "tokens": 2048})])
def test_score_host_vs_oracle(scorer, cuda, config, kw):
    sh = synth.make_shard(config, **kw)
    b = sh.batch
    cfg = _cfg(config)
    V = cfg.vocab
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    pool = [torch.empty((cfg.microbatch_rows, V), dtype=tdt, device=cuda) for _ in range(2)]
    got, tm = scorer.score_host(b.pinned(), cfg, pool, fill=True, seed=1234)
    ref = _oracle_step(b, cfg, 1234, sh.n_active)
    assert ref["status"] == 0 and ref["n_active"] == sh.n_active
    assert_partials_close(got, ref["partials"], ref["abs"], ref["n_border"], config)
    again, _ = scorer.score_host(b, cfg, pool, fill=True, seed=1234)
    assert np.array_equal(got, again)  # deterministic run to run
    info = scorer.last_step_info()
    assert info["micro_batches"] == -(-sh.n_active // cfg.microbatch_rows)
    assert info["h2d_bytes"] >= 16 * b.ids.size and info["kernel_launches"] > info["micro_batches"]


def _relaid(b: HostBatchArrays, order) -> HostBatchArrays:
    """The same batch with the turns' tokens stored in the host SoA in another order."""
    t = b.turns.copy()
    ids, lp, off = [], [], 0
    for k in order:
        s0, L = int(b.turns["src_off"][k]), int(b.turns["len"][k])
        ids.append(b.ids[s0:s0 + L])
        lp.append(b.lp[s0:s0 + L])
        t["src_off"][k] = off
        off += L
    return HostBatchArrays(t, np.concatenate(ids), np.concatenate(lp), b.reward, b.usable, b.group_off,
                           rollout_key=b.rollout_key)


def test_score_host_chunked_h2d_matches_single_copy(scorer, cuda):
    """The token SoA is copied in chunks of whole sequences that overlap the
    scoring (capi.cu plan_chunks). Storing the same turns in reverse order keeps
    the chunks (disjoint source ranges); a random order falls back to one copy.
    The packed batch is the same, so all three steps are bit-identical."""
    sh = synth.make_shard("c1", seed=99)
    b = sh.batch
    cfg = _cfg("c1")
    pool = [torch.empty((cfg.microbatch_rows, cfg.vocab), dtype=torch.float32, device=cuda) for _ in range(2)]
    runs = {}
    n_t = len(b.turns)
    for name, order in (("stored", range(n_t)), ("reversed", range(n_t - 1, -1, -1)),
                        ("shuffled", np.random.default_rng(5).permutation(n_t))):
        bb = b if name == "stored" else _relaid(b, order)
        runs[name] = scorer.score_host(bb.pinned(), cfg, pool, fill=True, seed=7)[0]
        runs[name + "_chunks"] = scorer.last_step_info()["h2d_chunks"]
    assert runs["stored_chunks"] > 1 and runs["reversed_chunks"] > 1 and runs["shuffled_chunks"] == 1
    assert np.array_equal(runs["stored"], runs["reversed"]) and np.array_equal(runs["stored"], runs["shuffled"])


def test_score_host_resident_pool_back_to_back(scorer, cuda):
    """A pool with one buffer per micro-batch: a fill step, then re-scoring the
    resident logits (fill=False), whose micro-batch launches overlap through
    programmatic dependent launch (capi.cu, PRORL_PDL) — bit-identical partials."""
    sh = synth.make_shard("c1", seed=99)  # 6 144 active rows: 7 micro-batches
    b = sh.batch.pinned()
    cfg = _cfg("c1")
    n_mb = (sh.n_active + cfg.microbatch_rows - 1) // cfg.microbatch_rows
    assert n_mb >= 3
    pool = [torch.empty((cfg.microbatch_rows, cfg.vocab), dtype=torch.float32, device=cuda) for _ in range(n_mb)]
    filled, _ = scorer.score_host(b, cfg, pool, fill=True, seed=99)
    for _ in range(3):
        resident, _ = scorer.score_host(b, cfg, pool, fill=False, seed=99)
        assert np.array_equal(filled, resident)


def test_score_host_error_paths(scorer, cuda):
    sh = synth.make_shard("c1")
    b = sh.batch
    cfg = _cfg("c1")
    pool = [torch.empty((cfg.microbatch_rows, cfg.vocab), dtype=torch.float32, device=cuda)]
    bad = HostBatchArrays(b.turns, b.ids.copy(), b.lp, b.reward, b.usable, b.group_off)
    bad.ids[5] = cfg.vocab + 1
    with pytest.raises(RolloutError) as e:
        scorer.score_host(bad, cfg, pool, fill=True)
    assert e.value.code == "shape_mismatch"
    short = HostBatchArrays(b.turns, b.ids[:-1], b.lp[:-1], b.reward, b.usable, b.group_off)
    with pytest.raises(RolloutError):
        scorer.score_host(short, cfg, pool, fill=True)
    # the ctx stays usable after an error
    scorer.score_host(b, cfg, pool, fill=True)


def test_full_c2_properties_and_sampled_rows(scorer, cuda):
    """BASELINE configs[1] at full size: size-independent properties of the
    whole step + a row sample checked against the oracle at full-size keys."""
    sh = synth.make_shard("c2")
    b = sh.batch
    cfg = ScoreConfig(vocab=151936, dtype="bf16", microbatch_rows=8192)
    pool = [torch.empty((cfg.microbatch_rows, cfg.vocab), dtype=torch.bfloat16, device=cuda) for _ in range(2)]
    got, _ = scorer.score_host(b.pinned(), cfg, pool, fill=True, seed=31)
    n = sh.n_active
    assert got[N.P_N_ACTIVE] == n
    assert sum(got[N.N_GLOBAL + 5 * k] for k in range(64)) == n
    assert got[N.P_CLIP_LO] + got[N.P_CLIP_HI] <= n
    assert abs(got[N.P_ADV_SUM]) < 1e-3 * got[N.P_N_ROLLOUTS]
    assert 0 < got[N.P_ENTROPY_SUM] / n < np.log(151936)
    assert got[N.P_N_ROLLOUTS] == b.usable.sum()
    # sampled rows at their full-size keys, through pack + gen + K2
    pk = scorer.pack(b.turns, dev(b.ids, cuda), dev(b.lp, cuda), b.n_rollouts, 151936, n)
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(n, 96, replace=False))
    tg = pk["act_target"].cpu().numpy()[idx]
    ol = pk["act_old_lp"].cpu().numpy()[idx]
    x = torch.empty((1, 151936), dtype=torch.bfloat16, device=cuda)
    lps, ents, olps, oents = [], [], [], []
    for j, i in enumerate(idx):
        scorer.gen_logits(x, 1, int(i), dev(tg[j:j + 1], cuda), dev(ol[j:j + 1], cuda), seed=31)
        lp, ent = scorer.logprob_entropy(x, dev(tg[j:j + 1], cuda))
        h = O.gen_logits(1, 151936, int(i), tg[j:j + 1], ol[j:j + 1], seed=31)
        olp, oent = O.logprob_entropy(h, tg[j:j + 1])
        lps.append(lp.item()); ents.append(ent.item()); olps.append(olp[0]); oents.append(oent[0])
    assert_rows_close(lps, olps, "sampled logp")
    assert_rows_close(ents, oents, "sampled entropy")


# ---------------------------------------------------------------- randomized ragged batches
def _random_batch(rng, V):
    n_seq = int(rng.integers(1, 40))
    turns, ids, lps = [], [], []
    src = 0
    for s in range(n_seq):
        if rng.random() < 0.15:
            continue                      # FAILED / dropped slot: empty sequence
        for _ in range(int(rng.integers(1, 12))):
            role = int(rng.choice([0, 1, 2, 2, 3]))
            L = int(rng.choice([0, 1, 2, int(rng.integers(1, 300))]))
            turns.append((src, s, L, role))
            ids.append(rng.integers(0, V, L))
            lps.append(-rng.random(L) * 4 if role == 2 else np.zeros(L))
            src += L
    t = np.zeros(len(turns), N.TURN_DTYPE)
    if turns:
        arr = np.array(turns, np.int64)
        t["src_off"], t["traj"], t["len"], t["role"] = arr[:, 0], arr[:, 1], arr[:, 2], arr[:, 3]
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)
    return t, cat(ids, np.int64), cat(lps, np.float64), n_seq


@pytest.mark.parametrize("seed", range(12))
def test_pack_random_ragged_batches(scorer, cuda, seed):
    rng = np.random.default_rng(1000 + seed)
    V = int(rng.choice([50, 32000, 151936]))
    t, ids, lp, n_seq = _random_batch(rng, V)
    st, ora = O.pack(t, ids, lp, n_seq, V)
    assert st == 0
    compare_pack(scorer.pack(t, dev(ids, cuda), dev(lp, cuda), n_seq, V, ora["n_active"]), ora)


@pytest.mark.parametrize("seed", range(6))
def test_score_host_random_ragged_batches(scorer, cuda, seed):
    rng = np.random.default_rng(2000 + seed)
    V = int(rng.choice([97, 1003, 4096]))
    t, ids, lp, n_seq = _random_batch(rng, V)
    # groups of random sizes over the slots, random binary rewards, a few FAILED
    sizes, left = [], n_seq
    while left > 0:
        k = int(min(left, rng.integers(1, 6)))
        sizes.append(k)
        left -= k
    goff = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    reward = rng.choice([0.0, 1.0], n_seq)
    usable = (rng.random(n_seq) > 0.1).astype(np.uint8)
    b = HostBatchArrays(t, ids, lp, reward, usable, goff)
    cfg = ScoreConfig(vocab=V, dtype="bf16", microbatch_rows=257)
    pool = [torch.empty((257, V), dtype=torch.bfloat16, device=cuda)]
    got, _ = scorer.score_host(b, cfg, pool, fill=True, seed=seed)
    st, ora = O.pack(t, ids, lp, n_seq, V)
    hb = O.host_batch(t, ids, lp, reward, usable, goff)
    ref = O.score_batch(hb, O.score_cfg(V, "bf16", microbatch_rows=257), seed, 2.0, nthreads=4)
    assert ref["status"] == 0 and ref["n_active"] == ora["n_active"]
    # random layouts: sums that cancel to ~0 by chance get the random-walk allowance (tests/parity.py)
    assert_partials_close(got, ref["partials"], ref["abs"], ref["n_border"], f"ragged{seed}", rw_rows=ref["n_active"])


def test_score_host_rejects_inconsistent_descriptors(scorer, cuda):
    sh = synth.make_shard("c1", seed=99)
    assert len(sh.batch.group_off) >= 3
    b = sh.batch
    cfg = _cfg("c1")
    pool = [torch.empty((cfg.microbatch_rows, cfg.vocab), dtype=torch.float32, device=cuda)]
    t = b.turns.copy()
    t["traj"][0], t["traj"][-1] = t["traj"][-1], t["traj"][0]        # unsorted
    with pytest.raises(RolloutError) as e:
        scorer.score_host(HostBatchArrays(t, b.ids, b.lp, b.reward, b.usable, b.group_off), cfg, pool, fill=True)
    assert e.value.code == "shape_mismatch"
    t = b.turns.copy()
    t["src_off"][3] = len(b.ids)                                      # points past the ids
    with pytest.raises(RolloutError):
        scorer.score_host(HostBatchArrays(t, b.ids, b.lp, b.reward, b.usable, b.group_off), cfg, pool, fill=True)
    g = b.group_off.copy()
    g[1] = g[2] + 1                                                    # not monotone
    with pytest.raises(RolloutError):
        scorer.score_host(HostBatchArrays(b.turns, b.ids, b.lp, b.reward, b.usable, g), cfg, pool, fill=True)
    scorer.score_host(b, cfg, pool, fill=True)                         # ctx still usable
