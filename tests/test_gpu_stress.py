"""Full-size and stress configurations (BASELINE.json configs[2..4] shards and
the C5 stress sweep's extremes): bit-exact packing in full, size-independent
properties of the whole step, and per-row parity on sampled rows at their
full-size keys."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2603_18815_b200 import _native as N
from paper_2603_18815_b200 import synth
from paper_2603_18815_b200.hotpath import ScoreConfig

pytestmark = pytest.mark.gpu

REL, FLOOR = 1e-5, 1e-3


def dev(a, d):
    return torch.from_numpy(np.ascontiguousarray(a)).to(d)


def _pack_both(scorer, cuda, sh, V):
    b = sh.batch
    st, ora = O.pack(b.turns, b.ids, b.lp, b.n_rollouts, V)
    assert st == 0 and ora["n_active"] == sh.n_active
    gpu = scorer.pack(b.turns, dev(b.ids, cuda), dev(b.lp, cuda), b.n_rollouts, V, sh.n_active)
    for k in ("tokens", "loss_mask", "turn_id", "seq_id", "pos_id", "old_lp", "cu_seqlens", "act_row",
              "act_target", "act_old_lp", "act_seq", "act_turn"):
        g = gpu[k].cpu().numpy()
        assert np.array_equal(g.view(np.uint8), ora[k].view(np.uint8)), k
    return gpu, ora


def _sampled_rows(scorer, cuda, gpu, b, V, dtype, seed, n_sample=48):
    n = int(gpu["n_active"].item())
    idx = np.sort(np.random.default_rng(seed).choice(n, min(n_sample, n), replace=False))
    ti = torch.from_numpy(idx).to(cuda)
    rows, seq = gpu["act_row"][ti].contiguous(), gpu["act_seq"][ti].contiguous()
    tg, ol = gpu["act_target"][ti].contiguous(), gpu["act_old_lp"][ti].contiguous()
    keys = scorer.row_keys(rows, seq, gpu["cu_seqlens"], dev(b.rollout_key, cuda))
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    x = torch.empty((len(idx), V), dtype=tdt, device=cuda)
    scorer.gen_logits_keyed(x, keys, tg, ol, seed=seed, vocab=V)
    lp, ent = scorer.logprob_entropy(x, tg)
    kh, th, oh = keys.cpu().numpy(), tg.cpu().numpy(), ol.cpu().numpy()
    olp, oent = [], []
    for j in range(len(idx)):
        h = O.gen_logits(1, V, int(kh[j]), th[j:j + 1], oh[j:j + 1], seed=seed, dtype=dtype)
        a, e = O.logprob_entropy(h, th[j:j + 1])
        olp.append(a[0])
        oent.append(e[0])
    for got, want in ((lp.cpu().numpy(), np.array(olp)), (ent.cpu().numpy(), np.array(oent))):
        err = np.abs(got.astype(np.float64) - want)
        assert np.all(err <= REL * np.maximum(np.abs(want), FLOOR)), np.max(err / np.maximum(np.abs(want), FLOOR))


def test_full_c3_pack_and_sampled_rows(scorer, cuda):
    sh = synth.make_shard("c3")
    gpu, _ = _pack_both(scorer, cuda, sh, 151936)
    _sampled_rows(scorer, cuda, gpu, sh.batch, 151936, "bf16", seed=11)


def test_c4_rank0_of_8_pack_and_sampled_rows(scorer, cuda):
    sh = synth.make_shard("c4", rank=0, world=8)
    assert sh.batch.n_tokens > 4_000_000
    gpu, _ = _pack_both(scorer, cuda, sh, 151936)
    _sampled_rows(scorer, cuda, gpu, sh.batch, 151936, "bf16", seed=12)


STRESS = [
    # tokens, turns, group, vocab, tasks   (C5 extremes: 64K tokens x 64 turns, group 32, V 262144)
    dict(tokens=65536, turns=64, group=32, vocab=262144, tasks=3),
    dict(tokens=1024, turns=1, group=4, vocab=32000, tasks=16),
    dict(tokens=20000, turns=40, group=16, vocab=151936, tasks=4),
]


@pytest.mark.parametrize("spec", STRESS)
def test_stress_whole_step_properties(scorer, cuda, spec):
    cfg = dict(index=4, dtype="bf16", asst_share=0.3, lengths="fixed", desc="C5 stress", **spec)
    sh = synth.make_shard(cfg, seed=2607 + spec["turns"])
    b = sh.batch
    V = spec["vocab"]
    gpu, ora = _pack_both(scorer, cuda, sh, V)
    sc = ScoreConfig(vocab=V, dtype="bf16", microbatch_rows=4096)
    pool = [torch.empty((sc.microbatch_rows, V), dtype=torch.bfloat16, device=cuda)]
    got, _ = scorer.score_host(b.pinned(), sc, pool, fill=True, seed=5)
    n = sh.n_active
    assert got[N.P_N_ACTIVE] == n
    counts = got[N.N_GLOBAL::5][:64]
    assert counts.sum() == n
    # turn ordinals >= 63 fold into bucket 63
    turns = ora["act_turn"].astype(np.int64)
    assert counts[63] == np.sum(turns >= 63)
    assert np.array_equal(counts[:63], np.bincount(np.minimum(turns, 63), minlength=64)[:63])
    assert 0 < got[N.P_ENTROPY_SUM] / n < np.log(V)
    assert got[N.P_CLIP_LO] + got[N.P_CLIP_HI] <= n
    assert got[N.P_N_ROLLOUTS] == b.usable.sum()
    _sampled_rows(scorer, cuda, gpu, b, V, "bf16", seed=5, n_sample=24)
