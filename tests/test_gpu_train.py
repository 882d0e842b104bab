"""K7 (one-pass training step: logprob/entropy + DAPO loss partials + dL/dlogits
from a single read of each logits row, on thread-block clusters) vs the fp64
oracle, and vs the two-pass K2+K4 -> K5 path it replaces.

Tolerances as the kernels it fuses: logp/entropy |g - o| <= 1e-5 max(|o|, 1e-3);
partial sums <= 1e-5 of the sum's condition scale, counts exact except rows
within 1e-5 of a clip bound; dL/dlogp 1e-5 relative (plus, with the KL term,
its sensitivity to logp times logp's own tolerance: a clipped row's KL-only
scale kl/N (1 - e^(ref - logp)) is a small difference when ref ~ logp);
gradient elements one bf16 rounding (2^-8 relative) for bf16, 1e-5 relative for
fp32, plus the row scale's tolerance. Rows whose clip decision is within 1e-5
of flipping (oracle `border`) are skipped for the gradient."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2603_18815_b200 import _native as N
from paper_2603_18815_b200.hotpath import LossConfig
from tests.parity import assert_partials_close, assert_rows_close

pytestmark = pytest.mark.gpu


def dev(a, d):
    return torch.from_numpy(np.ascontiguousarray(a)).to(d)


def _case(scorer, cuda, V, n, dtype, stride=None, seed=0, n_seq=11):
    rng = np.random.default_rng(seed)
    targets = rng.integers(0, V, n).astype(np.int32)
    old = (-0.05 - 2.95 * rng.random(n)).astype(np.float32)
    stride = stride or V
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    x = torch.empty((n, stride), dtype=tdt, device=cuda)
    scorer.gen_logits(x, n, 1000, dev(targets, cuda), dev(old, cuda), seed=seed + 5, sigma=2.0, vocab=V)
    host = O.gen_logits(n, V, 1000, targets, old, seed=seed + 5, sigma=2.0, dtype=dtype, row_stride=stride)
    adv = rng.normal(0, 1, n_seq).astype(np.float64)
    seq = rng.integers(0, n_seq, n).astype(np.int32)
    turn = rng.integers(-1, 70, n).astype(np.int16)
    return x, host, targets, old, adv, seq, turn


def _check_all(scorer, cuda, x, host, t, old, adv, seq, turn, V, dtype, n_global, rows=None, cfg=None, ref=None,
               inplace=False, inv_temp=1.0):
    kl = cfg.kl_coef if cfg else 0.0
    rd = None if rows is None else dev(rows, cuda)
    part, lp, ent, g, dl = scorer.score_grad(x, dev(t, cuda), dev(old, cuda), dev(adv, cuda), dev(seq, cuda),
                                             dev(turn, cuda), n_global, rows=rd, cfg=cfg, vocab=V,
                                             grad=x if inplace else None, want_dlogp=True,
                                             ref_lp=None if ref is None else dev(ref, cuda), inv_temp=inv_temp)
    torch.cuda.synchronize()
    olp, oent = O.logprob_entropy(host, t, rows=rows, vocab=V, inv_temp=inv_temp)
    assert_rows_close(lp.cpu().numpy(), olp, "logp")
    assert_rows_close(ent.cpu().numpy(), oent, "entropy")
    P, Q, nb = O.loss(olp, oent, old, adv.astype(np.float64), seq, turn, ref_lp=ref, kl_coef=kl)
    assert_partials_close(part.cpu().numpy(), P, Q, nb, "k7")
    og, odl, bd = O.logits_grad(host, t, old, adv.astype(np.float64), seq, n_global, rows=rows, vocab=V,
                                ref_lp=ref, kl_coef=kl, inv_temp=inv_temp)
    ok = bd == 0
    assert ok.sum() > 0.9 * len(ok)
    d = dl.cpu().numpy().astype(np.float64)
    # dL/dlogp to 1e-5, plus the KL term's sensitivity to logp times logp's own
    # tolerance (a KL-only row, ref ~ logp, is a small difference: its relative
    # error is the logp error amplified)
    tol_dl = 1e-5 * np.abs(odl) + 1e-12
    if ref is not None:
        tol_dl += kl / n_global * np.exp(ref.astype(np.float64) - olp) * 1e-5 * np.maximum(np.abs(olp), 1e-3)
    assert np.all(np.abs(d[ok] - odl[ok]) <= tol_dl[ok])
    r = np.arange(len(t)) if rows is None else rows
    got = g.float().cpu().numpy()[r, :V].astype(np.float64)
    # one bf16 rounding (fp32: 1e-5) plus the row scale's own tolerance (dL/dlogp)
    row_rel = (tol_dl / np.maximum(np.abs(odl), 1e-300))[:, None]
    tol = ((2.0 ** -8 if dtype == "bf16" else 1e-5) + row_rel) * np.abs(og) + 1e-30
    bad = (np.abs(got - og) > tol) & ok[:, None]
    assert not bad.any(), (np.argwhere(bad)[:5], got[bad][:5], og[bad][:5])
    return part, lp, ent, g, dl


@pytest.mark.parametrize("dtype,V,stride,n", [
    ("bf16", 32000, None, 300),
    ("bf16", 151936, None, 64),
    ("bf16", 262144, None, 20),
    ("fp32", 151936, None, 16),
    ("fp32", 32000, None, 90),
    ("bf16", 1003, 1008, 200),    # 3-element tail after the 16-B interior
    ("fp32", 4099, 4100, 60),     # 3-element tail, fp32
    ("bf16", 7, 8, 40),           # no interior at all: the whole row is tail
    ("bf16", 1003, None, 120),    # odd row stride: per-row head/tail phases differ
    ("bf16", 600000, None, 3),    # rows far larger than the shared-memory ring
    ("fp32", 5001, 5014, 50),     # padded odd stride, fp32
])
def test_score_grad_vs_oracle(scorer, cuda, dtype, V, stride, n):
    x, host, t, old, adv, seq, turn = _case(scorer, cuda, V, n, dtype, stride=stride, seed=V % 89 + n)
    _check_all(scorer, cuda, x, host, t, old, adv, seq, turn, V, dtype, n_global=5000.0)


def test_score_grad_matches_two_pass(scorer, cuda):
    """K7 == K2+K4 then K5 on the same rows, within the kernels' tolerances."""
    V, n = 151936, 512
    x, host, t, old, adv, seq, turn = _case(scorer, cuda, V, n, "bf16", seed=7)
    td, od, ad, sd, trd = (dev(a, cuda) for a in (t, old, adv, seq, turn))
    p1, lp1, ent1, g1, dl1 = scorer.score_grad(x, td, od, ad, sd, trd, 904452.0, want_dlogp=True)
    p2, lp2, ent2 = scorer.score_rows(x, td, od, ad, sd, trd)
    g2, dl2 = scorer.logits_grad(x, td, lp2, od, ad, sd, 904452.0, want_dlogp=True)
    torch.cuda.synchronize()
    a, b = lp1.double().cpu().numpy(), lp2.double().cpu().numpy()
    assert np.all(np.abs(a - b) <= 2e-5 * np.maximum(np.abs(b), 1e-3))
    a, b = ent1.double().cpu().numpy(), ent2.double().cpu().numpy()
    assert np.all(np.abs(a - b) <= 2e-5 * np.maximum(np.abs(b), 1e-3))
    P1, P2 = p1.cpu().numpy(), p2.cpu().numpy()
    assert P1[N.P_N_ACTIVE] == P2[N.P_N_ACTIVE] == n
    assert abs(P1[N.P_LOSS_SUM] - P2[N.P_LOSS_SUM]) <= 1e-5 * np.abs(P2[N.P_LOSS_SUM]) + 1e-6
    # gradients: same rows zero (clip decisions agree away from the border), values within 2 bf16 ulps
    G1, G2 = g1.float().cpu().numpy(), g2.float().cpu().numpy()
    assert np.all(np.abs(G1 - G2) <= 2.0 ** -7 * np.maximum(np.abs(G1), np.abs(G2)) + 1e-30)


def test_score_grad_rows_inplace_deterministic(scorer, cuda):
    V, n = 151936, 96
    x, host, t, old, adv, seq, turn = _case(scorer, cuda, V, n, "bf16", seed=11)
    rows = np.random.default_rng(2).permutation(n).astype(np.int32)
    x0 = x.clone()
    part, lp, ent, g, dl = _check_all(scorer, cuda, x, host, t, old, adv, seq, turn, V, "bf16", 333.0, rows=rows)
    # bit-identical on a second run (fixed reduction order, no atomics)
    part2, lp2, ent2, g2, dl2 = scorer.score_grad(x, dev(t, cuda), dev(old, cuda), dev(adv, cuda), dev(seq, cuda),
                                                  dev(turn, cuda), 333.0, rows=dev(rows, cuda), want_dlogp=True)
    assert torch.equal(part, part2) and torch.equal(lp, lp2) and torch.equal(g, g2)
    # in place: the gradient overwrites the logits and equals the out-of-place result
    xi = x0.clone()
    part3, lp3, *_ = scorer.score_grad(xi, dev(t, cuda), dev(old, cuda), dev(adv, cuda), dev(seq, cuda),
                                       dev(turn, cuda), 333.0, rows=dev(rows, cuda), grad=xi)
    torch.cuda.synchronize()
    assert torch.equal(xi, g) and torch.equal(part3, part) and torch.equal(lp3, lp)


def test_score_grad_kl_and_zero_advantage(scorer, cuda):
    V, n = 65536, 128
    x, host, t, old, adv, seq, turn = _case(scorer, cuda, V, n, "bf16", seed=21, n_seq=8)
    adv[3] = 0.0  # rows of sequence 3 have a zero gradient without the KL term
    lp0, _ = scorer.logprob_entropy(x, dev(t, cuda))
    ref = (lp0.cpu().numpy() + np.random.default_rng(3).normal(0, 0.4, n)).astype(np.float32)
    _check_all(scorer, cuda, x, host, t, old, adv, seq, turn, V, "bf16", 300.0, cfg=LossConfig(kl_coef=0.25),
               ref=ref)
    part, lp, ent, g, dl = scorer.score_grad(x, dev(t, cuda), dev(old, cuda), dev(adv, cuda), dev(seq, cuda),
                                             dev(turn, cuda), 300.0, want_dlogp=True)
    z = seq == 3
    assert z.any() and torch.count_nonzero(g[torch.from_numpy(z).to(cuda)]).item() == 0


def test_score_grad_edge_rows(scorer, cuda):
    """All-equal logits (H = ln V), one dominant logit (p -> 1), -inf entries,
    ties at the maximum in two distant warps' units, a max at a unit boundary."""
    V, n = 151936, 6
    rng = np.random.default_rng(5)
    xh = rng.normal(0, 2, (n, V)).astype(np.float32)
    xh[0] = 0.5
    xh[1, 1234] = 60.0
    xh[2, ::3] = -np.inf
    xh[3, 17] = xh[3, V - 17] = 30.0   # equal maxima in both halves of the row
    xh[4, V // 2] = 25.0              # max at the slice boundary
    t = np.array([5, 1234, 4, V - 17, V // 2, 9], np.int32)
    x = torch.from_numpy(xh).to(cuda).to(torch.bfloat16)
    host = x.view(torch.int16).cpu().numpy().view(np.uint16)
    old = np.full(n, -0.7, np.float32)
    adv = np.array([1.0, -1.0], np.float64)
    seq = np.array([0, 1, 0, 1, 0, 1], np.int32)
    turn = np.zeros(n, np.int16)
    part, lp, ent, g, dl = _check_all(scorer, cuda, x, host, t, old, adv, seq, turn, V, "bf16", 10.0)
    e = ent.cpu().numpy()
    assert abs(e[0] - np.log(V)) < 1e-4 and e[1] < 1e-6
    assert torch.isfinite(g.float()).all()


def test_score_grad_full_microbatch_properties(scorer, cuda):
    """A full C2 micro-batch (16 576 rows x 151 936): partials equal the fused
    K2+K4 pass, every gradient row sums to ~0 and is finite."""
    V, n = 151936, 16576
    rng = np.random.default_rng(31)
    t = rng.integers(0, V, n).astype(np.int32)
    old = (-0.05 - 2.95 * rng.random(n)).astype(np.float32)
    x = torch.empty((n, V), dtype=torch.bfloat16, device=cuda)
    scorer.gen_logits(x, n, 0, dev(t, cuda), dev(old, cuda), seed=9, sigma=2.0)
    adv = rng.normal(0, 1, 280).astype(np.float64)
    seq = np.sort(rng.integers(0, 280, n)).astype(np.int32)
    turn = rng.integers(0, 40, n).astype(np.int16)
    td, od, ad, sd, trd = (dev(a, cuda) for a in (t, old, adv, seq, turn))
    p2, lp2, _ = scorer.score_rows(x, td, od, ad, sd, trd)
    p1, lp1, _, g, _ = scorer.score_grad(x, td, od, ad, sd, trd, float(n), grad=x)   # in place
    torch.cuda.synchronize()
    P1, P2 = p1.cpu().numpy(), p2.cpu().numpy()
    assert P1[N.P_N_ACTIVE] == n
    for i in (N.P_LOSS_SUM, N.P_ENTROPY_SUM, N.P_LOGP_SUM, N.P_RATIO_SUM):
        assert abs(P1[i] - P2[i]) <= 1e-5 * abs(P2[i]) + 1e-6, (i, P1[i], P2[i])
    assert abs(P1[N.P_CLIP_LO] - P2[N.P_CLIP_LO]) <= 3
    s = x.float().sum(dim=1)
    mx = x.float().abs().amax(dim=1)
    assert torch.isfinite(s).all() and bool((s.abs() <= V * 2.0 ** -8 * mx + 1e-12).all())


def test_score_host_train_mode(scorer, cuda):
    """prorl_score_host in training mode (K7 per micro-batch): partials equal the
    forward step's, and each micro-batch's gradient equals prorl_score_grad on
    the same logits with the device-packed rows and GRPO advantages."""
    from paper_2603_18815_b200 import synth
    from paper_2603_18815_b200.hotpath import ScoreConfig
    from tests.test_gpu_parity import device_pack
    sh = synth.make_shard("c1", seed=5)
    b = sh.batch
    V, mb = 32000, 2048
    cfg = ScoreConfig(vocab=V, dtype="fp32", microbatch_rows=mb)
    n_mb = -(-sh.n_active // mb)
    pool = [torch.empty((mb, V), dtype=torch.float32, device=cuda) for _ in range(n_mb)]  # no buffer reuse
    gpool = [torch.empty_like(p) for p in pool]
    seen = []
    fwd, _ = scorer.score_host(b.pinned(), cfg, pool, fill=True, seed=7)
    trn, tm = scorer.score_host(b.pinned(), cfg, pool, fill=True, seed=7, train=True, grad_pool=gpool,
                                grad_fn=lambda r0, n, g, s: seen.append((r0, n, g, s)))
    torch.cuda.synchronize()
    assert [(r0, n) for r0, n, _, _ in seen] == [(j * mb, min(mb, sh.n_active - j * mb)) for j in range(n_mb)]
    assert all(g == gpool[j].data_ptr() and s == V for j, (_, _, g, s) in enumerate(seen))
    assert trn[N.P_N_ACTIVE] == fwd[N.P_N_ACTIVE] == sh.n_active
    for i in (N.P_LOSS_SUM, N.P_ENTROPY_SUM, N.P_LOGP_SUM, N.P_RATIO_SUM, N.P_ADV_SUM):
        assert abs(trn[i] - fwd[i]) <= 2e-5 * abs(fwd[i]) + 1e-6, (i, trn[i], fwd[i])
    # reference: prorl_score_grad on the same (regenerated) logits
    pk = device_pack(scorer, b, V, sh.n_active, cuda)
    adv, _ = scorer.grpo_adv(torch.from_numpy(b.reward).to(cuda), torch.from_numpy(b.usable).to(cuda),
                             torch.from_numpy(b.group_off).to(cuda))
    for j in range(n_mb):
        r0, n = j * mb, min(mb, sh.n_active - j * mb)
        sl = slice(r0, r0 + n)
        _, _, _, g_ref, _ = scorer.score_grad(pool[j][:n], pk["act_target"][sl], pk["act_old_lp"][sl], adv,
                                               pk["act_seq"][sl], pk["act_turn"][sl], float(sh.n_active))
        torch.cuda.synchronize()
        assert torch.equal(gpool[j][:n], g_ref[:n])
    # in place (no grad pool): the logits buffers end up holding the gradient
    trn2, _ = scorer.score_host(b.pinned(), cfg, pool, fill=True, seed=7, train=True)
    torch.cuda.synchronize()
    assert torch.equal(torch.from_numpy(trn2), torch.from_numpy(trn))
    for j in range(n_mb):
        n = min(mb, sh.n_active - j * mb)
        assert torch.equal(pool[j][:n], gpool[j][:n])


def test_score_grad_running_max_slack(scorer, cuda):
    """Rows whose maximum appears in a later warp unit just below / above the
    running-max slack (1 in log2 units = 0.69 nats) of an earlier near-max:
    the reference point then is not the exact maximum (or is raised), and
    logp / entropy / gradient must still meet the oracle tolerances."""
    V = 151936
    rng = np.random.default_rng(17)
    rows, targets = [], []
    for early, late, tgt_late in [(10.0, 10.6, True), (10.0, 10.6, False), (10.0, 10.68, True),
                                  (10.0, 10.8, True), (10.0, 30.0, True), (10.0, 9.5, False)]:
        r = rng.normal(0, 2, V).astype(np.float32)
        r[100] = early
        r[140000] = late
        rows.append(r)
        targets.append(140000 if tgt_late else 100)
    xh = np.stack(rows)
    x = torch.from_numpy(xh).to(cuda).to(torch.bfloat16)
    host = x.view(torch.int16).cpu().numpy().view(np.uint16)
    n = len(rows)
    t = np.array(targets, np.int32)
    old = np.full(n, -0.5, np.float32)
    adv = np.array([1.0, -1.0], np.float64)
    seq = (np.arange(n) % 2).astype(np.int32)
    turn = np.zeros(n, np.int16)
    _check_all(scorer, cuda, x, host, t, old, adv, seq, turn, V, "bf16", 10.0)
    # K2 uses the same running-max slack: forward-only logp / entropy on the same rows
    lp, ent = scorer.logprob_entropy(x, dev(t, cuda))
    olp, oent = O.logprob_entropy(host, t)
    assert_rows_close(lp.cpu().numpy(), olp, "K2 logp")
    assert_rows_close(ent.cpu().numpy(), oent, "K2 entropy")


@pytest.mark.parametrize("case", range(10))
def test_score_grad_randomized_layouts(scorer, cuda, case):
    """Seeded random layouts (vocab, row padding, dtype, rows indirection, in
    place, KL) through K7 vs the fp64 oracle."""
    rng = np.random.default_rng(1000 + case)
    dtype = "bf16" if rng.random() < 0.7 else "fp32"
    V = int(rng.choice([int(rng.integers(2, 300)), int(rng.integers(300, 20000)), int(rng.integers(20000, 200000))]))
    pad = int(rng.integers(0, 9)) if rng.random() < 0.5 else 0
    n = int(rng.integers(1, 40 if V > 50000 else 120))
    x, host, t, old, adv, seq, turn = _case(scorer, cuda, V, n, dtype, stride=V + pad, seed=case, n_seq=5)
    rows = rng.permutation(n).astype(np.int32) if rng.random() < 0.5 else None
    cfg, ref = None, None
    if rng.random() < 0.4:
        cfg = LossConfig(kl_coef=0.1)
        lp0, _ = scorer.logprob_entropy(x, dev(t, cuda), rows=None if rows is None else dev(rows, cuda), vocab=V)
        ref = (lp0.cpu().numpy() + rng.normal(0, 0.3, n)).astype(np.float32)
    inv_temp = float(rng.choice([1.0, 1.0, 0.7, 1.6]))
    if ref is not None and inv_temp != 1.0:  # reference logprobs near this temperature's logprobs
        lp0, _ = scorer.logprob_entropy(x, dev(t, cuda), rows=None if rows is None else dev(rows, cuda), vocab=V,
                                        inv_temp=inv_temp)
        ref = (lp0.cpu().numpy() + rng.normal(0, 0.3, n)).astype(np.float32)
    _check_all(scorer, cuda, x, host, t, old, adv, seq, turn, V, dtype, float(n * 3), rows=rows, cfg=cfg, ref=ref,
               inplace=rows is None and rng.random() < 0.5, inv_temp=inv_temp)


def test_score_grad_errors(scorer, cuda):
    """Layout / argument errors surface as rollout error codes, nothing launches."""
    from paper_2603_18815_b200.hotpath import RolloutError
    x = torch.zeros((4, 64), dtype=torch.bfloat16, device=cuda)
    t = torch.zeros(4, dtype=torch.int32, device=cuda)
    f = torch.zeros(4, dtype=torch.float32, device=cuda)
    tr = torch.zeros(4, dtype=torch.int16, device=cuda)
    a = torch.zeros(4, dtype=torch.float64, device=cuda)
    with pytest.raises(RolloutError) as e:   # gradient with another row stride
        scorer.score_grad(x, t, f, a, t, tr, 10.0, grad=torch.zeros((4, 72), dtype=torch.bfloat16, device=cuda))
    assert e.value.code == "shape_mismatch"
    with pytest.raises(RolloutError) as e:   # gradient with another 16-B phase
        buf = torch.zeros(4 * 64 + 1, dtype=torch.bfloat16, device=cuda)
        scorer.score_grad(x, t, f, a, t, tr, 10.0, grad=buf[1:].view(4, 64))
    assert e.value.code == "shape_mismatch"
    with pytest.raises(RolloutError) as e:   # no active rows in the global count
        scorer.score_grad(x, t, f, a, t, tr, 0.0)
    assert e.value.code == "malformed_request"
    with pytest.raises(RolloutError) as e:   # missing row arrays
        scorer.score_grad(x, t, None, a, t, tr, 10.0)
    assert e.value.code == "malformed_request"
    # zero rows: a no-op that leaves the partials untouched
    part, *_ = scorer.score_grad(x[:0], t[:0], f[:0], a, t[:0], tr[:0], 10.0)
    assert float(part.abs().sum()) == 0.0


def test_score_host_kl_reference_logprobs(scorer, cuda):
    """The k3 KL term through the whole step: reference logprobs
    come from provide_ref per micro-batch; forward and training mode equal the
    per-kernel path with ref_lp on the same logits; kl_coef without a source is
    rejected."""
    from paper_2603_18815_b200 import synth
    from paper_2603_18815_b200.hotpath import RolloutError, ScoreConfig
    from tests.test_gpu_parity import device_pack
    sh = synth.make_shard("c1", seed=6)
    b = sh.batch
    V, mb = 32000, 2048
    lcfg = LossConfig(kl_coef=0.25)
    cfg = ScoreConfig(vocab=V, dtype="fp32", microbatch_rows=mb, loss=lcfg)
    n_mb = -(-sh.n_active // mb)
    pool = [torch.empty((mb, V), dtype=torch.float32, device=cuda) for _ in range(n_mb)]
    gpool = [torch.empty_like(p) for p in pool]
    ref_all = torch.from_numpy((-0.05 - 2.5 * np.random.default_rng(4).random(sh.n_active)).astype(np.float32)).to(cuda)
    ref_fn = lambda row0, n, rows, seq, cu, tg: ref_all[row0:row0 + n]  # noqa: E731
    with pytest.raises(RolloutError) as e:
        scorer.score_host(b.pinned(), cfg, pool, fill=True, seed=7)
    assert e.value.code == "malformed_request"
    fwd, _ = scorer.score_host(b.pinned(), cfg, pool, fill=True, seed=7, ref_fn=ref_fn)
    trn, _ = scorer.score_host(b.pinned(), cfg, pool, fill=True, seed=7, ref_fn=ref_fn, train=True, grad_pool=gpool)
    torch.cuda.synchronize()
    pk = device_pack(scorer, b, V, sh.n_active, cuda)
    adv, _ = scorer.grpo_adv(torch.from_numpy(b.reward).to(cuda), torch.from_numpy(b.usable).to(cuda),
                             torch.from_numpy(b.group_off).to(cuda))
    acc = torch.zeros(N.N_PARTIALS, dtype=torch.float64, device=cuda)
    for j in range(n_mb):
        r0, n = j * mb, min(mb, sh.n_active - j * mb)
        sl = slice(r0, r0 + n)
        p, _, _ = scorer.score_rows(pool[j][:n], pk["act_target"][sl], pk["act_old_lp"][sl], adv, pk["act_seq"][sl],
                                    pk["act_turn"][sl], cfg=lcfg, ref_lp=ref_all[sl])
        acc += p
    ref = acc.cpu().numpy()
    assert ref[N.P_KL_SUM] > 0
    for got in (fwd, trn):
        for i in (N.P_LOSS_SUM, N.P_KL_SUM, N.P_ENTROPY_SUM, N.P_LOGP_SUM):
            assert abs(got[i] - ref[i]) <= 2e-5 * abs(ref[i]) + 1e-6, (i, got[i], ref[i])
