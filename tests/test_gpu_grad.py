"""K5 (backward of the DAPO surrogate through the log-softmax) vs the fp64 oracle.

Tolerances: dL/dlogp per row 1e-5 relative; gradient elements bf16: one bf16
rounding (|g - o| <= 2^-8 |o|) plus fp32 noise; fp32: 1e-5 relative. Rows
whose clip decision is within 1e-5 of flipping (oracle `border`) are skipped —
their gradient is legitimately all-or-nothing."""
import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def dev(a, d):
    return torch.from_numpy(np.ascontiguousarray(a)).to(d)


def _case(scorer, cuda, V, n, dtype, stride=None, seed=0, n_seq=11):
    rng = np.random.default_rng(seed)
    targets = rng.integers(0, V, n).astype(np.int32)
    old = (-1.0 - 0.6 * rng.random(n)).astype(np.float32)
    stride = stride or V
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    x = torch.empty((n, stride), dtype=tdt, device=cuda)
    scorer.gen_logits(x, n, 1000, dev(targets, cuda), dev(old, cuda), seed=seed + 5, sigma=2.0, vocab=V)
    host = O.gen_logits(n, V, 1000, targets, old, seed=seed + 5, sigma=2.0, dtype=dtype, row_stride=stride)
    adv = rng.normal(0, 1, n_seq).astype(np.float64)
    seq = rng.integers(0, n_seq, n).astype(np.int32)
    return x, host, targets, old, adv, seq


def _check(scorer, cuda, x, host, targets, old, adv, seq, V, dtype, n_global, rows=None, inplace=False):
    td = dev(targets, cuda)
    xr = x if rows is None else x
    lp, _ = scorer.logprob_entropy(xr, td, rows=None if rows is None else dev(rows, cuda), vocab=V)
    grad_in = x if inplace else None
    g, dl = scorer.logits_grad(x, td, lp, dev(old, cuda), dev(adv, cuda), dev(seq, cuda), n_global,
                               rows=None if rows is None else dev(rows, cuda), grad=grad_in, vocab=V,
                               want_dlogp=True)
    og, odl, bd = O.logits_grad(host, targets, old, adv.astype(np.float64), seq, n_global, rows=rows, vocab=V)
    ok = bd == 0
    assert ok.sum() > 0.9 * len(ok)
    d = dl.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(d[ok] - odl[ok]) <= 1e-5 * np.abs(odl[ok]) + 1e-12)
    gh = g.float().cpu().numpy()
    r = np.arange(len(targets)) if rows is None else rows
    got = gh[r, :V].astype(np.float64)
    want = og
    if dtype == "bf16":
        tol = 2.0 ** -8 * np.abs(want) + 1e-30
    else:
        tol = 1e-5 * np.abs(want) + 1e-30
    bad = (np.abs(got - want) > tol) & ok[:, None]
    assert not bad.any(), (np.argwhere(bad)[:5], got[bad][:5], want[bad][:5])
    # each gradient row sums to ~0 (sum_v (1[v=y] - p_v) = 0)
    scale = np.abs(want).max(axis=1) + 1e-30
    assert np.all(np.abs(got.sum(axis=1))[ok] <= (V * 2.0 ** -8 + 1e-3) * scale[ok])


@pytest.mark.parametrize("dtype,V,n", [("bf16", 32000, 96), ("fp32", 32000, 64), ("bf16", 1003, 70), ("bf16", 7, 40)])
def test_logits_grad_vs_oracle(scorer, cuda, dtype, V, n):
    x, host, t, old, adv, seq = _case(scorer, cuda, V, n, dtype, seed=V % 97)
    _check(scorer, cuda, x, host, t, old, adv, seq, V, dtype, n_global=5000.0)


def test_logits_grad_full_vocab_bf16(scorer, cuda):
    V = 151936
    x, host, t, old, adv, seq = _case(scorer, cuda, V, 24, "bf16", seed=3)
    _check(scorer, cuda, x, host, t, old, adv, seq, V, "bf16", n_global=904452.0)


def test_logits_grad_padded_stride_rows_inplace(scorer, cuda):
    V, stride = 5001, 5001 + 13
    x, host, t, old, adv, seq = _case(scorer, cuda, V, 90, "fp32", stride=stride, seed=9)
    rows = np.random.default_rng(1).permutation(90).astype(np.int32)
    # targets/old/seq are per call row i, logits row = rows[i]
    ref_x = x.clone()
    _check(scorer, cuda, x, host, t, old, adv, seq, V, "fp32", n_global=777.0, rows=rows)
    # in place == out of place
    td = dev(t, cuda)
    lp, _ = scorer.logprob_entropy(ref_x, td, rows=dev(rows, cuda), vocab=V)
    g_out, _ = scorer.logits_grad(ref_x, td, lp, dev(old, cuda), dev(adv, cuda), dev(seq, cuda), 777.0,
                                  rows=dev(rows, cuda), vocab=V)
    scorer.logits_grad(ref_x, td, lp, dev(old, cuda), dev(adv, cuda), dev(seq, cuda), 777.0, rows=dev(rows, cuda),
                       grad=ref_x, vocab=V)
    assert torch.equal(g_out[:, :V], ref_x[:, :V])


def test_logits_grad_with_kl(scorer, cuda):
    from paper_2603_18815_b200.hotpath import LossConfig
    V, n = 4099, 64
    x, host, t, old, adv, seq = _case(scorer, cuda, V, n, "bf16", seed=21)
    td = dev(t, cuda)
    lp, _ = scorer.logprob_entropy(x, td)
    ref = (lp.cpu().numpy() + np.random.default_rng(3).normal(0, 0.4, n)).astype(np.float32)
    cfg = LossConfig(kl_coef=0.25)
    g, dl = scorer.logits_grad(x, td, lp, dev(old, cuda), dev(adv, cuda), dev(seq, cuda), 300.0, cfg=cfg,
                               ref_lp=dev(ref, cuda), want_dlogp=True)
    og, odl, bd = O.logits_grad(host, t, old, adv.astype(np.float64), seq, 300.0, ref_lp=ref, kl_coef=0.25)
    ok = bd == 0
    d = dl.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(d[ok] - odl[ok]) <= 1e-5 * np.abs(odl[ok]) + 1e-10)
    got = g.float().cpu().numpy().astype(np.float64)
    assert not ((np.abs(got - og) > 2.0 ** -8 * np.abs(og) + 1e-30) & ok[:, None]).any()


def test_logits_grad_layout_errors(scorer, cuda):
    from paper_2603_18815_b200.hotpath import RolloutError
    x = torch.zeros((4, 64), dtype=torch.bfloat16, device=cuda)
    t = torch.zeros(4, dtype=torch.int32, device=cuda)
    f = torch.zeros(4, dtype=torch.float32, device=cuda)
    a = torch.zeros(4, dtype=torch.float64, device=cuda)
    bad = torch.zeros((4, 72), dtype=torch.bfloat16, device=cuda)
    with pytest.raises(RolloutError):
        scorer.logits_grad(x, t, f, f, a, t, 10.0, grad=bad)
    with pytest.raises(TypeError):  # advantages cross the C-ABI as fp64
        scorer.logits_grad(x, t, f, f, f, t, 10.0)


def test_logits_grad_dominant_and_masked_rows(scorer, cuda):
    """p_y -> 1 (the target gradient -g (1 - p_y) must not pick up the fp32
    rounding of the lse) and -inf (masked) logits."""
    V, n = 32000, 4
    rng = np.random.default_rng(8)
    xh = rng.normal(0, 2, (n, V)).astype(np.float32)
    xh[0, 77] = 60.0
    xh[1, ::5] = -np.inf
    xh[2] = 0.25
    t = np.array([77, 3, 9, 11], np.int32)
    x = torch.from_numpy(xh).to(cuda).to(torch.bfloat16)
    host = x.view(torch.int16).cpu().numpy().view(np.uint16)
    old = np.full(n, -0.7, np.float32)
    adv = np.array([1.0, -1.0], np.float64)
    seq = np.array([0, 1, 0, 1], np.int32)
    _check(scorer, cuda, x, host, t, old, adv, seq, V, "bf16", n_global=10.0)
