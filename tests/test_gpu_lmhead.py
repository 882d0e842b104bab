"""K6 fused LM head (tcgen05 GEMM + online-softmax epilogue) vs a plain
PyTorch float64 reference of the same op (the logits path it replaces):
logp = log_softmax(H W^T * inv_T)[y], entropy = -sum p log p.
Tolerance: 1e-5 * max(|ref|, 1e-3)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(H, W, t, inv_temp):
    x = (H.double() @ W.double().T) * inv_temp
    lse = torch.logsumexp(x, dim=1)
    logp = x.gather(1, t.long()[:, None])[:, 0] - lse
    p = torch.softmax(x, dim=1)
    ent = -(p * torch.log_softmax(x, dim=1)).sum(dim=1)
    return logp, ent


def _check(got, want, what):
    got = got.double().cpu().numpy()
    want = want.cpu().numpy()
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-3)
    assert np.all(rel <= 1e-5), (what, rel.max(), int(rel.argmax()), got[rel.argmax()], want[rel.argmax()])


@pytest.mark.parametrize("n,d,V,inv_temp", [(200, 256, 4099, 1.0), (129, 512, 1000, 1.0 / 0.7),
                                            (300, 2560, 151936, 1.0), (64, 4096, 32000, 1.0)])
def test_lmhead_vs_torch_fp64(scorer, cuda, n, d, V, inv_temp):
    g = torch.Generator(device=cuda).manual_seed(n + d)
    H = torch.randn(n, d, device=cuda, generator=g).to(torch.bfloat16)
    W = (torch.randn(V, d, device=cuda, generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    t = torch.randint(0, V, (n,), device=cuda, dtype=torch.int32, generator=g)
    lp, ent = scorer.lmhead_logprob(H, W, t, inv_temp=inv_temp)
    rlp, rent = _ref(H, W, t, inv_temp)
    _check(lp, rlp, "logp")
    _check(ent, rent, "entropy")


@pytest.mark.parametrize("n,d,V,scale,pad", [
    (1, 64, 1, 1.0, 0),        # one row, one vocabulary entry (logp = 0, H = 0)
    (5, 64, 7, 1.0, 0),        # V far below one 256-wide vocabulary chunk
    (130, 128, 257, 1.0, 0),   # one row and one vocab entry past a tile edge
    (257, 192, 5000, 40.0, 0),  # peaked softmax: logits spread over hundreds of nats
    (96, 320, 3001, 1.0, 64),  # hidden rows strided (padded leading dimension)
])
def test_lmhead_edges(scorer, cuda, n, d, V, scale, pad):
    g = torch.Generator(device=cuda).manual_seed(7 * n + V)
    Hfull = torch.randn(n, d + pad, device=cuda, generator=g).to(torch.bfloat16)
    H = Hfull[:, :d]
    W = (torch.randn(V, d, device=cuda, generator=g) * (scale / d ** 0.5)).to(torch.bfloat16)
    t = torch.randint(0, V, (n,), device=cuda, dtype=torch.int32, generator=g)
    if scale > 1:  # half the targets at the row's arg-max: logp -> 0 must keep its relative accuracy
        x = H.double() @ W.double().T
        t[::2] = x.argmax(dim=1).to(torch.int32)[::2]
    lp, ent = scorer.lmhead_logprob(H, W, t)
    rlp, rent = _ref(H, W, t, 1.0)
    if V == 1:
        assert torch.all(lp == 0) and torch.all(ent.abs() <= 1e-6)
        return
    if scale == 1.0:
        _check(lp, rlp, "logp")
        _check(ent, rent, "entropy")
        return
    # Peaked rows: the fp32 tensor-core accumulation of each logit (d products,
    # |x| up to ~150) perturbs x_v by up to ~u32 * sum_i |h_i w_vi|, and
    # logp = x_y - lse moves by at most twice that (SURVEY.md App. B.2 is exact
    # only for given logits; K6 computes them). Tolerance = the 1e-5 relative
    # bar plus that GEMM rounding bound.
    gemm = 2.0 * 2.0 ** -24 * (H.double().abs() @ W.double().abs().T).max(dim=1).values
    tol = 1e-5 * torch.clamp(rlp.abs(), min=1e-3) + gemm
    err = (lp.double() - rlp).abs()
    assert torch.all(err <= tol), ("logp", float((err / tol).max()))
    etol = 1e-5 * torch.clamp(rent, min=1e-3) + gemm * (1.0 + rent)
    assert torch.all((ent.double() - rent).abs() <= etol), "entropy"


def test_lmhead_empty_and_shape_errors(scorer, cuda):
    from paper_2603_18815_b200.hotpath import RolloutError
    W = torch.zeros(100, 64, device=cuda, dtype=torch.bfloat16)
    H = torch.zeros(0, 64, device=cuda, dtype=torch.bfloat16)
    t = torch.zeros(0, device=cuda, dtype=torch.int32)
    lp, ent = scorer.lmhead_logprob(H, W, t)
    assert lp.numel() == 0
    with pytest.raises(RolloutError) as e:
        scorer.lmhead_logprob(torch.zeros(4, 96, device=cuda, dtype=torch.bfloat16),
                              torch.zeros(100, 96, device=cuda, dtype=torch.bfloat16),
                              torch.zeros(4, device=cuda, dtype=torch.int32))
    assert e.value.code == "shape_mismatch"


def test_lmhead_matches_k2_on_materialised_logits(scorer, cuda):
    """Same rows through K6 and through K2 on explicitly materialised fp32 logits."""
    n, d, V = 256, 1024, 32000
    g = torch.Generator(device=cuda).manual_seed(5)
    H = torch.randn(n, d, device=cuda, generator=g).to(torch.bfloat16)
    W = (torch.randn(V, d, device=cuda, generator=g) * (3.0 / d ** 0.5)).to(torch.bfloat16)
    t = torch.randint(0, V, (n,), device=cuda, dtype=torch.int32, generator=g)
    lp6, ent6 = scorer.lmhead_logprob(H, W, t)
    logits = (H.double() @ W.double().T).float().contiguous()
    lp2, ent2 = scorer.logprob_entropy(logits, t)
    _check(lp6, lp2.double(), "logp vs K2")
    _check(ent6, ent2.double(), "entropy vs K2")


def test_lmhead_throughput_report(scorer, cuda):
    """Qwen3-4B LM head shape (d = 2560, V = 151936): report TFLOP/s (not a bench number)."""
    n, d, V = 16384, 2560, 151936
    H = torch.randn(n, d, device=cuda).to(torch.bfloat16)
    W = (torch.randn(V, d, device=cuda) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    t = torch.randint(0, V, (n,), device=cuda, dtype=torch.int32)
    scorer.lmhead_logprob(H, W, t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        scorer.lmhead_logprob(H, W, t)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    tflops = 2.0 * n * d * V / (ms / 1e3) / 1e12
    print(f"\nK6 lmhead: {n} rows x d {d} x V {V}: {ms:.2f} ms, {tflops:.0f} TFLOP/s, {n / ms * 1e3 / 1e6:.2f} M rows/s")
    assert tflops > 50


def test_score_host_lmhead_mode_matches_materialised_logits(scorer, cuda):
    """Whole step with the fused LM head (hidden-state source) == the same step
    on the explicitly materialised logits (pool source, K2+K4)."""
    from paper_2603_18815_b200 import _native as N
    from paper_2603_18815_b200 import synth
    from paper_2603_18815_b200.hotpath import ScoreConfig
    sh = synth.make_shard("c1", seed=99)
    b = sh.batch
    V, d, A = 32000, 256, sh.n_active
    g = torch.Generator(device=cuda).manual_seed(3)
    H = torch.randn(A, d, generator=g, device=cuda).to(torch.bfloat16)
    W = (torch.randn(V, d, generator=g, device=cuda) * (3.0 / d ** 0.5)).to(torch.bfloat16)
    calls = []

    def hidden_fn(row0, n, rows, seq, cu):
        calls.append((row0, n))
        return H[row0:row0 + n]

    got, _ = scorer.score_host_lmhead(b, ScoreConfig(vocab=V, dtype="bf16", microbatch_rows=1000), hidden_fn, W)
    assert calls[0] == (0, 1000) and sum(n for _, n in calls) == A
    logits = (H.double() @ W.double().T).float().contiguous()
    ref, _ = scorer.score_host(b, ScoreConfig(vocab=V, dtype="fp32", microbatch_rows=A), [logits], fill=False)
    assert got[N.P_N_ACTIVE] == ref[N.P_N_ACTIVE] == A
    for i in range(N.N_PARTIALS):
        if i in (N.P_CLIP_LO, N.P_CLIP_HI) or (i >= N.N_GLOBAL and (i - N.N_GLOBAL) % 5 == 4):
            assert abs(got[i] - ref[i]) <= 2, (i, got[i], ref[i])
        else:
            assert abs(got[i] - ref[i]) <= 1e-5 * max(abs(ref[i]), 1.0), (i, got[i], ref[i])


@pytest.mark.parametrize("n,V", [(40000, 8192), (9000, 151936), (37888, 16384)])
def test_lmhead_multi_wave_and_paced_schedules(scorer, cuda, n, V):
    """Row counts that give several waves of two-chunk CTA-pair units (no
    pacing), a single paced wave, and two full paced waves of one-chunk units
    (148 row tiles on 74 pairs: pacing counted across waves); sampled rows vs
    torch fp64."""
    d = 256
    g = torch.Generator(device=cuda).manual_seed(n)
    H = torch.randn(n, d, device=cuda, generator=g).to(torch.bfloat16)
    W = (torch.randn(V, d, device=cuda, generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    t = torch.randint(0, V, (n,), device=cuda, dtype=torch.int32, generator=g)
    lp, ent = scorer.lmhead_logprob(H, W, t)
    idx = torch.cat([torch.arange(0, 300, device=cuda), torch.arange(n - 300, n, device=cuda),
                     torch.randint(0, n, (400,), device=cuda, generator=g)])
    rlp, rent = _ref(H[idx], W, t[idx], 1.0)
    _check(lp[idx], rlp, "logp")
    _check(ent[idx], rent, "entropy")
