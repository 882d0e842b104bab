"""The library's own NCCL communicator (prorl_nccl_unique_id / _init / _allreduce),
exercised at world size 1 on the single GPU a test box has: NCCL is resolved at
run time (dlopen of the process's libnccl.so.2), the all-reduce runs inside
prorl_score_host, and a 1-rank sum is the identity — so the step with the
communicator must return exactly the partials of the step without it.
World > 1 host logic (sharding, partial merge) is covered by test_dist_gloo.py."""
import numpy as np
import pytest
import torch

from paper_2603_18815_b200 import _native as N
from paper_2603_18815_b200 import synth
from paper_2603_18815_b200.hotpath import RolloutError, ScoreConfig, Scorer, nccl_unique_id

pytestmark = pytest.mark.gpu


def test_nccl_world1_step_identity(cuda):
    sh = synth.make_shard("c1", seed=5)
    b = sh.batch
    cfg = ScoreConfig(vocab=32000, dtype="fp32", microbatch_rows=2048)
    pool = [torch.empty((cfg.microbatch_rows, cfg.vocab), dtype=torch.float32, device=cuda) for _ in range(2)]
    plain = Scorer(0)
    want, tm0 = plain.score_host(b.pinned(), cfg, pool, fill=True, seed=77)
    assert tm0[3] >= 0.0

    sc = Scorer(0)
    sc.nccl_init(1, 0, nccl_unique_id())
    got, tm = sc.score_host(b.pinned(), cfg, pool, fill=True, seed=77)
    assert np.array_equal(got, want)
    assert got[N.P_N_ACTIVE] == sh.n_active
    assert tm[3] >= 0.0

    # explicit all-reduce of a device vector through the same communicator
    x = torch.arange(N.N_PARTIALS, dtype=torch.float64, device=cuda)
    y = x.clone()
    sc.allreduce(y)
    torch.cuda.synchronize()
    assert torch.equal(x, y)


def test_nccl_init_rejects_bad_rank(cuda):
    sc = Scorer(0)
    with pytest.raises(RolloutError):
        sc.nccl_init(1, 3, nccl_unique_id())
    # the context stays usable
    sc.nccl_init(1, 0, nccl_unique_id())


def test_failed_step_sets_error_rank_flag(cuda):
    """A device-side rejection (token id >= vocab) is folded into
    partials[PRORL_P_ERR_RANKS] before the all-reduce, so with >1 ranks every
    peer would fail with peer_failed instead of summing a void shard; a host
    validation failure still enters the collective (no hang) and keeps its own
    status. At world size 1 the flag comes back to this rank."""
    from paper_2603_18815_b200.hotpath import HostBatchArrays
    sh = synth.make_shard("c1", seed=5)
    b = sh.batch
    cfg = ScoreConfig(vocab=32000, dtype="fp32", microbatch_rows=2048)
    pool = [torch.empty((cfg.microbatch_rows, cfg.vocab), dtype=torch.float32, device=cuda)]
    sc = Scorer(0)
    sc.nccl_init(1, 0, nccl_unique_id())
    bad = HostBatchArrays(b.turns, b.ids.copy(), b.lp, b.reward, b.usable, b.group_off)
    bad.ids[3] = cfg.vocab + 7
    with pytest.raises(RolloutError) as e:
        sc.score_host(bad, cfg, pool, fill=True)
    assert e.value.code == "shape_mismatch"
    short = HostBatchArrays(b.turns, b.ids[:-1], b.lp[:-1], b.reward, b.usable, b.group_off)
    with pytest.raises(RolloutError) as e:
        sc.score_host(short, cfg, pool, fill=True)
    assert e.value.code == "shape_mismatch"
    # the communicator and the ctx stay usable; the flag is clear on success
    got, _ = sc.score_host(b, cfg, pool, fill=True, seed=3)
    assert got[N.P_ERR_RANKS] == 0.0 and got[N.P_N_ACTIVE] == sh.n_active
