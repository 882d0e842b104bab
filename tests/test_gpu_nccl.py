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
