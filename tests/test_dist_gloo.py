"""N > 1 host path on CPU (gloo, world_size 2 and 4): deterministic LPT group
sharding, disjoint/complete shards, and the partials all-reduce.

Each rank scores its own groups with the CPU oracle (the device path is
replaced by the oracle here: there is no GPU) and the 332-double partials are
summed with torch.distributed (gloo), exactly as prorl_allreduce sums them over
NCCL on the GPUs. Because GRPO statistics are per group and the synthetic
logits of a row are keyed by (global rollout, position), the all-reduced
result must equal the single-rank result up to fp64 summation order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2603_18815_b200 import synth

CFG = dict(index=0, tasks=12, group=4, tokens=384, turns=7, vocab=1003, dtype="fp32", asst_share=0.45,
           lengths="lognormal", desc="test")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _score(shard):
    b = shard.batch
    hb = O.host_batch(b.turns, b.ids, b.lp, b.reward, b.usable, b.group_off, b.rollout_key)
    r = O.score_batch(hb, O.score_cfg(CFG["vocab"], CFG["dtype"]), 77, 2.0, nthreads=2)
    assert r["status"] == 0
    return r["partials"]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shard = synth.make_shard(CFG, rank=rank, world=world, seed=5)
    p = torch.from_numpy(_score(shard))
    groups = [None] * world
    dist.all_gather_object(groups, shard.groups)
    dist.all_reduce(p, op=dist.ReduceOp.SUM)
    if rank == 0:
        out.put((p.numpy().tolist(), groups))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_allreduce_equals_single_rank(world):
    full = synth.make_shard(CFG, seed=5)
    P1 = _score(full)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, groups = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # shards are disjoint and cover every informative group
    flat = [g for gs in groups for g in gs]
    assert sorted(flat) == sorted(full.groups) and len(flat) == len(set(flat))
    got = np.array(got)
    assert got[1] == P1[1]                       # N_active exact
    assert got[9] == P1[9]                       # N_rollouts exact
    np.testing.assert_allclose(got, P1, rtol=1e-11, atol=1e-9)


def test_lpt_balances_skewed_groups():
    from paper_2603_18815_b200.hotpath import shard_lpt
    rng = np.random.default_rng(0)
    load = np.exp(rng.normal(10, 0.6, 256)).astype(np.int64)  # C4-like skew
    for world in (2, 4, 8):
        owner = shard_lpt(load, world)
        per = np.bincount(owner, weights=load, minlength=world)
        assert per.max() / per.mean() < 1.02


def _fail_worker(rank, world, port, failing, out):
    """One step's collective-safe failure bookkeeping (prorl_fail_partials /
    prorl_step_status — what prorl_score_host does around its NCCL all-reduce)
    with the partials reduced over gloo: ranks in `failing` contribute the
    failure record, every rank decides its outcome from the reduced vector."""
    import ctypes as C
    from paper_2603_18815_b200 import _native as N
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shard = synth.make_shard(CFG, rank=rank, world=world, seed=5)
    p = _score(shard)
    own = N.PRORL_E_SHAPE if rank in failing else 0
    if own:
        N.lib.prorl_fail_partials(p.ctypes.data)
    t = torch.from_numpy(p)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    red = np.ascontiguousarray(t.numpy())
    st = N.lib.prorl_step_status(own, red.ctypes.data)
    msg = N.lib.prorl_last_error().decode() if st else ""
    out.put((rank, st, msg, float(red[N.P_ERR_RANKS])))
    dist.destroy_process_group()
    del C


@pytest.mark.parametrize("failing", [(), (1,), (0, 1)])
def test_collective_safe_failure_world2(failing):
    from paper_2603_18815_b200 import _native as N
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fail_worker, args=(r, world, port, failing, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, st, msg, err_ranks in res:
        assert err_ranks == len(failing)
        if rank in failing:
            assert st == N.PRORL_E_SHAPE                  # its own error wins
        elif failing:
            assert st == N.PRORL_E_PEER_FAILED and "peer_failed" in msg
        else:
            assert st == 0
