"""Benchmark: masked tokens/s scored (logprob + GRPO loss) on B200, % of the HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One *step* = one pass of the trainer-side hot path over one shard of the
synthetic batch of a BASELINE.json config — by default configs[2], the largest
single-GPU config (Qwen3-8B-shaped: 128 tasks x group 8, 16K-token ~30-turn
trajectories with heavy tool-observation masking, V = 151936, bf16 logits;
only informative groups are scored, as IterationStats::informative hands over):
H2D of the host SoA -> K1 pack -> K3 GRPO -> K2+K4 fused over every logits
micro-batch -> NCCL all-reduce of the partials -> D2H, all through the C-ABI
call prorl_score_host with pinned HOST buffers (the e2e number). `value` is
the same step with its inputs resident in HBM: the device segments
pack+GRPO+score+all-reduce timed with CUDA events on the launching stream.

The logits are the LM-head stand-in (the model forward is out of the
reference's scope): a pool of 3 micro-batch buffers (15 GB,
>> the 126 MB L2) filled by the synthetic generator during warm-up; micro-batch
j reads buffer j % 3, so no L2 reuse between micro-batches. Generation is not
inside the timed region.

Multi-GPU (torchrun): groups are sharded by deterministic LPT (no data-path
collective); the only collective is the NCCL all-reduce of the 332-double
partials inside each step. Timing is the max over ranks. Weak scaling (default)
gives every rank a config-sized shard (the global batch is N x the config's
tasks); the north-star 8-GPU run is the C4 batch split over 8 ranks:
    torchrun --nproc-per-node 8 bench.py --gpus 8 --config c4 --scaling strong

--impl reference: the reference's CPU path on this host's cores (see
run_reference), on the same workload and config dict.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIG_NAMES = {"c1": 0, "c2": 1, "c3": 2, "c4": 3}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--microbatch", type=int, default=16576)  # 148 SMs x 8 warps x 14 rows
    ap.add_argument("--pool", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-backward", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: the global batch grows with N (default); strong: one config-sized batch split N ways")
    return ap.parse_args()


def bytes_per_row(vocab: int, dtype: str) -> int:
    # V * sizeof(logit) + ~26 B of side arrays per active row
    # (target 4 + old_lp 4 + seq 4 + turn 2 + adv 4 + row bookkeeping 8)
    return vocab * (2 if dtype == "bf16" else 4) + 26


K_SCORE_FN = "k_scoreI13__nv_bfloat16Li16ELi2ELi4096ELi8ELb1E"  # the default fused bf16 K2+K4 instantiation


def k_score_stamp() -> str | None:
    """Digest of the SASS of the k_score instantiation the bench runs, read
    from the built library (cuobjdump): an ncu traffic capture is quoted only
    for the kernel binary it was taken on."""
    import hashlib
    lib = ROOT / "paper_2603_18815_b200" / "libprorl_hotpath.so"
    tool = "/usr/local/cuda/bin/cuobjdump" if Path("/usr/local/cuda/bin/cuobjdump").exists() else "cuobjdump"
    try:
        out = subprocess.run([tool, "-sass", str(lib)], capture_output=True, text=True, timeout=60).stdout
    except Exception:
        return None
    h, on, n = hashlib.sha256(), False, 0
    for line in out.splitlines():
        if "Function :" in line:
            on = K_SCORE_FN in line
        elif on and line.strip():
            h.update(line.strip().encode())
            n += 1
    return h.hexdigest()[:16] if n else None


def k_score_traffic(rows_per_launch: int):
    """(DRAM bytes per launch, note) from profiles/k_score_traffic.json — the
    `ncu --set full` capture summarised by scripts/ncu_summary.py full ... --traffic — or (None, why)
    when that capture was taken on other kernel sources."""
    tf = ROOT / "profiles" / "k_score_traffic.json"
    if not tf.exists():
        return None, "no capture (scripts/ncu_summary.py --traffic)"
    try:
        tj = json.loads(tf.read_text())
    except Exception as ex:
        return None, f"unreadable capture: {ex!r}"
    stamp = k_score_stamp()
    if stamp is None or tj.get("sass_stamp") != stamp:
        return None, "stale capture: the k_score binary differs from the one profiles/k_score_traffic.json was taken on"
    return tj["dram_bytes_per_row"] * rows_per_launch, f"ncu capture {tj.get('source', '?')} (kernel SASS stamp matches)"


def measured_peak_gbs():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def global_workload(c: dict, world: int, scaling: str) -> dict:
    """The step's global batch: weak scaling grows the task count with N (every
    rank scores ~one config-sized shard); strong scaling splits the config's."""
    g = dict(c)
    g["tasks"] = c["tasks"] * (world if scaling == "weak" else 1)
    return g


def workload_config(c: dict, config_id: str, gcfg: dict, world: int, scaling: str, n_groups: int,
                    n_active: int) -> dict:
    """The `config` dict — identical for our arm and the reference arm (it names
    the workload; how each arm ran it goes under "run")."""
    return {"workload": c["desc"], "config_id": config_id, "tasks_global": gcfg["tasks"],
            "group_size": c["group"], "global_batch": f"{n_groups} informative groups, {n_active} active rows",
            "seq_len": c["tokens"], "vocab": c["vocab"], "logits_dtype": c["dtype"],
            "parallelism": f"group-sharded dp{world}", "scaling": scaling, "seed": 2603 + c["index"]}


def cpu_reference(gcfg: dict, per_step_s: float, steps: int, warmup: int, microbatch: int) -> dict:
    """The reference's CPU path for this workload, timed on this host's cores.

    Inputs come from the reference's own compiled code (oracle/ref_workload.py:
    generate_workload, mock hash_token / token_logprob, TokenTrajectory::flatten,
    is_informative — oracle/_ref/libref.so); the arithmetic the reference does
    not have (logprob / entropy / GRPO / DAPO loss) is the CPU
    oracle (kind "port"), fp64, all host threads. Each step scores a systematic
    (stratified) sample of the batch's active rows — every stride-th row, a
    different offset per step — sized to ~per_step_s of CPU work; the time is
    the WALL clock of the scoring phases (the synthetic logits are generated
    between them, untimed: they stand in for the LM head) plus the whole
    batch's pack + GRPO wall time pro rata."""
    from oracle import oracle as O
    from oracle import ref_workload as RW
    rb = RW.build(gcfg)
    hb = RW.host_batch(rb)
    oc = O.score_cfg(gcfg["vocab"], gcfg["dtype"], microbatch_rows=microbatch)
    threads = os.cpu_count() or 1
    A = rb.n_active
    probe_rows = threads * 16
    probe = O.score_sample(hb, oc, 2603, 2.0, threads, stride=max(1, A // probe_rows), max_rows=probe_rows)
    rate = probe["n_scored"] / max(probe["timings"][1], 1e-6)
    per_step = int(min(max(rate * per_step_s, threads), A))
    stride = max(1, A // per_step)
    rows = secs = 0.0
    for s in range(warmup + steps):
        r = O.score_sample(hb, oc, 2603, 2.0, threads, stride=stride, offset=s % stride, max_rows=per_step)
        assert r["status"] == 0
        t = r["timings"][1] + r["timings"][0] * r["n_scored"] / max(A, 1)
        if s >= warmup:
            rows += r["n_scored"]
            secs += t
    return {"value": rows / secs, "unit": "masked tokens/s", "cores": threads, "kind": "port",
            "cpu_model": O.cpu_model(), "timing": "wall clock",
            "sample": f"every {stride}th active row of the {A}-row batch ({per_step} rows per step, offset = step "
                      f"mod {stride}); inputs from the reference's compiled generate_workload / hash_token / "
                      f"TokenTrajectory::flatten / is_informative; logits generation (LM-head stand-in) untimed; "
                      f"pack + GRPO of the whole batch pro rata",
            "seconds": secs, "rows": int(rows), "ms_per_step": 1000.0 * secs / max(steps, 1),
            "n_groups": len(rb.groups), "n_active": A}


def measure_backward(sc, pool, c, args, reps: int = 10) -> dict:
    """K5 (dL/dlogits, SURVEY §8 f rank 1) on one full logits micro-batch:
    reads pool[0] (2V B/row), writes the bf16 gradient into pool[1] (2V B/row).
    Not part of the forward metric; reported beside it."""
    import torch
    from paper_2603_18815_b200.hotpath import LossConfig
    n, V = pool[0].shape
    g = torch.Generator(device="cuda").manual_seed(7)
    targets = torch.randint(0, V, (n,), device="cuda", dtype=torch.int32, generator=g)
    logp, _ = sc.logprob_entropy(pool[0], targets)
    old = logp + 0.3 * (torch.rand(n, device="cuda", generator=g) - 0.5)
    adv = torch.randn(64, device="cuda", generator=g, dtype=torch.float64)
    seq = torch.randint(0, 64, (n,), device="cuda", dtype=torch.int32, generator=g)
    for _ in range(2):
        sc.logits_grad(pool[0], targets, logp, old, adv, seq, float(n), grad=pool[1])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        sc.logits_grad(pool[0], targets, logp, old, adv, seq, float(n), grad=pool[1])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    bpr = 2 * V * (2 if c["dtype"] == "bf16" else 4) + 26
    gbs = n * bpr / (ms / 1e3) / 1e9
    peak, kind = measured_peak_gbs()
    return {"kernel": "k_grad (K5: dL/dlogits, bf16 out)", "rows_per_launch": n, "ms_per_launch": ms,
            "rows_per_s": n / (ms / 1e3), "bytes_per_row": bpr, "achieved_gbs": gbs, "frac_of_measured": gbs / peak,
            "frac_of_nominal_8000": gbs / 8000.0}


def measure_train_whole_step(sc, host, cfg, pool, n_active, reps: int = 3) -> dict:
    """The whole per-GPU TRAINING step through the C-ABI (prorl_score_host,
    training mode): H2D, K1, K3, K7 per micro-batch (loss partials + bf16
    dL/dlogits into a gradient pool), all-reduce, D2H; device time.

    The logits pool holds 3 micro-batches, so the scoring bench re-scores
    stale logits (targets not planted -> ratio ~ 0 -> every negative-advantage
    row clips and has a zero gradient, whose pass B skips the exponentials).
    Here every micro-batch is regenerated in the step (fill) so the gradient
    density is the planted one (a few per cent of rows clip), and the
    generator's time - the LM-head stand-in, outside the metric - is measured
    on its own over the same micro-batch sizes and subtracted."""
    import numpy as np
    import torch
    from paper_2603_18815_b200 import _native as N
    gpool = [torch.empty_like(b) for b in pool]  # grad_buffers[j % n_pool]: one per logits buffer
    for _ in range(2):
        sc.score_host(host, cfg, pool, fill=True, seed=2603, train=True, grad_pool=gpool)
    torch.cuda.synchronize()
    tms = []
    for _ in range(reps):
        part, tm = sc.score_host(host, cfg, pool, fill=True, seed=2603, train=True, grad_pool=gpool)
        tms.append(tm)
    torch.cuda.synchronize()
    seg = np.mean(np.array(tms), axis=0)
    # generator alone over the same micro-batch sizes (planted targets, as in fill)
    mb, V = cfg.microbatch_rows, pool[0].shape[1]
    sizes = [min(mb, n_active - r) for r in range(0, n_active, mb)]
    tg = torch.randint(0, V, (mb,), device="cuda", dtype=torch.int32)
    ol = torch.full((mb,), -1.3, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gen_ms = []
    for _ in range(reps):
        e0.record()
        for j, n in enumerate(sizes):
            sc.gen_logits(pool[j % len(pool)], n, j * mb, tg, ol, seed=2603)
        e1.record()
        torch.cuda.synchronize()
        gen_ms.append(e0.elapsed_time(e1))
    gen = float(np.median(gen_ms))
    score = float(seg[2]) - gen
    dev_ms = float(seg[1] + seg[3]) + score
    e2e_ms = float(seg.sum()) - gen
    na = float(part[N.P_N_ACTIVE])
    del gpool
    torch.cuda.empty_cache()
    return {"path": "prorl_score_host training mode (K1, K3, K7 per micro-batch: loss + bf16 dL/dlogits, all-reduce)",
            "logits": "regenerated per micro-batch (planted targets); generator time measured alone and subtracted",
            "generator_ms": gen, "ms_per_step_device": dev_ms, "ms_per_step_e2e": e2e_ms, "score_ms": score,
            "clipped_rows_frac": float(part[N.P_CLIP_LO] + part[N.P_CLIP_HI]) / max(na, 1.0),
            "masked_tokens_per_s": n_active / (dev_ms / 1e3), "e2e_masked_tokens_per_s": n_active / (e2e_ms / 1e3),
            "hbm_gbs_k7": n_active * (2 * (2 if cfg.dtype == "bf16" else 4) * cfg.vocab + 30) / (score / 1e3) / 1e9}


def measure_train_step(sc, pool, c, args, reps: int = 10) -> dict:
    """K7 (one-pass training step: logprob/entropy + loss partials + dL/dlogits
    from ONE read of each logits row, thread-block clusters) on one full logits
    micro-batch, beside the two-pass K2+K4 -> K5 sequence it replaces. Reads
    pool[0], writes the bf16 gradient into pool[1]."""
    import torch
    from paper_2603_18815_b200 import _native as N
    n, V = pool[0].shape
    g = torch.Generator(device="cuda").manual_seed(7)
    targets = torch.randint(0, V, (n,), device="cuda", dtype=torch.int32, generator=g)
    logp, _ = sc.logprob_entropy(pool[0], targets)
    old = logp + 0.3 * (torch.rand(n, device="cuda", generator=g) - 0.5)
    adv = torch.randn(64, device="cuda", generator=g, dtype=torch.float64)
    seq = torch.randint(0, 64, (n,), device="cuda", dtype=torch.int32, generator=g)
    turn = torch.randint(0, 30, (n,), device="cuda", dtype=torch.int16, generator=g)
    part = torch.zeros(N.N_PARTIALS, dtype=torch.float64, device="cuda")
    lp = torch.empty(n, dtype=torch.float32, device="cuda")

    def one_pass():
        sc.score_grad(pool[0], targets, old, adv, seq, turn, float(n), grad=pool[1], partials=part, want_rows=False)

    def two_pass():
        _, lp2, _ = sc.score_rows(pool[0], targets, old, adv, seq, turn, partials=part)
        sc.logits_grad(pool[0], targets, lp2, old, adv, seq, float(n), grad=pool[1])

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    ms1 = timed(one_pass)
    ms2 = timed(two_pass)
    esz = 2 if c["dtype"] == "bf16" else 4
    bpr = 2 * V * esz + 30  # read the row + write its gradient; target, old, adv, seq, turn, row bookkeeping
    gbs = n * bpr / (ms1 / 1e3) / 1e9
    peak, kind = measured_peak_gbs()
    return {"kernel": "k_train (K7: K2+K4+K5, one HBM read + one HBM write per row; second pass from L2)",
            "rows_per_launch": n, "ms_per_launch": ms1, "rows_per_s": n / (ms1 / 1e3), "bytes_per_row": bpr,
            "achieved_gbs": gbs, "frac_of_measured": gbs / peak, "frac_of_nominal_8000": gbs / 8000.0,
            "two_pass_k2k4_k5_ms": ms2, "speedup_vs_two_pass": ms2 / ms1}


def measure_lmhead(sc, c, args, reps: int = 3) -> dict:
    """K6 (fused LM head + logprob, SURVEY §8 f rank 2) at the Qwen3-4B LM-head
    shape (d = 2560, V = config vocab): tcgen05 GEMM with the online-softmax
    epilogue; logits never reach HBM. Reported beside the forward metric."""
    import torch
    n, d, V = 16384, 2560, c["vocab"]
    g = torch.Generator(device="cuda").manual_seed(11)
    H = torch.randn(n, d, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(V, d, device="cuda", generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    t = torch.randint(0, V, (n,), device="cuda", dtype=torch.int32, generator=g)
    logits = torch.empty((n, V), dtype=torch.bfloat16, device="cuda")
    # K6 against what it replaces — cuBLAS bf16 GEMM writing the logits to HBM,
    # then K2 — and against that GEMM alone (the unfused path's floor: a fused
    # kernel at cuBLAS's GEMM speed with a free epilogue would reach
    # unfused / gemm); alternating rounds, best of each (the power-capped
    # clock drifts between rounds)
    runs = {"k6": lambda: sc.lmhead_logprob(H, W, t),
            "unfused": lambda: (torch.matmul(H, W.T, out=logits), sc.logprob_entropy(logits, t)),
            "gemm": lambda: torch.matmul(H, W.T, out=logits)}
    for f in runs.values():
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = {k: float("inf") for k in runs}
    for _ in range(3):
        for k, f in runs.items():
            e0.record()
            for _ in range(reps):
                f()
            e1.record()
            torch.cuda.synchronize()
            best[k] = min(best[k], e0.elapsed_time(e1) / reps)
    ms, unfused_ms, gemm_ms = best["k6"], best["unfused"], best["gemm"]
    del logits
    tf = 2.0 * n * d * V / (ms / 1e3) / 1e12
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    burst = float(peaks.get("bf16_tflops", 1590.0))
    sustained = float(peaks.get("bf16_tflops_sustained", 1400.0))
    del H, W
    return {"kernel": "k_lmhead (K6: tcgen05 LM head + online logsumexp)", "rows": n, "d_model": d, "vocab": V,
            "ms_per_launch": ms, "tflops": tf, "frac_of_measured_bf16_burst": tf / burst,
            "frac_of_measured_bf16_sustained": tf / sustained, "rows_per_s": n / (ms / 1e3),
            "unfused_cublas_gemm_plus_k2_ms": unfused_ms, "speedup_vs_unfused": unfused_ms / ms,
            "cublas_gemm_alone_ms": gemm_ms, "speedup_vs_gemm_alone": gemm_ms / ms,
            "fused_ceiling_at_cublas_gemm_speed": unfused_ms / gemm_ms,
            "logits_bytes_avoided": n * V * 2}


def measure_ingest(shard, reps: int = 3) -> dict:
    """Wire side of the step: the shard's /process responses (reference schema,
    handlers.cpp:57-91, serialised here) -> host SoA by the native parser on all
    host threads (prorl_ingest_responses). Host-only; reported beside the device
    step it would feed (it overlaps the previous step in a pipelined trainer)."""
    from paper_2603_18815_b200.hotpath import ingest_responses
    from tests.wire import to_responses
    b = shard.batch
    resp = to_responses(b)
    nbytes = sum(len(r) for r in resp)
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        got, n_active, _ = ingest_responses(resp, b.group_off)
        best = min(best, time.perf_counter() - t0)
    assert n_active == shard.n_active and len(got.ids) == len(b.ids)
    return {"wire_bytes": nbytes, "tokens": int(len(b.ids)), "ms": best * 1e3, "threads": os.cpu_count(),
            "wire_gb_per_s": nbytes / best / 1e9, "tokens_per_s": len(b.ids) / best,
            "masked_tokens_per_s": shard.n_active / best}


def measure_lmhead_step(sc, host, cfg, c, reps: int = 2) -> dict:
    """The whole step (pack, GRPO, K6 fused LM head + K4 loss, all-reduce) on the
    same shard with a hidden-state source instead of logits (d = 2560): the
    logits of the 0.9 M active rows never exist in HBM."""
    import torch
    from paper_2603_18815_b200.hotpath import ScoreConfig
    d, V = 2560, c["vocab"]
    H = torch.randn(cfg.microbatch_rows, d, device="cuda").to(torch.bfloat16)
    W = (torch.randn(V, d, device="cuda") * (2.0 / d ** 0.5)).to(torch.bfloat16)
    lcfg = ScoreConfig(vocab=V, dtype="bf16", microbatch_rows=cfg.microbatch_rows)
    fn = lambda row0, n, rows, seq, cu: H[:n]  # noqa: E731 — stand-in for the model's final hidden states
    sc.score_host_lmhead(host, lcfg, fn, W)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    seg = np.zeros(5)
    for _ in range(reps):
        _, tm = sc.score_host_lmhead(host, lcfg, fn, W)
        seg += tm
    wall = (time.perf_counter() - t0) / reps
    del H, W
    return {"path": "prorl_score_host with a hidden-state source (K1, K3, K6 tcgen05 LM head + K4, all-reduce)",
            "d_model": d, "ms_per_step_device": float(seg[1] + seg[2] + seg[3]) / reps, "ms_per_step_wall": wall * 1e3}


def run_reference(args):
    """--impl reference: the reference's CPU path for this workload on the host
    cores (cpu_reference: the reference's own compiled code for the inputs and
    the oracle port for the math the reference does not have),
    rank 0 only; the other ranks exit without work. Same metric, unit, config."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2603_18815_b200 import synth_spec as S  # pure Python: no product library on this path
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    c = S.CONFIGS[args.config]
    gcfg = global_workload(c, world, args.scaling)
    per_step = min(6.0, 150.0 / max(args.steps + args.warmup, 1))
    ref = cpu_reference(gcfg, per_step, args.steps, args.warmup, args.microbatch)
    value = ref["value"]
    line = {"metric": "masked tokens/sec scored (logprob+GRPO loss)", "value": value, "unit": "masked tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ref["ms_per_step"],
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": c["dtype"],
            "data": "synthetic", "impl": "reference",
            "config": workload_config(c, args.config, gcfg, world, args.scaling, ref["n_groups"], ref["n_active"]),
            "run": {"where": "rank 0's host cores", "threads": ref["cores"], "cpu_model": ref["cpu_model"],
                    "rows_scored": ref["rows"], "seconds": ref["seconds"]},
            "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "timing")},
            "e2e": {"value": value, "unit": "masked tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2603_18815_b200 import _native as N
    from paper_2603_18815_b200 import synth
    from paper_2603_18815_b200.hotpath import ScoreConfig, Scorer, finalize, nccl_unique_id

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    # PRORL_BENCH_DIST_BACKEND=gloo: orchestration check with several ranks
    # sharing fewer GPUs (the library's NCCL communicator then cannot form and
    # the partials are reduced through torch.distributed); numbers from such a
    # run are not scaling numbers.
    backend = os.environ.get("PRORL_BENCH_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1)
    coll = "cpu" if backend == "gloo" else "cuda"  # device of the torch.distributed tensors
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    c = synth.CONFIGS[args.config]
    # weak scaling: the global batch grows with the GPU count (tasks x N, same
    # seed), groups are LPT-sharded so every rank scores ~one config-sized shard;
    # strong scaling: the config's batch itself is LPT-sharded over the ranks
    gcfg = global_workload(c, world, args.scaling)
    shard = synth.make_shard(gcfg, rank=rank, world=world, seed=2603 + c["index"])
    host = shard.batch.pinned()
    cfg = ScoreConfig(vocab=c["vocab"], dtype=c["dtype"], microbatch_rows=args.microbatch)
    sc = Scorer(local)
    if world > 1 and backend != "nccl":
        torch_allreduce = True  # ranks may share a GPU: no library communicator
    elif world > 1:
        uid = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        try:
            sc.nccl_init(world, rank, uid[0])  # the library's own communicator: the all-reduce runs inside the step
            torch_allreduce = False
        except Exception as ex:  # keep the run alive: reduce the partials through torch.distributed instead
            print(f"warning: prorl_nccl_init failed ({ex}); all-reducing partials via torch.distributed",
                  file=sys.stderr)
            torch_allreduce = True
    else:
        torch_allreduce = False
    tdt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
    pool = [torch.empty((args.microbatch, c["vocab"]), dtype=tdt, device="cuda") for _ in range(args.pool)]
    stream = torch.cuda.current_stream()
    n_mb = (shard.n_active + args.microbatch - 1) // args.microbatch

    def step(fill: bool):
        """One step; with torch_allreduce the partials are summed over
        torch.distributed with the library's collective-safe bookkeeping
        (prorl_fail_partials / prorl_step_status), as prorl_score_host does
        around its own NCCL all-reduce."""
        if not torch_allreduce:
            return sc.score_host(host, cfg, pool, fill=fill, seed=2603)
        own, tm = 0, np.zeros(5, np.float32)
        try:
            p, tm = sc.score_host(host, cfg, pool, fill=fill, seed=2603)
        except N.RolloutError as ex:
            own, p = ex.status, np.zeros(N.N_PARTIALS)
            N.lib.prorl_fail_partials(p.ctypes.data)
        pt = torch.from_numpy(p).to(coll)
        dist.all_reduce(pt)
        p = np.ascontiguousarray(pt.cpu().numpy())
        N.check(N.lib.prorl_step_status(own, p.ctypes.data))
        return p, tm

    # warm-up: the first call fills the pool with generated logits (LM-head stand-in)
    for w in range(max(args.warmup, 1)):
        partials, tm = step(w == 0)
        if w == 0:  # the step whose logits match its targets (reported as "result")
            fill_partials = partials.copy()
    torch.cuda.synchronize()

    # totals over ranks (weak scaling: each rank scores its own groups)
    n_local = torch.tensor([shard.n_active], dtype=torch.float64, device=coll)
    per_rank = [shard.n_active]
    if world > 1:
        gathered = [torch.zeros_like(n_local) for _ in range(world)]
        dist.all_gather(gathered, n_local)
        per_rank = [int(x.item()) for x in gathered]
    n_total = int(sum(per_rank))
    lpt_imbalance = max(per_rank) / (sum(per_rank) / len(per_rank))
    n_groups = len(shard.groups)
    if world > 1:
        g_t = torch.tensor([float(n_groups)], dtype=torch.float64, device=coll)
        dist.all_reduce(g_t)
        n_groups = int(g_t.item())

    clocks = ClockSampler(local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    seg = np.zeros(5)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0.record(stream)
    for _ in range(args.steps):
        partials, tm = step(False)
        seg += tm
    ev1.record(stream)
    torch.cuda.synchronize()
    step_info = sc.last_step_info()  # the library's own count of what the last timed step launched / copied
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    # single-GPU kernel side measurements: N=1 only (at N>1 the whole-step ones
    # would put extra all-reduces on every rank, and one rank failing there
    # would leave its peers waiting in the collective)
    extras = world == 1 and not args.no_backward
    backward = measure_backward(sc, pool, c, args) if args.pool >= 2 and extras else None
    train_step = None
    if args.pool >= 2 and extras:
        try:
            train_step = measure_train_step(sc, pool, c, args)
            train_step["whole_step"] = measure_train_whole_step(sc, host, cfg, pool, shard.n_active)
        except Exception as ex:
            train_step = {"error": repr(ex)}
    lmhead = measure_lmhead(sc, c, args) if extras and c["dtype"] == "bf16" else None
    lmhead_step = None
    if lmhead is not None:
        del pool  # free the 15 GB logits pool: this path never materialises logits
        torch.cuda.empty_cache()
        lmhead_step = measure_lmhead_step(sc, host, cfg, c)
        lmhead_step["masked_tokens_per_s"] = shard.n_active / (lmhead_step["ms_per_step_device"] / 1e3)
    e2e_ms = ev0.elapsed_time(ev1)
    dev_ms = float(seg[1] + seg[2] + seg[3])  # pack+GRPO, score, all-reduce (inputs resident)
    score_ms = float(seg[2])
    t = torch.tensor([e2e_ms, dev_ms, score_ms], dtype=torch.float64, device=coll)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms, dev_ms, score_ms = (float(x) for x in t.tolist())
    K = args.steps
    value = n_total * K / (dev_ms / 1e3)
    e2e = n_total * K / (e2e_ms / 1e3)

    # roofline of the dominant kernel (fused K2+K4), from the live events
    bpr = bytes_per_row(c["vocab"], c["dtype"])
    local_rows = shard.n_active
    peak, peak_kind = measured_peak_gbs()
    achieved = local_rows * bpr * K / (seg[2] / 1e3) / 1e9  # rank-local bytes / rank-local score time
    traffic, traffic_note = k_score_traffic(min(args.microbatch, local_rows))

    if rank == 0:
        res = finalize(fill_partials)
        cpu = None
        ingest = None
        if world == 1 and not args.no_backward:
            try:
                ingest = measure_ingest(shard)
            except Exception as ex:
                ingest = {"error": repr(ex)}
        if world == 1 and not args.no_cpu_baseline:
            try:
                ref = cpu_reference(gcfg, args.cpu_seconds, 1, 0, args.microbatch)
                cpu = {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "timing",
                                           "seconds")}
            except Exception as ex:  # the baseline must not sink the GPU number
                cpu = {"error": repr(ex)}
        launches_per_step = step_info["kernel_launches"]  # K1 (turn scan + per-chunk token pass), K3, K2+K4 x n_mb, reduce, fold
        line = {
            "metric": "masked tokens/sec scored (logprob+GRPO loss)",
            "value": value, "unit": "masked tokens/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": dev_ms / K, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": c["dtype"], "data": "synthetic",
            "config": workload_config(c, args.config, gcfg, world, args.scaling, n_groups, n_total),
            "run": {"lpt_imbalance_max_over_mean": lpt_imbalance, "rank0_groups": len(shard.groups),
                    "rank0_active_rows": shard.n_active, "microbatch_rows": args.microbatch,
                    "micro_batches_per_step": n_mb, "h2d_chunks": step_info["h2d_chunks"], "logits_pool": f"{args.pool} x {args.microbatch} rows "
                    f"({args.pool * args.microbatch * c['vocab'] * (2 if c['dtype'] == 'bf16' else 4) / 1e9:.1f} GB)",
                    "l2": "inputs larger than L2 (logits pool >> 126 MB; no flush needed)"},
            "e2e": {"value": e2e, "unit": "masked tokens/s", "h2d_bytes_per_step": host.bytes_h2d(),
                    "d2h_bytes_per_step": N.N_PARTIALS * 8, "ms_per_step": e2e_ms / K},
            "gpu_launches": launches_per_step * K,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_note": traffic_note, "peak_kind": peak_kind, "frac_of_nominal_8000": achieved / 8000.0,
                         "kernel": "k_score<bf16," + N.lib.prorl_kernel_config().decode() + ",fused> (K2+K4)", "bytes_per_row": bpr},
            "segments_ms_per_step": {"h2d": seg[0] / K, "pack_grpo": seg[1] / K, "score": seg[2] / K,
                                     "allreduce": seg[3] / K, "d2h": seg[4] / K},
            "clocks": clk,
            "result": {"of": "the fill warm-up step (timed steps re-score the pooled logits; same cost)",
                       "loss": res["loss"], "entropy": res["entropy"], "clip_lo_frac": res["clip_lo_frac"],
                       "clip_hi_frac": res["clip_hi_frac"], "n_active": res["n_active"]},
            "cpu_baseline": cpu,
            "backward": backward,
            "train_step": train_step,
            "lmhead": lmhead,
            "lmhead_step": lmhead_step,
            "ingest": ingest,
        }
        print(json.dumps(line), flush=True)
    sc.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
