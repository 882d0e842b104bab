"""Python handle over the C-ABI (include/prorl_hotpath.h) for tests and the bench.

The product is the C/C++ library; this module only moves torch device
pointers / numpy host pointers across ctypes and maps status codes onto
`RolloutError` (the rollout::Error code convention, errors.hpp:10-18).
Every call runs the sm_100a kernels; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._native import RolloutError, check, ptr  # noqa: F401  (RolloutError re-exported)

_DT = {torch.bfloat16: N.PRORL_BF16, torch.float32: N.PRORL_FP32}


def _adv(adv: torch.Tensor) -> torch.Tensor:
    """Advantages cross the C-ABI as fp64 (prorl_grpo_adv's output type)."""
    if adv.dtype != torch.float64:
        raise TypeError(f"advantages must be float64 (got {adv.dtype})")
    return adv


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


@dataclass
class LossConfig:
    eps_lo: float = 0.2
    eps_hi: float = 0.28
    n_buckets: int = N.TURN_BUCKETS
    kl_coef: float = 0.0  # k3 KL vs the reference policy (1e-4); needs ref_lp

    def c(self) -> N.LossCfg:
        return N.LossCfg(self.eps_lo, self.eps_hi, self.n_buckets, self.kl_coef)


@dataclass
class ScoreConfig:
    """Mirror of the C++ rollout::train::ScoreConfig."""
    vocab: int
    dtype: str = "bf16"
    inv_temperature: float = 1.0
    adv_eps: float = 1e-6
    ddof: int = 1
    microbatch_rows: int = 16576  # 7 waves of the 148 x 16 K2 warps
    loss: LossConfig = None
    gate_tolerance: float = 0.0   # is_informative tolerance (K3 gate; the host batch must use the same)

    def c(self) -> N.ScoreCfg:
        loss = self.loss or LossConfig()
        return N.ScoreCfg(loss.c(), self.inv_temperature, self.adv_eps, self.ddof, self.vocab,
                          N.PRORL_BF16 if self.dtype == "bf16" else N.PRORL_FP32, self.microbatch_rows,
                          self.gate_tolerance)


class Scorer:
    """One prorl_ctx on one CUDA device."""

    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        check(N.lib.prorl_ctx_create(device, C.byref(h)))
        self.ctx = h

    def close(self) -> None:
        if self.ctx:
            N.lib.prorl_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check_errors(self, stream=None) -> None:
        check(N.lib.prorl_check_errors(self.ctx, _stream(stream)))

    # ---- K1 ----
    def pack(self, turns: np.ndarray, ids: torch.Tensor, lp: torch.Tensor, n_seq: int, vocab: int,
             n_active: int, stream=None) -> dict:
        dev = ids.device
        n_tok = ids.numel()
        t_dev = torch.from_numpy(turns.view(np.uint8).reshape(-1)).to(dev)
        e = lambda n, dt: torch.empty(max(n, 1), dtype=dt, device=dev)
        out = {
            "tokens": e(n_tok, torch.int32), "loss_mask": e(n_tok, torch.uint8), "turn_id": e(n_tok, torch.int16),
            "seq_id": e(n_tok, torch.int32), "pos_id": e(n_tok, torch.int32), "cu_seqlens": e(n_seq + 1, torch.int32),
            "old_lp": e(n_tok, torch.float32), "act_row": e(n_active, torch.int32),
            "act_target": e(n_active, torch.int32), "act_old_lp": e(n_active, torch.float32),
            "act_seq": e(n_active, torch.int32), "act_turn": e(n_active, torch.int16),
            "n_active": torch.zeros(1, dtype=torch.int64, device=dev),
        }
        pk = N.Packed(*[ptr(out[f]) for f, _ in N.Packed._fields_])
        check(N.lib.prorl_pack(self.ctx, ptr(t_dev), len(turns), ptr(ids), ptr(lp), n_tok, n_seq, vocab,
                               C.byref(pk), _stream(stream)))
        self.check_errors(stream)
        for k in ("tokens", "loss_mask", "turn_id", "seq_id", "pos_id", "old_lp"):
            out[k] = out[k][:n_tok]
        for k in ("act_row", "act_target", "act_old_lp", "act_seq", "act_turn"):
            out[k] = out[k][:n_active]
        return out

    # ---- K3 ----
    def grpo_adv(self, reward: torch.Tensor, usable: torch.Tensor, group_off: torch.Tensor, ddof: int = 1,
                 eps: float = 1e-6, tol: float = 0.0, partials: torch.Tensor | None = None, stream=None):
        adv = torch.empty(max(reward.numel(), 1), dtype=torch.float64, device=reward.device)
        ng = group_off.numel() - 1
        info = torch.empty(max(ng, 1), dtype=torch.uint8, device=reward.device)
        check(N.lib.prorl_grpo_adv(self.ctx, ptr(reward), ptr(usable), ptr(group_off), ng, ddof, eps, tol, ptr(adv),
                                   ptr(info), ptr(partials), _stream(stream)))
        return adv[:reward.numel()], info[:ng]

    # ---- K2 ----
    def logprob_entropy(self, logits: torch.Tensor, targets: torch.Tensor, rows: torch.Tensor | None = None,
                        inv_temp: float = 1.0, vocab: int | None = None, stream=None):
        n = targets.numel()
        logp = torch.empty(n, dtype=torch.float32, device=targets.device)
        ent = torch.empty(n, dtype=torch.float32, device=targets.device)
        V = vocab if vocab is not None else logits.shape[1]
        check(N.lib.prorl_logprob_entropy(self.ctx, ptr(logits), _DT[logits.dtype], logits.stride(0), V, ptr(rows),
                                          ptr(targets), n, inv_temp, ptr(logp), ptr(ent), _stream(stream)))
        return logp, ent

    # ---- K4 ----
    def clipped_loss(self, logp, entropy, old_lp, adv, row_seq, row_turn, cfg: LossConfig | None = None,
                     partials: torch.Tensor | None = None, ref_lp=None, stream=None) -> torch.Tensor:
        if partials is None:
            partials = torch.zeros(N.N_PARTIALS, dtype=torch.float64, device=logp.device)
        c = (cfg or LossConfig()).c()
        check(N.lib.prorl_clipped_loss(self.ctx, ptr(logp), ptr(entropy), ptr(old_lp), ptr(_adv(adv)), ptr(row_seq),
                                       ptr(row_turn), ptr(ref_lp), logp.numel(), C.byref(c), ptr(partials),
                                       _stream(stream)))
        return partials

    # ---- K2+K4 fused ----
    def score_rows(self, logits, targets, old_lp, adv, row_seq, row_turn, rows=None, inv_temp: float = 1.0,
                   cfg: LossConfig | None = None, partials=None, want_rows: bool = True, vocab: int | None = None,
                   ref_lp=None, stream=None):
        n = targets.numel()
        dev = targets.device
        if partials is None:
            partials = torch.zeros(N.N_PARTIALS, dtype=torch.float64, device=dev)
        logp = torch.empty(n, dtype=torch.float32, device=dev) if want_rows else None
        ent = torch.empty(n, dtype=torch.float32, device=dev) if want_rows else None
        c = (cfg or LossConfig()).c()
        V = vocab if vocab is not None else logits.shape[1]
        check(N.lib.prorl_score_rows(self.ctx, ptr(logits), _DT[logits.dtype], logits.stride(0), V, ptr(rows),
                                     ptr(targets), ptr(old_lp), ptr(_adv(adv)), ptr(row_seq), ptr(row_turn), ptr(ref_lp), n,
                                     inv_temp, C.byref(c), ptr(logp), ptr(ent), ptr(partials), _stream(stream)))
        return partials, logp, ent

    # ---- K5: backward through the log-softmax ----
    def logits_grad(self, logits, targets, logp, old_lp, adv, row_seq, n_global: float, rows=None,
                    inv_temp: float = 1.0, cfg: LossConfig | None = None, grad=None, vocab: int | None = None,
                    want_dlogp: bool = False, ref_lp=None, stream=None):
        """dL/dlogits (same dtype/layout as logits; grad=logits for in place)."""
        if grad is None:
            grad = torch.empty_like(logits)
        n = targets.numel()
        dl = torch.empty(n, dtype=torch.float32, device=targets.device) if want_dlogp else None
        c = (cfg or LossConfig()).c()
        V = vocab if vocab is not None else logits.shape[1]
        check(N.lib.prorl_logits_grad(self.ctx, ptr(logits), _DT[logits.dtype], logits.stride(0), V, ptr(rows),
                                      ptr(targets), ptr(logp), ptr(old_lp), ptr(_adv(adv)), ptr(row_seq), ptr(ref_lp), n,
                                      inv_temp,
                                      C.byref(c), float(n_global), ptr(grad), grad.stride(0), ptr(dl),
                                      _stream(stream)))
        return grad, dl

    # ---- K7: one-pass training step (K2 + K4 + K5 from one read of each row) ----
    def score_grad(self, logits, targets, old_lp, adv, row_seq, row_turn, n_global: float, rows=None,
                   inv_temp: float = 1.0, cfg: LossConfig | None = None, grad=None, partials=None,
                   want_rows: bool = True, want_dlogp: bool = False, vocab: int | None = None, ref_lp=None,
                   stream=None):
        """(partials, logp, entropy, grad, dlogp): score_rows + logits_grad with one HBM read of each row."""
        n = targets.numel()
        dev = targets.device
        if partials is None:
            partials = torch.zeros(N.N_PARTIALS, dtype=torch.float64, device=dev)
        if grad is None:
            grad = torch.empty_like(logits)
        logp = torch.empty(n, dtype=torch.float32, device=dev) if want_rows else None
        ent = torch.empty(n, dtype=torch.float32, device=dev) if want_rows else None
        dl = torch.empty(n, dtype=torch.float32, device=dev) if want_dlogp else None
        c = (cfg or LossConfig()).c()
        V = vocab if vocab is not None else logits.shape[1]
        check(N.lib.prorl_score_grad(self.ctx, ptr(logits), _DT[logits.dtype], logits.stride(0), V, ptr(rows),
                                     ptr(targets), ptr(old_lp), ptr(_adv(adv)), ptr(row_seq), ptr(row_turn), ptr(ref_lp), n,
                                     inv_temp, C.byref(c), float(n_global), ptr(logp), ptr(ent), ptr(partials),
                                     ptr(grad), grad.stride(0), ptr(dl), _stream(stream)))
        return partials, logp, ent, grad, dl

    # ---- K6: fused LM head (tcgen05) ----
    def lmhead_logprob(self, hidden: torch.Tensor, weight: torch.Tensor, targets: torch.Tensor,
                       inv_temp: float = 1.0, stream=None):
        """logp / entropy of softmax(hidden @ weight.T * inv_temp) without materialising the logits."""
        n, d = hidden.shape
        V = weight.shape[0]
        logp = torch.empty(n, dtype=torch.float32, device=hidden.device)
        ent = torch.empty(n, dtype=torch.float32, device=hidden.device)
        check(N.lib.prorl_lmhead_logprob(self.ctx, ptr(hidden), hidden.stride(0), ptr(weight), weight.stride(0), d, V,
                                         ptr(targets), n, inv_temp, ptr(logp), ptr(ent), _stream(stream)))
        return logp, ent

    # ---- synthetic LM head ----
    def gen_logits(self, out: torch.Tensor, n_rows: int, row_key0: int, targets=None, old_lp=None, seed: int = 0,
                   sigma: float = 2.0, vocab: int | None = None, stream=None) -> torch.Tensor:
        V = vocab if vocab is not None else out.shape[1]
        check(N.lib.prorl_gen_logits(self.ctx, ptr(out), _DT[out.dtype], out.stride(0), V, n_rows, row_key0,
                                     ptr(targets), ptr(old_lp), seed, sigma, _stream(stream)))
        return out

    def row_keys(self, rows, seq, cu_seqlens, rollout_key=None, stream=None) -> torch.Tensor:
        """Synthetic-logits keys of active rows (rollout_key[seq] * 2^20 + position)."""
        keys = torch.empty(max(rows.numel(), 1), dtype=torch.int64, device=rows.device)
        check(N.lib.prorl_row_keys(self.ctx, ptr(rows), ptr(seq), ptr(cu_seqlens), ptr(rollout_key), rows.numel(),
                                   ptr(keys), _stream(stream)))
        return keys[:rows.numel()]

    def gen_logits_keyed(self, out: torch.Tensor, keys: torch.Tensor, targets=None, old_lp=None, seed: int = 0,
                         sigma: float = 2.0, vocab: int | None = None, stream=None) -> torch.Tensor:
        V = vocab if vocab is not None else out.shape[1]
        check(N.lib.prorl_gen_logits_keyed(self.ctx, ptr(out), _DT[out.dtype], out.stride(0), V, keys.numel(),
                                           ptr(keys), ptr(targets), ptr(old_lp), seed, sigma, _stream(stream)))
        return out

    # ---- NCCL ----
    def nccl_init(self, world: int, rank: int, uid: bytes) -> None:
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        check(N.lib.prorl_nccl_init(self.ctx, world, rank, C.addressof(buf)))

    def allreduce(self, partials: torch.Tensor, stream=None) -> None:
        check(N.lib.prorl_allreduce(self.ctx, ptr(partials), partials.numel(), _stream(stream)))

    def score_host_lmhead(self, batch: "HostBatchArrays", cfg: ScoreConfig, hidden_fn, weight: torch.Tensor,
                          stream=None):
        """Whole step with the fused LM head (K6): hidden_fn(row0, n, rows, seq, cu) -> bf16 [n x d] device
        tensor (kept alive until the next call); weight bf16 [V x d]."""
        keep = []

        def cb(user, row0, n, rows, seq, cu, out_ptr, out_stride, strm):
            try:
                h = hidden_fn(row0, n, rows, seq, cu)
                keep[:] = [h]
                out_ptr[0] = h.data_ptr()
                out_stride[0] = h.stride(0)
                return 0
            except Exception:  # noqa: BLE001 — reported as a C status
                return -3
        fn = N.HIDDEN_FN(cb)
        hb = batch.c()
        dummy = (C.c_void_p * 1)(None)
        lp = N.LogitsPool(C.cast(dummy, C.c_void_p), 0, 0, 0, 0, 0.0, 0, None, None,
                          C.cast(fn, C.c_void_p), ptr(weight), weight.stride(0), weight.shape[1], 0,
                          0, 0, 0.0, None, None, None, None, None)
        out = np.zeros(N.N_PARTIALS, dtype=np.float64)
        tm = np.zeros(5, dtype=np.float32)
        sc = cfg.c()
        check(N.lib.prorl_score_host(self.ctx, C.byref(hb), C.byref(sc), C.byref(lp), ptr(out), ptr(tm),
                                     _stream(stream)))
        return out, tm

    def last_step_info(self) -> dict:
        """What the last score_host call did: kernel launches, micro-batches, H2D chunks and bytes."""
        si = N.StepInfo()
        check(N.lib.prorl_last_step_info(self.ctx, C.byref(si)))
        return {k: getattr(si, k) for k, _ in N.StepInfo._fields_}

    # ---- whole per-GPU step from host buffers ----
    def score_host(self, batch: "HostBatchArrays", cfg: ScoreConfig, pool: list[torch.Tensor], fill: bool,
                   seed: int = 0, sigma: float = 2.0, stream=None, train: bool = False, n_global: float = 0.0,
                   grad_pool: list[torch.Tensor] | None = None, grad_fn=None, ref_fn=None):
        """Whole step through prorl_score_host. train=True runs K7 per micro-batch (loss partials + dL/dlogits,
        in place or into grad_pool); grad_fn(row0, n, grad_ptr, row_stride) sees each micro-batch's gradient."""
        if grad_pool is not None and len(grad_pool) != len(pool):
            raise ValueError("grad_pool needs one buffer per logits buffer (grad_buffers[j % n_pool])")
        hb = batch.c()
        bufs = (C.c_void_p * len(pool))(*[ptr(b) for b in pool])
        gbufs = (C.c_void_p * len(grad_pool))(*[ptr(b) for b in grad_pool]) if grad_pool else None
        cb = None
        if grad_fn is not None:
            def _cb(user, row0, n, g, stride, strm):
                try:
                    grad_fn(row0, n, g, stride)
                    return 0
                except Exception:  # noqa: BLE001 — reported as a C status
                    return -3
            cb = N.GRAD_FN(_cb)
        rcb, keep = None, []
        if ref_fn is not None:
            def _rcb(user, row0, n, rows, seq, cu, targets, out_ptr, strm):
                try:
                    r = ref_fn(row0, n, rows, seq, cu, targets)  # fp32 device tensor [n]
                    keep[:] = [r]
                    out_ptr[0] = r.data_ptr()
                    return 0
                except Exception:  # noqa: BLE001 — reported as a C status
                    return -3
            rcb = N.REF_FN(_rcb)
        lp = N.LogitsPool(C.cast(bufs, C.c_void_p), len(pool), 1 if fill else 0, pool[0].stride(0), seed, sigma, 0,
                          None, None, None, None, 0, 0, 0, 1 if train else 0, 0, float(n_global),
                          C.cast(gbufs, C.c_void_p) if gbufs is not None else None,
                          C.cast(cb, C.c_void_p) if cb is not None else None, None,
                          C.cast(rcb, C.c_void_p) if rcb is not None else None, None)
        out = np.zeros(N.N_PARTIALS, dtype=np.float64)
        tm = np.zeros(5, dtype=np.float32)
        sc = cfg.c()
        check(N.lib.prorl_score_host(self.ctx, C.byref(hb), C.byref(sc), C.byref(lp), ptr(out), ptr(tm),
                                     _stream(stream)))
        return out, tm


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(N.lib.prorl_nccl_unique_id(C.addressof(buf)))
    return bytes(buf)


def shard_lpt(load: np.ndarray, world: int) -> np.ndarray:
    load = np.ascontiguousarray(load, dtype=np.int64)
    owner = np.zeros(len(load), dtype=np.int32)
    check(N.lib.prorl_shard_lpt(len(load), ptr(load), world, ptr(owner)))
    return owner


def ingest_responses(responses: list[bytes], group_off, tolerance: float = 0.0, threads: int = 0):
    """/process response JSON (handlers.cpp:57-91 schema) -> (HostBatchArrays, n_active, n_informative)
    via the native single-pass parser (prorl_ingest_responses)."""
    n = len(responses)
    bufs = (C.c_char_p * n)(*responses)
    lens = np.array([len(r) for r in responses], dtype=np.uint64)
    goff = np.ascontiguousarray(group_off, dtype=np.int32)
    res = N.IngestResult()
    check(N.lib.prorl_ingest_responses(C.cast(bufs, C.c_void_p), ptr(lens), ptr(goff), len(goff) - 1, tolerance,
                                       threads, C.byref(res)))
    try:
        b = res.batch

        def arr(p, n, dt):
            if n == 0 or not p:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint8)), shape=(n * np.dtype(dt).itemsize,)).view(
                dt).copy()
        out = HostBatchArrays(turns=arr(b.turns, b.n_turns, N.TURN_DTYPE), ids=arr(b.ids, b.n_tokens, np.int64),
                              lp=arr(b.lp, b.n_tokens, np.float64), reward=arr(b.reward, b.n_rollouts, np.float64),
                              usable=arr(b.usable, b.n_rollouts, np.uint8), group_off=goff.copy())
        return out, res.n_active, res.n_informative
    finally:
        N.lib.prorl_ingest_free(C.byref(res))


def synth_rewards(num_prompts: int, n: int, seed: int, p_informative: float = 0.5) -> np.ndarray:
    out = np.zeros(num_prompts * n, dtype=np.float64)
    check(N.lib.prorl_synth_rewards(num_prompts, n, seed, p_informative, ptr(out)))
    return out.reshape(num_prompts, n)


@dataclass
class HostBatchArrays:
    """Host SoA of one shard (prorl_host_batch). Arrays must stay alive."""
    turns: np.ndarray      # TURN_DTYPE
    ids: np.ndarray        # int64 wire TokenIds (types.hpp:12)
    lp: np.ndarray         # float64 wire logprobs (trajectory.hpp:31)
    reward: np.ndarray     # float64 per rollout slot
    usable: np.ndarray     # uint8 per rollout slot (0 = FAILED)
    group_off: np.ndarray  # int32 [n_groups+1]
    rollout_key: np.ndarray | None = None  # int64 global rollout identity per slot (synthetic-logits key)

    def c(self) -> N.HostBatch:
        return N.HostBatch(ptr(self.turns), len(self.turns), ptr(self.ids), ptr(self.lp), len(self.ids),
                           ptr(self.reward), ptr(self.usable), len(self.reward), ptr(self.group_off),
                           len(self.group_off) - 1, ptr(self.rollout_key))

    def pinned(self) -> "HostBatchArrays":
        """Copy into page-locked host memory (torch pinned tensors)."""
        def pin(a):
            t = torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1)).pin_memory()
            return t.numpy().view(a.dtype).reshape(a.shape)
        return HostBatchArrays(*(pin(getattr(self, f)) for f in
                                 ("turns", "ids", "lp", "reward", "usable", "group_off")),
                               rollout_key=None if self.rollout_key is None else pin(self.rollout_key))

    @property
    def n_tokens(self) -> int:
        return len(self.ids)

    @property
    def n_rollouts(self) -> int:
        return len(self.reward)

    @property
    def n_groups(self) -> int:
        return len(self.group_off) - 1

    def bytes_h2d(self) -> int:
        extra = 0 if self.rollout_key is None else self.rollout_key.nbytes
        return extra + sum(getattr(self, f).nbytes for f in ("turns", "ids", "lp", "reward", "usable", "group_off"))


def finalize(p: np.ndarray) -> dict:
    """Host-side finalisation of the all-reduced partials."""
    n = max(p[N.P_N_ACTIVE], 1.0)
    out = {
        "loss": p[N.P_LOSS_SUM] / n, "n_active": int(p[N.P_N_ACTIVE]), "entropy": p[N.P_ENTROPY_SUM] / n,
        "logp": p[N.P_LOGP_SUM] / n, "ratio": p[N.P_RATIO_SUM] / n, "clip_lo_frac": p[N.P_CLIP_LO] / n,
        "clip_hi_frac": p[N.P_CLIP_HI] / n, "kl_k1": p[N.P_KL1_SUM] / n, "kl_k3": p[N.P_KL_SUM] / n,
        "adv_sum": p[N.P_ADV_SUM],
        "n_rollouts": int(p[N.P_N_ROLLOUTS]),
    }
    per_turn = p[N.N_GLOBAL:].reshape(N.TURN_BUCKETS, N.N_PER_TURN)
    out["per_turn"] = [
        {"turn": k, "n": int(r[0]), "loss": r[1] / max(r[0], 1), "entropy": r[2] / max(r[0], 1),
         "logp": r[3] / max(r[0], 1), "clip_frac": r[4] / max(r[0], 1)}
        for k, r in enumerate(per_turn) if r[0] > 0]
    return out
