"""ctypes loader for the CPU oracle (oracle/liboracle.so) and the compiled
reference (oracle/_ref/libref.so).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() (as the
checker) and bench.py's cpu_baseline / --impl reference leg. The product path
(paper_2603_18815_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libref.so"
N_PARTIALS = 332

vp = C.c_void_p
i32, i64, u64, f32, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double


def build(ref: bool = True) -> None:
    """make -C oracle (liboracle.so, and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "liboracle.so"], check=True)
    if ref:
        subprocess.run([str(HERE / "build_ref.sh")], check=True, capture_output=True)


class OraclePacked(C.Structure):
    _fields_ = [(n, vp) for n in ("tokens", "loss_mask", "turn_id", "seq_id", "pos_id", "cu_seqlens", "old_lp",
                                  "act_row", "act_target", "act_old_lp", "act_seq", "act_turn")] + [("n_active", i64)]


class LossCfg(C.Structure):  # layout of prorl_loss_cfg (include/prorl_hotpath.h)
    _fields_ = [("eps_lo", f32), ("eps_hi", f32), ("n_buckets", i32), ("kl_coef", f32)]


class ScoreCfg(C.Structure):  # layout of prorl_score_cfg
    _fields_ = [("loss", LossCfg), ("inv_temperature", f32), ("adv_eps", f32), ("ddof", i32), ("vocab", i32),
                ("dtype", i32), ("microbatch_rows", i32), ("gate_tolerance", f64)]


class HostBatch(C.Structure):  # layout of prorl_host_batch
    _fields_ = [("turns", vp), ("n_turns", i64), ("ids", vp), ("lp", vp), ("n_tokens", i64), ("reward", vp),
                ("usable", vp), ("n_rollouts", i32), ("group_off", vp), ("n_groups", i32), ("rollout_key", vp)]


def host_batch(turns, ids, lp, reward, usable, group_off, rollout_key=None) -> HostBatch:
    return HostBatch(turns.ctypes.data, len(turns), ids.ctypes.data, lp.ctypes.data, len(ids), reward.ctypes.data,
                     usable.ctypes.data, len(reward), group_off.ctypes.data, len(group_off) - 1,
                     None if rollout_key is None else rollout_key.ctypes.data)


def score_cfg(vocab, dtype="bf16", inv_temperature=1.0, adv_eps=1e-6, ddof=1, eps_lo=0.2, eps_hi=0.28,
              n_buckets=64, microbatch_rows=16384, gate_tolerance=0.0) -> ScoreCfg:
    return ScoreCfg(LossCfg(eps_lo, eps_hi, n_buckets, 0), inv_temperature, adv_eps, ddof, vocab,
                    0 if dtype == "bf16" else 1, microbatch_rows, gate_tolerance)


def _p(a):
    return None if a is None else a.ctypes.data


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not ORACLE_SO.exists():
            build(ref=False)
        L = C.CDLL(str(ORACLE_SO))
        sig = {
            "oracle_fnv1a64": (u64, [vp, C.c_size_t, u64]),
            "oracle_hash_token": (i64, [u64, vp, i64, u64, i64]),
            "oracle_token_logprob": (f64, [i64]),
            "oracle_validate_turn": (C.c_int, [C.c_int, i64, i64, i64]),
            "oracle_flatten": (i64, [C.c_int, vp, vp, vp, i64, i64, vp, i64]),
            "oracle_usable_rewards": (C.c_int, [C.c_int, vp, vp, vp, vp]),
            "oracle_is_informative": (C.c_int, [C.c_int, vp, vp, vp, f64]),
            "oracle_pack": (C.c_int, [vp, i64, vp, vp, i64, i32, i32, C.POINTER(OraclePacked)]),
            "oracle_grpo": (None, [vp, vp, vp, i32, i32, f64, f64, vp, vp, vp, vp]),
            "oracle_gen_logits": (None, [vp, C.c_int, i64, i32, i64, i64, vp, vp, u64, f32]),
            "oracle_row_logprob": (None, [vp, C.c_int, i32, i32, f32, vp, vp]),
            "oracle_logprob_entropy": (None, [vp, C.c_int, i64, i32, vp, vp, i64, f32, vp, vp]),
            "oracle_loss": (None, [vp, vp, vp, vp, vp, vp, vp, i64, f32, f32, f32, C.c_int, vp, vp, vp]),
            "oracle_score_batch": (C.c_int, [vp, vp, u64, f32, C.c_int, i64, i64, vp, vp, vp, vp, vp, vp, vp]),
            "oracle_score_sample": (C.c_int, [vp, vp, u64, f32, C.c_int, i64, i64, i64, vp, vp, vp, vp, vp, vp]),
            "oracle_logits_grad": (None, [vp, C.c_int, i64, i32, vp, vp, vp, vp, vp, vp, i64, f32, f32, f32, f32, f64,
                                          vp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def ref_lib() -> C.CDLL | None:
    """The compiled reference, or None when it was not built (no /root/reference)."""
    if not REF_SO.exists():
        return None
    L = C.CDLL(str(REF_SO))
    sig = {
        "ref_validate_turn": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int]),
        "ref_flatten": (i64, [C.c_int, vp, vp, vp, vp, i64, i64, vp, i64]),
        "ref_usable_rewards": (C.c_int, [C.c_int, vp, vp, vp, vp]),
        "ref_is_informative": (C.c_int, [C.c_int, vp, vp, vp, f64]),
        "ref_fnv1a64": (u64, [vp, C.c_size_t]),
        "ref_hash_token": (i64, [u64, vp, i64, u64, i64]),
        "ref_hash_tokens": (None, [u64, vp, i64, u64, i64, i64, vp, vp]),
        "ref_token_logprob": (f64, [i64]),
        "ref_prompt_digest": (u64, [vp, i64]),
        "ref_generate_workload_rewards": (C.c_int, [C.c_int, C.c_int, u64, f64, vp]),
        "ref_process_response": (i64, [C.c_char_p, C.c_int, vp, vp, vp, vp, f64, C.c_int, C.c_char_p, vp, i64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


# ---- convenience wrappers ------------------------------------------------------

def pack(turns: np.ndarray, ids: np.ndarray, lp: np.ndarray, n_seq: int, vocab: int):
    """oracle_pack -> (status, dict of numpy arrays)."""
    n = len(ids)
    m = max(n, 1)
    out = {
        "tokens": np.zeros(m, np.int32), "loss_mask": np.zeros(m, np.uint8), "turn_id": np.zeros(m, np.int16),
        "seq_id": np.zeros(m, np.int32), "pos_id": np.zeros(m, np.int32), "cu_seqlens": np.zeros(n_seq + 1, np.int32),
        "old_lp": np.zeros(m, np.float32), "act_row": np.zeros(m, np.int32), "act_target": np.zeros(m, np.int32),
        "act_old_lp": np.zeros(m, np.float32), "act_seq": np.zeros(m, np.int32), "act_turn": np.zeros(m, np.int16),
    }
    pk = OraclePacked(*[_p(out[f]) for f, _ in OraclePacked._fields_[:-1]], 0)
    st = lib().oracle_pack(_p(turns), len(turns), _p(ids), _p(lp), n, n_seq, vocab, C.byref(pk))
    a = pk.n_active
    for k in ("tokens", "loss_mask", "turn_id", "seq_id", "pos_id", "old_lp"):
        out[k] = out[k][:n]
    for k in ("act_row", "act_target", "act_old_lp", "act_seq", "act_turn"):
        out[k] = out[k][:a]
    out["n_active"] = a
    return st, out


def grpo(reward, usable, group_off, ddof=1, eps=1e-6, tol=0.0):
    R, G = len(reward), len(group_off) - 1
    adv = np.zeros(max(R, 1), np.float64)
    info = np.zeros(max(G, 1), np.uint8)
    asum, nr = C.c_double(), C.c_double()
    lib().oracle_grpo(_p(np.ascontiguousarray(reward, np.float64)), _p(np.ascontiguousarray(usable, np.uint8)),
                      _p(np.ascontiguousarray(group_off, np.int32)), G, ddof, eps, tol, _p(adv), _p(info),
                      C.byref(asum), C.byref(nr))
    return adv[:R], info[:G], asum.value, nr.value


def gen_logits(n_rows, vocab, row_key0=0, targets=None, old_lp=None, seed=0, sigma=2.0, dtype="bf16",
               row_stride=None):
    stride = row_stride or vocab
    arr = np.zeros((n_rows, stride), np.uint16 if dtype == "bf16" else np.float32)
    lib().oracle_gen_logits(_p(arr), 0 if dtype == "bf16" else 1, stride, vocab, n_rows, row_key0,
                            _p(None if targets is None else np.ascontiguousarray(targets, np.int32)),
                            _p(None if old_lp is None else np.ascontiguousarray(old_lp, np.float32)), seed, sigma)
    return arr


def logprob_entropy(logits: np.ndarray, targets, rows=None, inv_temp=1.0, vocab=None):
    """logits: uint16 (bf16 bits) or float32 2-D array."""
    dtype = 0 if logits.dtype == np.uint16 else 1
    t = np.ascontiguousarray(targets, np.int32)
    n = len(t)
    lp, ent = np.zeros(n), np.zeros(n)
    r = None if rows is None else np.ascontiguousarray(rows, np.int32)
    lib().oracle_logprob_entropy(_p(logits), dtype, logits.shape[1], vocab or logits.shape[1], _p(r), _p(t), n,
                                 inv_temp, _p(lp), _p(ent))
    return lp, ent


def loss(logp, ent, old_lp, adv, row_seq, row_turn, eps_lo=0.2, eps_hi=0.28, n_buckets=64, ref_lp=None,
         kl_coef=0.0):
    P, Q = np.zeros(N_PARTIALS), np.zeros(N_PARTIALS)
    nb = C.c_int64(0)
    lib().oracle_loss(_p(np.ascontiguousarray(logp, np.float64)), _p(np.ascontiguousarray(ent, np.float64)),
                      _p(np.ascontiguousarray(old_lp, np.float32)), _p(np.ascontiguousarray(adv, np.float64)),
                      _p(np.ascontiguousarray(row_seq, np.int32)), _p(np.ascontiguousarray(row_turn, np.int16)),
                      _p(None if ref_lp is None else np.ascontiguousarray(ref_lp, np.float32)),
                      len(logp), eps_lo, eps_hi, kl_coef, n_buckets, _p(P), _p(Q), C.byref(nb))
    return P, Q, nb.value


def logits_grad(logits: np.ndarray, targets, old_lp, adv, row_seq, n_global, rows=None, inv_temp=1.0, eps_lo=0.2,
                eps_hi=0.28, vocab=None, ref_lp=None, kl_coef=0.0):
    """Oracle dL/dlogits (fp64) [n_rows x V], dL/dlogp [n_rows], border flags [n_rows]."""
    dtype = 0 if logits.dtype == np.uint16 else 1
    V = vocab or logits.shape[1]
    t = np.ascontiguousarray(targets, np.int32)
    n = len(t)
    g = np.zeros((n, V))
    dl = np.zeros(n)
    bd = np.zeros(n, np.uint8)
    r = None if rows is None else np.ascontiguousarray(rows, np.int32)
    lib().oracle_logits_grad(_p(logits), dtype, logits.shape[1], V, _p(r), _p(t),
                             _p(np.ascontiguousarray(old_lp, np.float32)), _p(np.ascontiguousarray(adv, np.float64)),
                             _p(np.ascontiguousarray(row_seq, np.int32)),
                             _p(None if ref_lp is None else np.ascontiguousarray(ref_lp, np.float32)), n, inv_temp,
                             eps_lo, eps_hi, kl_coef, n_global, _p(g), _p(dl), _p(bd))
    return g, dl, bd


def score_batch(hb_c, cfg_c, seed: int, sigma: float, nthreads: int = 1, row_begin: int = -1, row_end: int = -1,
                want_rows: bool = False, n_active_hint: int = 0):
    """Full CPU path (oracle_score_batch). hb_c / cfg_c: the ctypes structs of
    the product's C-ABI (prorl_host_batch / prorl_score_cfg) — same layout."""
    P, Q = np.zeros(N_PARTIALS), np.zeros(N_PARTIALS)
    nb, na = C.c_int64(0), C.c_int64(0)
    tm = np.zeros(3)
    lp = np.zeros(max(n_active_hint, 1)) if want_rows else None
    ent = np.zeros(max(n_active_hint, 1)) if want_rows else None
    st = lib().oracle_score_batch(C.addressof(hb_c), C.addressof(cfg_c), seed, sigma, nthreads, row_begin, row_end,
                                  _p(P), _p(Q), C.byref(nb), _p(lp), _p(ent), C.byref(na), _p(tm))
    return {"status": st, "partials": P, "abs": Q, "n_border": nb.value, "n_active": na.value, "timings": tm,
            "logp": lp, "entropy": ent}


def score_sample(hb_c, cfg_c, seed: int, sigma: float, nthreads: int, stride: int, offset: int = 0,
                 max_rows: int = -1):
    """Whole-step CPU path on the systematic sample of active rows offset, offset + stride, ...
    (oracle_score_sample). timings: [pack+GRPO wall s, scoring wall s, generation wall s]."""
    P, Q = np.zeros(N_PARTIALS), np.zeros(N_PARTIALS)
    nb, ns, na = C.c_int64(0), C.c_int64(0), C.c_int64(0)
    tm = np.zeros(3)
    st = lib().oracle_score_sample(C.addressof(hb_c), C.addressof(cfg_c), seed, sigma, nthreads, stride, offset,
                                   max_rows, _p(P), _p(Q), C.byref(nb), C.byref(ns), C.byref(na), _p(tm))
    return {"status": st, "partials": P, "abs": Q, "n_border": nb.value, "n_scored": ns.value, "n_active": na.value,
            "timings": tm}


def cpu_model() -> str:
    """The host CPU's model name (/proc/cpuinfo), for the baseline's record."""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
