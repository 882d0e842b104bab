"""ctypes binding of the C-ABI in include/prorl_hotpath.h.

The shared object is built in-tree (paper_2603_18815_b200/libprorl_hotpath.so,
see build.py). There is no fallback: if the library is missing or does not
load, importing this module raises — the product path is the sm_100a kernels
or nothing.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libprorl_hotpath.so"
if os.environ.get("PRORL_HOTPATH_LIB"):  # A/B of an experimental build (scripts/build_variant.sh); never a fallback
    LIB_PATH = Path(os.environ["PRORL_HOTPATH_LIB"]).resolve()

PRORL_BF16, PRORL_FP32 = 0, 1
# prorl_status (include/prorl_hotpath.h)
(PRORL_OK, PRORL_E_MALFORMED_TURN, PRORL_E_INCOMPLETE_GROUP, PRORL_E_MALFORMED_REQUEST) = (0, -1, -2, -3)
(PRORL_E_CUDA, PRORL_E_NCCL, PRORL_E_SHAPE, PRORL_E_TOKEN_RANGE, PRORL_E_PEER_FAILED) = (-10, -11, -12, -13, -14)
ROLE_SYSTEM, ROLE_USER, ROLE_ASSISTANT, ROLE_TOOL = 0, 1, 2, 3
TURN_BUCKETS, N_GLOBAL, N_PER_TURN = 64, 12, 5
N_PARTIALS = N_GLOBAL + TURN_BUCKETS * N_PER_TURN
(P_LOSS_SUM, P_N_ACTIVE, P_ENTROPY_SUM, P_LOGP_SUM, P_RATIO_SUM, P_CLIP_LO, P_CLIP_HI,
 P_KL1_SUM, P_ADV_SUM, P_N_ROLLOUTS, P_KL_SUM, P_ERR_RANKS) = range(12)

# Turn descriptor: must match prorl_turn_desc (24 bytes).
TURN_DTYPE = np.dtype([("src_off", "<i8"), ("traj", "<i4"), ("len", "<i4"), ("role", "u1"), ("pad", "u1", (7,))])
assert TURN_DTYPE.itemsize == 24

# Every symbol include/prorl_hotpath.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "prorl_abi_version", "prorl_kernel_config", "prorl_last_error", "prorl_status_code", "prorl_ctx_create", "prorl_ctx_destroy",
    "prorl_check_errors", "prorl_pack", "prorl_grpo_adv", "prorl_logprob_entropy", "prorl_clipped_loss",
    "prorl_score_rows", "prorl_nccl_unique_id", "prorl_nccl_init", "prorl_allreduce", "prorl_gen_logits",
    "prorl_gen_logits_keyed", "prorl_row_keys", "prorl_logits_grad", "prorl_score_grad", "prorl_lmhead_logprob", "prorl_ingest_responses", "prorl_ingest_free",
    "prorl_synth_rewards", "prorl_shard_lpt", "prorl_score_host", "prorl_fail_partials", "prorl_step_status",
    "prorl_last_step_info",
]

vp = C.c_void_p


class Packed(C.Structure):
    _fields_ = [(n, vp) for n in ("tokens", "loss_mask", "turn_id", "seq_id", "pos_id", "cu_seqlens", "old_lp",
                                  "act_row", "act_target", "act_old_lp", "act_seq", "act_turn", "n_active")]


class LossCfg(C.Structure):
    _fields_ = [("eps_lo", C.c_float), ("eps_hi", C.c_float), ("n_buckets", C.c_int32), ("kl_coef", C.c_float)]


class ScoreCfg(C.Structure):
    _fields_ = [("loss", LossCfg), ("inv_temperature", C.c_float), ("adv_eps", C.c_float), ("ddof", C.c_int32),
                ("vocab", C.c_int32), ("dtype", C.c_int32), ("microbatch_rows", C.c_int32),
                ("gate_tolerance", C.c_double)]


class HostBatch(C.Structure):
    _fields_ = [("turns", vp), ("n_turns", C.c_int64), ("ids", vp), ("lp", vp), ("n_tokens", C.c_int64),
                ("reward", vp), ("usable", vp), ("n_rollouts", C.c_int32), ("group_off", vp),
                ("n_groups", C.c_int32), ("rollout_key", vp)]


class StepInfo(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("micro_batches", C.c_int32), ("h2d_chunks", C.c_int32),
                ("h2d_bytes", C.c_int64)]


class IngestResult(C.Structure):
    _fields_ = [("batch", HostBatch), ("n_active", C.c_int64), ("n_informative", C.c_int32), ("pad_", C.c_int32),
                ("impl", vp)]


class LogitsPool(C.Structure):
    _fields_ = [("buffers", vp), ("n_pool", C.c_int32), ("fill", C.c_int32), ("row_stride", C.c_int64),
                ("seed", C.c_uint64), ("sigma", C.c_float), ("pad_", C.c_int32), ("provide", vp), ("user", vp),
                ("provide_hidden", vp), ("weight", vp), ("w_stride", C.c_int64), ("d_model", C.c_int32),
                ("pad2_", C.c_int32), ("train", C.c_int32), ("pad3_", C.c_int32), ("n_global", C.c_double),
                ("grad_buffers", vp), ("consume_grad", vp), ("grad_user", vp), ("provide_ref", vp), ("ref_user", vp)]

# prorl_ref_fn
REF_FN = C.CFUNCTYPE(C.c_int, vp, C.c_int64, C.c_int64, vp, vp, vp, vp, C.POINTER(vp), vp)

# prorl_grad_fn
GRAD_FN = C.CFUNCTYPE(C.c_int, vp, C.c_int64, C.c_int64, vp, C.c_int64, vp)

# prorl_hidden_fn
HIDDEN_FN = C.CFUNCTYPE(C.c_int, vp, C.c_int64, C.c_int64, vp, vp, vp, C.POINTER(vp), C.POINTER(C.c_int64), vp)


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a library first "
            "(python -m paper_2603_18815_b200.build or __graft_entry__.build()). There is no CPU fallback.")
    lib = C.CDLL(str(LIB_PATH))
    i32, i64, u64, f32, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double
    sig = {
        "prorl_abi_version": (C.c_int, []),
        "prorl_kernel_config": (C.c_char_p, []),
        "prorl_last_error": (C.c_char_p, []),
        "prorl_status_code": (C.c_char_p, [C.c_int]),
        "prorl_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
        "prorl_ctx_destroy": (C.c_int, [vp]),
        "prorl_check_errors": (C.c_int, [vp, vp]),
        "prorl_pack": (C.c_int, [vp, vp, i64, vp, vp, i64, i32, i32, C.POINTER(Packed), vp]),
        "prorl_grpo_adv": (C.c_int, [vp, vp, vp, vp, i32, i32, f32, f64, vp, vp, vp, vp]),
        "prorl_logprob_entropy": (C.c_int, [vp, vp, C.c_int, i64, i32, vp, vp, i64, f32, vp, vp, vp]),
        "prorl_clipped_loss": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, i64, C.POINTER(LossCfg), vp, vp]),
        "prorl_score_rows": (C.c_int, [vp, vp, C.c_int, i64, i32, vp, vp, vp, vp, vp, vp, vp, i64, f32,
                                       C.POINTER(LossCfg), vp, vp, vp, vp]),
        "prorl_logits_grad": (C.c_int, [vp, vp, C.c_int, i64, i32, vp, vp, vp, vp, vp, vp, vp, i64, f32,
                                        C.POINTER(LossCfg), f64, vp, i64, vp, vp]),
        "prorl_score_grad": (C.c_int, [vp, vp, C.c_int, i64, i32, vp, vp, vp, vp, vp, vp, vp, i64, f32,
                                       C.POINTER(LossCfg), f64, vp, vp, vp, vp, i64, vp, vp]),
        "prorl_ingest_responses": (C.c_int, [vp, vp, vp, i32, f64, i32, C.POINTER(IngestResult)]),
        "prorl_ingest_free": (C.c_int, [C.POINTER(IngestResult)]),
        "prorl_lmhead_logprob": (C.c_int, [vp, vp, i64, vp, i64, i32, i32, vp, i64, f32, vp, vp, vp]),
        "prorl_nccl_unique_id": (C.c_int, [vp]),
        "prorl_nccl_init": (C.c_int, [vp, C.c_int, C.c_int, vp]),
        "prorl_allreduce": (C.c_int, [vp, vp, C.c_int, vp]),
        "prorl_gen_logits": (C.c_int, [vp, vp, C.c_int, i64, i32, i64, i64, vp, vp, u64, f32, vp]),
        "prorl_gen_logits_keyed": (C.c_int, [vp, vp, C.c_int, i64, i32, i64, vp, vp, vp, u64, f32, vp]),
        "prorl_row_keys": (C.c_int, [vp, vp, vp, vp, vp, i64, vp, vp]),
        "prorl_synth_rewards": (C.c_int, [i32, i32, u64, f64, vp]),
        "prorl_shard_lpt": (C.c_int, [i32, vp, i32, vp]),
        "prorl_fail_partials": (None, [vp]),
        "prorl_step_status": (C.c_int, [C.c_int, vp]),
        "prorl_last_step_info": (C.c_int, [vp, C.POINTER(StepInfo)]),
        "prorl_score_host": (C.c_int, [vp, C.POINTER(HostBatch), C.POINTER(ScoreCfg), C.POINTER(LogitsPool), vp, vp,
                                       vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class RolloutError(RuntimeError):
    """Mirror of rollout::Error (errors.hpp:10-18): carries the stable code()."""

    def __init__(self, code: str, msg: str, status: int):
        super().__init__(msg)
        self.code = code
        self.status = status


def check(status: int) -> None:
    if status != 0:
        raise RolloutError(lib.prorl_status_code(status).decode(), lib.prorl_last_error().decode(), status)


def ptr(x) -> int | None:
    """Device/host address of a torch tensor or numpy array (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def loaded_library_path() -> str:
    return os.fspath(LIB_PATH)
