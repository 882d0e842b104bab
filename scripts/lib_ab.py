"""A/B two builds of the library on the same box, alternating: K7 (prorl_score_grad)
and K2+K4 (prorl_score_rows) on one C2-sized micro-batch rotated over 3 buffers.
Works across ABI versions (advantages fp32 in ABI 1, fp64 from ABI 2).

    python scripts/lib_ab.py LIB_A LIB_B [--vocab 151936] [--rows 16576] [--rounds 4]
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs=2)
ap.add_argument("--vocab", type=int, default=151936)
ap.add_argument("--rows", type=int, default=16576)
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--kinds", default="k7,k2")
a = ap.parse_args()

vp = C.c_void_p


class LossCfg(C.Structure):
    _fields_ = [("eps_lo", C.c_float), ("eps_hi", C.c_float), ("n_buckets", C.c_int32), ("kl_coef", C.c_float)]


def load(path):
    L = C.CDLL(str(Path(path).resolve()))
    L.prorl_abi_version.restype = C.c_int
    L.prorl_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.prorl_gen_logits.argtypes = [vp, vp, C.c_int, C.c_int64, C.c_int32, C.c_int64, C.c_int64, vp, vp, C.c_uint64,
                                   C.c_float, vp]
    L.prorl_score_grad.argtypes = [vp, vp, C.c_int, C.c_int64, C.c_int32, vp, vp, vp, vp, vp, vp, vp, C.c_int64,
                                   C.c_float, C.POINTER(LossCfg), C.c_double, vp, vp, vp, vp, C.c_int64, vp, vp]
    L.prorl_score_rows.argtypes = [vp, vp, C.c_int, C.c_int64, C.c_int32, vp, vp, vp, vp, vp, vp, vp, C.c_int64,
                                   C.c_float, C.POINTER(LossCfg), vp, vp, vp, vp]
    ctx = vp()
    assert L.prorl_ctx_create(0, C.byref(ctx)) == 0
    return L, ctx


n, V = a.rows, a.vocab
libs = [load(p) for p in a.libs]
g = torch.Generator(device="cuda").manual_seed(7)
t = torch.randint(0, V, (n,), device="cuda", dtype=torch.int32, generator=g)
old = -0.05 - 2.9 * torch.rand(n, device="cuda", generator=g)
xs = [torch.empty((n, V), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
st = torch.cuda.current_stream().cuda_stream
L0, c0 = libs[0]
for x in xs:
    L0.prorl_gen_logits(c0, x.data_ptr(), 0, V, V, n, 0, t.data_ptr(), old.data_ptr(), 3, 2.0, st)
gout = torch.empty_like(xs[0])
adv64 = torch.randn(64, device="cuda", generator=g, dtype=torch.float64)
adv32 = adv64.float()
seq = torch.randint(0, 64, (n,), device="cuda", dtype=torch.int32, generator=g)
turn = torch.randint(0, 30, (n,), device="cuda", dtype=torch.int16, generator=g)
part = torch.zeros(332, dtype=torch.float64, device="cuda")
cfg = LossCfg(0.2, 0.28, 64, 0.0)


def run(lib, kind, k):
    L, ctx = lib
    adv = adv64 if L.prorl_abi_version() >= 2 else adv32
    x = xs[k % 3]
    if kind == "k7":
        r = L.prorl_score_grad(ctx, x.data_ptr(), 0, V, V, None, t.data_ptr(), old.data_ptr(), adv.data_ptr(),
                               seq.data_ptr(), turn.data_ptr(), None, n, 1.0, C.byref(cfg), float(n), None, None,
                               part.data_ptr(), gout.data_ptr(), V, None, st)
    else:
        r = L.prorl_score_rows(ctx, x.data_ptr(), 0, V, V, None, t.data_ptr(), old.data_ptr(), adv.data_ptr(),
                               seq.data_ptr(), turn.data_ptr(), None, n, 1.0, C.byref(cfg), None, None,
                               part.data_ptr(), st)
    assert r == 0


def timed(lib, kind):
    for k in range(2):
        run(lib, kind, k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(a.reps):
        run(lib, kind, k)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


for kind in a.kinds.split(","):
    res = {0: [], 1: []}
    for r in range(a.rounds):
        for i in (0, 1) if r % 2 == 0 else (1, 0):
            res[i].append(timed(libs[i], kind))
    print(f"V={V} {kind}: A {min(res[0]):.4f} ms (all {['%.4f' % v for v in res[0]]})  "
          f"B {min(res[1]):.4f} ms (all {['%.4f' % v for v in res[1]]})  B/A {min(res[1]) / min(res[0]):.4f}")
