"""The C++ drop-in surface (include/rollout/..., rollout::train::score_groups):
build tests/cpp/test_scoring.cpp against the in-tree library and run it.
Host checks run without a GPU; the --gpu leg is checked against the oracle."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_18815_b200 import _native as N
from paper_2603_18815_b200 import build as B
from tests.parity import assert_partials_close

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "build" / "test_scoring"


@pytest.fixture(scope="module")
def binary():
    assert B.LIB.exists(), "libprorl_hotpath.so missing (conftest builds it on first use)"
    BIN.parent.mkdir(parents=True, exist_ok=True)
    src = ROOT / "tests" / "cpp" / "test_scoring.cpp"
    if not BIN.exists() or BIN.stat().st_mtime < max(src.stat().st_mtime, B.LIB.stat().st_mtime):
        cmd = ["g++", "-std=c++17", "-O2", "-Wall", f"-I{ROOT / 'include'}", f"-I{ROOT / 'include' / 'standalone'}",
               f"-I{B.json_include()}",
               "-I/usr/local/cuda/include", str(src), "-o", str(BIN), f"-L{B.PKG}", "-lprorl_hotpath",
               f"-Wl,-rpath,{B.PKG}", "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"]
        subprocess.run(cmd, check=True)
    return BIN


def test_cpp_host_checks(binary):
    r = subprocess.run([str(binary)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "host checks OK" in r.stdout


@pytest.mark.gpu
def test_cpp_score_groups_vs_oracle(binary):
    r = subprocess.run([str(binary), "--gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    t = np.zeros(len(d["turns"]), N.TURN_DTYPE)
    arr = np.array(d["turns"], np.int64)
    t["src_off"], t["traj"], t["len"], t["role"] = arr[:, 0], arr[:, 1], arr[:, 2], arr[:, 3]
    ids = np.array(d["ids"], np.int64)
    lp = np.array(d["lp"], np.float64)
    reward = np.array(d["reward"], np.float64)
    usable = np.array(d["usable"], np.uint8)
    goff = np.array(d["group_off"], np.int32)
    hb = O.host_batch(t, ids, lp, reward, usable, goff)
    ref = O.score_batch(hb, O.score_cfg(4099, "bf16", microbatch_rows=64), 4242, 2.0, nthreads=4)
    assert ref["status"] == 0 and ref["n_active"] == d["n_active_host"] == d["n_active"]
    got = np.array(d["partials"])
    P, Q = ref["partials"], ref["abs"]
    assert_partials_close(got, P, Q, ref["n_border"], "score_groups")
    # DeviceScorer::train_groups: same partials (K7), one gradient hand-off per
    # micro-batch, gradient rows finite and summing to ~0 (sum_v (1[v=y] - p_v) = 0)
    tp = np.array(d["train_partials"])
    assert_partials_close(tp, P, Q, ref["n_border"], "train_groups")
    n, mb = d["n_active"], 64
    assert d["grad_batches"] == [[r0, min(mb, n - r0)] for r0 in range(0, n, mb)]
    assert d["grad_finite"] == 1 and d["grad_nonzero_rows"] > 0
    assert d["grad_max_row_sum_rel"] <= 4099 * 2.0 ** -8


@pytest.mark.gpu
def test_cpp_score_responses_tool_vs_oracle(tmp_path):
    """tools/score_responses: wire JSON -> IngestedBatch -> DeviceScorer, all in C++."""
    from paper_2603_18815_b200 import synth
    from tests.wire import to_responses
    assert B.LIB.exists()
    exe = ROOT / "build" / "score_responses"
    src = ROOT / "tools" / "score_responses.cpp"
    if not exe.exists() or exe.stat().st_mtime < max(src.stat().st_mtime, B.LIB.stat().st_mtime):
        subprocess.run(["g++", "-std=c++17", "-O2", f"-I{ROOT / 'include'}", f"-I{ROOT / 'include' / 'standalone'}",
                        f"-I{B.json_include()}", "-I/usr/local/cuda/include", str(src), "-o", str(exe),
                        f"-L{B.PKG}", "-lprorl_hotpath", f"-Wl,-rpath,{B.PKG}", "-L/usr/local/cuda/lib64", "-lcudart",
                        "-Wl,-rpath,/usr/local/cuda/lib64"], check=True)
    sh = synth.make_shard("c1", seed=99)
    b = sh.batch
    assert all(b.group_off[1:] - b.group_off[:-1] == 4)
    path = tmp_path / "responses.jsonl"
    path.write_bytes(b"\n".join(to_responses(b)) + b"\n")
    r = subprocess.run([str(exe), str(path), "4", "32000", "fp32", "21"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["n_active"] == sh.n_active
    hb = O.host_batch(b.turns, b.ids, b.lp, b.reward, b.usable, b.group_off)  # keys = slot index, as the tool
    ref = O.score_batch(hb, O.score_cfg(32000, "fp32", microbatch_rows=4096), 21, 2.0, nthreads=4)
    got = np.array(d["partials"])
    P, Q = ref["partials"], ref["abs"]
    assert_partials_close(got, P, Q, ref["n_border"], "score_responses")
    assert d["grad_batches"] == 0
    # --train: the K7 training step through the facade, same metrics, one gradient hand-off per micro-batch
    r = subprocess.run([str(exe), str(path), "4", "32000", "fp32", "21", "--train"], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert_partials_close(np.array(d["partials"]), P, Q, ref["n_border"], "score_responses --train")
    assert d["grad_rows"] == sh.n_active and d["grad_batches"] == -(-sh.n_active // 4096)
