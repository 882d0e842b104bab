"""The drop-in boundary against the UNMODIFIED reference: tests/cpp/test_reference_seam.cpp
is compiled with the reference's own include root (-I/root/reference/proj/include
-Iinclude: every rollout:: type is the reference's, only the façade headers come
from this repo) and linked against the reference's handlers.cpp / harness.cpp /
mock policy (oracle/_ref/libref.so, compiled in place by oracle/build_ref.sh)
plus libprorl_hotpath.so. It runs build_process_response -> wire JSON ->
record_response -> build_host_batch; here the batch is checked against the
reference's own flatten() and the oracle's packing, and (GPU leg)
DeviceScorer::score_groups / train_groups against the oracle.

The binary is built where /root/reference exists (this container) and the
prebuilt one travels to the GPU box with the snapshot (build/ is git-ignored,
not gpurun-ignored).
"""
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
REF_INCLUDE = Path("/root/reference/proj/include")
BIN = ROOT / "build" / "test_reference_seam"
SRC = ROOT / "tests" / "cpp" / "test_reference_seam.cpp"


def build_seam() -> Path:
    """Compile the seam test against the reference headers (needs /root/reference)."""
    BIN.parent.mkdir(parents=True, exist_ok=True)
    deps = [SRC, B.LIB, O.REF_SO, *(ROOT / "include").rglob("*.h*")]
    if BIN.exists() and BIN.stat().st_mtime >= max(d.stat().st_mtime for d in deps):
        return BIN
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", f"-I{REF_INCLUDE}", f"-I{ROOT / 'include'}", f"-I{B.json_include()}",
           "-I/usr/local/cuda/include", str(SRC), "-o", str(BIN), f"-L{O.REF_SO.parent}", "-lref",
           f"-Wl,-rpath,{O.REF_SO.parent}", f"-L{B.PKG}", "-lprorl_hotpath", f"-Wl,-rpath,{B.PKG}",
           "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)
    return BIN


@pytest.fixture(scope="module")
def seam():
    if REF_INCLUDE.is_dir():
        assert O.REF_SO.exists(), "oracle/_ref/libref.so missing (conftest builds it when /root/reference exists)"
        return build_seam()
    if not BIN.exists():
        pytest.skip("no /root/reference here and no prebuilt build/test_reference_seam in the snapshot")
    return BIN


def _run(binary, *args):
    r = subprocess.run([str(binary), *args], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return json.loads(r.stdout.strip().splitlines()[-1])


def _host_batch(d):
    t = np.zeros(len(d["turns"]), N.TURN_DTYPE)
    arr = np.array(d["turns"], np.int64).reshape(-1, 4)
    t["src_off"], t["traj"], t["len"], t["role"] = arr[:, 0], arr[:, 1], arr[:, 2], arr[:, 3]
    return (t, np.array(d["ids"], np.int64), np.array(d["lp"], np.float64), np.array(d["reward"], np.float64),
            np.array(d["usable"], np.uint8), np.array(d["group_off"], np.int32))


def test_seam_host_batch_matches_reference_flatten_and_oracle(seam):
    d = _run(seam)
    t, ids, lp, reward, usable, goff = _host_batch(d)
    assert d["prompt_ids"] == sorted(d["prompt_ids"])        # App. B.1 group order
    exp = d["expect"]
    assert len(exp) == len(reward)
    # the batch's token stream is the reference's TokenTrajectory::flatten() of
    # every participating rollout, in (prompt_id, slot) order
    want_ids = [i for e in exp if e for i in e["flatten"]]
    assert ids.tolist() == want_ids
    st, pk = O.pack(t, ids, lp, len(reward), 4099)
    assert st == 0
    want_mask = [m for e in exp if e for m in e["mask"]]
    assert pk["loss_mask"].tolist() == want_mask             # role -> mask rule (trajectory.hpp:82-83)
    lens = [len(e["flatten"]) if e else 0 for e in exp]
    assert pk["cu_seqlens"].tolist() == np.concatenate([[0], np.cumsum(lens)]).tolist()
    assert pk["n_active"] == d["n_active"]
    # behaviour logprobs are the reference mock policy's token_logprob of each id (policy.cpp:51-53)
    a = pk["loss_mask"].astype(bool)
    assert np.array_equal(lp[a], -(1.0 + (ids[a] % 7) / 10.0))
    # FAILED rollouts and the non-informative group are in the batch with empty sequences
    assert usable.sum() == len(usable) - 1
    assert sum(1 for e in exp if e is None) >= 5


@pytest.mark.gpu
def test_seam_score_and_train_groups_vs_oracle(seam):
    d = _run(seam, "--gpu")
    t, ids, lp, reward, usable, goff = _host_batch(d)
    hb = O.host_batch(t, ids, lp, reward, usable, goff)     # keys = slot index, as SyntheticLogits
    ref = O.score_batch(hb, O.score_cfg(4099, "bf16", microbatch_rows=48), 77, 2.0, nthreads=4)
    assert ref["status"] == 0 and ref["n_active"] == d["n_active"]
    assert_partials_close(d["partials"], ref["partials"], ref["abs"], ref["n_border"], "seam score_groups")
    assert_partials_close(d["train_partials"], ref["partials"], ref["abs"], ref["n_border"], "seam train_groups")
    assert d["grad_rows"] == d["n_active"]


def test_reference_patch_applies_and_compiles(tmp_path):
    """integration/reference.patch (TrainerOptions::on_response, the 3-line hook
    at harness.cpp:273) applies to the unmodified reference, and the patched
    trainer/harness.cpp compiles together with a trainer TU that wires the hook
    to the façade's keep_trajectory."""
    if not REF_INCLUDE.is_dir():
        pytest.skip("no /root/reference here")
    import shutil
    ref = REF_INCLUDE.parent
    work = tmp_path / "proj"
    for rel in ("include/rollout/trainer/harness.hpp", "src/trainer/harness.cpp"):
        (work / rel).parent.mkdir(parents=True, exist_ok=True)
        shutil.copy(ref / rel, work / rel)
    subprocess.run(["patch", "-p1", "-d", str(tmp_path), "-i", str(ROOT / "integration" / "reference.patch")],
                   check=True, capture_output=True)
    inc = [f"-I{work / 'include'}", f"-I{REF_INCLUDE}", f"-I{ROOT / 'include'}", f"-I{B.json_include()}"]
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", *inc, str(work / "src/trainer/harness.cpp")], check=True)
    tu = tmp_path / "trainer.cpp"
    tu.write_text('''
#include "rollout/trainer/harness.hpp"
#include "rollout/trainer/scoring.hpp"
using namespace rollout::train;
void wire(TrainerOptions& opts, TrajectoryTable& table) {
  opts.on_response = [&table](const PromptGroup& g, int slot, const nlohmann::json& r) {
    keep_trajectory(table, g, slot, r);
  };
}
''')
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", *inc, str(tu)], check=True)
