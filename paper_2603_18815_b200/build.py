"""Build the sm_100a hot-path library in-tree.

    python -m paper_2603_18815_b200.build          # -> paper_2603_18815_b200/libprorl_hotpath.so

nvcc cross-compiles for sm_100a without a GPU, so this runs in the CPU
container too. Objects go to build/, the shared object next to this file so
it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = ROOT / "build" / "hotpath"
LIB = PKG / "libprorl_hotpath.so"

SOURCES = ["pack.cu", "grpo.cu", "score.cu", "grad.cu", "train.cu", "lmhead.cu", "synth.cu", "capi.cu", "workload.cpp", "ingest.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
              "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}"]


def json_include() -> str:
    """Directory holding nlohmann json.hpp (the reference's only third-party
    header, also used by the drop-in C++ headers). This image ships 3.11.3
    inside the venv's cudnn_frontend tree."""
    import glob
    import site
    env = os.environ.get("PRORL_JSON_DIR")
    if env and (Path(env) / "json.hpp").exists():
        return env
    for sp in site.getsitepackages() + [site.getusersitepackages(), sys.prefix]:
        for cand in glob.glob(os.path.join(sp, "**", "nlohmann", "json.hpp"), recursive=True):
            return str(Path(cand).parent)
    raise RuntimeError("nlohmann/json.hpp not found (set PRORL_JSON_DIR)")


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the sm_100a hot-path library cannot be built")


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h")) + list(INCLUDE.glob("rollout/**/*.hpp"))
    objs = []
    jobs = []
    for src in SOURCES:
        s = CSRC / src
        o = BUILD / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append((s, o))

    def compile_one(job):
        s, o = job
        if s.suffix == ".cpp":  # host-only C++: the host compiler directly, full optimisation
            cmd = [os.environ.get("CXX", "g++"), "-O3", "-std=c++17", "-fPIC", "-Wall", f"-I{INCLUDE}",
                   f"-I{CSRC}", f"-I{json_include()}", "-I/usr/local/cuda/include", "-c", str(s), "-o", str(o)]
        else:
            cmd = [nvcc(), *ARCH, *NVCC_FLAGS, f"-I{json_include()}", "-c", str(s), "-o", str(o)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed for {s.name}:\n{r.stderr}")
        if verbose:
            (BUILD / (s.stem + ".ptxas.txt")).write_text(r.stderr)

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        list(ex.map(compile_one, jobs))
    if force or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    p = build(verbose=True, force="--force" in sys.argv)
    print(p)
