"""Build ``_lib/libmeshchroma_b200.so`` in-tree with nvcc for sm_100a.

Every source under ``csrc/`` (CUDA kernels, the C-ABI, the host C++
coloring) goes into one shared library with a static CUDA runtime, so the
library loads through ctypes next to torch's own runtime without version
coupling.  The built file is git-ignored but travels to the GPU box with
the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB_NAME = "libmeshchroma_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"),
                 "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; cannot build the sm_100a extension")


def sources():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_native(force: bool = False, verbose: bool = False) -> Path:
    OUT_DIR.mkdir(exist_ok=True)
    target = OUT_DIR / LIB_NAME
    deps = sources() + list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) \
        + list((PKG.parent / "include").glob("*.h"))
    if not force and not _stale(target, deps):
        return target
    nvcc = _nvcc()
    objs = []
    jobs = []
    for src in sources():
        obj = OUT_DIR / (src.name + ".o")
        cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17",
               "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v" if verbose else "-O3",
               "-I", str(PKG.parent / "include"), "-c", str(src), "-o", str(obj)]
        if src.suffix == ".cu":
            cmd[5:5] = ["--expt-relaxed-constexpr"]
        cmd[5:5] = [f"-D{d}" for d in os.environ.get("MC_DEFINES", "").split() if d]
        jobs.append((src, cmd))
        objs.append(obj)
    procs = [(src, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                    stderr=subprocess.STDOUT, text=True))
             for src, cmd in jobs]
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append(f"--- {src.name}\n{out}")
        elif verbose and out:
            sys.stderr.write(out)
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(failed))
    tmp = target.with_suffix(".so.tmp")
    link = [nvcc, *ARCH, "-shared", "-cudart=static", "-o", str(tmp),
            *map(str, objs), "-lpthread", "-ldl", "-lrt"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    os.replace(tmp, target)
    for o in objs:
        o.unlink(missing_ok=True)
    return target


if __name__ == "__main__":
    print(build_native(force="--force" in sys.argv, verbose="-v" in sys.argv))
