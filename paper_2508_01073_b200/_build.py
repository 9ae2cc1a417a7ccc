"""Build the sm_100a shared library libwalkvec_b200.so in-tree with nvcc."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libwalkvec_b200.so"
SOURCES = ["abi.cu", "csr.cu", "walks.cu", "bfs.cu", "sgns.cu", "replica.cu", "synth.cu", "ingest.cu", "formats.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def needs_build() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "walkvec_b200.h"]
    return any(p.stat().st_mtime > mtime for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False, out: Path | None = None, defines=()) -> Path:
    """Compile the library (``out``/``defines``: A/B variants, loaded with WV_LIB=path)."""
    lib = Path(out) if out else LIB
    if not force and out is None and not needs_build():
        return LIB
    # one nvcc per translation unit in parallel (sgns.cu dominates), then one link
    objdir = ROOT / "build" / (lib.stem + "_obj")
    objdir.mkdir(parents=True, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]
    procs = []
    for s in SOURCES:
        cmd = [_nvcc(), *compile_flags, *[f"-D{d}" for d in defines], "-I", str(ROOT / "include"), "-c",
               "-o", str(objdir / (s + ".o")), str(CSRC / s)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        procs.append((s, subprocess.Popen(cmd)))
    failed = [s for s, p in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, f"nvcc {' '.join(failed)}")
    link = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(lib) + ".tmp"]
    link += [str(objdir / (s + ".o")) for s in SOURCES]
    subprocess.run(link, check=True)
    os.replace(str(lib) + ".tmp", lib)
    shutil.rmtree(objdir, ignore_errors=True)  # ~70 MB per variant; the repo snapshot travels to the GPU box
    return lib


if __name__ == "__main__":
    # python _build.py [-v] [--out path -DNAME=VAL ...]
    argv = sys.argv[1:]
    out = argv[argv.index("--out") + 1] if "--out" in argv else None
    defs = [a[2:] for a in argv if a.startswith("-D")]
    print(build(force=True, verbose="-v" in argv, out=out, defines=defs))
