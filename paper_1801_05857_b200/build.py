"""Build libgx.so in-tree for sm_100a (nvcc, one process per translation
unit, then one shared-library link)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
OUT = HERE / "libgx.so"
SOURCES = ["gx_table.cu", "gx_explore.cu"]
NVCC_FLAGS = ["-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v", f"-I{HERE.parent / 'include'}"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    return "nvcc"


def stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = list(CSRC.glob("*")) + [HERE.parent / "include" / "gx.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return OUT
    objdir = HERE / "build"
    objdir.mkdir(exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        log = objdir / (Path(src).stem + ".ptxas.log")
        cmd = [nvcc(), *NVCC_FLAGS, "-c", str(CSRC / src), "-o", str(obj)]
        procs.append((cmd, obj, log, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                      stderr=subprocess.STDOUT)))
    objs = []
    for cmd, obj, log, p in procs:
        out, _ = p.communicate()
        log.write_bytes(out)
        if p.returncode != 0:
            sys.stderr.write(out.decode(errors="replace")[-8000:])
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
        if verbose:
            sys.stdout.write(out.decode(errors="replace"))
        objs.append(str(obj))
    tmp = OUT.with_suffix(".so.tmp")
    subprocess.run([nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs,
                    "-o", str(tmp)], check=True)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
