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
SOURCES = ["gx_table.cu", "gx_explore.cu", "gx_micro.cu", "gx_shard.cu"]
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


def build(force: bool = False, verbose: bool = False, out: Path = OUT, defines=()) -> Path:
    """Compile and link libgx.so (defines: extra -D flags for a variant build
    written to `out`, used by the A/B sweep scripts)."""
    if not force and out == OUT and not stale():
        return OUT
    objdir = HERE / "build" / (out.stem if out != OUT else "")
    objdir.mkdir(parents=True, exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        log = objdir / (Path(src).stem + ".ptxas.log")
        cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", str(CSRC / src), "-o", str(obj)]
        procs.append((cmd, obj, log, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                      stderr=subprocess.STDOUT)))
    objs = []
    for cmd, obj, log, p in procs:
        txt, _ = p.communicate()
        log.write_bytes(txt)
        if p.returncode != 0:
            sys.stderr.write(txt.decode(errors="replace")[-8000:])
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
        if verbose:
            sys.stdout.write(txt.decode(errors="replace"))
        objs.append(str(obj))
    tmp = out.with_suffix(".so.tmp")
    subprocess.run([nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs,
                    "-o", str(tmp)], check=True)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    # python build.py [--force] [-v] [--out PATH -DNAME=VALUE ...]
    argv = sys.argv[1:]
    out = Path(argv[argv.index("--out") + 1]) if "--out" in argv else OUT
    defs = [a[2:] for a in argv if a.startswith("-D")]
    print(build(force="--force" in argv or out != OUT, verbose="-v" in argv, out=out, defines=defs))
