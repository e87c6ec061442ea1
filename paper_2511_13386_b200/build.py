"""Build libpk.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels
with the repo snapshot to the GPU box)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = ["pk_api.cu", "pk_fine.cu", "pk_fluid.cu"]
OUT = os.path.join(HERE, "libpk.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--threads", "0",
    # exact IEEE double arithmetic in numpy's operation order: no contraction
    "--fmad=false",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
]


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))]
    deps.append(os.path.join(HERE, "..", "include", "pk.h"))
    return any(os.path.getmtime(d) > t for d in deps)


FINE_PARTS = 9  # pk_fine.cu compiles once per PK_FINE_PART (one fine_kernel layout each)


def build(force: bool = False, verbose: bool = False, extra=(), jobs: int | None = None) -> str:
    """Compile the translation units in parallel (pk_fine.cu split by
    PK_FINE_PART, ptxas time dominates) into _obj/ and link libpk.so."""
    if not force and not needs_build():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    obj_dir = os.path.join(HERE, "_obj")
    os.makedirs(obj_dir, exist_ok=True)
    flags = [f for f in NVCC_FLAGS if f not in ("-shared",)]
    units = [("pk_api.cu", None), ("pk_fluid.cu", None)] + [("pk_fine.cu", k) for k in range(FINE_PARTS)]
    # the heavy layouts first
    units.sort(key=lambda u: 0 if u[1] is not None else 1)
    jobs = jobs or max(1, min(len(units), os.cpu_count() or 1))
    cmds, objs = [], []
    for src, part in units:
        obj = os.path.join(obj_dir, src[:-3] + (f"_{part}" if part is not None else "") + ".o")
        cmd = [nvcc, *flags, *extra, "-c", "-o", obj, os.path.join(HERE, "csrc", src)]
        if part is not None:
            cmd.insert(1, f"-DPK_FINE_PART={part}")
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        cmds.append(cmd)
        objs.append(obj)
    running, todo, failed = [], list(cmds), None
    while (todo or running) and failed is None:
        while todo and len(running) < jobs:
            c = todo.pop(0)
            if verbose:
                print(" ".join(c), file=sys.stderr)
            running.append((c, subprocess.Popen(c, cwd=os.path.join(HERE, "csrc"))))
        c, pr = running.pop(0)
        if pr.wait() != 0:
            failed = c
    for _, pr in running:
        pr.wait()
    if failed is not None:
        raise subprocess.CalledProcessError(1, failed)
    link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
            "-Xcompiler", "-fPIC", "-o", OUT, *objs]
    subprocess.run(link, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
