"""Build libspeedrec.so in-tree with nvcc for sm_100a (no JIT cache).

Every `csrc/*.cu` is one translation unit, compiled in parallel (the
unrolled k_mask_fit<D> instantiations live in their own units), then linked
into one shared library.
"""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspeedrec.so")
OBJ_DIR = os.path.join(_HERE, "_obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def _run(cmd):
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + res.stderr)
    return res.stderr


def build_library(force: bool = False, verbose: bool = False, extra_flags=None, out: str | None = None) -> str:
    """Compile csrc/*.cu for sm_100a and link `out` (default LIB_PATH).
    extra_flags: additional nvcc flags (A/B variants, tools/ab_variants.sh)."""
    out = out or LIB_PATH
    srcs = sorted(glob.glob(os.path.join(_HERE, "csrc", "*")))
    units = [p for p in srcs if p.endswith(".cu")]
    hdr = os.path.join(os.path.dirname(_HERE), "include", "speedrec.h")
    newest = max(os.path.getmtime(p) for p in srcs + [hdr])
    if not force and not extra_flags and os.path.exists(out) and os.path.getmtime(out) >= newest:
        return out
    tag = "" if not extra_flags else "_" + str(abs(hash(tuple(extra_flags))))
    os.makedirs(OBJ_DIR, exist_ok=True)
    objs = [os.path.join(OBJ_DIR, os.path.basename(u)[:-3] + tag + ".o") for u in units]
    cmds = [[NVCC] + FLAGS + list(extra_flags or []) + ["-c", "-o", o, u] for u, o in zip(units, objs)]
    with ThreadPoolExecutor(max(1, min(len(cmds), os.cpu_count() or 1))) as pool:
        logs = list(pool.map(_run, cmds))
    logs.append(_run([NVCC] + ARCH + ["-shared", "-o", out] + objs))
    if verbose:
        print("\n".join(logs))
    return out
