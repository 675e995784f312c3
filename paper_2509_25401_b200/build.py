"""Build the sm_100a C-ABI library in-tree (nvcc cross-compiles without a GPU).

    python -m paper_2509_25401_b200.build [--force] [-v]

Each translation unit compiles to its own object in parallel (objects are
rebuilt only when their source, a shared header or the flags change), then
one link produces _fo_b200.so.
"""

import concurrent.futures as cf
import hashlib
import os
import pathlib
import subprocess
import sys

HERE = pathlib.Path(__file__).resolve().parent
SOURCES = ["fo_symbols.cu", "fo_attention.cu", "fo_attention_cs.cu", "fo_gemm.cu",
           "fo_elementwise.cu", "fo_policy.cu", "fo_numerics.cu", "fo_capi.cu"]
OUT = HERE / "_fo_b200.so"
OBJ_DIR = HERE / "build"
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
]
EXTRA = os.environ.get("FO_NVCC_EXTRA", "").split()


def _deps():
    return list((HERE / "csrc").glob("*.cuh")) + [HERE.parent / "include" / "flashomni_b200.h"]


def _flags_tag():
    return hashlib.sha1(" ".join(NVCC_FLAGS + EXTRA).encode()).hexdigest()[:10]


def _obj(src):
    return OBJ_DIR / f"{pathlib.Path(src).stem}.{_flags_tag()}.o"


def _stale(target, deps):
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def needs_build():
    srcs = [HERE / "csrc" / s for s in SOURCES]
    return _stale(OUT, srcs + _deps())


def _compile(src, force, verbose):
    obj = _obj(src)
    path = HERE / "csrc" / src
    if not force and not _stale(obj, [path] + _deps()):
        return obj
    cmd = ["nvcc", *NVCC_FLAGS, *EXTRA, "-c", "-o", str(obj), str(path)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return obj


def build(force=False, verbose=False):
    if not force and not needs_build():
        return OUT
    OBJ_DIR.mkdir(exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose), SOURCES))
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(OUT),
           *[str(o) for o in objs]]
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
