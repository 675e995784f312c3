"""Build the sm_100a C-ABI library in-tree (nvcc cross-compiles without a GPU).

    python -m paper_2509_25401_b200.build
"""

import pathlib
import subprocess
import sys

HERE = pathlib.Path(__file__).resolve().parent
SOURCES = ["fo_symbols.cu", "fo_attention.cu", "fo_attention_cs.cu", "fo_gemm.cu",
           "fo_elementwise.cu", "fo_policy.cu", "fo_capi.cu"]
OUT = HERE / "_fo_b200.so"
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-shared",
]


def needs_build():
    if not OUT.exists():
        return True
    mtime = OUT.stat().st_mtime
    deps = [HERE / "csrc" / s for s in SOURCES] + list((HERE / "csrc").glob("*.cuh"))
    deps.append(HERE.parent / "include" / "flashomni_b200.h")
    return any(d.stat().st_mtime > mtime for d in deps)


def build(force=False, verbose=False):
    if not force and not needs_build():
        return OUT
    cmd = ["nvcc", *NVCC_FLAGS, "-o", str(OUT), *[str(HERE / "csrc" / s) for s in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
