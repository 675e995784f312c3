"""SASS instruction census of the built library (no GPU needed).

    python tools/sass_census.py [out.json]

Per kernel (demangled name), counts of the Blackwell-native instructions that
prove the tcgen05 / TMEM / TMA data path: UTCHMMA (tcgen05.mma, .2CTA =
cta_group::2), UTCBAR (tcgen05.commit), LDTM / STTM (tcgen05.ld / st),
UTMALDG / UTMASTG / UTMAPF (TMA load / store / L2 prefetch, .MULTICAST / .2CTA
variants), plus legacy HMMA (mma.sync) which must be absent from the hot
kernels. Static counts: instructions in the binary, not executions.
"""

import collections
import json
import pathlib
import re
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2509_25401_b200" / "_fo_b200.so"
OPS = re.compile(r"\b(UTCHMMA[A-Z0-9_.]*|UTCQMMA[A-Z0-9_.]*|UTCBAR[A-Z0-9_.]*|LDTM[A-Z0-9_.]*|"
                 r"STTM[A-Z0-9_.]*|UTMALDG[A-Z0-9_.]*|UTMASTG[A-Z0-9_.]*|UTMAPF[A-Z0-9_.]*|"
                 r"HMMA[A-Z0-9_.]*|UBLKCP[A-Z0-9_.]*|STG\.E\.ENL2\.256|STG\.E\.256)")


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()


def census(lib=LIB):
    sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True,
                          check=True).stdout
    per = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        if "Function :" in line:
            cur = line.split("Function :")[1].strip()
            per[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        for m in OPS.findall(line):
            # strip operand-specific suffixes that are not variants (e.g. LDTM.x32)
            per[cur][m.rstrip(".")] += 1
    names = list(per)
    pretty = demangle(names)
    return {p.replace("(anonymous namespace)", "anon").split("(")[0]: dict(sorted(per[n].items())) for n, p in zip(names, pretty)}


if __name__ == "__main__":
    res = {"library": str(LIB.relative_to(ROOT)), "arch": "sm_100a", "kernels": census()}
    text = json.dumps(res, indent=1)
    if len(sys.argv) > 1:
        pathlib.Path(sys.argv[1]).write_text(text + "\n")
    print(text)
