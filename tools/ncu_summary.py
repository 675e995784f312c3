"""Summarise ncu reports (run here, no GPU): key metrics per kernel -> JSON.

    python tools/ncu_summary.py out.json name=gpurun_out/x.ncu-rep [...] [--launches csv]
        [--current '{"config": "c4", "cached": 0.25, "skip": 0.5}']

--current also writes profiles/ncu_current.json: per kernel (short name) the
DRAM bytes per launch of these captures, which bench.py reports as
roofline.traffic when its workload matches.
"""

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
    "tensor_pipe_active_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "l2_to_sm_tma_bytes": "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "cluster": "launch__cluster_dim_x",
}
SCALE = {"dram_read_bytes": 1, "dram_write_bytes": 1, "l2_to_sm_tma_bytes": 1}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (u, v) for h, u, v in zip(hdr, units, vals)}, vals[hdr.index("Kernel Name")]


def to_base(unit, v):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3,
            "Ghz": 1, "cycle/nsecond": 1, "cycle/usecond": 1e-3}.get(unit, 1)
    return float(v.replace(",", "")) * mult


def main():
    out_path = sys.argv[1]
    res = {}
    launches = None
    args = sys.argv[2:]
    current = None
    if "--current" in args:
        k = args.index("--current")
        current = json.loads(args[k + 1])
        args = args[:k] + args[k + 2:]
    if "--launches" in args:
        k = args.index("--launches")
        launches = args[k + 1]
        args = args[:k] + args[k + 2:]
    for spec in args:
        name, rep = spec.split("=", 1)
        m, kname = raw(rep)
        d = {"kernel": kname[:120], "report": rep.split("/")[-1]}
        for key, met in METRICS.items():
            if met in m:
                unit, v = m[met]
                try:
                    d[key] = round(to_base(unit, v), 4)
                except ValueError:
                    d[key] = v
        res[name] = d
    if launches:
        agg = defaultdict(lambda: [0, 0.0])
        text = open(launches).read()
        text = text[text.index('"ID"'):] if '"ID"' in text else text
        for r in csv.DictReader(io.StringIO(text)):
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            kn = r["Kernel Name"].split("(")[0]
            mult = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
                    "msecond": 1e3}.get(r["Metric Unit"], 1)
            agg[kn][0] += 1
            agg[kn][1] += float(r["Metric Value"].replace(",", "")) * mult
        # shares among this engine's kernels (torch setup kernels listed, not counted)
        tot = sum(v[1] for k, v in agg.items() if "fo::" in k)
        res["launch_list"] = {k: {"launches": v[0], "total_us": round(v[1], 1),
                                  "avg_us": round(v[1] / v[0], 1),
                                  "share_of_engine": round(v[1] / tot, 4) if "fo::" in k else None}
                              for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}
    json.dump(res, open(out_path, "w"), indent=1)
    if current is not None:
        import pathlib

        kern = {}
        for name, d in res.items():
            if name == "launch_list" or "dram_read_bytes" not in d:
                continue
            short = d["kernel"].split("(")[0].split("<")[0].split("::")[-1].strip()
            kern[short] = {"dram_bytes_per_launch": d["dram_read_bytes"] + d.get("dram_write_bytes", 0),
                           "capture": name, "report": d["report"]}
        cur = {"source": pathlib.Path(out_path).name, "workload": current, "kernels": kern}
        pathlib.Path(out_path).with_name("ncu_current.json").write_text(json.dumps(cur, indent=1))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
