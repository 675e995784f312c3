# Round-2 closing pass 2 (final binary: per-block head pairing in GEMM-Q)
TAG=${1:-y}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for rep in a b; do
  timeout 900 python bench.py > gpurun_out/bench_r02_${TAG}$rep.json 2> /dev/null; echo "bench rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/bench_r02_${TAG}$rep.json'));print(d['value'],d['e2e']['value'],d['roofline']['frac'],d['breakdown_ms'],d['clocks']['sm_mhz'],d['clocks']['reasons'])"
done
for c in c1 c2 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_r02_$TAG.json 2> /dev/null; echo "$c rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/bench_${c}_r02_$TAG.json'));print('$c',d['value'],d.get('e2e',{}).get('value'),d['breakdown_ms'])"
done
timeout 600 python tools/gemm_time.py > gpurun_out/gemm_time_r02_$TAG.json 2>/dev/null; echo "gemm_time rc=$?"
timeout 600 python tools/gemm_time.py --seq 4096 > gpurun_out/gemm_time4k_r02_$TAG.json 2>/dev/null
timeout 1800 python tools/sweep.py --out gpurun_out/sweep_r02_$TAG.json > /dev/null 2> gpurun_out/sweep_r02_$TAG.err; echo "sweep rc=$?"
B="python bench.py --eager --steps 2 --warmup 3 --no-cpu --no-e2e --no-dense"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_$TAG.csv $B > /dev/null 2>&1; echo "launches rc=$?"
for r in 0.25 0.9; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_q2 -s 3 -c 1 -o gpurun_out/gq_r02_${TAG}_$r -f python tools/gemm_time.py --eager --ops q --ratios $r --orders 0 > /dev/null 2>&1; echo "ncu gq $r rc=$?"
done
