# Round-2 closing pass (tag $1): GPU tests, smoke, bench lines (C4 x2, C1, C2, C5),
# reference arm, the bench's ncu launch list
TAG=${1:-z}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for rep in a b; do
  timeout 900 python bench.py > gpurun_out/bench_r02_${TAG}$rep.json 2> gpurun_out/bench_r02_${TAG}$rep.err; echo "bench rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/bench_r02_${TAG}$rep.json'));print(d['value'],d['e2e']['value'],d['roofline']['frac'],d['breakdown_ms'],d['clocks'],d['gpu_launches'],d['cpu_baseline']['value'])"
done
for c in c1 c2 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_r02_$TAG.json 2> /dev/null; echo "$c rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/bench_${c}_r02_$TAG.json'));print('$c',d['value'],d['e2e']['value'],d['breakdown_ms'])"
done
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02_$TAG.json 2> gpurun_out/bench_ref_r02_$TAG.err; echo "ref rc=$?"
tail -c 600 gpurun_out/bench_ref_r02_$TAG.json
B="python bench.py --eager --steps 2 --warmup 3 --no-cpu --no-e2e --no-dense"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_$TAG.csv $B > /dev/null 2>&1; echo "launches rc=$?"
