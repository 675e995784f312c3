# bench lines of the other BASELINE configs (C1, C2, C5) and the default C4. $1 = tag
TAG=${1:-a}
set -x
for c in c4 c1 c2 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "$c rc=$?"
  tail -c 600 gpurun_out/bench_${c}_$TAG.json; tail -3 gpurun_out/bench_${c}_$TAG.err
done
