# Iteration run: GPU tests, bench line, GEMM sweep. $1 = tag
TAG=${1:-x}
set -x
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gputest_$TAG.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gputest_$TAG.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_$TAG.err
timeout 900 python tools/sweep.py --parts ${PARTS:-gemm} --out gpurun_out/sweep_$TAG.json > /dev/null 2> gpurun_out/sweep_$TAG.err; echo "sweep rc=$?"
tail -3 gpurun_out/sweep_$TAG.err
