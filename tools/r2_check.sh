# Round-2 state check: full -m gpu suite, bench line (with CPU legs)
TAG=${1:-c}
set -x
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gputest_$TAG.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/gputest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -c 3500 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
