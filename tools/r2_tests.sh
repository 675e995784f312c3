# GPU parity run: the bench-shape tests first, then the whole -m gpu suite
set -x
timeout 1200 python -m pytest tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/r2_benchshapes.log 2>&1; echo "rc=$?"
tail -30 gpurun_out/r2_benchshapes.log
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/r2_gputest.log 2>&1; echo "rc=$?"
tail -15 gpurun_out/r2_gputest.log
