set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest0.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_gputest0.log
timeout 600 python bench.py > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err; echo "bench rc=$?"
cat gpurun_out/r2_bench0.json
