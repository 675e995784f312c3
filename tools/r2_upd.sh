set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "gemm_o or update or engine or pipeline or run or materialize" > gpurun_out/gputest_f.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/gputest_f.log
tools/ab_lib.sh "python tools/gemm_time.py --ops disp,upd" tools/bin/new.so tools/bin/upd.so > gpurun_out/ab_f.txt 2>&1
cat gpurun_out/ab_f.txt
