# Full sweep (attention C4/C2, GEMM C3) + GEMM medians at both S. $1 = tag
TAG=${1:-s}
set -x
timeout 600 python tools/gemm_time.py > gpurun_out/gemm_time_$TAG.json 2> gpurun_out/gemm_time_$TAG.err; echo "rc=$?"
timeout 600 python tools/gemm_time.py --seq 4096 > gpurun_out/gemm_time4k_$TAG.json 2>> gpurun_out/gemm_time_$TAG.err; echo "rc=$?"
cat gpurun_out/gemm_time_$TAG.json gpurun_out/gemm_time4k_$TAG.json
timeout 1500 python tools/sweep.py --out gpurun_out/sweep_$TAG.json > /dev/null 2> gpurun_out/sweep_$TAG.err; echo "sweep rc=$?"
tail -3 gpurun_out/sweep_$TAG.err
