# Round-2 measurement pass on one B200: bench line, launch list, ncu --set full
# of the hot kernels at the bench workload (25% cached) and GEMM-Q / GEMM-O at
# 90% cached. Output names carry a tag ($1, default "a").
TAG=${1:-a}
set -x
timeout 900 python bench.py > gpurun_out/bench_r02_$TAG.json 2> gpurun_out/bench_r02_$TAG.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_r02_$TAG.json
B="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-dense"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-dense > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_attention_cs -s 1 -c 1 -o gpurun_out/attn_r02_$TAG -f $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_q -s 2 -c 2 -o gpurun_out/gq_r02_$TAG -f $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_o -s 2 -c 1 -o gpurun_out/go_r02_$TAG -f $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_q -s 2 -c 2 -o gpurun_out/gq90_r02_$TAG -f $B --cached 0.9 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_o -s 2 -c 1 -o gpurun_out/go90_r02_$TAG -f $B --cached 0.9 > /dev/null 2>&1
ls -la gpurun_out/
