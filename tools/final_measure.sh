set -x
python bench.py > gpurun_out/bench_r01_v5.json 2> gpurun_out/bench_v5.err
python tools/sweep.py --out gpurun_out/sweep_r01_v5.json > gpurun_out/sweep_v5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_v5.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-dense > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sparse_attention_cs -s 3 -c 1 -o gpurun_out/attn_v5 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-dense > /dev/null 2>&1
ncu --set full --clock-control none -k regex:gemm_q -s 3 -c 1 -o gpurun_out/gq_v5 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-dense > /dev/null 2>&1
ncu --set full --clock-control none -k regex:gemm_o -s 3 -c 1 -o gpurun_out/go_v5 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-dense > /dev/null 2>&1
ls -la gpurun_out/
