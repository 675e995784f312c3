# Round-2 final measurement pass on one B200 (tag $1): bench lines (C4 default,
# N=1), the bench's launch list, ncu --set full of the attention kernel at the
# bench workload and of GEMM-Q / GEMM-O dispatch / GEMM-O update at 25% and 90%
# cached (C3, S=33024), GEMM medians and the sparsity sweep.
TAG=${1:-f}
set -x
timeout 900 python bench.py > gpurun_out/bench_r02_$TAG.json 2> gpurun_out/bench_r02_$TAG.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_r02_$TAG.json
B="python bench.py --eager --steps 2 --warmup 3 --no-cpu --no-e2e --no-dense"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_$TAG.csv $B > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_attention_cs -s 2 -c 1 -o gpurun_out/attn_r02_$TAG -f $B > /dev/null 2>&1; echo "attn rc=$?"
for r in 0.25 0.9; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_q2 -s 3 -c 1 -o gpurun_out/gq_r02_${TAG}_$r -f python tools/gemm_time.py --eager --ops q --ratios $r --orders 0 > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_o_kernel -s 5 -c 1 -o gpurun_out/godisp_r02_${TAG}_$r -f python tools/gemm_time.py --eager --ops disp --ratios $r --orders 1 > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_o_update -s 5 -c 1 -o gpurun_out/goupd_r02_${TAG}_$r -f python tools/gemm_time.py --eager --ops upd --ratios $r --orders 1 > /dev/null 2>&1
done
timeout 600 python tools/gemm_time.py > gpurun_out/gemm_time_r02_$TAG.json 2>/dev/null; echo "gemm_time rc=$?"
timeout 600 python tools/gemm_time.py --seq 4096 > gpurun_out/gemm_time4k_r02_$TAG.json 2>/dev/null
timeout 1800 python tools/sweep.py --out gpurun_out/sweep_r02_$TAG.json > /dev/null 2> gpurun_out/sweep_r02_$TAG.err; echo "sweep rc=$?"
ls -la gpurun_out/ | grep $TAG
for c in c1 c2 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_r02_$TAG.json 2> /dev/null; echo "$c rc=$?"
done
timeout 600 python tools/external_check.py > gpurun_out/external_r02_$TAG.json 2>/dev/null; echo "external rc=$?"
