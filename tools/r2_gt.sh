set -x
python tools/gemm_time.py > gpurun_out/gt_graph.json 2>gpurun_out/gt.err; tail -3 gpurun_out/gt.err
python tools/gemm_time.py --seq 4096 > gpurun_out/gt4k_graph.json 2>>gpurun_out/gt.err
python tools/gemm_time.py --seq 4096 --eager > gpurun_out/gt4k_eager.json 2>>gpurun_out/gt.err
cat gpurun_out/gt_graph.json gpurun_out/gt4k_graph.json gpurun_out/gt4k_eager.json
timeout 1200 python tools/sweep.py --parts attn,flux --out gpurun_out/sweep_attn_g.json > /dev/null 2>>gpurun_out/gt.err; tail -3 gpurun_out/gt.err
