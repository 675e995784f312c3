# GEMM-Q: largest block distance of a two-block N=256 job (A/B)
cp tools/bin/d8.so paper_2509_25401_b200/_fo_b200.so
timeout 900 python -m pytest tests/test_gpu_bench_shapes.py -q -x -k "gq_job_list or gemm_q_c4 or fused" 2>&1 | tail -2
for rep in 1 2 3; do for v in rp0 dinf d32 d8; do
  cp tools/bin/$v.so paper_2509_25401_b200/_fo_b200.so
  echo "$v $(python tools/gemm_time.py --ops q --orders 0 --ratios 0.25,0.5,0.75,0.9,0.95 2>/dev/null) $(python tools/gemm_time.py --ops q --orders 0 --ratios 0.25,0.5,0.75 --seq 4096 2>/dev/null)"
done; done
cp tools/bin/dinf.so paper_2509_25401_b200/_fo_b200.so
