# GEMM-Q at S=4096: kernel durations (ncu) across cached ratios
for r in 0.0 0.5 0.9 1.0; do
  ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm_q2 -s 3 -c 1 python tools/gemm_time.py --eager --seq 4096 --ops q --ratios $r --orders 0 2>/dev/null | grep -E "gpu__time|sm__cycles|tensor" | sed "s/^/$r /"
done
