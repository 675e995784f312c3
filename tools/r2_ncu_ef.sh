for v in base pf0 el0; do
  cp tools/bin/$v.so paper_2509_25401_b200/_fo_b200.so
  for r in 0.25 0.9; do
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:gemm_o_kernel -s 5 -c 1 python tools/gemm_time.py --eager --ops disp --ratios $r --orders 1 2>/dev/null | grep -E "dram__|gpu__time|lts__" | sed "s/^/$v $r /"
  done
done
