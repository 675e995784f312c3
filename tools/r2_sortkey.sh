for rep in 1 2 3; do for v in k0 k1 k2; do
  cp tools/bin/$v.so paper_2509_25401_b200/_fo_b200.so
  echo "$v $(python tools/gemm_time.py --ops q --orders 0 --ratios 0.25,0.5,0.75,0.9,0.95 2>/dev/null)"
done; done
cp tools/bin/k0.so paper_2509_25401_b200/_fo_b200.so
