#!/bin/bash
# A/B timing of library variants on one box: tools/ab.sh tools/bin/a.so tools/bin/b.so ...
# (interleaved twice; attention / gemm ms from bench.py)
for rep in 1 2; do
  for so in "$@"; do
    cp "$so" paper_2509_25401_b200/_fo_b200.so
    r=$(timeout 300 python bench.py --no-cpu --no-e2e --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());b=d['breakdown_ms'];print(b['attention'],b['gemm_q'],b['gemm_o_dispatch'],d['dense_ms']['attention'])")
    echo "$(basename $so) rep$rep attn/gq/go/dense_attn: $r"
  done
done
