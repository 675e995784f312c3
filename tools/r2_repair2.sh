for rep in 1 2 3 4; do for v in rp0 rp1; do
  cp tools/bin/$v.so paper_2509_25401_b200/_fo_b200.so
  echo "$v $(python tools/gemm_time.py --ops q --orders 0 --ratios 0.75,0.9,0.95 2>/dev/null)"
done; done
bash tools/ab_lib.sh "python bench.py --config c1 --no-cpu --no-dense --steps 20 | python -c \"import json,sys;d=json.loads(sys.stdin.read());print(json.dumps({'v':d['value'],'q':d['breakdown_ms']['gemm_q']}))\"" tools/bin/rp0.so tools/bin/rp1.so
cp tools/bin/rp1.so paper_2509_25401_b200/_fo_b200.so
