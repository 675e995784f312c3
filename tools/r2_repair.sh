# GEMM-Q head pairs chosen per block: parity, then A/B of GEMM-Q / QKV medians and the bench
cp tools/bin/rp1.so paper_2509_25401_b200/_fo_b200.so
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/ab_lib.sh "python tools/gemm_time.py --ops q,qkv --orders 0 --ratios 0.25,0.5,0.75,0.9" tools/bin/rp0.so tools/bin/rp1.so
bash tools/ab_lib.sh "python tools/gemm_time.py --ops q --orders 0 --ratios 0.25,0.5,0.75,0.9 --seq 4096" tools/bin/rp0.so tools/bin/rp1.so
bash tools/ab_lib.sh "python bench.py --no-cpu --no-dense --steps 20 | python -c \"import json,sys;d=json.loads(sys.stdin.read());print(json.dumps({'v':d['value'],'q':d['breakdown_ms']['gemm_q'],'e2e':d['e2e']['value']}))\"" tools/bin/rp0.so tools/bin/rp1.so
cp tools/bin/rp1.so paper_2509_25401_b200/_fo_b200.so
