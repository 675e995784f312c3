timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_bench_shapes.py tests/test_engine.py tests/test_pipeline.py tests/test_gpu_sharded.py -q -x 2>&1 | tail -2
bash tools/ab_lib.sh "python bench.py --config c1 --no-cpu --no-e2e --steps 20 | python -c \"import json,sys;d=json.loads(sys.stdin.read());print(json.dumps({'c1':d['value'],'b':d['breakdown_ms']}))\"" tools/bin/pdl0.so tools/bin/pdl1.so
bash tools/ab_lib.sh "python tools/gemm_time.py --seq 4096 --ratios 0.0,0.5,0.9 --orders 1" tools/bin/pdl0.so tools/bin/pdl1.so
bash tools/ab_lib.sh "python bench.py --no-cpu --no-e2e --steps 20 | python -c \"import json,sys;d=json.loads(sys.stdin.read());print(json.dumps({'c4':d['value']}))\"" tools/bin/pdl0.so tools/bin/pdl1.so
