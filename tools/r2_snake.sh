timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_bench_shapes.py tests/test_pipeline.py -q -x 2>&1 | tail -2
bash tools/ab_lib.sh "python tools/gemm_time.py --seq 4096 --ops q --ratios 0.25,0.5,0.75,0.9 --orders 0" tools/bin/rr.so tools/bin/snake.so
bash tools/ab_lib.sh "python tools/gemm_time.py --ops q --ratios 0.0,0.25,0.5,0.75,0.9 --orders 0" tools/bin/rr.so tools/bin/snake.so
