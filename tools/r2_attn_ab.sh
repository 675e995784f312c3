# attention A/B: parity suite on the default build, C4 bench attention + FLUX sweep per variant
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_bench_shapes.py tests/test_engine.py tests/test_pipeline.py -q -x 2>&1 | tail -2
bash tools/ab_attn.sh "$@"
cp paper_2509_25401_b200/_fo_b200.so /tmp/keep.so
for so in "$@"; do
  cp $so paper_2509_25401_b200/_fo_b200.so
  echo "$(basename $so) flux: $(timeout 600 python tools/sweep.py --parts flux 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print([(r['kv_skip_ratio'],r['ms'],r['frac']) for r in d['attention_c2_flux']])")"
done
cp /tmp/keep.so paper_2509_25401_b200/_fo_b200.so
