# shared-ones V layout + double O staging: parity, then A/B (bench attention, dense, FLUX C2 sweep)
cp tools/bin/vs1.so paper_2509_25401_b200/_fo_b200.so
timeout 900 python -m pytest tests -m gpu -x -q -k "attention or attn or pair or smoke or bench_shapes" 2>&1 | tail -3
bash tools/ab_attn.sh tools/bin/vs0.so tools/bin/vs1.so
for rep in 1 2; do for v in vs0 vs1; do
  cp tools/bin/$v.so paper_2509_25401_b200/_fo_b200.so
  echo "$v flux $(timeout 300 python tools/sweep.py --parts flux 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print([(r['kv_skip_ratio'],r['ms']) for r in d['attention_c2_flux']])")"
done; done
cp tools/bin/vs1.so paper_2509_25401_b200/_fo_b200.so
