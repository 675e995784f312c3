# small layers: attention items in one global length order for the per-wave LPT
cp tools/bin/gl1.so paper_2509_25401_b200/_fo_b200.so
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c1 c2; do
bash tools/ab_lib.sh "python bench.py --config $c --no-cpu --no-dense --steps 20 | python -c \"import json,sys;d=json.loads(sys.stdin.read());print(json.dumps({'v':d['value'],'attn':d['breakdown_ms']['attention']}))\"" tools/bin/base.so tools/bin/gl1.so
done
for v in base gl1; do cp tools/bin/$v.so paper_2509_25401_b200/_fo_b200.so; echo "$v $(python tools/sweep.py --parts flux 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print([(r['kv_skip_ratio'],r['ms']) for r in d['attention_c2_flux']])")"; done
cp tools/bin/gl1.so paper_2509_25401_b200/_fo_b200.so
