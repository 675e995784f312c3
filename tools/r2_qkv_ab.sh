for rep in 1 2 3; do
  for f in 0 1; do
    echo "fused=$f rep$rep $(FO_FUSED_QKV=$f timeout 600 python bench.py --no-cpu --no-dense --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(json.dumps({'e2e':d['e2e']['value'],'launches':d['e2e']['gpu_launches_per_step'],'step':d['value']}))")"
  done
done
FO_FUSED_QKV=1 python tools/e2e_probe.py 2>&1 | tail -3
FO_FUSED_QKV=0 python tools/e2e_probe.py 2>&1 | tail -3
