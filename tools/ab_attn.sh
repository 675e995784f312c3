#!/bin/bash
# A/B of attention library variants: bench attention ms + dense attention ms, then
# the attention parity tests on the last variant. args: .so files
bash tools/ab_lib.sh "python bench.py --no-cpu --no-e2e --steps 20 | python -c \"import json,sys;d=json.loads(sys.stdin.read());b=d['breakdown_ms'];print(json.dumps({'attn':b['attention'],'dense':d['dense_ms']['attention'],'mhz':d['clocks']['sm_mhz']}))\"" "$@"
