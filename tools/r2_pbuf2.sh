# separate P buffer + own V producer warp: parity, A/B, phase timing
cp tools/bin/pbv.so paper_2509_25401_b200/_fo_b200.so
timeout 900 python -m pytest tests -m gpu -x -q -k "attention or attn or pair or smoke or bench_shapes or reference_suite" 2>&1 | tail -2
bash tools/ab_attn.sh tools/bin/base.so tools/bin/b_v.so tools/bin/pbv.so
cp tools/bin/tm.so paper_2509_25401_b200/_fo_b200.so
python tools/cs_timing.py 0.25 0.5 | tail -3
cp tools/bin/base.so paper_2509_25401_b200/_fo_b200.so
