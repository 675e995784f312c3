# speculative row max: parity, A/B (bench attention + dense), C4 phase timing
cp tools/bin/sp1.so paper_2509_25401_b200/_fo_b200.so
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/ab_attn.sh tools/bin/sp0.so tools/bin/sp1.so
cp tools/bin/tm.so paper_2509_25401_b200/_fo_b200.so
python tools/cs_timing.py 0.25 0.5 | tail -3
cp tools/bin/sp1.so paper_2509_25401_b200/_fo_b200.so
