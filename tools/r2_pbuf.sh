# separate P buffer in TMEM (QK two tiles ahead): parity, A/B, phase timing
cp tools/bin/pb1.so paper_2509_25401_b200/_fo_b200.so
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/ab_attn.sh tools/bin/base.so tools/bin/pb1.so
cp tools/bin/tm.so paper_2509_25401_b200/_fo_b200.so
python tools/cs_timing.py 0.25 0.5 | tail -3
python tools/cs_timing.py 0.0 0.9 4608 | grep "kernel span"
cp tools/bin/pb1.so paper_2509_25401_b200/_fo_b200.so
