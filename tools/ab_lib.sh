#!/bin/bash
# Interleaved A/B of library variants on one box:
#   tools/ab_lib.sh "<timing command>" tools/bin/a.so tools/bin/b.so ...
# Each variant is copied over paper_2509_25401_b200/_fo_b200.so and the timing
# command (printing one JSON line) runs in a fresh process; 3 rounds.
cmd=$1; shift
cp paper_2509_25401_b200/_fo_b200.so /tmp/_fo_b200.keep.so
for rep in 1 2 3; do
  for so in "$@"; do
    cp "$so" paper_2509_25401_b200/_fo_b200.so
    echo "$(basename $so) rep$rep $(timeout 600 bash -c "$cmd" 2>/dev/null | tail -1)"
  done
done
cp /tmp/_fo_b200.keep.so paper_2509_25401_b200/_fo_b200.so
