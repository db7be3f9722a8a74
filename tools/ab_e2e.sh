#!/bin/bash
# Interleaved e2e timing (host drop-in on c5): working tree (B) vs build_a (A).
cd "$(dirname "$0")/.."
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extra"
P='import json,sys; d=json.loads(sys.stdin.read()); print(round(d["e2e"]["value"], 1), round(d["e2e"]["ms_per_step"], 2))'
for r in 1 2; do
  echo -n "A: "; LOWBIT_LIB=paper_2205_09120_b200/build_a/liblowbit_a.so timeout 300 $CMD | python -c "$P"
  echo -n "B: "; timeout 300 $CMD | python -c "$P"
done
