#!/bin/bash
# Interleaved timing of config 5 on K5 across builds: working tree (B), build_a (A) and, if present, build_c (C).
cd "$(dirname "$0")/.."
CMD="python bench.py --steps 20 --warmup 3 --layout nibbles --config ${CFG:-c5} --no-cpu-baseline --no-e2e --no-extra"
P='import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"], 4))'
for r in 1 2 3; do
  echo -n "A: "; LOWBIT_LIB=paper_2205_09120_b200/build_a/liblowbit_a.so timeout 200 $CMD | python -c "$P"
  echo -n "B: "; timeout 200 $CMD | python -c "$P"
  if [ -f paper_2205_09120_b200/build_c/liblowbit_c.so ]; then
    echo -n "C: "; LOWBIT_LIB=paper_2205_09120_b200/build_c/liblowbit_c.so timeout 200 $CMD | python -c "$P"
  fi
done
