#!/bin/bash
# Interleaved A/B timing of the c4 conv: working-tree build (B) vs build_a (A), 3 rounds each.
cd "$(dirname "$0")/.."
for r in 1 2 3; do
  echo -n "A: "; LOWBIT_LIB=paper_2205_09120_b200/build_a/liblowbit_a.so KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1
  echo -n "B: "; KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1
done
