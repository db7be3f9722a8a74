#!/bin/bash
# K7 timing experiments on c4 (graph replay after an L2 flush; results invalid for flags that skip work):
# LOWBIT_HALO_DEBUG 1 no output stores, 2 one MMA pair per tile, 4 no conversion.
cd "$(dirname "$0")/.."
for d in ${DBG_LIST:-0 1 2 4 3 5 6 7}; do
  echo -n "dbg $d: "
  LOWBIT_HALO_DEBUG=$d KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1
done
