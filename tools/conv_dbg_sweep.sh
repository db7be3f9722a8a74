#!/bin/bash
# K6 timing experiments: c4 (pack + conv) per LOWBIT_CONV_DEBUG value (each its own process; results invalid
# for the flags that skip work).  1 no stores, 2 no MMAs, 4 no A loads, 8 no TMEM loads, 2048 no STS.
cd "$(dirname "$0")/.."
for d in ${DBG_LIST:-0 1 2 4 8 3 5 6 7 2048}; do
  echo -n "dbg $d: "
  LOWBIT_CONV_DEBUG=$d PROBE_B=64 timeout 120 python tools/conv_scale_probe.py 2>&1 | tail -1
done
