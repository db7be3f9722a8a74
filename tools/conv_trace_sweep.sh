#!/bin/bash
# K6 per-tile timelines (pair 0 leader) under timing-experiment flags (each OR 32 = trace on);
# also the c4 time per conv with the flag set.  Flags: see ConvF4Params::dbg in csrc/conv_fp4_pair.cu.
cd "$(dirname "$0")/.."
for d in ${DBG_LIST:-0 16 8 2048 1 2 2057 2059 4096}; do
  echo "=== dbg $d"
  LOWBIT_CONV_DEBUG=$((d | 32)) timeout 100 python tools/conv_trace.py 2>&1 | tail -28
  LOWBIT_CONV_DEBUG=$d PROBE_B=64 timeout 100 python tools/conv_scale_probe.py 2>&1 | tail -1
done
