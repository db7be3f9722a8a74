# usage: VARS="lib1 lib2" DBG="0 5" bash tools/fp4_variants.sh
for V in default ${VARS}; do
  for D in ${DBG:-0}; do
    if [ "$V" = default ]; then unset LOWBIT_LIB; else export LOWBIT_LIB=$PWD/variants/$V.so; fi
    r=$(LOWBIT_DEBUG_FP4=$D python bench.py --steps ${STEPS:-20} --warmup 3 --layout nibbles --config ${CFG:-c5} --no-cpu-baseline --no-e2e --no-extra | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks'].get('samples'))")
    echo "$V debug=$D $r"
  done
done
