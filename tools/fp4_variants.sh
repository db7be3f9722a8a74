# usage: VARS="lib1 lib2" DBG="0 5" REPS=3 bash tools/fp4_variants.sh  (tuning experiments)
for R in $(seq ${REPS:-1}); do
for V in default ${VARS}; do
  for D in ${DBG:-0}; do
    if [ "$V" = default ]; then unset LOWBIT_LIB; else export LOWBIT_LIB=$PWD/variants/$V.so; fi
    r=$(LOWBIT_DEBUG_FP4=$D M=${M:-1048576} NS=${NS:-1024} python tools/fp4_shape_sweep.py | tr '\n' ' ')
    echo "$V debug=$D $r"
  done
done
done
