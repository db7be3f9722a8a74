# K7 experiment: alternative builds (X...) against the in-tree library (H): conv suites on each X, then interleaved c4 timing
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/k7x.log
rm -f $L
for X in $XLIBS; do
LOWBIT_LIB=$X timeout -s KILL 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_conv.py tests/test_gpu_sign.py 2>&1 | tail -4 >> $L
echo "PYTEST $X = $?" >> $L
done
for r in 1 2 3; do
  echo -n "H: " >> $L; KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> $L
  for X in $XLIBS; do
  echo -n "$X: " >> $L; LOWBIT_LIB=$X KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> $L
  done
done
