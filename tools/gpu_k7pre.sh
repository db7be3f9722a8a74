cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/k7pre.log
rm -f $L
timeout -s KILL 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_conv.py -k "large_sums or config4" >> $L 2>&1
echo PYTEST=$? >> $L
