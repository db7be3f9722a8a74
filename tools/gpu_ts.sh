cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/ts.log
rm -f $L
timeout 300 python tools/ts_debug.py >> $L 2>&1
echo DBG=$? >> $L
timeout -s KILL 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_conv.py tests/test_gpu_sign.py >> $L 2>&1
echo PYTEST=$? >> $L
bash tools/ab_conv.sh >> $L 2>&1
