# K7: conv + sign tests on the working-tree build, then interleaved c4 timing A (build_a) / B (working tree)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/k7ab.log
rm -f $L
timeout -s KILL 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_conv.py tests/test_gpu_sign.py >> $L 2>&1
echo PYTEST=$? >> $L
bash tools/ab_conv.sh >> $L 2>&1
