# conv2d_lowbit through the C++ drop-in (config 4, 64 single-image calls) and the conv/host tests
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/convdropin.log
rm -f $L
timeout 900 python -m pytest -x -q tests/test_gpu_hardening.py tests/test_cpp_dropin.py tests/test_gpu_conv.py tests/test_gpu_sign.py >> $L 2>&1
echo "pytest exit $?" >> $L
for i in 1 2 3; do
  timeout 300 paper_2205_09120_b200/cpp/build/dropin_e2e conv 1 64 56 56 128 128 5 46 >> $L 2>&1
done
