# K7 correctness (conv tests + sign tests), c4 timing (product build, and build_c if present), a step trace
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/k7_time.log gpurun_out/k7_dbg2.log
timeout -s KILL 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_conv.py tests/test_gpu_sign.py > gpurun_out/pytest_k7.log 2>&1
echo PYTEST=$? >> gpurun_out/pytest_k7.log
for r in 1 2; do
  echo -n "B " >> gpurun_out/k7_time.log; KERNELS=2 timeout 120 python tools/conv_c4_time.py >> gpurun_out/k7_time.log 2>&1
  if [ -f paper_2205_09120_b200/build_c/liblowbit_c.so ]; then echo -n "C " >> gpurun_out/k7_time.log; LOWBIT_LIB=paper_2205_09120_b200/build_c/liblowbit_c.so KERNELS=2 timeout 120 python tools/conv_c4_time.py >> gpurun_out/k7_time.log 2>&1; fi
done
