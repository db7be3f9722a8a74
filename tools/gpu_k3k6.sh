cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/k3k6.log
rm -f $L
for r in 1 2; do
  echo -n "A " >> $L; LOWBIT_LIB=paper_2205_09120_b200/build_a/liblowbit_a.so timeout 300 python tools/k3k6_time.py >> $L 2>&1
  echo -n "B " >> $L; timeout 300 python tools/k3k6_time.py >> $L 2>&1
done
timeout -s KILL 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_conv.py tests/test_gpu_sign.py tests/test_gpu_parity.py >> $L 2>&1
echo PYTEST=$? >> $L
