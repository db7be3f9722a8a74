cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
for v in A B C; do
  case $v in A) export LOWBIT_LIB=paper_2205_09120_b200/build_a/liblowbit_a.so;; B) unset LOWBIT_LIB;; C) export LOWBIT_LIB=paper_2205_09120_b200/build_c/liblowbit_c.so;; esac
  echo "== $v" >> gpurun_out/k2k4.log
  timeout 300 python tools/k2_time.py >> gpurun_out/k2k4.log 2>&1
  timeout 120 python tools/k4_time.py >> gpurun_out/k2k4.log 2>&1
done; done
unset LOWBIT_LIB
timeout -s KILL 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_conv.py tests/test_gpu_parity.py > gpurun_out/pytest_k2k4.log 2>&1
echo PYTEST=$? >> gpurun_out/pytest_k2k4.log
