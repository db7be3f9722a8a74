cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/k4c.log
for r in 1 2 3; do timeout 120 python tools/k4_time.py >> gpurun_out/k4c.log 2>&1; done
timeout -s KILL 1200 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_conv.py tests/test_gpu_sign.py tests/test_gpu_parity.py > gpurun_out/pytest_k4c.log 2>&1
echo PYTEST=$? >> gpurun_out/pytest_k4c.log
