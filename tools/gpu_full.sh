# full GPU suite + default bench line (round 2 checks)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1
echo PYTEST=$? >> gpurun_out/pytest_full.log
KERNELS=2 timeout 120 python tools/conv_c4_time.py > gpurun_out/c4_time.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo BENCH=$? >> gpurun_out/pytest_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo SMOKE=$? >> gpurun_out/pytest_full.log
