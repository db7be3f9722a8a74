# A/B: committed build (A) vs working tree (B) on the c5 / c3 headline kernels, interleaved; then fp4 tests
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/k5ab.log
for r in 1 2 3; do
  for v in A B; do
    if [ $v = A ]; then export LOWBIT_LIB=paper_2205_09120_b200/build_a/liblowbit_a.so; else unset LOWBIT_LIB; fi
    for c in c5 c3; do
      echo -n "$v $c " >> gpurun_out/k5ab.log
      timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-extra --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" >> gpurun_out/k5ab.log
    done
  done
done
unset LOWBIT_LIB
timeout -s KILL 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fp4.py tests/test_gpu_parity.py > gpurun_out/pytest_k5.log 2>&1
echo PYTEST=$? >> gpurun_out/pytest_k5.log
