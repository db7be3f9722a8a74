# K5 variant (build_a) vs working tree: interleaved c5/c3 timing, then the fp4 suite on the variant
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/k5var.log
for r in 1 2 3; do
  for v in V B; do
    if [ $v = V ]; then export LOWBIT_LIB=paper_2205_09120_b200/build_a/liblowbit_a.so; else unset LOWBIT_LIB; fi
    for c in c5 c3; do
      echo -n "$v $c " >> gpurun_out/k5var.log
      timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-extra --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4))" >> gpurun_out/k5var.log
    done
  done
done
LOWBIT_LIB=paper_2205_09120_b200/build_a/liblowbit_a.so timeout -s KILL 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fp4.py > gpurun_out/pytest_k5var.log 2>&1
echo PYTEST=$? >> gpurun_out/pytest_k5var.log
