# e2e A/B/C: build_a, build_c, working tree (B), interleaved
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/e2eab.log
for r in 1 2; do for v in A C B; do
  case $v in A) export LOWBIT_LIB=paper_2205_09120_b200/build_a/liblowbit_a.so;; C) export LOWBIT_LIB=paper_2205_09120_b200/build_c/liblowbit_c.so;; B) unset LOWBIT_LIB;; esac
  echo -n "$v " >> gpurun_out/e2eab.log
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print(round(e['ms_per_step'],2), round(e['pageable']['ms_per_step'],1), round(d['ms_per_step'],4))" >> gpurun_out/e2eab.log
done; done
