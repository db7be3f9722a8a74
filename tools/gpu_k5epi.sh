# K5 epilogue experiments on the TUNING build
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/k5epi.log
rm -f $L
T=paper_2205_09120_b200/build_t/liblowbit_t.so
run() { echo -n "$1: " >> $L; shift; env "$@" LOWBIT_LIB=$T timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline --no-extra --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4))" >> $L; }
for r in 1 2; do
run "tma epilogue     " A=1
run "C evict_first    " LOWBIT_DEBUG_FP4=1024
run "C evict_normal   " LOWBIT_DEBUG_FP4=2048
done
