# K7 A/B + a trace of the TUNING build
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/k7ab.log
rm -f $L
timeout -s KILL 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_conv.py tests/test_gpu_sign.py >> $L 2>&1
echo PYTEST=$? >> $L
bash tools/ab_conv.sh >> $L 2>&1
for d in 32 672; do
echo "== dbg $d" >> $L
LOWBIT_LIB=paper_2205_09120_b200/build_t/liblowbit_t.so LOWBIT_HALO_DEBUG=$d timeout 120 python tools/halo_trace.py 2>&1 | grep "phases\|steady\|MMA waits" >> $L
done
