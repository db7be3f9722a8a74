cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/k7tr.log
rm -f $L
for lib in build_t/liblowbit_t.so build_d/liblowbit_d.so; do
for d in 32 160; do
echo "== $lib dbg $d" >> $L
LOWBIT_LIB=paper_2205_09120_b200/$lib LOWBIT_HALO_DEBUG=$d timeout 120 python tools/halo_trace.py >> $L 2>&1
done
done
