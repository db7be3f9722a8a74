cd "$(dirname "$0")/.."
mkdir -p gpurun_out
echo "== A (no sign check)" > gpurun_out/k7_trace.log
LOWBIT_LIB=paper_2205_09120_b200/build_a/liblowbit_at.so LOWBIT_HALO_DEBUG=32 timeout 120 python tools/halo_trace.py >> gpurun_out/k7_trace.log 2>&1
echo "== B (sign check)" >> gpurun_out/k7_trace.log
LOWBIT_LIB=paper_2205_09120_b200/build_t/liblowbit_t.so LOWBIT_HALO_DEBUG=32 timeout 120 python tools/halo_trace.py >> gpurun_out/k7_trace.log 2>&1
