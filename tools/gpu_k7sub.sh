# K7 work-item variants (TUNING build): sub 2 / NEPI 8 (default), sub 1 / NEPI 16, and traces
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/k7sub.log
rm -f $L
T=paper_2205_09120_b200/build_t/liblowbit_t.so
for r in 1 2; do
  echo -n "A(head) " >> $L; LOWBIT_LIB=paper_2205_09120_b200/build_a/liblowbit_a.so KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> $L
  echo -n "T sub2 " >> $L; LOWBIT_LIB=$T KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> $L
  echo -n "T sub1 " >> $L; LOWBIT_HALO_SUB=1 LOWBIT_LIB=$T KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> $L
done
echo "== sub2 trace" >> $L
LOWBIT_LIB=$T LOWBIT_HALO_DEBUG=32 timeout 120 python tools/halo_trace.py >> $L 2>&1
echo "== sub2 trace no epilogue" >> $L
LOWBIT_LIB=$T LOWBIT_HALO_DEBUG=160 timeout 120 python tools/halo_trace.py 2>&1 | grep "phases\|steady\|MMA waits" >> $L
