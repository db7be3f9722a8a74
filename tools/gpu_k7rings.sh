# K7 ring-depth experiments (TUNING build knobs): NEPI 16 raw 2 (default) / NEPI 8 raw 3 / NEPI 8 raw 2 / NEPI 8 raw 3 f4 2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/k7rings.log
export LOWBIT_LIB=paper_2205_09120_b200/build_t/liblowbit_t.so KERNELS=2
for r in 1 2; do
  echo -n "nepi16 raw2: " >> gpurun_out/k7rings.log; timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> gpurun_out/k7rings.log
  echo -n "nepi8 raw3: " >> gpurun_out/k7rings.log; LOWBIT_HALO_NEPI8=1 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> gpurun_out/k7rings.log
  echo -n "nepi8 raw2: " >> gpurun_out/k7rings.log; LOWBIT_HALO_NEPI8=1 LOWBIT_HALO_RAWST=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> gpurun_out/k7rings.log
  echo -n "nepi8 raw4 f4 2: " >> gpurun_out/k7rings.log; LOWBIT_HALO_NEPI8=1 LOWBIT_HALO_F4ST=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> gpurun_out/k7rings.log
done
LOWBIT_HALO_NEPI8=1 LOWBIT_HALO_DEBUG=32 timeout 120 python tools/halo_trace.py 2>&1 | grep "steady\|MMA waits" >> gpurun_out/k7rings.log
