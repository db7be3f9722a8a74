# K7 converter groups: 2 groups (working tree, f4 2 / raw 2), 1 group (build_c: f4 3 / raw 2), 1 group f4 2 (build_a + knob)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/k7cg.log
for r in 1 2; do
  echo -n "2 groups f4 2: " >> gpurun_out/k7cg.log; KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> gpurun_out/k7cg.log
  echo -n "1 group f4 3: " >> gpurun_out/k7cg.log; LOWBIT_LIB=paper_2205_09120_b200/build_c/liblowbit_c.so KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> gpurun_out/k7cg.log
  echo -n "1 group f4 2: " >> gpurun_out/k7cg.log; LOWBIT_LIB=paper_2205_09120_b200/build_a/liblowbit_a.so LOWBIT_HALO_F4ST=2 KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> gpurun_out/k7cg.log
done
