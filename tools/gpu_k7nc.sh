# K7: 8 converter warps + 16 epilogue (working tree) vs 16 converter warps + 8 epilogue (build_c)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/k7nc.log
for r in 1 2; do
  echo -n "conv8 epi16: " >> gpurun_out/k7nc.log; KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> gpurun_out/k7nc.log
  echo -n "conv16 epi8: " >> gpurun_out/k7nc.log; LOWBIT_LIB=paper_2205_09120_b200/build_c/liblowbit_c.so KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> gpurun_out/k7nc.log
done
LOWBIT_LIB=paper_2205_09120_b200/build_c/liblowbit_c.so timeout -s KILL 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_conv.py tests/test_gpu_sign.py >> gpurun_out/k7nc.log 2>&1
echo PYTEST=$? >> gpurun_out/k7nc.log
