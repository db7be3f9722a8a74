# K5 (c5 headline) source-level ncu capture with full-rate warp sampling
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra --no-e2e"
timeout 300 $CMD > gpurun_out/k5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 2 -k regex:gemm_fp4_pair -s 1 -c 1 -o gpurun_out/k5_r02 $CMD > gpurun_out/k5_ncu.log 2>&1
echo NCU=$? >> gpurun_out/k5_plain.log
