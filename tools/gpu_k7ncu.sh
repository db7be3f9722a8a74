cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 python tools/conv_once.py > gpurun_out/k7ncu_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:conv_fp4_halo -s 2 -c 1 -o gpurun_out/k7_prod python tools/conv_once.py > gpurun_out/k7_ncu.log 2>&1
echo NCU=$? >> gpurun_out/k7ncu_plain.log
