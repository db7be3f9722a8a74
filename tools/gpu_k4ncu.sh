cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 python tools/k4_time.py > gpurun_out/k4b.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_encode_ring -s 1 -c 1 -o gpurun_out/k4_ring python tools/k4_time.py > gpurun_out/k4_ncu.log 2>&1
echo NCU=$? >> gpurun_out/k4b.log
