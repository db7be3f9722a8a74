cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/e2e.log
nproc >> gpurun_out/e2e.log
export LOWBIT_LIB=paper_2205_09120_b200/build_t/liblowbit_t.so
for th in 8 12 16 24; do for mb in 16 32; do
  LOWBIT_COPY_THREADS=$th LOWBIT_STAGE_MB=$mb timeout 300 python tools/e2e_pageable_time.py >> gpurun_out/e2e.log 2>&1
done; done
