# K7 experiment isolation: TUNING builds of HEAD (T) and the experiment (D) with ring / epilogue-warp knobs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/k7x2.log
rm -f $L
T=paper_2205_09120_b200/build_t/liblowbit_t.so
D=paper_2205_09120_b200/build_d/liblowbit_d.so
run() { echo -n "$1: " >> $L; shift; env "$@" KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> $L; }
for r in 1 2; do
run "T          " LOWBIT_LIB=$T
run "T f4st2    " LOWBIT_LIB=$T LOWBIT_HALO_F4ST=2
run "T nepi8    " LOWBIT_LIB=$T LOWBIT_HALO_NEPI8=1
run "D          " LOWBIT_LIB=$D
run "D nepi8    " LOWBIT_LIB=$D LOWBIT_HALO_NEPI8=1
run "D nobias   " LOWBIT_LIB=$D LOWBIT_HALO_DEBUG=8192
run "D nepi8 nob" LOWBIT_LIB=$D LOWBIT_HALO_NEPI8=1 LOWBIT_HALO_DEBUG=8192
run "D noepi    " LOWBIT_LIB=$D LOWBIT_HALO_DEBUG=128
run "T noepi    " LOWBIT_LIB=$T LOWBIT_HALO_DEBUG=128
done
