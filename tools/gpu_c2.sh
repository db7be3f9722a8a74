cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/c2.log
rm -f $L
timeout -s KILL 600 python -m pytest -q -x -p no:cacheprovider tests -m gpu -k "grouped or c2 or sweep" >> $L 2>&1
echo PYTEST=$? >> $L
for r in 1 2 3; do
  echo -n "A " >> $L; LOWBIT_LIB=paper_2205_09120_b200/build_a/liblowbit_a.so timeout 120 python tools/c2_grouped_time.py >> $L 2>&1
  echo -n "B " >> $L; timeout 120 python tools/c2_grouped_time.py >> $L 2>&1
done
