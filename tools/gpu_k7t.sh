# timing only: in-tree library (H) against $XLIBS on c4 (bench's cold / back-to-back method)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/k7t.log
rm -f $L
for r in 1 2; do
  echo -n "H: " >> $L; timeout 120 python tools/c4_flushed.py 2>&1 | tail -1 >> $L
  for X in $XLIBS; do
  echo -n "$X: " >> $L; LOWBIT_LIB=$X timeout 120 python tools/c4_flushed.py 2>&1 | tail -1 >> $L
  done
done
