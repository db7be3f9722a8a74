set -x
python -m pytest tests/test_gpu_fp4.py -x -q 2>&1 | tail -15
for L in nibbles lanes; do python bench.py --steps 20 --warmup 3 --layout $L --no-cpu-baseline --no-e2e --no-extra; done
