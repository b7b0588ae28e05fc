set -x
python bench.py --config C1 --steps 5 --warmup 3 --batches 64 2>&1 | tail -5
timeout 900 python bench.py --steps 10 --warmup 3 2>&1 | tail -15
