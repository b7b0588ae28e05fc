# C5 bench at several chunk sizes (TGL_CHUNK_ROOTS), values only
for c in 1048576 262144 131072 65536; do
  v=$(TGL_CHUNK_ROOTS=$c python bench.py --steps 10 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'])")
  echo "chunk=$c $v"
done
