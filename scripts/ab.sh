# A/B of library variants on one config with tools/ktime.py (one process per variant):
#   bash scripts/ab.sh OUTDIR [ktime args] -- lib1.so lib2.so ...   ("product" = the in-tree library)
out=$1; shift
args=()
while [ "$1" != "--" ]; do args+=("$1"); shift; done; shift
mkdir -p $out
for v in "$@"; do
  if [ "$v" = product ]; then lib=""; else lib=$PWD/$v; fi
  TGL_LIB_PATH=$lib python tools/ktime.py "${args[@]}" 2>&1 | tail -1 | sed "s|^|$v |" >> $out/ktime.txt
done
cat $out/ktime.txt
