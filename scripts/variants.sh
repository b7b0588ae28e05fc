# tools/sweep.py default setting for each prebuilt tools/variants/lib*.so
for f in tools/variants/lib*.so; do
  echo -n "$f "; TGL_LIB_PATH=$PWD/$f python tools/sweep.py --only handle=aux "$@" 2>&1 | grep handle
done
