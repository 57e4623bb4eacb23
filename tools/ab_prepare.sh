# A/B of gls_prepare wall time across library builds, alternating: bash tools/ab_prepare.sh lib1.so lib2.so
for rep in 1 2 3; do
  for lib in "$@"; do
    echo "== $lib"
    GG_LIB_PATH=$lib python tools/prof_prepare.py --n 10000 40000 --reps 3 2>&1 | grep "rep=2"
  done
done
