for rep in 1 2 3; do
  for v in 0 128 256; do
    echo "== GG_DGEMM_SMALL_K=$v"
    GG_DGEMM_SMALL_K=$v python tools/prof_prepare.py --n 10000 40000 --reps 3 2>&1 | grep "rep=2"
  done
done
