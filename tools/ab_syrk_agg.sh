# A/B of gls_prepare wall time across GG_SYRK_AGG values, alternating: bash tools/ab_syrk_agg.sh 1 2 3
for rep in 1 2 3; do
  for a in "$@"; do
    echo "== GG_SYRK_AGG=$a"
    GG_SYRK_AGG=$a python tools/prof_prepare.py --n 10000 40000 --reps 3 2>&1 | grep "rep=2"
  done
done
