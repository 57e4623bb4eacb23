# A/B of the int8 TRSM tile variants at configs 3 and 1 (alternating; clocks in the last field)
run() { python bench.py --config $1 --steps $2 --warmup 2 --no-e2e --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$3', 'c$1', d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['parity'] and d['parity']['max_rel'])"; }
for rep in 1 2; do
  GG_I8_QUAD=0 run 3 4 dual
  GG_I8_QUAD=1 GG_I8_QUAD_ILV=0 run 3 4 quad
  GG_I8_QUAD=1 GG_I8_QUAD_ILV=1 run 3 4 quad-ilv
done
for rep in 1 2; do
  GG_I8_QUAD=0 run 1 10 dual
  GG_I8_QUAD=1 GG_I8_QUAD_ILV=1 run 1 10 quad-ilv
done
