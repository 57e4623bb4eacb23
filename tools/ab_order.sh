for rep in 1 2; do for o in 0 1; do
  GG_I8_ORDER=$o python bench.py --config 1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('c1 order=$o', d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"
done; done
for rep in 1 2; do for o in 0 1; do
  GG_I8_ORDER=$o python bench.py --config 3 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('c3 order=$o', d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['parity'])"
done; done
