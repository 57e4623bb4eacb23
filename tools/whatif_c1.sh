# config-1 what-ifs of the int8 TRSM (timing only; results invalid for whatif != 0)
run() { python bench.py --config 1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('whatif=$1', d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"; }
for rep in 1 2; do for w in 0 1 2 4 6 7; do GG_I8_WHATIF=$w run $w; done; done
