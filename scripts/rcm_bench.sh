set -e
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']; print(sys.argv[1], round(d['value'],4), c['iterations'], c['format'], c.get('setup_s'), round(d['roofline']['frac'],3), d['throughput']['effective_GBps'])" "$1"; }
for c in 128 256; do
python bench.py --config C6 --c $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | summ "C6c$c lattice"
python bench.py --config C6 --c $c --steps 5 --warmup 3 --no-cpu-baseline --reorder rcm 2>/dev/null | summ "C6c$c lattice+rcm"
python bench.py --config C6 --c $c --steps 5 --warmup 3 --no-cpu-baseline --relabel 7 2>/dev/null | summ "C6c$c random"
python bench.py --config C6 --c $c --steps 5 --warmup 3 --no-cpu-baseline --relabel 7 --reorder rcm 2>/dev/null | summ "C6c$c random+rcm"
done
