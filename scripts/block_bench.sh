# N3 block CG vs the independent multi-RHS solves on C4 (k = 16), one B200 (R5)
for s in pcg block; do
  python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --solver $s 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print('$s', round(d['value'],4), c['iterations'], round(d['roofline']['frac'],3), round(d['roofline']['achieved']), d['e2e']['value'])"
done
