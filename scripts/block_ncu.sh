# per-kernel launch times of one block CG iteration on C4 (ncu launch list; R5)
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:bcg_ -s 40 -c 14 --csv --log-file gpurun_out/block_ncu.csv \
  python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --solver block > gpurun_out/block_ncu.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/block_ncu.csv')) if len(r)>14 and r[0]!='ID']
cur={}
for r in rows:
    cur.setdefault((r[0], r[4][:60]), {})[r[12]] = r[14]
for (i,k),v in cur.items():
    print(i, k, v.get('gpu__time_duration.sum'), v.get('dram__bytes_read.sum'), v.get('dram__bytes_write.sum'))
PY
