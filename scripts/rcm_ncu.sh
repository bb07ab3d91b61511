# ncu evidence for N4: K1b DRAM bytes on C6 c=256, randomly numbered vs RCM-ordered.
# PCG_PERSIST=0 PCG_NO_GRAPH=1: the 3-pass schedule as direct launches (K1b a separate kernel ncu can see).
set -e
mkdir -p gpurun_out
for v in "random:--relabel 7" "rcm:--relabel 7 --reorder rcm"; do
  name=${v%%:*}; args=${v#*:}
  PCG_PERSIST=0 PCG_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:k1b_kernel -s 20 -c 1 --csv --log-file gpurun_out/rcm_ncu_$name.csv \
    python bench.py --config C6 --c 256 --steps 1 --warmup 3 --no-cpu-baseline $args > gpurun_out/rcm_ncu_$name.log 2>&1
done
