# round-end evidence: GPU suite, smoke, default bench, ncu launch list of the same command
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/final_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
tail -1 gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_bench_c5.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/final_bench_c5.log | cut -c1-400
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/final_launches_c5.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu_c5.log 2>&1; echo "ncu rc=$?"
