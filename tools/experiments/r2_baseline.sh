# round-2 re-entry: full -m gpu suite, bench line, ncu launch list, one --set full capture
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2_pytest_gpu.log 2>&1; tail -3 gpurun_out/r2_pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -c 400 gpurun_out/r2_bench.json; tail -3 gpurun_out/r2_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 5 --warmup 3 --no-sweep --no-solve --no-cpu-baseline --no-full-oracle > gpurun_out/r2_ncu_launch.log 2>&1; tail -2 gpurun_out/r2_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:symv_tma -s 6 -c 2 -o gpurun_out/r2_symv_tma_full \
  python bench.py --steps 3 --warmup 3 --no-sweep --no-solve --no-cpu-baseline --no-full-oracle > gpurun_out/r2_ncu_full.log 2>&1; tail -2 gpurun_out/r2_ncu_full.log
