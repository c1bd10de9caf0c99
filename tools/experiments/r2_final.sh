# round-end evidence: full -m gpu suite, default bench line, ncu launch list + --set full of the fused kernel
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2F_pytest_gpu.log 2>&1; tail -3 gpurun_out/r2F_pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/r2F_bench.json 2> gpurun_out/r2F_bench.err; tail -c 300 gpurun_out/r2F_bench.json; grep "\[bench\]" gpurun_out/r2F_bench.err; tail -2 gpurun_out/r2F_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2F_launches.csv \
  python bench.py --steps 5 --warmup 3 --no-sweep --no-solve --no-cpu-baseline --no-full-oracle > gpurun_out/r2F_ncu_launch.log 2>&1; tail -1 gpurun_out/r2F_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:symv_tma -s 3 -c 2 -o gpurun_out/r2F_symv_tma_full \
  python bench.py --steps 3 --warmup 3 --no-sweep --no-solve --no-cpu-baseline --no-full-oracle > gpurun_out/r2F_ncu_full.log 2>&1; tail -1 gpurun_out/r2F_ncu_full.log
