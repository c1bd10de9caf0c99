# round-end evidence (session 5): full -m gpu suite, smoke, default bench line, f1 A/B timing (dense A*(w) vs the
# matrix-light product), ncu launch list of the bench + --set full of symv_gather and the fused graded kernel
mkdir -p gpurun_out
( time timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 ) > gpurun_out/r2H_pytest_gpu.log 2>&1; tail -18 gpurun_out/r2H_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2H_smoke.log 2>&1; tail -2 gpurun_out/r2H_smoke.log
( time timeout 1500 python bench.py ) > gpurun_out/r2H_bench.json 2> gpurun_out/r2H_bench.err; tail -c 300 gpurun_out/r2H_bench.json; grep "\[bench\]" gpurun_out/r2H_bench.err | tail -30; tail -4 gpurun_out/r2H_bench.err
for d in 80 100; do
  for fg in 0 1; do
    echo "== d=$d DRSDP_FUSED_GATHER=$fg"
    DRSDP_FUSED_GATHER=$fg timeout 300 python tools/alm_profile.py $d 8,16,32,64 30 2>&1 | tail -5
  done
done > gpurun_out/r2H_gather_ab.log 2>&1
cat gpurun_out/r2H_gather_ab.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2H_launches.csv \
  python bench.py --steps 5 --warmup 3 --no-sweep --no-solve --no-cpu-baseline --no-full-oracle > gpurun_out/r2H_ncu_launch.log 2>&1; tail -1 gpurun_out/r2H_ncu_launch.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:symv_gather -s 4 -c 2 -o gpurun_out/r2H_symv_gather_full \
  python tools/alm_profile.py 100 16 2 > gpurun_out/r2H_ncu_gather.log 2>&1; tail -1 gpurun_out/r2H_ncu_gather.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2H_alm100_launches.csv \
  python tools/alm_profile.py 100 16 3 > gpurun_out/r2H_ncu_alm_launch.log 2>&1; tail -1 gpurun_out/r2H_ncu_alm_launch.log
