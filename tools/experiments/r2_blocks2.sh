# f2 after the dense block tiles for the segmented sums: parity, timings, launch list, chain solves
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_blocks.py -x -q > gpurun_out/r2b2_tests.log 2>&1; tail -3 gpurun_out/r2b2_tests.log
timeout 300 python tools/alm_profile.py chain:20:120 2,8,16,32,64 30 > gpurun_out/r2b2_prof120.log 2>&1; cat gpurun_out/r2b2_prof120.log
timeout 300 python tools/alm_profile.py chain:20:20 2,8,16 30 > gpurun_out/r2b2_prof20.log 2>&1; cat gpurun_out/r2b2_prof20.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b2_chain_launches.csv \
    python tools/alm_profile.py chain:20:120 16 2 > gpurun_out/r2b2_ncu.log 2>&1; tail -1 gpurun_out/r2b2_ncu.log
timeout 1000 python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --solve-d 10 --solve-chain 20:20,20:60,20:120 --solve-time-limit 240 > gpurun_out/r2b2_bench.json 2> gpurun_out/r2b2_bench.err; grep "\[bench\]" gpurun_out/r2b2_bench.err
