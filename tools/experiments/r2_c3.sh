# block kernels after the segsum / Gram latency fixes: parity, timing, chain bench lines; then racecheck
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_blocks.py -x -q > gpurun_out/r2c3_tests.log 2>&1; tail -2 gpurun_out/r2c3_tests.log
timeout 300 python tools/alm_profile.py chain:20:120 2,16,64,128 30 > gpurun_out/r2c3_prof120.log 2>&1; cat gpurun_out/r2c3_prof120.log
timeout 300 python tools/alm_profile.py 100 16,128 20 > gpurun_out/r2c3_alm100.log 2>&1; cat gpurun_out/r2c3_alm100.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --solve-d 10 --solve-chain 20:20,20:40,20:60,20:80,20:100,20:120,10:10,30:10,40:10 --solve-time-limit 120 > gpurun_out/r2c3_bench.json 2> gpurun_out/r2c3_bench.err; grep "\[bench\]" gpurun_out/r2c3_bench.err
bash tools/experiments/r2_sanitize.sh racecheck
