mkdir -p gpurun_out
DRSDP_VERBOSE=1 timeout 2800 python tools/solve_run.py 100 2700 4 > gpurun_out/solve_r34_100_long.log 2> gpurun_out/solve_r34_100_long_v.log
tail -1 gpurun_out/solve_r34_100_long.log | cut -c1-420
