mkdir -p gpurun_out
DRSDP_VERBOSE=1 timeout 1150 python tools/solve_run.py 100 1080 4 sigma0=16.0 > gpurun_out/z100.log 2> gpurun_out/z100_v.log
tail -1 gpurun_out/z100.log | cut -c1-420
