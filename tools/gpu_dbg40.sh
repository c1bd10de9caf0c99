mkdir -p gpurun_out
DRSDP_DEBUG_RTR=1 timeout 300 python tools/solve_run.py 40 200 4 max_outer=21 max_rtr=80 > gpurun_out/solve_40_dbg.log 2> gpurun_out/solve_40_dbg.err
tail -3 gpurun_out/solve_40_dbg.log | cut -c1-200
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_d40.csv python tools/solve_run.py 40 2 > gpurun_out/ncu_d40.log 2>&1
tail -2 gpurun_out/ncu_d40.log
