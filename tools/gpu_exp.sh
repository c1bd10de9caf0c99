mkdir -p gpurun_out
timeout 200 python tools/solve_run.py 10,20,40 100 > gpurun_out/solve_rep.log 2>&1; grep '"d"' gpurun_out/solve_rep.log | cut -c1-200
DRSDP_VERBOSE=1 timeout 800 python tools/solve_run.py 100 700 8 > gpurun_out/exp_D100b.log 2> gpurun_out/exp_D100b.err; tail -2 gpurun_out/exp_D100b.err | cut -c1-300
