mkdir -p gpurun_out
DRSDP_VERBOSE=1 timeout 700 python tools/solve_run.py 100 600 8 sigma0=10.0 sigma_min=10.0 > gpurun_out/exp_D100c.log 2> gpurun_out/exp_D100c.err; tail -2 gpurun_out/exp_D100c.err | cut -c1-300
