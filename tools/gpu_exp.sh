mkdir -p gpurun_out
DRSDP_VERBOSE=1 timeout 800 python tools/solve_run.py 100 700 32 sigma0=10.0 sigma_min=10.0 escape_max=64 > gpurun_out/exp_D100d.log 2> gpurun_out/exp_D100d.err; tail -2 gpurun_out/exp_D100d.err | cut -c1-300
