mkdir -p gpurun_out
DRSDP_VERBOSE=1 timeout 800 python tools/solve_run.py 100 660 32 sigma0=10.0 sigma_min=10.0 escape_max=32 eps_scale=1.0 > gpurun_out/exp_D100e.log 2> gpurun_out/exp_D100e.err; tail -2 gpurun_out/exp_D100e.err | cut -c1-300
