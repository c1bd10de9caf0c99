mkdir -p gpurun_out
DRSDP_VERBOSE=1 timeout 800 python tools/solve_run.py 100 660 32 sigma0=10.0 sigma_min=10.0 escape_max=32 max_tcg=1000 > gpurun_out/exp_D100f.log 2> gpurun_out/exp_D100f.err; tail -2 gpurun_out/exp_D100f.err | cut -c1-300
