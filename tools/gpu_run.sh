mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
DRSDP_VERBOSE=1 timeout 900 python tools/solve_run.py 150 720 32 sigma0=10.0 sigma_min=10.0 escape_max=32 > gpurun_out/exp_D150.log 2> gpurun_out/exp_D150.err; tail -2 gpurun_out/exp_D150.err | cut -c1-300
