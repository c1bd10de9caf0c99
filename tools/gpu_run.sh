mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
DRSDP_VERBOSE=1 timeout 900 python tools/solve_run.py 150 600 16 escape_max=16 > gpurun_out/solve_150.log 2> gpurun_out/solve_150.err; tail -4 gpurun_out/solve_150.err; grep '"d"' gpurun_out/solve_150.log | cut -c1-300
