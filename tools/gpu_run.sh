mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 200 python tools/solve_run.py 10,40 120 > gpurun_out/solve_10_40.log 2>&1; grep '"d"' gpurun_out/solve_10_40.log | cut -c1-300
DRSDP_VERBOSE=1 timeout 500 python tools/solve_run.py 100 420 > gpurun_out/solve_100.log 2> gpurun_out/solve_100.err; tail -2 gpurun_out/solve_100.log | cut -c1-300; tail -5 gpurun_out/solve_100.err
