mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 200 python tools/quick_sweep.py 16384,32768 16,32,64 > gpurun_out/sweep.log 2>&1; cut -c1-110 gpurun_out/sweep.log
timeout 200 python tools/solve_run.py 10,40,10,40 60 > gpurun_out/solve_rep.log 2>&1; grep '"d"' gpurun_out/solve_rep.log | cut -c1-170
