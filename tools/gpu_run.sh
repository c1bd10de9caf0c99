mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/solve_run.py 10,20,40 120 > gpurun_out/solve_rep.log 2>&1; grep '"d"' gpurun_out/solve_rep.log | cut -c1-230
timeout 200 python tools/quick_sweep.py 16384,32768 16,64 > gpurun_out/sweep_tma.log 2>&1; cut -c1-140 gpurun_out/sweep_tma.log
