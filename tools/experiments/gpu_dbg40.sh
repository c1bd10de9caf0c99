mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 400 python tools/solve_run.py 10,40 300 > gpurun_out/solve_40.log 2>&1
tail -4 gpurun_out/solve_40.log | cut -c1-400
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_d40.csv python tools/solve_run.py 40 2 > gpurun_out/ncu_d40.log 2>&1
tail -2 gpurun_out/ncu_d40.log
