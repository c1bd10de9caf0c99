mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "fixed_eval" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 200 python tools/quick_sweep.py 16384,32768 8,16 > gpurun_out/sweep_symm.log 2>&1; cut -c1-140 gpurun_out/sweep_symm.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:symm -c 20 --csv --log-file gpurun_out/launch_symm.csv python tools/quick_sweep.py 32768 16 > /dev/null 2>&1; python tools/ncu_summary.py launches gpurun_out/launch_symm.csv | head -5
