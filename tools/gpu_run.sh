mkdir -p gpurun_out
timeout 200 python tools/quick_sweep.py 4096,16384,32768 8 > gpurun_out/sweep.log 2>&1; cut -c1-110 gpurun_out/sweep.log
timeout 600 python -m pytest tests -m gpu -x -q -k "upper_triangle" > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
