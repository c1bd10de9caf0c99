mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "fixed_eval or operator or alm" > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
timeout 200 python tools/quick_sweep.py 16384,32768 8,16,32,64 > gpurun_out/sweep_tma.log 2>&1; cat gpurun_out/sweep_tma.log | cut -c1-150
DRSDP_NO_TMA=1 timeout 100 python tools/quick_sweep.py 32768 16,64 > gpurun_out/sweep_old.log 2>&1; cat gpurun_out/sweep_old.log | cut -c1-150
timeout 200 python tools/eig_time.py 821,5051,11326 2>&1 | tail -3
