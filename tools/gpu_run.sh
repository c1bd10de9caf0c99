mkdir -p gpurun_out
DRSDP_SYMM16=1 timeout 200 python tools/quick_sweep.py 16384,32768 16 > gpurun_out/sweep_s16.log 2>&1; cut -c1-110 gpurun_out/sweep_s16.log
DRSDP_SYMM16=1 timeout 300 python -m pytest tests -m gpu -x -q -k "upper_triangle or full_size_sampled" > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
