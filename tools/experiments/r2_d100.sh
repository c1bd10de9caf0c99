# d = 100 (BASELINE configs[2]) with the dense eigen step + Gram-preconditioned tCG (new defaults)
mkdir -p gpurun_out
DRSDP_VERBOSE=1 timeout 1900 python tools/solve_run.py 100 1800 4 > gpurun_out/r2_d100_a.log 2> gpurun_out/r2_d100_a.err; tail -1 gpurun_out/r2_d100_a.log | cut -c1-400
