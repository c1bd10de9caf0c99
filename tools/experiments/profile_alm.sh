# fp64 unit co-issue microbenchmark, ALM evaluation timings at d = 80 / 100, and the per-kernel
# launch list of a few ALM evaluations at d = 100 (p = 16, 128, 512)
mkdir -p gpurun_out
./tools/microbench/fp64_mixed > gpurun_out/r2_fp64_mixed.json 2>&1; cat gpurun_out/r2_fp64_mixed.json
python tools/alm_profile.py 80 16,128,240 30 > gpurun_out/r2_alm80.log 2>&1; cat gpurun_out/r2_alm80.log
python tools/alm_profile.py 100 16,128,512 10 > gpurun_out/r2_alm100.log 2>&1 && cat gpurun_out/r2_alm100.log &&
python tools/alm_profile.py 100 16,128,512 2 > gpurun_out/r2_alm100_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_alm100_launches.csv \
    python tools/alm_profile.py 100 16,128,512 2 > gpurun_out/r2_alm100_ncu.log 2>&1; tail -2 gpurun_out/r2_alm100_ncu.log
# upper-triangle product at p = 16 with V_I^T in registers (DRSDP_SYMM16=1) against the full read
DRSDP_SYMM16=1 python -m pytest tests -m gpu -q -x -k "upper_triangle or full_size_sampled" > gpurun_out/r2_symm16_tests.log 2>&1; tail -2 gpurun_out/r2_symm16_tests.log
python tools/quick_sweep.py 16384,32768 8,16 > gpurun_out/r2_sweep_full.log 2>&1; cat gpurun_out/r2_sweep_full.log
DRSDP_SYMM16=1 python tools/quick_sweep.py 16384,32768 8,16 > gpurun_out/r2_sweep_symm16.log 2>&1; cat gpurun_out/r2_sweep_symm16.log
# trust-region trace of the first outer iterations at d = 100 (accept / reject, radius, tCG exits)
DRSDP_VERBOSE=1 DRSDP_DEBUG_RTR=1 timeout 300 python tools/solve_run.py 100 120 4 precond_mu=0.1 max_outer=4 > gpurun_out/r2_d100_rtrdbg.log 2> gpurun_out/r2_d100_rtrdbg.err; grep -c rtr gpurun_out/r2_d100_rtrdbg.err
