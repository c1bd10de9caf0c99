# gram-tile / gather-assemble changes: ALM parity, timings; then compute-sanitizer racecheck
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "alm_eval or operator or solve_d10 or solve_d20 or preconditioned or lanczos_eigen" > gpurun_out/r2c_tests.log 2>&1; tail -2 gpurun_out/r2c_tests.log
python tools/alm_profile.py 100 16,128,512 10 > gpurun_out/r2c_alm100.log 2>&1; cat gpurun_out/r2c_alm100.log
python tools/alm_profile.py 80 16,128,240 30 > gpurun_out/r2c_alm80.log 2>&1; cat gpurun_out/r2c_alm80.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report analysis python tools/sanitize_cases.py > gpurun_out/r2c_racecheck.log 2>&1; tail -15 gpurun_out/r2c_racecheck.log
