# certified d = 150 solve (tests/test_long_solves.py: oracle-recomputed residues + rank-one rounding certificate)
# next to a d = 100 run with the penalty boost of reading R41 (both share the GPU: wall times are inflated)
mkdir -p gpurun_out
( DRSDP_LONG=1 DRSDP_VERBOSE=1 timeout 4000 python -m pytest tests/test_long_solves.py -m gpu -s -q -k "150" > gpurun_out/r2L_long150.log 2> gpurun_out/r2L_long150.err ) &
( DRSDP_VERBOSE=1 timeout 3100 python tools/solve_run.py 100 3000 4 escape_max=64 sigma_boost=5e-4 max_outer=1000 > gpurun_out/r2L_boost100.log 2> gpurun_out/r2L_boost100.err ) &
wait
tail -5 gpurun_out/r2L_long150.log | cut -c1-600
tail -1 gpurun_out/r2L_boost100.log | cut -c1-420; grep "k=" gpurun_out/r2L_boost100.err | tail -3 | cut -c1-300
