# reading R39 v2 (per-block escape columns) + unrolled segsum: block parity, chain traces, ncu captures
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_blocks.py tests/test_gpu_parity.py -x -q -k "block or chain or alm_eval or operator or solve_d10 or solve_d20" > gpurun_out/r2c2_tests.log 2>&1; tail -3 gpurun_out/r2c2_tests.log
run() { tag=$1; shift; DRSDP_VERBOSE=1 timeout 400 python tools/solve_run.py "$@" > gpurun_out/r2_$tag.log 2> gpurun_out/r2_$tag.err; tail -1 gpurun_out/r2_$tag.log | cut -c1-400; }
run c2_chain20 chain:20:20 300 2
run c2_chain60 chain:20:60 300 2
run c2_chain120 chain:20:120 300 2
timeout 300 python tools/alm_profile.py chain:20:120 2,16,64 30 > gpurun_out/r2c2_prof120.log 2>&1; cat gpurun_out/r2c2_prof120.log
timeout 300 python tools/alm_profile.py 80 16,128 20 > gpurun_out/r2c2_alm80.log 2>&1; cat gpurun_out/r2c2_alm80.log
bash tools/experiments/r2_ncu_more.sh
