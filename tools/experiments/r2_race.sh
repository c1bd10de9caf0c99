# bitwise repeatability of the matrix-light HVP product (race check), then the extra ncu evidence
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "bitwise_repeatable" > gpurun_out/r2R_bitwise_on.log 2>&1; tail -8 gpurun_out/r2R_bitwise_on.log | cut -c1-300
DRSDP_FUSED_GATHER=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "bitwise_repeatable" > gpurun_out/r2R_bitwise_off.log 2>&1; tail -3 gpurun_out/r2R_bitwise_off.log | cut -c1-300
for i in 1 2; do DRSDP_FUSED_GATHER=1 timeout 200 python tools/solve_run.py 70 150 4 2>/dev/null | tail -1 | cut -c1-200; done
for i in 1 2; do DRSDP_FUSED_GATHER=0 timeout 200 python tools/solve_run.py 70 150 4 2>/dev/null | tail -1 | cut -c1-200; done
bash tools/experiments/r2_extra.sh
