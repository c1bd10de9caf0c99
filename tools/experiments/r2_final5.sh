# final build (matrix-light HVP product off by default after the race finding): full -m gpu suite, smoke, default
# bench; then, for information, the bitwise-repeatability test and two d = 70 solves with DRSDP_FUSED_GATHER=1 (4 gather warps)
mkdir -p gpurun_out
( time timeout 1800 python -m pytest tests -m gpu -q -x --durations=5 ) > gpurun_out/r2Z_pytest_gpu.log 2>&1; tail -12 gpurun_out/r2Z_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2Z_smoke.log 2>&1; tail -2 gpurun_out/r2Z_smoke.log
( time timeout 1500 python bench.py ) > gpurun_out/r2Z_bench.json 2> gpurun_out/r2Z_bench.err; tail -c 300 gpurun_out/r2Z_bench.json; grep "\[bench\]" gpurun_out/r2Z_bench.err | tail -12
DRSDP_FUSED_GATHER=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "bitwise_repeatable" > gpurun_out/r2Z_bitwise_on_ngw4.log 2>&1; tail -6 gpurun_out/r2Z_bitwise_on_ngw4.log | cut -c1-300
for i in 1 2; do DRSDP_FUSED_GATHER=1 timeout 200 python tools/solve_run.py 70 150 4 2>/dev/null | tail -1 | cut -c1-200; done
