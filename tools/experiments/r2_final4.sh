# round-end re-verification of the final build (NVTX ranges, reading R41, DRSDP_MAX_P 4096): full -m gpu suite,
# smoke, default bench line; trajectory sensitivity of the d = 60 / 70 / 80 solves to the matrix-light HVP product;
# an NVTX-filtered launch list of the truncated-CG phase
mkdir -p gpurun_out
( time timeout 1800 python -m pytest tests -m gpu -q -x --durations=5 ) > gpurun_out/r2K_pytest_gpu.log 2>&1; tail -12 gpurun_out/r2K_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2K_smoke.log 2>&1; tail -2 gpurun_out/r2K_smoke.log
( time timeout 1500 python bench.py ) > gpurun_out/r2K_bench.json 2> gpurun_out/r2K_bench.err; tail -c 300 gpurun_out/r2K_bench.json; grep "\[bench\]" gpurun_out/r2K_bench.err | tail -12
for fg in 0 1; do
  for d in 60 70 80; do
    echo "== d=$d DRSDP_FUSED_GATHER=$fg"
    DRSDP_FUSED_GATHER=$fg timeout 200 python tools/solve_run.py $d 150 4 2>/dev/null | tail -1 | cut -c1-330
  done
done > gpurun_out/r2K_gather_solves.log 2>&1
cat gpurun_out/r2K_gather_solves.log
for sb in 1e-3 1e-2; do
  echo "== sigma_boost=$sb d=40,60,80"
  timeout 400 python tools/solve_run.py 40,60,80 150 4 sigma_boost=$sb 2>/dev/null | grep '^{' | cut -c1-330
done > gpurun_out/r2K_boost_solves.log 2>&1
cat gpurun_out/r2K_boost_solves.log
timeout 600 ncu --nvtx --nvtx-include "drsdp:tcg/" --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/r2K_nvtx_tcg_launches.csv python tools/solve_run.py 40 60 4 > gpurun_out/r2K_nvtx.log 2>&1; tail -1 gpurun_out/r2K_nvtx.log | cut -c1-200
