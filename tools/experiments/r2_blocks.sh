# f2 (multi-block clique-chain relaxation): GPU parity, chain solves, block evaluation timings
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_blocks.py -x -q > gpurun_out/r2_blocks_tests.log 2>&1; tail -15 gpurun_out/r2_blocks_tests.log
timeout 300 python tools/alm_profile.py chain:20:120 2,8,16,32 30 > gpurun_out/r2_blocks_prof.log 2>&1; cat gpurun_out/r2_blocks_prof.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --solve-d 10 --solve-chain 20:20,20:60,20:120,30:10 --solve-time-limit 300 > gpurun_out/r2_blocks_bench.json 2> gpurun_out/r2_blocks_bench.err; tail -3 gpurun_out/r2_blocks_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2_blocks_bench.json').read().strip().splitlines()[-1])
for s in d.get('chain_solves', []): print({k: s[k] for k in ('q','t','seconds','status','outer_iters','p_max','eta_p','eta_d','eta_g','dual_obj','n_hvp')})
"
# does DFMA co-issue with DMMA? (decides whether a mixed-pipe symmetric-half kernel can beat the DMMA bound)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/fp64_mixed tools/microbench/fp64_mixed.cu && ./gpurun_out/fp64_mixed > gpurun_out/r2_fp64_mixed.json; cat gpurun_out/r2_fp64_mixed.json; rm -f gpurun_out/fp64_mixed
# dense ALM evaluation at d = 80 (solve sizes): wall times and the ncu per-kernel launch list
timeout 300 python tools/alm_profile.py 80 16,128,240 20 > gpurun_out/r2_alm80.log 2>&1; cat gpurun_out/r2_alm80.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_alm80_launches.csv \
    python tools/alm_profile.py 80 16,128,240 2 > gpurun_out/r2_alm80_ncu.log 2>&1; tail -1 gpurun_out/r2_alm80_ncu.log
