# fused cost+grad+HVP (EPI_BOTH): parity, then the bench line, launch list and one ncu --set full capture
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_sharded.py -x -q -k "fixed or fused or host or row_blocks or abi" > gpurun_out/r2both_tests.log 2>&1; tail -3 gpurun_out/r2both_tests.log
timeout 900 python bench.py --no-solve --no-cpu-baseline --no-full-oracle > gpurun_out/r2both_bench.json 2> gpurun_out/r2both_bench.err; tail -c 300 gpurun_out/r2both_bench.json; tail -3 gpurun_out/r2both_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2both_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['clocks']); print(d['roofline'])
for s in d['sweep']: print(s['n'], s['p'], s['eval'], round(s['us'],1), round(s['tflops'],2))
"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2both_launches.csv \
  python bench.py --steps 5 --warmup 3 --no-sweep --no-solve --no-cpu-baseline --no-full-oracle > gpurun_out/r2both_ncu_launch.log 2>&1; tail -1 gpurun_out/r2both_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:symv_tma -s 3 -c 2 -o gpurun_out/r2both_full \
  python bench.py --steps 3 --warmup 3 --no-sweep --no-solve --no-cpu-baseline --no-full-oracle > gpurun_out/r2both_ncu_full.log 2>&1; tail -1 gpurun_out/r2both_ncu_full.log
