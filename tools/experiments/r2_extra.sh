# extra ncu evidence: launch list of the n = 4096, p = 16 step (launch-sequence bound) and --set full of gram_kernel
mkdir -p gpurun_out
timeout 300 python bench.py --n 4096 --p 16 --steps 50 --warmup 5 --no-sweep --no-solve --no-cpu-baseline --no-full-oracle > gpurun_out/r2X_bench4096.json 2> gpurun_out/r2X_bench4096.err; tail -c 400 gpurun_out/r2X_bench4096.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2X_launches4096.csv \
  python bench.py --n 4096 --p 16 --steps 5 --warmup 3 --no-sweep --no-solve --no-cpu-baseline --no-full-oracle > gpurun_out/r2X_ncu4096.log 2>&1; tail -1 gpurun_out/r2X_ncu4096.log | cut -c1-200
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gram_kernel|gram_final" -s 4 -c 4 -o gpurun_out/r2X_gram_full \
  python bench.py --steps 3 --warmup 3 --no-sweep --no-solve --no-cpu-baseline --no-full-oracle > gpurun_out/r2X_ncu_gram.log 2>&1; tail -1 gpurun_out/r2X_ncu_gram.log | cut -c1-200
