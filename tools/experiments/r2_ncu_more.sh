# ncu --set full captures beyond the graded kernel: ALM evaluation kernels at d = 100 (p = 16, 128),
# the upper-triangle product at p = 8, the multi-block kernels at q = 20, t = 120
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_tile|segsum|assemble_alm|gather_assemble|symv_tma_kernel" -s 12 -c 10 \
  -o gpurun_out/r2_alm100_full python tools/alm_profile.py 100 16,128 2 > gpurun_out/r2_alm100_full.log 2>&1; tail -1 gpurun_out/r2_alm100_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"symm_" -s 4 -c 4 \
  -o gpurun_out/r2_symm_full python bench.py --steps 2 --warmup 3 --p 8 --no-sweep --no-solve --no-cpu-baseline --no-full-oracle > gpurun_out/r2_symm_full.log 2>&1; tail -1 gpurun_out/r2_symm_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"blk_|segsum" -s 10 -c 8 \
  -o gpurun_out/r2_chain_full python tools/alm_profile.py chain:20:120 16 2 > gpurun_out/r2_chain_full.log 2>&1; tail -1 gpurun_out/r2_chain_full.log
