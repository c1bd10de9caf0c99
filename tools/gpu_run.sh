mkdir -p gpurun_out
for d in 100 80; do
  DRSDP_VERBOSE=1 timeout 1300 python tools/solve_run.py $d 1200 > gpurun_out/solve_r34_$d.log 2> gpurun_out/solve_r34_${d}_v.log
  tail -1 gpurun_out/solve_r34_$d.log | cut -c1-400
done
