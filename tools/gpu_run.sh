mkdir -p gpurun_out
i=0
for args in "escape_max=32" "mode=1" "escape_max=32 mode=1"; do
  i=$((i+1))
  DRSDP_VERBOSE=1 timeout 560 python tools/solve_run.py 100 480 4 $args > gpurun_out/x100_$i.log 2> gpurun_out/x100_${i}_v.log
  echo "$args"; tail -1 gpurun_out/x100_$i.log | cut -c1-420
done
