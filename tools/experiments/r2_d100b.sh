# d = 100: escape gate (R36) and stall factor (R30) variants, 540 s each
mkdir -p gpurun_out
run() { tag=$1; shift; DRSDP_VERBOSE=1 timeout 620 python tools/solve_run.py "$@" > gpurun_out/r2_d100_$tag.log 2> gpurun_out/r2_d100_$tag.err; tail -1 gpurun_out/r2_d100_$tag.log | cut -c1-420; grep "\[drsdp\]" gpurun_out/r2_d100_$tag.err | tail -2 | cut -c1-300; }
run g10 100 540 4 escape_gate=10.0
run s10 100 540 4 stall_factor=10.0
run g10s10 100 540 4 escape_gate=10.0 stall_factor=10.0
