# chain solve traces (q = 20, t = 10 / 20) then d = 100 variants (escape gate R36, stall factor R30)
mkdir -p gpurun_out
run() { tag=$1; shift; DRSDP_VERBOSE=1 timeout 700 python tools/solve_run.py "$@" > gpurun_out/r2_$tag.log 2> gpurun_out/r2_$tag.err; tail -1 gpurun_out/r2_$tag.log | cut -c1-420; grep "\[drsdp\]" gpurun_out/r2_$tag.err | tail -2 | cut -c1-300; }
run chain10 chain:20:10 200 2
run chain20 chain:20:20 200 2
run d100_g10 100 540 4 escape_gate=10.0
run d100_s10 100 540 4 stall_factor=10.0
run d100_g10s10 100 540 4 escape_gate=10.0 stall_factor=10.0
