# tightness diagnostic: solves started from the tabu-search vertex (tools/experiments/vertex_start.py)
mkdir -p gpurun_out
DRSDP_VERBOSE=1 timeout 200 python tools/experiments/vertex_start.py 80 150 > gpurun_out/r2V_80.log 2> gpurun_out/r2V_80.err &
DRSDP_VERBOSE=1 timeout 800 python tools/experiments/vertex_start.py 100 700 > gpurun_out/r2V_100.log 2> gpurun_out/r2V_100.err &
DRSDP_VERBOSE=1 timeout 800 python tools/experiments/vertex_start.py 100 700 escape_max=32 > gpurun_out/r2V_100e32.log 2> gpurun_out/r2V_100e32.err &
wait
for t in 80 100 100e32; do echo "== $t"; head -1 gpurun_out/r2V_$t.log; tail -1 gpurun_out/r2V_$t.log | cut -c1-420; grep "k=" gpurun_out/r2V_$t.err | tail -2 | cut -c1-300; done
