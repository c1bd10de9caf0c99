# reading R40 (multiplier hold) experiments: d = 40 / 80 sanity, then d = 100 variants concurrently
mkdir -p gpurun_out
python -m paper_2512_04406_b200.build > /dev/null
run() { tag=$1; shift; DRSDP_VERBOSE=1 timeout $T python tools/solve_run.py "$@" > gpurun_out/r2H_$tag.log 2> gpurun_out/r2H_$tag.err; }
T=300 run d80h 80 240 4 hold_max=10 hold_tau=1e-2 escape_max=32 stall_factor=10.0
T=300 run d80h3 80 240 4 hold_max=10 hold_tau=1e-3 escape_max=64 stall_factor=10.0
for t in d80h d80h3; do echo "== $t"; tail -1 gpurun_out/r2H_$t.log | cut -c1-400; done
T=3000 run H1 100 2900 4 hold_max=10 hold_tau=1e-2 escape_max=32 stall_factor=10.0 &
T=3000 run H2 100 2900 4 hold_max=10 hold_tau=1e-3 escape_max=64 stall_factor=10.0 &
T=3000 run C1 100 2900 4 escape_max=64 stall_factor=10.0 &
wait
for t in H1 H2 C1; do echo "== $t"; tail -1 gpurun_out/r2H_$t.log | cut -c1-400; grep "k=" gpurun_out/r2H_$t.err | tail -2 | cut -c1-300; done
