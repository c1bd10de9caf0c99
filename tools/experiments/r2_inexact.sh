# inexact inner solves (a few trust-region iterations per outer iteration, as the paper's iteration counts and
# times imply: ~100 HVPs per outer iteration at q = 80): d = 40 / 80 sanity, then d = 100 variants concurrently
mkdir -p gpurun_out
run() { tag=$1; shift; DRSDP_VERBOSE=1 timeout $T python tools/solve_run.py "$@" > gpurun_out/r2I_$tag.log 2> gpurun_out/r2I_$tag.err; }
summ() { for t in "$@"; do echo "== $t"; tail -1 gpurun_out/r2I_$t.log | cut -c1-330; grep "k=" gpurun_out/r2I_$t.err | tail -1 | cut -c1-250; done; }
T=150 run a40 40 120 4 max_rtr=4 max_tcg=50 max_outer=3000 &
T=150 run d40 40 120 4 max_rtr=4 max_tcg=20 max_outer=3000 &
T=150 run a80 80 140 4 max_rtr=4 max_tcg=50 max_outer=3000 &
T=150 run d80 80 140 4 max_rtr=4 max_tcg=20 max_outer=3000 &
T=150 run c80 80 140 4 max_rtr=10 max_tcg=100 max_outer=3000 &
wait; summ a40 d40 a80 d80 c80
T=1000 run a100 100 900 4 max_rtr=4 max_tcg=50 max_outer=20000 &
T=1000 run d100 100 900 4 max_rtr=4 max_tcg=20 max_outer=20000 &
T=1000 run c100 100 900 4 max_rtr=10 max_tcg=100 max_outer=20000 &
T=1000 run e100 100 900 16 max_rtr=4 max_tcg=50 escape_max=16 max_outer=20000 &
wait; summ a100 d100 c100 e100
