# d = 80 regression hunt: eigen step (Lanczos vs dense) x tCG preconditioner (R35)
mkdir -p gpurun_out
run() { tag=$1; shift; DRSDP_VERBOSE=1 timeout 400 python tools/solve_run.py "$@" > gpurun_out/r2v_$tag.log 2> gpurun_out/r2v_$tag.err; tail -1 gpurun_out/r2v_$tag.log | cut -c1-330; }
run A 80 300 4
run B 80 300 4 eig_method=1
run C 80 300 4 eig_method=1 precond_mu=0.0
run D 80 300 4 precond_mu=0.0
run E 40 300 4 eig_method=2
