# d = 80 / 100 solves with the Gram-preconditioned tCG (reading R35); one log per configuration
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "precond" > gpurun_out/r2_prec_tests.log 2>&1; tail -1 gpurun_out/r2_prec_tests.log
run() { tag=$1; shift; DRSDP_VERBOSE=1 timeout 720 python tools/solve_run.py "$@" > gpurun_out/r2_$tag.log 2> gpurun_out/r2_$tag.err; tail -1 gpurun_out/r2_$tag.log | cut -c1-400; }
run E1 80 300 4 precond_mu=0.01
run E2 80 300 4 precond_mu=0.1
run E3 100 600 4 precond_mu=0.01
run E4 100 600 4 precond_mu=0.1
run E5 100 600 4 precond_mu=0.01 sigma0=16.0 escape_max=16
