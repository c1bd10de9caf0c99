# BASELINE configs[3] (d = 150 Erdos-Renyi): certified solve (oracle-recomputed residues, rounding certificate)
mkdir -p gpurun_out
DRSDP_LONG=1 DRSDP_VERBOSE=1 timeout 3500 python -m pytest tests/test_long_solves.py -m gpu -x -q -s -k "150" > gpurun_out/r2_long150.log 2> gpurun_out/r2_long150.err; tail -5 gpurun_out/r2_long150.log | cut -c1-600
