# certified d = 150 solve alone on the GPU (clean solve time next to the certificate)
mkdir -p gpurun_out
DRSDP_LONG=1 DRSDP_VERBOSE=1 timeout 2300 python -m pytest tests/test_long_solves.py -m gpu -s -q -k "150" > gpurun_out/r2S_long150.log 2> gpurun_out/r2S_long150.err
tail -3 gpurun_out/r2S_long150.log | cut -c1-700
