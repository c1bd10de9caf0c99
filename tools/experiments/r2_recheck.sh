# re-entry check: full -m gpu suite, smoke, default bench line
mkdir -p gpurun_out
python -c "import torch; print(torch.cuda.get_device_name(0))"
( time timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 ) > gpurun_out/r2G_pytest_gpu.log 2>&1; tail -25 gpurun_out/r2G_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2G_smoke.log 2>&1; tail -2 gpurun_out/r2G_smoke.log
( time timeout 1500 python bench.py ) > gpurun_out/r2G_bench.json 2> gpurun_out/r2G_bench.err; tail -c 300 gpurun_out/r2G_bench.json; grep "\[bench\]" gpurun_out/r2G_bench.err | tail -30; tail -4 gpurun_out/r2G_bench.err
