# fused kernel: 1 CTA/SM 4-stage ring vs 2 CTAs/SM 2-stage rings (DRSDP_BOTH_DUO), bench step only
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or full_size_sampled" > gpurun_out/r2duo_tests0.log 2>&1; tail -1 gpurun_out/r2duo_tests0.log
DRSDP_BOTH_DUO=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or full_size_sampled" > gpurun_out/r2duo_tests1.log 2>&1; tail -1 gpurun_out/r2duo_tests1.log
for v in 0 1 0 1; do
DRSDP_BOTH_DUO=$v timeout 300 python bench.py --steps 100 --warmup 5 --no-sweep --no-solve --no-cpu-baseline --no-full-oracle > gpurun_out/r2duo_$v.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2duo_$v.json').read().strip().splitlines()[-1])
print('DUO=$v', round(d['value'],1), round(d['roofline']['per_launch_ms'],4), round(d['roofline']['frac'],4), d['clocks'])"
done
# DMMA block product: block parity and chain timings
timeout 900 python -m pytest tests/test_gpu_blocks.py -x -q > gpurun_out/r2duo_blocks.log 2>&1; tail -2 gpurun_out/r2duo_blocks.log
timeout 300 python tools/alm_profile.py chain:20:120 2,16,64,128 30 2>&1 | tail -4
timeout 300 python tools/alm_profile.py chain:20:20 16 30 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --solve-d 10 --solve-chain 20:20,20:120,40:10 --solve-time-limit 200 > gpurun_out/r2duo_chain.json 2> gpurun_out/r2duo_chain.err; grep "\[bench\]" gpurun_out/r2duo_chain.err
