# f1: matrix-light HVP product (symv_gather.cu) — parity, then A/B timing against the dense A*(w) path
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "alm_eval" > gpurun_out/r2G_parity.log 2>&1; tail -3 gpurun_out/r2G_parity.log
for d in 80 100; do
  for fg in 0 1 2; do
    echo "== d=$d DRSDP_FUSED_GATHER=$fg"
    DRSDP_FUSED_GATHER=$fg timeout 300 python tools/alm_profile.py $d 8,16,32,64,128,256 30 2>&1 | tail -6
  done
done > gpurun_out/r2G_ab.log 2>&1
cat gpurun_out/r2G_ab.log
