# per-kernel device times of the ALM cost+grad / HVP at d = 100 (p = 16, 128) after the gram-tile /
# gather-assemble changes (ncu launch list; cold-cache, serialised)
mkdir -p gpurun_out
python tools/alm_profile.py 100 16,128 2 > gpurun_out/r2d_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_alm100_launches.csv \
    python tools/alm_profile.py 100 16,128 2 > gpurun_out/r2d_ncu.log 2>&1; tail -2 gpurun_out/r2d_ncu.log
