mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 400 python tools/alm_profile.py 80 16,64,128,240 30 2>&1 | tail -6
timeout 400 python tools/alm_profile.py 150 64,256,512 10 2>&1 | tail -4
