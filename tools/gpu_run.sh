mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "fixed_m_mode" > gpurun_out/pt.log 2>&1; tail -25 gpurun_out/pt.log | grep -E "assert|Error|passed|failed|where" | head -12
