mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rA > gpurun_out/pt.log 2>&1; grep -E "passed|failed|FAILED|objects|background|rel L2|^E  " gpurun_out/pt.log | tail -30
