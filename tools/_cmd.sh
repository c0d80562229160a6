mkdir -p gpurun_out/e2e2
SFM_TIMING=1 timeout 600 python tools/e2e_breakdown.py 3 > gpurun_out/e2e2/log.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
