mkdir -p gpurun_out/gj5
SFM_B200_LIB=$PWD/paper_2510_15271_b200/variants/gjp.so timeout 300 python tools/pcg_sweep.py 3 2 1e-8:8 > gpurun_out/gj5/log.txt 2>&1
timeout 300 python tools/pcg_sweep.py 3 8 1e-8:8 > gpurun_out/gj5/sweep.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "pcg or config3 or sharded or camera_kinds" 2>&1 | tail -2
