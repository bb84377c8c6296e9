./build/fused_probe 8 992 4 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_launch_modes.py -q -x 2>&1 | tail -2
for sr in 1 0; do
TTKV_SCORE_ROWS=$sr timeout 300 python tools/hbm_step.py 256 131072 6 4 | sed "s/^/ROWS=$sr /"
TTKV_SCORE_ROWS=$sr timeout 300 python tools/hbm_step.py 4096 32768 3 4 | sed "s/^/ROWS=$sr /"
done
timeout 300 python tools/ls_trace.py 1 8 2>&1 | tail -6
