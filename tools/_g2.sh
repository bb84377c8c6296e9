mkdir -p gpurun_out
timeout 300 python tools/ls_trace.py 1 8 > gpurun_out/g2_ls_trace.txt 2>&1
TTKV_FUSED_SELECT=0 timeout 300 python tools/ls_trace.py 1 8 > gpurun_out/g2_ls_trace_nofused.txt 2>&1
./build/fused_probe 8 992 4 > gpurun_out/g2_fused_probe.txt 2>&1
