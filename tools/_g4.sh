mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hbm or extreme or long_fast or one_layer" > gpurun_out/g4_pt.log 2>&1; echo "rc=$?" >> gpurun_out/g4_pt.log
timeout 300 python tools/ls_trace.py 1 8 > gpurun_out/g4_ls_trace.txt 2>&1
for c in 3 2 1; do
TTKV_SPEC_CPS=$c timeout 400 python bench.py --layer-sequential --slow-tier device --no-cpu-baseline --steps 200 2>>gpurun_out/g4.err | tail -1 > gpurun_out/g4_ls_spec$c.json
done
TTKV_SPEC_CPS=2 timeout 300 python tools/ls_trace.py 1 8 > gpurun_out/g4_ls_trace2.txt 2>&1
