mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hbm or extreme or long_fast or one_layer or hot_shape" > gpurun_out/g3_pt.log 2>&1; echo "rc=$?" >> gpurun_out/g3_pt.log
timeout 900 python -m pytest tests/test_gpu_launch_modes.py -q -x >> gpurun_out/g3_pt.log 2>&1; echo "rc=$?" >> gpurun_out/g3_pt.log
timeout 300 python tools/ls_trace.py 1 8 > gpurun_out/g3_ls_trace.txt 2>&1
timeout 400 python bench.py --layer-sequential --slow-tier device --no-cpu-baseline 2>>gpurun_out/g3.err | tail -1 > gpurun_out/g3_ls_spec.json
TTKV_SPEC=0 timeout 400 python bench.py --layer-sequential --slow-tier device --no-cpu-baseline 2>>gpurun_out/g3.err | tail -1 > gpurun_out/g3_ls_union.json
