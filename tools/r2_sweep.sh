#!/usr/bin/env bash
# One B200, round 2: the parity suite and every bench line (writes
# gpurun_out/r2/; the committed profiles/r2_* files are copied from there).
#   gpurun --timeout 3600 -- 'bash tools/r2_sweep.sh'
set -x
O=gpurun_out/r2; mkdir -p $O
nvidia-smi --query-gpu=name,pci.bus_id,clocks.max.sm,clocks.max.mem --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu > $O/gpu_tests.txt 2>&1; echo "rc=$?" >> $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
B="timeout 600 python bench.py"
$B > $O/bench_cfg2.json 2> $O/bench_cfg2.err
$B --impl reference > $O/bench_reference_cfg2.json 2> $O/bench_reference_cfg2.err
$B --workload cfg1 > $O/bench_cfg1.json 2>> $O/bench.err
$B --workload cfg3 --no-cpu-baseline > $O/bench_cfg3.json 2>> $O/bench.err
$B --group-select --no-cpu-baseline > $O/bench_cfg2_gs.json 2>> $O/bench.err
for c in cfg1 cfg2 cfg3; do
  $B --workload $c --slow-tier device --no-cpu-baseline 2>> $O/bench.err | tail -1 > $O/bench_${c}_hbm.json
done
$B --layer-sequential --slow-tier device --no-cpu-baseline 2>> $O/bench.err | tail -1 > $O/bench_cfg2_layer_sequential_hbm.json
TTKV_SPEC=1 $B --layer-sequential --slow-tier device --no-cpu-baseline 2>> $O/bench.err | tail -1 > $O/bench_cfg2_layer_sequential_hbm_spec.json
$B --layer-sequential --no-cpu-baseline 2>> $O/bench.err | tail -1 > $O/bench_cfg2_layer_sequential.json
TTKV_SLOW_TC5=1 $B --slow-tier device --no-cpu-baseline 2>> $O/bench.err | tail -1 > $O/bench_cfg2_hbm_tcgen05.json
TTKV_SHARE_DEVICE=1 TTKV_DIST_BACKEND=gloo $B --gpus 2 --no-cpu-baseline 2>> $O/bench.err | tail -1 > $O/bench_n2_shared_device_gloo.json
timeout 900 python bench.py --workload cfg5 --no-cpu-baseline > $O/bench_cfg5.json 2>> $O/bench.err
echo done
