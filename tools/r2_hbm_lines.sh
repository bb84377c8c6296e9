#!/usr/bin/env bash
# One B200: the HBM-tier bench lines of both slow kernels on the same box
# (writes gpurun_out/r2h/; copied to profiles/r2_bench_*hbm*.json).
#   gpurun --timeout 2400 -- 'bash tools/r2_hbm_lines.sh'
set -x
O=gpurun_out/r2h; mkdir -p $O
B="timeout 600 python bench.py --no-cpu-baseline --slow-tier device"
for c in cfg1 cfg2 cfg3; do
  $B --workload $c 2>> $O/err | tail -1 > $O/bench_${c}_hbm.json
  TTKV_SLOW_TC5=1 $B --workload $c 2>> $O/err | tail -1 > $O/bench_${c}_hbm_tcgen05.json
done
$B --layer-sequential 2>> $O/err | tail -1 > $O/bench_cfg2_layer_sequential_hbm.json
TTKV_SLOW_TC5=1 $B --layer-sequential 2>> $O/err | tail -1 > $O/bench_cfg2_layer_sequential_hbm_tcgen05.json
TTKV_SPEC=1 $B --layer-sequential 2>> $O/err | tail -1 > $O/bench_cfg2_layer_sequential_hbm_spec.json
echo done
