#!/usr/bin/env bash
# One B200: ncu captures of the round's dominant kernels + the launch list of
# the default bench command (read back here with tools/ncu_summary.py and
# tools/stamp_traffic.py).
#   gpurun --timeout 1800 -- 'bash tools/r2_profile.sh'
set -x
mkdir -p gpurun_out
NCU="ncu --clock-control none"
# launch list of the exact default bench command (cold cache, serialised)
$NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2_launches_cfg2.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_launches_cfg2.log 2>&1
# the PCIe-streaming slow kernel, one launch of the cfg2 bench step
$NCU --set full --import-source on -k regex:'slow_attn_kernel' -s 4 -c 1 -f \
  -o gpurun_out/r2_slow_cfg2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/r2_slow_cfg2.log 2>&1
# the HBM-resident tensor-core slow kernel, cfg2 with --slow-tier device
$NCU --set full --import-source on -k regex:'slow_attn_tc' -s 4 -c 1 -f \
  -o gpurun_out/r2_slowtc_cfg2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --slow-tier device > gpurun_out/r2_slowtc_cfg2.log 2>&1
echo done
