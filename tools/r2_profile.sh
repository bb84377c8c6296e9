#!/usr/bin/env bash
# One B200, round 2: ncu launch lists and full captures of the kernels the
# bench lines depend on, plus compute-sanitizer over tools/sanitize_subset.py
# (writes gpurun_out/r2p/; read back here with tools/ncu_summary.py and
# tools/stamp_traffic.py).
#   gpurun --timeout 3600 -- 'bash tools/r2_profile.sh'
set -x
O=gpurun_out/r2p; mkdir -p $O
NCU="timeout 900 ncu --clock-control none"
# launch list of the exact default bench command (cold cache, serialised)
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/launches_cfg2.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/launches_cfg2.log 2>&1
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/launches_cfg2_hbm.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --slow-tier device > $O/launches_cfg2_hbm.log 2>&1
$NCU --metrics gpu__time_duration.sum,launch__grid_size --csv --log-file $O/launches_ls_hbm.csv \
  python bench.py --layer-sequential --slow-tier device --steps 2 --warmup 3 --no-cpu-baseline \
  > $O/launches_ls_hbm.log 2>&1
# the PCIe-streaming slow kernel (headline), one launch of the cfg2 bench step
$NCU --set full --import-source on -k regex:'slow_attn_kernel' -s 4 -c 1 -f -o $O/slow_cfg2 \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/slow_cfg2.log 2>&1
# the HBM-resident tensor-core slow kernel, cfg2 with --slow-tier device
$NCU --set full --import-source on -k regex:'slow_attn_tc_kernel' -s 4 -c 1 -f -o $O/slowtc_cfg2 \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --slow-tier device > $O/slowtc_cfg2.log 2>&1
# one layer of layer-sequential cfg2 (S = 8): fused selection, fast tier, combine
$NCU --set full --import-source on -k regex:'select_fused|fast_attn_tc|combine_kernel' -s 6 -c 3 -f \
  -o $O/layer_kernels python tools/hbm_step.py 8 131072 3 4 > $O/layer_kernels.log 2>&1
# the speculative record stream and its combine (opt-in), same layer
TTKV_SPEC=1 $NCU --set full --import-source on -k regex:'spec' -s 4 -c 2 -f -o $O/spec_kernels \
  python tools/hbm_step.py 8 131072 3 4 > $O/spec_kernels.log 2>&1
# sanitizer
for t in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $t python tools/sanitize_subset.py > $O/sanitizer_$t.txt 2>&1
  echo "rc=$?" >> $O/sanitizer_$t.txt
done
echo done
