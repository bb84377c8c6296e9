mkdir -p gpurun_out
NCU="ncu --clock-control none"
$NCU --set full --import-source on -k regex:'slow_attn_tc' -s 1 -c 1 -f -o gpurun_out/tc_cfg2 python tools/hbm_step.py 256 131072 2 4 > gpurun_out/tc_cfg2.log 2>&1
