#!/usr/bin/env bash
# One B200: the round's measurements in one go (writes gpurun_out/f_*; the
# committed profiles/ files are copied from these).
#   gpurun --timeout 2700 -- 'bash tools/refresh_profiles.sh'
set -x
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/f_pt.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
python bench.py --impl reference > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err
for c in cfg1 cfg2 cfg3; do
  python bench.py --workload $c --slow-tier device --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/f_hbm_$c.json
done
python bench.py --layer-sequential --slow-tier device --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/f_hbm_ls.json
python bench.py --layer-sequential --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/f_host_ls.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_hbm.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --slow-tier device > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
  --log-file gpurun_out/f_launches_ls_hbm.csv \
  python bench.py --layer-sequential --slow-tier device --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:slow_attn_tc -s 2 -c 1 \
  -o gpurun_out/f_slowtc python tools/hbm_step.py 256 131072 3 > /dev/null 2>&1
echo done
