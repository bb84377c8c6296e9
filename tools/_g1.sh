mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/g1_pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g1_pt.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
for c in cfg1 cfg2 cfg3; do
  timeout 400 python bench.py --workload $c --slow-tier device --no-cpu-baseline 2>>gpurun_out/g1_hbm.err | tail -1 > gpurun_out/g1_hbm_$c.json
done
timeout 400 python bench.py --layer-sequential --slow-tier device --no-cpu-baseline 2>>gpurun_out/g1_hbm.err | tail -1 > gpurun_out/g1_hbm_ls.json
echo done
