mkdir -p gpurun_out
for ch in 8 16 32 64 128 256; do
  TTKV_SLOW_CH=$ch timeout 300 python tools/hbm_step.py 256 131072 6 4 2>&1 | sed "s/^/CH=$ch /"
done
for ch in 8 18 32 64; do
  TTKV_SLOW_CH=$ch timeout 300 python tools/hbm_step.py 8 131072 20 4 2>&1 | sed "s/^/S8 CH=$ch /"
done
