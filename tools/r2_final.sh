#!/usr/bin/env bash
# One B200, end of round 2: the sweep, then the profiles, then the native
# drivers and the host-issue probe (gpurun_out/r2, r2p, r2q).
#   gpurun --timeout 7000 -- 'bash tools/r2_final.sh'
bash tools/r2_sweep.sh
bash tools/r2_misc.sh
O=gpurun_out/r2q; mkdir -p $O
./build/host_issue_probe 32 1 32768 1 > $O/host_issue_cfg1_hbm.txt 2>&1
TTKV_GRAPH=0 ./build/host_issue_probe 32 1 32768 1 > $O/host_issue_cfg1_hbm_nograph.txt 2>&1
./build/host_issue_probe 256 4 131072 1 > $O/host_issue_cfg2_hbm.txt 2>&1
bash tools/r2_profile.sh
