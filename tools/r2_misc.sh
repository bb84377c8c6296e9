O=gpurun_out/r2q; mkdir -p $O
timeout 300 compute-sanitizer --tool racecheck ./build/racecheck_control > $O/racecheck_control.txt 2>&1; echo "rc=$?" >> $O/racecheck_control.txt
./build/racecheck_control >> $O/racecheck_control.txt 2>&1
timeout 600 ./build/decode_cli 256 4 131072 10 0 > $O/decode_cli_host.txt 2>&1
timeout 600 ./build/decode_cli 256 4 131072 50 1 > $O/decode_cli_hbm.txt 2>&1
