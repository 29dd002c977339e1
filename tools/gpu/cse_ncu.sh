# full ncu capture of the sweep tile kernel on cfg2 (variant in $1)
SPG_CSE=$1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cse_tile -c 1 -o gpurun_out/cse_v$1 -f python tools/cse_probe.py 32 1 > gpurun_out/cse_ncu_v$1.log 2>&1
