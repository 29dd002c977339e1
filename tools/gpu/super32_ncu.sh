# L = 32 super-block GEMM at 27 % / 55 % skipped: timing, then a full ncu capture at 55 %
set -x
timeout 300 python tools/profile_leaf.py 32 1e-6 > gpurun_out/super32_time.log 2>&1
timeout 300 python tools/profile_leaf.py 32 1e-4 >> gpurun_out/super32_time.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:leaf_gemm_super32 -c 1 -o gpurun_out/super32 -f python tools/profile_leaf.py 32 1e-4 > gpurun_out/super32_ncu.log 2>&1
