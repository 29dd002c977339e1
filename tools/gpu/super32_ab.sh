# L = 32 super-block GEMM: quadrant ownership (default) vs one warp per block (SPG_SUPER32_QUAD=0); gemm paths must stay bitwise
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_distributed_panels.py tests/test_gpu_bstream.py -x -q > gpurun_out/super32_tests.log 2>&1; echo rc=$? >> gpurun_out/super32_tests.log
for d in 1e-8 1e-6 1e-4; do
  timeout 300 python tools/profile_leaf.py 32 $d >> gpurun_out/super32_quad.log 2>&1
  SPG_SUPER32_QUAD=0 timeout 300 python tools/profile_leaf.py 32 $d >> gpurun_out/super32_block.log 2>&1
done
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:leaf_gemm_super32 -c 1 -o gpurun_out/super32q -f python tools/profile_leaf.py 32 1e-4 > gpurun_out/super32q_ncu.log 2>&1
