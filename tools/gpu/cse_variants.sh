# sweep variants on cfg2: parity tests (default path, then the list path and
# without the level s-1 fold), host-timed sweeps per variant and grid size
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_sharding.py tests/test_gpu_reference_cases.py tests/test_distributed_panels.py -x -q -m gpu > gpurun_out/t_cse.log 2>&1; echo rc=$? >> gpurun_out/t_cse.log
SPG_CSE_LISTS=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_sharding.py -x -q -m gpu > gpurun_out/t_cse_lists.log 2>&1; echo rc=$? >> gpurun_out/t_cse_lists.log
SPG_CSE_FOLD=2 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_sharding.py -x -q -m gpu > gpurun_out/t_cse_fold.log 2>&1; echo rc=$? >> gpurun_out/t_cse_fold.log; SPG_CSE_FOLD=2 SPG_CSE_LISTS=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_sharding.py -x -q -m gpu >> gpurun_out/t_cse_fold.log 2>&1; echo rc=$? >> gpurun_out/t_cse_fold.log
for nt in ${NTS:-32 64 128}; do
for cfg in ${CFGS:-"SPG_CSE=8 SPG_CSE_LISTS=1" "SPG_CSE=8"}; do
  tag=$(echo $cfg | tr ' =' '__')_$nt
  env $cfg python tools/cse_probe.py $nt 6 > gpurun_out/probe_$tag.txt 2>&1
done; done
