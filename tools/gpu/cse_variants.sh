# sweep variants on cfg2: parity tests (default path, then the list path),
# host-timed sweeps per variant, ncu durations of every sweep kernel
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_sharding.py tests/test_gpu_reference_cases.py -x -q -m gpu > gpurun_out/t_cse.log 2>&1; echo rc=$? >> gpurun_out/t_cse.log
SPG_CSE_LISTS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/t_cse_lists.log 2>&1; echo rc=$? >> gpurun_out/t_cse_lists.log
for cfg in "SPG_CSE=6" "SPG_CSE=8 SPG_CSE_LISTS=1" "SPG_CSE=8"; do
  tag=$(echo $cfg | tr ' =' '__')
  env $cfg python tools/cse_probe.py 32 8 > gpurun_out/probe_$tag.txt 2>&1
  env $cfg timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv python tools/cse_probe.py 32 2 > gpurun_out/ncu_$tag.csv 2>&1
done
